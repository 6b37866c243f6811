// sort.cu -- the library's own radix sort and max-scan (no CUB on the hot path).
//
// Where they are used: the a3 access table ("sort the access table by
// item, then transaction id"; the paper uses thrust), the GPUTx K-set order (sort by
// rank), a7 commit positions (sort by the scheme's order key) and phase B of
// partitioned TPC-C (sort the received requests by item, then global transaction id).
//
// gc_sort: stable LSD radix sort of u64 keys (optionally carrying a u32 value) over a bit
// range, 8-bit digits, three kernels per pass:
//   count   -- one block per 4,096-key tile: per-digit counts of its tile (smem atomics),
//              written digit-major so that one exclusive scan gives every (digit, tile) its
//              output base;
//   scan    -- one block per digit row scans it across the tiles, one warp the 256 row
//              totals (two kernels);
//   scatter -- one block per tile, each warp a contiguous 512-key run in 32-key chunks:
//              a key's rank among equal digits is __match_any_sync + popc in its chunk plus
//              its warp's running count (smem), so the scatter is stable (warp multisplit);
//              the tile is reordered in shared memory first, so each digit's run goes out
//              as consecutive addresses.
// The number of keys may live in device memory (n_dev): grids are sized for the host
// capacity and tiles past n exit, so a caller whose n is known only on the device (the
// phase-B exchange) sorts without a host synchronisation.
//
// gc_scan_max2: inclusive max-scan of two u32 arrays at once (segment starts and last
// writes of the access table), reduce-then-scan in three kernels.
#include <cstdint>

#include <cooperative_groups.h>

#include "internal.h"

namespace cg = cooperative_groups;

namespace gcctb {

typedef unsigned long long u64;
typedef uint32_t u32;

constexpr int SORT_THREADS = 256;
constexpr int SORT_WARPS = SORT_THREADS / 32;
constexpr int SORT_PER = 16;                              // keys per thread
constexpr int SORT_TILE = SORT_THREADS * SORT_PER;        // 4,096 keys per tile
constexpr int SORT_WTILE = 32 * SORT_PER;                 // 512 keys per warp, contiguous

static __device__ __forceinline__ u64 n_of(const u64 *n_dev, u64 n_host) { return n_dev ? *n_dev : n_host; }

// per-tile digit counts, digit-major (counts[d * tiles + t]); tiles past n write zeros
__global__ void __launch_bounds__(SORT_THREADS) sort_count_kernel(const u64 *keys, const u64 *n_dev, u64 n_host,
                                                                   int shift, u32 *counts, u32 tiles) {
    __shared__ u32 h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const u64 n = n_of(n_dev, n_host);
    const u64 base = (u64)blockIdx.x * SORT_TILE;
    if (base < n) {
#pragma unroll
        for (int r = 0; r < SORT_PER; r++) {
            const u64 i = base + (u64)r * SORT_THREADS + threadIdx.x;
            if (i < n) atomicAdd(&h[(keys[i] >> shift) & 0xFF], 1u);
        }
    }
    __syncthreads();
    counts[(u64)threadIdx.x * tiles + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan (digit-major) of the counts of the tiles that hold keys, in two kernels:
// one block per digit row scans that row across the tiles (coalesced, in place) and
// records the row total; then one warp turns the 256 totals into each row's base
// (rowbase[d]).  A key's output position is rowbase[digit] + row offset of its tile + its
// place inside the tile.
__global__ void __launch_bounds__(1024) sort_rowscan_kernel(u32 *counts, u32 tiles, const u64 *n_dev, u64 n_host,
                                                             u32 *rowsum) {
    __shared__ u32 wsum[32];
    const u64 n = n_of(n_dev, n_host);
    const u32 active = (u32)((n + SORT_TILE - 1) / SORT_TILE);
    u32 *row = counts + (u64)blockIdx.x * tiles;
    const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u32 carry = 0;
    for (u32 t0 = 0; t0 < active; t0 += 1024) {
        const u32 t = t0 + threadIdx.x;
        const u32 c = t < active ? row[t] : 0u;
        u32 x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= (u32)o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            u32 v = wsum[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 y = __shfl_up_sync(0xFFFFFFFFu, v, o);
                if (lane >= (u32)o) v += y;
            }
            wsum[lane] = v;   // inclusive over warps
        }
        __syncthreads();
        const u32 before = (warp ? wsum[warp - 1] : 0u) + carry;
        if (t < active) row[t] = before + x - c;   // exclusive within the row
        carry += wsum[31];
        __syncthreads();
    }
    if (threadIdx.x == 0) rowsum[blockIdx.x] = carry;
}

__global__ void sort_rowbase_kernel(u32 *rowsum) {   // one warp: exclusive scan of 256 totals, in place
    const u32 lane = threadIdx.x;
    u32 v[8], acc = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        v[k] = rowsum[lane * 8 + k];
        acc += v[k];
    }
    u32 x = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= (u32)o) x += y;
    }
    u32 run = x - acc;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        rowsum[lane * 8 + k] = run;
        run += v[k];
    }
}

// stable scatter of one tile, staged through shared memory so the global writes are
// coalesced runs per digit: warp w owns keys [w * 512, (w + 1) * 512) of the tile in
// 32-key chunks processed in order.  Phase 1 counts each warp's digits (a chunk's equal
// digits form one __match_any_sync group whose lowest lane adds the group size); phase 2
// scans them into each warp's first slot of each digit inside the tile's digit-sorted
// order; phase 3 places every key there (+ its rank in its group) in shared memory;
// phase 4 writes the tile's keys out in that order, each digit's run at its global base
// (gbase[d], filled by the caller before the first __syncthreads here).
struct ScatterSmem {
    u32 wc[SORT_WARPS][256];
    u32 tstart[256], gbase[256];
    u32 ws[SORT_WARPS];
};
template <bool PAIRS>
__device__ __forceinline__ void scatter_tile(ScatterSmem &S, u64 *sk, u32 *sv, const u64 *keys, const u32 *vals,
                                             u64 *keys_out, u32 *vals_out, u64 n, int shift, u32 tile) {
    const u32 tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const u64 tb = (u64)tile * SORT_TILE;
    const u32 cnt = (u32)(n - tb < SORT_TILE ? n - tb : SORT_TILE);
    const u64 w0 = tb + (u64)warp * SORT_WTILE;
#pragma unroll
    for (int w = 0; w < SORT_WARPS; w++) S.wc[w][tid] = 0;
    __syncthreads();
    u64 k[SORT_PER];
    u32 dg[SORT_PER];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int c = 0; c < SORT_PER; c++) {
        const u64 i = w0 + (u64)c * 32 + lane;
        const bool ok = i < n;
        k[c] = ok ? keys[i] : 0ull;
        dg[c] = ok ? (u32)((k[c] >> shift) & 0xFF) : 256u;
    }
#pragma unroll
    for (int c = 0; c < SORT_PER; c++) {
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, dg[c]);
        if (dg[c] < 256u && (peers & lt) == 0) S.wc[warp][dg[c]] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    {   // thread `tid` owns digit `tid`: its count in the tile, and the warps' prefixes
        u32 pre[SORT_WARPS], tot = 0;
#pragma unroll
        for (int w = 0; w < SORT_WARPS; w++) {
            pre[w] = tot;
            tot += S.wc[w][tid];
        }
        // exclusive scan of the 256 digit totals across the block (digit = thread)
        u32 x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= (u32)o) x += y;
        }
        if (lane == 31) S.ws[warp] = x;
        __syncthreads();
        u32 before = 0;
        for (u32 w = 0; w < warp; w++) before += S.ws[w];
        const u32 start = before + x - tot;   // first slot of digit `tid` in the tile's order
        S.tstart[tid] = start;
#pragma unroll
        for (int w = 0; w < SORT_WARPS; w++) S.wc[w][tid] = start + pre[w];
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < SORT_PER; c++) {
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, dg[c]);
        if (dg[c] < 256u) {
            const u32 slot = S.wc[warp][dg[c]] + __popc(peers & lt);
            sk[slot] = k[c];
            if (PAIRS) sv[slot] = vals[w0 + (u64)c * 32 + lane];
        }
        __syncwarp();
        if (dg[c] < 256u && (peers & lt) == 0) S.wc[warp][dg[c]] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (u32 i = tid; i < cnt; i += SORT_THREADS) {   // consecutive slots of a digit: consecutive addresses
        const u64 key = sk[i];
        const u32 d = (u32)((key >> shift) & 0xFF);
        const u32 pos = S.gbase[d] + (i - S.tstart[d]);
        keys_out[pos] = key;
        if (PAIRS) vals_out[pos] = sv[i];
    }
}

template <bool PAIRS>
__global__ void __launch_bounds__(SORT_THREADS) sort_scatter_kernel(const u64 *keys, const u32 *vals, u64 *keys_out,
                                                                     u32 *vals_out, const u64 *n_dev, u64 n_host,
                                                                     int shift, const u32 *offs, const u32 *rowbase,
                                                                     u32 tiles) {
    __shared__ ScatterSmem S;
    extern __shared__ __align__(16) unsigned char sort_smem[];
    u64 *sk = reinterpret_cast<u64 *>(sort_smem);
    u32 *sv = reinterpret_cast<u32 *>(sort_smem + SORT_TILE * sizeof(u64));
    const u64 n = n_of(n_dev, n_host);
    if ((u64)blockIdx.x * SORT_TILE >= n) return;   // uniform
    S.gbase[threadIdx.x] = rowbase[threadIdx.x] + offs[(u64)threadIdx.x * tiles + blockIdx.x];
    scatter_tile<PAIRS>(S, sk, sv, keys, vals, keys_out, vals_out, n, shift, blockIdx.x);
}

// Small sorts (a7 commit positions, the GPUTx rank order: n <= GC_COOP_MAX_TILES tiles)
// in ONE cooperative launch, one block per tile: per pass the tile counts, a grid barrier,
// every block derives its tile's digit bases from all tiles' counts (a 256 x tiles scan
// it repeats for itself), the stable scatter above, a grid barrier.  Passes above the
// largest key's top byte are skipped on the device (the keys' range -- e.g. TicToc's
// commit timestamps -- is known only there); if the skipped passes leave the keys in the
// other buffer than the host-side ping-pong expects, a final copy puts them there.
#ifndef GC_COOP_MAX_TILES
#define GC_COOP_MAX_TILES 128u
#endif
template <bool PAIRS>
__global__ void __launch_bounds__(SORT_THREADS) sort_coop_kernel(u64 *ka, u32 *va, u64 *kb, u32 *vb, u64 n, int lo_bit,
                                                                  int hi_bit, u32 *counts, u64 *bmax) {
    __shared__ ScatterSmem S;
    __shared__ u64 smax[SORT_WARPS];
    __shared__ u32 dtot[256];
    extern __shared__ __align__(16) unsigned char sort_smem[];
    u64 *sk = reinterpret_cast<u64 *>(sort_smem);
    u32 *sv = reinterpret_cast<u32 *>(sort_smem + SORT_TILE * sizeof(u64));
    cg::grid_group grid = cg::this_grid();
    const u32 tiles = gridDim.x, t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const u64 tb = (u64)t * SORT_TILE;
    // largest key (grid-wide): each block publishes its tile's maximum
    {
        u64 m = 0;
        for (u64 i = tb + tid; i < n && i < tb + SORT_TILE; i += SORT_THREADS) m = max(m, ka[i]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, (u64)__shfl_xor_sync(0xFFFFFFFFu, m, o));
        if (lane == 0) smax[warp] = m;
        __syncthreads();
        if (tid == 0) {
            u64 x = 0;
            for (int w = 0; w < SORT_WARPS; w++) x = max(x, smax[w]);
            bmax[t] = x;
        }
    }
    grid.sync();
    u64 kmax = 0;
    for (u32 b = 0; b < tiles; b++) kmax = max(kmax, bmax[b]);   // (same value in every block)
    u64 *src = ka, *dst = kb;
    u32 *vs = va, *vd = vb;
    int total = 0, done = 0;
    for (int sh = lo_bit; sh < hi_bit; sh += 8) total++;
    for (int sh = lo_bit; sh < hi_bit; sh += 8) {
        if (sh >= 64 || (kmax >> sh) == 0) break;   // every remaining digit is 0: identity
        // 1. tile digit counts
        if (tid < 256) dtot[tid] = 0;
        __syncthreads();
        for (u64 i = tb + tid; i < n && i < tb + SORT_TILE; i += SORT_THREADS) atomicAdd(&dtot[(src[i] >> sh) & 0xFF], 1u);
        __syncthreads();
        counts[(u64)tid * tiles + t] = dtot[tid];
        grid.sync();
        // 2. this tile's base of each digit: all tiles' counts of smaller digits, plus the
        // counts of this digit in the tiles before
        {
            u32 tot = 0, pre = 0;
            const u32 *row = counts + (u64)tid * tiles;
            for (u32 b = 0; b < tiles; b++) {
                const u32 c = row[b];
                tot += c;
                if (b < t) pre += c;
            }
            u32 x = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 y = __shfl_up_sync(0xFFFFFFFFu, x, o);
                if (lane >= (u32)o) x += y;
            }
            __syncthreads();   // S.ws is reused by the scatter
            if (lane == 31) S.ws[warp] = x;
            __syncthreads();
            u32 before = 0;
            for (u32 w = 0; w < warp; w++) before += S.ws[w];
            S.gbase[tid] = before + x - tot + pre;
        }
        // 3. stable scatter
        if (tb < n) scatter_tile<PAIRS>(S, sk, sv, src, vs, dst, vd, n, sh, t);
        grid.sync();
        u64 *tk = src; src = dst; dst = tk;
        u32 *tv = vs; vs = vd; vd = tv;
        done++;
    }
    if ((total - done) & 1) {   // the host expects the result after `total` swaps
        for (u64 i = (u64)t * SORT_THREADS + tid; i < n; i += (u64)tiles * SORT_THREADS) {
            dst[i] = src[i];
            if (PAIRS) vd[i] = vs[i];
        }
    }
}

size_t gc_sort_temp_bytes(uint64_t cap) {
    const u64 tiles = (cap + SORT_TILE - 1) / SORT_TILE;
    return (size_t)(256 * (tiles ? tiles : 1) + 256) * sizeof(u32) + 256;
}
constexpr size_t SORT_SMEM = (size_t)SORT_TILE * (sizeof(u64) + sizeof(u32));   // 48 KB staging

cudaError_t gc_sort(u64 *keys, u32 *vals, u64 *keys_alt, u32 *vals_alt, uint64_t cap, const u64 *n_dev,
                    int lo_bit, int hi_bit, void *temp, size_t temp_bytes, cudaStream_t s, u64 **keys_out,
                    u32 **vals_out) {
    u64 *ka = keys, *kb = keys_alt;
    u32 *va = vals, *vb = vals_alt;
    *keys_out = ka;
    if (vals_out) *vals_out = va;
    if (cap == 0 || hi_bit <= lo_bit) return cudaSuccess;
    const u64 tiles = (cap + SORT_TILE - 1) / SORT_TILE;
    if (gc_sort_temp_bytes(cap) > temp_bytes || tiles > 0xFFFFFFFFull) return cudaErrorInvalidValue;
    u32 *counts = reinterpret_cast<u32 *>(temp);
    u32 *rowsum = counts + 256 * tiles;
    // (per call: the attribute belongs to the current device's context)
    cudaError_t ea = cudaFuncSetAttribute(va ? (const void *)sort_scatter_kernel<true> : (const void *)sort_scatter_kernel<false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SORT_SMEM);
    if (ea) return ea;
    if (!n_dev && tiles <= GC_COOP_MAX_TILES) {   // one cooperative launch (see sort_coop_kernel)
        const void *f = va ? (const void *)sort_coop_kernel<true> : (const void *)sort_coop_kernel<false>;
        cudaError_t ec = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SORT_SMEM);
        if (ec) return ec;
        u64 n = cap;
        int lo = lo_bit, hi = hi_bit;
        u64 *bmax = reinterpret_cast<u64 *>(rowsum);
        void *args[] = {&ka, &va, &kb, &vb, &n, &lo, &hi, &counts, &bmax};
        ec = cudaLaunchCooperativeKernel(f, dim3((unsigned)tiles), dim3(SORT_THREADS), args, SORT_SMEM, s);
        if (ec) return ec;
        int passes = 0;
        for (int sh = lo_bit; sh < hi_bit; sh += 8) passes++;
        if (passes & 1) {
            *keys_out = kb;
            if (vals_out) *vals_out = vb;
        }
        return cudaSuccess;
    }
    for (int sh = lo_bit; sh < hi_bit; sh += 8) {
        sort_count_kernel<<<(unsigned)tiles, SORT_THREADS, 0, s>>>(ka, n_dev, cap, sh, counts, (u32)tiles);
        sort_rowscan_kernel<<<256, 1024, 0, s>>>(counts, (u32)tiles, n_dev, cap, rowsum);
        sort_rowbase_kernel<<<1, 32, 0, s>>>(rowsum);
        if (va)
            sort_scatter_kernel<true><<<(unsigned)tiles, SORT_THREADS, SORT_SMEM, s>>>(ka, va, kb, vb, n_dev, cap, sh,
                                                                                     counts, rowsum, (u32)tiles);
        else
            sort_scatter_kernel<false><<<(unsigned)tiles, SORT_THREADS, SORT_SMEM, s>>>(ka, nullptr, kb, nullptr, n_dev,
                                                                                      cap, sh, counts, rowsum, (u32)tiles);
        u64 *tk = ka; ka = kb; kb = tk;
        u32 *tv = va; va = vb; vb = tv;
    }
    *keys_out = ka;
    if (vals_out) *vals_out = va;
    return cudaGetLastError();
}

// ------------------------------------------------------------------ max-scan of two arrays
constexpr int SCAN_THREADS = 256, SCAN_PER = 8, SCAN_TILE = SCAN_THREADS * SCAN_PER;

__global__ void __launch_bounds__(SCAN_THREADS) scan_reduce_kernel(const u32 *a, const u32 *b, u64 n, u32 *bm) {
    __shared__ u32 ra[SCAN_THREADS / 32], rb[SCAN_THREADS / 32];
    const u64 t0 = (u64)blockIdx.x * SCAN_TILE;
    u32 ma = 0, mb = 0;
    for (int r = 0; r < SCAN_PER; r++) {
        const u64 i = t0 + (u64)r * SCAN_THREADS + threadIdx.x;
        if (i < n) {
            ma = max(ma, a[i]);
            mb = max(mb, b[i]);
        }
    }
    ma = __reduce_max_sync(0xFFFFFFFFu, ma);
    mb = __reduce_max_sync(0xFFFFFFFFu, mb);
    if ((threadIdx.x & 31) == 0) {
        ra[threadIdx.x >> 5] = ma;
        rb[threadIdx.x >> 5] = mb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < SCAN_THREADS / 32; w++) {
            ma = max(ma, ra[w]);
            mb = max(mb, rb[w]);
        }
        bm[2 * blockIdx.x] = ra[0] > ma ? ra[0] : ma;
        bm[2 * blockIdx.x + 1] = rb[0] > mb ? rb[0] : mb;
    }
}

// exclusive max-scan of the block maxima (pairs), one block of 1,024 threads, each a
// contiguous chunk (independent loads), then a scan of the chunk maxima
__global__ void __launch_bounds__(1024) scan_blocks_kernel(u32 *bm, u64 tiles) {
    __shared__ u32 pa[1024], pb[1024];
    const u64 per = (tiles + 1023) / 1024, lo = (u64)threadIdx.x * per, hi = lo + per < tiles ? lo + per : tiles;
    u32 ma = 0, mb = 0;
    for (u64 t = lo; t < hi; t++) {
        ma = max(ma, bm[2 * t]);
        mb = max(mb, bm[2 * t + 1]);
    }
    pa[threadIdx.x] = ma;
    pb[threadIdx.x] = mb;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const u32 xa = threadIdx.x >= (unsigned)o ? pa[threadIdx.x - o] : 0u;
        const u32 xb = threadIdx.x >= (unsigned)o ? pb[threadIdx.x - o] : 0u;
        __syncthreads();
        pa[threadIdx.x] = max(pa[threadIdx.x], xa);
        pb[threadIdx.x] = max(pb[threadIdx.x], xb);
        __syncthreads();
    }
    u32 ca = threadIdx.x ? pa[threadIdx.x - 1] : 0u, cb = threadIdx.x ? pb[threadIdx.x - 1] : 0u;
    for (u64 t = lo; t < hi; t++) {
        const u32 xa = bm[2 * t], xb = bm[2 * t + 1];
        bm[2 * t] = ca;
        bm[2 * t + 1] = cb;
        ca = max(ca, xa);
        cb = max(cb, xb);
    }
}

// block-local inclusive max-scan with the carry of the tiles before; out may alias in
__global__ void __launch_bounds__(SCAN_THREADS) scan_apply_kernel(const u32 *a, const u32 *b, u64 n, const u32 *bm,
                                                                   u32 *oa, u32 *ob) {
    __shared__ u32 wa[SCAN_THREADS / 32], wb[SCAN_THREADS / 32];
    const u64 t0 = (u64)blockIdx.x * SCAN_TILE;
    u32 ca = bm[2 * blockIdx.x], cb = bm[2 * blockIdx.x + 1];
    const u32 lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int r = 0; r < SCAN_PER; r++) {
        const u64 i = t0 + (u64)r * SCAN_THREADS + threadIdx.x;
        u32 xa = i < n ? a[i] : 0u, xb = i < n ? b[i] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {   // warp inclusive max-scan
            const u32 ya = __shfl_up_sync(0xFFFFFFFFu, xa, o), yb = __shfl_up_sync(0xFFFFFFFFu, xb, o);
            if (lane >= (u32)o) {
                xa = max(xa, ya);
                xb = max(xb, yb);
            }
        }
        if (lane == 31) {
            wa[warp] = xa;
            wb[warp] = xb;
        }
        __syncthreads();
        u32 pa = ca, pb = cb;
        for (u32 w = 0; w < warp; w++) {
            pa = max(pa, wa[w]);
            pb = max(pb, wb[w]);
        }
        if (i < n) {
            oa[i] = max(pa, xa);
            ob[i] = max(pb, xb);
        }
        for (u32 w = 0; w < SCAN_THREADS / 32; w++) {   // carry into the next round
            ca = max(ca, wa[w]);
            cb = max(cb, wb[w]);
        }
        __syncthreads();
    }
}

size_t gc_scan_temp_bytes(uint64_t n) { return (size_t)(2 * ((n + SCAN_TILE - 1) / SCAN_TILE + 1)) * sizeof(u32); }

cudaError_t gc_scan_max2(const u32 *a, const u32 *b, u32 *oa, u32 *ob, uint64_t n, void *temp, size_t temp_bytes,
                         cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (gc_scan_temp_bytes(n) > temp_bytes) return cudaErrorInvalidValue;
    const u64 tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    u32 *bm = reinterpret_cast<u32 *>(temp);
    scan_reduce_kernel<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(a, b, n, bm);
    scan_blocks_kernel<<<1, 1024, 0, s>>>(bm, tiles);
    scan_apply_kernel<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(a, b, n, bm, oa, ob);
    return cudaGetLastError();
}


// Lazy module loading (the CUDA 12 default) may synchronise the context the first time a
// kernel is launched -- which deadlocks once kernels of one process wait on each other
// across streams (CC_FLAG_PART_P2P between the dbs of one process).  cc_part_connect*
// loads every kernel up front.
template <class F>
static void preload1(F f) {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, f);
}
void preload_sort_kernels() {
    preload1(sort_count_kernel); preload1(sort_rowscan_kernel); preload1(sort_rowbase_kernel);
    preload1(sort_scatter_kernel<true>);
    preload1(sort_scatter_kernel<false>); preload1(sort_coop_kernel<true>); preload1(sort_coop_kernel<false>); preload1(scan_reduce_kernel); preload1(scan_blocks_kernel);
    preload1(scan_apply_kernel);
}
}  // namespace gcctb
