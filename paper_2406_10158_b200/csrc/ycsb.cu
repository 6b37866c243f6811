// ycsb.cu -- YCSB workload on the device: table initialiser, primary-key index,
// a1 batch generator, the workload policy the executor is instantiated with, and the
// a3 access gather for the deterministic schemes.
//
// YCSB: 2^20*10 rows, 16 single-tuple accesses per transaction,
// Zipfian keys (theta), write fraction W.  Row = 16 x u64 (128 B, one L2 line pair
// of sectors; reading Z11).  Op semantics (Z11): out = fp(row) = sum_j rotl(r[j], j);
// a write also sets r[f] = r[f]*0x9E3779B97F4A7C15 + ((gid<<4)|i) + 1 and r[15] += 1.
#include <cstdio>
#include <cstdlib>

#include "exec.cuh"

namespace gcctb {

struct YcsbWL {
    static constexpr int MAXK = 16;
    static constexpr int ROW_WORDS = 16;
    static constexpr bool STAGE_TILE_LANE = false;   // tile mode: the 40 B entry stays in registers
    using Params = YcsbParams;
    // One access of a transaction and its private workspace ("private
    // workspace"): the value read and the buffered new values of a write.
    struct Lane {
        u32 rec;
        bool act, w;
        uint8_t field;
        u64 out, nf, n15;
        u64 cv;   // thread mode: control word seen (OCC snapshot / lock-time word, TO / MVCC saved word)
    };

    // Index lookup: lower bound of key in the sorted key array, returns
    // the row or ~0 for KeyNotFound.  Dense key range: direct addressing
    // (f-3); else descend the cache-line tree (one 128 B node of 16 keys per level:
    // count keys < key); CC_FLAG_INDEX_BINARY: the paper's branch-free binary search.
    static GC_DEV bool is_dense(int mode) { return mode == IDX_DENSE || mode == IDX_DENSE_ID; }
    static GC_DEV u64 lookup(const YcsbParams &y, u64 key) {
        if (is_dense(y.mode)) return dense_lookup(y, key);
        if (y.mode == IDX_TREE) return tree_lookup(y, key);
        if (y.mode == IDX_EYTZ) return eytz_lookup(y, key);
        return binary_lookup(y, key);
    }
    // Eytzinger layout (f-3): node i (1-based) has children 2i, 2i+1; descend branch-free
    // (i = 2i + [key > node]) to below the leaves, then strip the trailing right turns:
    // the remaining node is the lower bound (0: every key is smaller).  The top levels are
    // shared by every lookup and stay cached; one dependent load per level below them.
    static GC_DEV u64 eytz_lookup(const YcsbParams &y, u64 key) {
        u64 i = 1;
        while (i <= y.eytz_n) i = 2 * i + (__ldg(y.eytz_keys + i) < key);
        i >>= __ffsll((long long)~i);
        if (i == 0 || __ldg(y.eytz_keys + i) != key) return ~0ull;
        return __ldg(y.eytz_rows + i);
    }
    static GC_DEV u64 dense_lookup(const YcsbParams &y, u64 key) {
        const u64 pos = key - y.idx_k0;   // wraps above idx_n for key < k0
        if (pos >= y.idx_n) return ~0ull;
        return y.mode == IDX_DENSE_ID ? pos : __ldg(y.idx_rows + pos);
    }
    static GC_DEV u64 tree_lookup(const YcsbParams &y, u64 key) {
        u64 node = 0;
        for (int l = y.tree.n_levels - 1; l >= 0; l--) {
            const u64 *nd = y.tree.lv[l] + node * 16;
            u32 j = 0;
#pragma unroll
            for (int w = 0; w < 8; w++) {
                u64 a, b;
                asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(nd + 2 * w));
                j += (a < key) + (b < key);
            }
            if (j == 16) return ~0ull;   // key above every key
            node = node * 16 + j;
        }
        const u64 pos = node;
        if (pos >= y.idx_n || __ldg(y.idx_keys + pos) != key) return ~0ull;
        return __ldg(y.idx_rows + pos);
    }
    static GC_DEV u64 binary_lookup(const YcsbParams &y, u64 key) {
        const u64 *b = y.idx_keys;
        u64 n = y.idx_n;
        while (n > 1) {
            const u64 half = n >> 1;
            b = (__ldg(b + half) < key) ? b + half : b;
            n -= half;
        }
        u64 pos = (u64)(b - y.idx_keys);
        u64 kv = __ldg(b);
        if (kv < key) {
            pos++;
            kv = pos < y.idx_n ? __ldg(y.idx_keys + pos) : ~0ull;
        }
        return (pos >= y.idx_n || kv != key) ? ~0ull : __ldg(y.idx_rows + pos);
    }

    // Thread mode: resolve every access up front (read/write sets are predetermined,
    // PAPER.md:446) into the staged lanes; the K searches of the tree / binary index run
    // in lockstep for memory-level parallelism (u32 keys and positions: 2 x 16 registers).
    template <class LA>
    static GC_DEV u32 load_all(const ExecParams &p, const YcsbParams &y, u32 gid, LA L) {
        const u64 base = (u64)gid * p.K;
        const u32 K = p.K;
        for (u32 i = 0; i < K; i++) {
            Lane &Li = L[i];
            const uint8_t op = y.ops[base + i];
            Li.act = true;
            Li.field = op & 0x0F;
            Li.w = op >> 7;
            if (p.acc_rec) Li.rec = p.acc_rec[base + i];   // resolved by a3
        }
        if (p.acc_rec) return K;
        bool ok = true;
        if (is_dense(y.mode) || y.mode == IDX_EYTZ) {
            for (u32 i = 0; i < K; i++) {
                const u64 key = y.keys[base + i];
                const u64 r = is_dense(y.mode) ? dense_lookup(y, key) : eytz_lookup(y, key);
                ok &= r != ~0ull;
                L[i].rec = (u32)r;
            }
        } else if (y.mode == IDX_TREE) {
            // descents in lockstep, TG keys at a time (TG x 8 independent 16 B loads per level
            // in flight; all 16 at once spilled ~700 B per thread)
            constexpr int TG = 2;
            for (u32 i0 = 0; i0 < K; i0 += TG) {
                u32 key[TG], node[TG];
#pragma unroll
                for (int g = 0; g < TG; g++) {
                    key[g] = i0 + g < K ? y.keys[base + i0 + g] : 0u;
                    node[g] = 0;
                }
                for (int l = y.tree.n_levels - 1; l >= 0; l--) {
                    const u64 *lv = y.tree.lv[l];
#pragma unroll
                    for (int g = 0; g < TG; g++) {
                        const u64 *nd = lv + (u64)node[g] * 16;
                        u32 j = 0;
#pragma unroll
                        for (int w = 0; w < 8; w++) {
                            u64 a, b;
                            asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(nd + 2 * w));
                            j += (a < key[g]) + (b < key[g]);
                        }
                        if (i0 + g < K) ok &= j < 16;
                        node[g] = node[g] * 16 + (j < 16 ? j : 0);
                    }
                }
#pragma unroll
                for (int g = 0; g < TG; g++)
                    if (i0 + g < K) {
                        if (node[g] >= y.idx_n || __ldg(y.idx_keys + node[g]) != key[g]) ok = false;
                        else L[i0 + g].rec = (u32)__ldg(y.idx_rows + node[g]);
                    }
            }
        } else {   // the paper's binary search, lower bound; BG searches in lockstep
            constexpr int BG = 4;
            for (u32 i0 = 0; i0 < K; i0 += BG) {
                u32 key[BG], lo[BG];
#pragma unroll
                for (int g = 0; g < BG; g++) {
                    key[g] = i0 + g < K ? y.keys[base + i0 + g] : 0u;
                    lo[g] = 0;
                }
                u64 n = y.idx_n;
                while (n > 1) {
                    const u64 half = n >> 1;
#pragma unroll
                    for (int g = 0; g < BG; g++)
                        lo[g] = (__ldg(y.idx_keys + lo[g] + half) < key[g]) ? lo[g] + (u32)half : lo[g];
                    n -= half;
                }
#pragma unroll
                for (int g = 0; g < BG; g++)
                    if (i0 + g < K) {
                        u64 pos = lo[g];
                        u64 kv = __ldg(y.idx_keys + pos);
                        if (kv < key[g]) {
                            pos++;
                            kv = pos < y.idx_n ? __ldg(y.idx_keys + pos) : ~0ull;
                        }
                        if (pos >= y.idx_n || kv != key[g]) ok = false;
                        else L[i0 + g].rec = (u32)__ldg(y.idx_rows + pos);
                    }
            }
        }
        if (!ok) return 0xFFFFFFFFu;
        for (u32 i = 0; i < K; i++) prefetch_access(p, y, L[i]);
        return K;
    }

    // Tile mode: lane i resolves access i.
    static GC_DEV bool load_lane(const ExecParams &p, const YcsbParams &y, u32 gid, u32 i, Lane &L) {
        L.act = i < p.K;
        if (!L.act) return true;
        const u64 a = (u64)gid * p.K + i;
        const uint8_t op = y.ops[a];
        L.field = op & 0x0F;
        L.w = op >> 7;
        if (p.acc_rec) {
            L.rec = p.acc_rec[a];
            prefetch_access(p, y, L);
            return true;
        }
        const u64 r = lookup(y, y.keys[a]);
        L.rec = (u32)r;
        if (r != ~0ull) prefetch_access(p, y, L);
        return r != ~0ull;
    }

    // bring the row (both 64 B halves) and the CC word into L2 while the scheme's ordered
    // accesses to the word are still pending
    static GC_DEV void prefetch_access(const ExecParams &p, const YcsbParams &y, const Lane &L) {
        const u64 *rw = y.rows + (u64)L.rec * 16u;
        prefetch_l2(rw);
        prefetch_l2(rw + 8);
        prefetch_l2(p.scheme == CC_MVCC ? mvcc_lo(p, L.rec) : cw(p, L.rec));
    }

    static GC_DEV u64 *row(const YcsbParams &y, const Lane &L) { return y.rows + (u64)L.rec * 16u; }

    // CC_FLAG_WARM: wait until the prefetched row and control word are in L2 -- one load
    // per 32 B sector, folded into a value the caller consumes before its first CC step
    static GC_DEV u64 warm(const ExecParams &p, const YcsbParams &y, const Lane &L) {
        const u64 *rw = y.rows + (u64)L.rec * 16u;
        const u64 *w = p.scheme == CC_MVCC ? mvcc_lo(p, L.rec) : cw(p, L.rec);
        return ld_cg(rw) ^ ld_cg(rw + 4) ^ ld_cg(rw + 8) ^ ld_cg(rw + 12) ^ ld_relaxed(w);
    }

    // op semantics (Z11): out = fp(row); a write buffers r[f]*G + ((gid<<4)|i) + 1 and
    // r[15] + 1 (installed at commit by the scheme).
    static GC_DEV void read(const YcsbParams &, Lane &L, u32 gid, u32 i, const u64 *src) {
        u64 r[16];
#pragma unroll
        for (int j = 0; j < 4; j++) ld_cg_v4(src + 4 * j, r[4 * j], r[4 * j + 1], r[4 * j + 2], r[4 * j + 3]);
        u64 fp = 0, rf = 0;
#pragma unroll
        for (int j = 0; j < 16; j++) {
            fp += rotl64(r[j], j);
            rf = (j == (int)L.field) ? r[j] : rf;
        }
        L.out = fp;
        if (L.w) {
            L.nf = rf * 0x9E3779B97F4A7C15ull + ((((u64)gid) << 4) | (u64)i) + 1ull;
            L.n15 = r[15] + 1ull;
        }
    }

    static GC_DEV void install(const YcsbParams &, const Lane &L, u64 *dst) {
        st_cg(dst + L.field, L.nf);
        st_cg(dst + 15, L.n15);
    }

    static GC_DEV void copy_row(const Lane &, const u64 *src, u64 *dst) {
#pragma unroll
        for (int j = 0; j < 4; j += 2) {   // two 32 B loads in flight (all four spilled)
            u64 a, b, c, d, e, f, g, h;
            ld_cg_v4(src + 4 * j, a, b, c, d);
            ld_cg_v4(src + 4 * j + 4, e, f, g, h);
            st_cg_v4(dst + 4 * j, a, b, c, d);
            st_cg_v4(dst + 4 * j + 4, e, f, g, h);
        }
    }

    template <class LA>
    static GC_DEV void emit_txn(const ExecParams &p, const YcsbParams &, u32 gid, LA L, u32 n) {
        if (!p.read_out) return;
        for (u32 i = 0; i < n; i++) p.read_out[(u64)gid * p.K + i] = L[i].out;
    }
    template <class Tile>
    static GC_DEV void emit_tile(Tile &, const ExecParams &p, const YcsbParams &, u32 gid, const Lane &L, u32 i) {
        if (p.read_out && L.act) p.read_out[(u64)gid * p.K + i] = L.out;
    }
};

// ---------------------------------------------------------------- executor launch
template <int S>
static cudaError_t launch_s(const ExecParams &p, const YcsbParams &y, int grid, int block, size_t smem,
                            cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    auto go = [&](auto kern) {
        if (smem > 32 * 1024) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (getenv("GCCTB_DEBUG_LAUNCH")) {
            cudaFuncAttributes fa{};
            cudaFuncGetAttributes(&fa, kern);
            fprintf(stderr, "launch lanes=%u grid=%d block=%d smem=%zu set=%d static=%zu maxdyn=%d regs=%d maxthr=%d\n",
                    p.lanes, grid, block, smem, (int)e, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes, fa.numRegs,
                    fa.maxThreadsPerBlock);
        }
        if (e == cudaSuccess) kern<<<grid, block, smem, s>>>(p, y);
    };
    switch (p.lanes) {
        case 4: go(exec_tile_kernel<S, YcsbWL, 4>); break;
        case 8: go(exec_tile_kernel<S, YcsbWL, 8>); break;
        case 16: go(exec_tile_kernel<S, YcsbWL, 16>); break;
        case 32: go(exec_tile_kernel<S, YcsbWL, 32>); break;
        default: go(exec_thread_kernel<S, YcsbWL>); break;
    }
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_ycsb_exec(const ExecParams &p, const YcsbParams &y, int grid, int block, size_t smem,
                             cudaStream_t s) {
    switch (p.scheme) {
        case CC_TPL_NW: return launch_s<CC_TPL_NW>(p, y, grid, block, smem, s);
        case CC_TPL_WD: return launch_s<CC_TPL_WD>(p, y, grid, block, smem, s);
        case CC_TO: return launch_s<CC_TO>(p, y, grid, block, smem, s);
        case CC_MVCC: return launch_s<CC_MVCC>(p, y, grid, block, smem, s);
        case CC_SILO: return launch_s<CC_SILO>(p, y, grid, block, smem, s);
        case CC_TICTOC: return launch_s<CC_TICTOC>(p, y, grid, block, smem, s);
        case CC_GPUTX: return launch_s<CC_GPUTX>(p, y, grid, block, smem, s);
        case CC_GACCO: return launch_s<CC_GACCO>(p, y, grid, block, smem, s);
    }
    return cudaErrorInvalidValue;
}

template <class F>
static int occ_of(F f, int block, size_t smem = 0) {
    int nb = 0;
    if (smem > 32 * 1024) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, block, smem);
    return nb;
}

template <int S>
static int occ_s(int lanes, int block, size_t smem) {
    switch (lanes) {
        case 4: return occ_of(exec_tile_kernel<S, YcsbWL, 4>, block, smem);
        case 8: return occ_of(exec_tile_kernel<S, YcsbWL, 8>, block, smem);
        case 16: return occ_of(exec_tile_kernel<S, YcsbWL, 16>, block, smem);
        case 32: return occ_of(exec_tile_kernel<S, YcsbWL, 32>, block, smem);
        default: return occ_of(exec_thread_kernel<S, YcsbWL>, block, smem);
    }
}

size_t ycsb_lane_bytes() { return sizeof(YcsbWL::Lane); }
size_t exec_th_bytes() { return sizeof(Th); }
int ycsb_exec_max_blocks_per_sm(int scheme, int lanes, int block, size_t smem) {
    switch (scheme) {
        case CC_TPL_NW: return occ_s<CC_TPL_NW>(lanes, block, smem);
        case CC_TPL_WD: return occ_s<CC_TPL_WD>(lanes, block, smem);
        case CC_TO: return occ_s<CC_TO>(lanes, block, smem);
        case CC_MVCC: return occ_s<CC_MVCC>(lanes, block, smem);
        case CC_SILO: return occ_s<CC_SILO>(lanes, block, smem);
        case CC_TICTOC: return occ_s<CC_TICTOC>(lanes, block, smem);
        case CC_GPUTX: return occ_s<CC_GPUTX>(lanes, block, smem);
        case CC_GACCO: return occ_s<CC_GACCO>(lanes, block, smem);
    }
    return 0;
}

// ---------------------------------------------------------------- a3 gather
// One thread per transaction: resolve its accesses and emit the access-table sort
// keys (rec << 27) | (gid << 6) | (i << 1) | is_write.
__global__ void ycsb_gather_kernel(ExecParams p, YcsbParams y, uint32_t *acc_rec,
                                   unsigned long long *keys_out) {
    const u64 a = (u64)blockIdx.x * blockDim.x + threadIdx.x;   // one thread per access
    if (a >= (u64)p.n_txn * p.K) return;
    const u32 gid = (u32)(a / p.K), i = (u32)(a % p.K);
    u64 r = YcsbWL::lookup(y, y.keys[a]);
    if (r == ~0ull) {   // reported; record 0 keeps every later a3 / exec access in bounds
        atomicCAS(&p.ctl->err.v, 0ull, (u64)CC_ERR_KEY_NOT_FOUND);
        r = 0;
    }
    acc_rec[a] = (uint32_t)r;
    keys_out[a] = (r << 27) | ((u64)gid << 6) | ((u64)i << 1) | (u64)(y.ops[a] >> 7);
}

cudaError_t launch_ycsb_gather(const ExecParams &p, const YcsbParams &y, PrepBufs &b,
                               cudaStream_t s) {
    const int blk = 256;
    const u64 n = (u64)p.n_txn * p.K;
    ycsb_gather_kernel<<<(unsigned)((n + blk - 1) / blk), blk, 0, s>>>(p, y, b.acc_rec, b.keys_in);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- table + index init
// Row initialiser: the device copy of the seeded input generator (inputs/ycsb.py):
// word j of row k = mix64(seed ^ (16k + j)) for j < 15, word 15 = 0.
__global__ void ycsb_init_rows_kernel(u64 *rows, uint64_t first, uint64_t n, uint64_t seed) {
    const uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;   // word index
    if (w >= n * 16) return;
    const uint64_t k = first + w / 16, j = w % 16;
    rows[w] = (j == 15) ? 0ull : mix64(seed ^ (16ull * k + j));
}

cudaError_t launch_ycsb_init_rows(u64 *rows, uint64_t first, uint64_t n, uint64_t seed,
                                  cudaStream_t s) {
    const uint64_t words = n * 16;
    ycsb_init_rows_kernel<<<(unsigned)((words + 255) / 256), 256, 0, s>>>(rows, first, n, seed);
    return cudaGetLastError();
}

__global__ void identity_index_kernel(u64 *keys, u64 *rowids, uint64_t n) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { keys[i] = i; rowids[i] = i; }
}

cudaError_t launch_identity_index(u64 *keys, u64 *rowids, uint64_t n, cudaStream_t s) {
    identity_index_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(keys, rowids, n);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- a1 generator
// The definition (readings Z12, Z13), per transaction:
//   op i: draw k = 0,1,..: u = rng(seed, gid, 1<<56 | i<<24 | k), rank = Zipf(u) by
//   binary search in the threshold table, key = ((rank-1)*A) mod n, until distinct;
//   sort keys ascending; write iff (rng(seed,gid,2<<56|i) >> 11) < floor(W*2^53);
//   field = rng(seed,gid,3<<56|i) mod 15.
// One warp per transaction: lane i draws op i's first candidate (k = 0) -- the binary
// searches of a transaction's ops run in parallel, not one after another as in the
// paper's one-thread loop -- then the warp resolves duplicates in op order (op i redraws
// k = 1, 2, ... while it equals an earlier op's key: the same draw sequence as the serial
// definition, so the keys are bit-identical), ranks the K distinct keys (ascending) and
// writes them; lane i writes op byte i.
__device__ __forceinline__ u32 ycsb_draw(uint64_t seed, u32 gid, u32 i, u64 k, uint64_t n, const u64 *T,
                                         uint64_t A) {
    const u64 u = rng3(seed, gid, (1ull << 56) | ((u64)i << 24) | k);
    u64 lo = 0, hi = n;   // count = #{j : T[j] <= u}
    while (lo < hi) {
        const u64 mid = lo + (hi - lo) / 2;
        if (__ldg(T + mid) <= u) lo = mid + 1; else hi = mid;
    }
    if (lo > n - 1) lo = n - 1;
    return (u32)((lo * A) % n);   // (rank - 1) * A mod n
}

__global__ void ycsb_gen_kernel(uint32_t *keys, uint8_t *ops, uint32_t n_txn, uint32_t K,
                                uint64_t n, u64 wthr, uint64_t seed, const u64 *T,
                                uint64_t A, u64 *err) {
    const u32 lane = threadIdx.x & 31u;
    const u32 gid = (u32)(((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (gid >= n_txn) return;   // warp-uniform
    constexpr unsigned FULL = 0xFFFFFFFFu;
    u32 mine = lane < K ? ycsb_draw(seed, gid, lane, 0, n, T, A) : 0xFFFFFFFFu;
    for (u32 i = 1; i < K; i++) {
        u32 ki = __shfl_sync(FULL, mine, (int)i);
        for (u64 k = 1;; k++) {
            if (!__any_sync(FULL, lane < i && mine == ki)) break;   // distinct from ops 0..i-1
            if (k >= (1u << 24)) {
                if (lane == 0) atomicCAS(err, 0ull, (u64)CC_ERR_CONFIG);   // the batch's error word
                return;
            }
            ki = ycsb_draw(seed, gid, i, k, n, T, A);   // (every lane: the same redraw)
        }
        if (lane == i) mine = ki;
    }
    u32 rank = 0;   // keys are distinct: position = number of smaller keys
    for (u32 j = 0; j < K; j++) {
        const u32 kj = __shfl_sync(FULL, mine, (int)j);
        rank += (lane < K && kj < mine) ? 1u : 0u;
    }
    if (lane < K) {
        const u64 base = (u64)gid * K;
        keys[base + rank] = mine;
        const u64 um = rng3(seed, gid, (2ull << 56) | lane);
        const u64 uf = rng3(seed, gid, (3ull << 56) | lane);
        uint8_t op = (uint8_t)(uf % 15u);
        if ((um >> 11) < wthr) op |= 0x80u;
        ops[base + lane] = op;
    }
}

cudaError_t launch_ycsb_gen(uint32_t *keys, uint8_t *ops, uint32_t n_txn, uint32_t K,
                            uint64_t n_rows, double W, uint64_t seed, const u64 *T,
                            uint64_t mult, u64 *err, cudaStream_t s) {
    if (K > 32) return cudaErrorInvalidValue;
    const u64 wthr = (u64)(W * 9007199254740992.0);
    const int blk = 128;   // 4 transactions per block
    const u64 threads = (u64)n_txn * 32;
    ycsb_gen_kernel<<<(unsigned)((threads + blk - 1) / blk), blk, 0, s>>>(keys, ops, n_txn, K, n_rows, wthr,
                                                                          seed, T, mult, err);
    return cudaGetLastError();
}

}  // namespace gcctb

namespace gcctb {
__global__ void index_lookup_kernel(YcsbParams y, const u64 *keys, uint64_t n, u64 *out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = YcsbWL::lookup(y, keys[i]);
}
cudaError_t launch_index_lookup(const YcsbParams &y, const u64 *keys, uint64_t n, u64 *out, cudaStream_t s) {
    if (n) index_lookup_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(y, keys, n, out);
    return cudaGetLastError();
}
// Eytzinger copy: sorted position j (in-order number m = j + 1 of a complete tree of height
// h) sits at depth h-1-ctz(m), index m >> (ctz(m)+1) within its level, i.e. BFS slot
// 2^(h-1-ctz(m)) + (m >> (ctz(m)+1)); positions >= n hold the ~0 padding.
__global__ void eytz_build_kernel(const u64 *keys, const u64 *rows, uint64_t n, int h, u64 *ek, u64 *er) {
    const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t slots = (1ull << h) - 1;
    if (j >= slots) return;
    const uint64_t m = j + 1;
    const int t = __ffsll((long long)m) - 1;
    const uint64_t i = (1ull << (h - 1 - t)) + (m >> (t + 1));
    ek[i] = j < n ? keys[j] : ~0ull;
    er[i] = j < n ? rows[j] : ~0ull;
    if (j == 0) { ek[0] = ~0ull; er[0] = ~0ull; }   // slot 0 unused
}
cudaError_t launch_eytz_build(const u64 *keys, const u64 *rows, uint64_t n, int h, u64 *ek, u64 *er,
                              cudaStream_t s) {
    const uint64_t slots = (1ull << h) - 1;
    eytz_build_kernel<<<(unsigned)((slots + 255) / 256), 256, 0, s>>>(keys, rows, n, h, ek, er);
    return cudaGetLastError();
}
// one tree level: out[c] = in[min(16c + 15, n_in - 1)] (the last key of node c), ~0 padding
__global__ void tree_level_kernel(const u64 *in, uint64_t n_in, u64 *out, uint64_t n_out_padded) {
    const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_out_padded) return;
    const uint64_t n_nodes = (n_in + 15) / 16;
    out[c] = c < n_nodes ? in[min(16 * c + 15, n_in - 1)] : ~0ull;
}
cudaError_t launch_tree_level(const u64 *in, uint64_t n_in, u64 *out, uint64_t n_out_padded, cudaStream_t s) {
    tree_level_kernel<<<(unsigned)((n_out_padded + 255) / 256), 256, 0, s>>>(in, n_in, out, n_out_padded);
    return cudaGetLastError();
}
__global__ void fill_u64_kernel(u64 *p, u64 v, uint64_t n) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
cudaError_t launch_fill_u64(u64 *p, u64 v, uint64_t n, cudaStream_t s) {
    if (n) fill_u64_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, v, n);
    return cudaGetLastError();
}

void preload_ycsb_kernels() {   // (see preload_prep_kernels) every executor instantiation
    const int lanes[5] = {1, 4, 8, 16, 32};
    for (int sc = 0; sc < CC_NUM_SCHEMES; sc++)
        for (int l : lanes) ycsb_exec_max_blocks_per_sm(sc, l, 256, 0);
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, ycsb_gen_kernel);
    cudaFuncGetAttributes(&a, ycsb_gather_kernel);
    cudaFuncGetAttributes(&a, fill_u64_kernel);
    cudaFuncGetAttributes(&a, index_lookup_kernel);
}
}  // namespace gcctb
