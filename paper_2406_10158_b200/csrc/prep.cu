// prep.cu -- a2 CC-state reset, a3 preprocessing for the deterministic schemes
// (access table, GaccO lock table, GPUTx ranks / K-sets) and a7 result emission.
//
// Access table: every access becomes the 64-bit sort key
//   (rec << 27) | (gid << 6) | (i << 1) | is_write
// so one radix sort groups accesses per item with transaction ids ascending (keys arrive
// in (gid, i) order and the sort is stable, so only the record bits are sorted).  Each
// sorted position then needs the start of its item's segment and the last write at or
// before it: one fused max-scan of (head ? p : 0, write ? p + 1 : 0).  The paper uses
// thrust sort + scan; here both are the library's own kernels (sort.cu).
#include <cstdlib>

#include "exec.cuh"

namespace gcctb {

constexpr int KEY_SHIFT = 27;
constexpr u64 GID_MASK = (1ull << 21) - 1;

// ------------------------------------------------------------------ a2 reset
// a2 prologue of a submit, one launch: the retry ring and retry queues, the per-
// transaction results and the control block; then the batch's own a1 error word is
// folded into the fresh control block (block 0, after its reset), so a failed generation
// stops the submit before anything executes.  The CC words themselves (the throughput
// window starts "from the initialization of the CC method", Z19) are zeroed
// by the submit that used them, on the reset stream, while the next submit runs on the
// other word set (cc_submit); every scheme's initial words are zeros.
__global__ void a2_kernel(u64 *ring, uint32_t ring_words, Ctl *ctl, uint8_t *committed, uint32_t *restarts,
                          u64 *ohi, u64 *olo, uint32_t n_txn, const u64 *batch_err) {
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    if (blockIdx.x == 0) {
        for (uint32_t r = threadIdx.x; r < sizeof(Ctl) / 8; r += blockDim.x) reinterpret_cast<u64 *>(ctl)[r] = 0ull;
        __syncthreads();
        if (threadIdx.x == 0 && batch_err) {
            const u64 e = *batch_err;
            if (e) ctl->err.v = e;
        }
    }
    for (uint64_t r = tid; r < ring_words; r += stride) ring[r] = 0ull;
    for (uint64_t i = tid; i < n_txn; i += stride) {
        committed[i] = 0;
        restarts[i] = 0;
        ohi[i] = ~0ull;
        olo[i] = ~0ull;
    }
}

// The background zeroing of a used word set (a2, reset stream): 32 B evict-first stores
// (st.global.cs), so the 84-168 MB it writes beside the next submit's executor do not
// displace that executor's control words and hot rows from L2 (GC_ZERO_CS=0: memset;
// measured neutral on the bench, 100.6 / 101.0 vs 101.3 / 99.5 M txn/s, profiles/
// r02_bench_v21_zero_ab.txt).
#ifndef GC_ZERO_CS
#define GC_ZERO_CS 1
#endif
#ifndef GC_ZERO_BLOCKS_PER_SM_X4
#define GC_ZERO_BLOCKS_PER_SM_X4 2   // blocks per SM x 4 (2: one block per two SMs)
#endif
#ifndef GC_ZERO_THREADS
#define GC_ZERO_THREADS 256
#endif
__global__ void zero_cs_kernel(u64 *p, uint64_t n4) {   // n4: 32 B units
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride)
        asm volatile("st.global.cs.v4.u64 [%0], {%1, %1, %1, %1};" ::"l"(p + 4 * i), "l"(0ull) : "memory");
}
cudaError_t launch_zero_words(u64 *p, uint64_t words, cudaStream_t s) {
    if (!GC_ZERO_CS || (words & 3)) return cudaMemsetAsync(p, 0, words * 8, s);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // a small grid: the zeroing runs beside the next submit's executor and has ~two submits
    // to finish; a full-GPU grid competes with that executor for issue slots
    zero_cs_kernel<<<(unsigned)(sms * GC_ZERO_BLOCKS_PER_SM_X4 / 4 > 0 ? sms * GC_ZERO_BLOCKS_PER_SM_X4 / 4 : 1),
                     GC_ZERO_THREADS, 0, s>>>(p, words / 4);
    return cudaGetLastError();
}

cudaError_t launch_a2(u64 *ring, uint32_t ring_words, Ctl *ctl, uint8_t *committed, uint32_t *restarts, u64 *ohi,
                      u64 *olo, uint32_t n_txn, const u64 *batch_err, cudaStream_t s) {
    const uint64_t work = ring_words > n_txn ? ring_words : n_txn;
    const unsigned g = (unsigned)((work + 1023) / 1024);
    a2_kernel<<<g < 2 ? 2 : g, 256, 0, s>>>(ring, ring_words, ctl, committed, restarts, ohi, olo, n_txn, batch_err);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ a3 kernels
// markers for the fused max-scan: segment heads (their own position) and writes (p + 1)
__global__ void a3_marks_kernel(const u64 *keys, uint32_t *head_at, uint32_t *write_at, uint64_t n) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const u64 k = keys[p];
    head_at[p] = (p == 0 || (keys[p - 1] >> KEY_SHIFT) != (k >> KEY_SHIFT)) ? (uint32_t)p : 0u;
    write_at[p] = (k & 1ull) ? (uint32_t)(p + 1) : 0u;   // write marker for the last-write scan
}

// GaccO lock table: queue position of each access inside its item's segment
// ("recording which transaction currently owns each data item").  An item's
// segment is named by its first sorted position, which also indexes its cursor.  acc_rdy:
// the cursor value at which the last earlier write of the item has installed (its queue
// position + 1; 0 if no write precedes the access): from then on the row holds exactly what
// the access would read at its turn, since only reads sit between that write and it.
__global__ void positions_kernel(const u64 *keys, const uint32_t *seg_of, const uint32_t *lw_scan,
                                 uint32_t K, uint32_t *acc_seg, uint32_t *acc_pos, uint32_t *acc_rdy,
                                 uint32_t *sorted_pos, uint32_t *cursor, uint64_t n) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const u64 k = keys[p];
    const uint64_t gid = (k >> 6) & GID_MASK, i = (k >> 1) & 31u;
    const uint64_t a = gid * K + i;
    const uint32_t seg = seg_of[p];
    acc_seg[a] = seg;
    acc_pos[a] = (uint32_t)p - seg;
    const uint32_t q = p > seg ? lw_scan[p - 1] : 0u;   // last write before p, + 1
    acc_rdy[a] = q > seg ? q - seg : 0u;
    sorted_pos[a] = (uint32_t)p;
    if (seg == (uint32_t)p) cursor[p] = 0u;
}

// GPUTx ranks (PAPER.md:218 read per Z1): rank(T) = 1 + max rank over the conflicting
// earlier transactions.  In each item's id-ordered segment a read depends on the last
// earlier write; a write on the last earlier write and every read since (Z2: reads do
// not conflict).  Dataflow pass: lanes claim transactions in increasing id (so every
// predecessor is claimed by a running lane) and wait for predecessor ranks.
constexpr uint32_t RANK_UNSET = 0xFFFFFFFFu;

template <int G>
__global__ void __launch_bounds__(1024) gputx_rank_kernel(
    const u64 *keys, const uint32_t *sorted_pos, const uint32_t *seg_of,
    const uint32_t *lw, uint32_t *rank, uint32_t n_txn, uint32_t K, Ctl *ctl,
    u64 watchdog_ns, uint32_t poll_cap_ns, uint32_t *acc_dep) {
    // a tile of G lanes per transaction, lane i resolves the predecessors of access i
    auto tile = cg::tiled_partition<G>(cg::this_thread_block());
    const uint32_t li = tile.thread_rank();
    const u64 deadline = globaltimer_ns() + watchdog_ns;
    for (;;) {
        u64 s = 0;
        if (li == 0) s = atomicAdd(&ctl->rank_head.v, 1ull);
        s = tile.shfl(s, 0);
        if (s >= n_txn) return;
        const uint32_t gid = (uint32_t)s;
        uint32_t r = 0, dep = 0;
        bool fail = false;
        if (li < K) {
            const uint32_t p = sorted_pos[(u64)gid * K + li];
            const uint32_t s0 = seg_of[p];   // first position of this item's segment
            const bool w = keys[p] & 1ull;
            const uint32_t q = (p > s0) ? lw[p - 1] : 0u;   // last write before p (+1)
            const bool has_q = q > s0;                        // inside this segment
            const uint32_t lo = has_q ? q - 1 : s0;           // first predecessor to visit
            const uint32_t hi = w ? p : (has_q ? q : s0);     // reads: only that write
            // A rank is written once (release), so a relaxed load that sees a value sees the
            // final one and nothing else is read through it: the predecessors' ranks are
            // loaded 8 at a time (independent loads), and only the unset ones are polled.
            // (A write after a long run of reads -- a hot item -- otherwise paid one
            // dependent L2 round trip per read.)
            constexpr int B = 8;
            bool first = has_q;   // the chunk at lo starts with the item's last earlier write
            for (uint32_t x = lo; x < hi && !fail; x += B) {
                uint32_t u[B], ru[B];
#pragma unroll
                for (int j = 0; j < B; j++)
                    u[j] = (x + j < hi) ? (uint32_t)((__ldg(keys + x + j) >> 6) & GID_MASK) : 0xFFFFFFFFu;
#pragma unroll
                for (int j = 0; j < B; j++) ru[j] = (u[j] != 0xFFFFFFFFu) ? ld_relaxed32(&rank[u[j]]) : 0u;
#pragma unroll
                for (int j = 0; j < B; j++) {
                    unsigned ns = 8;
                    while (ru[j] == RANK_UNSET && !fail) {
                        if (globaltimer_ns() > deadline || ld_relaxed(&ctl->err.v)) {
                            atomicCAS(&ctl->err.v, 0ull, (u64)CC_ERR_WATCHDOG);
                            fail = true;
                            break;
                        }
                        __nanosleep(ns);
                        ns = ns < poll_cap_ns ? ns * 2 : poll_cap_ns;
                        ru[j] = ld_relaxed32(&rank[u[j]]);
                    }
                    if (u[j] != 0xFFFFFFFFu) r = max(r, ru[j] + 1);
                }
                if (first) {   // dependency of the access's row read: that write's K-set, + 1
                    dep = ru[0] + 1;
                    first = false;
                }
            }
            // (the executor may read the row once K-set dep - 1 has completed, before its
            // own gate: only reads sit between that write and this access in id order)
            acc_dep[(u64)gid * K + li] = dep;
        }
        if (tile.any(fail)) return;
        r = cg::reduce(tile, r, cg::greater<uint32_t>());
        if (li == 0) {
            // relaxed: readers use only the value itself (nothing is published through it),
            // so the MEMBAR of a release store would only lengthen the chain
            st_relaxed32(&rank[gid], r);   // (max_rank: from the rank sort, not an atomic per txn)
        }
    }
}

__global__ void fill_u32_kernel(uint32_t *a, uint32_t v, uint64_t n) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = v;
}
__global__ void iota_kernel(uint32_t *a, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = i;
}

// K-set boundaries over the rank-sorted transactions (sorted ranks as u64 sort keys)
__global__ void rank_bounds_kernel(const u64 *rs, uint32_t *start, uint32_t *count,
                                   uint32_t *done, uint32_t n) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint32_t r = (uint32_t)rs[p];
    if (p == 0 || (uint32_t)rs[p - 1] != r) { start[r] = p; done[r] = 0; }
}
__global__ void rank_count_kernel(const u64 *rs, const uint32_t *start, uint32_t *count,
                                  uint32_t n, Ctl *ctl) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint32_t r = (uint32_t)rs[p];
    if (p == n - 1 || (uint32_t)rs[p + 1] != r) count[r] = p + 1 - start[r];
    if (p == n - 1) ctl->max_rank.v = r;   // ranks sorted ascending: the last is the max
}
// sort keys of a u32 (rank) or u64 (order key) array, with the identity permutation
__global__ void keys_iota_kernel(const uint32_t *r32, const u64 *r64, u64 *keys, uint32_t *idx, uint32_t n) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    keys[g] = r32 ? (u64)r32[g] : r64[g];
    idx[g] = g;
}
__global__ void copy_u32_kernel(const uint32_t *src, uint32_t *dst, uint32_t n) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) dst[g] = src[g];
}

int rank_kernel_grid() {
    int dev = 0, sms = 148, nb = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, gputx_rank_kernel<32>, 256, 0);
    // a quarter of the resident capacity: fewer transactions waiting on predecessors poll
    // less, and the long chains resolve faster (configs[1] theta 0.6: rank pass 0.81 ->
    // 0.73 ms; theta 0.8: 13.5 -> 6.6 ms; profiles/r01_gputx_rank_sweep.txt)
    const int g = (nb > 0 ? nb : 1) * sms / 4;
    return g > 0 ? g : 1;
}

static int bits_for(uint64_t x) {
    int b = 1;
    while (b < 64 && (1ull << b) <= x) b++;
    return b;
}

size_t prep_cub_bytes(uint64_t n_acc, uint64_t n_txn) {
    const size_t a = gc_sort_temp_bytes(n_acc > n_txn ? n_acc : n_txn), b = gc_scan_temp_bytes(n_acc);
    return (a > b ? a : b) + 256;
}

cudaError_t launch_prep_common(const ExecParams &p, PrepBufs &b, uint64_t n_records, bool gputx,
                               int grid, cudaStream_t s, int rank_block) {
    const uint64_t n = (uint64_t)p.n_txn * p.K;
    const int blk = 256;
    const unsigned g = (unsigned)((n + blk - 1) / blk);
    cudaError_t e;
    const int end_bit = KEY_SHIFT + bits_for(n_records);
    // keys arrive in (gid, i) order; a stable LSD sort on the record bits alone keeps
    // transaction ids ascending within each item (3 passes for 2^24 records, not 7)
    u64 *sk = nullptr;
    e = gc_sort(b.keys_in, nullptr, b.keys_out, nullptr, n, nullptr, KEY_SHIFT, end_bit > 64 ? 64 : end_bit,
                b.cub_tmp, b.cub_bytes, s, &sk, nullptr);
    if (e) return e;
    // per sorted position: its segment's first position (seg_start) and the last write at
    // or before it, + 1 (seg_id's storage)
    a3_marks_kernel<<<g, blk, 0, s>>>(sk, b.head_flag, b.lw, n);
    e = gc_scan_max2(b.head_flag, b.lw, b.seg_start, b.seg_id, n, b.cub_tmp, b.cub_bytes, s);
    if (e) return e;
    positions_kernel<<<g, blk, 0, s>>>(sk, b.seg_start, b.seg_id, p.K, b.acc_seg, b.acc_pos, b.acc_rdy,
                                       b.sorted_pos, b.cursor, n);
    if (!gputx) return cudaGetLastError();
    fill_u32_kernel<<<(p.n_txn + blk - 1) / blk, blk, 0, s>>>(b.rank, RANK_UNSET, p.n_txn);
    // experiment knobs (environment): poll cap and a grid divisor for the rank pass
    static const uint32_t poll_cap = getenv("GCCTB_RANK_POLL_NS") ? (uint32_t)atoi(getenv("GCCTB_RANK_POLL_NS")) : 512u;
    static const int grid_div = getenv("GCCTB_RANK_GRID_DIV") ? atoi(getenv("GCCTB_RANK_GRID_DIV")) : 1;
    if (grid_div > 1) grid = grid / grid_div > 0 ? grid / grid_div : 1;
    if (p.K <= 16)
        gputx_rank_kernel<16><<<grid, rank_block, 0, s>>>(sk, b.sorted_pos, b.seg_start, b.seg_id, b.rank, p.n_txn,
                                                          p.K, p.ctl, p.watchdog_ns, poll_cap, b.acc_rdy);
    else
        gputx_rank_kernel<32><<<grid, rank_block, 0, s>>>(sk, b.sorted_pos, b.seg_start, b.seg_id, b.rank, p.n_txn,
                                                          p.K, p.ctl, p.watchdog_ns, poll_cap, b.acc_rdy);
    // K-sets: transactions sorted by rank (stable: ids ascending inside a K-set)
    const unsigned gt = (p.n_txn + blk - 1) / blk;
    u64 *k1 = sk == b.keys_in ? b.keys_out : b.keys_in, *k2 = sk;   // the access keys are dead now
    keys_iota_kernel<<<gt, blk, 0, s>>>(b.rank, nullptr, k1, b.gid_in, p.n_txn);
    u64 *rk = nullptr;
    uint32_t *ro = nullptr;
    e = gc_sort(k1, b.gid_in, k2, b.rank_sorted, p.n_txn, nullptr, 0, bits_for(p.n_txn), b.cub_tmp, b.cub_bytes, s,
                &rk, &ro);
    if (e) return e;
    copy_u32_kernel<<<gt, blk, 0, s>>>(ro, b.rank_order, p.n_txn);
    rank_bounds_kernel<<<gt, blk, 0, s>>>(rk, b.rank_start, b.rank_count, b.rank_done, p.n_txn);
    rank_count_kernel<<<gt, blk, 0, s>>>(rk, b.rank_start, b.rank_count, p.n_txn, p.ctl);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ a7 emission
__global__ void commit_pos_kernel(const uint32_t *sorted_gid, const uint8_t *committed,
                                  uint32_t *pos_out, uint32_t n) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const uint32_t g = sorted_gid[p];
    pos_out[g] = committed[g] ? p : 0xFFFFFFFFu;
}

__global__ void gather_hi_kernel(const u64 *hi, const uint32_t *perm, u64 *out, uint32_t n) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n) out[p] = hi[perm[p]];
}

// a7 copy-out, one launch: per transaction the results (commit positions from `pos`, or --
// 2PL, pos == null -- the dense lock-point ticket itself, see dense_ticket_pos_kernel),
// the committed / restart totals; the last block to finish writes the stats words
// (stats_body).  (Round 1 used three launches: positions, copy-out, stats.)
__device__ void stats_body(const Ctl *c, uint64_t *stats, const unsigned long long *stages,
                           unsigned long long *sticky);
__global__ void copy_out_kernel(const ExecParams p, cc_result r, const uint32_t *pos, uint64_t *mirror) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t c = 0, a = 0;
    if (i < p.n_txn) {
        c = p.committed[i];
        a = p.restarts[i];
        if (c && p.order_lo[i] >= 0xFFFFFFFFull)   // the 32-bit commit-position sort would be wrong
            atomicCAS(&p.ctl->err.v, 0ull, (u64)CC_ERR_TS_OVERFLOW);
        r.committed[i] = (uint8_t)c;
        if (r.restarts) r.restarts[i] = a;
        if (r.order_hi) r.order_hi[i] = p.order_hi[i];
        if (r.order_lo) r.order_lo[i] = p.order_lo[i];
        if (r.commit_pos) r.commit_pos[i] = pos ? pos[i] : (c ? (uint32_t)p.order_lo[i] : 0xFFFFFFFFu);
    }
    c = __reduce_add_sync(0xFFFFFFFFu, c);
    a = __reduce_add_sync(0xFFFFFFFFu, a);
    if ((threadIdx.x & 31) == 0) {
        if (c) atomicAdd(&p.ctl->done.v, (u64)c);
        if (a) atomicAdd(&p.ctl->aborts.v, (u64)a);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();   // this block's totals before its finish count
        const u64 f = atomicAdd(&p.ctl->fin.v, 1ull);
        if (f == gridDim.x - 1) {   // every block's totals are in
            __threadfence();
            st_relaxed(&p.ctl->fin.v, 0ull);   // (for a later copy-out of the same control block)
            if (r.stats) stats_body(p.ctl, r.stats, p.stages, p.sticky);
            if (mirror && mirror != r.stats) stats_body(p.ctl, mirror, p.stages, nullptr);   // cc_sync's copy
        }
    }
}

// sum the per-thread stage slots (stages[8 + t*8 + k]) into stages[0..7]
__global__ void stages_reduce_kernel(unsigned long long *stages, uint64_t n_threads) {
    __shared__ unsigned long long acc[STAGE_WORDS];
    if (threadIdx.x < STAGE_WORDS) acc[threadIdx.x] = 0;
    __syncthreads();
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_threads;
         t += (uint64_t)gridDim.x * blockDim.x)
        for (int k = 0; k < STAGE_WORDS; k++) {
            const unsigned long long v = stages[STAGE_WORDS + t * STAGE_WORDS + k];
            if (v) atomicAdd(&acc[k], v);
        }
    __syncthreads();
    if (threadIdx.x < STAGE_WORDS && acc[threadIdx.x]) atomicAdd(&stages[threadIdx.x], acc[threadIdx.x]);
}
cudaError_t launch_stages_reduce(unsigned long long *stages, uint64_t n_threads, cudaStream_t s) {
    stages_reduce_kernel<<<148, 256, 0, s>>>(stages, n_threads);
    return cudaGetLastError();
}

__device__ void stats_body(const Ctl *c, uint64_t *stats, const unsigned long long *stages,
                           unsigned long long *sticky) {
    if (c->err.v && sticky) atomicCAS(sticky, 0ull, c->err.v);   // survives the next submit's reset
    stats[0] = c->done.v;
    stats[1] = c->aborts.v;
    stats[2] = c->done.v + c->aborts.v;
    stats[3] = c->err.v;
    stats[4] = c->max_rank.v;
    stats[5] = c->ts.v;
    for (int k = 6; k < CC_STATS_WORDS; k++) stats[k] = 0;
    if (stages)
        for (int k = 0; k < 7; k++) stats[8 + k] = stages[k];
}
__global__ void stats_kernel(const Ctl *c, uint64_t *stats, const unsigned long long *stages,
                             unsigned long long *sticky) {
    stats_body(c, stats, stages, sticky);
}

// 2PL: the lock-point ticket is drawn only by attempts that commit, so the committed
// set's tickets are exactly 0 .. n_committed-1 and the ticket is the commit position
__global__ void dense_ticket_pos_kernel(const u64 *lo, const uint8_t *committed, uint32_t *pos_out,
                                        uint32_t n) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n) pos_out[g] = committed[g] ? (uint32_t)lo[g] : 0xFFFFFFFFu;
}

// TO / MVCC / Silo: the committed order keys are distinct integers below R (the last
// timestamp + 1, or the number of tickets drawn), so a transaction's commit position is
// the number of committed keys below its own -- a bitmap over [0, R) and a prefix count
// of its set bits (five small kernels instead of four radix passes of four kernels each).
// The kernels loop over [0, R) with R read on the device, so the grids do not depend on it.
constexpr int BM_CHUNK = 1024;   // words per chunk: one block scans one chunk
__device__ __forceinline__ u64 bm_range(const u64 *rptr, u64 radd) {
    const u64 r = *rptr + radd;
    return r < RANK_BITMAP_BITS ? r : RANK_BITMAP_BITS;   // beyond: reported by bm_set_kernel
}

__global__ void bm_zero_kernel(uint32_t *bm, const u64 *rptr, u64 radd) {
    const u64 words = (bm_range(rptr, radd) + 31) / 32;
    for (u64 w = (u64)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += (u64)gridDim.x * blockDim.x) bm[w] = 0u;
}
__global__ void bm_set_kernel(const u64 *lo, const uint8_t *committed, uint32_t *bm, uint32_t n, Ctl *ctl) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n || !committed[g]) return;
    if (lo[g] >= RANK_BITMAP_BITS) {   // a 32-bit ticket range is beyond the bitmap (never seen)
        atomicCAS(&ctl->err.v, 0ull, (u64)CC_ERR_TS_OVERFLOW);
        return;
    }
    atomicOr(&bm[lo[g] >> 5], 1u << (lo[g] & 31));
}
// per chunk of 1,024 words: exclusive prefix of the words' popcounts, and the chunk total
__global__ void __launch_bounds__(BM_CHUNK) bm_chunk_kernel(const uint32_t *bm, uint32_t *pre, uint32_t *csum,
                                                           const u64 *rptr, u64 radd) {
    __shared__ uint32_t ws[BM_CHUNK / 32];
    const u64 words = (bm_range(rptr, radd) + 31) / 32, chunks = (words + BM_CHUNK - 1) / BM_CHUNK;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (u64 c = blockIdx.x; c < chunks; c += gridDim.x) {
        const u64 w = c * BM_CHUNK + threadIdx.x;
        const uint32_t v = w < words ? __popc(bm[w]) : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) ws[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t t = ws[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, t, o);
                if (lane >= (uint32_t)o) t += y;
            }
            ws[lane] = t;
        }
        __syncthreads();
        if (w < words) pre[w] = (warp ? ws[warp - 1] : 0u) + x - v;
        if (threadIdx.x == 0) csum[c] = ws[31];
        __syncthreads();
    }
}
// exclusive scan of the chunk totals, one block (loops with a carry)
__global__ void __launch_bounds__(1024) bm_csum_kernel(uint32_t *csum, const u64 *rptr, u64 radd) {
    __shared__ uint32_t ws[32];
    const u64 words = (bm_range(rptr, radd) + 31) / 32, chunks = (words + BM_CHUNK - 1) / BM_CHUNK;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t carry = 0;
    for (u64 c0 = 0; c0 < chunks; c0 += 1024) {
        const u64 c = c0 + threadIdx.x;
        const uint32_t v = c < chunks ? csum[c] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane == 31) ws[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t t = ws[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, t, o);
                if (lane >= (uint32_t)o) t += y;
            }
            ws[lane] = t;
        }
        __syncthreads();
        if (c < chunks) csum[c] = carry + (warp ? ws[warp - 1] : 0u) + x - v;
        carry += ws[31];
        __syncthreads();
    }
}
__global__ void bm_pos_kernel(const u64 *lo, const uint8_t *committed, const uint32_t *bm, const uint32_t *pre,
                              const uint32_t *csum, uint32_t *pos, uint32_t n) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    if (!committed[g]) { pos[g] = 0xFFFFFFFFu; return; }
    const u64 k = lo[g], w = k >> 5;
    if (k >= RANK_BITMAP_BITS) { pos[g] = 0xFFFFFFFFu; return; }
    pos[g] = csum[w / BM_CHUNK] + pre[w] + __popc(bm[w] & ((1u << (k & 31)) - 1u));
}

// TicToc: every committed transaction drew one ticket 0..n-1 -- the order by key_lo is
// the inverse permutation, no sort
__global__ void ticket_perm_kernel(const u64 *lo, const uint8_t *committed, uint32_t *perm, uint32_t n) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < n && committed[g] && lo[g] < n) perm[lo[g]] = g;
}

cudaError_t launch_finalize(const ExecParams &p, const cc_result &res, PrepBufs &b,
                            bool deterministic, bool two_pass, cudaStream_t s, bool dense_ticket, bool lo_dense,
                            const RankBitmap *rb, uint64_t *stats_mirror) {
    const uint32_t n = p.n_txn;
    const int blk = 256;
    const unsigned g = (n + blk - 1) / blk;
    // commit positions: a stable radix sort of the order keys (lo, then hi when used)
    uint32_t *pos = b.acc_pos;   // reuse as n-sized scratch after execution
    if (dense_ticket) {
        pos = nullptr;   // copy_out takes the ticket as the position
    } else if (deterministic) {
        iota_kernel<<<g, blk, 0, s>>>(b.rank_order, n);
        commit_pos_kernel<<<g, blk, 0, s>>>(b.rank_order, p.committed, pos, n);
    } else if (rb && !two_pass) {   // TO / MVCC / Silo: bitmap + prefix count
        const bool ts = p.scheme == CC_TO || p.scheme == CC_MVCC;
        const u64 *rptr = ts ? &p.ctl->ts.v : &p.ctl->ticket.v;
        const u64 radd = ts ? 1 : 0;
        const int gs = 148 * 4;
        bm_zero_kernel<<<gs, 256, 0, s>>>(rb->bits, rptr, radd);
        bm_set_kernel<<<g, blk, 0, s>>>(p.order_lo, p.committed, rb->bits, n, p.ctl);
        bm_chunk_kernel<<<gs, BM_CHUNK, 0, s>>>(rb->bits, rb->pre, rb->csum, rptr, radd);
        bm_csum_kernel<<<1, 1024, 0, s>>>(rb->csum, rptr, radd);
        bm_pos_kernel<<<g, blk, 0, s>>>(p.order_lo, p.committed, rb->bits, rb->pre, rb->csum, pos, n);
    } else {
        u64 *k1 = b.keys_in, *k2 = b.keys_out;   // n_acc >= n scratch
        u64 *sk = k2;
        uint32_t *perm = b.rank_order;
        cudaError_t e;
        if (lo_dense) {   // TicToc: tickets are drawn only by committing attempts -- 0..n-1
            ticket_perm_kernel<<<g, blk, 0, s>>>(p.order_lo, p.committed, perm, n);
        } else {
            keys_iota_kernel<<<g, blk, 0, s>>>(nullptr, p.order_lo, k1, b.gid_in, n);
            // key_lo is a ticket, a 31-bit timestamp or a gid: 32 bits suffice (copy_out flags
            // a value >= 2^32 - 1 as an overflow), 4 radix passes instead of 8
            e = gc_sort(k1, b.gid_in, k2, b.rank_order, n, nullptr, 0, 32, b.cub_tmp, b.cub_bytes, s, &sk, &perm);
            if (e) return e;
        }
        if (two_pass) {   // then by key_hi (stable): TicToc's (commit_ts, ticket), partitioned (phase, ...)
            u64 *hk = sk == k1 ? k2 : k1;
            uint32_t *hv = perm == b.gid_in ? b.rank_order : b.gid_in;
            gather_hi_kernel<<<g, blk, 0, s>>>(p.order_hi, perm, hk, n);
            // TicToc: key_hi = commit_ts (48 bits); partitioned: the phase bits (63, rank << 48)
            e = gc_sort(hk, perm, sk, hv, n, nullptr, 0, lo_dense ? 48 : 64, b.cub_tmp, b.cub_bytes, s, &sk, &perm);
            if (e) return e;
        }
        commit_pos_kernel<<<g, blk, 0, s>>>(perm, p.committed, pos, n);
    }
    copy_out_kernel<<<g, blk, 0, s>>>(p, res, pos, stats_mirror);   // + the stats words (last block; res.stats is set)
    return cudaGetLastError();
}

// f-4: fold an error raised while a batch was prepared ahead into the submit's control block
__global__ void merge_err_kernel(const Ctl *src, Ctl *dst) {
    const u64 e = src->err.v;
    if (e) atomicCAS(&dst->err.v, 0ull, e);
    dst->max_rank.v = src->max_rank.v;   // GPUTx: the prepared rank pass counted the K-sets
}
cudaError_t launch_merge_err(const Ctl *src, Ctl *dst, cudaStream_t s) {
    merge_err_kernel<<<1, 1, 0, s>>>(src, dst);
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
void preload_prep_kernels() {
    preload1(a2_kernel); preload1(zero_cs_kernel); preload1(a3_marks_kernel); preload1(positions_kernel);
    preload1(gputx_rank_kernel<16>); preload1(gputx_rank_kernel<32>); preload1(fill_u32_kernel); preload1(iota_kernel);
    preload1(rank_bounds_kernel); preload1(rank_count_kernel); preload1(keys_iota_kernel); preload1(copy_u32_kernel);
    preload1(commit_pos_kernel); preload1(gather_hi_kernel); preload1(copy_out_kernel); preload1(stages_reduce_kernel);
    preload1(stats_kernel); preload1(dense_ticket_pos_kernel); preload1(ticket_perm_kernel); preload1(merge_err_kernel);
    preload1(bm_zero_kernel); preload1(bm_set_kernel); preload1(bm_chunk_kernel);
    preload1(bm_csum_kernel); preload1(bm_pos_kernel);
}
}  // namespace gcctb
