// internal.h -- structures shared by the host driver (db.cu) and the kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/gcctb.h"

// Words per record of the single-word schemes' control-word array: 1 (packed 8 B SoA) or,
// with CC_FLAG_META_PAD, GC_META_PAD_WORDS (one word per 32 B sector);
// the array is allocated for the padded layout.
constexpr unsigned GC_META_PAD_WORDS = 4;

namespace gcctb {

// Device control block of one submit (reset by the a2 reset kernel).  Every hot
// counter lives in its own 256 B block so that claims, tickets, timestamps and the
// error word never share an L2 line (and usually not an L2 slice).
struct alignas(256) Counter {
    unsigned long long v;
    unsigned long long pad[31];
};
struct Ctl {
    Counter head;       // claim counter over [0, n_txn)
    Counter tail;       // retry-ring append counter (producers): seal bit 63 | reserved slots
    Counter rhead;      // retry-ring claim counter (consumers)
    Counter done;       // committed transactions (counted at emission)
    Counter ts;         // TO/MVCC timestamp allocator (first ts = 1)
    Counter ticket;     // lock-point / serialization-point ticket
    Counter err;        // first device error (cc_status), 0 = none
    Counter aborts;     // sum of restarts (counted at emission)
    Counter max_rank;   // GPUTx: number of K-sets - 1
    Counter rank_head;  // GPUTx rank-pass claim counter
    Counter rtail;      // sealed retry-batch size + 1 (0: not sealed yet)
    Counter events;     // CC_FLAG_EVENTS: event sequence counter
    Counter pacing;     // TO/MVCC: transactions in retry backoff right now (adaptive cap)
    Counter kdone;      // GPUTx: K-sets completed so far (they complete in order)
    Counter pacing_lk;  // transactions in post-lock-wait jitter right now (adaptive cap)
    Counter warm_hits;  // CC_FLAG_WARM: sink for the warm loads (practically never incremented)
    Counter fin;        // a7: blocks of the copy-out launch that have finished (last one: stats)
};
// one event of the debug log: 24 bytes
struct Event {
    unsigned long long seq;   // global order (atomic counter)
    uint32_t gid, rec;        // transaction, record (global record id)
    uint32_t attempt;         // restart ordinal of the attempt
    uint32_t kind;            // 0 read, 1 write (install), 2 commit, 3 abort
};

enum { KIND_YCSB = 1, KIND_TPCC = 2 };

// retry queues: one FIFO word per hashed control word (GC_RETRY_FIFO), after the ring
constexpr uint32_t GC_RQ_N = 1u << 16;
// Workload-independent execution parameters.
struct ExecParams {
    int scheme;
    uint32_t n_txn;
    uint32_t K;                  // accesses per transaction slot (YCSB ops_per_txn)
    uint32_t wd;
    uint32_t flags;
    uint32_t lanes;              // lanes per transaction (1 = thread per txn)
    uint32_t claim_chunk;        // fresh ids claimed per atomic (>= 1)
    unsigned long long watchdog_ns;
    Ctl *ctl;
    unsigned long long *meta;    // CC words: 1 x u64 per record, MVCC 2 x u64 (lo, hi)
    uint32_t meta_stride = 1;    // words per record for the single-word schemes (1 or GC_META_PAD_WORDS)
    uint32_t meta_shift = 0;     // log2(meta_stride)
    unsigned long long *arena;   // MVCC version nodes: ARENA_HDR header words + the row
    uint32_t to_backoff_cap;     // TO/MVCC backoff cap exponent (0: adaptive); experiment
                                 // knob, environment GCCTB_TO_BACKOFF_CAP
    unsigned long long mvcc_split;   // MVCC words: 0 = interleaved (lo, hi) pairs; else lo at
                                     // meta[r], hi at meta[mvcc_split + r] (CC_FLAG_MVCC_SPLIT)
    unsigned long long *ring;    // retry batch (compacted aborted ids), n_txn slots
    void *ws;                    // thread mode: per-worker access workspace in global memory when
                                 // it does not fit shared memory (else null: dynamic smem)
    uint32_t ring_cap;
    uint32_t rq_herd_2pl;        // 2PL: pacing transactions from which exclusive retriers queue
    unsigned long long *rq;      // retry queues (GC_RETRY_FIFO): GC_RQ_N words after the ring,
                                 // ticket (low 32) | serving (high 32), hashed by control word
    // per-transaction internal results
    uint8_t *committed;
    uint32_t *restarts;
    unsigned long long *order_hi;
    unsigned long long *order_lo;
    unsigned long long *read_out;  // caller buffer (may be null)
    // deterministic-scheme tables (a3)
    const uint32_t *acc_rec;     // resolved record of each access (n_txn*K) or null
    const uint32_t *acc_seg;     // GaccO: segment (item) id of each access
    const uint32_t *acc_pos;     // GaccO: queue position of each access
    const uint32_t *acc_rdy;     // GaccO: cursor value at which the item's last earlier write
                                 // has installed (0: none before it in the queue); GPUTx:
                                 // 1 + the K-set of that write (0: none)
    uint32_t *cursor;            // GaccO: per-segment owner cursor
    const uint32_t *rank_order;  // GPUTx: transactions sorted by rank
    const uint32_t *rank_of;     // GPUTx: rank of each transaction
    uint32_t *rank_done;         // GPUTx: completed count per rank
    const uint32_t *rank_count;  // GPUTx: size of each rank (K-set)
    const uint8_t *skip;         // partitioned TPC-C: 1 = distributed txn, left to phase B
    uint32_t *latch;             // CC_FLAG_LATCHED: one 32-bit latch per control word
    unsigned long long *stages;  // CC_FLAG_STAGES: accumulated cycles per stage (STAGE_*)
    unsigned long long *sticky;  // first device error of any submit since the last cc_sync
    Event *events;               // CC_FLAG_EVENTS: event log (capacity events_cap)
    unsigned long long events_cap;
    unsigned long long *trace;   // GC_TRACE_COMMIT experiment builds only (else null)
};
// stage-time breakdown (Exp-6): cycles summed over workers
enum { STAGE_INDEX = 0, STAGE_TS = 1, STAGE_WAIT = 2, STAGE_CC = 3, STAGE_ABORT = 4,
       STAGE_USEFUL = 5, STAGE_ATTEMPTS = 6, STAGE_WORDS = 8 };

// Cache-line search tree over a sorted key array (same lower-bound result as the
// binary search of PAPER.md:344): the sorted array, padded with ~0 to a multiple of 16,
// is the leaf level; level l+1 holds the last key of every 16-entry node of level l;
// the top level has <= 16 entries.  levels[0] = leaves.
// MVCC history node = header word (begin ts << 32 | previous node) padded to 32 B, then
// the row, so node rows stay 32 B aligned for 256-bit loads
constexpr unsigned ARENA_HDR = 4;
constexpr int IDX_MAX_LEVELS = 10;
// Lookup modes; every mode returns the same lower-bound result for the same index.
// Dense modes (f-3 direct addressing) apply when the keys are k0, k0+1, ..., k0+n-1:
// the position is key - k0, no probe at all; IDX_DENSE_ID also has row id == position.
enum { IDX_TREE = 0, IDX_BINARY = 1, IDX_DENSE = 2, IDX_DENSE_ID = 3, IDX_EYTZ = 4 };
struct TreeIndex {
    const unsigned long long *lv[IDX_MAX_LEVELS];
    unsigned long long len[IDX_MAX_LEVELS];   // padded lengths (multiples of 16)
    int n_levels;
};

// YCSB workload parameters.
struct YcsbParams {
    const uint32_t *keys;        // n_txn*K primary keys
    const uint8_t *ops;          // n_txn*K op bytes: bit7 write, bits 0..3 field
    const unsigned long long *idx_keys;  // sorted-array index
    const unsigned long long *idx_rows;
    unsigned long long idx_n;
    TreeIndex tree;              // same keys, cache-line tree layout (f-3)
    const unsigned long long *eytz_keys;   // same keys in Eytzinger (BFS) order, 1-based,
    const unsigned long long *eytz_rows;   // padded with ~0 to 2^h - 1 entries (f-3)
    unsigned long long eytz_n;             // 2^h - 1
    int mode;                    // IDX_TREE / IDX_BINARY (the paper's) / IDX_DENSE / IDX_DENSE_ID
    unsigned long long idx_k0;   // first key (dense modes)
    unsigned long long *rows;    // 16 x u64 per row
    unsigned long long n_rows;
};

// Deterministic-scheme preprocessing buffers (a3), sized n_acc = n_txn*K.
struct PrepBufs {
    unsigned long long *keys_in, *keys_out;   // (rec << 27) | (gid << 6) | (i << 1) | w
    uint32_t *acc_rec, *acc_seg, *acc_pos, *acc_rdy, *sorted_pos;
    uint32_t *head_flag;   // scan input: p at a segment head, else 0
    uint32_t *lw;          // scan input: p + 1 at a write, else 0
    uint32_t *seg_start;   // per sorted position: first position of its item's segment
    uint32_t *seg_id;      // per sorted position: last write at or before it, + 1 (0: none)
    uint32_t *cursor;
    uint32_t *rank, *rank_sorted, *gid_in, *rank_order, *rank_count, *rank_done, *rank_start;
    void *cub_tmp;
    size_t cub_bytes;
};

// launchers (defined in the .cu files)
// a2 prologue: ring + retry queues (ring_words), control block, per-transaction results,
// then the batch's a1 error word (may be null) folded into the control block
cudaError_t launch_a2(unsigned long long *ring, uint32_t ring_words, Ctl *ctl, uint8_t *committed,
                      uint32_t *restarts, unsigned long long *ohi, unsigned long long *olo, uint32_t n_txn,
                      const unsigned long long *batch_err, cudaStream_t s);
// `smem` bytes of dynamic shared memory: the per-worker contexts (exec_th_bytes() per
// working lane: every lane in tile mode, 2^wd per warp in thread mode), then in thread
// mode the workers' staged accesses unless ExecParams::ws holds them in global memory
cudaError_t launch_ycsb_exec(const ExecParams &p, const YcsbParams &y, int grid, int block, size_t smem,
                             cudaStream_t s);
int ycsb_exec_max_blocks_per_sm(int scheme, int lanes, int block, size_t smem);
size_t ycsb_lane_bytes();
size_t exec_th_bytes();
size_t tpcc_lane_bytes();
cudaError_t launch_ycsb_gather(const ExecParams &p, const YcsbParams &y, PrepBufs &b,
                               cudaStream_t s);
// rank_block: threads per block of the GPUTx rank kernel (256 inline; 1024 on the prep
// stream, so that its few blocks occupy few SMs beside the executor)
cudaError_t launch_prep_common(const ExecParams &p, PrepBufs &b, uint64_t n_records,
                               bool gputx, int grid, cudaStream_t s, int rank_block = 256);
cudaError_t launch_merge_err(const Ctl *src, Ctl *dst, cudaStream_t s);
// a7 commit positions of TO / MVCC / Silo by bitmap (bits: 2^31 / 32 words, pre: one u32
// per word, csum: one per 1,024 words); null: radix sort
struct RankBitmap {
    uint32_t *bits, *pre, *csum;
};
constexpr unsigned long long RANK_BITMAP_BITS = 1ull << 31;   // 31-bit timestamps
cudaError_t launch_finalize(const ExecParams &p, const cc_result &res, PrepBufs &b,
                            bool deterministic, bool two_pass, cudaStream_t s, bool dense_ticket = false,
                            bool lo_dense = false, const RankBitmap *rb = nullptr,
                            uint64_t *stats_mirror = nullptr);   // also written with the stats
size_t prep_cub_bytes(uint64_t n_acc, uint64_t n_txn);
// sort.cu: stable LSD radix sort of u64 keys (+ optional u32 values) on bits [lo, hi),
// keys_alt / vals_alt the ping-pong buffers, n = *n_dev if given (device-resident count,
// cap the host-side capacity that sizes the grids) else cap; *keys_out / *vals_out
// receive whichever buffer holds the result.  gc_scan_max2: inclusive max-scan of two u32
// arrays (out may alias in).
size_t gc_sort_temp_bytes(uint64_t cap);
cudaError_t gc_sort(unsigned long long *keys, uint32_t *vals, unsigned long long *keys_alt, uint32_t *vals_alt,
                    uint64_t cap, const unsigned long long *n_dev, int lo_bit, int hi_bit, void *temp,
                    size_t temp_bytes, cudaStream_t s, unsigned long long **keys_out, uint32_t **vals_out);
size_t gc_scan_temp_bytes(uint64_t n);
cudaError_t gc_scan_max2(const uint32_t *a, const uint32_t *b, uint32_t *oa, uint32_t *ob, uint64_t n, void *temp,
                         size_t temp_bytes, cudaStream_t s);
cudaError_t launch_stages_reduce(unsigned long long *stages, uint64_t n_threads, cudaStream_t s);

struct TpccParams;
cudaError_t launch_tpcc_exec(const ExecParams &p, const TpccParams &y, int grid, int block, size_t smem,
                             cudaStream_t s);
int tpcc_exec_max_blocks_per_sm(int scheme, int lanes, int block, size_t smem);
cudaError_t launch_tpcc_gather(const ExecParams &p, const TpccParams &y, PrepBufs &b,
                               uint64_t n_records, cudaStream_t s);
cudaError_t launch_tpcc_pop(int table, unsigned long long *rows, unsigned long long first,
                            unsigned long long n, unsigned long long seed, uint32_t c_load,
                            cudaStream_t s);
cudaError_t build_name_index(const unsigned long long *cu, uint32_t n_cust,
                             unsigned long long first_row, unsigned long long seed,
                             uint32_t c_load, uint32_t *idx_start, uint32_t *idx_count,
                             uint32_t *idx_rows, uint32_t n_groups, cudaStream_t s);
cudaError_t launch_tpcc_gen(uint32_t *tx, uint32_t n_txn, unsigned long long seed, uint32_t W,
                            uint32_t w_lo, uint32_t w_hi, uint32_t no_pm, uint32_t c_last_run,
                            uint32_t c_id_c, uint32_t c_item_c, unsigned long long *err, cudaStream_t s);

struct PartReq;
struct PartResp;
cudaError_t part_classify_pack(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr,
                               uint32_t n_txn, uint8_t *skip, unsigned long long *cnt,
                               unsigned long long *off, unsigned long long *cursor, PartReq *out,
                               cudaStream_t s);
cudaError_t part_apply(PartReq *req, uint64_t n, const TpccParams &y, PartResp *resp,
                       unsigned long long *k1, unsigned long long *k2, uint32_t *i1, uint32_t *i2,
                       void *tmp, size_t tmp_bytes, Ctl *ctl, cudaStream_t s);
size_t part_sort_bytes(uint64_t n);
cudaError_t part_finish(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr,
                        uint32_t n_txn, const uint8_t *skip, const PartReq *sent,
                        const PartResp *resp, uint64_t n_sent, PartResp *stage,
                        uint8_t *committed, unsigned long long *ohi, unsigned long long *olo,
                        unsigned long long *read_out, cudaStream_t s, bool two_pc = false);
// 2PC phase B (f-2): prepare/grant on the owner, decide on the home, commit on the owner,
// repack the pending transactions for the next round
cudaError_t part_grant(PartReq *req, uint64_t n, const TpccParams &y, PartResp *resp, uint8_t *vote,
                       unsigned long long *k1, unsigned long long *k2, uint32_t *i1, uint32_t *i2,
                       void *tmp, size_t tmp_bytes, Ctl *ctl, cudaStream_t s, bool ts_rule = false);
cudaError_t part_decide(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr, uint32_t n_txn,
                        uint8_t *skip, const PartReq *sent, const PartResp *resp, uint64_t n_sent,
                        PartResp *stage, uint8_t *committed, unsigned long long *ohi,
                        unsigned long long *olo, unsigned long long *read_out, uint32_t *restarts,
                        uint32_t round, unsigned long long *dec, cudaStream_t s);
cudaError_t part_commit(const PartReq *req, uint64_t n, const uint8_t *vote, const unsigned long long *dec,
                        const TpccParams &y, cudaStream_t s);
// CC_FLAG_PART_P2P (part.cu): window layout [flags | inbox world x cap | staging max_txn x K]
struct PeerTab;
size_t p2p_window_bytes(uint32_t world, uint32_t cap, uint32_t max_txn);
cudaError_t p2p_send(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr, uint32_t n_txn, uint8_t *skip,
                     unsigned long long *cnt, unsigned long long *cursor, const PeerTab &pt, uint32_t cap,
                     unsigned long long epoch, Ctl *ctl, bool all, cudaStream_t s);
cudaError_t p2p_phase_b(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr, uint32_t n_txn,
                        const uint8_t *skip, const PeerTab &pt, uint32_t cap, unsigned long long epoch,
                        unsigned long long *rc, PartReq *recv, unsigned long long *k1, unsigned long long *k2,
                        uint32_t *i1, uint32_t *i2, void *tmp, size_t tmp_bytes, uint8_t *committed,
                        unsigned long long *ohi, unsigned long long *olo, unsigned long long *read_out, Ctl *ctl,
                        unsigned long long watchdog_ns, cudaStream_t s);
cudaError_t part_repack(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr, uint32_t n_txn,
                        const uint8_t *skip, unsigned long long *cnt, unsigned long long *off,
                        unsigned long long *cursor, PartReq *out, cudaStream_t s);

cudaError_t launch_ycsb_init_rows(unsigned long long *rows, uint64_t first, uint64_t n,
                                  uint64_t seed, cudaStream_t s);
cudaError_t launch_identity_index(unsigned long long *keys, unsigned long long *rows,
                                  uint64_t n, cudaStream_t s);
cudaError_t launch_eytz_build(const unsigned long long *keys, const unsigned long long *rows, uint64_t n,
                              int h, unsigned long long *ekeys, unsigned long long *erows, cudaStream_t s);
cudaError_t launch_tree_level(const unsigned long long *in, uint64_t n_in, unsigned long long *out,
                              uint64_t n_out_padded, cudaStream_t s);
cudaError_t launch_index_lookup(const YcsbParams &y, const unsigned long long *keys, uint64_t n,
                                unsigned long long *out, cudaStream_t s);
cudaError_t launch_fill_u64(unsigned long long *p, unsigned long long v, uint64_t n, cudaStream_t s);
// zero `words` u64 words (background a2 of a used CC word set): evict-first stores
cudaError_t launch_zero_words(unsigned long long *p, uint64_t words, cudaStream_t s);
cudaError_t launch_ycsb_gen(uint32_t *keys, uint8_t *ops, uint32_t n_txn, uint32_t K,
                            uint64_t n_rows, double W, uint64_t seed,
                            const unsigned long long *T, uint64_t mult, unsigned long long *err,
                            cudaStream_t s);

// roof.cu: out = {gather GB/s, CAS/s L2-resident, CAS/s > L2, hand-off ns (row), hop ns,
//                 hand-off ns (row, acquire polls)}
cudaError_t roofline_probe(cudaStream_t s, int num_sms, double out[6]);
// roof.cu: GB/s of random 32 / 64 / 128 / 256 B reads over 1 GiB
cudaError_t gather_sweep(cudaStream_t s, int num_sms, double out[4]);

// load every kernel of the library now (lazy module loading may otherwise synchronise the
// context at a first launch while kernels of this process wait on each other)
void preload_prep_kernels();
void preload_sort_kernels();
void preload_part_kernels();
void preload_tpcc_kernels();
void preload_ycsb_kernels();

}  // namespace gcctb
