/*
 * gcctb.h -- C ABI of the B200-native batched-OLTP concurrency-control library
 * (libgcctb.so).  Re-designs the hot path measured by the gCCTB testbed of
 * "GPU-Accelerated OLTP: An In-Depth Analysis of Concurrency Control Schemes"
 * (arXiv 2406.10158).  Citations are PAPER.md / SPEC.md line numbers.
 *
 * Problem statement: tables and indexes are resident in device
 * memory; transactions consist only of reads and writes whose read/write sets are
 * known before execution; a batch is executed with one worker per transaction under
 * one concurrency-control (CC) scheme until every transaction commits; results stay
 * in device memory.
 *
 * Conventions for every entry point:
 *   - Plain C types only; every call returns cc_status; no C++ exception crosses the ABI.
 *   - Argument / configuration errors return before anything is enqueued.
 *   - Device work is asynchronous on the db's stream.  Asynchronous faults (a CUDA
 *     error, the device watchdog, timestamp overflow) surface at the next cc_sync() /
 *     cc_submit(); after a CUDA fault the db is sticky-failed (CC_ERR_STATE).
 *   - Ownership: the db owns every device allocation it makes (tables, indexes, CC
 *     metadata, version arena, queues, batches).  The caller owns result buffers and
 *     any host / device source buffers it passes in (they are read before return for
 *     host sources, or before the next stream operation completes for device sources).
 *   - A db is not re-entrant: one host thread at a time.
 *   - cc_last_error(db) returns a message for the last failing call (valid until the
 *     next call on that db).
 */
#ifndef GCCTB_H
#define GCCTB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CC_OK = 0,
    CC_ERR_INVALID_ARG = 1,
    CC_ERR_CONFIG = 2,            /* ConfigError */
    CC_ERR_OOM = 3,
    CC_ERR_CUDA = 4,
    CC_ERR_NCCL = 5,
    CC_ERR_KEY_NOT_FOUND = 6,     /* KeyNotFound */
    CC_ERR_TS_OVERFLOW = 7,       /* TimestampOverflow at 2^31-1 */
    CC_ERR_VERSION_EXHAUSTED = 8, /* VersionExhausted */
    CC_ERR_WATCHDOG = 9,          /* WatchdogTimeout */
    CC_ERR_STATE = 10,            /* sticky after a device fault */
    CC_ERR_UNSUPPORTED = 11
} cc_status;

/* The eight schemes of PAPER.md Table I. */
typedef enum {
    CC_TPL_NW = 0,  /* 2PL no-wait */
    CC_TPL_WD = 1,  /* 2PL wait-die */
    CC_TO = 2,      /* basic timestamp ordering */
    CC_MVCC = 3,    /* multi-version TO */
    CC_SILO = 4,    /* OCC */
    CC_TICTOC = 5,  /* OCC */
    CC_GPUTX = 6,   /* conflict-graph ranks / K-sets */
    CC_GACCO = 7    /* preprocessed lock table */
} cc_scheme;

#define CC_NUM_SCHEMES 8

typedef struct cc_db_s *cc_db;
typedef struct cc_batch_s *cc_batch;

/* ---------------------------------------------------------------- db lifetime */
typedef struct {
    int device;        /* CUDA device ordinal */
    void *stream;      /* cudaStream_t to run on; NULL = the library creates one */
    int rank;          /* partition id of this process (0 for a single GPU) */
    int world;         /* number of partitions (1 for a single GPU) */
} cc_db_desc;

/* Create a db bound to (device, stream).  *out receives the handle. */
cc_status cc_db_create(const cc_db_desc *desc, cc_db *out);
/* Free every device allocation of the db (waits for its stream first). */
cc_status cc_db_destroy(cc_db db);
/* Message of the last failing call on db (never NULL; "" when none). */
const char *cc_last_error(cc_db db);
/* Library build string (arch, version).  Never NULL. */
const char *cc_version(void);

/* ------------------------------------------------------- tables and indexes
 * Row store: one fixed-size array of tuples per table; all CC-managed tables share
 * one monotonically increasing record id space.
 * Table size is fixed for the life of the db (no insert/delete). */

/* Create a table of `rows` rows of `row_bytes` bytes (multiple of 8), zero-filled.
 * *table_id receives its id.  Errors: INVALID_ARG (row_bytes==0 or not a multiple of
 * 8, rows==0), OOM. */
cc_status cc_table_create(cc_db db, const char *name, uint32_t row_bytes, uint64_t rows,
                          uint32_t *table_id);
/* Copy n rows from src (host if src_on_device==0, else device) into rows
 * [first_row, first_row+n).  Synchronous for host sources. */
cc_status cc_table_load(cc_db db, uint32_t table_id, uint64_t first_row, uint64_t n,
                        const void *src, int src_on_device);
/* Copy rows [first_row, first_row+n) to dst (host or device).  Waits for the db
 * stream, so it observes every submitted batch. */
cc_status cc_table_read(cc_db db, uint32_t table_id, uint64_t first_row, uint64_t n,
                        void *dst, int dst_on_device);
/* Number of rows / row bytes of a table. */
cc_status cc_table_info(cc_db db, uint32_t table_id, uint64_t *rows, uint32_t *row_bytes);

/* Sorted-array index over table_id: sorted_keys[i] strictly ascending,
 * row_ids[i] < rows(table).  A lookup returns the lower-bound match of the paper's binary
 * search; when the keys form a dense range k0..k0+n-1 it is resolved by
 * direct addressing (no probe), else by a cache-line search tree over the same sorted
 * array; CC_FLAG_INDEX_BINARY / CC_FLAG_INDEX_TREE /
 * CC_FLAG_INDEX_EYTZ force a method (the Eytzinger copy of the keys and row ids is built
 * with the index: 2 x 2^ceil(log2(n+1)) u64).
 * INVALID_ARG unless strictly ascending.  *index_id receives the id. */
cc_status cc_index_create(cc_db db, uint32_t table_id, const uint64_t *sorted_keys,
                          const uint64_t *row_ids, uint64_t n, int src_on_device,
                          uint32_t *index_id);

/* Batch index lookup (SPEC.md:47 index_lookup): rows_out[i] = row id of keys[i], or
 * 2^64-1 when the key is absent (KeyNotFound).  keys / rows_out are device
 * arrays of n u64 (caller-owned).  flags: CC_FLAG_INDEX_BINARY selects the paper's
 * binary search, CC_FLAG_INDEX_TREE the cache-line tree, CC_FLAG_INDEX_EYTZ the
 * Eytzinger layout, otherwise direct addressing on
 * a dense key range and the tree elsewhere; results are identical.  Async. */
cc_status cc_index_lookup(cc_db db, uint32_t index_id, const uint64_t *keys, uint64_t n,
                          uint64_t *rows_out, uint32_t flags);

/* ----------------------------------------------------------------- YCSB
 * YCSB table: n_rows rows of 16 x u64 (128 B); word j of row k is
 * mix64(seed ^ (16k + j)) for j < 15 and word 15 (a write counter) is 0, where mix64
 * is the splitmix64 finaliser (reading Z11).  Creates table "usertable" and
 * its primary-key index (key k -> row k), generated on the device. */
typedef struct {
    uint64_t n_rows;
    uint64_t seed;
} cc_ycsb_db_desc;
cc_status cc_load_ycsb(cc_db db, const cc_ycsb_db_desc *desc);

/* On-device YCSB batch generator.
 * A device-side generator failure (a transaction whose distinct keys could not be drawn:
 * CONFIG) is recorded in the batch itself; every cc_submit of the batch then executes
 * nothing and cc_sync returns CONFIG.  STATE while a partitioned submit is pending.
 * thresholds: u64[n_rows] Zipf inverse-CDF table (see inputs/ycsb.py), host or device
 * per thresholds_on_device; it is read during the call (device) or copied (host).
 * Key = ((rank-1) * scramble_mult) mod n_rows; duplicates within a transaction are
 * resampled; each transaction's keys are sorted ascending; each access writes with
 * probability write_frac; field in [0, 15). */
typedef struct {
    uint32_t n_txn;
    uint32_t ops_per_txn;      /* K, 1..16 */
    double write_frac;         /* W in [0, 1] */
    uint64_t seed;
    const uint64_t *thresholds;
    int thresholds_on_device;
    uint64_t scramble_mult;    /* must be coprime with n_rows */
} cc_ycsb_gen_desc;
cc_status cc_batch_gen_ycsb(cc_db db, const cc_ycsb_gen_desc *g, cc_batch *out);

/* Import a YCSB-form batch: keys u32[n_txn*K] (primary keys of "usertable", sorted
 * ascending and distinct within each transaction), ops u8[n_txn*K] (bit7 = write,
 * bits 0..3 = field < 15).  KEY_NOT_FOUND surfaces at submit for unknown keys.
 * src_on_device: 0 host buffers, copied before return; 1 device buffers;
 * CC_SRC_HOST_ASYNC (2) host buffers (pinned for a true overlap) copied on the db's copy
 * stream without waiting, so the transfer overlaps work already queued on the db stream;
 * the caller keeps them unchanged until the first cc_submit of the batch has completed
 * (cc_sync).  Submits of the batch wait for its copy on the device. */
#define CC_SRC_HOST_ASYNC 2
cc_status cc_batch_import_ycsb(cc_db db, const uint32_t *keys, const uint8_t *ops,
                               uint32_t n_txn, uint32_t ops_per_txn, int src_on_device,
                               cc_batch *out);
/* Export a YCSB batch to host buffers (keys u32[n*K], ops u8[n*K]). */
cc_status cc_batch_export_ycsb(cc_db db, cc_batch b, uint32_t *keys, uint8_t *ops);
/* Batch geometry. */
cc_status cc_batch_info(cc_db db, cc_batch b, uint32_t *n_txn, uint32_t *ops_per_txn,
                        uint32_t *kind);
/* Release a batch.  Its device buffers (and any buffers cc_prepare attached to it) go to
 * a per-db pool and are reused, in stream order, by the next batch of the same kind and
 * shape, so that a steady stream of batches makes no cudaMalloc / cudaFree calls (each is
 * an implicit device synchronisation).  Never blocks the host: the reuse waits on the
 * device for the old batch's readers (db stream, and the prep stream via an event).  The
 * handle is invalid afterwards (it may come back from a later gen / import).  STATE for
 * the batch of a pending partitioned submit.  cc_pool_trim / cc_db_destroy free the pool. */
cc_status cc_batch_free(cc_db db, cc_batch b);
/* Free the pooled buffers of released batches (waits for the db's streams). */
cc_status cc_pool_trim(cc_db db);
/* Process-wide counters of the driver's device allocations: number of cudaMalloc and
 * cudaFree calls and bytes allocated since the library was loaded (any pointer may be
 * NULL).  A steady batch loop (gen / prepare / submit / free) leaves the first two
 * unchanged once the pool holds its batches (bench.py asserts it over the timed region). */
cc_status cc_mem_stats(cc_db db, uint64_t *n_allocs, uint64_t *n_frees, uint64_t *bytes_allocated);

/* ----------------------------------------------------------------- TPC-C
 * TPC-C NewOrder + Payment.  Creates, in this order, the CC-managed
 * tables WAREHOUSE, DISTRICT, CUSTOMER, STOCK for warehouses [w_first, w_first+w_count)
 * of `warehouses` (record ids consecutive), the immutable ITEM table
 * (outside CC, Z16), the reserved-slot tables ORDER, NEW_ORDER, ORDER_LINE (15 per
 * transaction), HISTORY for max_txn transactions (inserts become private slot writes,
 * Z15), and the immutable customer last-name index.  Population per TPC-C §4.3.3 from
 * `seed` (row layouts: inputs/tpcc.py), generated on the device. */
typedef struct {
    uint32_t warehouses;   /* total W */
    uint32_t w_first;      /* first warehouse held by this db (partitioning), 0 for 1 GPU */
    uint32_t w_count;      /* warehouses held (w_count = warehouses for 1 GPU) */
    uint32_t max_txn;      /* capacity of the reserved-slot tables */
    uint64_t seed;
} cc_tpcc_db_desc;
cc_status cc_load_tpcc(cc_db db, const cc_tpcc_db_desc *desc);

/* Table ids of the TPC-C tables: ids[0..8] = W, D, C, S, I, O, NO, OL, H. */
cc_status cc_tpcc_tables(cc_db db, uint32_t ids[9]);

/* On-device TPC-C generator: NewOrder with probability
 * neworder_permyriad/10,000 (else Payment), home warehouse uniform in [w_lo, w_hi),
 * TPC-C §2.4.1 / §2.5.1 inputs (NURand customers/items/last names, 1% remote supply,
 * 15% remote Payment, 60% by name), NewOrder lines distinct and sorted by stock key.
 * Transaction descriptors are 40 x u32. */
typedef struct {
    uint32_t n_txn;
    uint32_t neworder_permyriad;
    uint64_t seed;
    uint32_t w_lo, w_hi;
} cc_tpcc_gen_desc;
cc_status cc_batch_gen_tpcc(cc_db db, const cc_tpcc_gen_desc *g, cc_batch *out);
/* Import / export TPC-C descriptors (u32[n_txn*40]). */
cc_status cc_batch_import_tpcc(cc_db db, const uint32_t *tx, uint32_t n_txn, int src_on_device,
                               cc_batch *out);
cc_status cc_batch_export_tpcc(cc_db db, cc_batch b, uint32_t *tx);

/* ------------------------------------------------------------ execution */
#define CC_FLAG_IMMEDIATE_RETRY 0x1u /* paper mode: the worker re-runs its own aborted
                                        transaction at once instead of
                                        appending it to the retry queue */
#define CC_FLAG_TIMING 0x2u          /* record CUDA events around each phase; read them
                                        with cc_timing_read() */
#define CC_FLAG_PARTITIONED 0x4u     /* TPC-C over warehouse partitions (a8): cc_submit runs
                                        phase A (local transactions, chosen scheme) and
                                        packs phase-B requests; finish with cc_part_send /
                                        cc_part_apply / cc_part_finish */
#define CC_FLAG_PART_ALL 0x8u        /* as PARTITIONED, but every transaction takes phase B
                                        (exercises phase B on one partition) */
#define CC_FLAG_LATCHED 0x20u        /* Exp-7: every control-word mutation
                                        under a 32-bit per-word latch instead of one 64-bit CAS */
#define CC_FLAG_STAGES 0x40u         /* Exp-6: per-stage cycle
                                        accounting into cc_stats.stage_cycles */
#define CC_FLAG_EVENTS 0x80u         /* debug event log: every row read / install
                                        and every commit / abort gets a global sequence number;
                                        read it with cc_events_read (capacity: cc_events_capacity) */
#define CC_FLAG_INDEX_BINARY 0x10u   /* index lookups by plain binary search over the sorted
                                        array (the paper's index) instead of the
                                        default cache-line search tree over the same array
                                        (identical results) */
#define CC_FLAG_FLAT_JITTER 0x200u   /* ablation: after waiting out a conflicting lock, retry
                                        with a flat 0..255 ns jitter instead of a window that
                                        doubles per restart (retry pacing) */
#define CC_FLAG_PART_2PC 0x800u      /* with CC_FLAG_PARTITIONED, the six non-deterministic
                                        schemes: distributed transactions in 2PC rounds under
                                        the scheme's round rule (cc_part_decide /
                                        cc_part_commit / cc_part_next, f-2) */
#define CC_FLAG_MVCC_SPLIT 0x400u    /* MVCC metadata layout ablation (PAPER.md:636
                                        attributes MVCC's gap to TO to its timestamps and version
                                        pointers being interleaved): the timestamp words in one
                                        dense array and the version-pointer words in another,
                                        instead of Table II's interleaved 16 B per record */
#define CC_FLAG_INDEX_TREE 0x100u    /* force the cache-line search tree even on a dense key
                                        range (default there: direct addressing, key - k0) */
#define CC_FLAG_WARM 0x2000u        /* tile mode, YCSB, the six non-deterministic schemes:
                                        before a transaction's first attempt every lane waits
                                        until its prefetched row and control word have
                                        reached L2 (one load per 32 B sector), so a lock /
                                        pending write is held across L2 latencies only, not
                                        across its cold rows' HBM misses.  Same results. */
#define CC_FLAG_META_PAD 0x10000u    /* single-word schemes: one control word per 32 B sector instead of
                                        packed 8 B words (the north star's metadata padded against
                                        false sharing in L2).  Same results;
                                        measured per workload */
#define CC_FLAG_L2_PERSIST 0x8000u   /* ablation: an L2 access-policy window (persisting) over the
                                        control words during the executor; reserves the device's
                                        persisting L2 set-aside on first use (measured
                                        slower on the bench).  Same results */
#define CC_FLAG_PART_P2P 0x4000u     /* with CC_FLAG_PARTITIONED (deterministic phase B): the exchange
                                        runs inside the library over peer memory -- requests and
                                        responses are stored straight into the peers' exchange
                                        windows, published by system-scope release flags -- so the
                                        submit enqueues phase A, phase B and a7 on the db stream and
                                        completes without the host (cc_part_window / connect) */
#define CC_FLAG_INDEX_EYTZ 0x1000u   /* index lookups in the Eytzinger (BFS) layout of the same
                                        sorted keys: a branch-free
                                        descent over a complete binary tree padded to 2^h - 1
                                        keys; same lower-bound result as the binary search */

typedef struct {
    cc_scheme scheme;
    uint32_t wd;            /* warp density: 2^wd working lanes per warp, 0..5 */
    uint32_t bs;            /* block size: warps per block, 1..32 */
    uint32_t flags;         /* CC_FLAG_* */
    uint32_t grid;          /* blocks; 0 = resident capacity (persistent grid) */
    uint32_t lanes_per_txn; /* 0/1: one lane per transaction (the paper's model, wd and bs
                               apply); 4/8/16/32: a tile of that many lanes runs one
                               transaction, lane i owning access i (must be >= ops per
                               transaction; wd is ignored; 32 gives every transaction a
                               warp of its own).  TPC-C batches use 32-lane
                               tiles for any value > 1 */
    double watchdog_s;      /* device watchdog in seconds (0 = 30 s) */
    uint32_t claim_chunk;   /* fresh transaction ids a worker claims per atomic (0 = 1) */
} cc_exec_desc;

/* Per-transaction results, owned by the caller: all DEVICE pointers, or all HOST pointers
 * (a mix is INVALID_ARG).  Host buffers are filled by copies the submit enqueues at its end
 * from library-owned device staging (pinned memory: asynchronous, complete at cc_sync;
 * pageable memory: the copy waits for the submit); a host-driven partitioned submit
 * (CC_FLAG_PARTITIONED without CC_FLAG_PART_P2P) takes device buffers only (UNSUPPORTED).
 * Any may be NULL except committed.  n = n_txn of the batch, K = ops_per_txn.
 *   committed u8[n]   1 iff the transaction committed
 *   restarts  u32[n]  number of aborted attempts
 *   order_hi/lo u64[n] the scheme's serialization-order key;
 *                     ascending (hi, lo) is a valid serial order of the committed set
 *   commit_pos u32[n] dense position of the transaction in that order
 *   read_out  u64[n*K] per-op value read (YCSB: fingerprint of the row read);
 *             TPC-C: u64[n*48] per transaction (NewOrder: o_id, total, then per line
 *             s_quantity before, 'B'/'G', ol_amount; Payment: c_id, c_balance, c_credit)
 *   stats     u64[CC_STATS_WORDS] device counters (see cc_stats)               */
#define CC_STATS_WORDS 16
typedef struct {
    uint8_t *committed;
    uint32_t *restarts;
    uint64_t *order_hi;
    uint64_t *order_lo;
    uint32_t *commit_pos;
    uint64_t *read_out;
    uint64_t *stats;
} cc_result;

/* Host view of the stats words. */
typedef struct {
    uint64_t commits;       /* committed transactions */
    uint64_t aborts;        /* sum of restarts (abort rate = aborts / commits) */
    uint64_t attempts;
    uint64_t error;         /* device-side cc_status (0 = ok) */
    uint64_t max_rank;      /* GPUTx: number of K-sets - 1 */
    uint64_t ts_last;       /* TO/MVCC: last timestamp drawn */
    uint64_t reserved[2];
    /* CC_FLAG_STAGES: SM cycles summed over workers (tile mode: each tile's leader lane):
     * [0] index lookup  [1] timestamp allocation  [2] waiting  [3] CC manager (rest of
     * committed attempts)  [4] aborted attempts minus their ts allocation, plus retry
     * pacing  [5] useful row work  [6] attempts.  Preprocessing time is the a3 phase of
     * cc_timing_read. */
    uint64_t stage_cycles[7];
    uint64_t sm_clock_khz;  /* nominal SM clock, to convert cycles */
} cc_stats;

/* Run batch b under desc->scheme: reset the scheme's CC state (a2), preprocess
 * (GPUTx/GaccO, a3), execute with compaction of aborts into a retry queue until every
 * transaction commits (a4-a6), then emit results (a7).  Asynchronous on the db stream.
 * a2 (reading Z19): the db keeps two sets of control words, all zeros in
 * the initial state of every scheme; a submit executes on a clean set and, once its
 * executor is done, the set is zeroed on a background (reset) stream while the next
 * submit runs on the other set (a partitioned submit zeroes its set in stream before the
 * set's next use instead).  The db stream waits for that zeroing only when the set is
 * reused; cc_join / cc_sync cover it. */
cc_status cc_submit(cc_db db, cc_batch b, const cc_exec_desc *desc, const cc_result *res);

/* Pipelined preprocessing (GaccO's preprocessing
 * can be pipelined with execution).  Runs a3 of `scheme` -- GPUTx K-set ranks or GaccO
 * queue positions -- for batch b on the db's second (preprocessing) stream into buffers
 * owned by b, waiting only for b's own generation / import, so it overlaps whatever the
 * main stream is executing (e.g. the previous batch).  The next cc_submit of b with the
 * same scheme consumes it and skips a3 (results identical to an inline a3); one
 * cc_prepare feeds one submit.  flags: the CC_FLAG_INDEX_* bits.  Other schemes: no-op.
 * Partitioned submits ignore it (their access sets depend on the per-submit phase split)
 * and prepare inline.  Errors raised during the preparation (e.g. KEY_NOT_FOUND) surface
 * at the consuming submit's cc_sync.  Asynchronous.  INVALID_ARG for an unknown batch,
 * STATE while a partitioned submit is pending. */
cc_status cc_prepare(cc_db db, cc_batch b, cc_scheme scheme, uint32_t flags);
/* ------------------------------------------- partitioned TPC-C (a8)
 * Rank r of `world` (cc_db_desc) holds warehouses [r*W/world, (r+1)*W/world).  After a
 * cc_submit with CC_FLAG_PARTITIONED:
 *   cc_part_send   waits, returns the device buffer of phase-B requests (48-byte records,
 *                  grouped by destination rank in rank order) and counts[world] on the host;
 *   -- the caller exchanges requests with an all-to-all (NCCL via torch.distributed) --
 *   cc_part_apply  applies n received requests (device) on the items this rank owns: per
 *                  item, in global transaction order (every TPC-C write is a
 *                  read-modify-write of one item), writing n 48-byte responses (device, same
 *                  order as received);
 *   -- the caller returns responses with the reverse all-to-all --
 *   cc_part_finish takes the responses aligned with this rank's send buffer, assembles the
 *                  outputs and reserved slots of its distributed transactions and completes
 *                  the submit (a7).  Order keys: phase A (rank << 48 | scheme key, key_lo),
 *                  phase B (1 << 63, global gid = rank * n_txn + gid).
 * Buffers passed in are caller-owned device memory. */
cc_status cc_part_send(cc_db db, const void **send, uint64_t *counts);
cc_status cc_part_apply(cc_db db, void *recv, uint64_t n, void *resp);
cc_status cc_part_finish(cc_db db, const void *resp, uint64_t n_sent);

/* Scheme-native phase B (cc_submit with CC_FLAG_PARTITIONED |
 * CC_FLAG_PART_2PC, the six non-deterministic schemes; GPUTx / GaccO are deterministic and
 * keep the gid-ordered chains): the distributed transactions run in two-phase-commit rounds
 * instead of the deterministic chains.  Per round, every rank (collectively):
 *   cc_part_send    requests of its pending distributed transactions, as above;
 *   -- all-to-all #1 --
 *   cc_part_apply   PREPARE: the owner grants the round's requests item by item in global
 *                   transaction order, no-wait, and answers with the values read and the
 *                   vote in word 5 of each response.  2PL: shared unless an exclusive was
 *                   granted, exclusive only on a free item.  TO / MVCC / Silo / TicToc,
 *                   with the round's timestamps ts = (round, global gid): an access is
 *                   granted unless an earlier write to the item was granted this round
 *                   (TO: a read or write behind a pending older write waits -- here:
 *                   retries next round; a write behind granted older reads is in
 *                   timestamp order; OCC: the first writer takes the write lock, a read
 *                   behind it would fail validation);
 *   -- reverse all-to-all #2 --
 *   cc_part_decide  DECIDE on the home: a transaction commits iff every access was granted;
 *                   committed ones are assembled with order key (1 << 63 | round, global
 *                   gid), aborted ones count a restart; *dec = device buffer of n_sent u64
 *                   decisions (1 commit / 0 abort) aligned with this round's send buffer;
 *   -- all-to-all #3 of the decisions, same counts as #1 --
 *   cc_part_commit  COMMIT on the owner: n decisions aligned with the `recv` buffer given
 *                   to this round's cc_part_apply (kept alive by the caller); installs the
 *                   granted writes of committed transactions;
 *   cc_part_next    packs the still-pending transactions for the next round and returns
 *                   their number (waits).  Loop while any rank has pending transactions
 *                   (the oldest pending transaction is granted everything it asks for, so
 *                   every round commits at least one); then cc_part_finish(db, NULL, 0).
 * STATE outside a 2PC partitioned submit; UNSUPPORTED (at cc_submit) for other schemes. */
cc_status cc_part_decide(cc_db db, const void *resp, uint64_t n_sent, const void **dec);
cc_status cc_part_commit(cc_db db, const void *recv, const void *dec, uint64_t n);
cc_status cc_part_next(cc_db db, uint64_t *pending);

/* In-library exchange over peer memory (CC_FLAG_PART_P2P; the north
 * star's "all-to-all exchange of remote accesses over NVLink each round", fused with the
 * kernels that produce and consume it).  Each rank's db owns an exchange window in device
 * memory: system-scope flags, an inbox of cap request slots per source rank (cap =
 * max_txn x 18 accesses: a source can never overflow it) and the staging array of its own
 * transactions' phase-B responses.  A partitioned submit with CC_FLAG_PART_P2P then runs on
 * the db stream, with no host synchronisation and no collective call:
 *   pack + send    requests are stored by the pack kernel straight into the owners'
 *                  inboxes (NVLink stores to a peer GPU), then one release flag per owner
 *                  carries (epoch, count);
 *   phase A        the local transactions under the scheme (as without P2P);
 *   receive        wait for every source's flag of this epoch, compact, sort by (item, gid);
 *   apply + reply  each item's chain in global gid order, every response stored straight
 *                  into its home's staging array, then one release flag per home;
 *   finish         wait for every owner's flag, assemble, a7.
 * Results are those of cc_part_send / apply / finish (the same phase-B kernels decide what
 * is applied and returned).  All ranks must issue the same sequence of P2P submits.
 *   cc_part_window   allocates this db's window (TPC-C must be loaded; world from
 *                    cc_db_desc) and returns its handle: a CUDA IPC handle plus the shape;
 *   cc_part_connect  maps the windows of all ranks, handles[world] indexed by rank (as
 *                    gathered by the caller, e.g. all_gather over torch.distributed);
 *   cc_part_connect_local  the same for `n` dbs of this process (ranks 0..n-1, one GPU or
 *                    several with peer access), by plain device pointers.
 * Errors: CONFIG (shapes differ, > 64 ranks), STATE (already connected), CUDA (IPC). */
typedef struct {
    unsigned char ipc[64];   /* cudaIpcMemHandle_t of the window */
    uint32_t rank, world, cap, max_txn;
} cc_ipc_handle;
cc_status cc_part_window(cc_db db, cc_ipc_handle *out);
cc_status cc_part_connect(cc_db db, const cc_ipc_handle *handles);
cc_status cc_part_connect_local(cc_db *dbs, int n);

/* Debug event log (CC_FLAG_EVENTS).  Each event is 24 bytes: u64 seq, u32 gid,
 * u32 record (global id; 0xFFFFFFFF for commit/abort), u32 attempt, u32 kind (0 read,
 * 1 write/install, 2 commit, 3 abort).  cc_events_capacity allocates room for `cap`
 * events; cc_events_read waits, copies min(n, cap) events of the last submit to host
 * memory and returns the number recorded (larger than cap means overflow). */
cc_status cc_events_capacity(cc_db db, uint64_t cap);
cc_status cc_events_read(cc_db db, void *dst, uint64_t cap, uint64_t *n_events);

/* Make the db stream wait (on the device; the host does not block) for the library's
 * background work enqueued so far: the zeroing of the CC words a submit used, which runs
 * on a reset stream beside the next submit (the a2 of PAPER.md:472, Z19, off the critical
 * path).  A CUDA event recorded on the db stream after cc_join covers all of it -- what a
 * caller timing a sequence of submits wants.  Submits order themselves; cc_sync waits for
 * everything.  CUDA on a launch error. */
cc_status cc_join(cc_db db);

/* Wait for the db stream; surface asynchronous errors -- the first device error of any
 * submit since the previous cc_sync (sticky across submits); if st != NULL copy the stats
 * of the last submit into it. */
cc_status cc_sync(cc_db db, cc_stats *st);

/* Phase timing (CC_FLAG_TIMING): accumulated milliseconds per phase over the submits
 * since the last reset: ms[0]=reset(a2) ms[1]=prep(a3) ms[2]=exec(a4-a6)
 * ms[3]=emit(a7) ms[4]=whole submit; *n_submits receives the count.  Waits for the
 * stream.  reset != 0 clears the accumulators. */
cc_status cc_timing_read(cc_db db, double ms[5], uint64_t *n_submits, int reset);

/* Device-side snapshot of every table's bytes: save=1 copies tables -> snapshot,
 * save=0 restores.  Used to reset the db between measurement repetitions. */
cc_status cc_snapshot(cc_db db, int save);

/* Memory-system ceilings for the roofline fractions (SURVEY.md §8(d) "Which roofline
 * bounds the path"; the north star's "achieved fraction of the HBM/L2-atomic roofline").
 * Runs three microbenchmarks on the db stream and waits for them:
 *   gather_gbs      random 128 B line reads (the row read of every access) over 1 GiB;
 *   cas_l2_per_s    64-bit CAS on distinct random words of an L2-resident 16 MiB array;
 *   cas_hbm_per_s   the same over 256 MiB (larger than L2, like the CC words at configs[1]);
 *   handoff_row_ns  one hop of a token passed around one warp per SM: relaxed poll,
 *                   acquire, 128 B row read, 2-word install, release -- the per-record
 *                   hand-off that serialises conflicting accesses (GaccO queue, lock
 *                   release -> next acquire);
 *   handoff_ns      the bare token hop (poll + release) without the row;
 *   handoff_acq_row_ns  handoff_row_ns with ld.acquire polls instead of relaxed polls
 *                   followed by one fence.acq_rel (the executor's wait idiom).
 * Allocates ~1.3 GiB of scratch for the call and frees it.  A hand-off figure of -1
 * means the ring timed out (blocks not co-resident).  Errors: INVALID_ARG (null),
 * OOM, CUDA. */
typedef struct {
    double gather_gbs;
    double cas_l2_per_s;
    double cas_hbm_per_s;
    double handoff_row_ns;
    double handoff_ns;
    double handoff_acq_row_ns;
} cc_roofline;
cc_status cc_roofline_probe(cc_db db, cc_roofline *out);
/* Access-size sweep of the gather ceiling (check the 128 B figure against
 * other sizes and ncu): GB/s of random, size-aligned reads of 32, 64, 128 and 256 B over
 * 1 GiB, 8 or 16 in flight per thread (the better), on the db stream; waits.  Allocates
 * 1 GiB of scratch for the call.  Errors: INVALID_ARG (null), OOM, CUDA. */
cc_status cc_gather_sweep(cc_db db, double gbs[4]);

#ifdef __cplusplus
}
#endif
#endif /* GCCTB_H */
