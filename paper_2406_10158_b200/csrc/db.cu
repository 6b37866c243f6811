// db.cu -- host driver behind the C ABI (include/gcctb.h).  It owns every device
// allocation, enqueues the a1..a7 kernels on the db stream, and turns device errors
// into cc_status.  No torch types anywhere: plain pointers and sizes.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <atomic>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"
#include "tpcc.h"

namespace gcctb {
cudaError_t launch_part_all(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr, uint32_t n_txn,
                            uint8_t *skip, unsigned long long *cnt, unsigned long long *off,
                            unsigned long long *cursor, PartReq *out, cudaStream_t s);
int rank_kernel_grid();
}  // namespace gcctb

using namespace gcctb;
typedef unsigned long long u64;

// largest per-block shared-memory footprint of an executor (contexts + thread-mode staged
// accesses): above it the staged accesses move to a global workspace, and the rest of
// the 228 KB per SM stays free for the L1 share the executor's loads use
#ifndef GC_STAGE_SMEM_MAX
#define GC_STAGE_SMEM_MAX (180u * 1024u)
#endif

// Every device allocation / free the driver makes goes through dalloc / dfree, which count
// them (cc_mem_stats): the bench asserts that a timed loop of steps makes none (a
// cudaMalloc / cudaFree is an implicit device synchronisation).
static std::atomic<uint64_t> g_allocs{0}, g_frees{0}, g_alloc_bytes{0};
template <class T>
static cudaError_t dalloc(T **p, size_t bytes) {
    g_allocs++;
    g_alloc_bytes += bytes ? bytes : 16;
    return cudaMalloc((void **)p, bytes ? bytes : 16);
}
static void dfree(void *p) {
    if (!p) return;
    g_frees++;
    cudaFree(p);
}

struct Table {
    std::string name;
    uint32_t row_bytes;
    uint64_t rows;
    uint64_t base;   // first record id (CC-managed tables)
    bool cc;         // has CC words (false: immutable or private reserved slots)
    void *d;
};
struct Index {
    uint32_t table;
    uint64_t n;
    u64 *keys;     // sorted keys, padded with ~0 to a multiple of 16 (tree leaves)
    u64 *rowids;
    std::vector<u64 *> levels;   // cache-line tree levels above the leaves
    std::vector<uint64_t> lens;
    int dense = 0;   // 0, IDX_DENSE (keys k0..k0+n-1) or IDX_DENSE_ID (and row id == position)
    u64 k0 = 0;
    u64 *eytz_keys = nullptr, *eytz_rows = nullptr;   // Eytzinger copy, 1-based (f-3)
    uint64_t eytz_n = 0;                              // 2^h - 1
};

// Lookup mode for a submit / lookup: forced by the flags, else direct addressing on a
// dense key range, else the cache-line tree (all return the same rows, f-3).
static int index_mode(const Index &ix, uint32_t flags) {
    if (flags & CC_FLAG_INDEX_BINARY) return IDX_BINARY;
    if (flags & CC_FLAG_INDEX_EYTZ) return IDX_EYTZ;
    if ((flags & CC_FLAG_INDEX_TREE) || !ix.dense) return IDX_TREE;
    return ix.dense;
}

// Build the separator levels of the cache-line search tree over ix.keys (device).
static cudaError_t build_tree(Index &ix, cudaStream_t s) {
    uint64_t n_in = ix.n;
    const u64 *in = ix.keys;
    uint64_t padded = (n_in + 15) / 16 * 16;
    ix.lens.push_back(padded);
    while (padded > 16) {
        const uint64_t nodes = padded / 16;
        const uint64_t out_padded = (nodes + 15) / 16 * 16;
        u64 *out = nullptr;
        cudaError_t e = dalloc(&out, out_padded * 8);
        if (e) return e;
        e = launch_tree_level(in, n_in, out, out_padded, s);
        if (e) return e;
        ix.levels.push_back(out);
        ix.lens.push_back(out_padded);
        in = out;
        n_in = nodes;
        padded = out_padded;
    }
    // Eytzinger layout of the same keys: a complete tree of 2^h - 1 slots (1-based)
    int h = 1;
    while (((1ull << h) - 1) < ix.n) h++;
    ix.eytz_n = (1ull << h) - 1;
    cudaError_t e = dalloc(&ix.eytz_keys, (ix.eytz_n + 1) * 8);
    if (!e) e = dalloc(&ix.eytz_rows, (ix.eytz_n + 1) * 8);
    if (!e) e = launch_eytz_build(ix.keys, ix.rowids, ix.n, h, ix.eytz_keys, ix.eytz_rows, s);
    if (e) return e;
    return cudaStreamSynchronize(s);
}


static TreeIndex tree_of(const Index &ix) {
    TreeIndex t{};
    t.n_levels = 1 + (int)ix.levels.size();
    t.lv[0] = ix.keys;
    t.len[0] = ix.lens[0];
    for (size_t k = 0; k < ix.levels.size() && k + 1 < (size_t)IDX_MAX_LEVELS; k++) {
        t.lv[k + 1] = ix.levels[k];
        t.len[k + 1] = ix.lens[k + 1];
    }
    return t;
}

static void index_params(const Index &ix, uint32_t flags, YcsbParams &y) {
    y.idx_keys = ix.keys;
    y.idx_rows = ix.rowids;
    y.idx_n = ix.n;
    y.tree = tree_of(ix);
    y.mode = index_mode(ix, flags);
    y.idx_k0 = ix.k0;
    y.eytz_keys = ix.eytz_keys;
    y.eytz_rows = ix.eytz_rows;
    y.eytz_n = ix.eytz_n;
}

struct cc_batch_s {
    uint32_t kind;
    uint32_t n_txn;
    uint32_t K;
    uint32_t *keys;   // YCSB
    uint8_t *ops;     // YCSB
    uint32_t *tx;     // TPC-C descriptors
    u64 *err = nullptr;            // a1 error word of this batch (generator failure), merged at submit
    cudaEvent_t ready = nullptr;   // recorded on the db stream after generation / import
    cudaEvent_t idle = nullptr;    // pooled: the prep stream's last read of the batch (cc_batch_free)
    bool idle_rec = false;
    // f-4: a3 results prepared ahead on the prep stream, slot 0 = GPUTx, 1 = GaccO
    struct Prepared {
        PrepBufs b{};
        std::vector<void *> allocs;
        Ctl *ctl = nullptr;            // errors raised during the prepare (merged at submit)
        cudaEvent_t done = nullptr;    // prep finished (prep stream)
        cudaEvent_t consumed = nullptr;   // the consuming submit's finalize finished (db stream)
        bool has_consumer = false;
        bool valid = false;
    } prep[2];
};

struct TpccState {
    bool loaded = false;
    uint32_t W = 0, w_first = 0, w_count = 0, max_txn = 0;
    uint64_t seed = 0;
    uint32_t c_load = 0, c_run = 0, c_id = 0, c_item = 0;
    uint32_t ids[9] = {0};
    uint32_t *nidx_start = nullptr, *nidx_count = nullptr, *nidx_rows = nullptr;
};

struct Pending {
    cudaEvent_t ev[5];
};

struct cc_db_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaStream_t prep_stream = nullptr;   // f-4: a3 of the next batch (cc_prepare)
    cudaStream_t copy_stream = nullptr;   // asynchronous host imports (src_on_device == 2)
    cudaEvent_t copy_after = nullptr;     // orders an async import after the db stream's work
    int rank = 0, world = 1;
    int num_sms = 148;
    size_t persist_l2 = 0;     // L2 set aside for persisting accesses (the control words), bytes
    size_t max_window = 0;     // largest access-policy window
    std::string err;
    cc_status sticky = CC_OK;
    std::vector<Table> tables;
    std::vector<Index> indexes;
    uint64_t n_records = 0;
    uint32_t *latch = nullptr;          // CC_FLAG_LATCHED
    uint64_t latch_records = 0;
    u64 *stages = nullptr;              // CC_FLAG_STAGES accumulators
    Event *events = nullptr;            // CC_FLAG_EVENTS log
    uint64_t events_cap = 0;
    int clock_khz = 0;
    u64 *meta = nullptr;                 // meta_buf[0]
    uint64_t meta_records = 0;
    // a2 off the critical path: two sets of CC words.  A submit executes on one set while
    // the set its predecessor used is zeroed on reset_stream (every scheme's initial words
    // are zeros); a partitioned submit leaves its set dirty, zeroed in stream before reuse.
    u64 *meta_buf[2] = {nullptr, nullptr};
    int meta_cur = 0;
    uint64_t meta_dirty[2] = {0, 0};          // words to zero in stream before the next use
    bool meta_cleaning[2] = {false, false};   // a zeroing on reset_stream is in flight
    cudaEvent_t meta_used[2] = {nullptr, nullptr}, meta_clean[2] = {nullptr, nullptr};
    cudaStream_t reset_stream = nullptr;
    int ycsb_table = -1, ycsb_index = -1;
    TpccState tpcc;
    struct Part {
        bool pending = false;         // a partitioned submit awaits cc_part_finish
        bool all = false;             // CC_FLAG_PART_ALL: every transaction is distributed
        uint32_t cap_txn = 0;
        uint8_t *skip = nullptr;
        PartReq *send = nullptr;
        PartResp *stage = nullptr;
        unsigned long long *cnt = nullptr, *off = nullptr, *cursor = nullptr;   // [world + 1]
        uint64_t recv_cap = 0;
        unsigned long long *k1 = nullptr, *k2 = nullptr;
        uint32_t *i1 = nullptr, *i2 = nullptr;
        void *tmp = nullptr;
        size_t tmp_bytes = 0;
        ExecParams p{};
        TpccParams tp{};
        cc_result res{};
        cc_batch b = nullptr;
        bool timing = false;
        Pending ev{};
        bool two_pc = false;          // CC_FLAG_PART_2PC: phase B in 2PC rounds (f-2)
        uint32_t round = 0;
        uint8_t *vote = nullptr;      // owner: grant of every received request (this round)
        uint64_t vote_cap = 0;
        unsigned long long *dec = nullptr;   // home: decision of every sent request
        // CC_FLAG_PART_P2P: in-library exchange over peer memory
        void *win = nullptr;                 // this rank's window [flags | inbox | staging]
        uint32_t win_cap = 0, win_txn = 0;   // request slots per source, transactions
        PeerTab pt{};                        // every rank's window, as pointers of this process
        bool connected = false;
        std::vector<void *> ipc_open;        // peers' windows opened through CUDA IPC
        unsigned long long epoch = 0;        // partitioned P2P submits so far (all ranks in step)
        unsigned long long *rc = nullptr;    // [2 world + 1]: counts, offsets, total received
        PartReq *recv = nullptr;             // compacted inboxes (world x cap)
    } part;
    // per-submit scratch (grown on demand)
    Ctl *ctl = nullptr;
    u64 *stats_scratch = nullptr;
    u64 *sticky_dev = nullptr;
    uint32_t cap_txn = 0;
    uint64_t cap_acc = 0;
    uint8_t *committed = nullptr;
    uint32_t *restarts = nullptr;
    u64 *ohi = nullptr, *olo = nullptr;
    u64 *ring = nullptr;
    uint32_t ring_cap = 0;
    RankBitmap rank_bm{};               // a7 commit positions of TO / MVCC / Silo
    cc_result hres[2]{};                // device staging of results requested in host memory
    cudaEvent_t hres_out[2]{};          // the copy-out of the submit that last used staging set k
    bool hres_used[2] = {false, false};
    int hres_next = 0;                  // alternating: a submit's copy-out overlaps the next one
    uint32_t hres_txn = 0, hres_words = 0;
    void *ws = nullptr;                 // thread-mode staging workspace (global fallback)
    uint64_t ws_bytes = 0;
    u64 *arena = nullptr;
    uint64_t arena_nodes = 0;
    uint32_t arena_row_words = 0;
    PrepBufs prep{};
    std::vector<void *> prep_allocs;
    std::vector<void *> snap;
    std::vector<Pending> pending;
    std::vector<Pending> free_events;
    double acc[5] = {0, 0, 0, 0, 0};
    uint64_t n_timed = 0;
    cc_stats last{};
    std::vector<cc_batch_s *> batches;
    // freed batches kept with their device buffers for reuse by a batch of the same shape:
    // no cudaMalloc / cudaFree (a device-wide sync) between steps.  Reuse is ordered after
    // the old batch's work by the db stream (and, if it was prepared, by prep_idle).
    std::vector<cc_batch_s *> pool;
};

static cc_status fail(cc_db db, cc_status st, const char *fmt, ...) {
    if (db) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        db->err = buf;
        if (st == CC_ERR_CUDA) db->sticky = CC_ERR_STATE;
    }
    return st;
}

#define CUDA_TRY(db, x)                                                                   \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess)                                                            \
            return fail(db, e_ == cudaErrorMemoryAllocation ? CC_ERR_OOM : CC_ERR_CUDA,   \
                        "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

#define CHECK_DB(db)                                                         \
    do {                                                                     \
        if (!(db)) return CC_ERR_INVALID_ARG;                                \
        if ((db)->sticky != CC_OK) return (db)->sticky;                      \
        if (cudaSetDevice((db)->device) != cudaSuccess)                      \
            return fail(db, CC_ERR_CUDA, "cudaSetDevice(%d) failed", (db)->device); \
    } while (0)


extern "C" {

const char *cc_version(void) { return "gcctb-b200 0.1 (sm_100a, CUDA " "12.9)"; }

const char *cc_last_error(cc_db db) { return db ? db->err.c_str() : "null db"; }

cc_status cc_db_create(const cc_db_desc *desc, cc_db *out) {
    if (!desc || !out) return CC_ERR_INVALID_ARG;
    if (desc->world < 1 || desc->rank < 0 || desc->rank >= desc->world) return CC_ERR_INVALID_ARG;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return CC_ERR_CUDA;
    if (desc->device < 0 || desc->device >= ndev) return CC_ERR_INVALID_ARG;
    cc_db db = new cc_db_s();
    db->device = desc->device;
    db->rank = desc->rank;
    db->world = desc->world;
    if (cudaSetDevice(db->device) != cudaSuccess) { delete db; return CC_ERR_CUDA; }
    cudaDeviceGetAttribute(&db->num_sms, cudaDevAttrMultiProcessorCount, db->device);
    cudaDeviceGetAttribute(&db->clock_khz, cudaDevAttrClockRate, db->device);
    if (desc->stream) {
        db->stream = (cudaStream_t)desc->stream;
    } else {
        if (cudaStreamCreateWithFlags(&db->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete db;
            return CC_ERR_CUDA;
        }
        db->own_stream = true;
    }
    int lo_prio = 0, hi_prio = 0;   // the prep stream yields to everything else
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    if (cudaStreamCreateWithPriority(&db->prep_stream, cudaStreamNonBlocking, lo_prio) != cudaSuccess) {
        delete db;
        return CC_ERR_CUDA;
    }
    if (cudaStreamCreateWithFlags(&db->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithPriority(&db->reset_stream, cudaStreamNonBlocking, lo_prio) != cudaSuccess ||
        cudaEventCreateWithFlags(&db->meta_used[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&db->meta_used[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&db->meta_clean[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&db->meta_clean[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&db->copy_after, cudaEventDisableTiming) != cudaSuccess) {
        delete db;
        return CC_ERR_CUDA;
    }
    if (dalloc(&db->ctl, sizeof(Ctl)) || dalloc(&db->stats_scratch, 8 * CC_STATS_WORDS) ||
        dalloc(&db->sticky_dev, 8)) {
        delete db;
        return CC_ERR_OOM;
    }
    cudaMemset(db->sticky_dev, 0, 8);
    cudaMemset(db->ctl, 0, sizeof(Ctl));
    *out = db;
    return CC_OK;
}

static void free_scratch(cc_db db) {
    dfree(db->committed); dfree(db->restarts); dfree(db->ohi); dfree(db->olo);
    dfree(db->ring);
    for (void *p : db->prep_allocs) dfree(p);
    db->prep_allocs.clear();
    db->committed = nullptr; db->restarts = nullptr; db->ohi = db->olo = nullptr; db->ring = nullptr;
    db->cap_txn = 0;
    db->cap_acc = 0;
}

static void free_batch_mem(cc_batch b) {
    dfree(b->keys);
    dfree(b->ops);
    dfree(b->tx);
    dfree(b->err);
    if (b->ready) cudaEventDestroy(b->ready);
    if (b->idle) cudaEventDestroy(b->idle);
    for (auto &q : b->prep) {
        for (void *a : q.allocs) dfree(a);
        dfree(q.ctl);
        if (q.done) cudaEventDestroy(q.done);
        if (q.consumed) cudaEventDestroy(q.consumed);
    }
    delete b;
}

cc_status cc_db_destroy(cc_db db) {
    if (!db) return CC_ERR_INVALID_ARG;
    cudaSetDevice(db->device);
    cudaStreamSynchronize(db->stream);
    for (auto &t : db->tables) dfree(t.d);
    for (auto &i : db->indexes) {
        dfree(i.keys);
        dfree(i.rowids);
        for (u64 *l : i.levels) dfree(l);
        dfree(i.eytz_keys);
        dfree(i.eytz_rows);
    }
    for (void *p : db->snap) dfree(p);
    cudaStreamSynchronize(db->prep_stream);
    for (auto *b : db->batches) free_batch_mem(b);
    for (auto *b : db->pool) free_batch_mem(b);
    dfree(db->tpcc.nidx_start); dfree(db->tpcc.nidx_count); dfree(db->tpcc.nidx_rows);
    for (auto &pe : db->pending) for (auto &e : pe.ev) cudaEventDestroy(e);
    for (auto &pe : db->free_events) for (auto &e : pe.ev) cudaEventDestroy(e);
    free_scratch(db);
    dfree(db->part.skip); dfree(db->part.send); dfree(db->part.stage);
    dfree(db->part.cnt); dfree(db->part.off); dfree(db->part.cursor);
    dfree(db->part.k1); dfree(db->part.k2); dfree(db->part.i1); dfree(db->part.i2);
    dfree(db->part.tmp);
    dfree(db->part.vote);
    dfree(db->part.dec);
    for (void *p : db->part.ipc_open) cudaIpcCloseMemHandle(p);
    dfree(db->part.win);
    dfree(db->part.rc);
    dfree(db->part.recv);
    dfree(db->arena);
    dfree(db->ws);
    for (int k = 0; k < 2; k++) {
        cc_result &h = db->hres[k];
        dfree(h.committed); dfree(h.restarts); dfree(h.order_hi); dfree(h.order_lo);
        dfree(h.commit_pos); dfree(h.read_out); dfree(h.stats);
        if (db->hres_out[k]) cudaEventDestroy(db->hres_out[k]);
    }
    dfree(db->rank_bm.bits);
    dfree(db->rank_bm.pre);
    dfree(db->rank_bm.csum);
    dfree(db->latch);
    dfree(db->stages);
    dfree(db->events);
    cudaStreamSynchronize(db->reset_stream);
    dfree(db->meta_buf[0]);
    dfree(db->meta_buf[1]);
    dfree(db->ctl);
    dfree(db->stats_scratch);
    dfree(db->sticky_dev);
    if (db->own_stream) cudaStreamDestroy(db->stream);
    cudaStreamDestroy(db->prep_stream);
    cudaStreamSynchronize(db->copy_stream);
    cudaStreamDestroy(db->copy_stream);
    cudaEventDestroy(db->copy_after);
    cudaStreamDestroy(db->reset_stream);
    for (int k = 0; k < 2; k++) {
        cudaEventDestroy(db->meta_used[k]);
        cudaEventDestroy(db->meta_clean[k]);
    }
    delete db;
    return CC_OK;
}

// ---------------------------------------------------------------- tables
static cc_status create_table(cc_db db, const char *name, uint32_t row_bytes, uint64_t rows, bool cc,
                              uint32_t *table_id) {
    if (!table_id || row_bytes == 0 || row_bytes % 8 || rows == 0)
        return fail(db, CC_ERR_INVALID_ARG, "cc_table_create: bad row_bytes/rows");
    if (cc && db->n_records + rows > (1ull << 32))
        return fail(db, CC_ERR_CONFIG, "cc_table_create: more than 2^32 records");
    Table t;
    t.name = name ? name : "";
    t.row_bytes = row_bytes;
    t.rows = rows;
    t.base = db->n_records;
    t.cc = cc;
    CUDA_TRY(db, dalloc(&t.d, (size_t)row_bytes * rows));
    CUDA_TRY(db, cudaMemsetAsync(t.d, 0, (size_t)row_bytes * rows, db->stream));
    if (cc) {
        // CC metadata: 2 words per record so MVCC's (lo, hi) pair fits (Table II: 16 B),
        // GC_META_PAD_WORDS words per record for the padded layout (CC_FLAG_META_PAD)
        // (two sets: see cc_db_s::meta_buf), zeroed: every scheme's initial state
        const uint64_t need = db->n_records + rows;
        u64 *mb[2] = {nullptr, nullptr};
        for (int k = 0; k < 2; k++) {
            CUDA_TRY(db, dalloc(&mb[k], need * 8 * GC_META_PAD_WORDS));   // room for the padded layout
            CUDA_TRY(db, cudaMemsetAsync(mb[k], 0, need * 8 * GC_META_PAD_WORDS, db->stream));
        }
        CUDA_TRY(db, cudaStreamSynchronize(db->stream));
        CUDA_TRY(db, cudaStreamSynchronize(db->reset_stream));
        for (int k = 0; k < 2; k++) {
            dfree(db->meta_buf[k]);
            db->meta_buf[k] = mb[k];
            db->meta_dirty[k] = 0;
            db->meta_cleaning[k] = false;
        }
        db->meta = mb[0];
        db->meta_cur = 0;
        db->meta_records = need;
        db->n_records = need;
    }
    db->tables.push_back(t);
    *table_id = (uint32_t)db->tables.size() - 1;
    return CC_OK;
}

cc_status cc_table_create(cc_db db, const char *name, uint32_t row_bytes, uint64_t rows,
                          uint32_t *table_id) {
    CHECK_DB(db);
    return create_table(db, name, row_bytes, rows, true, table_id);
}

cc_status cc_table_info(cc_db db, uint32_t table_id, uint64_t *rows, uint32_t *row_bytes) {
    CHECK_DB(db);
    if (table_id >= db->tables.size()) return fail(db, CC_ERR_INVALID_ARG, "bad table id");
    if (rows) *rows = db->tables[table_id].rows;
    if (row_bytes) *row_bytes = db->tables[table_id].row_bytes;
    return CC_OK;
}

cc_status cc_table_load(cc_db db, uint32_t table_id, uint64_t first_row, uint64_t n,
                        const void *src, int src_on_device) {
    CHECK_DB(db);
    if (table_id >= db->tables.size() || !src) return fail(db, CC_ERR_INVALID_ARG, "bad args");
    Table &t = db->tables[table_id];
    if (first_row + n > t.rows) return fail(db, CC_ERR_INVALID_ARG, "row range out of table");
    char *dst = (char *)t.d + first_row * t.row_bytes;
    CUDA_TRY(db, cudaMemcpyAsync(dst, src, n * t.row_bytes,
                                 src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                 db->stream));
    if (!src_on_device) CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    return CC_OK;
}

cc_status cc_table_read(cc_db db, uint32_t table_id, uint64_t first_row, uint64_t n, void *dst,
                        int dst_on_device) {
    CHECK_DB(db);
    if (table_id >= db->tables.size() || !dst) return fail(db, CC_ERR_INVALID_ARG, "bad args");
    Table &t = db->tables[table_id];
    if (first_row + n > t.rows) return fail(db, CC_ERR_INVALID_ARG, "row range out of table");
    const char *src = (const char *)t.d + first_row * t.row_bytes;
    CUDA_TRY(db, cudaMemcpyAsync(dst, src, n * t.row_bytes,
                                 dst_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                 db->stream));
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    return CC_OK;
}

cc_status cc_index_create(cc_db db, uint32_t table_id, const uint64_t *sorted_keys,
                          const uint64_t *row_ids, uint64_t n, int src_on_device,
                          uint32_t *index_id) {
    CHECK_DB(db);
    if (table_id >= db->tables.size() || !sorted_keys || !row_ids || !index_id || n == 0)
        return fail(db, CC_ERR_INVALID_ARG, "cc_index_create: bad args");
    std::vector<uint64_t> hk, hr;
    const uint64_t *k = sorted_keys, *r = row_ids;
    if (src_on_device) {
        hk.resize(n); hr.resize(n);
        CUDA_TRY(db, cudaMemcpy(hk.data(), sorted_keys, n * 8, cudaMemcpyDeviceToHost));
        CUDA_TRY(db, cudaMemcpy(hr.data(), row_ids, n * 8, cudaMemcpyDeviceToHost));
        k = hk.data(); r = hr.data();
    }
    for (uint64_t i = 0; i < n; i++) {
        if (i && k[i] <= k[i - 1]) return fail(db, CC_ERR_INVALID_ARG, "index keys not strictly ascending");
        if (k[i] == ~0ull) return fail(db, CC_ERR_INVALID_ARG, "key 2^64-1 is reserved");
        if (r[i] >= db->tables[table_id].rows) return fail(db, CC_ERR_INVALID_ARG, "row id out of table");
    }
    Index ix{table_id, n, nullptr, nullptr, {}, {}};
    bool dk = true, dr = true;
    for (uint64_t i = 0; i < n; i++) {
        dk &= k[i] == k[0] + i;
        dr &= r[i] == i;
    }
    ix.dense = dk ? (dr ? IDX_DENSE_ID : IDX_DENSE) : 0;
    ix.k0 = k[0];
    const uint64_t padded = (n + 15) / 16 * 16;
    CUDA_TRY(db, dalloc(&ix.keys, padded * 8));
    CUDA_TRY(db, dalloc(&ix.rowids, n * 8));
    CUDA_TRY(db, launch_fill_u64(ix.keys + n, ~0ull, padded - n, db->stream));
    CUDA_TRY(db, cudaMemcpyAsync(ix.keys, k, n * 8, cudaMemcpyHostToDevice, db->stream));
    CUDA_TRY(db, cudaMemcpyAsync(ix.rowids, r, n * 8, cudaMemcpyHostToDevice, db->stream));
    CUDA_TRY(db, build_tree(ix, db->stream));
    db->indexes.push_back(ix);
    *index_id = (uint32_t)db->indexes.size() - 1;
    return CC_OK;
}

cc_status cc_index_lookup(cc_db db, uint32_t index_id, const uint64_t *keys, uint64_t n, uint64_t *rows_out,
                          uint32_t flags) {
    CHECK_DB(db);
    if (index_id >= db->indexes.size() || (n && (!keys || !rows_out)))
        return fail(db, CC_ERR_INVALID_ARG, "cc_index_lookup: bad args");
    const Index &ix = db->indexes[index_id];
    YcsbParams y{};
    index_params(ix, flags, y);
    CUDA_TRY(db, launch_index_lookup(y, (const u64 *)keys, n, (u64 *)rows_out, db->stream));
    return CC_OK;
}

// ---------------------------------------------------------------- YCSB
cc_status cc_load_ycsb(cc_db db, const cc_ycsb_db_desc *d) {
    CHECK_DB(db);
    if (!d || d->n_rows == 0 || d->n_rows > 0xFFFFFFFFull)
        return fail(db, CC_ERR_INVALID_ARG, "cc_load_ycsb: bad n_rows");
    if (db->ycsb_table >= 0) return fail(db, CC_ERR_CONFIG, "YCSB table already loaded");
    uint32_t tid;
    cc_status st = cc_table_create(db, "usertable", 128, d->n_rows, &tid);
    if (st) return st;
    Table &t = db->tables[tid];
    CUDA_TRY(db, launch_ycsb_init_rows((u64 *)t.d, 0, d->n_rows, d->seed, db->stream));
    Index ix{tid, d->n_rows, nullptr, nullptr, {}, {}};
    ix.dense = IDX_DENSE_ID;   // key i -> row i
    ix.k0 = 0;
    const uint64_t padded = (d->n_rows + 15) / 16 * 16;
    CUDA_TRY(db, dalloc(&ix.keys, padded * 8));
    CUDA_TRY(db, dalloc(&ix.rowids, d->n_rows * 8));
    CUDA_TRY(db, launch_fill_u64(ix.keys + d->n_rows, ~0ull, padded - d->n_rows, db->stream));
    CUDA_TRY(db, launch_identity_index(ix.keys, ix.rowids, d->n_rows, db->stream));
    CUDA_TRY(db, build_tree(ix, db->stream));
    db->indexes.push_back(ix);
    db->ycsb_table = (int)tid;
    db->ycsb_index = (int)db->indexes.size() - 1;
    return CC_OK;
}

static cudaError_t batch_ready(cc_db db, cc_batch b, cudaStream_t s = nullptr) {
    if (!b->ready) {
        cudaError_t e = cudaEventCreateWithFlags(&b->ready, cudaEventDisableTiming);
        if (e) return e;
    }
    return cudaEventRecord(b->ready, s ? s : db->stream);
}

static cc_status new_batch(cc_db db, uint32_t n_txn, uint32_t K, cc_batch *out, uint32_t kind = KIND_YCSB) {
    if (db->part.pending) return fail(db, CC_ERR_STATE, "a partitioned submit is pending (cc_part_finish first)");
    for (size_t i = 0; i < db->pool.size(); i++) {
        cc_batch b = db->pool[i];
        if (b->kind != kind || b->n_txn != n_txn || b->K != K) continue;
        db->pool.erase(db->pool.begin() + i);
        for (auto &q : b->prep) q.valid = false;
        // the new contents are written on the db stream: after the prep stream's last read
        if (b->idle_rec) CUDA_TRY(db, cudaStreamWaitEvent(db->stream, b->idle, 0));
        b->idle_rec = false;
        CUDA_TRY(db, cudaMemsetAsync(b->err, 0, 8, db->stream));
        db->batches.push_back(b);
        *out = b;
        return CC_OK;
    }
    cc_batch b = new cc_batch_s();
    b->kind = kind;
    b->n_txn = n_txn;
    b->K = K;
    b->keys = nullptr;
    b->ops = nullptr;
    b->tx = nullptr;
    cudaError_t e = kind == KIND_YCSB
                        ? (dalloc(&b->keys, (size_t)n_txn * K * 4) ?: dalloc(&b->ops, (size_t)n_txn * K))
                        : dalloc(&b->tx, (size_t)n_txn * TPCC_TX_WORDS * 4);
    if (!e) e = dalloc(&b->err, 8);
    if (!e) e = cudaMemsetAsync(b->err, 0, 8, db->stream);
    if (e) {
        dfree(b->keys);
        dfree(b->ops);
        dfree(b->tx);
        dfree(b->err);
        delete b;
        return fail(db, CC_ERR_OOM, "batch allocation failed");
    }
    db->batches.push_back(b);
    *out = b;
    return CC_OK;
}

cc_status cc_batch_gen_ycsb(cc_db db, const cc_ycsb_gen_desc *g, cc_batch *out) {
    CHECK_DB(db);
    if (!g || !out || !g->thresholds) return fail(db, CC_ERR_INVALID_ARG, "cc_batch_gen_ycsb: null");
    if (db->ycsb_table < 0) return fail(db, CC_ERR_CONFIG, "no YCSB table loaded");
    const uint64_t n = db->tables[db->ycsb_table].rows;
    if (g->ops_per_txn == 0 || g->ops_per_txn > 16 || g->ops_per_txn > n || g->n_txn == 0 ||
        g->n_txn > (1u << 21) || !(g->write_frac >= 0.0 && g->write_frac <= 1.0))
        return fail(db, CC_ERR_CONFIG, "cc_batch_gen_ycsb: bad geometry (K 1..16, n_txn <= 2^21, W in [0,1])");
    cc_batch b;
    cc_status st = new_batch(db, g->n_txn, g->ops_per_txn, &b);
    if (st) return st;
    const u64 *T = (const u64 *)g->thresholds;
    u64 *tmp = nullptr;
    if (!g->thresholds_on_device) {
        CUDA_TRY(db, dalloc(&tmp, n * 8));
        CUDA_TRY(db, cudaMemcpyAsync(tmp, g->thresholds, n * 8, cudaMemcpyHostToDevice, db->stream));
        T = tmp;
    }
    CUDA_TRY(db, launch_ycsb_gen(b->keys, b->ops, g->n_txn, g->ops_per_txn, n, g->write_frac,
                                 g->seed, T, g->scramble_mult % n, b->err, db->stream));
    if (tmp) {
        CUDA_TRY(db, cudaStreamSynchronize(db->stream));
        dfree(tmp);
    }
    CUDA_TRY(db, batch_ready(db, b));
    *out = b;
    return CC_OK;
}

cc_status cc_batch_import_ycsb(cc_db db, const uint32_t *keys, const uint8_t *ops, uint32_t n_txn,
                               uint32_t K, int src_on_device, cc_batch *out) {
    CHECK_DB(db);
    if (!keys || !ops || !out || n_txn == 0 || K == 0 || K > 16 || n_txn > (1u << 21))
        return fail(db, CC_ERR_INVALID_ARG, "cc_batch_import_ycsb: bad args (K 1..16, n_txn <= 2^21)");
    if (db->ycsb_table < 0) return fail(db, CC_ERR_CONFIG, "no YCSB table loaded");
    cc_batch b;
    cc_status st = new_batch(db, n_txn, K, &b);
    if (st) return st;
    if (src_on_device == CC_SRC_HOST_ASYNC) {   // copy stream; overlaps the db stream's work
        CUDA_TRY(db, cudaEventRecord(db->copy_after, db->stream));   // a pooled buffer's old readers
        CUDA_TRY(db, cudaStreamWaitEvent(db->copy_stream, db->copy_after, 0));
        CUDA_TRY(db, cudaMemcpyAsync(b->keys, keys, (size_t)n_txn * K * 4, cudaMemcpyHostToDevice, db->copy_stream));
        CUDA_TRY(db, cudaMemcpyAsync(b->ops, ops, (size_t)n_txn * K, cudaMemcpyHostToDevice, db->copy_stream));
        CUDA_TRY(db, batch_ready(db, b, db->copy_stream));
        *out = b;
        return CC_OK;
    }
    const cudaMemcpyKind kind = src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CUDA_TRY(db, cudaMemcpyAsync(b->keys, keys, (size_t)n_txn * K * 4, kind, db->stream));
    CUDA_TRY(db, cudaMemcpyAsync(b->ops, ops, (size_t)n_txn * K, kind, db->stream));
    if (!src_on_device) CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    CUDA_TRY(db, batch_ready(db, b));
    *out = b;
    return CC_OK;
}

cc_status cc_batch_export_ycsb(cc_db db, cc_batch b, uint32_t *keys, uint8_t *ops) {
    CHECK_DB(db);
    if (!b || !keys || !ops || b->kind != KIND_YCSB) return fail(db, CC_ERR_INVALID_ARG, "bad batch");
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    CUDA_TRY(db, cudaMemcpy(keys, b->keys, (size_t)b->n_txn * b->K * 4, cudaMemcpyDeviceToHost));
    CUDA_TRY(db, cudaMemcpy(ops, b->ops, (size_t)b->n_txn * b->K, cudaMemcpyDeviceToHost));
    return CC_OK;
}

cc_status cc_batch_info(cc_db db, cc_batch b, uint32_t *n_txn, uint32_t *K, uint32_t *kind) {
    if (!db || !b) return CC_ERR_INVALID_ARG;
    if (n_txn) *n_txn = b->n_txn;
    if (K) *K = b->K;
    if (kind) *kind = b->kind;
    return CC_OK;
}

cc_status cc_batch_free(cc_db db, cc_batch b) {
    if (!db || !b) return CC_ERR_INVALID_ARG;
    for (size_t i = 0; i < db->batches.size(); i++)
        if (db->batches[i] == b) {
            if (db->part.pending && db->part.b == b)
                return fail(db, CC_ERR_STATE, "the batch of a pending partitioned submit");
            bool prepared = false;
            for (auto &q : b->prep) prepared |= !q.allocs.empty();
            // a prepare may still read the batch: the next writer (db stream) waits for this
            // event when the buffers are reused -- no host synchronisation here
            if (prepared) {
                if (!b->idle) CUDA_TRY(db, cudaEventCreateWithFlags(&b->idle, cudaEventDisableTiming));
                CUDA_TRY(db, cudaEventRecord(b->idle, db->prep_stream));
                b->idle_rec = true;
            }
            db->pool.push_back(b);
            db->batches.erase(db->batches.begin() + i);
            return CC_OK;
        }
    return fail(db, CC_ERR_INVALID_ARG, "unknown batch");
}

cc_status cc_pool_trim(cc_db db) {
    CHECK_DB(db);
    CUDA_TRY(db, cudaStreamSynchronize(db->prep_stream));
    CUDA_TRY(db, cudaStreamSynchronize(db->copy_stream));
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    for (auto *b : db->pool) free_batch_mem(b);
    db->pool.clear();
    return CC_OK;
}

cc_status cc_mem_stats(cc_db db, uint64_t *n_allocs, uint64_t *n_frees, uint64_t *bytes_allocated) {
    if (!db) return CC_ERR_INVALID_ARG;
    if (n_allocs) *n_allocs = g_allocs.load();
    if (n_frees) *n_frees = g_frees.load();
    if (bytes_allocated) *bytes_allocated = g_alloc_bytes.load();
    return CC_OK;
}


// ---------------------------------------------------------------- TPC-C
static uint64_t host_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t host_prand(uint64_t seed, uint64_t table, uint64_t row, uint64_t field) {
    return host_mix64(seed ^ (table << 56) ^ (row << 8) ^ field);
}

cc_status cc_load_tpcc(cc_db db, const cc_tpcc_db_desc *d) {
    CHECK_DB(db);
    if (!d || d->warehouses == 0 || d->w_count == 0 || d->w_first + d->w_count > d->warehouses ||
        d->max_txn == 0 || d->warehouses > 65535)
        return fail(db, CC_ERR_INVALID_ARG, "cc_load_tpcc: bad warehouse range / max_txn");
    if (db->tpcc.loaded) return fail(db, CC_ERR_CONFIG, "TPC-C already loaded");
    TpccState &T = db->tpcc;
    T.W = d->warehouses;
    T.w_first = d->w_first;
    T.w_count = d->w_count;
    T.max_txn = d->max_txn;
    T.seed = d->seed;
    // NURand constants (TPC-C §2.1.6; inputs/tpcc.py nurand_consts)
    uint64_t c[4];
    for (int k = 0; k < 4; k++) c[k] = host_prand(d->seed, TPCC_T_CONST, 0, k);
    T.c_load = (uint32_t)(c[0] % 256);
    T.c_run = (uint32_t)((T.c_load + 65 + c[1] % 55) % 256);
    T.c_id = (uint32_t)(c[2] % 1024);
    T.c_item = (uint32_t)(c[3] % 8192);
    const uint64_t wc = d->w_count;
    const struct { const char *n; uint32_t words; uint64_t rows; bool cc; } spec[9] = {
        {"warehouse", TPCC_W_WORDS, wc, true},
        {"district", TPCC_D_WORDS, wc * TPCC_DIST, true},
        {"customer", TPCC_C_WORDS, wc * TPCC_DIST * TPCC_CUST, true},
        {"stock", TPCC_S_WORDS, wc * TPCC_STOCK, true},
        {"item", TPCC_I_WORDS, TPCC_ITEMS, false},
        {"order", TPCC_O_WORDS, d->max_txn, false},
        {"new_order", TPCC_NO_WORDS, d->max_txn, false},
        {"order_line", TPCC_OL_WORDS, (uint64_t)d->max_txn * TPCC_MAXOL, false},
        {"history", TPCC_H_WORDS, d->max_txn, false}};
    for (int k = 0; k < 9; k++) {
        cc_status st = create_table(db, spec[k].n, spec[k].words * 8, spec[k].rows, spec[k].cc, &T.ids[k]);
        if (st) return st;
    }
    const int pop_tab[5] = {TPCC_T_W, TPCC_T_D, TPCC_T_C, TPCC_T_S, TPCC_T_I};
    const uint64_t first[5] = {d->w_first, (uint64_t)d->w_first * TPCC_DIST,
                               (uint64_t)d->w_first * TPCC_DIST * TPCC_CUST, (uint64_t)d->w_first * TPCC_STOCK, 0};
    for (int k = 0; k < 5; k++)
        CUDA_TRY(db, launch_tpcc_pop(pop_tab[k], (u64 *)db->tables[T.ids[k]].d, first[k],
                                     db->tables[T.ids[k]].rows, d->seed, T.c_load, db->stream));
    const uint32_t n_cust = (uint32_t)(wc * TPCC_DIST * TPCC_CUST), n_groups = (uint32_t)(wc * TPCC_DIST * 1000);
    CUDA_TRY(db, dalloc(&T.nidx_start, n_groups * 4ull));
    CUDA_TRY(db, dalloc(&T.nidx_count, n_groups * 4ull));
    CUDA_TRY(db, dalloc(&T.nidx_rows, n_cust * 4ull));
    CUDA_TRY(db, build_name_index((const u64 *)db->tables[T.ids[2]].d, n_cust, first[2], d->seed, T.c_load,
                                  T.nidx_start, T.nidx_count, T.nidx_rows, n_groups, db->stream));
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    T.loaded = true;
    return CC_OK;
}

cc_status cc_tpcc_tables(cc_db db, uint32_t ids[9]) {
    CHECK_DB(db);
    if (!db->tpcc.loaded || !ids) return fail(db, CC_ERR_CONFIG, "TPC-C not loaded");
    for (int k = 0; k < 9; k++) ids[k] = db->tpcc.ids[k];
    return CC_OK;
}

cc_status cc_batch_gen_tpcc(cc_db db, const cc_tpcc_gen_desc *g, cc_batch *out) {
    CHECK_DB(db);
    const TpccState &T = db->tpcc;
    if (!g || !out) return fail(db, CC_ERR_INVALID_ARG, "null args");
    if (!T.loaded) return fail(db, CC_ERR_CONFIG, "TPC-C not loaded");
    if (g->n_txn == 0 || g->n_txn > T.max_txn || g->n_txn > (1u << 21) || g->w_hi <= g->w_lo ||
        g->w_hi > T.W || g->neworder_permyriad > 10000)
        return fail(db, CC_ERR_CONFIG, "cc_batch_gen_tpcc: bad n_txn (<= max_txn, 2^21) / warehouse range");
    cc_batch b;
    cc_status st = new_batch(db, g->n_txn, TPCC_K, &b, KIND_TPCC);
    if (st) return st;
    CUDA_TRY(db, launch_tpcc_gen(b->tx, g->n_txn, g->seed, T.W, g->w_lo, g->w_hi, g->neworder_permyriad,
                                 T.c_run, T.c_id, T.c_item, b->err, db->stream));
    CUDA_TRY(db, batch_ready(db, b));
    *out = b;
    return CC_OK;
}

cc_status cc_batch_import_tpcc(cc_db db, const uint32_t *tx, uint32_t n_txn, int src_on_device, cc_batch *out) {
    CHECK_DB(db);
    if (!tx || !out || n_txn == 0) return fail(db, CC_ERR_INVALID_ARG, "null args");
    if (!db->tpcc.loaded) return fail(db, CC_ERR_CONFIG, "TPC-C not loaded");
    if (n_txn > db->tpcc.max_txn || n_txn > (1u << 21)) return fail(db, CC_ERR_CONFIG, "n_txn > max_txn");
    if (!src_on_device) {   // validate ranges of host descriptors before anything is enqueued
        for (uint32_t g = 0; g < n_txn; g++) {
            const uint32_t *t = tx + (uint64_t)g * TPCC_TX_WORDS;
            const TpccState &T = db->tpcc;
            auto local = [&](uint32_t w) { return w >= T.w_first && w < T.w_first + T.w_count; };
            bool ok = t[TX_TYPE] <= 1 && local(t[TX_W]) && t[TX_D] < TPCC_DIST && t[TX_CD] < TPCC_DIST;
            if (t[TX_TYPE] == 0) {
                ok = ok && t[TX_OLCNT] >= 1 && t[TX_OLCNT] <= TPCC_MAXOL && t[TX_C] < TPCC_CUST;
                for (uint32_t j = 0; ok && j < t[TX_OLCNT]; j++)
                    ok = t[TX_ITEM + j] < TPCC_ITEMS && local(t[TX_SUPQ + j] >> 8);
            } else {
                ok = ok && local(t[TX_CW]) && (t[TX_C] < TPCC_CUST || (t[TX_C] == 0xFFFFFFFFu && t[TX_CLAST] < 1000));
            }
            if (!ok) return fail(db, CC_ERR_KEY_NOT_FOUND, "TPC-C descriptor %u out of range", g);
        }
    }
    cc_batch b;
    cc_status st = new_batch(db, n_txn, TPCC_K, &b, KIND_TPCC);
    if (st) return st;
    CUDA_TRY(db, cudaMemcpyAsync(b->tx, tx, (size_t)n_txn * TPCC_TX_WORDS * 4,
                                 src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, db->stream));
    if (!src_on_device) CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    CUDA_TRY(db, batch_ready(db, b));
    *out = b;
    return CC_OK;
}

cc_status cc_batch_export_tpcc(cc_db db, cc_batch b, uint32_t *tx) {
    CHECK_DB(db);
    if (!b || !tx || b->kind != KIND_TPCC) return fail(db, CC_ERR_INVALID_ARG, "bad batch");
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    CUDA_TRY(db, cudaMemcpy(tx, b->tx, (size_t)b->n_txn * TPCC_TX_WORDS * 4, cudaMemcpyDeviceToHost));
    return CC_OK;
}

// ---------------------------------------------------------------- execution
static cudaError_t alloc_prep(PrepBufs &b, std::vector<void *> &allocs, uint64_t na, uint32_t nt);

static cc_status ensure_scratch(cc_db db, uint32_t n_txn, uint64_t n_acc) {
    if (n_txn <= db->cap_txn && n_acc <= db->cap_acc) return CC_OK;
    cudaStreamSynchronize(db->stream);
    free_scratch(db);
    const uint32_t nt = n_txn;
    const uint64_t na = n_acc < nt ? nt : n_acc;
    CUDA_TRY(db, dalloc(&db->committed, nt));
    CUDA_TRY(db, dalloc(&db->restarts, (size_t)nt * 4));
    CUDA_TRY(db, dalloc(&db->ohi, (size_t)nt * 8));
    CUDA_TRY(db, dalloc(&db->olo, (size_t)nt * 8));
    const uint32_t cap = nt;   // each id is appended to the retry batch at most once
    CUDA_TRY(db, dalloc(&db->ring, ((size_t)cap + GC_RQ_N) * 8));   // + the retry queues
    db->ring_cap = cap;
    CUDA_TRY(db, alloc_prep(db->prep, db->prep_allocs, na, nt));
    db->cap_txn = nt;
    db->cap_acc = na;
    return CC_OK;
}

// a3 buffers for n_acc accesses / n_txn transactions (allocations recorded in `allocs`)
static cudaError_t alloc_prep(PrepBufs &b, std::vector<void *> &allocs, uint64_t na, uint32_t nt) {
    auto A = [&](auto **p, size_t bytes) -> cudaError_t {
        cudaError_t e = dalloc(p, bytes);
        if (e == cudaSuccess) allocs.push_back((void *)*p);
        return e;
    };
#define PTRY(x) do { cudaError_t e_ = (x); if (e_) return e_; } while (0)
    PTRY(A(&b.keys_in, na * 8));
    PTRY(A(&b.keys_out, na * 8));
    PTRY(A(&b.acc_rec, na * 4));
    PTRY(A(&b.acc_seg, na * 4));
    PTRY(A(&b.acc_pos, na * 4));
    PTRY(A(&b.acc_rdy, na * 4));
    PTRY(A(&b.sorted_pos, na * 4));
    PTRY(A(&b.head_flag, na * 4));
    PTRY(A(&b.seg_id, na * 4));
    PTRY(A(&b.seg_start, na * 4));
    PTRY(A(&b.lw, na * 4));
    PTRY(A(&b.cursor, na * 4));
    PTRY(A(&b.rank, (size_t)nt * 4));
    PTRY(A(&b.rank_sorted, (size_t)nt * 4));
    PTRY(A(&b.gid_in, (size_t)nt * 4));
    PTRY(A(&b.rank_order, (size_t)nt * 4));
    PTRY(A(&b.rank_count, (size_t)nt * 4));
    PTRY(A(&b.rank_done, (size_t)nt * 4));
    PTRY(A(&b.rank_start, (size_t)nt * 4));
    b.cub_bytes = prep_cub_bytes(na, nt);
    PTRY(A((char **)&b.cub_tmp, b.cub_bytes));
#undef PTRY
    return cudaSuccess;
}

static cc_status ensure_arena(cc_db db, uint64_t nodes, uint32_t row_words) {
    if (nodes <= db->arena_nodes && row_words == db->arena_row_words) return CC_OK;
    cudaStreamSynchronize(db->stream);
    dfree(db->arena);
    db->arena = nullptr;
    db->arena_nodes = 0;
    CUDA_TRY(db, dalloc(&db->arena, nodes * (ARENA_HDR + row_words) * 8));
    db->arena_nodes = nodes;
    db->arena_row_words = row_words;
    return CC_OK;
}

static Pending get_events(cc_db db) {
    Pending p;
    if (!db->free_events.empty()) {
        p = db->free_events.back();
        db->free_events.pop_back();
        return p;
    }
    for (auto &e : p.ev) cudaEventCreate(&e);
    return p;
}

static cc_status ensure_part(cc_db db, uint32_t n_txn) {
    auto &P = db->part;
    if (!P.cnt) {
        CUDA_TRY(db, dalloc(&P.cnt, (db->world + 1) * 8ull));
        CUDA_TRY(db, dalloc(&P.off, (db->world + 1) * 8ull));
        CUDA_TRY(db, dalloc(&P.cursor, (db->world + 1) * 8ull));
    }
    if (n_txn <= P.cap_txn) return CC_OK;
    cudaStreamSynchronize(db->stream);
    dfree(P.skip); dfree(P.send); dfree(P.stage); dfree(P.dec);
    CUDA_TRY(db, dalloc(&P.dec, (size_t)n_txn * TPCC_K * 8));
    CUDA_TRY(db, dalloc(&P.skip, n_txn));
    CUDA_TRY(db, dalloc(&P.send, (size_t)n_txn * TPCC_K * sizeof(PartReq)));
    CUDA_TRY(db, dalloc(&P.stage, (size_t)n_txn * TPCC_K * sizeof(PartResp)));
    P.cap_txn = n_txn;
    return CC_OK;
}

// kernel-side workload parameters of batch b (YCSB or TPC-C)
static cc_status wl_params(cc_db db, cc_batch b, uint32_t flags, YcsbParams &y, TpccParams &tp) {
    if (b->kind == KIND_TPCC) {
        const TpccState &T = db->tpcc;
        tp.tx = b->tx;
        tp.wh = (u64 *)db->tables[T.ids[0]].d;
        tp.di = (u64 *)db->tables[T.ids[1]].d;
        tp.cu = (u64 *)db->tables[T.ids[2]].d;
        tp.st = (u64 *)db->tables[T.ids[3]].d;
        tp.it = (const u64 *)db->tables[T.ids[4]].d;
        tp.o = (u64 *)db->tables[T.ids[5]].d;
        tp.no = (u64 *)db->tables[T.ids[6]].d;
        tp.ol = (u64 *)db->tables[T.ids[7]].d;
        tp.h = (u64 *)db->tables[T.ids[8]].d;
        tp.bW = db->tables[T.ids[0]].base;
        tp.bD = db->tables[T.ids[1]].base;
        tp.bC = db->tables[T.ids[2]].base;
        tp.bS = db->tables[T.ids[3]].base;
        tp.W = T.W;
        tp.w_first = T.w_first;
        tp.nidx_start = T.nidx_start;
        tp.nidx_count = T.nidx_count;
        tp.nidx_rows = T.nidx_rows;
        tp.entry_date = 20240601;   // per-submit constant date (no wall clock)
    } else {
        if (db->ycsb_table < 0) return fail(db, CC_ERR_CONFIG, "no YCSB table loaded");
        const Table &t = db->tables[db->ycsb_table];
        const Index &ix = db->indexes[db->ycsb_index];
        y.keys = b->keys;
        y.ops = b->ops;
        index_params(ix, flags, y);
        y.rows = (u64 *)t.d;
        y.n_rows = t.rows;
    }
    return CC_OK;
}

// Results requested in host memory: 0 device, 1 host (pinned or pageable), -1 mixed
static int result_kind(const cc_result *r) {
    const void *ptrs[7] = {r->committed, r->restarts, r->order_hi, r->order_lo, r->commit_pos, r->read_out, r->stats};
    int kind = -2;
    for (const void *q : ptrs) {
        if (!q) continue;
        cudaPointerAttributes a{};
        const bool host = cudaPointerGetAttributes(&a, q) != cudaSuccess || a.type == cudaMemoryTypeHost ||
                          a.type == cudaMemoryTypeUnregistered;
        cudaGetLastError();   // an unregistered pointer may leave an error behind on older runtimes
        const int k = host ? 1 : 0;
        if (kind == -2) kind = k;
        else if (kind != k) return -1;
    }
    return kind < 0 ? 0 : kind;
}

// device staging for host-memory results: two sets, so one submit's copy-out (on the
// copy stream) overlaps the next submit (grown on demand, never inside a P2P round)
static cc_status ensure_hres(cc_db db, uint32_t n_txn, uint32_t words) {
    if (n_txn <= db->hres_txn && words <= db->hres_words) return CC_OK;
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    CUDA_TRY(db, cudaStreamSynchronize(db->copy_stream));
    for (int k = 0; k < 2; k++) {
        cc_result &h = db->hres[k];
        dfree(h.committed); dfree(h.restarts); dfree(h.order_hi); dfree(h.order_lo); dfree(h.commit_pos);
        dfree(h.read_out); dfree(h.stats);
        h = cc_result{};
        CUDA_TRY(db, dalloc(&h.committed, n_txn));
        CUDA_TRY(db, dalloc(&h.restarts, n_txn * 4ull));
        CUDA_TRY(db, dalloc(&h.order_hi, n_txn * 8ull));
        CUDA_TRY(db, dalloc(&h.order_lo, n_txn * 8ull));
        CUDA_TRY(db, dalloc(&h.commit_pos, n_txn * 4ull));
        CUDA_TRY(db, dalloc(&h.read_out, (uint64_t)n_txn * words * 8));
        CUDA_TRY(db, dalloc(&h.stats, 8 * CC_STATS_WORDS));
        if (!db->hres_out[k]) CUDA_TRY(db, cudaEventCreateWithFlags(&db->hres_out[k], cudaEventDisableTiming));
        db->hres_used[k] = false;
    }
    db->hres_txn = n_txn;
    db->hres_words = words;
    return CC_OK;
}

// copy the staged results of a submit (set k) to the caller's host buffers on the copy
// stream, after the submit's work on the db stream; cc_sync waits for it
static cc_status copy_results_out(cc_db db, int k, const cc_result *user, uint32_t n_txn, uint32_t words) {
    const cc_result &h = db->hres[k];
    CUDA_TRY(db, cudaEventRecord(db->copy_after, db->stream));
    CUDA_TRY(db, cudaStreamWaitEvent(db->copy_stream, db->copy_after, 0));
    auto cp = [&](void *dst, const void *src, size_t bytes) -> cudaError_t {
        return dst ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, db->copy_stream) : cudaSuccess;
    };
    CUDA_TRY(db, cp(user->committed, h.committed, n_txn));
    CUDA_TRY(db, cp(user->restarts, h.restarts, n_txn * 4ull));
    CUDA_TRY(db, cp(user->order_hi, h.order_hi, n_txn * 8ull));
    CUDA_TRY(db, cp(user->order_lo, h.order_lo, n_txn * 8ull));
    CUDA_TRY(db, cp(user->commit_pos, h.commit_pos, n_txn * 4ull));
    CUDA_TRY(db, cp(user->read_out, h.read_out, (uint64_t)n_txn * words * 8));
    CUDA_TRY(db, cp(user->stats, h.stats, 8 * CC_STATS_WORDS));
    CUDA_TRY(db, cudaEventRecord(db->hres_out[k], db->copy_stream));
    db->hres_used[k] = true;
    return CC_OK;
}

cc_status cc_submit(cc_db db, cc_batch b, const cc_exec_desc *desc, const cc_result *res_in) {
    CHECK_DB(db);
    if (!b || !desc || !res_in || !res_in->committed)
        return fail(db, CC_ERR_INVALID_ARG, "cc_submit: null batch/desc/result");
    // results in host memory are staged in library-owned device buffers and copied out at
    // the end of the submit (pinned: asynchronously on the db stream)
    const int rkind = result_kind(res_in);
    if (rkind < 0) return fail(db, CC_ERR_INVALID_ARG, "cc_submit: result pointers mix host and device memory");
    const uint32_t out_words = b->kind == KIND_TPCC ? TPCC_OUT_WORDS : b->K;
    cc_result staged{};
    int hk = 0;
    const cc_result *res = res_in;
    if (rkind == 1) {
        if ((desc->flags & (CC_FLAG_PARTITIONED | CC_FLAG_PART_ALL)) && !(desc->flags & CC_FLAG_PART_P2P))
            return fail(db, CC_ERR_UNSUPPORTED, "host result buffers: not with a host-driven partitioned submit");
        cc_status st0 = ensure_hres(db, b->n_txn, out_words);
        if (st0) return st0;
        hk = db->hres_next;
        db->hres_next ^= 1;
        // the set's previous copy-out must have drained before this submit overwrites it
        if (db->hres_used[hk]) CUDA_TRY(db, cudaStreamWaitEvent(db->stream, db->hres_out[hk], 0));
        staged = db->hres[hk];
        if (!res_in->read_out) staged.read_out = nullptr;
        res = &staged;
    }
    if ((unsigned)desc->scheme >= CC_NUM_SCHEMES) return fail(db, CC_ERR_INVALID_ARG, "bad scheme");
    if (desc->wd > 5 || desc->bs < 1 || desc->bs > 32)
        return fail(db, CC_ERR_INVALID_ARG, "wd must be 0..5 and bs 1..32 (PAPER.md:480-484)");
    const bool is_tpcc = b->kind == KIND_TPCC;
    if (b->ready) CUDA_TRY(db, cudaStreamWaitEvent(db->stream, b->ready, 0));   // async imports
    {
        const uint32_t L = desc->lanes_per_txn;
        if (!(L <= 1 || L == 4 || L == 8 || L == 16 || L == 32) || (!is_tpcc && L > 1 && L < b->K))
            return fail(db, CC_ERR_INVALID_ARG, "lanes_per_txn must be 0/1 or 4/8/16/32 (YCSB: >= ops per txn)");
    }
    const int scheme = (int)desc->scheme;
    const bool det = scheme == CC_GPUTX || scheme == CC_GACCO;
    const uint64_t n_acc = (uint64_t)b->n_txn * b->K;
    cc_status st = ensure_scratch(db, b->n_txn, n_acc);
    if (st) return st;
    if (scheme == CC_MVCC) {
        st = ensure_arena(db, n_acc, is_tpcc ? TPCC_C_WORDS : 16);   // one history node per access slot
        if (st) return st;
    }

    ExecParams p{};
    p.scheme = scheme;
    p.n_txn = b->n_txn;
    p.K = b->K;
    p.wd = desc->wd;
    p.flags = desc->flags;
    p.lanes = desc->lanes_per_txn <= 1 ? 1 : (is_tpcc ? 32 : desc->lanes_per_txn);
    p.claim_chunk = desc->claim_chunk ? desc->claim_chunk : 1;
    {   // experiment knob (not part of the ABI): TO/MVCC retry backoff cap exponent
        static const int to_cap = getenv("GCCTB_TO_BACKOFF_CAP") ? atoi(getenv("GCCTB_TO_BACKOFF_CAP")) : 0;
        p.to_backoff_cap = (uint32_t)(to_cap > 0 && to_cap < 20 ? to_cap : 0);
    }
    p.watchdog_ns = (u64)((desc->watchdog_s > 0 ? desc->watchdog_s : 30.0) * 1e9);
    p.ctl = db->ctl;
    p.sticky = db->sticky_dev;
    const int mk = db->meta_cur;   // the word set this submit executes on
    p.meta = db->meta_buf[mk];
    p.arena = db->arena;
    p.ring = db->ring;
    p.ring_cap = db->ring_cap;
    p.rq = db->ring + db->ring_cap;
    p.rq_herd_2pl = is_tpcc ? 256u : 2048u;   // retry-queue threshold for 2PL (see exec.cuh)
    p.committed = db->committed;
    p.restarts = db->restarts;
    p.order_hi = db->ohi;
    p.order_lo = db->olo;
    p.read_out = (u64 *)res->read_out;
    YcsbParams y{};
    TpccParams tp{};
    st = wl_params(db, b, desc->flags, y, tp);
    if (st) return st;

    if (desc->flags & CC_FLAG_LATCHED) {   // one 32-bit latch per control word (Exp-7)
        if (db->latch_records < db->n_records) {
            cudaStreamSynchronize(db->stream);
            dfree(db->latch);
            db->latch = nullptr;
            CUDA_TRY(db, dalloc(&db->latch, db->n_records * 8));
            db->latch_records = db->n_records;
        }
        CUDA_TRY(db, launch_fill_u64((u64 *)db->latch, 0ull, db->n_records, db->stream));
        p.latch = db->latch;
    }
    if (desc->flags & CC_FLAG_STAGES) {   // 8 totals + 8 words per thread of the grid (<= 2^21 threads)
        const uint64_t words = 8ull + 8ull * (1ull << 21);
        if (!db->stages) CUDA_TRY(db, dalloc(&db->stages, words * 8));
        CUDA_TRY(db, launch_fill_u64(db->stages, 0ull, words, db->stream));
        p.stages = db->stages;
    }
    if (desc->flags & CC_FLAG_EVENTS) {
        if (!db->events) return fail(db, CC_ERR_CONFIG, "CC_FLAG_EVENTS needs cc_events_capacity first");
        p.events = db->events;
        p.events_cap = db->events_cap;
    }
    const bool timing = desc->flags & CC_FLAG_TIMING;
    const bool partitioned = (desc->flags & (CC_FLAG_PARTITIONED | CC_FLAG_PART_ALL)) != 0;
    const bool two_pc = (desc->flags & CC_FLAG_PART_2PC) != 0;
    if (two_pc && (!partitioned || scheme == CC_GPUTX || scheme == CC_GACCO))
        return fail(db, CC_ERR_UNSUPPORTED,
                    "CC_FLAG_PART_2PC: non-deterministic schemes with CC_FLAG_PARTITIONED only");
    const bool p2p = (desc->flags & CC_FLAG_PART_P2P) != 0;
    if (p2p && (!partitioned || two_pc))
        return fail(db, CC_ERR_UNSUPPORTED, "CC_FLAG_PART_P2P: with CC_FLAG_PARTITIONED, deterministic phase B only");
    if (p2p && (!db->part.connected || b->n_txn > db->part.win_txn))
        return fail(db, CC_ERR_STATE, "CC_FLAG_PART_P2P: cc_part_connect first (window for %u transactions)",
                    db->part.win_txn);
    if (partitioned) {
        const TpccState &T = db->tpcc;
        if (!is_tpcc) return fail(db, CC_ERR_UNSUPPORTED, "partitioned execution is TPC-C only (YCSB: replicas)");
        if (db->part.pending) return fail(db, CC_ERR_STATE, "previous partitioned submit not finished");
        if (T.W % db->world || T.w_count != T.W / db->world || T.w_first != db->rank * T.w_count)
            return fail(db, CC_ERR_CONFIG, "partitioning needs equal contiguous warehouse ranges per rank");
        if ((uint64_t)db->world * b->n_txn > (1ull << 24))
            return fail(db, CC_ERR_CONFIG, "world * n_txn must be <= 2^24 (global gid bits)");
        st = ensure_part(db, b->n_txn);
        if (st) return st;
    }
    Pending ev{};
    if (timing) {
        ev = get_events(db);
        CUDA_TRY(db, cudaEventRecord(ev.ev[0], db->stream));
    }
#if GC_TRACE_COMMIT
    {   // experiment builds: histogram of commit / abort times (tools/trace_tail.py)
        const char *tp_ = getenv("GCCTB_TRACE_PTR");
        p.trace = tp_ ? (unsigned long long *)strtoull(tp_, nullptr, 0) : nullptr;
    }
#endif
    // a2: reset CC state (every record of every table)
    p.mvcc_split = (scheme == CC_MVCC && (desc->flags & CC_FLAG_MVCC_SPLIT)) ? db->n_records : 0;
    p.meta_stride = (scheme != CC_MVCC && (desc->flags & CC_FLAG_META_PAD)) ? GC_META_PAD_WORDS : 1u;
    p.meta_shift = p.meta_stride == 1 ? 0u : 2u;
    static_assert(GC_META_PAD_WORDS == 4, "meta_shift assumes 4 words per padded record");
    // CC_FLAG_L2_PERSIST (ablation, off by default): an access-policy window marks the
    // scheme's word array persisting and everything else streaming from the a2 reset until
    // after the executor (a random 8 B word otherwise costs a ~128 B DRAM fetch, profiles/
    // r02_gather_sweep.md).  Measured a loss on the bench (profiles/r02_l2_persist.md): the
    // set-aside shrinks L2 for the other kernels, and persisting lines outlive the window
    // (and an L2 flush), so a back-to-back gain is partly stale warm lines.
    bool persist = false;
    if ((desc->flags & CC_FLAG_L2_PERSIST) && !det) {
        if (!db->persist_l2) {   // device-wide set-aside, reserved on first use
            int pmax = 0, wmax = 0;
            cudaDeviceGetAttribute(&pmax, cudaDevAttrMaxPersistingL2CacheSize, db->device);
            cudaDeviceGetAttribute(&wmax, cudaDevAttrMaxAccessPolicyWindowSize, db->device);
            if (pmax > 0 && wmax > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)pmax) == cudaSuccess) {
                db->persist_l2 = (size_t)pmax;
                db->max_window = (size_t)wmax;
            }
            cudaGetLastError();
        }
        persist = db->persist_l2 > 0;
    }
    if (persist) {
        const uint64_t words = scheme == CC_MVCC ? 2 * db->n_records : (uint64_t)db->n_records * p.meta_stride;
        cudaStreamAttrValue a{};
        a.accessPolicyWindow.base_ptr = p.meta;
        a.accessPolicyWindow.num_bytes = (size_t)(words * 8 < db->max_window ? words * 8 : db->max_window);
        const double ratio = (double)db->persist_l2 / (double)a.accessPolicyWindow.num_bytes;
        a.accessPolicyWindow.hitRatio = (float)(ratio < 1.0 ? ratio : 1.0);
        a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        CUDA_TRY(db, cudaStreamSetAttribute(db->stream, cudaStreamAttributeAccessPolicyWindow, &a));
    }
    // (GaccO / GPUTx keep no per-record control word: their cursors and K-set counters are
    // reset by a3, so only the ring and the control block are cleared for them)
    // (GaccO / GPUTx keep no per-record control word)
    if (!det) {
        if (db->meta_cleaning[mk]) {   // zeroed behind the previous submit on the reset stream
            CUDA_TRY(db, cudaStreamWaitEvent(db->stream, db->meta_clean[mk], 0));
            db->meta_cleaning[mk] = false;
        }
        if (db->meta_dirty[mk]) {
            CUDA_TRY(db, cudaMemsetAsync(p.meta, 0, db->meta_dirty[mk] * 8, db->stream));
            db->meta_dirty[mk] = 0;
        }
    }
    CUDA_TRY(db, launch_a2(db->ring, db->ring_cap + GC_RQ_N, db->ctl, db->committed, db->restarts, db->ohi,
                           db->olo, b->n_txn, b->err, db->stream));   // a1 failure: nothing executes
    {   // test hook (not part of the ABI): the TO / MVCC timestamp counter starts at
        // GCCTB_TS_BASE instead of 0, so the 31-bit overflow path is reachable
        const char *tb = getenv("GCCTB_TS_BASE");
        const unsigned long long base = tb ? strtoull(tb, nullptr, 0) : 0ull;
        if (base) CUDA_TRY(db, launch_fill_u64(&db->ctl->ts.v, base, 1, db->stream));
    }
    if (partitioned && p2p) {   // a8 over peer memory: requests go straight into the owners' windows
        const uint32_t wpr = db->tpcc.W / db->world;
        db->part.epoch++;
        CUDA_TRY(db, p2p_send(tp, db->rank, db->world, wpr, b->n_txn, db->part.skip, db->part.cnt, db->part.cursor,
                              db->part.pt, db->part.win_cap, db->part.epoch, db->ctl,
                              (desc->flags & CC_FLAG_PART_ALL) != 0, db->stream));
        p.skip = db->part.skip;
    } else if (partitioned) {   // a8: classify local / distributed, pack phase-B requests per owner
        const uint32_t wpr = db->tpcc.W / db->world;
        CUDA_TRY(db, part_classify_pack(tp, db->rank, db->world, wpr, b->n_txn, db->part.skip, db->part.cnt,
                                        db->part.off, db->part.cursor, db->part.send, db->stream));
        if (desc->flags & CC_FLAG_PART_ALL) {
            CUDA_TRY(db, launch_part_all(tp, db->rank, db->world, wpr, b->n_txn, db->part.skip, db->part.cnt,
                                         db->part.off, db->part.cursor, db->part.send, db->stream));
        }
        p.skip = db->part.skip;
    }
    if (timing) CUDA_TRY(db, cudaEventRecord(ev.ev[1], db->stream));
    // a3: preprocessing for the conflict-graph schemes
    cc_batch_s::Prepared *used = nullptr;   // f-4: a3 done ahead by cc_prepare
    if (det) {
        PrepBufs *pb = &db->prep;
        auto &q = b->prep[scheme == CC_GPUTX ? 0 : 1];
        if (!partitioned && q.valid) {
            CUDA_TRY(db, cudaStreamWaitEvent(db->stream, q.done, 0));
            CUDA_TRY(db, launch_merge_err(q.ctl, db->ctl, db->stream));
            pb = &q.b;
            q.valid = false;
            used = &q;
        } else {
            if (is_tpcc) CUDA_TRY(db, launch_tpcc_gather(p, tp, db->prep, db->n_records, db->stream));
            else CUDA_TRY(db, launch_ycsb_gather(p, y, db->prep, db->stream));
            CUDA_TRY(db, launch_prep_common(p, db->prep, db->n_records, scheme == CC_GPUTX,
                                            rank_kernel_grid(), db->stream));
        }
        p.acc_rec = pb->acc_rec;
        p.acc_seg = pb->acc_seg;
        p.acc_pos = pb->acc_pos;
        p.acc_rdy = pb->acc_rdy;
        p.cursor = pb->cursor;
        p.rank_order = pb->rank_order;
        p.rank_of = pb->rank;
        p.rank_done = pb->rank_done;
        p.rank_count = pb->rank_count;
    }
    if (timing) CUDA_TRY(db, cudaEventRecord(ev.ev[2], db->stream));
    // a4-a6: persistent executor
    const int block = 32 * (int)desc->bs;
    // thread mode: each working lane's staged read/write set (K lanes of the workload's
    // access record) in dynamic shared memory, or -- when a block's working lanes need more
    // than GC_STAGE_SMEM_MAX -- in a global workspace with the same strided layout
    // (plus, in every mode, each working lane's context -- exec_th_bytes() -- in shared memory)
    size_t smem = 0;
    uint64_t ws_per_block = 0;
    if (p.lanes == 1) {
        const uint64_t working = (uint64_t)desc->bs << desc->wd;
        const uint64_t bytes = working * (is_tpcc ? TPCC_K : b->K) * (is_tpcc ? tpcc_lane_bytes() : ycsb_lane_bytes());
        smem = (size_t)(working * exec_th_bytes());
        if (smem + bytes <= GC_STAGE_SMEM_MAX) smem += (size_t)bytes;
        else ws_per_block = bytes;
    } else {   // TPC-C tile lanes keep their access entry in shared memory too (else global)
        smem = (size_t)block * exec_th_bytes();
        const uint64_t bytes = is_tpcc ? (uint64_t)block * tpcc_lane_bytes() : 0;
        if (smem + bytes <= GC_STAGE_SMEM_MAX) smem += (size_t)bytes;
        else ws_per_block = bytes;
    }
    int grid = (int)desc->grid;
    if (grid <= 0) {
        const int per_sm = is_tpcc ? tpcc_exec_max_blocks_per_sm(scheme, (int)p.lanes, block, smem)
                                   : ycsb_exec_max_blocks_per_sm(scheme, (int)p.lanes, block, smem);
        if (per_sm <= 0) return fail(db, CC_ERR_CONFIG, "executor cannot launch %d threads/block", block);
        grid = per_sm * db->num_sms;
    }
    if ((uint64_t)grid * block > (1ull << 21)) return fail(db, CC_ERR_CONFIG, "grid x block > 2^21 threads");
    if (ws_per_block) {
        const uint64_t need = ws_per_block * (uint64_t)grid;
        if (need > db->ws_bytes) {
            CUDA_TRY(db, cudaStreamSynchronize(db->stream));
            dfree(db->ws);
            db->ws = nullptr;
            db->ws_bytes = 0;
            CUDA_TRY(db, dalloc(&db->ws, need));
            db->ws_bytes = need;
        }
        p.ws = db->ws;
    }
    if (is_tpcc) CUDA_TRY(db, launch_tpcc_exec(p, tp, grid, block, smem, db->stream));
    else CUDA_TRY(db, launch_ycsb_exec(p, y, grid, block, smem, db->stream));
    if (persist) {
        cudaStreamAttrValue a{};
        a.accessPolicyWindow.num_bytes = 0;   // later work on the stream: normal caching
        CUDA_TRY(db, cudaStreamSetAttribute(db->stream, cudaStreamAttributeAccessPolicyWindow, &a));
    }
    if (!det) {   // this word set is zeroed for its next user while the next submit runs on the other
        const uint64_t words = scheme == CC_MVCC ? 2 * db->n_records : db->n_records * p.meta_stride;
        if (partitioned) {
            db->meta_dirty[mk] = words;   // phase B may still use it; zeroed in stream at reuse
        } else {
            CUDA_TRY(db, cudaEventRecord(db->meta_used[mk], db->stream));
            CUDA_TRY(db, cudaStreamWaitEvent(db->reset_stream, db->meta_used[mk], 0));
            CUDA_TRY(db, launch_zero_words(p.meta, words, db->reset_stream));
            CUDA_TRY(db, cudaEventRecord(db->meta_clean[mk], db->reset_stream));
            db->meta_cleaning[mk] = true;
            db->meta_cur = mk ^ 1;
        }
    }
    if (p.stages) CUDA_TRY(db, launch_stages_reduce(p.stages, (uint64_t)grid * block, db->stream));
    if (timing) CUDA_TRY(db, cudaEventRecord(ev.ev[3], db->stream));
    if (partitioned && p2p) {   // phase B through the windows, then a7: the submit is complete
        auto &P = db->part;
        const uint32_t wpr = db->tpcc.W / db->world;
        CUDA_TRY(db, p2p_phase_b(tp, db->rank, db->world, wpr, b->n_txn, P.skip, P.pt, P.win_cap, P.epoch, P.rc, P.recv,
                                 P.k1, P.k2, P.i1, P.i2, P.tmp, P.tmp_bytes, p.committed, p.order_hi, p.order_lo,
                                 p.read_out, db->ctl, p.watchdog_ns, db->stream));
        if (timing) CUDA_TRY(db, cudaEventRecord(ev.ev[3], db->stream));
        cc_result r = *res;
        if (!r.stats) r.stats = (uint64_t *)db->stats_scratch;
        CUDA_TRY(db, launch_finalize(p, r, db->prep, false, true, db->stream, false, false, nullptr,
                                     (uint64_t *)db->stats_scratch));
        if (rkind == 1) {
            cc_status st1 = copy_results_out(db, hk, res_in, b->n_txn, out_words);
            if (st1) return st1;
        }
        if (timing) {
            CUDA_TRY(db, cudaEventRecord(ev.ev[4], db->stream));
            db->pending.push_back(ev);
        }
        return CC_OK;
    }
    if (partitioned) {   // phase B happens in cc_part_apply / cc_part_finish
        db->part.pending = true;
        db->part.p = p;
        db->part.tp = tp;
        db->part.res = *res;
        db->part.b = b;
        db->part.timing = timing;
        db->part.ev = ev;
        db->part.two_pc = two_pc;
        db->part.round = 0;
        return CC_OK;
    }
    // a7: commit positions + result copy-out
    cc_result r = *res;
    if (!r.stats) r.stats = (uint64_t *)db->stats_scratch;
    const bool bitmap_rank = scheme == CC_TO || scheme == CC_MVCC || scheme == CC_SILO;
    if (bitmap_rank && !db->rank_bm.bits) {   // once per db: 512 MB for the 31-bit key range
        CUDA_TRY(db, cudaStreamSynchronize(db->stream));
        CUDA_TRY(db, dalloc(&db->rank_bm.bits, RANK_BITMAP_BITS / 8));
        CUDA_TRY(db, dalloc(&db->rank_bm.pre, RANK_BITMAP_BITS / 8));
        CUDA_TRY(db, dalloc(&db->rank_bm.csum, RANK_BITMAP_BITS / 32 / 1024 * 4 + 64));
    }
    CUDA_TRY(db, launch_finalize(p, r, db->prep, det, scheme == CC_TICTOC, db->stream,
                                 scheme == CC_TPL_NW || scheme == CC_TPL_WD, scheme == CC_TICTOC,
                                 bitmap_rank ? &db->rank_bm : nullptr, (uint64_t *)db->stats_scratch));
    if (used) {   // a later cc_prepare of this batch may overwrite the buffers after this point
        CUDA_TRY(db, cudaEventRecord(used->consumed, db->stream));
        used->has_consumer = true;
    }

    if (rkind == 1) {
        cc_status st1 = copy_results_out(db, hk, res_in, b->n_txn, out_words);
        if (st1) return st1;
    }
    if (timing) {
        CUDA_TRY(db, cudaEventRecord(ev.ev[4], db->stream));
        db->pending.push_back(ev);
    }
    return CC_OK;
}


cc_status cc_prepare(cc_db db, cc_batch b, cc_scheme scheme, uint32_t flags) {
    CHECK_DB(db);
    if (!b) return fail(db, CC_ERR_INVALID_ARG, "cc_prepare: null batch");
    if ((unsigned)scheme >= CC_NUM_SCHEMES) return fail(db, CC_ERR_INVALID_ARG, "bad scheme");
    if (scheme != CC_GPUTX && scheme != CC_GACCO) return CC_OK;   // nothing to prepare
    bool known = false;
    for (auto *x : db->batches) known |= x == b;
    if (!known || !b->ready) return fail(db, CC_ERR_INVALID_ARG, "cc_prepare: unknown batch");
    if (db->part.pending) return fail(db, CC_ERR_STATE, "partitioned submit pending");
    auto &q = b->prep[scheme == CC_GPUTX ? 0 : 1];
    const uint64_t n_acc = (uint64_t)b->n_txn * b->K;
    if (q.allocs.empty()) {
        CUDA_TRY(db, alloc_prep(q.b, q.allocs, n_acc < b->n_txn ? b->n_txn : n_acc, b->n_txn));
        CUDA_TRY(db, dalloc(&q.ctl, sizeof(Ctl)));
        CUDA_TRY(db, cudaEventCreateWithFlags(&q.done, cudaEventDisableTiming));
        CUDA_TRY(db, cudaEventCreateWithFlags(&q.consumed, cudaEventDisableTiming));
    }
    YcsbParams y{};
    TpccParams tp{};
    cc_status st = wl_params(db, b, flags, y, tp);
    if (st) return st;
    ExecParams p{};
    p.scheme = (int)scheme;
    p.n_txn = b->n_txn;
    p.K = b->K;
    p.flags = flags;
    p.ctl = q.ctl;
    p.watchdog_ns = 30000000000ull;
    cudaStream_t ps = db->prep_stream;
    CUDA_TRY(db, cudaStreamWaitEvent(ps, b->ready, 0));   // only the batch's own generation
    if (q.has_consumer) CUDA_TRY(db, cudaStreamWaitEvent(ps, q.consumed, 0));
    CUDA_TRY(db, cudaMemsetAsync(q.ctl, 0, sizeof(Ctl), ps));
    if (b->kind == KIND_TPCC) CUDA_TRY(db, launch_tpcc_gather(p, tp, q.b, db->n_records, ps));
    else CUDA_TRY(db, launch_ycsb_gather(p, y, q.b, ps));
    // the rank kernel shares the GPU with the executor: 1024-thread blocks on 1/8 of the SMs
    const int rg = db->num_sms / 8;
    CUDA_TRY(db, launch_prep_common(p, q.b, db->n_records, scheme == CC_GPUTX, rg > 0 ? rg : 1, ps, 1024));
    CUDA_TRY(db, cudaEventRecord(q.done, ps));
    q.valid = true;
    return CC_OK;
}

cc_status cc_part_send(cc_db db, const void **send, uint64_t *counts) {
    CHECK_DB(db);
    if (!db->part.pending || !send || !counts) return fail(db, CC_ERR_STATE, "no partitioned submit pending");
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    std::vector<unsigned long long> c(db->world);
    CUDA_TRY(db, cudaMemcpy(c.data(), db->part.cnt, db->world * 8ull, cudaMemcpyDeviceToHost));
    for (int k = 0; k < db->world; k++) counts[k] = c[k];
    *send = db->part.send;
    return CC_OK;
}

cc_status cc_part_apply(cc_db db, void *recv, uint64_t n, void *resp) {
    CHECK_DB(db);
    auto &P = db->part;
    if (!P.pending) return fail(db, CC_ERR_STATE, "no partitioned submit pending");
    if (n && (!recv || !resp)) return fail(db, CC_ERR_INVALID_ARG, "null buffers");
    if (n > P.recv_cap) {
        cudaStreamSynchronize(db->stream);
        dfree(P.k1); dfree(P.k2); dfree(P.i1); dfree(P.i2); dfree(P.tmp);
        CUDA_TRY(db, dalloc(&P.k1, n * 8));
        CUDA_TRY(db, dalloc(&P.k2, n * 8));
        CUDA_TRY(db, dalloc(&P.i1, n * 4));
        CUDA_TRY(db, dalloc(&P.i2, n * 4));
        P.tmp_bytes = part_sort_bytes(n);
        CUDA_TRY(db, dalloc((char **)&P.tmp, P.tmp_bytes));
        P.recv_cap = n;
    }
    if (P.two_pc) {   // PREPARE: grant per item in gid order, vote in resp[k].v[5]
        if (n > P.vote_cap) {
            cudaStreamSynchronize(db->stream);
            dfree(P.vote);
            P.vote = nullptr;
            CUDA_TRY(db, dalloc(&P.vote, n));
            P.vote_cap = n;
        }
        const bool ts_rule = P.p.scheme != CC_TPL_NW && P.p.scheme != CC_TPL_WD;
        CUDA_TRY(db, part_grant((PartReq *)recv, n, P.tp, (PartResp *)resp, P.vote, P.k1, P.k2, P.i1, P.i2,
                                P.tmp, P.tmp_bytes, db->ctl, db->stream, ts_rule));
        return CC_OK;
    }
    CUDA_TRY(db, part_apply((PartReq *)recv, n, P.tp, (PartResp *)resp, P.k1, P.k2, P.i1, P.i2, P.tmp,
                            P.tmp_bytes, db->ctl, db->stream));
    return CC_OK;
}

cc_status cc_part_decide(cc_db db, const void *resp, uint64_t n_sent, const void **dec) {
    CHECK_DB(db);
    auto &P = db->part;
    if (!P.pending || !P.two_pc) return fail(db, CC_ERR_STATE, "no 2PC partitioned submit pending");
    if (!dec || (n_sent && !resp)) return fail(db, CC_ERR_INVALID_ARG, "null buffers");
    const uint32_t wpr = db->tpcc.W / db->world;
    CUDA_TRY(db, part_decide(P.tp, db->rank, db->world, wpr, P.b->n_txn, P.skip, P.send, (const PartResp *)resp,
                             n_sent, P.stage, P.p.committed, P.p.order_hi, P.p.order_lo, P.p.read_out,
                             P.p.restarts, P.round, P.dec, db->stream));
    *dec = P.dec;
    return CC_OK;
}

cc_status cc_part_commit(cc_db db, const void *recv, const void *dec, uint64_t n) {
    CHECK_DB(db);
    auto &P = db->part;
    if (!P.pending || !P.two_pc) return fail(db, CC_ERR_STATE, "no 2PC partitioned submit pending");
    if (n && (!recv || !dec)) return fail(db, CC_ERR_INVALID_ARG, "null buffers");
    if (n > P.vote_cap) return fail(db, CC_ERR_INVALID_ARG, "more decisions than requests granted this round");
    CUDA_TRY(db, part_commit((const PartReq *)recv, n, P.vote, (const unsigned long long *)dec, P.tp, db->stream));
    return CC_OK;
}

cc_status cc_part_next(cc_db db, uint64_t *pending) {
    CHECK_DB(db);
    auto &P = db->part;
    if (!P.pending || !P.two_pc) return fail(db, CC_ERR_STATE, "no 2PC partitioned submit pending");
    if (!pending) return fail(db, CC_ERR_INVALID_ARG, "null pending");
    const uint32_t wpr = db->tpcc.W / db->world;
    CUDA_TRY(db, part_repack(P.tp, db->rank, db->world, wpr, P.b->n_txn, P.skip, P.cnt, P.off, P.cursor, P.send,
                             db->stream));
    unsigned long long c = 0;
    CUDA_TRY(db, cudaMemcpyAsync(&c, P.cnt + db->world, 8, cudaMemcpyDeviceToHost, db->stream));
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    *pending = c;
    P.round++;
    return CC_OK;
}

cc_status cc_part_finish(cc_db db, const void *resp, uint64_t n_sent) {
    CHECK_DB(db);
    auto &P = db->part;
    if (!P.pending) return fail(db, CC_ERR_STATE, "no partitioned submit pending");
    const uint32_t wpr = db->tpcc.W / db->world;
    CUDA_TRY(db, part_finish(P.tp, db->rank, db->world, wpr, P.b->n_txn, P.skip, P.send, (const PartResp *)resp,
                             n_sent, P.stage, P.p.committed, P.p.order_hi, P.p.order_lo, P.p.read_out,
                             db->stream, P.two_pc));
    if (P.timing) CUDA_TRY(db, cudaEventRecord(P.ev.ev[3], db->stream));
    cc_result r = P.res;
    if (!r.stats) r.stats = (uint64_t *)db->stats_scratch;
    CUDA_TRY(db, launch_finalize(P.p, r, db->prep, false, true, db->stream, false, false, nullptr,
                                 (uint64_t *)db->stats_scratch));
    if (P.timing) {
        CUDA_TRY(db, cudaEventRecord(P.ev.ev[4], db->stream));
        db->pending.push_back(P.ev);
    }
    P.pending = false;
    return CC_OK;
}

// ---------------------------------------------------------------- P2P exchange windows
static cc_status ensure_window(cc_db db) {
    auto &P = db->part;
    if (P.win) return CC_OK;
    if (!db->tpcc.loaded) return fail(db, CC_ERR_CONFIG, "cc_part_window: TPC-C not loaded");
    if (db->world > P2P_MAXW) return fail(db, CC_ERR_CONFIG, "cc_part_window: at most %d ranks", P2P_MAXW);
    P.win_txn = db->tpcc.max_txn;
    P.win_cap = P.win_txn * TPCC_K;   // a source can send at most every access of its batch
    const size_t bytes = p2p_window_bytes(db->world, P.win_cap, P.win_txn);
    CUDA_TRY(db, dalloc(&P.win, bytes));
    CUDA_TRY(db, cudaMemsetAsync(P.win, 0, P2P_FLAG_BYTES, db->stream));
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    return CC_OK;
}

static void window_ptrs(void *base, uint32_t world, uint32_t cap, PartReq **inbox, PartResp **stage,
                        unsigned long long **flags) {
    char *b = (char *)base;
    *flags = (unsigned long long *)b;
    *inbox = (PartReq *)(b + P2P_FLAG_BYTES);
    *stage = (PartResp *)(b + P2P_FLAG_BYTES + (size_t)world * cap * sizeof(PartReq));
}

static void preload_all_kernels() {
    static std::atomic<uint64_t> done{0};   // once per device (modules load per context)
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load() & bit) return;
    preload_prep_kernels();
    preload_sort_kernels();
    preload_part_kernels();
    preload_tpcc_kernels();
    preload_ycsb_kernels();
    done |= bit;
}

static cc_status p2p_buffers(cc_db db) {
    preload_all_kernels();
    auto &P = db->part;
    const uint64_t capn = (uint64_t)db->world * P.win_cap;
    if (!P.rc) CUDA_TRY(db, dalloc(&P.rc, (2ull * db->world + 1) * 8));
    if (!P.recv) CUDA_TRY(db, dalloc(&P.recv, capn * sizeof(PartReq)));
    if (capn > P.recv_cap) {   // sort buffers of phase B (shared with the host-driven exchange)
        CUDA_TRY(db, cudaStreamSynchronize(db->stream));
        dfree(P.k1); dfree(P.k2); dfree(P.i1); dfree(P.i2); dfree(P.tmp);
        CUDA_TRY(db, dalloc(&P.k1, capn * 8));
        CUDA_TRY(db, dalloc(&P.k2, capn * 8));
        CUDA_TRY(db, dalloc(&P.i1, capn * 4));
        CUDA_TRY(db, dalloc(&P.i2, capn * 4));
        P.tmp_bytes = part_sort_bytes(capn);
        CUDA_TRY(db, dalloc((char **)&P.tmp, P.tmp_bytes));
        P.recv_cap = capn;
    }
    cc_status st = ensure_part(db, P.win_txn);
    if (st) return st;
    // everything a P2P submit of up to win_txn transactions can need is allocated now: a
    // cudaMalloc inside a submit may block the host until the device idles, while another
    // rank's kernels of this process already wait on the device for this rank's requests
    st = ensure_scratch(db, P.win_txn, (uint64_t)P.win_txn * TPCC_K);
    if (st) return st;
    st = ensure_arena(db, (uint64_t)P.win_txn * TPCC_K, TPCC_C_WORDS);
    if (st) return st;
    st = ensure_hres(db, P.win_txn, TPCC_OUT_WORDS);   // host-memory results of a P2P submit
    if (st) return st;
    P.connected = true;
    return CC_OK;
}

cc_status cc_part_window(cc_db db, cc_ipc_handle *out) {
    CHECK_DB(db);
    if (!out) return fail(db, CC_ERR_INVALID_ARG, "null handle");
    cc_status st = ensure_window(db);
    if (st) return st;
    cudaIpcMemHandle_t h;
    CUDA_TRY(db, cudaIpcGetMemHandle(&h, db->part.win));
    static_assert(sizeof(h) == sizeof(out->ipc), "IPC handle size");
    memcpy(out->ipc, &h, sizeof h);
    out->rank = (uint32_t)db->rank;
    out->world = (uint32_t)db->world;
    out->cap = db->part.win_cap;
    out->max_txn = db->part.win_txn;
    return CC_OK;
}

cc_status cc_part_connect(cc_db db, const cc_ipc_handle *handles) {
    CHECK_DB(db);
    auto &P = db->part;
    if (!handles) return fail(db, CC_ERR_INVALID_ARG, "null handles");
    cc_status st = ensure_window(db);
    if (st) return st;
    if (P.connected) return fail(db, CC_ERR_STATE, "cc_part_connect: already connected");
    for (int r = 0; r < db->world; r++) {
        const cc_ipc_handle &h = handles[r];
        if (h.rank != (uint32_t)r || h.world != (uint32_t)db->world || h.cap != P.win_cap || h.max_txn != P.win_txn)
            return fail(db, CC_ERR_CONFIG, "cc_part_connect: handle %d does not match this db's window", r);
        void *base = P.win;
        if (r != db->rank) {
            cudaIpcMemHandle_t ih;
            memcpy(&ih, h.ipc, sizeof ih);
            CUDA_TRY(db, cudaIpcOpenMemHandle(&base, ih, cudaIpcMemLazyEnablePeerAccess));
            P.ipc_open.push_back(base);
        }
        window_ptrs(base, db->world, P.win_cap, &P.pt.inbox[r], &P.pt.stage[r], &P.pt.flags[r]);
    }
    return p2p_buffers(db);
}

cc_status cc_part_connect_local(cc_db *dbs, int n) {
    if (!dbs || n < 1 || n > P2P_MAXW) return CC_ERR_INVALID_ARG;
    for (int r = 0; r < n; r++) {
        cc_db db = dbs[r];
        CHECK_DB(db);
        if (db->rank != r || db->world != n) return fail(db, CC_ERR_CONFIG, "cc_part_connect_local: db %d is not rank %d of %d", r, r, n);
        cc_status st = ensure_window(db);
        if (st) return st;
        if (db->part.connected) return fail(db, CC_ERR_STATE, "cc_part_connect_local: already connected");
    }
    for (int r = 0; r < n; r++) {
        auto &P = dbs[r]->part;
        for (int q = 0; q < n; q++) {
            const auto &Q = dbs[q]->part;
            if (Q.win_cap != P.win_cap || Q.win_txn != P.win_txn) return fail(dbs[r], CC_ERR_CONFIG, "window shapes differ");
            window_ptrs(Q.win, n, Q.win_cap, &P.pt.inbox[q], &P.pt.stage[q], &P.pt.flags[q]);
        }
        cudaSetDevice(dbs[r]->device);
        cc_status st = p2p_buffers(dbs[r]);
        if (st) return st;
    }
    return CC_OK;
}

cc_status cc_events_capacity(cc_db db, uint64_t cap) {
    CHECK_DB(db);
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    dfree(db->events);
    db->events = nullptr;
    db->events_cap = 0;
    if (cap) {
        CUDA_TRY(db, dalloc(&db->events, cap * sizeof(Event)));
        db->events_cap = cap;
    }
    return CC_OK;
}

cc_status cc_events_read(cc_db db, void *dst, uint64_t cap, uint64_t *n_events) {
    CHECK_DB(db);
    if (!n_events) return fail(db, CC_ERR_INVALID_ARG, "null n_events");
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    Ctl c;
    CUDA_TRY(db, cudaMemcpy(&c, db->ctl, sizeof c, cudaMemcpyDeviceToHost));
    *n_events = c.events.v;
    uint64_t n = c.events.v < cap ? c.events.v : cap;
    if (n > db->events_cap) n = db->events_cap;
    if (n && dst) CUDA_TRY(db, cudaMemcpy(dst, db->events, n * sizeof(Event), cudaMemcpyDeviceToHost));
    return CC_OK;
}

static cc_status drain_timing(cc_db db) {
    for (auto &pe : db->pending) {
        float ms[4];
        for (int i = 0; i < 4; i++) CUDA_TRY(db, cudaEventElapsedTime(&ms[i], pe.ev[i], pe.ev[i + 1]));
        float tot;
        CUDA_TRY(db, cudaEventElapsedTime(&tot, pe.ev[0], pe.ev[4]));
        for (int i = 0; i < 4; i++) db->acc[i] += ms[i];
        db->acc[4] += tot;
        db->n_timed++;
        db->free_events.push_back(pe);
    }
    db->pending.clear();
    return CC_OK;
}

cc_status cc_join(cc_db db) {
    CHECK_DB(db);
    for (int k = 0; k < 2; k++)
        if (db->meta_cleaning[k]) CUDA_TRY(db, cudaStreamWaitEvent(db->stream, db->meta_clean[k], 0));
    return CC_OK;
}

cc_status cc_sync(cc_db db, cc_stats *out) {
    CHECK_DB(db);
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    CUDA_TRY(db, cudaStreamSynchronize(db->reset_stream));
    CUDA_TRY(db, cudaStreamSynchronize(db->copy_stream));   // host-memory results of the submits
    CUDA_TRY(db, cudaGetLastError());
    u64 w[CC_STATS_WORDS];
    CUDA_TRY(db, cudaMemcpy(w, db->stats_scratch, sizeof w, cudaMemcpyDeviceToHost));
    cc_stats s{};
    s.commits = w[0];
    s.aborts = w[1];
    s.attempts = w[2];
    s.error = w[3];
    s.max_rank = w[4];
    s.ts_last = w[5];
    for (int k = 0; k < 7; k++) s.stage_cycles[k] = w[8 + k];
    s.sm_clock_khz = (uint64_t)db->clock_khz;
    db->last = s;
    if (out) *out = s;
    Ctl c;
    CUDA_TRY(db, cudaMemcpy(&c, db->ctl, sizeof c, cudaMemcpyDeviceToHost));
    u64 sticky = 0;
    CUDA_TRY(db, cudaMemcpy(&sticky, db->sticky_dev, 8, cudaMemcpyDeviceToHost));
    CUDA_TRY(db, cudaMemset(db->sticky_dev, 0, 8));
    const u64 e = sticky ? sticky : (c.err.v ? c.err.v : w[3]);
    if (e) {
        static const char *names[] = {"ok", "invalid arg", "config", "oom", "cuda", "nccl",
                                      "key not found", "timestamp overflow", "version exhausted",
                                      "watchdog timeout", "state", "unsupported"};
        return fail(db, (cc_status)e, "device reported: %s", e < 12 ? names[e] : "?");
    }
    return CC_OK;
}

cc_status cc_timing_read(cc_db db, double ms[5], uint64_t *n_submits, int reset) {
    CHECK_DB(db);
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    cc_status st = drain_timing(db);
    if (st) return st;
    if (ms) for (int i = 0; i < 5; i++) ms[i] = db->acc[i];
    if (n_submits) *n_submits = db->n_timed;
    if (reset) {
        for (double &a : db->acc) a = 0;
        db->n_timed = 0;
    }
    return CC_OK;
}

cc_status cc_snapshot(cc_db db, int save) {
    CHECK_DB(db);
    if (save) {
        for (void *p : db->snap) dfree(p);
        db->snap.clear();
        for (auto &t : db->tables) {
            void *p = nullptr;
            CUDA_TRY(db, dalloc(&p, (size_t)t.row_bytes * t.rows));
            db->snap.push_back(p);
            CUDA_TRY(db, cudaMemcpyAsync(p, t.d, (size_t)t.row_bytes * t.rows, cudaMemcpyDeviceToDevice,
                                         db->stream));
        }
    } else {
        if (db->snap.size() != db->tables.size()) return fail(db, CC_ERR_CONFIG, "no snapshot saved");
        for (size_t i = 0; i < db->tables.size(); i++) {
            auto &t = db->tables[i];
            CUDA_TRY(db, cudaMemcpyAsync(t.d, db->snap[i], (size_t)t.row_bytes * t.rows,
                                         cudaMemcpyDeviceToDevice, db->stream));
        }
    }
    return CC_OK;
}

cc_status cc_roofline_probe(cc_db db, cc_roofline *out) {
    CHECK_DB(db);
    if (!out) return fail(db, CC_ERR_INVALID_ARG, "null output");
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    double v[6] = {0, 0, 0, 0, 0, 0};
    CUDA_TRY(db, roofline_probe(db->stream, db->num_sms, v));
    out->gather_gbs = v[0];
    out->cas_l2_per_s = v[1];
    out->cas_hbm_per_s = v[2];
    out->handoff_row_ns = v[3];
    out->handoff_ns = v[4];
    out->handoff_acq_row_ns = v[5];
    return CC_OK;
}

cc_status cc_gather_sweep(cc_db db, double gbs[4]) {
    CHECK_DB(db);
    if (!gbs) return fail(db, CC_ERR_INVALID_ARG, "null output");
    CUDA_TRY(db, cudaStreamSynchronize(db->stream));
    for (int k = 0; k < 4; k++) gbs[k] = 0;
    CUDA_TRY(db, gather_sweep(db->stream, db->num_sms, gbs));
    return CC_OK;
}

}  // extern "C"
