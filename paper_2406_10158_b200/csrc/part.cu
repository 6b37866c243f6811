// part.cu -- warehouse-partitioned TPC-C across GPUs.
//
// Rank g owns warehouses [w_first, w_first + w_count).  A transaction runs on the
// owner of its home warehouse.  Phase A: transactions whose every access is local run
// under the chosen CC scheme (the normal executor; distributed ones are skipped).
// Phase B: every access of a distributed transaction becomes a request to the item's
// owner (all-to-all #1).  Every TPC-C write is a read-modify-write of one item that
// depends only on that item and the transaction's inputs, so each owner sorts the
// requests it received by (item, global gid) and applies each item's chain in gid
// order -- one thread per item, no locks -- returning the value each access read
// (all-to-all #2).  The home rank assembles outputs and the reserved O/NO/OL/H slots.
// Result: Phase A (any interleaving across ranks: disjoint data) then Phase B in global
// gid order, a serial order; the order key is (rank << 48 | scheme key) for Phase A
// and (1 << 63, gid) for Phase B.

#include "exec.cuh"
#include "tpcc.h"

namespace gcctb {

struct PartDev {
    uint32_t rank, world, wpr;   // warehouses per rank (contiguous ranges)
    uint32_t n_local;            // local transactions per rank (gid_global = rank*n_local + gid)
};

__device__ __forceinline__ uint32_t owner_of(const PartDev &pd, uint32_t w) { return w / pd.wpr; }

// ---------------------------------------------------------------- classify
__global__ void part_classify_kernel(TpccParams y, PartDev pd, uint32_t n_txn, uint8_t *skip,
                                     unsigned long long *n_req_dest /*[world]*/, bool all) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_txn) return;
    const uint32_t *t = y.tx + (u64)g * TPCC_TX_WORDS;
    bool dist = all;
    if (t[TX_TYPE] == 0) {
        for (uint32_t j = 0; j < t[TX_OLCNT]; j++) dist |= owner_of(pd, t[TX_SUPQ + j] >> 8) != pd.rank;
    } else {
        dist |= owner_of(pd, t[TX_CW]) != pd.rank;
    }
    skip[g] = dist ? 1 : 0;
    if (!dist) return;
    // count requests per destination (W, D home; C at c_w's owner; stock at supply_w's owner)
    const uint32_t n = t[TX_TYPE] == 0 ? 3 + t[TX_OLCNT] : 3;
    for (uint32_t i = 0; i < n; i++) {
        uint32_t dest = pd.rank;
        if (i == 2 && t[TX_TYPE] == 1) dest = owner_of(pd, t[TX_CW]);
        if (i >= 3) dest = owner_of(pd, t[TX_SUPQ + i - 3] >> 8);
        atomicAdd(&n_req_dest[dest], 1ull);
    }
}

__global__ void part_scan_kernel(const unsigned long long *cnt, unsigned long long *off,
                                 unsigned long long *cursor, uint32_t world) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        unsigned long long s = 0;
        for (uint32_t k = 0; k < world; k++) {
            off[k] = s;
            cursor[k] = s;
            s += cnt[k];
        }
        off[world] = s;
    }
}

__global__ void part_pack_kernel(TpccParams y, PartDev pd, uint32_t n_txn, const uint8_t *skip,
                                 unsigned long long *cursor, PartReq *out) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_txn || skip[g] != 1) return;   // 0: local (phase A), 2: done (2PC)
    const uint32_t *t = y.tx + (u64)g * TPCC_TX_WORDS;
    const uint32_t type = t[TX_TYPE], w = t[TX_W], d = t[TX_D];
    const uint32_t n = type == 0 ? 3 + t[TX_OLCNT] : 3;
    for (uint32_t i = 0; i < n; i++) {
        PartReq r{};
        r.gid = pd.rank * pd.n_local + g;
        r.home = pd.rank | (i << 16);
        r.type_d = type | (d << 8);
        r.home_w = w | (d << 16);
        r.last = 0xFFFFFFFFu;
        uint32_t dest = pd.rank;
        const uint32_t lw = w - pd.rank * pd.wpr;
        if (i == 0) {
            r.kind = 0;
            r.row = lw;
            r.amount = type == 1 ? t[TX_HAMT] : 0;
        } else if (i == 1) {
            r.kind = 1;
            r.row = lw * TPCC_DIST + d;
            r.amount = type == 1 ? t[TX_HAMT] : 0;
        } else if (i == 2) {
            r.kind = 2;
            const uint32_t cw = type == 0 ? w : t[TX_CW], cd = type == 0 ? d : t[TX_CD];
            dest = owner_of(pd, cw);
            const uint32_t lcw = cw - dest * pd.wpr;
            r.cust = lcw * TPCC_DIST + cd;
            r.c_ids = cw | (cd << 16);
            r.amount = type == 1 ? t[TX_HAMT] : 0;
            if (t[TX_C] == 0xFFFFFFFFu) {
                r.row = 0xFFFFFFFFu;
                r.last = t[TX_CLAST];
            } else {
                r.row = r.cust * TPCC_CUST + t[TX_C];
            }
        } else {
            r.kind = 3;
            const uint32_t sw = t[TX_SUPQ + i - 3] >> 8;
            dest = owner_of(pd, sw);
            r.row = (sw - dest * pd.wpr) * TPCC_STOCK + t[TX_ITEM + i - 3];
            r.amount = t[TX_SUPQ + i - 3] & 0xFF;
            r.type_d |= (sw != w ? 1u : 0u) << 16;
        }
        const unsigned long long pos = atomicAdd(&cursor[dest], 1ull);
        out[pos] = r;
    }
}

// ---------------------------------------------------------------- apply (owner side)
// resolve by-name customers on the owner's immutable index, then build sort keys
// (kind << 60) | (row << 24) | (gid mod 2^24)
__global__ void part_keys_kernel(PartReq *req, uint64_t n, TpccParams y, unsigned long long *keys,
                                 uint32_t *idx, Ctl *ctl, const unsigned long long *n_dev = nullptr) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (n_dev ? *n_dev : n)) return;
    PartReq &r = req[k];
    if (r.kind == 2 && r.row == 0xFFFFFFFFu) {
        const uint32_t grp = r.cust * 1000u + r.last;
        const uint32_t c = y.nidx_count[grp];
        if (c == 0) {
            atomicCAS(&ctl->err.v, 0ull, (u64)CC_ERR_KEY_NOT_FOUND);
            r.row = 0;
        } else {
            r.row = y.nidx_rows[y.nidx_start[grp] + (c + 1) / 2 - 1];   // ceil(n/2), §2.5.2.2
        }
    }
    keys[k] = ((u64)r.kind << 60) | ((u64)r.row << 24) | (u64)(r.gid & 0xFFFFFFu);
    idx[k] = (uint32_t)k;
}

// One phase-B access on the owner: the values it reads (its response) and, if `apply`,
// its read-modify-write of the row.  Responses are identical with or without `apply`
// (2PC computes them at grant time and writes at commit time; the row cannot change in
// between, the grant being exclusive).
__device__ bool part_is_write(const PartReq &r) {
    return r.kind == 1 || r.kind == 3 || (r.type_d & 1u);   // D, S always; W, C for Payment
}

__device__ PartResp part_access(const PartReq &r, const TpccParams &y, bool apply) {
    PartResp o{};
    const bool pay = r.type_d & 1u;
    if (r.kind == 0) {
        u64 *w = y.wh + (u64)r.row * TPCC_W_WORDS;
        if (pay) {
            if (apply) w[0] += r.amount;             // w_ytd += h
            o.v[0] = w[2];
            o.v[1] = w[3];                           // w_name
        } else {
            o.v[0] = (uint32_t)w[1];                 // w_tax
        }
    } else if (r.kind == 1) {
        u64 *d = y.di + (u64)r.row * TPCC_D_WORDS;
        if (pay) {
            if (apply) d[0] += r.amount;             // d_ytd += h
            o.v[0] = d[2];
            o.v[1] = d[3];                           // d_name
        } else {
            const u64 w1 = d[1];
            o.v[0] = (uint32_t)w1;                   // d_tax
            o.v[1] = w1 >> 32;                       // o_id = d_next_o_id
            if (apply) d[1] = (w1 & 0xFFFFFFFFull) | (((w1 >> 32) + 1) << 32);
        }
    } else if (r.kind == 2) {
        u64 *c = y.cu + (u64)r.row * TPCC_C_WORDS;
        const u64 w3 = c[3];
        if (pay) {
            const u64 h = r.amount;
            const u64 bal = c[0] - h;
            if (apply) {
                c[0] = bal;
                c[1] += h;
                c[2] = (c[2] & ~0xFFFFFFFFull) | (u64)((uint32_t)c[2] + 1);
                if (((w3 >> 32) & 0xFFFF) == 0x4342) {   // "BC" (R7)
                    u64 *cd = c + TPCC_CDATA_OFF;
                    for (int k = TPCC_CDATA_WORDS - 1; k >= 4; k--) cd[k] = cd[k - 4];
                    const u64 cc = r.row % TPCC_CUST;
                    cd[0] = (cc + 1) | ((u64)((r.c_ids >> 16) + 1) << 32);
                    cd[1] = (u64)((r.c_ids & 0xFFFF) + 1) | ((u64)((r.home_w >> 16) + 1) << 32);
                    cd[2] = (u64)(r.home_w & 0xFFFF) + 1;
                    cd[3] = h;
                }
            }
            o.v[0] = r.row % TPCC_CUST;
            o.v[1] = bal;
        }
        o.v[2] = w3;
    } else {
        u64 *s = y.st + (u64)r.row * TPCC_S_WORDS;
        const u64 w0 = s[0];
        const uint32_t q = (uint32_t)w0, qty = r.amount;
        if (apply) {
            const uint32_t nq = (q >= qty + 10) ? q - qty : q - qty + 91;
            s[0] = (u64)nq | ((u64)((uint32_t)(w0 >> 32) + 1) << 32);
            s[1] += qty;
            if ((r.type_d >> 16) & 1u) s[2] = (s[2] & ~0xFFFFFFFFull) | (u64)((uint32_t)s[2] + 1);
        }
        const uint32_t dd = (r.type_d >> 8) & 0xFF;
        o.v[0] = q;
        bool orig = false;
        const uint8_t *sd = reinterpret_cast<const uint8_t *>(s + 33);
        for (int i = 0; i + 8 <= 50 && !orig; i++) {
            bool m = true;
            for (int k = 0; k < 8 && m; k++) m = sd[i + k] == (uint8_t)"ORIGINAL"[k];
            orig = m;
        }
        o.v[1] = orig;
        o.v[2] = s[3 + 3 * dd];
        o.v[3] = s[4 + 3 * dd];
        o.v[4] = s[5 + 3 * dd];
    }
    return o;
}

// one thread per item chain: apply the accesses in gid order, recording what each read
__global__ void part_chain_kernel(const unsigned long long *skeys, const uint32_t *sidx, uint64_t n,
                                  const PartReq *req, TpccParams y, PartResp *resp) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    if (p > 0 && (skeys[p - 1] >> 24) == (skeys[p] >> 24)) return;   // chain head only
    for (uint64_t q = p; q < n && (skeys[q] >> 24) == (skeys[p] >> 24); q++)
        resp[sidx[q]] = part_access(req[sidx[q]], y, true);
}

// ---------------------------------------------------------------- 2PC rounds (f-2)
// Scheme-native phase B for the 2PL family.  A round is 2PC:
// PREPARE -- each owner grants the round's lock requests item by item in global gid order,
// no-wait (a shared request is granted unless an exclusive one was, an exclusive one only
// on a free item) and answers with the values read plus the vote (v[5]); DECIDE -- the home
// commits a transaction iff every access was granted, assembles it, and sends the decision
// of every access back; COMMIT -- owners install the granted writes of committed
// transactions.  Locks live for one round (granted at prepare, released when the round
// ends), so the transactions committed in one round held all their locks together and are
// conflict-free: the order key is (2^63 | round, global gid).  The oldest pending
// transaction wins every item it asks for, so every round commits at least one (wait-die's
// priority: the older proceeds, the younger dies and retries next round).
// ts_rule (TO / MVCC / Silo / TicToc): with the round's timestamps (round, gid) every
// item's chain is in timestamp order, so the only conflict left inside a round is an access
// behind an older granted (pending) write -- TO makes it wait, MVCC's reader of an older
// pending version waits for it, OCC's writer holds the write lock and a reader behind it
// fails validation: it is denied and retries next round.  A write behind granted older
// reads is in timestamp order and is granted (2PL refuses it: the shared holders).  The
// committed set of a round is serializable in (round, gid) order, and the oldest pending
// transaction is granted everything, so every round commits at least one.
__global__ void part_grant_kernel(const unsigned long long *skeys, const uint32_t *sidx, uint64_t n,
                                  const PartReq *req, TpccParams y, PartResp *resp, uint8_t *vote,
                                  bool ts_rule) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    if (p > 0 && (skeys[p - 1] >> 24) == (skeys[p] >> 24)) return;   // chain head only
    bool ex = false;
    uint32_t sh = 0;
    for (uint64_t q = p; q < n && (skeys[q] >> 24) == (skeys[p] >> 24); q++) {
        const PartReq &r = req[sidx[q]];
        const bool w = part_is_write(r);
        const bool g = (w && !ts_rule) ? (!ex && sh == 0) : !ex;
        if (g) {
            if (w) ex = true;
            else sh++;
        }
        PartResp o = part_access(r, y, false);
        o.v[5] = g;
        resp[sidx[q]] = o;
        vote[sidx[q]] = g;
    }
}

__global__ void part_commit_kernel(const PartReq *req, uint64_t n, const uint8_t *vote,
                                   const unsigned long long *dec, TpccParams y) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    if (vote[k] && dec[k] && part_is_write(req[k])) part_access(req[k], y, true);
}

// ---------------------------------------------------------------- finish (home side)
__global__ void part_stage_kernel(const PartReq *sent, const PartResp *resp, uint64_t n, PartDev pd,
                                  PartResp *stage) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t g = sent[k].gid - pd.rank * pd.n_local, lane = sent[k].home >> 16;
    stage[(u64)g * TPCC_K + lane] = resp[k];
}

__device__ __forceinline__ bool item_original(const u64 *ir) {
    const uint8_t *s = reinterpret_cast<const uint8_t *>(ir + 4);
    for (int i = 0; i + 8 <= 50; i++) {
        bool m = true;
        for (int k = 0; k < 8 && m; k++) m = s[i + k] == (uint8_t)"ORIGINAL"[k];
        if (m) return true;
    }
    return false;
}

// assemble outputs + reserved slots of one distributed transaction from its accesses'
// responses (same formulas as the executor's emission) and mark it committed with `hi`
__device__ void part_assemble_one(const TpccParams &y, const PartDev &pd, uint32_t g, const PartResp *st,
                                  uint8_t *committed, unsigned long long *ohi, unsigned long long *olo,
                                  unsigned long long *read_out, u64 hi) {
    const uint32_t *t = y.tx + (u64)g * TPCC_TX_WORDS;
    u64 *out = read_out ? read_out + (u64)g * TPCC_OUT_WORDS : nullptr;
    const uint32_t w = t[TX_W], d = t[TX_D];
    if (t[TX_TYPE] == 0) {
        const u64 w_tax = st[0].v[0], d_tax = st[1].v[0], o_id = st[1].v[1], disc = (uint32_t)st[2].v[2];
        const uint32_t n = t[TX_OLCNT];
        u64 sum = 0;
        for (uint32_t j = 0; j < n; j++) {
            const uint32_t i = t[TX_ITEM + j], sw = t[TX_SUPQ + j] >> 8, qty = t[TX_SUPQ + j] & 0xFF;
            const u64 *ir = y.it + (u64)i * TPCC_I_WORDS;
            const u64 amount = (u64)qty * (uint32_t)ir[0];
            sum += amount;
            const PartResp &s = st[3 + j];
            u64 *ol = y.ol + ((u64)g * TPCC_MAXOL + j) * TPCC_OL_WORDS;
            ol[0] = o_id | ((u64)(j + 1) << 32);
            ol[1] = (u64)(d + 1) | ((u64)(w + 1) << 32);
            ol[2] = (u64)(i + 1) | ((u64)(sw + 1) << 32);
            ol[3] = qty;
            ol[4] = amount;
            ol[5] = s.v[2];
            ol[6] = s.v[3];
            ol[7] = s.v[4];
            if (out) {
                out[2 + 3 * j] = s.v[0];
                out[3 + 3 * j] = (s.v[1] && item_original(ir)) ? 'B' : 'G';
                out[4 + 3 * j] = amount;
            }
        }
        u64 *o = y.o + (u64)g * TPCC_O_WORDS;
        o[0] = o_id; o[1] = d + 1; o[2] = w + 1; o[3] = t[TX_C] + 1; o[4] = y.entry_date; o[5] = n;
        o[6] = t[TX_ALLLOCAL]; o[7] = 0;
        u64 *no = y.no + (u64)g * TPCC_NO_WORDS;
        no[0] = o_id; no[1] = d + 1; no[2] = w + 1; no[3] = 0;
        if (out) {
            const long long num = (long long)sum * (long long)(10000 - disc) * (long long)(10000 + w_tax + d_tax);
            out[0] = o_id;
            out[1] = (u64)((num + 50000000ll) / 100000000ll);
        }
    } else {
        const u64 c1 = st[2].v[0] + 1;
        u64 *h = y.h + (u64)g * TPCC_H_WORDS;
        h[0] = c1 | ((u64)(t[TX_CD] + 1) << 32);
        h[1] = (u64)(t[TX_CW] + 1) | ((u64)(d + 1) << 32);
        h[2] = (u64)w + 1;
        h[3] = y.entry_date;
        h[4] = t[TX_HAMT];
        h[5] = st[0].v[0];
        h[6] = (st[0].v[1] & 0xFFFFull) | (0x20202020ull << 16) | ((st[1].v[0] & 0xFFFFull) << 48);
        h[7] = (st[1].v[0] >> 16) | ((st[1].v[1] & 0xFFFFull) << 48);
        if (out) {
            out[0] = c1;
            out[1] = st[2].v[1];
            out[2] = (st[2].v[2] >> 32) & 0xFFFF;
        }
    }
    committed[g] = 1;
    ohi[g] = hi;
    olo[g] = (u64)pd.rank * pd.n_local + g;
}

// Phase A keys get the rank prefix; distributed transactions (deterministic phase B) are
// assembled with key (2^63, gid).  In 2PC mode they were assembled round by round.
__global__ void part_assemble_kernel(TpccParams y, PartDev pd, uint32_t n_txn, const uint8_t *skip,
                                     const PartResp *stage, uint8_t *committed, unsigned long long *ohi,
                                     unsigned long long *olo, unsigned long long *read_out, bool two_pc) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_txn) return;
    if (!skip[g]) {
        ohi[g] |= (u64)pd.rank << 48;
        return;
    }
    if (two_pc) return;
    part_assemble_one(y, pd, g, stage + (u64)g * TPCC_K, committed, ohi, olo, read_out, 1ull << 63);
}

// 2PC DECIDE (home): commit iff every access of the transaction was granted this round
__global__ void part_decide_kernel(TpccParams y, PartDev pd, uint32_t n_txn, uint8_t *skip, const PartResp *stage,
                                   uint8_t *committed, unsigned long long *ohi, unsigned long long *olo,
                                   unsigned long long *read_out, uint32_t *restarts, uint32_t round) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_txn || skip[g] != 1) return;
    const uint32_t *t = y.tx + (u64)g * TPCC_TX_WORDS;
    const uint32_t n = t[TX_TYPE] == 0 ? 3 + t[TX_OLCNT] : 3;
    const PartResp *st = stage + (u64)g * TPCC_K;
    bool all = true;
    for (uint32_t i = 0; i < n; i++) all &= st[i].v[5] != 0;
    if (all) {
        part_assemble_one(y, pd, g, st, committed, ohi, olo, read_out, (1ull << 63) | round);
        skip[g] = 2;   // done
    } else {
        restarts[g] += 1;   // aborted this round, retried in the next
    }
}

// decision of every access sent this round (aligned with the send buffer)
__global__ void part_dec_kernel(const PartReq *sent, uint64_t n, PartDev pd, const uint8_t *skip,
                                unsigned long long *dec) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    dec[k] = skip[sent[k].gid - pd.rank * pd.n_local] == 2 ? 1ull : 0ull;
}

// next round: requests of the still-pending distributed transactions; cnt[world] counts them
__global__ void part_recount_kernel(TpccParams y, PartDev pd, uint32_t n_txn, const uint8_t *skip,
                                    unsigned long long *cnt) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_txn || skip[g] != 1) return;
    const uint32_t *t = y.tx + (u64)g * TPCC_TX_WORDS;
    const uint32_t n = t[TX_TYPE] == 0 ? 3 + t[TX_OLCNT] : 3;
    for (uint32_t i = 0; i < n; i++) {
        uint32_t dest = pd.rank;
        if (i == 2 && t[TX_TYPE] == 1) dest = owner_of(pd, t[TX_CW]);
        if (i >= 3) dest = owner_of(pd, t[TX_SUPQ + i - 3] >> 8);
        atomicAdd(&cnt[dest], 1ull);
    }
    atomicAdd(&cnt[pd.world], 1ull);
}

// ---------------------------------------------------------------- launchers
cudaError_t part_classify_pack(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr, uint32_t n_txn,
                               uint8_t *skip, unsigned long long *cnt, unsigned long long *off,
                               unsigned long long *cursor, PartReq *out, cudaStream_t s) {
    const PartDev pd{rank, world, wpr, n_txn};
    cudaMemsetAsync(cnt, 0, world * 8ull, s);
    part_classify_kernel<<<(n_txn + 255) / 256, 256, 0, s>>>(y, pd, n_txn, skip, cnt, false);
    part_scan_kernel<<<1, 1, 0, s>>>(cnt, off, cursor, world);
    part_pack_kernel<<<(n_txn + 255) / 256, 256, 0, s>>>(y, pd, n_txn, skip, cursor, out);
    return cudaGetLastError();
}

// CC_FLAG_PART_ALL: every transaction takes the phase-B path (tests phase B on 1 GPU)
cudaError_t launch_part_all(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr, uint32_t n_txn,
                            uint8_t *skip, unsigned long long *cnt, unsigned long long *off,
                            unsigned long long *cursor, PartReq *out, cudaStream_t s) {
    const PartDev pd{rank, world, wpr, n_txn};
    cudaMemsetAsync(cnt, 0, world * 8ull, s);
    part_classify_kernel<<<(n_txn + 255) / 256, 256, 0, s>>>(y, pd, n_txn, skip, cnt, true);
    part_scan_kernel<<<1, 1, 0, s>>>(cnt, off, cursor, world);
    part_pack_kernel<<<(n_txn + 255) / 256, 256, 0, s>>>(y, pd, n_txn, skip, cursor, out);
    return cudaGetLastError();
}

cudaError_t part_apply(PartReq *req, uint64_t n, const TpccParams &y, PartResp *resp, unsigned long long *k1,
                       unsigned long long *k2, uint32_t *i1, uint32_t *i2, void *tmp, size_t tmp_bytes, Ctl *ctl,
                       cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    part_keys_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(req, n, y, k1, i1, ctl);
    u64 *sk = nullptr;
    uint32_t *si = nullptr;
    cudaError_t e = gc_sort(k1, i1, k2, i2, n, nullptr, 0, 62, tmp, tmp_bytes, s, &sk, &si);
    if (e) return e;
    part_chain_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sk, si, n, req, y, resp);
    return cudaGetLastError();
}

size_t part_sort_bytes(uint64_t n) { return gc_sort_temp_bytes(n) + 256; }

cudaError_t part_finish(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr, uint32_t n_txn,
                        const uint8_t *skip, const PartReq *sent, const PartResp *resp, uint64_t n_sent,
                        PartResp *stage, uint8_t *committed, unsigned long long *ohi, unsigned long long *olo,
                        unsigned long long *read_out, cudaStream_t s, bool two_pc) {
    const PartDev pd{rank, world, wpr, n_txn};
    if (n_sent && !two_pc)
        part_stage_kernel<<<(unsigned)((n_sent + 255) / 256), 256, 0, s>>>(sent, resp, n_sent, pd, stage);
    part_assemble_kernel<<<(n_txn + 127) / 128, 128, 0, s>>>(y, pd, n_txn, skip, stage, committed, ohi, olo,
                                                             read_out, two_pc);
    return cudaGetLastError();
}

// 2PC PREPARE on the owner: resolve + sort like part_apply, then grant per item chain
cudaError_t part_grant(PartReq *req, uint64_t n, const TpccParams &y, PartResp *resp, uint8_t *vote,
                       unsigned long long *k1, unsigned long long *k2, uint32_t *i1, uint32_t *i2, void *tmp,
                       size_t tmp_bytes, Ctl *ctl, cudaStream_t s, bool ts_rule) {
    if (n == 0) return cudaSuccess;
    part_keys_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(req, n, y, k1, i1, ctl);
    u64 *sk = nullptr;
    uint32_t *si = nullptr;
    cudaError_t e = gc_sort(k1, i1, k2, i2, n, nullptr, 0, 62, tmp, tmp_bytes, s, &sk, &si);
    if (e) return e;
    part_grant_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sk, si, n, req, y, resp, vote, ts_rule);
    return cudaGetLastError();
}

// 2PC DECIDE on the home: stage the returned votes / values, decide, emit decisions
cudaError_t part_decide(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr, uint32_t n_txn,
                        uint8_t *skip, const PartReq *sent, const PartResp *resp, uint64_t n_sent, PartResp *stage,
                        uint8_t *committed, unsigned long long *ohi, unsigned long long *olo,
                        unsigned long long *read_out, uint32_t *restarts, uint32_t round, unsigned long long *dec,
                        cudaStream_t s) {
    const PartDev pd{rank, world, wpr, n_txn};
    if (n_sent)
        part_stage_kernel<<<(unsigned)((n_sent + 255) / 256), 256, 0, s>>>(sent, resp, n_sent, pd, stage);
    part_decide_kernel<<<(n_txn + 127) / 128, 128, 0, s>>>(y, pd, n_txn, skip, stage, committed, ohi, olo,
                                                           read_out, restarts, round);
    if (n_sent) part_dec_kernel<<<(unsigned)((n_sent + 255) / 256), 256, 0, s>>>(sent, n_sent, pd, skip, dec);
    return cudaGetLastError();
}

// 2PC COMMIT on the owner
cudaError_t part_commit(const PartReq *req, uint64_t n, const uint8_t *vote, const unsigned long long *dec,
                        const TpccParams &y, cudaStream_t s) {
    if (n) part_commit_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(req, n, vote, dec, y);
    return cudaGetLastError();
}

// next 2PC round: pack the pending transactions' requests; cnt[world] = pending count
cudaError_t part_repack(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr, uint32_t n_txn,
                        const uint8_t *skip, unsigned long long *cnt, unsigned long long *off,
                        unsigned long long *cursor, PartReq *out, cudaStream_t s) {
    const PartDev pd{rank, world, wpr, n_txn};
    cudaMemsetAsync(cnt, 0, (world + 1) * 8ull, s);
    part_recount_kernel<<<(n_txn + 255) / 256, 256, 0, s>>>(y, pd, n_txn, skip, cnt);
    part_scan_kernel<<<1, 1, 0, s>>>(cnt, off, cursor, world);
    part_pack_kernel<<<(n_txn + 255) / 256, 256, 0, s>>>(y, pd, n_txn, skip, cursor, out);
    return cudaGetLastError();
}

// ================================================================ exchange over peer memory
// The deterministic phase B without the host in the loop (CC_FLAG_PART_P2P).  Every rank
// owns an exchange window in its device memory -- flags, an inbox of `cap` request slots
// per source rank, and the staging array of its own transactions' responses -- and maps
// the windows of its peers (CUDA IPC across processes / GPUs over NVLink; plain pointers
// between dbs of one process).  One partitioned cc_submit then runs, on the db stream:
//   pack    the sender writes each request straight into the owner's inbox (a remote store
//           over NVLink, a local one for itself) -- the pack and the transfer are one kernel;
//   signal  one release store per owner (system scope): epoch << 32 | number of requests;
//   [phase A executes meanwhile on this rank]
//   wait    until every source's flag carries this epoch, then compact the inboxes;
//   chain   sort by (item, global gid), apply each item's chain in gid order and store every
//           response straight into the home's staging array (compute + transfer fused);
//   signal  one release store per home: epoch;
//   wait    for every owner, then assemble the distributed transactions and emit (a7).
// The same kernels as the host-driven exchange decide what is applied and returned, so the
// results are identical; only the transport differs.  A round's inbox is compacted before
// its owner signals, and a sender packs its next round only after every owner's signal, so
// windows are reused without further synchronisation.
static __device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
static __device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
static __device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__global__ void p2p_pack_kernel(TpccParams y, PartDev pd, uint32_t n_txn, const uint8_t *skip,
                                unsigned long long *cursor, PeerTab pt, uint32_t cap, Ctl *ctl) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_txn || skip[g] != 1) return;
    const uint32_t *t = y.tx + (u64)g * TPCC_TX_WORDS;
    const uint32_t type = t[TX_TYPE], w = t[TX_W], d = t[TX_D];
    const uint32_t n = type == 0 ? 3 + t[TX_OLCNT] : 3;
    for (uint32_t i = 0; i < n; i++) {
        PartReq r{};
        r.gid = pd.rank * pd.n_local + g;
        r.home = pd.rank | (i << 16);
        r.type_d = type | (d << 8);
        r.home_w = w | (d << 16);
        r.last = 0xFFFFFFFFu;
        uint32_t dest = pd.rank;
        const uint32_t lw = w - pd.rank * pd.wpr;
        if (i == 0) {
            r.kind = 0;
            r.row = lw;
            r.amount = type == 1 ? t[TX_HAMT] : 0;
        } else if (i == 1) {
            r.kind = 1;
            r.row = lw * TPCC_DIST + d;
            r.amount = type == 1 ? t[TX_HAMT] : 0;
        } else if (i == 2) {
            r.kind = 2;
            const uint32_t cw = type == 0 ? w : t[TX_CW], cd = type == 0 ? d : t[TX_CD];
            dest = owner_of(pd, cw);
            const uint32_t lcw = cw - dest * pd.wpr;
            r.cust = lcw * TPCC_DIST + cd;
            r.c_ids = cw | (cd << 16);
            r.amount = type == 1 ? t[TX_HAMT] : 0;
            if (t[TX_C] == 0xFFFFFFFFu) {
                r.row = 0xFFFFFFFFu;
                r.last = t[TX_CLAST];
            } else {
                r.row = r.cust * TPCC_CUST + t[TX_C];
            }
        } else {
            r.kind = 3;
            const uint32_t sw = t[TX_SUPQ + i - 3] >> 8;
            dest = owner_of(pd, sw);
            r.row = (sw - dest * pd.wpr) * TPCC_STOCK + t[TX_ITEM + i - 3];
            r.amount = t[TX_SUPQ + i - 3] & 0xFF;
            r.type_d |= (sw != w ? 1u : 0u) << 16;
        }
        const unsigned long long pos = atomicAdd(&cursor[dest], 1ull);
        if (pos < cap) pt.inbox[dest][(u64)pd.rank * cap + pos] = r;   // into the owner's window
        else atomicCAS(&ctl->err.v, 0ull, (u64)CC_ERR_CONFIG);      // exchange capacity exceeded
    }
}

// flags: req[s] at flags[s * P2P_FLAG_STRIDE], resp[d] at flags[(P2P_MAXW + d) * P2P_FLAG_STRIDE]
__global__ void p2p_signal_req_kernel(PeerTab pt, PartDev pd, const unsigned long long *cursor, uint32_t cap,
                                      unsigned long long epoch) {
    const uint32_t d = threadIdx.x;
    if (d >= pd.world) return;
    const unsigned long long c = cursor[d] < cap ? cursor[d] : cap;
    fence_sys();   // the pack kernel's stores (ordered before this kernel) precede the flag
    st_release_sys(pt.flags[d] + (u64)pd.rank * P2P_FLAG_STRIDE, (epoch << 32) | c);
}

// wait for every source's requests of this epoch; rc[s] = count, rc[world + s] = offset,
// rc[2 * world] = total
__global__ void p2p_wait_req_kernel(const unsigned long long *flags, PartDev pd, unsigned long long epoch,
                                    unsigned long long *rc, Ctl *ctl, u64 watchdog_ns) {
    const uint32_t s = threadIdx.x;
    const u64 deadline = globaltimer_ns() + watchdog_ns;
    if (s < pd.world) {
        unsigned long long v;
        unsigned ns = 32;
        while (((v = ld_acquire_sys(flags + (u64)s * P2P_FLAG_STRIDE)) >> 32) != epoch) {
            if (globaltimer_ns() > deadline) {
                atomicCAS(&ctl->err.v, 0ull, (u64)CC_ERR_WATCHDOG);
                v = epoch << 32;   // count 0: nothing from this source
                break;
            }
            __nanosleep(ns);
            ns = ns < 1024 ? ns * 2 : 1024;
        }
        rc[s] = v & 0xFFFFFFFFull;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long o = 0;
        for (uint32_t k = 0; k < pd.world; k++) {
            rc[pd.world + k] = o;
            o += rc[k];
        }
        rc[2 * pd.world] = o;
    }
}

__global__ void p2p_compact_kernel(const PartReq *inbox, const unsigned long long *rc, uint32_t world, uint32_t cap,
                                   PartReq *recv) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (uint64_t)world * cap) return;
    const uint32_t s = (uint32_t)(k / cap), j = (uint32_t)(k % cap);
    if (j < rc[s]) recv[rc[world + s] + j] = inbox[k];
}

// one thread per item chain, in gid order; each response goes straight to its home's
// staging array (remote store): slot (local gid, access lane)
__global__ void p2p_chain_kernel(const unsigned long long *skeys, const uint32_t *sidx, const unsigned long long *n_dev,
                                 const PartReq *req, TpccParams y, PeerTab pt, uint32_t n_local) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t n = *n_dev;
    if (p >= n) return;
    if (p > 0 && (skeys[p - 1] >> 24) == (skeys[p] >> 24)) return;   // chain head only
    for (uint64_t q = p; q < n && (skeys[q] >> 24) == (skeys[p] >> 24); q++) {
        const PartReq &r = req[sidx[q]];
        const uint32_t home = r.home & 0xFFFFu, lane = r.home >> 16;
        pt.stage[home][(u64)(r.gid - home * n_local) * TPCC_K + lane] = part_access(r, y, true);
    }
}

__global__ void p2p_signal_resp_kernel(PeerTab pt, PartDev pd, unsigned long long epoch) {
    const uint32_t h = threadIdx.x;
    if (h >= pd.world) return;
    fence_sys();   // the chain kernel's remote stores precede the flag
    st_release_sys(pt.flags[h] + (u64)(P2P_MAXW + pd.rank) * P2P_FLAG_STRIDE, epoch << 32);
}

__global__ void p2p_wait_resp_kernel(const unsigned long long *flags, PartDev pd, unsigned long long epoch, Ctl *ctl,
                                     u64 watchdog_ns) {
    const uint32_t d = threadIdx.x;
    if (d >= pd.world) return;
    const u64 deadline = globaltimer_ns() + watchdog_ns;
    unsigned ns = 32;
    while ((ld_acquire_sys(flags + (u64)(P2P_MAXW + d) * P2P_FLAG_STRIDE) >> 32) != epoch) {
        if (globaltimer_ns() > deadline) {
            atomicCAS(&ctl->err.v, 0ull, (u64)CC_ERR_WATCHDOG);
            return;
        }
        __nanosleep(ns);
        ns = ns < 1024 ? ns * 2 : 1024;
    }
}

size_t p2p_window_bytes(uint32_t world, uint32_t cap, uint32_t max_txn) {
    return P2P_FLAG_BYTES + (size_t)world * cap * sizeof(PartReq) + (size_t)max_txn * TPCC_K * sizeof(PartResp);
}

// send side: classify, pack into the owners' windows, signal (before phase A)
cudaError_t p2p_send(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr, uint32_t n_txn, uint8_t *skip,
                     unsigned long long *cnt, unsigned long long *cursor, const PeerTab &pt, uint32_t cap,
                     unsigned long long epoch, Ctl *ctl, bool all, cudaStream_t s) {
    const PartDev pd{rank, world, wpr, n_txn};
    cudaMemsetAsync(cnt, 0, world * 8ull, s);
    cudaMemsetAsync(cursor, 0, world * 8ull, s);
    part_classify_kernel<<<(n_txn + 255) / 256, 256, 0, s>>>(y, pd, n_txn, skip, cnt, all);
    p2p_pack_kernel<<<(n_txn + 255) / 256, 256, 0, s>>>(y, pd, n_txn, skip, cursor, pt, cap, ctl);
    p2p_signal_req_kernel<<<1, P2P_MAXW, 0, s>>>(pt, pd, cursor, cap, epoch);
    return cudaGetLastError();
}

// owner side (after phase A) and home side: phase B through the windows, then assemble
cudaError_t p2p_phase_b(const TpccParams &y, uint32_t rank, uint32_t world, uint32_t wpr, uint32_t n_txn,
                        const uint8_t *skip, const PeerTab &pt, uint32_t cap, unsigned long long epoch,
                        unsigned long long *rc, PartReq *recv, unsigned long long *k1, unsigned long long *k2,
                        uint32_t *i1, uint32_t *i2, void *tmp, size_t tmp_bytes, uint8_t *committed,
                        unsigned long long *ohi, unsigned long long *olo, unsigned long long *read_out, Ctl *ctl,
                        u64 watchdog_ns, cudaStream_t s) {
    const PartDev pd{rank, world, wpr, n_txn};
    const unsigned long long *myflags = pt.flags[rank];
    p2p_wait_req_kernel<<<1, P2P_MAXW, 0, s>>>(myflags, pd, epoch, rc, ctl, watchdog_ns);
    const uint64_t capn = (uint64_t)world * cap;
    const unsigned gb = (unsigned)((capn + 255) / 256);
    p2p_compact_kernel<<<gb, 256, 0, s>>>(pt.inbox[rank], rc, world, cap, recv);
    const unsigned long long *n_dev = rc + 2 * world;
    part_keys_kernel<<<gb, 256, 0, s>>>(recv, capn, y, k1, i1, ctl, n_dev);
    u64 *sk = nullptr;
    uint32_t *si = nullptr;
    cudaError_t e = gc_sort(k1, i1, k2, i2, capn, n_dev, 0, 62, tmp, tmp_bytes, s, &sk, &si);
    if (e) return e;
    p2p_chain_kernel<<<gb, 256, 0, s>>>(sk, si, n_dev, recv, y, pt, n_txn);
    p2p_signal_resp_kernel<<<1, P2P_MAXW, 0, s>>>(pt, pd, epoch);
    p2p_wait_resp_kernel<<<1, P2P_MAXW, 0, s>>>(myflags, pd, epoch, ctl, watchdog_ns);
    part_assemble_kernel<<<(n_txn + 127) / 128, 128, 0, s>>>(y, pd, n_txn, skip, pt.stage[rank], committed, ohi, olo,
                                                             read_out, false);
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
void preload_part_kernels() {
    preload1(part_classify_kernel); preload1(part_scan_kernel); preload1(part_pack_kernel); preload1(part_keys_kernel);
    preload1(part_chain_kernel); preload1(part_grant_kernel); preload1(part_commit_kernel); preload1(part_stage_kernel);
    preload1(part_assemble_kernel); preload1(part_decide_kernel); preload1(part_dec_kernel); preload1(part_recount_kernel);
    preload1(p2p_pack_kernel); preload1(p2p_signal_req_kernel); preload1(p2p_wait_req_kernel); preload1(p2p_compact_kernel);
    preload1(p2p_chain_kernel); preload1(p2p_signal_resp_kernel); preload1(p2p_wait_resp_kernel);
}
}  // namespace gcctb
