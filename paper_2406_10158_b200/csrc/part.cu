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
#include <cub/cub.cuh>

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
                                 uint32_t *idx, Ctl *ctl) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
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
    size_t bytes = tmp_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, bytes, k1, k2, i1, i2, (int)n, 0, 62, s);
    if (e) return e;
    part_chain_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(k2, i2, n, req, y, resp);
    return cudaGetLastError();
}

size_t part_sort_bytes(uint64_t n) {
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, (const unsigned long long *)nullptr, (unsigned long long *)nullptr,
                                    (const uint32_t *)nullptr, (uint32_t *)nullptr, (int)n, 0, 62);
    return b + 256;
}

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
    size_t bytes = tmp_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, bytes, k1, k2, i1, i2, (int)n, 0, 62, s);
    if (e) return e;
    part_grant_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(k2, i2, n, req, y, resp, vote, ts_rule);
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

}  // namespace gcctb
