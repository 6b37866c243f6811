// tpcc.cu -- TPC-C NewOrder/Payment on the device: the initial
// population (device copy of the seeded input generator, inputs/tpcc.py), the
// immutable customer last-name index, the a1 batch generator, the workload policy the
// executor is instantiated with, and the a3 access gather for GPUTx/GaccO.
//
// Semantics: money i64 cents, rates 1/10,000; inserts
// are writes to per-transaction reserved slots (Z15); Item and the name index are
// immutable and outside CC (Z16); NewOrder's rollback omitted (Z17); totals rounded
// half up (Z18); NewOrder increments d_next_o_id (Z14).

#include "exec.cuh"
#include "tpcc.h"

namespace gcctb {

// ---------------------------------------------------------------- population
__device__ __forceinline__ u64 prand(u64 seed, u64 table, u64 row, u64 field) {
    return mix64(seed ^ (table << 56) ^ (row << 8) ^ field);
}
// 8 letters 'A' + (byte % 26) from one prand word, only the first `keep` bytes
__device__ __forceinline__ u64 letters_word(u64 seed, u64 table, u64 row, u64 field, int keep) {
    const u64 r = prand(seed, table, row, field);
    u64 out = 0;
#pragma unroll
    for (int b = 0; b < 8; b++)
        if (b < keep) out |= (u64)('A' + (uint32_t)((r >> (8 * b)) & 0xFF) % 26u) << (8 * b);
    return out;
}
__device__ __forceinline__ void put_letters(u64 *w, u64 seed, u64 table, u64 row, u64 field0, int n) {
    for (int k = 0; k < (n + 7) / 8; k++) {
        const int keep = n - 8 * k < 8 ? n - 8 * k : 8;
        w[k] = letters_word(seed, table, row, field0 + k, keep);
    }
}
// 10% of rows: "ORIGINAL" at byte offset (r >> 8) % 43 of the 50-letter string at w
__device__ __forceinline__ void put_original(u64 *w, u64 seed, u64 table, u64 row) {
    const u64 r = prand(seed, table, row, 2);
    if (r % 10 != 0) return;
    const int off = (int)((r >> 8) % 43);
    const char *o = "ORIGINAL";
    uint8_t *b = reinterpret_cast<uint8_t *>(w);
    for (int k = 0; k < 8; k++) b[off + k] = (uint8_t)o[k];
}

__constant__ char c_syl[10][6] = {"BAR", "OUGHT", "ABLE", "PRI", "PRES", "ESE", "ANTI", "CALLY", "ATION", "EING"};
__constant__ uint8_t c_syl_len[10] = {3, 5, 4, 3, 4, 3, 4, 5, 5, 4};

__device__ __forceinline__ void last_name(uint32_t num, u64 out[2]) {
    uint8_t b[16];
    for (int k = 0; k < 16; k++) b[k] = 0;
    int p = 0;
    const uint32_t dig[3] = {num / 100, (num / 10) % 10, num % 10};
    for (int k = 0; k < 3; k++)
        for (int c = 0; c < c_syl_len[dig[k]]; c++) b[p++] = (uint8_t)c_syl[dig[k]][c];
    out[0] = out[1] = 0;
    for (int k = 0; k < 16; k++) out[k / 8] |= (u64)b[k] << (8 * (k % 8));
}

__device__ __forceinline__ uint32_t cust_last_num(u64 seed, uint32_t c_load, u64 row) {
    const uint32_t c = (uint32_t)(row % TPCC_CUST);
    if (c < 1000) return c;
    const u64 a = prand(seed, TPCC_T_C, row, 5) % 256, b = prand(seed, TPCC_T_C, row, 6) % 1000;
    return (uint32_t)(((a | b) + c_load) % 1000);
}

// one thread per row of each table; global row ids g = first + local index
__global__ void tpcc_pop_kernel(int table, u64 *rows, u64 first, u64 n, u64 seed, uint32_t c_load) {
    const u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const u64 g = first + k;
    if (table == TPCC_T_W) {
        u64 *w = rows + k * TPCC_W_WORDS;
        w[0] = 30000000ull;
        w[1] = prand(seed, TPCC_T_W, g, 1) % 2001;
        put_letters(w + 2, seed, TPCC_T_W, g, 16, 10);
        for (int j = 0; j < 12; j++) w[4 + j] = prand(seed, TPCC_T_W, g, 32 + j);
    } else if (table == TPCC_T_D) {
        u64 *w = rows + k * TPCC_D_WORDS;
        w[0] = 3000000ull;
        w[1] = (prand(seed, TPCC_T_D, g, 1) % 2001) | (3001ull << 32);
        put_letters(w + 2, seed, TPCC_T_D, g, 16, 10);
        for (int j = 0; j < 12; j++) w[4 + j] = prand(seed, TPCC_T_D, g, 32 + j);
    } else if (table == TPCC_T_C) {
        u64 *w = rows + k * TPCC_C_WORDS;
        w[0] = (u64)(-1000ll);
        w[1] = 1000;
        w[2] = 1;
        const u64 credit = (prand(seed, TPCC_T_C, g, 2) % 10 == 0) ? 0x4342ull : 0x4347ull;
        w[3] = (prand(seed, TPCC_T_C, g, 3) % 5001) | (credit << 32);
        last_name(cust_last_num(seed, c_load, g), w + 4);
        const int flen = 8 + (int)(prand(seed, TPCC_T_C, g, 4) % 9);
        put_letters(w + 6, seed, TPCC_T_C, g, 16, flen);   // c_first: 8..16 letters
        if (flen <= 8) w[7] = 0;
        for (int j = 0; j < 17; j++) w[8 + j] = prand(seed, TPCC_T_C, g, 64 + j);
        put_letters(w + TPCC_CDATA_OFF, seed, TPCC_T_C, g, 128, 500);
    } else if (table == TPCC_T_S) {
        u64 *w = rows + k * TPCC_S_WORDS;
        w[0] = 10 + prand(seed, TPCC_T_S, g, 1) % 91;
        w[1] = 0;
        w[2] = 0;
        put_letters(w + 3, seed, TPCC_T_S, g, 16, 240);
        put_letters(w + 33, seed, TPCC_T_S, g, 64, 50);
        put_original(w + 33, seed, TPCC_T_S, g);
    } else {   // items
        u64 *w = rows + k * TPCC_I_WORDS;
        const u64 price = 100 + prand(seed, TPCC_T_I, g, 1) % 9901;
        const u64 im = 1 + prand(seed, TPCC_T_I, g, 3) % 10000;
        w[0] = price | (im << 32);
        put_letters(w + 1, seed, TPCC_T_I, g, 16, 24);
        put_letters(w + 4, seed, TPCC_T_I, g, 64, 50);
        put_original(w + 4, seed, TPCC_T_I, g);
        w[11] = prand(seed, TPCC_T_I, g, 200);
    }
}

cudaError_t launch_tpcc_pop(int table, u64 *rows, u64 first, u64 n, u64 seed, uint32_t c_load,
                            cudaStream_t s) {
    tpcc_pop_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(table, rows, first, n, seed, c_load);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- name index
// Immutable (Z16): per (w, d, last) group the customers sorted by (c_first, c_id)
// (TPC-C §2.5.2.2; ties by c_id, reading R5).  Built once at load.
__global__ void name_key_kernel(const u64 *cu, uint32_t n, u64 *key, uint32_t *val, u64 seed,
                                uint32_t c_load, u64 first_row) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const u64 g = first_row + k;
    const uint32_t wd = (uint32_t)(k / TPCC_CUST);     // local (w*10+d)
    key[k] = wd * 1000u + cust_last_num(seed, c_load, g);
    val[k] = k;                                         // local customer row
}

__device__ __forceinline__ u64 bswap64(u64 x) {
    const uint32_t lo = __byte_perm((uint32_t)x, 0, 0x0123), hi = __byte_perm((uint32_t)(x >> 32), 0, 0x0123);
    return ((u64)lo << 32) | hi;
}

__global__ void name_group_kernel(const u64 *skey, uint32_t *vals, uint32_t n, uint32_t *start,
                                  uint32_t *count, const u64 *cu) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    if (p != 0 && skey[p - 1] == skey[p]) return;   // one thread per group head
    uint32_t e = p + 1;
    while (e < n && skey[e] == skey[p]) e++;
    start[skey[p]] = p;
    count[skey[p]] = e - p;
    // insertion sort of the group by (c_first big-endian bytes, row)
    for (uint32_t a = p + 1; a < e; a++) {
        const uint32_t v = vals[a];
        const u64 f0 = bswap64(cu[(u64)v * TPCC_C_WORDS + 6]), f1 = bswap64(cu[(u64)v * TPCC_C_WORDS + 7]);
        int b = (int)a - 1;
        while (b >= (int)p) {
            const uint32_t u = vals[b];
            const u64 g0 = bswap64(cu[(u64)u * TPCC_C_WORDS + 6]), g1 = bswap64(cu[(u64)u * TPCC_C_WORDS + 7]);
            const bool gt = g0 > f0 || (g0 == f0 && (g1 > f1 || (g1 == f1 && u > v)));
            if (!gt) break;
            vals[b + 1] = u;
            b--;
        }
        vals[b + 1] = v;
    }
}

cudaError_t build_name_index(const u64 *cu, uint32_t n_cust, u64 first_row, u64 seed, uint32_t c_load,
                             uint32_t *idx_start, uint32_t *idx_count, uint32_t *idx_rows,
                             uint32_t n_groups, cudaStream_t s) {
    u64 *k1 = nullptr, *k2 = nullptr, *sk = nullptr;
    uint32_t *v1 = nullptr, *v2 = nullptr, *sv = nullptr;
    void *tmp = nullptr;
    const size_t bytes = gc_sort_temp_bytes(n_cust);
    cudaError_t e;
    if ((e = cudaMalloc(&k1, n_cust * 8ull)) || (e = cudaMalloc(&k2, n_cust * 8ull)) ||
        (e = cudaMalloc(&v1, n_cust * 4ull)) || (e = cudaMalloc(&v2, n_cust * 4ull)) || (e = cudaMalloc(&tmp, bytes)))
        return e;
    cudaMemsetAsync(idx_count, 0, n_groups * 4ull, s);
    name_key_kernel<<<(n_cust + 255) / 256, 256, 0, s>>>(cu, n_cust, k1, v1, seed, c_load, first_row);
    int hb = 1;   // group keys < n_groups
    while (hb < 32 && (1ull << hb) < n_groups) hb++;
    e = gc_sort(k1, v1, k2, v2, n_cust, nullptr, 0, hb, tmp, bytes, s, &sk, &sv);
    if (!e) e = cudaMemcpyAsync(idx_rows, sv, n_cust * 4ull, cudaMemcpyDeviceToDevice, s);
    if (!e) name_group_kernel<<<(n_cust + 255) / 256, 256, 0, s>>>(sk, idx_rows, n_cust, idx_start, idx_count, cu);
    if (!e) e = cudaStreamSynchronize(s);
    cudaFree(k1); cudaFree(k2); cudaFree(v1); cudaFree(v2); cudaFree(tmp);
    return e ? e : cudaGetLastError();
}

// ---------------------------------------------------------------- a1 generator
// One thread per transaction, the same draws as orc_tpcc_gen (TPC-C §2.4.1, §2.5.1,
// NURand §2.1.6): rng(seed, gid, stream << 56 | j << 24 | k).
enum { S_TYPE = 1, S_W, S_D, S_CA, S_CB, S_OLCNT, S_ITEMA, S_ITEMB, S_SUP, S_SUPW, S_QTY,
       S_BYNAME, S_REMOTE, S_CW, S_CD, S_LASTA, S_LASTB, S_HAMT };

__device__ __forceinline__ u64 draw(u64 seed, uint32_t g, u64 stream, u64 j, u64 k) {
    return rng3(seed, g, (stream << 56) | (j << 24) | k);
}
__device__ __forceinline__ u64 urand(u64 u, u64 lo, u64 hi) { return lo + u % (hi - lo + 1); }
__device__ __forceinline__ u64 nurand(u64 ua, u64 ub, u64 A, u64 x, u64 y, u64 C) {
    return (((urand(ua, 0, A) | urand(ub, x, y)) + C) % (y - x + 1)) + x;
}

__global__ void tpcc_gen_kernel(uint32_t *txo, uint32_t n_txn, u64 seed, uint32_t W, uint32_t w_lo,
                                uint32_t w_hi, uint32_t no_pm, uint32_t c_last_run, uint32_t c_id_c,
                                uint32_t c_item_c, u64 *err) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_txn) return;
    uint32_t t[TPCC_TX_WORDS];
    for (int k = 0; k < TPCC_TX_WORDS; k++) t[k] = 0;
    const uint32_t w = w_lo + (uint32_t)(draw(seed, g, S_W, 0, 0) % (w_hi - w_lo));
    const uint32_t d = (uint32_t)(draw(seed, g, S_D, 0, 0) % TPCC_DIST);
    t[TX_W] = w;
    t[TX_D] = d;
    if (draw(seed, g, S_TYPE, 0, 0) % 10000 < no_pm) {
        t[TX_TYPE] = 0;
        t[TX_CW] = w;
        t[TX_CD] = d;
        t[TX_C] = (uint32_t)nurand(draw(seed, g, S_CA, 0, 0), draw(seed, g, S_CB, 0, 0), 1023, 1, TPCC_CUST, c_id_c) - 1;
        t[TX_CLAST] = 0xFFFFFFFFu;
        const uint32_t n = (uint32_t)urand(draw(seed, g, S_OLCNT, 0, 0), 5, 15);
        t[TX_OLCNT] = n;
        uint32_t items[TPCC_MAXOL], sq[TPCC_MAXOL];
        uint32_t all_local = 1;
        for (uint32_t j = 0; j < n; j++) {
            for (u64 k = 0;; k++) {
                if (k > 4096) {
                    atomicCAS(err, 0ull, (u64)CC_ERR_CONFIG);   // the batch's error word
                    return;
                }
                const uint32_t i = (uint32_t)nurand(draw(seed, g, S_ITEMA, j, k), draw(seed, g, S_ITEMB, j, k), 8191, 1,
                                                    TPCC_ITEMS, c_item_c) - 1;
                bool dup = false;
                for (uint32_t q = 0; q < j; q++) dup |= items[q] == i;
                if (!dup) { items[j] = i; break; }
            }
            uint32_t sw = w;
            if (W > 1 && draw(seed, g, S_SUP, j, 0) % 100 == 0) {
                const uint32_t o = (uint32_t)(draw(seed, g, S_SUPW, j, 0) % (W - 1));
                sw = o >= w ? o + 1 : o;
            }
            if (sw != w) all_local = 0;
            sq[j] = (sw << 8) | (uint32_t)urand(draw(seed, g, S_QTY, j, 0), 1, 10);
        }
        for (uint32_t a = 1; a < n; a++) {
            const uint32_t ki = items[a], ks = sq[a];
            int b = (int)a - 1;
            while (b >= 0 && ((sq[b] >> 8) > (ks >> 8) || ((sq[b] >> 8) == (ks >> 8) && items[b] > ki))) {
                items[b + 1] = items[b];
                sq[b + 1] = sq[b];
                b--;
            }
            items[b + 1] = ki;
            sq[b + 1] = ks;
        }
        for (uint32_t j = 0; j < n; j++) {
            t[TX_ITEM + j] = items[j];
            t[TX_SUPQ + j] = sq[j];
        }
        t[TX_ALLLOCAL] = all_local;
    } else {
        t[TX_TYPE] = 1;
        uint32_t cw = w, cd = d;
        if (W > 1 && draw(seed, g, S_REMOTE, 0, 0) % 100 < 15) {
            const uint32_t o = (uint32_t)(draw(seed, g, S_CW, 0, 0) % (W - 1));
            cw = o >= w ? o + 1 : o;
            cd = (uint32_t)(draw(seed, g, S_CD, 0, 0) % TPCC_DIST);
        }
        t[TX_CW] = cw;
        t[TX_CD] = cd;
        if (draw(seed, g, S_BYNAME, 0, 0) % 100 < 60) {
            t[TX_C] = 0xFFFFFFFFu;
            t[TX_CLAST] = (uint32_t)nurand(draw(seed, g, S_LASTA, 0, 0), draw(seed, g, S_LASTB, 0, 0), 255, 0, 999, c_last_run);
        } else {
            t[TX_C] = (uint32_t)nurand(draw(seed, g, S_CA, 0, 0), draw(seed, g, S_CB, 0, 0), 1023, 1, TPCC_CUST, c_id_c) - 1;
            t[TX_CLAST] = 0xFFFFFFFFu;
        }
        t[TX_HAMT] = (uint32_t)urand(draw(seed, g, S_HAMT, 0, 0), 100, 500000);
    }
    uint32_t *o = txo + (u64)g * TPCC_TX_WORDS;
    for (int k = 0; k < TPCC_TX_WORDS; k++) o[k] = t[k];
}

cudaError_t launch_tpcc_gen(uint32_t *tx, uint32_t n_txn, u64 seed, uint32_t W, uint32_t w_lo, uint32_t w_hi,
                            uint32_t no_pm, uint32_t c_last_run, uint32_t c_id_c, uint32_t c_item_c, u64 *err,
                            cudaStream_t s) {
    tpcc_gen_kernel<<<(n_txn + 127) / 128, 128, 0, s>>>(tx, n_txn, seed, W, w_lo, w_hi, no_pm, c_last_run, c_id_c,
                                                        c_item_c, err);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- workload policy
struct TpccWL {
    static constexpr int MAXK = TPCC_K;          // W, D, C + up to 15 stock lines
    static constexpr int ROW_WORDS = TPCC_C_WORDS;   // largest CC row (MVCC node payload)
    static constexpr bool STAGE_TILE_LANE = true;    // tile mode: the ~110 B entry lives in shared memory
    using Params = TpccParams;
    enum { KW = 0, KD = 1, KC = 2, KS = 3 };
    struct Lane {
        u32 rec;
        bool act, w;
        uint8_t kind, type;   // kind: W/D/C/S; type: 0 NewOrder, 1 Payment
        u32 line;             // stock line index
        u32 qty, sw, item, price, brand_i;
        u64 v0, v1, v2, v3;   // values read / buffered new values (per kind)
        u64 s0, s1, s2, s3;   // string payload (w_name / d_name / s_dist) or the BC record
        u64 cv;               // thread mode: control word seen (OCC snapshot / lock-time word, TO / MVCC saved word)
    };

    static GC_DEV u64 *row(const TpccParams &y, const Lane &L) {
        switch (L.kind) {
            case KW: return y.wh + (u64)(L.rec - y.bW) * TPCC_W_WORDS;
            case KD: return y.di + (u64)(L.rec - y.bD) * TPCC_D_WORDS;
            case KC: return y.cu + (u64)(L.rec - y.bC) * TPCC_C_WORDS;
            default: return y.st + (u64)(L.rec - y.bS) * TPCC_S_WORDS;
        }
    }
    static GC_DEV int row_words(const Lane &L) {
        return L.kind == KC ? TPCC_C_WORDS : (L.kind == KS ? TPCC_S_WORDS : TPCC_W_WORDS);
    }

    // customer of a Payment: by id, or by last name through the immutable index (Z16)
    static GC_DEV int64_t customer_of(const TpccParams &y, const uint32_t *t) {
        if (t[TX_C] != 0xFFFFFFFFu) return t[TX_C];
        const uint32_t lw = t[TX_CW] - y.w_first;
        const uint32_t grp = (lw * TPCC_DIST + t[TX_CD]) * 1000u + t[TX_CLAST];
        const uint32_t n = y.nidx_count[grp];
        if (n == 0) return -1;
        const uint32_t row = y.nidx_rows[y.nidx_start[grp] + (n + 1) / 2 - 1];   // ceil(n/2), §2.5.2.2
        return row % TPCC_CUST;
    }

    static GC_DEV bool load_lane(const ExecParams &p, const TpccParams &y, u32 gid, u32 i, Lane &L) {
        const uint32_t *t = y.tx + (u64)gid * TPCC_TX_WORDS;
        const uint32_t type = t[TX_TYPE];
        const uint32_t n = type == 0 ? 3 + t[TX_OLCNT] : 3;
        L.act = i < n;
        L.type = (uint8_t)type;
        if (!L.act) return true;
        if (p.acc_rec) L.rec = p.acc_rec[(u64)gid * p.K + i];
        const uint32_t lw = t[TX_W] - y.w_first;
        if (i == 0) {
            L.kind = KW;
            L.w = type == 1;
            if (!p.acc_rec) L.rec = (u32)(y.bW + lw);
        } else if (i == 1) {
            L.kind = KD;
            L.w = true;
            if (!p.acc_rec) L.rec = (u32)(y.bD + (u64)lw * TPCC_DIST + t[TX_D]);
        } else if (i == 2) {
            L.kind = KC;
            L.w = type == 1;
            if (!p.acc_rec) {
                const int64_t c = type == 0 ? (int64_t)t[TX_C] : customer_of(y, t);
                if (c < 0) return false;
                const uint32_t cw = (type == 0 ? t[TX_W] : t[TX_CW]) - y.w_first;
                const uint32_t cd = type == 0 ? t[TX_D] : t[TX_CD];
                L.rec = (u32)(y.bC + ((u64)cw * TPCC_DIST + cd) * TPCC_CUST + (u64)c);
            }
        } else {
            L.kind = KS;
            L.w = true;
            L.line = i - 3;
            L.item = t[TX_ITEM + L.line];
            L.sw = t[TX_SUPQ + L.line] >> 8;
            L.qty = t[TX_SUPQ + L.line] & 0xFF;
            if (!p.acc_rec) L.rec = (u32)(y.bS + (u64)(L.sw - y.w_first) * TPCC_STOCK + L.item);
            const u64 *ir = y.it + (u64)L.item * TPCC_I_WORDS;   // Item: immutable, outside CC
            L.price = (u32)ir[0];
            L.brand_i = has_original(reinterpret_cast<const uint8_t *>(ir + 4));
        }
        if (!p.skip || !p.skip[gid]) prefetch_access(p, y, L);
        return true;
    }

    static GC_DEV void prefetch_access(const ExecParams &p, const TpccParams &y, const Lane &L) {
        const u64 *rw = row(y, L);
        const int n = row_words(L);
        for (int k = 0; k < n && k < 40; k += 16) prefetch_l2(rw + k);   // the fields read
        prefetch_l2(p.scheme == CC_MVCC ? mvcc_lo(p, L.rec) : cw(p, L.rec));
    }

    static GC_DEV u64 warm(const ExecParams &, const TpccParams &, const Lane &) { return 0; }


    template <class LA>
    static GC_DEV u32 load_all(const ExecParams &p, const TpccParams &y, u32 gid, LA L) {
        const uint32_t *t = y.tx + (u64)gid * TPCC_TX_WORDS;
        const u32 n = t[TX_TYPE] == 0 ? 3 + t[TX_OLCNT] : 3;
        for (u32 i = 0; i < n; i++)
            if (!load_lane(p, y, gid, i, L[i])) return 0xFFFFFFFFu;
        return n;
    }

    // the same test on s_data read through L2 as words: the 8-byte window at byte offset
    // i < 43 of the 50 letters, assembled from two adjacent little-endian words in registers
    // (a byte array here lived in local memory)
    static GC_DEV bool has_original_words(const u64 *src) {
        constexpr u64 ORIG = 0x4C414E494749524Full;   // "ORIGINAL" as a little-endian u64
        bool found = false;
        u64 a = ld_cg(src);
#pragma unroll
        for (int j = 0; j < 6; j++) {
            const u64 b = ld_cg(src + j + 1);
#pragma unroll
            for (int r = 0; r < 8; r++) {
                if (8 * j + r > 42) break;
                const u64 win = r ? ((a >> (8 * r)) | (b << (64 - 8 * r))) : a;
                found |= win == ORIG;
            }
            a = b;
        }
        return found;
    }

    static GC_DEV bool has_original(const uint8_t *s) {
        for (int i = 0; i + 8 <= 50; i++) {
            bool m = true;
            for (int k = 0; k < 8 && m; k++) m = s[i + k] == (uint8_t)"ORIGINAL"[k];
            if (m) return true;
        }
        return false;
    }

    // Read the fields the transaction needs and compute its buffered new values
    // (every write is a read-modify-write of the item's own row, so it can be
    // installed at commit from this snapshot under every scheme).
    static GC_DEV void read(const TpccParams &y, Lane &L, u32 gid, u32, const u64 *src) {
        const uint32_t *t = y.tx + (u64)gid * TPCC_TX_WORDS;
        switch (L.kind) {
            case KW:
                if (L.type == 0) {
                    L.v0 = (u32)ld_cg(src + 1);                          // w_tax
                } else {
                    L.v1 = ld_cg(src) + t[TX_HAMT];                     // w_ytd += h
                    L.s0 = ld_cg(src + 2);                              // w_name
                    L.s1 = ld_cg(src + 3);
                }
                break;
            case KD: {
                const u64 w1 = ld_cg(src + 1);
                if (L.type == 0) {
                    L.v0 = (u32)w1;                                     // d_tax
                    L.v1 = w1 >> 32;                                    // o_id = d_next_o_id
                    L.v2 = (w1 & 0xFFFFFFFFull) | ((L.v1 + 1) << 32);   // d_next_o_id += 1
                } else {
                    L.v1 = ld_cg(src) + t[TX_HAMT];                     // d_ytd += h
                    L.s0 = ld_cg(src + 2);
                    L.s1 = ld_cg(src + 3);
                }
                break;
            }
            case KC: {
                const u64 w3 = ld_cg(src + 3);
                L.v3 = w3;                                              // discount | credit
                if (L.type == 1) {
                    const u64 h = t[TX_HAMT];
                    L.v0 = ld_cg(src) - h;                              // c_balance -= h
                    L.v1 = ld_cg(src + 1) + h;                          // c_ytd_payment += h
                    const u64 w2 = ld_cg(src + 2);
                    L.v2 = (w2 & ~0xFFFFFFFFull) | (u64)((u32)w2 + 1);  // c_payment_cnt += 1
                    // the 32-byte record a "BC" customer prepends to c_data (R7)
                    const u64 c = (L.rec - y.bC) % TPCC_CUST;
                    L.s0 = (c + 1) | ((u64)(t[TX_CD] + 1) << 32);
                    L.s1 = (u64)(t[TX_CW] + 1) | ((u64)(t[TX_D] + 1) << 32);
                    L.s2 = (u64)t[TX_W] + 1;
                    L.s3 = h;
                }
                break;
            }
            default: {
                const u64 w0 = ld_cg(src), w2 = ld_cg(src + 2);
                const u32 q = (u32)w0;
                const u32 nq = (q >= L.qty + 10) ? q - L.qty : q - L.qty + 91;
                L.v0 = (u64)nq | ((u64)((u32)(w0 >> 32) + 1) << 32);   // s_quantity, s_order_cnt += 1
                L.v1 = ld_cg(src + 1) + L.qty;                          // s_ytd += qty
                L.v2 = (L.sw != t[TX_W]) ? ((w2 & ~0xFFFFFFFFull) | (u64)((u32)w2 + 1)) : w2;   // remote
                const u32 d = t[TX_D];
                L.s0 = ld_cg(src + 3 + 3 * d);                          // s_dist_{d}
                L.s1 = ld_cg(src + 4 + 3 * d);
                L.s2 = ld_cg(src + 5 + 3 * d);
                const bool bs = has_original_words(src + 33);
                L.v3 = (u64)q | ((u64)(bs && L.brand_i) << 32);         // q before, brand-generic
                break;
            }
        }
    }

    static GC_DEV void install(const TpccParams &y, const Lane &L, u64 *dst) {
        switch (L.kind) {
            case KW:
                st_cg(dst, L.v1);
                break;
            case KD:
                if (L.type == 0) st_cg(dst + 1, L.v2);
                else st_cg(dst, L.v1);
                break;
            case KC: {
                st_cg(dst, L.v0);
                st_cg(dst + 1, L.v1);
                st_cg(dst + 2, L.v2);
                if (((L.v3 >> 32) & 0xFFFF) == 0x4342) {   // "BC": c_data = rec32 || c_data[0:472] (R7)
                    u64 *cd = dst + TPCC_CDATA_OFF;
                    for (int k = TPCC_CDATA_WORDS - 1; k >= 4; k--) st_cg(cd + k, ld_cg(cd + k - 4));
                    st_cg(cd + 0, L.s0);
                    st_cg(cd + 1, L.s1);
                    st_cg(cd + 2, L.s2);
                    st_cg(cd + 3, L.s3);
                }
                break;
            }
            default:
                st_cg(dst, L.v0);
                st_cg(dst + 1, L.v1);
                st_cg(dst + 2, L.v2);
                break;
        }
    }

    static GC_DEV void copy_row(const Lane &L, const u64 *src, u64 *dst) {
        const int n = row_words(L);
        for (int j = 0; j < n; j += 2) {
            u64 a, b;
            ld_cg_v2(src + j, a, b);
            st_cg_v2(dst + j, a, b);
        }
    }

    // h_data = w_name[10] || 4 spaces || d_name[10] (TPC-C §2.5.2.2)
    static GC_DEV void h_data(u64 ws0, u64 ws1, u64 ds0, u64 ds1, u64 out[3]) {
        out[0] = ws0;
        out[1] = (ws1 & 0xFFFFull) | (0x20202020ull << 16) | ((ds0 & 0xFFFFull) << 48);
        out[2] = (ds0 >> 16) | ((ds1 & 0xFFFFull) << 48);
    }

    static GC_DEV u64 total_of(u64 sum, u64 disc, u64 w_tax, u64 d_tax) {
        const long long num = (long long)sum * (long long)(10000 - disc) * (long long)(10000 + w_tax + d_tax);
        return (u64)((num + 50000000ll) / 100000000ll);   // round half up (Z18)
    }

    // private writes after commit: outputs and the reserved O / NO / OL / H slots (Z15)
    static GC_DEV void write_line(const ExecParams &p, const TpccParams &y, u32 gid, const uint32_t *t,
                                  const Lane &L, u64 o_id) {
        const u64 amount = (u64)L.qty * L.price;
        u64 *ol = y.ol + ((u64)gid * TPCC_MAXOL + L.line) * TPCC_OL_WORDS;
        st_cg(ol + 0, o_id | ((u64)(L.line + 1) << 32));
        st_cg(ol + 1, (u64)(t[TX_D] + 1) | ((u64)(t[TX_W] + 1) << 32));
        st_cg(ol + 2, (u64)(L.item + 1) | ((u64)(L.sw + 1) << 32));
        st_cg(ol + 3, L.qty);
        st_cg(ol + 4, amount);
        st_cg(ol + 5, L.s0);
        st_cg(ol + 6, L.s1);
        st_cg(ol + 7, L.s2);
        if (p.read_out) {
            u64 *out = p.read_out + (u64)gid * TPCC_OUT_WORDS + 2 + 3 * L.line;
            out[0] = (u32)L.v3;
            out[1] = (L.v3 >> 32) ? 'B' : 'G';
            out[2] = amount;
        }
    }

    static GC_DEV void write_header(const ExecParams &p, const TpccParams &y, u32 gid, const uint32_t *t,
                                    u64 w_v0, u64 w_s0, u64 w_s1, u64 d_v0, u64 d_v1, u64 d_s0, u64 d_s1,
                                    u64 c_v0, u64 c_v3, u32 c_rec, u64 sum) {
        u64 *out = p.read_out ? p.read_out + (u64)gid * TPCC_OUT_WORDS : nullptr;
        const u64 c1 = (c_rec - y.bC) % TPCC_CUST + 1;
        if (t[TX_TYPE] == 0) {
            const u64 o_id = d_v1;
            u64 *o = y.o + (u64)gid * TPCC_O_WORDS;
            st_cg(o + 0, o_id);
            st_cg(o + 1, t[TX_D] + 1);
            st_cg(o + 2, t[TX_W] + 1);
            st_cg(o + 3, c1);
            st_cg(o + 4, y.entry_date);
            st_cg(o + 5, t[TX_OLCNT]);
            st_cg(o + 6, t[TX_ALLLOCAL]);
            st_cg(o + 7, 0);
            u64 *no = y.no + (u64)gid * TPCC_NO_WORDS;
            st_cg(no + 0, o_id);
            st_cg(no + 1, t[TX_D] + 1);
            st_cg(no + 2, t[TX_W] + 1);
            st_cg(no + 3, 0);
            if (out) {
                out[0] = o_id;
                out[1] = total_of(sum, (u32)c_v3, w_v0, d_v0);
            }
        } else {
            u64 *h = y.h + (u64)gid * TPCC_H_WORDS;
            st_cg(h + 0, c1 | ((u64)(t[TX_CD] + 1) << 32));
            st_cg(h + 1, (u64)(t[TX_CW] + 1) | ((u64)(t[TX_D] + 1) << 32));
            st_cg(h + 2, (u64)t[TX_W] + 1);
            st_cg(h + 3, y.entry_date);
            st_cg(h + 4, t[TX_HAMT]);
            u64 hd[3];
            h_data(w_s0, w_s1, d_s0, d_s1, hd);
            st_cg(h + 5, hd[0]);
            st_cg(h + 6, hd[1]);
            st_cg(h + 7, hd[2]);
            if (out) {
                out[0] = c1;
                out[1] = c_v0;
                out[2] = (c_v3 >> 32) & 0xFFFF;
            }
        }
    }

    template <class LA>
    static GC_DEV void emit_txn(const ExecParams &p, const TpccParams &y, u32 gid, LA L, u32 n) {
        const uint32_t *t = y.tx + (u64)gid * TPCC_TX_WORDS;
        u64 sum = 0;
        for (u32 i = 3; i < n; i++) {
            sum += (u64)L[i].qty * L[i].price;
            write_line(p, y, gid, t, L[i], L[1].v1);
        }
        write_header(p, y, gid, t, L[0].v0, L[0].s0, L[0].s1, L[1].v0, L[1].v1, L[1].s0, L[1].s1, L[2].v0,
                     L[2].v3, L[2].rec, sum);
    }

    template <class Tile>
    static GC_DEV void emit_tile(Tile &tile, const ExecParams &p, const TpccParams &y, u32 gid, const Lane &L,
                                 u32 i) {
        const uint32_t *t = y.tx + (u64)gid * TPCC_TX_WORDS;
        const u64 w_v0 = tile.shfl(L.v0, 0), w_s0 = tile.shfl(L.s0, 0), w_s1 = tile.shfl(L.s1, 0);
        const u64 d_v0 = tile.shfl(L.v0, 1), d_v1 = tile.shfl(L.v1, 1), d_s0 = tile.shfl(L.s0, 1),
                  d_s1 = tile.shfl(L.s1, 1);
        const u64 c_v0 = tile.shfl(L.v0, 2), c_v3 = tile.shfl(L.v3, 2);
        const u32 c_rec = tile.shfl(L.rec, 2);
        const u64 amt = (L.act && L.kind == KS) ? (u64)L.qty * L.price : 0ull;
        const u64 sum = cg::reduce(tile, amt, cg::plus<u64>());
        if (L.act && L.kind == KS) write_line(p, y, gid, t, L, d_v1);
        if (i == 0) write_header(p, y, gid, t, w_v0, w_s0, w_s1, d_v0, d_v1, d_s0, d_s1, c_v0, c_v3, c_rec, sum);
    }
};

// ---------------------------------------------------------------- launchers
template <int S>
static cudaError_t launch_s(const ExecParams &p, const TpccParams &y, int grid, int block, size_t smem,
                            cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    auto go = [&](auto kern) {
        if (smem > 32 * 1024) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) kern<<<grid, block, smem, s>>>(p, y);
    };
    if (p.lanes > 1) go(exec_tile_kernel<S, TpccWL, 32>);
    else go(exec_thread_kernel<S, TpccWL>);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_tpcc_exec(const ExecParams &p, const TpccParams &y, int grid, int block, size_t smem,
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
static int occ_of(F f, int block, size_t smem) {
    int nb = 0;
    if (smem > 32 * 1024) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, block, smem);
    return nb;
}
template <int S>
static int occ_s(int lanes, int block, size_t smem) {
    return lanes > 1 ? occ_of(exec_tile_kernel<S, TpccWL, 32>, block, smem)
                     : occ_of(exec_thread_kernel<S, TpccWL>, block, smem);
}
size_t tpcc_lane_bytes() { return sizeof(TpccWL::Lane); }
int tpcc_exec_max_blocks_per_sm(int scheme, int lanes, int block, size_t smem) {
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

// a3 gather: one thread per transaction; unused access slots get a sentinel record
// (all-ones in the record bits) so they sort after every real item and are skipped.
__global__ void tpcc_gather_kernel(ExecParams p, TpccParams y, uint32_t *acc_rec, unsigned long long *keys,
                                   u64 sentinel) {
    const u32 gid = blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= p.n_txn) return;
    ExecParams q = p;
    q.acc_rec = nullptr;
    const u64 base = (u64)gid * p.K;
    const uint32_t *t = y.tx + (u64)gid * TPCC_TX_WORDS;
    const u32 n = (p.skip && p.skip[gid]) ? 0 : (t[TX_TYPE] == 0 ? 3 + t[TX_OLCNT] : 3);
    for (u32 i = 0; i < (u32)p.K; i++) {
        if (i < n) {
            TpccWL::Lane L;
            if (!TpccWL::load_lane(q, y, gid, i, L)) {   // reported; sentinel keeps a3 / exec in bounds
                atomicCAS(&p.ctl->err.v, 0ull, (u64)CC_ERR_KEY_NOT_FOUND);
                acc_rec[base + i] = 0xFFFFFFFFu;
                keys[base + i] = (sentinel << 27) | ((u64)gid << 6) | ((u64)i << 1);
                continue;
            }
            acc_rec[base + i] = L.rec;
            keys[base + i] = ((u64)L.rec << 27) | ((u64)gid << 6) | ((u64)i << 1) | (u64)L.w;
        } else {
            acc_rec[base + i] = 0xFFFFFFFFu;
            keys[base + i] = (sentinel << 27) | ((u64)gid << 6) | ((u64)i << 1);
        }
    }
}

cudaError_t launch_tpcc_gather(const ExecParams &p, const TpccParams &y, PrepBufs &b, uint64_t n_records,
                               cudaStream_t s) {
    int bits = 1;
    while (bits < 37 && (1ull << bits) <= n_records) bits++;
    tpcc_gather_kernel<<<(p.n_txn + 127) / 128, 128, 0, s>>>(p, y, b.acc_rec, b.keys_in, (1ull << bits) - 1);
    return cudaGetLastError();
}


void preload_tpcc_kernels() {   // (see preload_prep_kernels) every executor instantiation
    for (int sc = 0; sc < CC_NUM_SCHEMES; sc++) {
        tpcc_exec_max_blocks_per_sm(sc, 1, 256, 0);
        tpcc_exec_max_blocks_per_sm(sc, 32, 256, 0);
    }
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, tpcc_gen_kernel);
    cudaFuncGetAttributes(&a, tpcc_gather_kernel);
}
}  // namespace gcctb
