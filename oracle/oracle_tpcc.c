/*
 * oracle_tpcc.c -- CPU ORACLE, TEST INFRASTRUCTURE ONLY (see oracle_ycsb.c header).
 *
 * Serial semantics of the two TPC-C transactions the paper evaluates (PAPER.md:467-468:
 * NewOrder and Payment, "together 88% of the default workload mix"), restricted to
 * reads and writes, with the readings of SURVEY.md §8(c) and
 * money in i64 cents, rates in 1/10,000, inserts become writes to
 * per-transaction reserved slots (Z15), Item and the customer last-name order are
 * immutable (Z16), NewOrder's 1% rollback omitted (Z17), totals rounded half up (Z18),
 * NewOrder increments d_next_o_id (Z14).  Row layouts: inputs/tpcc.py docstring
 * (a specification both sides implement independently).
 *
 * Also the TPC-C a1 batch generator, step by step (TPC-C §2.4.1 / §2.5.1 input
 * generation; NURand per §2.1.6), and the by-name customer selection (§2.5.2.2:
 * the row at position ceil(n/2) of the customers with that last name sorted by
 * c_first; ties in c_first broken by c_id -- reading R5).
 *
 * Pins (tests/test_oracle_tpcc.py): TPC-C §3.3.2 consistency conditions 1-4, 8-9 in
 * delta form, per-customer and per-stock conservation, a hand-worked NewOrder total,
 * NURand range / non-uniformity, remote rates, and serial-order sensitivity;
 * tests/test_oracle_pins.py: a hand-worked BC Payment (c_data rewrite, h_data, history,
 * tests/golden/tpcc_payment_bc.json) and orc_tpcc_accesses against the rows a replay
 * writes / the rows whose perturbation changes the output.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_CONFIG 2
#define ORC_ERR_OOM 3
#define ORC_ERR_KEY 6

/* ---- layout (inputs/tpcc.py) ---- */
#define TW_WORDS 16
#define TD_WORDS 16
#define TC_WORDS 88
#define TS_WORDS 40
#define TI_WORDS 12
#define TO_WORDS 8
#define TNO_WORDS 4
#define TOL_WORDS 8
#define TH_WORDS 8
#define NDIST 10
#define NCUST 3000
#define NSTOCK 100000
#define NITEM 100000
#define MAXOL 15
#define CDATA_OFF 25
#define CDATA_WORDS 63

/* txn descriptor: 40 u32 */
#define TX_WORDS 40
enum { TX_TYPE = 0, TX_W, TX_D, TX_CW, TX_CD, TX_C, TX_CLAST, TX_HAMT, TX_OLCNT, TX_ALLLOCAL,
       TX_ITEM = 10, TX_SUPQ = 25 };

typedef struct {
    uint32_t W;
    uint64_t *wh, *di, *cu, *st;   /* CC tables */
    const uint64_t *it;            /* immutable items */
    uint64_t *o, *no, *ol, *h;     /* reserved slots: o/no/h [n_txn], ol [n_txn*15] */
    uint64_t entry_date;
} orc_tpcc_db;

static uint64_t orc_mix64t(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static uint64_t orc_rng3(uint64_t seed, uint64_t a, uint64_t b) {
    return orc_mix64t(orc_mix64t(seed ^ orc_mix64t(a)) ^ b);
}

/* ---------------------------------------------------------------- generator (a1) */
enum { S_TYPE = 1, S_W, S_D, S_CA, S_CB, S_OLCNT, S_ITEMA, S_ITEMB, S_SUP, S_SUPW, S_QTY,
       S_BYNAME, S_REMOTE, S_CW, S_CD, S_LASTA, S_LASTB, S_HAMT };

static uint64_t draw(uint64_t seed, uint32_t gid, uint64_t stream, uint64_t j, uint64_t k) {
    return orc_rng3(seed, gid, (stream << 56) | (j << 24) | k);
}
/* rand(lo, hi) inclusive, TPC-C §2.1.5 */
static uint64_t urand(uint64_t u, uint64_t lo, uint64_t hi) { return lo + u % (hi - lo + 1); }
/* NURand(A, x, y) = (((rand(0,A) | rand(x,y)) + C) % (y-x+1)) + x, TPC-C §2.1.6 */
static uint64_t nurand(uint64_t ua, uint64_t ub, uint64_t A, uint64_t x, uint64_t y, uint64_t C) {
    return (((urand(ua, 0, A) | urand(ub, x, y)) + C) % (y - x + 1)) + x;
}

/* gen parameters: no_permyriad = NewOrder share in 1/10,000; home warehouses
 * [w_lo, w_hi); c_id/c_last/ol_i_id NURand constants; remote percentages. */
int orc_tpcc_gen(uint64_t seed, uint32_t W, uint32_t w_lo, uint32_t w_hi, uint32_t n_txn,
                 uint32_t no_permyriad, uint32_t c_last_run, uint32_t c_id_c, uint32_t c_item_c,
                 uint32_t *tx_out) {
    if (W == 0 || w_hi <= w_lo || w_hi > W) return ORC_ERR_CONFIG;
    for (uint32_t g = 0; g < n_txn; g++) {
        uint32_t *t = tx_out + (uint64_t)g * TX_WORDS;
        memset(t, 0, TX_WORDS * 4);
        const uint32_t w = w_lo + (uint32_t)(draw(seed, g, S_W, 0, 0) % (w_hi - w_lo));
        const uint32_t d = (uint32_t)(draw(seed, g, S_D, 0, 0) % NDIST);
        t[TX_W] = w;
        t[TX_D] = d;
        if (draw(seed, g, S_TYPE, 0, 0) % 10000 < no_permyriad) {   /* NewOrder, §2.4.1 */
            t[TX_TYPE] = 0;
            t[TX_CW] = w;
            t[TX_CD] = d;
            t[TX_C] = (uint32_t)nurand(draw(seed, g, S_CA, 0, 0), draw(seed, g, S_CB, 0, 0), 1023, 1, NCUST, c_id_c) - 1;
            t[TX_CLAST] = 0xFFFFFFFFu;
            const uint32_t n = (uint32_t)urand(draw(seed, g, S_OLCNT, 0, 0), 5, 15);
            t[TX_OLCNT] = n;
            uint32_t items[MAXOL], sq[MAXOL];
            uint32_t all_local = 1;
            for (uint32_t j = 0; j < n; j++) {
                for (uint64_t k = 0;; k++) {   /* distinct items per order (reading R6) */
                    if (k > 4096) return ORC_ERR_CONFIG;
                    uint32_t i = (uint32_t)nurand(draw(seed, g, S_ITEMA, j, k), draw(seed, g, S_ITEMB, j, k),
                                                  8191, 1, NITEM, c_item_c) - 1;
                    int dup = 0;
                    for (uint32_t q = 0; q < j; q++) dup |= (items[q] == i);
                    if (!dup) { items[j] = i; break; }
                }
                uint32_t sw = w;
                if (W > 1 && draw(seed, g, S_SUP, j, 0) % 100 == 0) {   /* 1% remote supply, §2.4.1.5 */
                    uint32_t o = (uint32_t)(draw(seed, g, S_SUPW, j, 0) % (W - 1));
                    sw = o >= w ? o + 1 : o;
                }
                if (sw != w) all_local = 0;
                const uint32_t qty = (uint32_t)urand(draw(seed, g, S_QTY, j, 0), 1, 10);
                sq[j] = (sw << 8) | qty;
            }
            /* lines in stock-key order (supply_w, i): the global lock order (Z23) */
            for (uint32_t a = 1; a < n; a++) {
                uint32_t ki = items[a], ks = sq[a];
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
        } else {   /* Payment, §2.5.1 */
            t[TX_TYPE] = 1;
            uint32_t cw = w, cd = d;
            if (W > 1 && draw(seed, g, S_REMOTE, 0, 0) % 100 < 15) {   /* 15% remote customer */
                uint32_t o = (uint32_t)(draw(seed, g, S_CW, 0, 0) % (W - 1));
                cw = o >= w ? o + 1 : o;
                cd = (uint32_t)(draw(seed, g, S_CD, 0, 0) % NDIST);
            }
            t[TX_CW] = cw;
            t[TX_CD] = cd;
            if (draw(seed, g, S_BYNAME, 0, 0) % 100 < 60) {   /* 60% by last name */
                t[TX_C] = 0xFFFFFFFFu;
                t[TX_CLAST] = (uint32_t)nurand(draw(seed, g, S_LASTA, 0, 0), draw(seed, g, S_LASTB, 0, 0), 255, 0, 999, c_last_run);
            } else {
                t[TX_C] = (uint32_t)nurand(draw(seed, g, S_CA, 0, 0), draw(seed, g, S_CB, 0, 0), 1023, 1, NCUST, c_id_c) - 1;
                t[TX_CLAST] = 0xFFFFFFFFu;
            }
            t[TX_HAMT] = (uint32_t)urand(draw(seed, g, S_HAMT, 0, 0), 100, 500000);
        }
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------- by-name lookup */
/* §2.5.2.2: customers of (w, d) whose c_last equals the name of number `last`, sorted by
 * c_first (16-byte, memcmp order; ties by c_id, reading R5); the row at position
 * ceil(n/2) (1-based).  Plain scan of all 3,000 customers. */
static int orc_last_bytes(uint32_t num, uint8_t out[16]) {
    static const char *syl[10] = {"BAR", "OUGHT", "ABLE", "PRI", "PRES", "ESE", "ANTI", "CALLY", "ATION", "EING"};
    memset(out, 0, 16);
    size_t p = 0;
    const uint32_t dig[3] = {num / 100, (num / 10) % 10, num % 10};
    for (int k = 0; k < 3; k++) {
        size_t l = strlen(syl[dig[k]]);
        memcpy(out + p, syl[dig[k]], l);
        p += l;
    }
    return 0;
}

int64_t orc_tpcc_by_name(const uint64_t *cu, uint32_t w, uint32_t d, uint32_t last) {
    uint8_t name[16];
    orc_last_bytes(last, name);
    uint32_t ids[NCUST];
    uint32_t n = 0;
    const uint64_t base = ((uint64_t)w * NDIST + d) * NCUST;
    for (uint32_t c = 0; c < NCUST; c++)
        if (memcmp(cu + (base + c) * TC_WORDS + 4, name, 16) == 0) ids[n++] = c;
    if (n == 0) return -1;
    /* insertion sort by (c_first bytes, c_id) */
    for (uint32_t a = 1; a < n; a++) {
        uint32_t v = ids[a];
        const uint8_t *fv = (const uint8_t *)(cu + (base + v) * TC_WORDS + 6);
        int b = (int)a - 1;
        while (b >= 0) {
            const uint8_t *fb = (const uint8_t *)(cu + (base + ids[b]) * TC_WORDS + 6);
            int c = memcmp(fb, fv, 16);
            if (c > 0 || (c == 0 && ids[b] > v)) { ids[b + 1] = ids[b]; b--; }
            else break;
        }
        ids[b + 1] = v;
    }
    return ids[(n + 1) / 2 - 1];
}

/* ---------------------------------------------------------------- transactions */
static uint32_t lo32(uint64_t x) { return (uint32_t)x; }
static uint32_t hi32(uint64_t x) { return (uint32_t)(x >> 32); }
static int has_original(const uint8_t *s, int n) {
    for (int i = 0; i + 8 <= n; i++)
        if (memcmp(s + i, "ORIGINAL", 8) == 0) return 1;
    return 0;
}

/* NewOrder (TPC-C §2.4.2, reads and writes only).  out[0] = o_id, out[1] = total,
 * out[2+3j .. 4+3j] = (s_quantity before the update, brand-generic 'B'/'G', ol_amount)
 * for line j in stock-key order. */
static void orc_neworder(orc_tpcc_db *db, uint32_t g, const uint32_t *t, uint64_t *out) {
    const uint32_t w = t[TX_W], d = t[TX_D], c = t[TX_C], n = t[TX_OLCNT];
    const uint64_t *wr = db->wh + (uint64_t)w * TW_WORDS;
    uint64_t *dr = db->di + ((uint64_t)w * NDIST + d) * TD_WORDS;
    const uint64_t *cr = db->cu + (((uint64_t)w * NDIST + d) * NCUST + c) * TC_WORDS;
    const uint64_t w_tax = lo32(wr[1]);
    const uint64_t d_tax = lo32(dr[1]);
    const uint32_t o_id = hi32(dr[1]);
    dr[1] = (dr[1] & 0xFFFFFFFFull) | ((uint64_t)(o_id + 1) << 32);   /* d_next_o_id += 1 (Z14) */
    const uint64_t disc = lo32(cr[3]);
    uint64_t *o = db->o + (uint64_t)g * TO_WORDS;
    o[0] = o_id; o[1] = d + 1; o[2] = w + 1; o[3] = c + 1; o[4] = db->entry_date; o[5] = n;
    o[6] = t[TX_ALLLOCAL]; o[7] = 0;
    uint64_t *no = db->no + (uint64_t)g * TNO_WORDS;
    no[0] = o_id; no[1] = d + 1; no[2] = w + 1; no[3] = 0;
    int64_t sum = 0;
    out[0] = o_id;
    for (uint32_t j = 0; j < n; j++) {
        const uint32_t i = t[TX_ITEM + j], sw = t[TX_SUPQ + j] >> 8, qty = t[TX_SUPQ + j] & 0xFF;
        const uint64_t *ir = db->it + (uint64_t)i * TI_WORDS;
        uint64_t *sr = db->st + ((uint64_t)sw * NSTOCK + i) * TS_WORDS;
        const uint64_t price = lo32(ir[0]);
        const uint32_t q = lo32(sr[0]);
        const uint32_t nq = (q >= qty + 10) ? q - qty : q - qty + 91;
        sr[0] = (uint64_t)nq | ((uint64_t)(hi32(sr[0]) + 1) << 32);   /* s_order_cnt += 1 */
        sr[1] += qty;                                                  /* s_ytd += qty */
        if (sw != w) sr[2] = (sr[2] & ~0xFFFFFFFFull) | (uint64_t)(lo32(sr[2]) + 1);   /* s_remote_cnt */
        const int64_t amount = (int64_t)qty * (int64_t)price;
        sum += amount;
        const int brand = has_original((const uint8_t *)(ir + 4), 50) && has_original((const uint8_t *)(sr + 33), 50);
        uint64_t *ol = db->ol + ((uint64_t)g * MAXOL + j) * TOL_WORDS;
        ol[0] = (uint64_t)o_id | ((uint64_t)(j + 1) << 32);
        ol[1] = (uint64_t)(d + 1) | ((uint64_t)(w + 1) << 32);
        ol[2] = (uint64_t)(i + 1) | ((uint64_t)(sw + 1) << 32);
        ol[3] = qty;
        ol[4] = (uint64_t)amount;
        memcpy(ol + 5, sr + 3 + 3 * d, 24);   /* ol_dist_info = s_dist_{d} */
        out[2 + 3 * j] = q;
        out[3 + 3 * j] = brand ? 'B' : 'G';
        out[4 + 3 * j] = (uint64_t)amount;
    }
    /* total = round_half_up(sum * (1 - disc) * (1 + w_tax + d_tax)) in 1/10^8 (Z18) */
    const int64_t num = sum * (int64_t)(10000 - disc) * (int64_t)(10000 + w_tax + d_tax);
    out[1] = (uint64_t)((num + 50000000) / 100000000);
}

/* Payment (TPC-C §2.5.2).  out[0] = c_id (1-based), out[1] = c_balance after, out[2] = credit. */
static int orc_payment(orc_tpcc_db *db, uint32_t g, const uint32_t *t, uint64_t *out) {
    const uint32_t w = t[TX_W], d = t[TX_D], cw = t[TX_CW], cd = t[TX_CD];
    const uint64_t h = t[TX_HAMT];
    uint64_t *wr = db->wh + (uint64_t)w * TW_WORDS;
    uint64_t *dr = db->di + ((uint64_t)w * NDIST + d) * TD_WORDS;
    wr[0] += h;                                      /* w_ytd += h_amount */
    dr[0] += h;                                      /* d_ytd += h_amount */
    int64_t c = t[TX_C];
    if (t[TX_C] == 0xFFFFFFFFu) {
        c = orc_tpcc_by_name(db->cu, cw, cd, t[TX_CLAST]);
        if (c < 0) return ORC_ERR_KEY;
    }
    uint64_t *cr = db->cu + (((uint64_t)cw * NDIST + cd) * NCUST + (uint64_t)c) * TC_WORDS;
    cr[0] -= h;                                      /* c_balance -= h_amount */
    cr[1] += h;                                      /* c_ytd_payment += h_amount */
    cr[2] = (cr[2] & ~0xFFFFFFFFull) | (uint64_t)(lo32(cr[2]) + 1);   /* c_payment_cnt += 1 */
    const uint32_t credit = hi32(cr[3]) & 0xFFFF;
    if (credit == 0x4342) {   /* "BC": c_data = rec32 || c_data[0:472] (reading R7) */
        uint64_t *cd_w = cr + CDATA_OFF;
        memmove(cd_w + 4, cd_w, (CDATA_WORDS - 4) * 8);
        cd_w[0] = (uint64_t)(c + 1) | ((uint64_t)(cd + 1) << 32);
        cd_w[1] = (uint64_t)(cw + 1) | ((uint64_t)(d + 1) << 32);
        cd_w[2] = (uint64_t)(w + 1);
        cd_w[3] = h;
    }
    uint64_t *hr = db->h + (uint64_t)g * TH_WORDS;
    hr[0] = (uint64_t)(c + 1) | ((uint64_t)(cd + 1) << 32);
    hr[1] = (uint64_t)(cw + 1) | ((uint64_t)(d + 1) << 32);
    hr[2] = w + 1;
    hr[3] = db->entry_date;
    hr[4] = h;
    uint8_t hd[24];
    memcpy(hd, wr + 2, 10);                          /* h_data = w_name || 4 spaces || d_name */
    memset(hd + 10, ' ', 4);
    memcpy(hd + 14, dr + 2, 10);
    memcpy(hr + 5, hd, 24);
    out[0] = (uint64_t)c + 1;
    out[1] = cr[0];
    out[2] = credit;
    return ORC_OK;
}

/* out stride per transaction */
#define TPCC_OUT_WORDS 48

int orc_tpcc_replay(uint32_t W, uint64_t *wh, uint64_t *di, uint64_t *cu, uint64_t *st,
                    const uint64_t *it, uint64_t *o, uint64_t *no, uint64_t *ol, uint64_t *h,
                    uint64_t entry_date, uint32_t n_txn, const uint32_t *tx,
                    const uint32_t *order, uint32_t n_order, uint64_t *out) {
    orc_tpcc_db db = {W, wh, di, cu, st, it, o, no, ol, h, entry_date};
    for (uint32_t p = 0; p < n_order; p++) {
        const uint32_t g = order[p];
        if (g >= n_txn) return ORC_ERR_CONFIG;
        const uint32_t *t = tx + (uint64_t)g * TX_WORDS;
        uint64_t *ou = out + (uint64_t)g * TPCC_OUT_WORDS;
        if (t[TX_W] >= W || t[TX_CW] >= W) return ORC_ERR_KEY;
        if (t[TX_TYPE] == 0) orc_neworder(&db, g, t, ou);
        else {
            int st = orc_payment(&db, g, t, ou);
            if (st) return st;
        }
    }
    return ORC_OK;
}

/* CC-managed records touched by a transaction (global record id space W|D|C|S, the
 * order PAPER.md:343 "arranged consecutively"), ascending; used for GPUTx ranks and
 * GaccO queues of TPC-C batches.  Returns the count; mode bit0 = write. */
int orc_tpcc_accesses(uint32_t W, const uint64_t *cu, const uint32_t *t, uint64_t *rec, uint8_t *mode) {
    const uint64_t bW = 0, bD = W, bC = W + (uint64_t)W * NDIST, bS = bC + (uint64_t)W * NDIST * NCUST;
    const uint32_t w = t[TX_W], d = t[TX_D];
    int n = 0;
    if (t[TX_TYPE] == 0) {
        rec[n] = bW + w; mode[n++] = 0;
        rec[n] = bD + (uint64_t)w * NDIST + d; mode[n++] = 1;
        rec[n] = bC + ((uint64_t)w * NDIST + d) * NCUST + t[TX_C]; mode[n++] = 0;
        for (uint32_t j = 0; j < t[TX_OLCNT]; j++) {
            rec[n] = bS + (uint64_t)(t[TX_SUPQ + j] >> 8) * NSTOCK + t[TX_ITEM + j];
            mode[n++] = 1;
        }
    } else {
        int64_t c = t[TX_C];
        if (t[TX_C] == 0xFFFFFFFFu) c = orc_tpcc_by_name(cu, t[TX_CW], t[TX_CD], t[TX_CLAST]);
        if (c < 0) return -1;
        rec[n] = bW + w; mode[n++] = 1;
        rec[n] = bD + (uint64_t)w * NDIST + d; mode[n++] = 1;
        rec[n] = bC + ((uint64_t)t[TX_CW] * NDIST + t[TX_CD]) * NCUST + (uint64_t)c; mode[n++] = 1;
    }
    return n;
}
