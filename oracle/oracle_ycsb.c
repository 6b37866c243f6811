/*
 * oracle_ycsb.c -- CPU ORACLE, TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this code.  It shares no code, header, table or constant generator
 * with the CUDA library under paper_2406_10158_b200/; neither side includes the other.
 *
 * What it computes (plain, slow, single-threaded, obviously correct):
 *   - the serial semantics exec(t, S) of one YCSB transaction (SURVEY.md §8(c),
 *     reading Z11; keys distinct and ascending per PAPER.md:414 / SPEC.md:112);
 *   - serial replay of a batch in a given order (the definition of serializability
 *     the paper claims for every scheme);
 *   - the a1 batch generator, step by step (PAPER.md:457-465 YCSB 16 accesses,
 *     Zipf(theta), write fraction W; readings Z12, Z13);
 *   - GPUTx ranks = longest path in the id-ordered conflict DAG (PAPER.md:218 with
 *     reading Z1, reads do not conflict with reads per Z2);
 *   - GaccO queue positions: per item, the rank of the accessing transaction id
 *     among all transactions accessing the item.
 *
 * Parity pins (tests/test_oracle_*.py, -m "not gpu"): write-counter conservation,
 * read-only identity, commutation of disjoint transactions, order sensitivity of
 * shared keys, Zipf hottest-key frequency vs the Hurwitz-zeta closed form, binomial
 * bounds on W, SPEC.md worked examples for ranks / access tables (tests/golden/),
 * and same-rank non-conflict + minimality for ranks.  The fingerprint fp() and the
 * affine write are readings (Z11) with no paper value; tests/test_oracle_pins.py pins
 * them with closed forms on rows of special structure (single words, top bits, all-ones,
 * zero / one fields), so a wrong rotation, word, field, "+1" or counter fails.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_KEY 6      /* KeyNotFound */
#define ORC_ERR_CONFIG 2   /* ConfigError */
#define ORC_ERR_OOM 3

/* ---- counter-based generator (the oracle's own copy; same definition as the
 *      device generator by specification, never by shared code) ---- */
static uint64_t orc_mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t orc_rng(uint64_t seed, uint64_t a, uint64_t b) {
    return orc_mix64(orc_mix64(seed ^ orc_mix64(a)) ^ b);
}

static uint64_t orc_rotl(uint64_t x, unsigned r) {
    r &= 63u;
    if (r == 0) return x;
    return (x << r) | (x >> (64u - r));
}

/* fp(r) = sum_j rotl64(r[j], j) mod 2^64 -- reading Z11 (full-row fingerprint). */
uint64_t orc_ycsb_fp(const uint64_t *row) {
    uint64_t s = 0;
    for (unsigned j = 0; j < 16; j++) s += orc_rotl(row[j], j);
    return s;
}

/* exec(t, S) for one YCSB transaction, reading Z11:
 *   op i (key k, field f): out_i = fp(row_k); if write:
 *     row_k[f] = row_k[f] * 0x9E3779B97F4A7C15 + ((gid << 4) | i) + 1,  row_k[15] += 1.
 * Keys are primary keys = row ordinals (SPEC.md:55 identity index); a key outside
 * the table is KeyNotFound. */
int orc_ycsb_exec(uint64_t *rows, uint64_t n_rows, uint32_t gid, uint32_t K,
                  const uint32_t *keys, const uint8_t *ops, uint64_t *out) {
    for (uint32_t i = 0; i < K; i++) {
        uint64_t key = keys[i];
        if (key >= n_rows) return ORC_ERR_KEY;
        uint64_t *row = rows + 16u * key;
        out[i] = orc_ycsb_fp(row);
        if (ops[i] & 0x80u) {
            unsigned f = ops[i] & 0x0Fu;
            row[f] = row[f] * 0x9E3779B97F4A7C15ull + ((((uint64_t)gid) << 4) | i) + 1u;
            row[15] += 1u;
        }
    }
    return ORC_OK;
}

/* Serial replay: S := S0 (rows, in place); for t in order: (out_t, S) := exec(t, S).
 * SURVEY.md §8(c) "The definition", step 4.  out has n_txn*K slots (txns not in
 * `order` keep whatever the caller put there). */
int orc_ycsb_replay(uint64_t *rows, uint64_t n_rows, uint32_t n_txn, uint32_t K,
                    const uint32_t *keys, const uint8_t *ops,
                    const uint32_t *order, uint32_t n_order, uint64_t *out) {
    for (uint32_t p = 0; p < n_order; p++) {
        uint32_t t = order[p];
        if (t >= n_txn) return ORC_ERR_CONFIG;
        int st = orc_ycsb_exec(rows, n_rows, t, K, keys + (uint64_t)t * K,
                               ops + (uint64_t)t * K, out + (uint64_t)t * K);
        if (st) return st;
    }
    return ORC_OK;
}

/* Zipf rank from a uniform u64: rank = min(#{j : T[j] <= u}, n-1) + 1 (inputs/ycsb.py
 * zipf_thresholds contract).  Plain binary search for the count. */
static uint64_t orc_zipf_rank(const uint64_t *T, uint64_t n, uint64_t u) {
    uint64_t lo = 0, hi = n; /* count of T[j] <= u lies in [lo, hi] */
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (T[mid] <= u) lo = mid + 1; else hi = mid;
    }
    if (lo > n - 1) lo = n - 1;
    return lo + 1;
}

#define ORC_STREAM_KEY 1ull
#define ORC_STREAM_MODE 2ull
#define ORC_STREAM_FIELD 3ull

/* a1, YCSB:
 *   for each txn gid, op i: draw k = 0,1,... u = rng(seed, gid, KEY<<56 | i<<24 | k),
 *     rank = Zipf(u), key = ((rank-1) * A) mod n, until key differs from keys 0..i-1
 *     (resample duplicates);
 *   sort the txn's keys ascending;
 *   then per sorted position i: write iff (rng(seed,gid,MODE<<56|i) >> 11) < floor(W*2^53)
 *     (Bernoulli(W) per access, reading Z12), field = rng(seed,gid,FIELD<<56|i) mod 15.
 * Output: keys u32[n_txn*K], ops u8 (bit7 write, bits0..3 field). */
int orc_ycsb_gen(uint64_t seed, uint64_t n_rows, uint32_t n_txn, uint32_t K, double W,
                 const uint64_t *T, uint64_t A, uint32_t *keys_out, uint8_t *ops_out) {
    if (n_rows < K || K == 0 || K > 64 || n_rows > 0xFFFFFFFFull) return ORC_ERR_CONFIG;
    if (!(W >= 0.0 && W <= 1.0)) return ORC_ERR_CONFIG;
    uint64_t wthr = (uint64_t)(W * 9007199254740992.0); /* W * 2^53, exact scaling */
    for (uint32_t gid = 0; gid < n_txn; gid++) {
        uint32_t *kk = keys_out + (uint64_t)gid * K;
        for (uint32_t i = 0; i < K; i++) {
            for (uint64_t k = 0;; k++) {
                if (k >= (1u << 24)) return ORC_ERR_CONFIG;
                uint64_t u = orc_rng(seed, gid, (ORC_STREAM_KEY << 56) | ((uint64_t)i << 24) | k);
                uint64_t rank = orc_zipf_rank(T, n_rows, u);
                uint64_t key = ((rank - 1) * A) % n_rows;
                int dup = 0;
                for (uint32_t j = 0; j < i; j++) if (kk[j] == key) { dup = 1; break; }
                if (!dup) { kk[i] = (uint32_t)key; break; }
            }
        }
        /* insertion sort ascending */
        for (uint32_t i = 1; i < K; i++) {
            uint32_t v = kk[i];
            int32_t j = (int32_t)i - 1;
            while (j >= 0 && kk[j] > v) { kk[j + 1] = kk[j]; j--; }
            kk[j + 1] = v;
        }
        for (uint32_t i = 0; i < K; i++) {
            uint64_t um = orc_rng(seed, gid, (ORC_STREAM_MODE << 56) | i);
            uint64_t uf = orc_rng(seed, gid, (ORC_STREAM_FIELD << 56) | i);
            uint8_t op = (uint8_t)(uf % 15u);
            if ((um >> 11) < wthr) op |= 0x80u;
            ops_out[(uint64_t)gid * K + i] = op;
        }
    }
    return ORC_OK;
}

/* GPUTx rank, PAPER.md:218 read per Z1: rank(T) = 0 if no earlier transaction
 * conflicts with T, else 1 + max over conflicting earlier T' of rank(T'); two
 * accesses to the same item conflict iff at least one writes (Z2).
 * Plain per-item scan of all earlier accesses: O(sum over items of count^2). */
int orc_gputx_ranks(uint32_t n_txn, uint32_t K, const uint32_t *keys, const uint8_t *ops,
                    uint64_t n_items, uint32_t *rank_out) {
    uint64_t n_acc = (uint64_t)n_txn * K;
    int64_t *head = (int64_t *)malloc(sizeof(int64_t) * (n_items ? n_items : 1));
    int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (n_acc ? n_acc : 1));
    if (!head || !next) { free(head); free(next); return ORC_ERR_OOM; }
    for (uint64_t i = 0; i < n_items; i++) head[i] = -1;
    for (uint32_t t = 0; t < n_txn; t++) {
        uint32_t r = 0;
        for (uint32_t i = 0; i < K; i++) {
            uint64_t a = (uint64_t)t * K + i;
            uint64_t item = keys[a];
            if (item >= n_items) { free(head); free(next); return ORC_ERR_KEY; }
            int w = (ops[a] & 0x80u) != 0;
            for (int64_t b = head[item]; b >= 0; b = next[b]) {
                int wb = (ops[b] & 0x80u) != 0;
                if (w || wb) {
                    uint32_t cand = rank_out[b / K] + 1u;
                    if (cand > r) r = cand;
                }
            }
        }
        rank_out[t] = r;
        for (uint32_t i = 0; i < K; i++) { /* publish t's accesses after computing rank */
            uint64_t a = (uint64_t)t * K + i;
            next[a] = head[keys[a]];
            head[keys[a]] = (int64_t)a;
        }
    }
    free(head); free(next);
    return ORC_OK;
}

/* GaccO lock-table queue position of each access:
 * pos(t, i) = number of accesses to item keys[t*K+i] by transactions with id < t. */
int orc_gacco_positions(uint32_t n_txn, uint32_t K, const uint32_t *keys, uint64_t n_items,
                        uint32_t *pos_out) {
    uint32_t *cnt = (uint32_t *)calloc(n_items ? n_items : 1, sizeof(uint32_t));
    if (!cnt) return ORC_ERR_OOM;
    for (uint64_t a = 0; a < (uint64_t)n_txn * K; a++) {
        if (keys[a] >= n_items) { free(cnt); return ORC_ERR_KEY; }
        pos_out[a] = cnt[keys[a]]++;
    }
    free(cnt);
    return ORC_OK;
}
