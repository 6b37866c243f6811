// exec.cuh -- the persistent transaction executor and the
// eight CC schemes, generic over a workload policy WL.
//
// Execution model (B200 design):
//  * one persistent grid at resident capacity; every working lane (2^wd per warp,
//    PAPER.md:480) claims transactions in increasing id from a device ticket, so
//    every transaction anyone waits on is already running on a resident lane (H1);
//  * an aborted attempt releases its CC state, bumps restarts[gid] and appends gid to
//    a device retry ring with a warp-aggregated atomic (a6), from which lanes claim
//    again after the fresh ids are exhausted; CC_FLAG_IMMEDIATE_RETRY restores the
//    paper's "the thread immediately restarts";
//  * each committing attempt emits its serialization-order key.
//
// WL must provide: MAXK, Txn {gid, n, wmask, rec[]}, Ws, load(), row(), read_op(),
// install(), copy_row(), emit(), ROW_WORDS.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "internal.h"

namespace gcctb {
namespace cg = cooperative_groups;

enum { RES_OK = 0, RES_ABORT = 1, RES_FATAL = 2 };

// ------------------------------------------------------------------ thread context
struct Th {
    u64 deadline;
    const ExecParams *p;
};

GC_DEV void set_err(Ctl *c, u64 code) { atomicCAS(&c->err, 0ull, code); }

GC_DEV bool dead(Th &th) {
    if (ld_relaxed(&th.p->ctl->err) != 0) return true;
    if (globaltimer_ns() > th.deadline) {
        set_err(th.p->ctl, CC_ERR_WATCHDOG);
        return true;
    }
    return false;
}

struct Spin {
    unsigned ns = 20;
    GC_DEV bool wait(Th &th) {   // false -> give up (error / watchdog)
        __nanosleep(ns);
        ns = ns < 320 ? ns + ns / 2 + 8 : 320;
        return !dead(th);
    }
};

// warp-aggregated fetch-add over the currently converged lanes
GC_DEV u64 agg_fetch_add(u64 *ctr) {
    cg::coalesced_group g = cg::coalesced_threads();
    u64 base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(ctr, (u64)g.size());
    base = g.shfl(base, 0);
    return base + g.thread_rank();
}
GC_DEV void agg_add(u64 *ctr) {
    cg::coalesced_group g = cg::coalesced_threads();
    if (g.thread_rank() == 0) atom_add_acqrel(ctr, (u64)g.size());
}

// ------------------------------------------------------------------ 2PL (Table II)
// word = [62] shared | [61:31] holder count | [30:0] holder (wait-die: min age of the
// holders, Z7; age = gid + 1).  0 = free.
constexpr u64 TPL_S = 1ull << 62;
constexpr u64 M31 = 0x7FFFFFFFull;
GC_DEV u32 tpl_cnt(u64 v) { return (u32)((v >> 31) & M31); }
GC_DEV u32 tpl_holder(u64 v) { return (u32)(v & M31); }
GC_DEV u64 tpl_make(bool s, u64 cnt, u64 holder) {
    return (s ? TPL_S : 0ull) | ((cnt & M31) << 31) | (holder & M31);
}

template <bool WD>
GC_DEV int tpl_acquire(u64 *w, bool ex, u32 age, Th &th) {
    u64 v = ld_relaxed(w);
    Spin sp;
    for (;;) {
        u64 nv;
        bool conflict;
        if (ex) {
            conflict = (v != 0);
            nv = tpl_make(false, 1, age);
        } else {
            conflict = (v != 0) && !(v & TPL_S);
            nv = (v == 0) ? tpl_make(true, 1, age)
                          : tpl_make(true, tpl_cnt(v) + 1, min(age, tpl_holder(v)));
        }
        if (conflict) {
            // no-wait: abort at once.  wait-die: an older requester
            // (smaller age) waits, a younger one dies.
            if (!WD || !(age < tpl_holder(v))) return RES_ABORT;
            if (!sp.wait(th)) return RES_FATAL;
            v = ld_relaxed(w);
            continue;
        }
        u64 old = cas_acqrel(w, v, nv);
        if (old == v) return RES_OK;
        v = old;
    }
}

GC_DEV void tpl_release(u64 *w, bool ex) {
    if (ex) {
        st_release(w, 0ull);
        return;
    }
    u64 v = ld_relaxed(w);
    for (;;) {
        u64 nv = (tpl_cnt(v) <= 1) ? 0ull : v - (1ull << 31);
        u64 old = cas_acqrel(w, v, nv);
        if (old == v) return;
        v = old;
    }
}

template <bool WD, class WL>
GC_DEV int run_tpl(Th &th, typename WL::Txn &t, typename WL::Ws &ws, const typename WL::Params &y) {
    const ExecParams &p = *th.p;
    const u32 age = t.gid + 1;
    int i = 0, r = RES_OK;
    for (; i < (int)t.n; i++) {
        const bool ex = (t.wmask >> i) & 1;
        r = tpl_acquire<WD>(&p.meta[t.rec[i]], ex, age, th);
        if (r != RES_OK) break;
        WL::read_op(y, t, i, WL::row(y, t.rec[i]), ws);  // row is stable under the lock
    }
    if (r != RES_OK) {
        for (int j = 0; j < i; j++) tpl_release(&p.meta[t.rec[j]], (t.wmask >> j) & 1);
        return r;
    }
    // lock point: every lock held, none released -> ticket is a valid serial order (strict 2PL)
    const u64 ticket = agg_fetch_add(&p.ctl->ticket);
    for (int j = 0; j < (int)t.n; j++)
        if ((t.wmask >> j) & 1) WL::install(y, t, j, WL::row(y, t.rec[j]), ws);
    for (int j = 0; j < (int)t.n; j++) tpl_release(&p.meta[t.rec[j]], (t.wmask >> j) & 1);
    t.key_hi = 0;
    t.key_lo = ticket;
    return RES_OK;
}

// ------------------------------------------------------------------ TO (Table II)
// word = [62] pending (uncommitted write) | [61:31] RTS | [30:0] WTS.
// While pending, WTS holds the pending writer's ts (the writer keeps the committed
// word to restore on abort).  Reading rules follow PAPER.md:188 with reading Z4.
constexpr u64 TO_P = 1ull << 62;
GC_DEV u64 to_rts(u64 v) { return (v >> 31) & M31; }
GC_DEV u64 to_wts(u64 v) { return v & M31; }
GC_DEV u64 to_make(bool pend, u64 rts, u64 wts) {
    return (pend ? TO_P : 0ull) | ((rts & M31) << 31) | (wts & M31);
}

GC_DEV bool draw_ts(Th &th, u64 &ts) {
    ts = agg_fetch_add(&th.p->ctl->ts) + 1;   // a fresh timestamp per attempt
    if (ts > M31) {                            // 31-bit field
        set_err(th.p->ctl, CC_ERR_TS_OVERFLOW);
        return false;
    }
    return true;
}

template <class WL>
GC_DEV int run_to(Th &th, typename WL::Txn &t, typename WL::Ws &ws, const typename WL::Params &y) {
    const ExecParams &p = *th.p;
    u64 ts;
    if (!draw_ts(th, ts)) return RES_FATAL;
    u64 saved[WL::MAXK];
    u32 pend = 0;
    int r = RES_OK;
    for (int i = 0; i < (int)t.n && r == RES_OK; i++) {
        u64 *w = &p.meta[t.rec[i]];
        const u64 *row = WL::row(y, t.rec[i]);
        Spin sp;
        if ((t.wmask >> i) & 1) {
            // write (read-modify-write): ts must be newer than RTS and WTS
            u64 v = ld_acquire(w);
            for (;;) {
                if (v & TO_P) {
                    if (to_wts(v) < ts) {   // older pending writer: wait for it (Z4)
                        if (!sp.wait(th)) { r = RES_FATAL; break; }
                        v = ld_acquire(w);
                        continue;
                    }
                    r = RES_ABORT;
                    break;
                }
                if (ts < to_rts(v) || ts < to_wts(v)) { r = RES_ABORT; break; }
                u64 old = cas_acqrel(w, v, to_make(true, to_rts(v), ts));
                if (old == v) break;
                v = old;
            }
            if (r != RES_OK) break;
            saved[i] = v;
            pend |= 1u << i;
            WL::read_op(y, t, i, row, ws);     // stable: we own the pending bit
        } else {
            // read: ts must be newer than WTS; wait on an older pending writer; then read
            // the row between two loads of the word and raise RTS with a CAS
            for (;;) {
                u64 v = ld_acquire(w);
                if (ts < to_wts(v)) { r = RES_ABORT; break; }
                if (v & TO_P) {
                    if (!sp.wait(th)) { r = RES_FATAL; break; }
                    continue;
                }
                WL::read_op(y, t, i, row, ws);
                fence_acqrel();
                if (to_rts(v) >= ts) {
                    if (ld_relaxed(w) == v) break;
                    continue;
                }
                if (cas_acqrel(w, v, to_make(false, ts, to_wts(v))) == v) break;
            }
        }
    }
    if (r != RES_OK) {
        for (int j = 0; j < (int)t.n; j++)
            if ((pend >> j) & 1) st_release(&p.meta[t.rec[j]], saved[j]);
        return r;
    }
    for (int j = 0; j < (int)t.n; j++)
        if ((pend >> j) & 1) {
            WL::install(y, t, j, WL::row(y, t.rec[j]), ws);
            st_release(&p.meta[t.rec[j]], to_make(false, ts, ts));
        }
    t.key_hi = 0;
    t.key_lo = ts;
    return RES_OK;
}

// ------------------------------------------------------------------ MVCC (Table II)
// meta[2r]   lo = TO word (pending | RTS | WTS); while pending WTS = pending writer ts
// meta[2r+1] hi = version pointer word: [63:32] begin ts of the in-place head version,
//                 [31:0] arena index of the previous version (NONE = 0xFFFFFFFF).
// History nodes (arena, one per write op of the batch):
//   word0 = (begin << 32) | prev, word1 = 0, words 2.. = row content (immutable once
//   published).  Writes are buffered and installed at commit (Z6).
constexpr u64 VNONE = 0xFFFFFFFFull;

template <class WL>
GC_DEV int run_mvcc(Th &th, typename WL::Txn &t, typename WL::Ws &ws, const typename WL::Params &y) {
    const ExecParams &p = *th.p;
    u64 ts;
    if (!draw_ts(th, ts)) return RES_FATAL;
    u64 saved_wts[WL::MAXK];
    u32 pend = 0;
    int r = RES_OK;
    for (int i = 0; i < (int)t.n && r == RES_OK; i++) {
        u64 *lo = &p.meta[2ull * t.rec[i]];
        u64 *hi = lo + 1;
        const u64 *row = WL::row(y, t.rec[i]);
        Spin sp;
        if ((t.wmask >> i) & 1) {
            // writes append only at the head: ts > head WTS and ts >= RTS (Z6)
            u64 v = ld_acquire(lo);
            for (;;) {
                if (v & TO_P) {
                    if (to_wts(v) < ts) {
                        if (!sp.wait(th)) { r = RES_FATAL; break; }
                        v = ld_acquire(lo);
                        continue;
                    }
                    r = RES_ABORT;
                    break;
                }
                if (ts < to_rts(v) || ts < to_wts(v)) { r = RES_ABORT; break; }
                u64 old = cas_acqrel(lo, v, to_make(true, to_rts(v), ts));
                if (old == v) break;
                v = old;
            }
            if (r != RES_OK) break;
            saved_wts[i] = to_wts(v);
            pend |= 1u << i;
            WL::read_op(y, t, i, row, ws);
        } else {
            // read the version whose interval holds ts; never aborts
            for (;;) {
                u64 v = ld_acquire(lo);
                if ((v & TO_P) && to_wts(v) < ts) {   // older pending writer: its version is ours
                    if (!sp.wait(th)) { r = RES_FATAL; break; }
                    continue;
                }
                u64 h = ld_acquire(hi);
                if ((h >> 32) <= ts) {   // head visible: read in place, validate, raise RTS
                    WL::read_op(y, t, i, row, ws);
                    fence_acqrel();
                    if (ld_relaxed(hi) != h) continue;
                    if (to_rts(v) >= ts) {
                        if (ld_relaxed(lo) == v) break;
                        continue;
                    }
                    u64 nv = (v & ~(M31 << 31)) | ((ts & M31) << 31);
                    if (cas_acqrel(lo, v, nv) == v) break;
                    continue;
                }
                // walk the history chain for the newest version with begin <= ts
                u64 idx = h & VNONE;
                bool found = false;
                while (idx != VNONE) {
                    const u64 *node = p.arena + idx * (2 + WL::ROW_WORDS);
                    u64 h0 = ld_cg(node);
                    if ((h0 >> 32) <= ts) {
                        WL::read_op(y, t, i, node + 2, ws);
                        found = true;
                        break;
                    }
                    idx = h0 & VNONE;
                }
                if (!found) {
                    set_err(p.ctl, CC_ERR_VERSION_EXHAUSTED);
                    r = RES_FATAL;
                }
                break;
            }
        }
    }
    if (r != RES_OK) {
        for (int j = 0; j < (int)t.n; j++)
            if ((pend >> j) & 1) {   // restore the committed word, keeping raised RTS
                u64 *lo = &p.meta[2ull * t.rec[j]];
                u64 v = ld_relaxed(lo);
                for (;;) {
                    u64 old = cas_acqrel(lo, v, to_make(false, to_rts(v), saved_wts[j]));
                    if (old == v) break;
                    v = old;
                }
            }
        return r;
    }
    for (int j = 0; j < (int)t.n; j++)
        if ((pend >> j) & 1) {
            u64 *lo = &p.meta[2ull * t.rec[j]];
            u64 *hi = lo + 1;
            u64 *row = WL::row(y, t.rec[j]);
            const u64 nidx = (u64)t.gid * p.K + j;
            u64 *node = p.arena + nidx * (2 + WL::ROW_WORDS);
            const u64 h = ld_relaxed(hi);
            st_cg(node, ((h >> 32) << 32) | (h & VNONE));   // old head -> history node
            WL::copy_row(row, node + 2);
            fence_acqrel();
            st_release(hi, (ts << 32) | nidx);                // publish, then install
            fence_acqrel();
            WL::install(y, t, j, row, ws);
            st_release(lo, to_make(false, ts, ts));
        }
    t.key_hi = 0;
    t.key_lo = ts;
    return RES_OK;
}

// ------------------------------------------------------------------ Silo (Table II)
// word = [63] lock | [62:0] TID.  Read phase snapshots (word, row, word); commit locks
// the write set no-wait, draws the serialization-point ticket,
// validates the read set, installs with TID = 1 + max observed (epoch dropped,
// PAPER.md:416; Z8).
constexpr u64 LOCKB = 1ull << 63;

template <class WL>
GC_DEV bool occ_read_phase(Th &th, typename WL::Txn &t, typename WL::Ws &ws,
                           const typename WL::Params &y, u64 *obs) {
    const ExecParams &p = *th.p;
    for (int i = 0; i < (int)t.n; i++) {
        u64 *w = &p.meta[t.rec[i]];
        const u64 *row = WL::row(y, t.rec[i]);
        Spin sp;
        for (;;) {
            u64 v1 = ld_acquire(w);
            if (v1 & LOCKB) {   // a committer holds it: wait (Z10)
                if (!sp.wait(th)) return false;
                continue;
            }
            WL::read_op(y, t, i, row, ws);
            fence_acqrel();
            if (ld_relaxed(w) == v1) {
                obs[i] = v1;
                break;
            }
        }
    }
    return true;
}

template <class WL>
GC_DEV int occ_lock_writes(Th &th, typename WL::Txn &t, u64 *pre, u32 &locked) {
    const ExecParams &p = *th.p;
    locked = 0;
    for (int i = 0; i < (int)t.n; i++) {
        if (!((t.wmask >> i) & 1)) continue;
        u64 *w = &p.meta[t.rec[i]];
        u64 v = ld_relaxed(w);
        for (;;) {
            if (v & LOCKB) return RES_ABORT;   // no-wait in the write phase
            u64 old = cas_acqrel(w, v, v | LOCKB);
            if (old == v) break;
            v = old;
        }
        pre[i] = v;
        locked |= 1u << i;
    }
    return RES_OK;
}

template <class WL>
GC_DEV void occ_unlock(const ExecParams &p, typename WL::Txn &t, const u64 *pre, u32 locked) {
    for (int j = 0; j < (int)t.n; j++)
        if ((locked >> j) & 1) st_release(&p.meta[t.rec[j]], pre[j]);
}

template <class WL>
GC_DEV int run_silo(Th &th, typename WL::Txn &t, typename WL::Ws &ws, const typename WL::Params &y) {
    const ExecParams &p = *th.p;
    u64 obs[WL::MAXK], pre[WL::MAXK];
    if (!occ_read_phase<WL>(th, t, ws, y, obs)) return RES_FATAL;
    u32 locked;
    if (occ_lock_writes<WL>(th, t, pre, locked) != RES_OK) {
        occ_unlock<WL>(p, t, pre, locked);
        return RES_ABORT;
    }
    const u64 ticket = agg_fetch_add(&p.ctl->ticket);   // serialization point
    fence_acqrel();
    u64 tid = 0;
    for (int i = 0; i < (int)t.n; i++) {
        const bool wr = (t.wmask >> i) & 1;
        const u64 cur = wr ? pre[i] : ld_acquire(&p.meta[t.rec[i]]);
        if (cur != obs[i]) {   // TID changed, or locked by another transaction
            occ_unlock<WL>(p, t, pre, locked);
            return RES_ABORT;
        }
        tid = max(tid, obs[i]);
    }
    tid = (tid + 1) & ~LOCKB;
    for (int j = 0; j < (int)t.n; j++)
        if ((t.wmask >> j) & 1) {
            WL::install(y, t, j, WL::row(y, t.rec[j]), ws);
            st_release(&p.meta[t.rec[j]], tid);
        }
    t.key_hi = 0;
    t.key_lo = ticket;
    return RES_OK;
}

// ------------------------------------------------------------------ TicToc (Table II)
// word = [63] lock | [62:48] delta | [47:0] WTS, RTS = WTS + delta.
constexpr u64 M48 = (1ull << 48) - 1;
constexpr u64 DMAX = 0x7FFFull;
GC_DEV u64 tt_wts(u64 v) { return v & M48; }
GC_DEV u64 tt_rts(u64 v) { return (v & M48) + ((v >> 48) & DMAX); }

template <class WL>
GC_DEV int run_tictoc(Th &th, typename WL::Txn &t, typename WL::Ws &ws, const typename WL::Params &y) {
    const ExecParams &p = *th.p;
    u64 obs[WL::MAXK], pre[WL::MAXK];
    if (!occ_read_phase<WL>(th, t, ws, y, obs)) return RES_FATAL;
    u32 locked;
    if (occ_lock_writes<WL>(th, t, pre, locked) != RES_OK) {
        occ_unlock<WL>(p, t, pre, locked);
        return RES_ABORT;
    }
    // commit_ts = max(max over writes of RTS+1, max over reads of WTS)
    u64 cts = 0;
    for (int i = 0; i < (int)t.n; i++) {
        if ((t.wmask >> i) & 1) cts = max(cts, tt_rts(pre[i]) + 1);
        cts = max(cts, tt_wts(obs[i]));
    }
    for (int i = 0; i < (int)t.n; i++) {
        if ((t.wmask >> i) & 1) {
            if (tt_wts(pre[i]) != tt_wts(obs[i])) {
                occ_unlock<WL>(p, t, pre, locked);
                return RES_ABORT;
            }
            continue;
        }
        if (tt_rts(obs[i]) >= cts) continue;   // version valid through cts already
        u64 *w = &p.meta[t.rec[i]];
        u64 v = ld_acquire(w);
        for (;;) {
            if (tt_wts(v) != tt_wts(obs[i]) || (v & LOCKB)) {
                occ_unlock<WL>(p, t, pre, locked);
                return RES_ABORT;
            }
            if (tt_rts(v) >= cts) break;
            u64 nw = tt_wts(v);
            if (cts - nw > DMAX) nw = cts - DMAX;   // delta overflow: shift WTS up (Z9)
            u64 old = cas_acqrel(w, v, ((cts - nw) << 48) | nw);
            if (old == v) break;
            v = old;
        }
    }
    const u64 ticket = agg_fetch_add(&p.ctl->ticket);   // after validation, before install
    for (int j = 0; j < (int)t.n; j++)
        if ((t.wmask >> j) & 1) {
            WL::install(y, t, j, WL::row(y, t.rec[j]), ws);
            st_release(&p.meta[t.rec[j]], cts & M48);
        }
    t.key_hi = cts;
    t.key_lo = ticket;
    return RES_OK;
}

// ------------------------------------------------------------------ GaccO
// Every access waits until the item's cursor reaches its preprocessed queue position,
// performs the access, then advances the cursor (release after the op, Z3).
template <class WL>
GC_DEV int run_gacco(Th &th, typename WL::Txn &t, typename WL::Ws &ws, const typename WL::Params &y) {
    const ExecParams &p = *th.p;
    const u64 base = (u64)t.gid * p.K;
    for (int i = 0; i < (int)t.n; i++) {
        const u32 seg = p.acc_seg[base + i], pos = p.acc_pos[base + i];
        u32 *cur = &p.cursor[seg];
        Spin sp;
        while (ld_acquire32(cur) != pos)
            if (!sp.wait(th)) return RES_FATAL;
        u64 *row = WL::row(y, t.rec[i]);
        WL::read_op(y, t, i, row, ws);
        if ((t.wmask >> i) & 1) WL::install(y, t, i, row, ws);
        st_release32(cur, pos + 1);
    }
    t.key_hi = 0;
    t.key_lo = t.gid;
    return RES_OK;
}

// ------------------------------------------------------------------ GPUTx
// K-set k runs once every transaction of K-set k-1 has completed; inside a K-set there
// is no concurrency control.
template <class WL>
GC_DEV int run_gputx(Th &th, typename WL::Txn &t, typename WL::Ws &ws, const typename WL::Params &y) {
    const ExecParams &p = *th.p;
    const u32 k = p.rank_of[t.gid];
    if (k > 0) {
        Spin sp;
        while (ld_acquire32(&p.rank_done[k - 1]) < p.rank_count[k - 1])
            if (!sp.wait(th)) return RES_FATAL;
    }
    for (int i = 0; i < (int)t.n; i++) {
        u64 *row = WL::row(y, t.rec[i]);
        WL::read_op(y, t, i, row, ws);
        if ((t.wmask >> i) & 1) WL::install(y, t, i, row, ws);
    }
    atom_add_release32(&p.rank_done[k], 1u);
    t.key_hi = 0;
    t.key_lo = t.gid;
    return RES_OK;
}

template <int S, class WL>
GC_DEV int run_scheme(Th &th, typename WL::Txn &t, typename WL::Ws &ws, const typename WL::Params &y) {
    if constexpr (S == CC_TPL_NW) return run_tpl<false, WL>(th, t, ws, y);
    else if constexpr (S == CC_TPL_WD) return run_tpl<true, WL>(th, t, ws, y);
    else if constexpr (S == CC_TO) return run_to<WL>(th, t, ws, y);
    else if constexpr (S == CC_MVCC) return run_mvcc<WL>(th, t, ws, y);
    else if constexpr (S == CC_SILO) return run_silo<WL>(th, t, ws, y);
    else if constexpr (S == CC_TICTOC) return run_tictoc<WL>(th, t, ws, y);
    else if constexpr (S == CC_GACCO) return run_gacco<WL>(th, t, ws, y);
    else return run_gputx<WL>(th, t, ws, y);
}

// ------------------------------------------------------------------ retry ring (a6)
// Bounded MPMC ring of (seq << 32 | gid) slots; slot k of the retry sequence lives at
// ring[k & (cap-1)], its consumer clears it after reading.
GC_DEV void ring_push(Th &th, u32 gid) {
    const ExecParams &p = *th.p;
    const u64 r = agg_fetch_add(&p.ctl->tail);
    u64 *slot = p.ring + (r & (p.ring_cap - 1));
    Spin sp;
    while (ld_relaxed(slot) != 0)   // previous lap not consumed yet
        if (!sp.wait(th)) return;
    st_release(slot, (((r + 1) & 0xFFFFFFFFull) << 32) | gid);
}

GC_DEV bool ring_take(Th &th, u64 k, u32 &gid) {
    const ExecParams &p = *th.p;
    u64 *slot = p.ring + (k & (p.ring_cap - 1));
    const u64 want = (k + 1) & 0xFFFFFFFFull;
    Spin sp;
    for (;;) {
        const u64 v = ld_acquire(slot);
        if ((v >> 32) == want) {
            gid = (u32)v;
            st_relaxed(slot, 0ull);
            return true;
        }
        if (ld_acquire(&p.ctl->done) >= p.n_txn) return false;
        if (!sp.wait(th)) return false;
    }
}

// Randomised, bounded exponential backoff after an abort.  Lanes of one warp run in
// lockstep, so two transactions with crossed read/write sets can otherwise lock,
// fail each other's validation and retry in perfect symmetry forever (an OCC livelock
// the paper's immediate restart, is exposed to as well).  Delay is
// uniform in [0, min(64 ns << restarts, 16 us)) from a hash of (gid, restarts).
GC_DEV void abort_backoff(u32 gid, u32 restarts) {
    const u32 sh = restarts < 8 ? restarts : 8;
    const u32 cap = 64u << sh;
    u32 d = (u32)(mix64(((u64)gid << 32) | restarts) % cap);
    while (d > 0) {
        const u32 s = d < 1000u ? d : 1000u;
        __nanosleep(s);
        d -= s;
    }
}

// ------------------------------------------------------------------ the kernel
template <int S, class WL>
__global__ void __launch_bounds__(1024) exec_kernel(ExecParams p, typename WL::Params y) {
    const u32 lane = threadIdx.x & 31u;
    if (lane >= (1u << p.wd)) return;   // idle lanes exit at once
    constexpr bool DET = (S == CC_GPUTX || S == CC_GACCO);
    Th th;
    th.p = &p;
    th.deadline = globaltimer_ns() + p.watchdog_ns;
    typename WL::Txn t;
    typename WL::Ws ws;
    for (;;) {
        if (dead(th)) return;
        const u64 s = agg_fetch_add(&p.ctl->head);
        u32 gid;
        if (s < p.n_txn) {
            gid = (S == CC_GPUTX) ? p.rank_order[s] : (u32)s;
        } else {
            if (DET || (p.flags & CC_FLAG_IMMEDIATE_RETRY)) return;
            if (!ring_take(th, s - p.n_txn, gid)) return;
        }
        if (!WL::load(p, y, gid, t)) {
            set_err(p.ctl, CC_ERR_KEY_NOT_FOUND);
            return;
        }
        for (;;) {
            const int r = run_scheme<S, WL>(th, t, ws, y);
            if (r == RES_OK) {
                WL::emit(p, y, t, ws);
                p.order_hi[gid] = t.key_hi;
                p.order_lo[gid] = t.key_lo;
                p.committed[gid] = 1;
                agg_add(&p.ctl->done);
                break;
            }
            if (r == RES_FATAL) return;
            const u32 nr = p.restarts[gid] + 1;   // single owner of gid at a time
            p.restarts[gid] = nr;
            agg_add(&p.ctl->aborts);
            abort_backoff(gid, nr);
            if (p.flags & CC_FLAG_IMMEDIATE_RETRY) continue;
            ring_push(th, gid);
            break;
        }
    }
}

}  // namespace gcctb
