// exec.cuh -- the persistent transaction executor and the
// eight CC schemes, generic over a workload policy WL.
//
// Two execution modes share the queue and the control-word protocols:
//  * thread mode (lanes = 1): one lane per transaction, 2^wd working lanes per warp,
//    bs warps per block -- the paper's launch model;
//  * tile mode (lanes = G in {4,8,16,32}): a tile of G lanes runs one transaction,
//    lane i owns access i.  Index lookups, CC words and rows of all accesses are issued
//    in parallel; commit / abort / wait decisions are tile ballots (vote.any/all), the
//    warp-level structure the north star asks for.  Same protocols, same order keys.
//
// Queue (a6): round 1 claims fresh ids in increasing order from a device ticket; an
// abort while fresh ids remain releases the CC state, bumps restarts[gid], backs off
// and compacts gid into the retry batch; round 2 drains that batch once it is sealed;
// aborts after that retry in place.  Every transaction a worker waits
// on has a smaller id or is held by a running worker, so nothing waits on an
// unscheduled block.
#pragma once
#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>

#include "common.cuh"
#include "internal.h"

// Executor launch bounds: one 1024-thread block per SM by default (64 registers, no
// spills); the build can trade registers for resident transactions with
// -DGC_EXEC_MAXT=512 -DGC_EXEC_MINB=3 (40 registers, 1536 threads per SM).
#ifndef GC_EXEC_MAXT
#define GC_EXEC_MAXT 1024
#endif
#ifndef GC_EXEC_MINB
#define GC_EXEC_MINB 1
#endif

namespace gcctb {
namespace cg = cooperative_groups;

enum { RES_OK = 0, RES_ABORT = 1, RES_FATAL = 2 };
constexpr u32 NO_TXN = 0xFFFFFFFFu;

// ------------------------------------------------------------------ thread context
// claim state of a worker (queue, a6); lives in its shared-memory context
struct Claim {
    bool exhausted = false;
    bool sealed = false;
    bool fresh = false;      // the last id returned was a fresh one (restarts = 0)
    u64 tail = 0;
    u64 next = 0, end = 0;   // fresh ids claimed ahead (chunked claims), processed in order
};

struct Th {
    u64 deadline;
    const ExecParams *p;
    u32 gid, attempt;     // current attempt (event log)
    u32 polls;
    bool timing;          // CC_FLAG_STAGES
    u64 *st;              // this worker's STAGE_WORDS accumulators (global memory), or null
    u64 *cw;   // lock word whose holder caused the last abort (nullptr: none)
    u64 cv;    // wait until (*cw & cv) == 0: the conflicting lock is free
    u32 hot;   // tile mode: 1 + lane of the lock that caused this transaction's last abort
    u64 *turn; // GC_RETRY_FIFO: the retry queue whose turn this worker holds (nullptr: none)
    bool cw_ex;   // the access that died on *cw wanted it exclusively (a write)
    u64 *tq;      // TO / MVCC: control word of the write whose timestamp check killed the attempt
    u64 a_t0, a_u0, a_w0, a_s0;   // CC_FLAG_STAGES: the current attempt's start snapshot
    Claim cl;                     // the worker's claim state (leader lane in tile mode)
};

GC_DEV void set_err(Ctl *c, u64 code) { atomicCAS(&c->err.v, 0ull, code); }

// control word of a record (single-word schemes): packed 8 B SoA words, or with
// CC_FLAG_META_PAD one word per 32 B sector (f-3; the north star's metadata "padded to
// avoid false sharing in L2"), a per-submit choice (ExecParams in shared memory keeps the
// runtime stride off the register budget).  MVCC: mvcc_lo / _hi.
GC_DEV u64 *cw(const ExecParams &p, u32 rec) {
    // re-read at every use (volatile): a stride held in a register across the transaction
    // loop made four tile kernels spill; the shared-memory load is ~30 cycles
    return p.meta + ((u64)rec << *reinterpret_cast<const volatile uint32_t *>(&p.meta_shift));
}

GC_DEV bool dead(Th &th) {
    if (globaltimer_ns() > th.deadline) {
        set_err(th.p->ctl, CC_ERR_WATCHDOG);
        return true;
    }
    if ((++th.polls & 15u) == 0 && ld_relaxed(&th.p->ctl->err.v) != 0) return true;
    return false;
}

struct Spin {
    unsigned ns = 16;
    unsigned cap = 256;   // max sleep between polls (ns)
    GC_DEV Spin() {}
    GC_DEV explicit Spin(unsigned max_ns) : ns(max_ns < 16 ? max_ns : 16), cap(max_ns) {}
    GC_DEV bool wait(Th &th) {   // false -> give up (error / watchdog)
        const u64 t0 = th.timing ? clk64() : 0;
        __nanosleep(ns);
        ns = ns < cap ? ns * 2 : cap;
        const bool alive = !dead(th);
        if (th.timing) th.st[STAGE_WAIT] += clk64() - t0;
        return alive;
    }
};

// stage timer: adds the elapsed cycles of its scope to one accumulator
struct StageClock {
    Th &th;
    int k;
    u64 t0;
    GC_DEV StageClock(Th &t, int stage) : th(t), k(stage), t0(t.timing ? clk64() : 0) {}
    GC_DEV ~StageClock() {
        if (th.timing) th.st[k] += clk64() - t0;
    }
};

// debug event log (CC_FLAG_EVENTS): each event takes a global sequence
// number right after the access it describes
GC_DEV u64 log_event(const Th &th, u32 rec, u32 kind) {
    const ExecParams &p = *th.p;
    if (!p.events) return ~0ull;
    const u64 k = atomicAdd(&p.ctl->events.v, 1ull);
    if (k >= p.events_cap) return ~0ull;   // overflow: the count tells the host
    Event &ev = p.events[k];
    ev.seq = k;
    ev.gid = th.gid;
    ev.rec = rec;
    ev.attempt = th.attempt;
    ev.kind = kind;
    return k;
}

// A read whose re-check failed (seqlock / RTS CAS lost) is repeated in the same attempt:
// its logged event did not happen logically, so it becomes kind 4 (retracted).
GC_DEV void retract_read(const Th &th, u64 k) {
    if (k != ~0ull) th.p->events[k].kind = 4u;
}

// row work (the "useful" stage) done through these wrappers
template <class WL>
GC_DEV u64 rd(Th &th, const typename WL::Params &y, typename WL::Lane &L, u32 gid, u32 i, const u64 *src) {
    {
        StageClock c(th, STAGE_USEFUL);
        WL::read(y, L, gid, i, src);
    }
    if (th.p->events) {
        fence_acqrel();
        return log_event(th, L.rec, 0);   // before the caller's re-check of the word
    }
    return ~0ull;
}
template <class WL>
GC_DEV void inst(Th &th, const typename WL::Params &y, const typename WL::Lane &L, u64 *dst) {
    {
        StageClock c(th, STAGE_USEFUL);
        WL::install(y, L, dst);
    }
    if (th.p->events) {
        fence_acqrel();
        log_event(th, L.rec, 1);
    }
}

// per-attempt attribution: a committed attempt's time not spent in row
// work, waits or timestamp allocation is CC-manager time; an aborted attempt's whole time
// minus its timestamp allocation is abort time (its row work and waits included).
// (the snapshot lives in the worker's shared-memory context, not in registers held across
// the attempt)
struct AttemptClock {
    Th &th;
    GC_DEV explicit AttemptClock(Th &t) : th(t) {
        if (t.timing) {
            t.a_t0 = clk64();
            t.a_u0 = t.st[STAGE_USEFUL];
            t.a_w0 = t.st[STAGE_WAIT];
            t.a_s0 = t.st[STAGE_TS];
        }
    }
    GC_DEV void done(bool committed) {
        if (!th.timing) return;
        const u64 el = clk64() - th.a_t0;
        const u64 du = th.st[STAGE_USEFUL] - th.a_u0, dw = th.st[STAGE_WAIT] - th.a_w0, ds = th.st[STAGE_TS] - th.a_s0;
        th.st[STAGE_ATTEMPTS] += 1;
        if (committed) {
            th.st[STAGE_CC] += el > du + dw + ds ? el - du - dw - ds : 0;
        } else {
            th.st[STAGE_USEFUL] = th.a_u0;
            th.st[STAGE_WAIT] = th.a_w0;
            th.st[STAGE_ABORT] += el > ds ? el - ds : 0;
        }
    }
};

GC_DEV void stages_init(Th &th, const ExecParams &p, bool on) {
    th.timing = p.stages != nullptr && on;
    th.st = nullptr;
    if (th.timing) {   // per-thread slot, reduced by stages_reduce after the kernel
        const u64 tid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
        th.st = p.stages + STAGE_WORDS + tid * STAGE_WORDS;
        for (int k = 0; k < STAGE_WORDS; k++) th.st[k] = 0;
    }
}

// warp-aggregated fetch-add over the currently converged lanes
GC_DEV u64 agg_fetch_add(u64 *ctr) {
    cg::coalesced_group g = cg::coalesced_threads();
    u64 base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(ctr, (u64)g.size());
    base = g.shfl(base, 0);
    return base + g.thread_rank();
}

// ------------------------------------------------------------------ control-word ops
// Latch-free by default: every read-transform-update of a control word is one 64-bit
// CAS.  With CC_FLAG_LATCHED (Exp-7) every
// mutation of a control word happens under a 32-bit per-word latch instead (acquire
// spin, read, compare, write, release); reads stay plain loads.
GC_DEV void latch_acquire(uint32_t *l) {
    unsigned ns = 8;
    for (;;) {
        uint32_t old;
        asm volatile("atom.acquire.gpu.global.cas.b32 %0, [%1], 0, 1;" : "=r"(old) : "l"(l) : "memory");
        if (old == 0) return;
        __nanosleep(ns);
        ns = ns < 128 ? ns * 2 : 128;
    }
}
GC_DEV void latch_release(uint32_t *l) { st_release32(l, 0u); }
GC_DEV uint32_t *latch_of(const ExecParams &p, const u64 *w) {
    return p.latch + (p.scheme == CC_MVCC ? (w - p.meta) : (w - p.meta) >> p.meta_shift);
}

GC_DEV u64 w_cas(const ExecParams &p, u64 *w, u64 expect, u64 desired) {
    if (!p.latch) return cas_acqrel(w, expect, desired);
    uint32_t *l = latch_of(p, w);
    latch_acquire(l);
    const u64 old = ld_relaxed(w);
    if (old == expect) st_relaxed(w, desired);
    latch_release(l);
    return old;
}
// CAS that acquires a lock / pending bit: acquire ordering suffices (see cas_acquire)
GC_DEV u64 w_cas_acq(const ExecParams &p, u64 *w, u64 expect, u64 desired) {
    if (!p.latch) return cas_acquire(w, expect, desired);
    uint32_t *l = latch_of(p, w);
    latch_acquire(l);
    const u64 old = ld_relaxed(w);
    if (old == expect) st_relaxed(w, desired);
    latch_release(l);
    return old;
}
GC_DEV void w_store(const ExecParams &p, u64 *w, u64 v) {   // release store
    if (!p.latch) { st_release(w, v); return; }
    uint32_t *l = latch_of(p, w);
    latch_acquire(l);
    st_relaxed(w, v);
    latch_release(l);
}
GC_DEV void w_store_relaxed(const ExecParams &p, u64 *w, u64 v) {   // after an explicit fence
    if (!p.latch) { st_relaxed(w, v); return; }
    w_store(p, w, v);
}
GC_DEV void w_add(const ExecParams &p, u64 *w, u64 v) {
    if (!p.latch) { atom_add_relaxed(w, v); return; }
    uint32_t *l = latch_of(p, w);
    latch_acquire(l);
    st_relaxed(w, ld_relaxed(w) + v);
    latch_release(l);
}

// Randomised, bounded exponential backoff after an abort that no single lock explains
// (validation failures, timestamp conflicts).  Lanes of one warp run in lockstep, so
// two transactions with crossed read/write sets can otherwise lock, fail each other's
// validation and retry in perfect symmetry forever (an OCC livelock the paper's
// immediate restart, is exposed to as well).  Delay is uniform in
// [0, 64 ns << min(restarts, cap)) from a hash of (gid, restarts); cap = 10 (~65 us)
// keeps batch tails short.  Timestamp schemes adapt the cap to the number of
// transactions backing off at that moment: 10 while few do (a moderately contended
// batch: a fixed 1 ms cap made single stragglers sleep the batch long, TO at theta=0.6
// 46-72 M vs 103-109 M txn/s), 12 from LO, 14 (~1 ms) from 4*LO (LO = 1,024 for TO, 256
// for MVCC, which aborts less) -- basic TO under a read-hot key otherwise retries in a
// storm that burns 31-bit timestamps (cap 10 at theta=0.8: 1.4 M vs 4.9 M).
// profiles/r01_probe_v6..v11, v18.
#ifndef GC_BACKOFF_CAP
#define GC_BACKOFF_CAP 10u   // lock / OCC schemes: 64 ns << 10 = 65 us
#endif
// Timestamp schemes, lowest tier: while fewer than GC_BACKOFF_LO transactions back off (the
// tail of a moderately contended batch), the cap drops to GC_BACKOFF_LO_CAP (~8 us).
// YCSB configs[1] theta=0.6: MVCC 112 -> 120, TO 108 -> 113 M txn/s; TPC-C 64 warehouses
// TO 15.5 -> 19.4 M; theta=0.8 and 1 warehouse unchanged.  For the lock / OCC schemes the
// same tier was neutral to -6 % (profiles/r01_pacing_v42/), so they keep the fixed cap.
#ifndef GC_BACKOFF_LO
#define GC_BACKOFF_LO 32
#endif
#ifndef GC_BACKOFF_LO_CAP
#define GC_BACKOFF_LO_CAP 7u
#endif
template <int S>
GC_DEV void abort_backoff(const ExecParams &p, u32 gid, u32 restarts) {
    constexpr bool TS = S == CC_TO || S == CC_MVCC;
    u32 CAP = GC_BACKOFF_CAP;
    u64 n = 0;
    if (TS) n = atomicAdd(&p.ctl->pacing.v, 1ull);   // transactions backing off now
    if (TS) {
        constexpr u64 LO = S == CC_TO ? 1024 : 256;   // MVCC aborts less: fewer back off at once
        CAP = p.to_backoff_cap ? p.to_backoff_cap : (n < LO ? 10u : (n < 4 * LO ? 12u : 14u));
    }
    if (TS && GC_BACKOFF_LO > 0 && !p.to_backoff_cap && n < (u64)GC_BACKOFF_LO) CAP = GC_BACKOFF_LO_CAP;
    const u32 sh = restarts < CAP ? restarts : CAP;
    const u32 cap = 64u << sh;
    u32 d = (u32)(mix64(((u64)gid << 32) | restarts) % cap);
    while (d > 0) {
        const u32 s = d < 1000u ? d : 1000u;
        __nanosleep(s);
        d -= s;
    }
    if (TS) atomicAdd(&p.ctl->pacing.v, (u64)-1ll);
}

// Waits on a hand-off chain (GaccO turn, GPUTx K-set gate) poll with ld.acquire and need
// no fence after the wait: the fence.acq_rel that used to follow relaxed polls cost ~0.3 us
// per hop (ring microbenchmark 1.48 -> 1.17 us; GaccO configs[1] theta 0.6 1.28 ->
// 1.04 ms, theta 0.8 19.1 -> 15.3 ms; profiles/r01_gacco_poll.txt).  GC_GACCO_SPIN caps
// the sleep between polls.
#ifndef GC_GACCO_SPIN
#define GC_GACCO_SPIN 32
#endif
// A GaccO access knows its queue position and reads the item's cursor, so it knows how
// many hand-offs (>= ~1.2 us each, measured) are still ahead of it: far waiters sleep in
// proportion to that distance with relaxed polls, and only the next in line polls with
// acquire loads.  Hundreds of waiters polling one hot cursor at full rate otherwise
// saturate its L2 slice and slow the very hand-offs they wait for.
#ifndef GC_GACCO_HOP_NS
#define GC_GACCO_HOP_NS 600
#endif
#ifndef GC_GACCO_MAX_SLEEP_NS
#define GC_GACCO_MAX_SLEEP_NS 50000u
#endif
// Wait until the item's cursor has reached `target` (the cursor only grows, one hand-off at
// a time; it never passes our own position before we release it).
GC_DEV bool gacco_reach(Th &th, u32 *cur, u32 target) {
    u32 c = ld_acquire32(cur);
    if ((int)(target - c) <= 0) return true;
    const u64 t0 = th.timing ? clk64() : 0;
    bool ok = true;
    while ((int)(target - c) > 1) {
        const u32 d = target - c - 1;
        const u32 ns = d * GC_GACCO_HOP_NS;
        __nanosleep(ns < GC_GACCO_MAX_SLEEP_NS ? ns : GC_GACCO_MAX_SLEEP_NS);
        if (dead(th)) { ok = false; break; }
        c = ld_relaxed32(cur);
    }
    if (th.timing) th.st[STAGE_WAIT] += clk64() - t0;
    if (!ok) return false;
    Spin sp(GC_GACCO_SPIN);
    while ((int)(target - ld_acquire32(cur)) > 0)   // the poll that sees it is the acquire
        if (!sp.wait(th)) return false;
    return true;
}

// One GaccO access: it owns the item from its turn (cursor == pos) until it
// advances the cursor.  Its row read is hoisted to the moment the item's last earlier write
// has installed (cursor >= rdy, acc_rdy from a3): only reads sit between that write and
// this access, so the row then already holds what the access reads at its turn.  The turn,
// the install and the hand-off stay in queue order; what leaves the hand-off chain's
// critical path is the row read (an L2 round trip per hop on a read-hot item).
// GC_GACCO_HOIST=0 reads at the turn (ablation).
#ifndef GC_GACCO_HOIST
#define GC_GACCO_HOIST 1
#endif
template <class WL>
GC_DEV bool gacco_access(Th &th, const typename WL::Params &y, typename WL::Lane &L, u32 gid, u32 i,
                         u32 *cur, u32 pos, u32 rdy) {
    u64 *row = WL::row(y, L);
    if (GC_GACCO_HOIST) {
        if (!gacco_reach(th, cur, rdy)) return false;
        rd<WL>(th, y, L, gid, i, row);
        if (!gacco_reach(th, cur, pos)) return false;
    } else {
        if (!gacco_reach(th, cur, pos)) return false;
        rd<WL>(th, y, L, gid, i, row);
    }
    if (L.w) inst<WL>(th, y, L, row);
#if defined(GC_EXP_GACCO_RELAXED_READ) && GC_EXP_GACCO_RELAXED_READ
    // timing ablation only: a read's hand-off without release semantics (the PTX model
    // does not order the row load before a relaxed store; never shipped)
    if (!L.w) { st_relaxed32(cur, pos + 1); return true; }
#endif
    st_release32(cur, pos + 1);
    return true;
}

// GPUTx K-set gate: wait until K-set k-1 has completed.  K-sets complete
// in order and ctl->kdone counts them (set by each set's last finisher), so a waiter knows
// how far the frontier is: the next set polls tightly, sets further ahead sleep about as
// long as the K-sets in between take (~1.5 us each at least, the measured hand-off).
// Thousands of waiters polling the one kdone word at sub-microsecond periods saturated
// its L2 slice, which also serves the rank_done counters of the frontier.
#ifndef GC_KSET_MAX_SLEEP_NS
#define GC_KSET_MAX_SLEEP_NS 50000u
#endif
#ifndef GC_KSET_TIGHT_DIST
#define GC_KSET_TIGHT_DIST 1   // distances polled tightly (kdone lags the last finisher by a round trip)
#endif
GC_DEV unsigned kset_sleep_ns(u64 dist) {
    if (dist <= GC_KSET_TIGHT_DIST) return 32u;
    const u64 ns = 1500ull * (dist - GC_KSET_TIGHT_DIST);
    return ns < GC_KSET_MAX_SLEEP_NS ? (unsigned)ns : GC_KSET_MAX_SLEEP_NS;
}
// wait until K-set k-1 is the frontier (every earlier K-set complete)
GC_DEV bool kset_near(Th &th, const ExecParams &p, u32 k) {
    const u64 t0 = th.timing ? clk64() : 0;
    bool ok = true;
    for (;;) {
        const u64 done = ld_relaxed(&p.ctl->kdone.v);
        if (done + 1 >= k) break;
        __nanosleep(kset_sleep_ns(k - done));
        if (dead(th)) { ok = false; break; }
    }
    if (th.timing) th.st[STAGE_WAIT] += clk64() - t0;
    return ok;
}
// GC_KSET_KDONE=1: the gate polls ctl->kdone, which only each K-set's last finisher
// writes (one release store after its acq_rel count increment, which reads from every
// earlier finisher's release increment), instead of the K-set's counter rank_done[k-1]:
// with the counter polled, a K-set's few hundred waiters loaded the very word its
// finishers were incrementing.  Measured slower (configs[1] bench launch, theta 0.6: 1.47 ->
// 1.54 ms per submit, theta 0.8: 15.8 -> 16.6 ms; profiles/r02_probe_kset_kdone.log): the
// finisher's extra store is on the chain.  0 (default): poll the counter.
#ifndef GC_KSET_KDONE
#define GC_KSET_KDONE 0
#endif
GC_DEV bool kset_wait(Th &th, const ExecParams &p, u32 k) {
    const u64 t0 = th.timing ? clk64() : 0;
    bool ok = true;
    // acquire polls: the one that sees K-set k-1 complete orders its installs before our
    // accesses (no fence after the wait)
    if (GC_KSET_KDONE) {
        u64 done;
        while ((done = ld_acquire(&p.ctl->kdone.v)) < k) {
            __nanosleep(kset_sleep_ns(k - done));
            if (dead(th)) { ok = false; break; }
        }
    } else {
        while (ld_acquire32(&p.rank_done[k - 1]) < p.rank_count[k - 1]) {
            const u64 done = ld_relaxed(&p.ctl->kdone.v);
            __nanosleep(kset_sleep_ns(k > done ? k - done : 1));
            if (dead(th)) { ok = false; break; }
        }
    }
    if (th.timing) th.st[STAGE_WAIT] += clk64() - t0;
    return ok;
}
// Experiment builds (-DGC_TRACE_COMMIT=1, tools/trace_kset.py): trace[2050 + k] = when
// K-set k completed, trace[4098 + k] = when the first member of K-set k passed its gate.
GC_DEV void kset_trace(const ExecParams &p, u32 k, int what) {
#if defined(GC_TRACE_COMMIT) && GC_TRACE_COMMIT
    if (!p.trace || k >= 2048) return;
    const u64 t = globaltimer_ns();
    if (what == 0) p.trace[2050 + k] = t;
    else atomicMin(&p.trace[4098 + k], t);
#endif
}
#ifndef GC_GPUTX_EARLY
#define GC_GPUTX_EARLY 1
#endif
GC_DEV void kset_done(const ExecParams &p, u32 k) {
    if (GC_KSET_KDONE) {
        const u32 old = atom_add_acqrel32(&p.rank_done[k], 1u);
        if (old + 1 == p.rank_count[k]) st_release(&p.ctl->kdone.v, (u64)k + 1);   // K-sets finish in order
    } else {
        const u32 old = atom_add_release32(&p.rank_done[k], 1u);
        if (old + 1 == p.rank_count[k]) {
            atomicMax(&p.ctl->kdone.v, (u64)k + 1);
            kset_trace(p, k, 0);
        }
    }
}

// Retry pacing after an abort.  If a held lock caused it, wait -- holding nothing, so
// no-wait / OCC semantics are unchanged -- until that lock is free (2PL holder count 0,
// OCC lock bit clear), bounded, add a little jitter, and retry; otherwise use the
// randomised backoff.  This replaces a blind sleep (during which the lock is often
// already free) by one L2 round trip, without turning a busy shared lock into a storm.
#ifndef GC_JITTER_MAX_SHIFT
#define GC_JITTER_MAX_SHIFT 11   // post-wait jitter window cap: 32 ns << 11 = 65 us
#endif
// Adaptive cap: while fewer than GC_JITTER_LO transactions are pacing after a lock wait,
// the window stops growing at 32 ns << GC_JITTER_LO_SHIFT (~8 us; 0: static cap only).
// A moderately contended batch ends in a tail of a few hot-record retriers whose 65 us
// windows left the lock idle; a herd (theta >= 0.8, one TPC-C warehouse) keeps the wide
// windows.  YCSB configs[1] theta=0.6, tuned launch: tpl_nw 107 -> 123, tpl_wd 126 ->
// 142 M txn/s; theta=0.8 and TPC-C at 1 / 64 warehouses unchanged; a static 8 us cap
// instead cost wait-die 40 % at theta=0.8 (profiles/r01_pacing_v39_v40/).
#ifndef GC_JITTER_LO
#define GC_JITTER_LO 32
#endif
#ifndef GC_JITTER_LO_SHIFT
#define GC_JITTER_LO_SHIFT 8
#endif
// Retry queues (GC_RETRY_FIFO): an exclusive request killed by a held lock (2PL writes, the
// OCC lock phase) takes a ticket in the FIFO of that lock's control word (hashed, GC_RQ_N queues) and
// waits -- holding nothing, so no-wait / wait-die / OCC semantics are unchanged -- for its
// turn, then for the lock to be free, and retries at once, in place; the turn passes on
// when that attempt ends, committed or not.  The random jitter that keeps a herd of
// retriers from colliding in lockstep is replaced by an order, so a hot lock's retriers
// hand it on one after another instead of leaving it idle for a jitter window.  (Readers
// keep the jitter: queued one at a time they lost the sharing -- YCSB theta 0.6 wait-die
// 141 -> 73 M txn/s, profiles/r02_probe_fifo_v1.log.)
#ifndef GC_RETRY_FIFO
#define GC_RETRY_FIFO 1
#endif
// Queue only while at least this many transactions pace after a lock wait (a herd); below
// it the jitter stays (measured, configs[1] tile 16, profiles/r02_probe_fifo_v5_herd.log:
// queueing from 64 pacers cost 2PL 10-25 % at theta 0.6-0.8, from 1024 it is neutral there
// and 2-8x faster at theta 0.99; Silo / TicToc gain from 64 at theta >= 0.8 and are neutral
// at 0.6).  The 2PL threshold is per workload (ExecParams::rq_herd_2pl, set by the host):
// TPC-C, whose warehouse / district rows are hot for every transaction, gains from 256
// (one warehouse +10 %, 64 warehouses +7-11 %, profiles/r02_probe_tpcc_herd2pl.log) where
// YCSB at theta 0.6 loses 21 %.
#ifndef GC_RQ_HERD_2PL
#define GC_RQ_HERD_2PL 2048
#endif
#ifndef GC_RQ_HERD_OCC
#define GC_RQ_HERD_OCC 64
#endif
#ifndef GC_RQ_TURN_NS
#define GC_RQ_TURN_NS 1500u   // sleep per turn ahead (about one attempt on a hot lock)
#endif
GC_DEV u64 *rq_of(const ExecParams &p, const u64 *w) {
    const u64 h = ((u64)(uintptr_t)w >> 3) * 0x9E3779B97F4A7C15ull;
    return p.rq + (h >> 48);   // GC_RQ_N = 2^16
}
GC_DEV void rq_release(Th &th) {
    if (th.turn) {
        atomicAdd(th.turn, 1ull << 32);
        th.turn = nullptr;
    }
}
// take a ticket in the queue of control word w and wait for the turn (holding nothing)
GC_DEV void rq_wait(Th &th, const u64 *w) {
    u64 *q = rq_of(*th.p, w);
    const u64 old = atomicAdd(q, 1ull);
    const u32 t = (u32)old;
    u32 sv = (u32)(old >> 32);
    while (sv != t) {   // far waiters sleep in proportion to the turns ahead,
        const u32 d = t - sv;   // the next in line polls
        const u32 ns = d > 30u ? 50000u : (d - 1) * GC_RQ_TURN_NS;
        __nanosleep(ns < 64u ? 64u : ns);
        if (dead(th)) break;
        sv = (u32)(ld_relaxed(q) >> 32);
    }
    th.turn = q;
}
// TO / MVCC (ablation, GC_TS_FIFO): a write killed by its timestamp check queues the same
// way once at least GC_RQ_HERD_TS transactions back off (instead of the randomised
// exponential backoff, whose window reaches ~1 ms in a herd).  Measured (tile 16,
// profiles/r02_probe_ts_fifo.log): TO unchanged (theta 0.99 0.27 M txn/s either way: its
// aborts are read-timestamp conflicts, not a queue); MVCC theta 0.99 0.91 -> 1.24 but theta
// 0.8 13.0 -> 9.0.  Off.
#ifndef GC_TS_FIFO
#define GC_TS_FIFO 0
#endif
#ifndef GC_RQ_HERD_TS
#define GC_RQ_HERD_TS 1024
#endif
// wait (holding nothing) until the lock that killed the attempt is free, bounded
GC_DEV void wait_lock_free(Th &th, u32 restarts) {
    const u32 sh = restarts < 10 ? restarts : 10;
    const u64 limit = globaltimer_ns() + (64ull << sh) + 1000ull;
    unsigned ns = 32;
    while ((ld_relaxed(th.cw) & th.cv) != 0 && globaltimer_ns() < limit) {
        __nanosleep(ns);
        ns = ns < 256 ? ns * 2 : 256;
    }
}
template <int S>
GC_DEV void retry_pace(Th &th, u32 gid, u32 restarts) {
    if (th.cw) {
        // how many transactions pace after a lock wait right now (this one included)
        const u64 n = (GC_JITTER_LO > 0 || GC_RETRY_FIFO) ? atomicAdd(&th.p->ctl->pacing_lk.v, 1ull) : 0ull;
        const bool flat = (th.p->flags & CC_FLAG_FLAT_JITTER) != 0;
        u64 HERD = (S == CC_TPL_NW || S == CC_TPL_WD)
                       ? (th.p->rq_herd_2pl ? (u64)th.p->rq_herd_2pl : (u64)GC_RQ_HERD_2PL)
                       : (u64)GC_RQ_HERD_OCC;
        if (HERD > (u64)(th.p->n_txn >> 3)) HERD = th.p->n_txn >> 3;   // small batches: an eighth pacing is a herd
        if (GC_RETRY_FIFO && th.cw_ex && n >= HERD && !flat) {   // a herd: queue
            rq_wait(th, th.cw);   // held through the next attempt (in place), released after it
            wait_lock_free(th, restarts);
        } else {
            const u32 jcap = (GC_JITTER_LO > 0 && n < (u64)GC_JITTER_LO) ? (u32)GC_JITTER_LO_SHIFT
                                                                         : (u32)GC_JITTER_MAX_SHIFT;
            wait_lock_free(th, restarts);
            // then a random delay whose window doubles per restart: waiters released by
            // the same unlock must not retry in lockstep (a herd livelock at theta >= 0.9)
            const u32 win = flat ? 256u : 32u << (restarts < jcap ? restarts : jcap);
            u32 d = (u32)(mix64(((u64)gid << 32) | restarts) % win);
            while (d > 0) {
                const u32 s = d < 1000u ? d : 1000u;
                __nanosleep(s);
                d -= s;
            }
        }
        if (GC_JITTER_LO > 0 || GC_RETRY_FIFO) atomicAdd(&th.p->ctl->pacing_lk.v, (u64)-1ll);
        th.cw = nullptr;
        return;
    }
    if ((S == CC_TO || S == CC_MVCC) && GC_TS_FIFO && th.tq) {
        const u64 *w = th.tq;
        th.tq = nullptr;
        if (ld_relaxed(&th.p->ctl->pacing.v) >= (u64)GC_RQ_HERD_TS) {   // a herd: queue
            atomicAdd(&th.p->ctl->pacing.v, 1ull);
            rq_wait(th, w);
            atomicAdd(&th.p->ctl->pacing.v, (u64)-1ll);
            return;
        }
    }
    abort_backoff<S>(*th.p, gid, restarts);
}

// ------------------------------------------------------------------ queue (a6)
// Round 1 is the fresh batch, claimed in increasing id.  While fresh ids remain, an
// aborted transaction is compacted into the retry batch (`ring`): the converged workers
// of a warp that append at the same moment take their slots with ONE atomicAdd on the
// ring's tail word (ballot/popc through a coalesced group, the leader adds the group size
// and shuffles the base back), then each writes its entry with a release store.  Each id
// is appended at most once before the fresh ids run out, so n_txn slots always suffice.
// The tail word carries a seal bit: the first worker that finds the fresh ids exhausted
// sets it with one atomicOr, whose return value is the exact number of appends that won
// a slot; it publishes that size (rtail = size + 1).  An append whose atomicAdd returns a
// sealed word was refused and retries in place; round 2 consumes the sealed batch with
// one atomicAdd per claim, waiting on an entry only in the rare case that its appender
// has reserved the slot but not yet written it.  Aborts after exhaustion retry in place
// after their backoff.  Workers exit when both rounds are drained.
constexpr u64 RING_SEALED = 1ull << 63;    // tail word: seal bit | number of reserved slots
constexpr u64 RING_VALID = 1ull << 63;     // ring entry: written | hot lane << 32 | gid

GC_DEV bool try_append_retry(Th &th, u32 gid) {
    const ExecParams &p = *th.p;
    Ctl *c = p.ctl;
    // exhaustion is monotone: after it nothing is appended (and the seal follows)
    if (ld_relaxed(&c->head.v) >= p.n_txn) return false;
    cg::coalesced_group g = cg::coalesced_threads();
    u64 old = 0;
    if (g.thread_rank() == 0) old = atomicAdd(&c->tail.v, (u64)g.size());   // one atomic per group
    old = g.shfl(old, 0);
    if (old & RING_SEALED) return false;   // refused: the batch was sealed first
    const u64 r = old + g.thread_rank();
    // release: restarts[gid] (and everything this attempt released) precede the entry
    st_release(p.ring + r, RING_VALID | ((u64)th.hot << 32) | gid);
    return true;
}


// Claim work for one worker: a fresh id, else a retry-batch entry, else NO_TXN.
template <int S>
GC_DEV u32 claim_work(Th &th, Claim &cl) {
    const ExecParams &p = *th.p;
    Ctl *c = p.ctl;
    constexpr bool DET = (S == CC_GPUTX || S == CC_GACCO);
    if (!cl.exhausted) {
        // chunked claims: one atomic per `claim_chunk` ids; ids stay increasing per worker
        // and across workers' chunks, so every waited-on transaction is already claimed
        if (cl.next >= cl.end) {
            cl.next = atomicAdd(&c->head.v, (u64)p.claim_chunk);
            cl.end = cl.next + p.claim_chunk;
        }
        const u64 s = cl.next++;
        th.hot = 0;
        cl.fresh = true;
        if (s < p.n_txn) return (S == CC_GPUTX) ? p.rank_order[s] : (u32)s;
        cl.exhausted = true;
    }
    cl.fresh = false;
    if (DET || (p.flags & CC_FLAG_IMMEDIATE_RETRY)) return NO_TXN;
    if (!cl.sealed) {
        u64 t = ld_relaxed(&c->rtail.v);
        if (t == 0) {
            const u64 old = atomicOr(&c->tail.v, RING_SEALED);
            if (!(old & RING_SEALED)) {   // this worker sealed: the size is exact
                t = old + 1;
                st_relaxed(&c->rtail.v, t);
            } else {
                Spin sp;
                while ((t = ld_relaxed(&c->rtail.v)) == 0)
                    if (!sp.wait(th)) return NO_TXN;
            }
        }
        cl.tail = t - 1;
        cl.sealed = true;
    }
    if (cl.tail == 0 || ld_relaxed(&c->rhead.v) >= cl.tail) return NO_TXN;
    const u64 r = atomicAdd(&c->rhead.v, 1ull);
    if (r >= cl.tail) return NO_TXN;
    u64 e = ld_acquire(p.ring + r);   // pairs with the appender's release store
    if (!(e & RING_VALID)) {          // reserved before the seal, not yet written
        Spin sp(64);
        while (!((e = ld_acquire(p.ring + r)) & RING_VALID))
            if (!sp.wait(th)) return NO_TXN;
    }
    th.hot = (u32)(e >> 32) & 0x7FFFFFFFu;
    return (u32)e;
}

// ------------------------------------------------------------------ 2PL (Table II)
// word = [63] writer intent (wait-die) | [62] shared | [61:31] holder count | [30:0]
// holder (wait-die: min age of the holders, Z7; age = gid + 1).  Free <=> count == 0
// (shared releases are a single atomic subtract and may leave stale bits behind; any
// acquisition of a free word rewrites all of them).
// Writer intent: an exclusive requester that waits on a shared-held lock sets it, and so
// does a starving one that dies there (TPL_INTENT_AFTER restarts); while it is set a new shared requester counts as conflicting
// (wait-die decides), so the lock drains.  Without it a hot read-mostly lock never drains:
// its recorded min holder age can belong to a long-gone older reader (shared releases do
// not rewrite it), so even the oldest writer compares itself against that stale age, dies
// instead of waiting, and starves (tile mode, YCSB theta=0.9: watchdog).
constexpr u64 TPL_WW = 1ull << 63;
constexpr u64 TPL_S = 1ull << 62;
constexpr u64 M31 = 0x7FFFFFFFull;
constexpr u64 TPL_ONE = 1ull << 31;
GC_DEV u32 tpl_cnt(u64 v) { return (u32)((v >> 31) & M31); }
GC_DEV u32 tpl_holder(u64 v) { return (u32)(v & M31); }
GC_DEV u64 tpl_make(bool s, u64 cnt, u64 holder) {
    return (s ? TPL_S : 0ull) | ((cnt & M31) << 31) | (holder & M31);
}

// One acquisition step.  Returns 0 granted, 1 wait (wait-die older requester, or the
// CAS lost a race), 2 die (conflict under no-wait, or younger requester).
// Tile-mode TO: restarts after which a transaction's accesses are stepped one lane at a
// time (measured, profiles/r01_probe_v16_*: 8 halves TO at theta=0.6, 32 keeps it; the
// same for wait-die cost 4.7x at theta=0.8 and was dropped)
#ifndef GC_TO_SEQ_AFTER
#define GC_TO_SEQ_AFTER 32
#endif
constexpr u32 TO_SEQ_AFTER = GC_TO_SEQ_AFTER;
// Restarts from which tile-mode TO steps one lane at a time while at least 1,024
// transactions back off (a herd; 0: off).  configs[1], M txn/s (profiles/
// r02_probe_to_seq_herd.log): theta 0.99 0.27 -> 0.33 (the paper's thread launch: 0.30),
// theta 0.9 0.93 -> 0.90, theta 0.6 unchanged; from 2 restarts: 0.35 / 0.79.
#ifndef GC_TO_SEQ_HERD
#define GC_TO_SEQ_HERD 6
#endif

// A waiting writer always announces intent (TPL_WW); a dying one only once it has restarted
// this often -- the stale-age starvation needs it, and announcing earlier makes readers die
// needlessly (measured, YCSB tile 16: every writer at once: theta 0.6 96M -> 53M txn/s;
// dying writers after 8 restarts: theta 0.8 6.1M -> 1.9M).
constexpr u32 TPL_INTENT_AFTER = 32;
// no-wait writer intent (ablation): a writer that has died this often on a shared-held
// lock announces itself too, and new readers then die on the announced lock so it drains
// (0: off -- readers never conflict with an announcement under no-wait).  Measured slower
// (configs[1] tile 16, exec ms: theta 0.6 0.51 -> 0.54 / 0.64 from 8 / 2 restarts, theta 0.8
// 5.9 -> 7.1 / 9.1; profiles/r02_probe_nw_intent.log).
#ifndef GC_NW_INTENT_AFTER
#define GC_NW_INTENT_AFTER 0
#endif
#ifndef GC_WD_SEQ_AFTER
#define GC_WD_SEQ_AFTER 0
#endif

template <bool WD>
GC_DEV bool tpl_intent(u32 attempt) {
    return WD ? attempt >= TPL_INTENT_AFTER : (GC_NW_INTENT_AFTER > 0 && attempt >= (u32)GC_NW_INTENT_AFTER);
}
template <bool WD>
GC_DEV int tpl_try(const ExecParams &p, u64 *w, bool ex, u32 age, u64 &seen, bool intent) {
    u64 v = ld_relaxed(w);
    for (;;) {   // latch-free read-transform-CAS loop
        const u32 cnt = tpl_cnt(v);
        bool conflict;
        u64 nv;
        if (ex) {
            conflict = cnt != 0;
            nv = tpl_make(false, 1, age);
        } else {
            conflict = cnt != 0 && (!(v & TPL_S) || ((WD || GC_NW_INTENT_AFTER > 0) && (v & TPL_WW)));
            nv = cnt == 0 ? tpl_make(true, 1, age) : tpl_make(true, cnt + 1, min(age, tpl_holder(v)));
        }
        if (conflict) {
            // no-wait: abort at once.  wait-die: an older requester
            // (smaller age) waits, a younger one dies.
            seen = v;
            const bool wait = WD && age < tpl_holder(v);
            if ((WD ? (wait || intent) : intent) && ex && (v & TPL_S) && !(v & TPL_WW)) {   // writer intent (TPL_WW)
                const u64 old = w_cas_acq(p, w, v, v | TPL_WW);
                if (old != v) { v = old; continue; }
            }
            return wait ? 1 : 2;
        }
        const u64 old = w_cas_acq(p, w, v, nv);
        if (old == v) return 0;
        v = old;
    }
}

GC_DEV void tpl_release_relaxed(const ExecParams &p, u64 *w, bool ex) {
    if (ex) w_store_relaxed(p, w, 0ull);
    else w_add(p, w, (u64)(-(long long)TPL_ONE));
}

// ------------------------------------------------------------------ TO (Table II)
// word = [62] pending (uncommitted write) | [61:31] RTS | [30:0] WTS.  While pending,
// WTS holds the pending writer's ts (the writer keeps the committed word to restore
// on abort).  Reading rules follow PAPER.md:188 with reading Z4.
constexpr u64 TO_P = 1ull << 62;
GC_DEV u64 to_rts(u64 v) { return (v >> 31) & M31; }
GC_DEV u64 to_wts(u64 v) { return v & M31; }
GC_DEV u64 to_make(bool pend, u64 rts, u64 wts) {
    return (pend ? TO_P : 0ull) | ((rts & M31) << 31) | (wts & M31);
}

// ------------------------------------------------------------------ MVCC (Table II)
// meta[2r]   lo = TO word (pending | RTS | WTS); while pending WTS = pending writer ts
// meta[2r+1] hi = version pointer word: [63:32] begin ts of the in-place head version,
//                 [31:0] 1 + arena index of the previous version (0: none), so the
//                 initial state of every scheme's words is all zeros.
// History nodes (one per write op of the batch): word0 = the hi word
// of the version they replaced ((begin << 32) | prev), word1 = 0, then the row content.
constexpr u64 VIDX = 0xFFFFFFFFull;   // hi / node word: 1 + previous node index, 0 = none

// ------------------------------------------------------------------ OCC (Table II)
constexpr u64 LOCKB = 1ull << 63;    // Silo: [63] lock | [62:0] TID
constexpr u64 M48 = (1ull << 48) - 1; // TicToc: [63] lock | [62:48] delta | [47:0] WTS
constexpr u64 DMAX = 0x7FFFull;
GC_DEV u64 tt_wts(u64 v) { return v & M48; }
GC_DEV u64 tt_rts(u64 v) { return (v & M48) + ((v >> 48) & DMAX); }

// Per-access step outcomes used by both modes
enum { ST_DONE = 0, ST_WAIT = 1, ST_ABORT = 2, ST_RETRY = 3 };   // RETRY: lost a CAS race, go again at once

// TO access step for one item (write = read-modify-write).  On success for a write the
// row is read under the pending bit; for a read it is read between two word loads.
template <class WL>
GC_DEV int to_step(Th &th, const ExecParams &p, const typename WL::Params &y, typename WL::Lane &L,
                   u32 gid, u32 i, u64 ts, bool &pend, u64 &saved) {
    u64 *w = cw(p, L.rec);
    const u64 *row = WL::row(y, L);
    const u64 v = ld_acquire(w);
    if (L.w) {
        if (v & TO_P) return to_wts(v) < ts ? ST_WAIT : ST_ABORT;   // older pending: wait (Z4)
        if (ts < to_rts(v) || ts < to_wts(v)) return ST_ABORT;
        if (w_cas_acq(p, w, v, to_make(true, to_rts(v), ts)) != v) return ST_RETRY;
        pend = true;
        saved = v;
        rd<WL>(th, y, L, gid, i, row);   // stable: we own the pending bit
        return ST_DONE;
    }
    if (ts < to_wts(v)) return ST_ABORT;
    if (v & TO_P) return ST_WAIT;
    const u64 ev = rd<WL>(th, y, L, gid, i, row);
    fence_acqrel();
    const bool ok = (to_rts(v) >= ts) ? ld_relaxed(w) == v : w_cas_acq(p, w, v, to_make(false, ts, to_wts(v))) == v;   // after the fence above
    if (ok) return ST_DONE;
    retract_read(th, ev);
    return ST_RETRY;
}

template <class WL>
GC_DEV void to_commit(Th &th, const ExecParams &p, const typename WL::Params &y, typename WL::Lane &L, u64 ts) {
    // the pending bit was taken with an acquire-only CAS: a release fence orders it before
    // the installs, so an optimistic reader that sees new row bytes also sees the bit
    fence_acqrel();
    inst<WL>(th, y, L, WL::row(y, L));
    fence_acqrel();
    w_store_relaxed(p, cw(p, L.rec), to_make(false, ts, ts));
}

// MVCC access step (Z6): writes append at the head only; reads never abort.
// MVCC word pair of a record: interleaved (lo, hi), Table II's 16 B, or split arrays
// (CC_FLAG_MVCC_SPLIT: lo words as dense as TO's; the PAPER.md:636 ablation)
GC_DEV u64 *mvcc_lo(const ExecParams &p, u32 rec) { return p.mvcc_split ? p.meta + rec : p.meta + 2ull * rec; }
GC_DEV u64 *mvcc_hi(const ExecParams &p, u32 rec) {
    return p.mvcc_split ? p.meta + p.mvcc_split + rec : p.meta + 2ull * rec + 1;
}

template <class WL>
GC_DEV int mvcc_step(Th &th, const ExecParams &p, const typename WL::Params &y, typename WL::Lane &L,
                     u32 gid, u32 i, u64 ts, bool &pend, u64 &saved_wts) {
    u64 *lo = mvcc_lo(p, L.rec);
    u64 *hi = mvcc_hi(p, L.rec);
    const u64 *row = WL::row(y, L);
    const u64 v = ld_acquire(lo);
    if (L.w) {
        if (v & TO_P) return to_wts(v) < ts ? ST_WAIT : ST_ABORT;
        if (ts < to_rts(v) || ts < to_wts(v)) return ST_ABORT;
        if (w_cas_acq(p, lo, v, to_make(true, to_rts(v), ts)) != v) return ST_RETRY;
        pend = true;
        saved_wts = to_wts(v);
        rd<WL>(th, y, L, gid, i, row);
        return ST_DONE;
    }
    if ((v & TO_P) && to_wts(v) < ts) return ST_WAIT;   // older pending writer: its version is ours
    const u64 h = ld_acquire(hi);
    if ((h >> 32) <= ts) {   // head visible: read in place, validate, raise RTS
        const u64 ev = rd<WL>(th, y, L, gid, i, row);
        fence_acqrel();
        bool ok = ld_relaxed(hi) == h;
        if (ok) {
            if (to_rts(v) >= ts) ok = ld_relaxed(lo) == v;
            else ok = w_cas_acq(p, lo, v, (v & ~(M31 << 31)) | ((ts & M31) << 31)) == v;   // after the fence
        }
        if (ok) return ST_DONE;
        retract_read(th, ev);
        return ST_RETRY;
    }
    // walk the history chain for the newest version with begin <= ts
    u64 idx = h & VIDX;
    while (idx != 0) {
        const u64 *node = p.arena + (idx - 1) * (ARENA_HDR + WL::ROW_WORDS);
        const u64 h0 = ld_cg(node);
        if ((h0 >> 32) <= ts) {
            rd<WL>(th, y, L, gid, i, node + ARENA_HDR);
            return ST_DONE;
        }
        idx = h0 & VIDX;
    }
    set_err(p.ctl, CC_ERR_VERSION_EXHAUSTED);
    return ST_ABORT;
}

template <class WL>
GC_DEV void mvcc_restore(const ExecParams &p, typename WL::Lane &L, u64 saved_wts) {
    u64 *lo = mvcc_lo(p, L.rec);
    u64 v = ld_relaxed(lo);
    for (;;) {   // keep RTS raised by readers while we were pending
        const u64 old = w_cas(p, lo, v, to_make(false, to_rts(v), saved_wts));
        if (old == v) return;
        v = old;
    }
}

template <class WL>
GC_DEV void mvcc_commit(Th &th, const ExecParams &p, const typename WL::Params &y, typename WL::Lane &L,
                        u32 gid, u32 i, u64 ts) {
    u64 *lo = mvcc_lo(p, L.rec);
    u64 *hi = mvcc_hi(p, L.rec);
    u64 *row = WL::row(y, L);
    const u64 nidx = (u64)gid * p.K + i;
    u64 *node = p.arena + nidx * (ARENA_HDR + WL::ROW_WORDS);
    st_cg(node, ld_relaxed(hi));   // old head -> history node (begin, prev)
    WL::copy_row(L, row, node + ARENA_HDR);
    fence_acqrel();
    w_store(p, hi, (ts << 32) | (nidx + 1));   // publish the history, then install in place
    fence_acqrel();
    inst<WL>(th, y, L, row);
    fence_acqrel();
    w_store_relaxed(p, lo, to_make(false, ts, ts));
}

// OCC read-phase step: snapshot (word, row, word); spin while locked (Z10).
template <class WL>
GC_DEV int occ_snap_step(Th &th, const ExecParams &p, const typename WL::Params &y, typename WL::Lane &L,
                         u32 gid, u32 i, u64 &obs) {
    u64 *w = cw(p, L.rec);
    const u64 v1 = ld_acquire(w);
    if (v1 & LOCKB) return ST_WAIT;
    const u64 ev = rd<WL>(th, y, L, gid, i, WL::row(y, L));
    fence_acqrel();
    if (ld_relaxed(w) != v1) {
        retract_read(th, ev);
        return ST_RETRY;
    }
    obs = v1;
    return ST_DONE;
}

// no-wait write lock
GC_DEV bool occ_lock(const ExecParams &p, u64 *w, u64 &pre, u64 &seen) {
    u64 v = ld_relaxed(w);
    for (int k = 0; k < 8; k++) {
        seen = v;
        if (v & LOCKB) return false;
        const u64 old = w_cas_acq(p, w, v, v | LOCKB);
        if (old == v) {
            pre = v;
            return true;
        }
        v = old;
    }
    return false;
}

// TicToc read-set validation of one item against commit_ts (Z9)
GC_DEV bool tictoc_validate(const ExecParams &p, u64 *w, u64 obs, u64 cts) {
    if (tt_rts(obs) >= cts) return true;   // version valid through cts already
    u64 v = ld_acquire(w);
    for (;;) {
        if (tt_wts(v) != tt_wts(obs) || (v & LOCKB)) return false;
        if (tt_rts(v) >= cts) return true;
        u64 nw = tt_wts(v);
        if (cts - nw > DMAX) nw = cts - DMAX;   // delta overflow: shift WTS up (Z9)
        const u64 old = w_cas(p, w, v, ((cts - nw) << 48) | nw);
        if (old == v) return true;
        v = old;
    }
}

// N1 intra-warp conflict detection.  Among the converged lanes of a warp that are about to
// CAS a lock word, those naming the same record with at least one exclusive request are
// arbitrated locally, by transaction age (gid + 1; smaller = older): the oldest goes on
// to its CAS, the others take the scheme's conflict outcome at once without touching the
// word -- no-wait / OCC write locks: abort; wait-die: the younger dies.  Equivalent to the
// oldest winning the CAS race (a schedule the racing CASes could produce), but without the
// losing CASes on a hot word, and lockstep lanes stop killing each other symmetrically
// (the oldest always survives the local round).  Lanes alone on their record, or sharing
// it only in shared mode, are unaffected.
GC_DEV bool warp_lock_loser(u32 rec, bool ex, u32 age) {
    const unsigned act = __activemask();
    const unsigned peers = __match_any_sync(act, rec);
    const unsigned exm = __ballot_sync(act, ex) & peers;
    if ((peers & (peers - 1)) == 0 || exm == 0) return false;   // alone, or all shared
    return __reduce_min_sync(peers, age) != age;
}

GC_DEV bool draw_ts_overflow(u64 ts, const ExecParams &p) {
    if (ts > M31) {   // 31-bit field
        set_err(p.ctl, CC_ERR_TS_OVERFLOW);
        return true;
    }
    return false;
}

// ===================================================================== thread mode
// One lane per transaction; accesses processed in ascending key order.  The transaction's
// read/write set -- one WL::Lane per access: record, mode, the value read, the buffered new
// values and the control-word value it saw (OCC snapshot / lock-time word, TO / MVCC saved
// word) -- is staged in shared memory (the OCC "private workspace"): a
// strided array, element i of worker w at base[i * stride + w].  When the launch's working
// lanes do not fit (dense wd, large bs) the same layout lives in a global workspace instead.
// Either way no per-access state sits in registers or local memory (no spills).
// Register budget: the executors run 1024-thread blocks, i.e. at most 64 registers, and a
// row read alone needs 32 for its 16 words in flight.  So the per-worker context (Th) and
// the block-uniform ExecParams live in shared memory: a kernel parameter whose address is
// taken (th.p) would otherwise be copied to local memory, and Th's rarely used fields
// (deadline, pacing state, stage pointers) would hold registers across the whole loop.
extern __shared__ __align__(16) unsigned char gc_dyn_smem[];
__shared__ __align__(16) unsigned char gc_exec_params[sizeof(ExecParams)];   // raw: no __shared__ constructor
GC_DEV void exec_params_copy(const ExecParams &p) {
    if (threadIdx.x == 0) *reinterpret_cast<ExecParams *>(gc_exec_params) = p;
    __syncthreads();
}
GC_DEV const ExecParams *exec_params_smem(const ExecParams &) {
    return reinterpret_cast<const ExecParams *>(gc_exec_params);
}

template <class Lane>
struct Staged {
    Lane *b;
    u32 s;
    GC_DEV Lane &operator[](u32 i) const { return b[(u64)i * s]; }
};

template <int S, class WL, class LA>
GC_DEV int run_thread(Th &th, u32 gid, LA L, u32 n, const typename WL::Params &y, u64 &key_hi, u64 &key_lo) {
    const ExecParams &p = *th.p;
    if constexpr (S == CC_TPL_NW || S == CC_TPL_WD) {
        constexpr bool WD = S == CC_TPL_WD;
        const u32 age = gid + 1;
        u32 i = 0;
        int r = RES_OK;
        for (; i < n; i++) {
            typename WL::Lane &Li = L[i];
            Spin sp;
            int st;
            u64 seen = 0;
            if (warp_lock_loser(Li.rec, Li.w, age)) st = ST_ABORT;   // an older lane of this warp takes it
            else
                while ((st = tpl_try<WD>(p, cw(p, Li.rec), Li.w, age, seen, tpl_intent<WD>(th.attempt))) == ST_WAIT)
                    if (!sp.wait(th)) { st = -1; break; }
            if (st == ST_ABORT) { th.cw = cw(p, Li.rec); th.cv = M31 << 31; th.cw_ex = Li.w; }   // until free
            if (st != ST_DONE) { r = st < 0 ? RES_FATAL : RES_ABORT; break; }
            rd<WL>(th, y, Li, gid, i, WL::row(y, Li));   // stable under the lock
        }
        if (r != RES_OK) {
            fence_acqrel();
            for (u32 j = 0; j < i; j++) tpl_release_relaxed(p, cw(p, L[j].rec), L[j].w);
            return r;
        }
        // lock point: every lock held, none released -> a valid serial order (strict 2PL)
        key_lo = agg_fetch_add(&p.ctl->ticket.v);
        key_hi = 0;
        for (u32 j = 0; j < n; j++)
            if (L[j].w) inst<WL>(th, y, L[j], WL::row(y, L[j]));
        fence_acqrel();
        for (u32 j = 0; j < n; j++) tpl_release_relaxed(p, cw(p, L[j].rec), L[j].w);
        return RES_OK;
    } else if constexpr (S == CC_TO || S == CC_MVCC) {
        u64 ts;
        {
            StageClock c(th, STAGE_TS);
            ts = agg_fetch_add(&p.ctl->ts.v) + 1;   // fresh ts per attempt
        }
        if (draw_ts_overflow(ts, p)) return RES_FATAL;
        u32 pendm = 0;
        int r = RES_OK;
        for (u32 i = 0; i < n && r == RES_OK; i++) {
            typename WL::Lane &Li = L[i];
            Spin sp;
            for (;;) {
                bool pend = false;
                const int st = (S == CC_TO) ? to_step<WL>(th, p, y, Li, gid, i, ts, pend, Li.cv)
                                            : mvcc_step<WL>(th, p, y, Li, gid, i, ts, pend, Li.cv);
                if (pend) pendm |= 1u << i;
                if (st == ST_DONE) break;
                if (st == ST_ABORT) {
                    if (GC_TS_FIFO && Li.w) th.tq = (S == CC_TO) ? cw(p, Li.rec) : mvcc_lo(p, Li.rec);
                    r = RES_ABORT;
                    break;
                }
                if (st == ST_RETRY) continue;
                if (!sp.wait(th)) { r = RES_FATAL; break; }
            }
        }
        if (r != RES_OK) {
            for (u32 j = 0; j < n; j++)
                if ((pendm >> j) & 1) {
                    if (S == CC_TO) w_store(p, cw(p, L[j].rec), L[j].cv);
                    else mvcc_restore<WL>(p, L[j], L[j].cv);
                }
            return r;
        }
        for (u32 j = 0; j < n; j++)
            if ((pendm >> j) & 1) {
                if (S == CC_TO) to_commit<WL>(th, p, y, L[j], ts);
                else mvcc_commit<WL>(th, p, y, L[j], gid, j, ts);
            }
        key_hi = 0;
        key_lo = ts;
        return RES_OK;
    } else if constexpr (S == CC_SILO || S == CC_TICTOC) {
        // read phase: L[i].cv = the word observed with the snapshot
        for (u32 i = 0; i < n; i++) {
            Spin sp;
            int st;
            while ((st = occ_snap_step<WL>(th, p, y, L[i], gid, i, L[i].cv)) != ST_DONE)
                if (st == ST_WAIT && !sp.wait(th)) return RES_FATAL;
        }
        // write-set locks (no-wait).  The lock-time word `pre` is checked against
        // the snapshot at once -- Silo: pre == obs; TicToc: same WTS -- the check validation
        // would make (the word cannot change while we hold its lock); for TicToc the write's
        // slot then keeps `pre` (its RTS enters commit_ts, and an abort restores it).
        u32 locked = 0;
        bool ok = true;
        const u32 age = gid + 1;
        for (u32 i = 0; i < n && ok; i++) {
            typename WL::Lane &Li = L[i];
            if (!Li.w) continue;
            u64 seen = 0, pre = 0;
            if (warp_lock_loser(Li.rec, true, age)) {   // an older lane of this warp locks it
                ok = false;
                th.cw = cw(p, Li.rec);
                th.cv = LOCKB;
                th.cw_ex = true;
                break;
            }
            if (occ_lock(p, cw(p, Li.rec), pre, seen)) {
                locked |= 1u << i;
                if (S == CC_SILO ? pre != Li.cv : tt_wts(pre) != tt_wts(Li.cv)) {
                    ok = false;
                    w_store(p, cw(p, Li.rec), pre);   // changed since the read: unlock, abort
                    locked &= ~(1u << i);
                } else {
                    Li.cv = pre;
                }
            } else {
                ok = false;
                if (seen & LOCKB) { th.cw = cw(p, Li.rec); th.cv = LOCKB; th.cw_ex = true; }   // until unlocked
            }
        }
        u64 ticket = 0, cts = 0;
        if (ok && S == CC_SILO) {
            ticket = agg_fetch_add(&p.ctl->ticket.v);   // serialization point
            fence_acqrel();
            // relaxed: the fence above orders them after the locks and the ticket, and
            // nothing is read through them.  (Acquire loads here were 16 dependent L2 round
            // trips, each invalidating the SM's L1 -- the read-only index included: RO in
            // the paper's launch ran 2.5 ms with the dense index, 425 ms with the binary
            // search.)
            for (u32 i = 0; i < n && ok; i++)
                if (!L[i].w) ok = ld_relaxed(cw(p, L[i].rec)) == L[i].cv;
        }
        if (ok && S == CC_TICTOC) {
            for (u32 i = 0; i < n; i++) {   // commit_ts
                const u64 v = L[i].cv;
                if (L[i].w) cts = max(cts, tt_rts(v) + 1);
                cts = max(cts, tt_wts(v));
            }
            for (u32 i = 0; i < n && ok; i++)
                if (!L[i].w) ok = tictoc_validate(p, cw(p, L[i].rec), L[i].cv, cts);
            if (ok) ticket = agg_fetch_add(&p.ctl->ticket.v);   // after validation
        }
        if (!ok) {
            fence_acqrel();
            for (u32 j = 0; j < n; j++)
                if ((locked >> j) & 1) w_store_relaxed(p, cw(p, L[j].rec), L[j].cv);
            return RES_ABORT;
        }
        u64 nw;
        if (S == CC_SILO) {
            u64 tid = 0;
            for (u32 i = 0; i < n; i++) tid = max(tid, L[i].cv);
            nw = (tid + 1) & ~LOCKB;   // TID = 1 + max observed (epoch dropped)
            key_hi = 0;
        } else {
            nw = cts & M48;
            key_hi = cts;
        }
        key_lo = ticket;
        if (S == CC_TICTOC) fence_acqrel();   // locks (acquire-only CAS) before the installs (Silo: fenced above)
        for (u32 j = 0; j < n; j++)
            if (L[j].w) inst<WL>(th, y, L[j], WL::row(y, L[j]));
        fence_acqrel();
        for (u32 j = 0; j < n; j++)
            if (L[j].w) w_store_relaxed(p, cw(p, L[j].rec), nw);
        return RES_OK;
    } else if constexpr (S == CC_GACCO) {
        // wait for the turn, access, advance the cursor (release after the op, Z3)
        const u64 base = (u64)gid * p.K;
        for (u32 i = 0; i < n; i++) {
            const u32 seg = p.acc_seg[base + i], pos = p.acc_pos[base + i], rdy = p.acc_rdy[base + i];
            if (!gacco_access<WL>(th, y, L[i], gid, i, &p.cursor[seg], pos, rdy)) return RES_FATAL;
        }
        key_hi = 0;
        key_lo = gid;
        return RES_OK;
    } else {   // GPUTx: K-set k runs after K-set k-1 completes; no CC inside
        const u32 k = p.rank_of[gid];
        if (k > 0 && !kset_wait(th, p, k)) return RES_FATAL;
        for (u32 i = 0; i < n; i++) {
            u64 *row = WL::row(y, L[i]);
            rd<WL>(th, y, L[i], gid, i, row);
            if (L[i].w) inst<WL>(th, y, L[i], row);
        }
        kset_done(p, k);
        key_hi = 0;
        key_lo = gid;
        return RES_OK;
    }
}

template <int S, class WL>
__global__ void __launch_bounds__(GC_EXEC_MAXT, GC_EXEC_MINB) exec_thread_kernel(ExecParams p, typename WL::Params y) {
    const u32 lane = threadIdx.x & 31u;
    exec_params_copy(p);
    if (lane >= (1u << p.wd)) return;   // idle lanes exit at once
    if (ld_relaxed(&p.ctl->err.v) != 0) return;   // a3 failed (e.g. KEY_NOT_FOUND): nothing runs
    constexpr bool DET = (S == CC_GPUTX || S == CC_GACCO);
    // shared memory: [Th of every working lane][staged lanes (unless p.ws)]
    const u32 per_warp = 1u << p.wd, per_block = (blockDim.x >> 5) * per_warp;
    const u32 w_in_block = (threadIdx.x >> 5) * per_warp + lane;
    Th &th = reinterpret_cast<Th *>(gc_dyn_smem)[w_in_block];
    th.p = exec_params_smem(p);
    th.polls = 0;
    th.cw = nullptr;
    th.cv = 0;
    th.hot = 0;
    th.turn = nullptr;
    th.tq = nullptr;
    stages_init(th, p, true);
    th.deadline = globaltimer_ns() + p.watchdog_ns;
    // the worker's staged read/write set: shared memory, or the global workspace
    th.cl = Claim{};
    Claim &cl = th.cl;
    using Lane = typename WL::Lane;
    Staged<Lane> L;
    if (p.ws) {
        L.b = reinterpret_cast<Lane *>(p.ws) + (u64)blockIdx.x * per_block + w_in_block;
        L.s = gridDim.x * per_block;
    } else {
        L.b = reinterpret_cast<Lane *>(gc_dyn_smem + (size_t)per_block * sizeof(Th)) + w_in_block;
        L.s = per_block;
    }
    for (;;) {
        const u32 gid = claim_work<S>(th, cl);
        if (gid == NO_TXN) break;
        if (p.skip && p.skip[gid]) {   // distributed (partitioned TPC-C): phase B handles it
            if (S == CC_GPUTX) kset_done(p, p.rank_of[gid]);
            continue;
        }
        u32 n;
        {
            StageClock c(th, STAGE_INDEX);
            n = WL::load_all(p, y, gid, L);
        }
        if (n == 0xFFFFFFFFu) {
            set_err(p.ctl, CC_ERR_KEY_NOT_FOUND);
            break;
        }
        bool stop = false, next = false;
        while (!stop && !next) {
            u64 kh, kl;
            th.gid = gid;
            th.attempt = p.restarts[gid];
            AttemptClock ac(th);
            const int r = run_thread<S, WL>(th, gid, L, n, y, kh, kl);
            rq_release(th);   // GC_RETRY_FIFO: this attempt used its turn
            ac.done(r == RES_OK);
            if (p.events && r != RES_FATAL) log_event(th, 0xFFFFFFFFu, r == RES_OK ? 2u : 3u);
            if (r == RES_OK) {
                {
                    StageClock c(th, STAGE_USEFUL);
                    WL::emit_txn(p, y, gid, L, n);   // outputs + private reserved-slot writes
                }
                p.order_hi[gid] = kh;
                p.order_lo[gid] = kl;
                p.committed[gid] = 1;
                next = true;
            } else if (r == RES_FATAL || DET) {
                stop = true;
            } else {
                const u32 nr = p.restarts[gid] + 1;   // single owner of gid at a time
                p.restarts[gid] = nr;
                StageClock c(th, STAGE_ABORT);
                retry_pace<S>(th, gid, nr);
                if (dead(th)) { stop = true; break; }   // the watchdog also bounds abort-only livelocks
                // (a worker that holds a retry-queue turn retries in place)
                if (!(p.flags & CC_FLAG_IMMEDIATE_RETRY) && !th.turn && try_append_retry(th, gid)) next = true;   // a6
            }
        }
        if (stop) break;
    }
}

// ===================================================================== tile mode
// G lanes per transaction; lane i owns access i.  Every loop below is tile-uniform:
// the exit conditions are tile votes, so all lanes execute the same collectives.
// Restarts from which a retry takes the lock that killed its last attempt first, alone
// (round 1: from 2, against hot-lock livelocks at one TPC-C warehouse).  It lengthens every
// retried critical section by one round trip, and with the retry queues the herds no
// longer need it from the start: from 2 restarts vs never, configs[1] tile 16, exec ms:
// tpl_nw theta 0.6 0.51 -> 0.45, theta 0.8 5.9 -> 5.2; TPC-C one warehouse tpl_nw 0.21 ->
// 0.23 M txn/s; Silo / TicToc within noise (profiles/r02_probe_hot_first.log).  It stays
// as a livelock breaker for long-starved transactions: a small batch with extreme
// contention (2,053 x 16 ops on 1,024 rows, too few transactions for a herd) livelocked
// without it.
#ifndef GC_HOT_FIRST_AFTER
#define GC_HOT_FIRST_AFTER 64
#endif
template <int S, class WL, class Tile>
GC_DEV int run_tile(Tile &tile, Th &th, u32 gid, typename WL::Lane &L,
                    const typename WL::Params &y, u64 &key_hi, u64 &key_lo) {
    const ExecParams &p = *th.p;
    const u32 li = tile.thread_rank();
    const bool act = L.act;
    if constexpr (S == CC_TPL_NW || S == CC_TPL_WD) {
        constexpr bool WD = S == CC_TPL_WD;
        const u32 age = gid + 1;
        bool held = false;
        // Parallel acquisition (every lane CASes its lock at once) is the fast path.  Under
        // extreme contention every dying attempt still holds its other locks for a moment,
        // and those transient holds can keep a hot lock busy forever (TPC-C at 1 warehouse:
        // W is never free when a Payment's lanes look).  So a retry under no-wait takes the
        // lock that killed its previous attempt first, alone, and the rest in parallel once
        // it holds it: a retry that meets the hot lock busy dies holding nothing.
        const u32 first = (WD || th.attempt < GC_HOT_FIRST_AFTER) ? 0u : th.hot;   // 1 + that lock's lane, 0: none
        // wait-die under extreme contention (experiment knob): from GC_WD_SEQ_AFTER restarts
        // on, take the locks one lane at a time in access (key) order, as the paper's
        // one-thread launch does
        const bool seq = WD && GC_WD_SEQ_AFTER > 0 && th.attempt >= GC_WD_SEQ_AFTER;
        Spin sp;
        for (;;) {
            int st = ST_DONE;
            u64 seen = 0;
            bool mine = act && !held;
            if (first && !tile.shfl(held || !act, first - 1)) mine = mine && li == first - 1;
            if (seq) {
                const unsigned want = tile.ballot(mine);
                mine = mine && li == (u32)(__ffs(want) - 1);
            }
            if (mine) {
                if (warp_lock_loser(L.rec, L.w, age)) st = ST_ABORT;   // an older tile of this warp takes it
                else st = tpl_try<WD>(p, cw(p, L.rec), L.w, age, seen, tpl_intent<WD>(th.attempt));
                held = st == ST_DONE;
            }
            const unsigned dying = tile.ballot(st == ST_ABORT);
            if (dying) {
                if (held) tpl_release_relaxed(p, cw(p, L.rec), L.w);
                const int src = __ffs(dying) - 1;   // remember one conflicting lock for the retry
                th.cw = (u64 *)tile.shfl((u64)cw(p, L.rec), src);
                th.cw_ex = tile.shfl((int)L.w, src) != 0;
                th.cv = M31 << 31;                   // wait until its holder count is 0
                th.hot = (u32)src + 1;               // and take it first next time
                return RES_ABORT;
            }
            if (tile.all(!act || held)) break;
            if (!tile.any(st == ST_WAIT)) continue;   // ordered: the next lane's turn
            if (tile.any(!sp.wait(th))) {
                if (held) tpl_release_relaxed(p, cw(p, L.rec), L.w);
                return RES_FATAL;
            }
        }
        // lock point: the ticket's atomic is issued before the row reads, so its round trip
        // overlaps them instead of lengthening the critical section; the shuffle before the
        // releases makes every lane wait for it (a conflicting successor draws its ticket
        // only after acquiring a lock released here)
        u64 ticket = 0;
        if (li == 0) ticket = atomicAdd(&p.ctl->ticket.v, 1ull);
        if (act) rd<WL>(th, y, L, gid, li, WL::row(y, L));   // stable under the lock
        if (act && L.w) inst<WL>(th, y, L, WL::row(y, L));
        key_lo = tile.shfl(ticket, 0);
        key_hi = 0;
        fence_acqrel();
        if (act) tpl_release_relaxed(p, cw(p, L.rec), L.w);
        return RES_OK;
    } else if constexpr (S == CC_TO || S == CC_MVCC) {
        u64 ts = 0;
        {
            StageClock c(th, STAGE_TS);
            if (li == 0) ts = atomicAdd(&p.ctl->ts.v, 1ull) + 1;
            ts = tile.shfl(ts, 0);
        }
        if (draw_ts_overflow(ts, p)) return RES_FATAL;
        bool done = !act, pend = false;
        u64 saved = 0;
        // Basic TO under heavy contention: an attempt doomed by one conflict would still
        // raise the read timestamps of all its other items at once and abort their writers
        // (tile mode at theta=0.99: 5 K txn/s).  After TO_SEQ_AFTER restarts a transaction
        // steps one lane at a time in access order and stops at the first conflict, as the
        // paper's one-thread-per-transaction launch does.
        bool seq = S == CC_TO && th.attempt >= TO_SEQ_AFTER;
        if (S == CC_TO && GC_TO_SEQ_HERD > 0 && !seq && th.attempt >= (u32)GC_TO_SEQ_HERD) {
            u64 n = 0;   // in a herd (many backing off) step one lane at a time sooner
            if (li == 0) n = ld_relaxed(&p.ctl->pacing.v);
            seq = tile.shfl(n, 0) >= 1024;
        }
        Spin sp;
        for (;;) {
            int st = ST_DONE;
            bool mine = !done;
            if (seq) {
                const unsigned want = tile.ballot(mine);
                mine = mine && li == (u32)(__ffs(want) - 1);
            }
            if (mine) {
                st = (S == CC_TO) ? to_step<WL>(th, p, y, L, gid, li, ts, pend, saved)
                                  : mvcc_step<WL>(th, p, y, L, gid, li, ts, pend, saved);
                done = st == ST_DONE;
            }
            if (tile.any(st == ST_ABORT)) {
                if (pend) {
                    if (S == CC_TO) w_store(p, cw(p, L.rec), saved);
                    else mvcc_restore<WL>(p, L, saved);
                }
                if (GC_TS_FIFO) {   // a write whose timestamp check failed: its word names the queue
                    const unsigned wab = tile.ballot(st == ST_ABORT && L.w);
                    th.tq = nullptr;
                    if (wab) {
                        const int src = __ffs(wab) - 1;
                        th.tq = (u64 *)tile.shfl((u64)((S == CC_TO) ? cw(p, L.rec) : mvcc_lo(p, L.rec)), src);
                    }
                }
                return RES_ABORT;
            }
            if (tile.all(done)) break;
            if (tile.any(st == ST_RETRY)) continue;   // lost a CAS race: go again at once
            if (seq && !tile.any(st == ST_WAIT)) continue;   // sequential: the next lane's turn
            if (tile.any(!sp.wait(th))) {
                if (pend) {
                    if (S == CC_TO) w_store(p, cw(p, L.rec), saved);
                    else mvcc_restore<WL>(p, L, saved);
                }
                return RES_FATAL;
            }
        }
        if (pend) {
            if (S == CC_TO) to_commit<WL>(th, p, y, L, ts);
            else mvcc_commit<WL>(th, p, y, L, gid, li, ts);
        }
        key_hi = 0;
        key_lo = ts;
        return RES_OK;
    } else if constexpr (S == CC_SILO || S == CC_TICTOC) {
        u64 obs = 0, pre = 0;
        bool done = !act;
        Spin sp;
        for (;;) {   // read phase
            int st = ST_DONE;
            if (!done) {
                st = occ_snap_step<WL>(th, p, y, L, gid, li, obs);
                done = st == ST_DONE;
            }
            if (tile.all(done)) break;
            if (tile.any(st == ST_RETRY)) continue;
            if (tile.any(!sp.wait(th))) return RES_FATAL;
        }
        bool locked = false, bad = false;
        u64 seen = 0;
        // write-set locks: all at once; a retry takes the lock that was busy last time
        // first, alone (see 2PL)
        const u32 first = th.attempt < GC_HOT_FIRST_AFTER ? 0u : th.hot;
        const u32 age = gid + 1;
        if (first && li == first - 1 && act && L.w) {
            if (warp_lock_loser(L.rec, true, age)) { bad = true; seen = LOCKB; }   // an older tile locks it
            else { locked = occ_lock(p, cw(p, L.rec), pre, seen); bad = !locked; }
        }
        if (!tile.any(bad) && act && L.w && !locked) {
            if (warp_lock_loser(L.rec, true, age)) { bad = true; seen = LOCKB; }
            else { locked = occ_lock(p, cw(p, L.rec), pre, seen); bad = !locked; }
        }
        {
            const unsigned busy = tile.ballot(bad && (seen & LOCKB));
            th.hot = 0;
            if (busy) {
                const int src = __ffs(busy) - 1;
                th.cw = (u64 *)tile.shfl((u64)cw(p, L.rec), src);
                th.cw_ex = true;
                th.cv = LOCKB;                       // wait until unlocked
                th.hot = (u32)src + 1;
            }
        }
        u64 ticket = 0, cts = 0;
        if (!tile.any(bad)) {
            if (S == CC_SILO) {
                if (li == 0) ticket = atomicAdd(&p.ctl->ticket.v, 1ull);   // serialization point
                ticket = tile.shfl(ticket, 0);
                fence_acqrel();
                if (act) bad = L.w ? (pre != obs) : (ld_relaxed(cw(p, L.rec)) != obs);   // see run_thread
            } else {
                u64 c = 0;
                if (act) c = max(L.w ? tt_rts(pre) + 1 : 0ull, tt_wts(obs));
                cts = cg::reduce(tile, c, cg::greater<u64>());
                if (act) bad = L.w ? (tt_wts(pre) != tt_wts(obs)) : !tictoc_validate(p, cw(p, L.rec), obs, cts);
                if (!tile.any(bad)) {
                    if (li == 0) ticket = atomicAdd(&p.ctl->ticket.v, 1ull);   // after validation
                    ticket = tile.shfl(ticket, 0);
                }
            }
        }
        if (tile.any(bad)) {
            if (locked) w_store(p, cw(p, L.rec), pre);
            return RES_ABORT;
        }
        u64 nw;
        if (S == CC_SILO) {
            const u64 tid = cg::reduce(tile, act ? obs : 0ull, cg::greater<u64>());
            nw = (tid + 1) & ~LOCKB;
            key_hi = 0;
        } else {
            nw = cts & M48;
            key_hi = cts;
        }
        key_lo = ticket;
        if (S == CC_TICTOC && act && L.w) fence_acqrel();   // locks (acquire-only CAS) before the installs
        if (act && L.w) inst<WL>(th, y, L, WL::row(y, L));
        fence_acqrel();
        if (act && L.w) w_store_relaxed(p, cw(p, L.rec), nw);
        return RES_OK;
    } else if constexpr (S == CC_GACCO) {
        int st = ST_DONE;
        if (act) {   // each lane waits for its own item's turn: overlapped across items
            const u64 a = (u64)gid * p.K + li;
            const u32 seg = p.acc_seg[a], pos = p.acc_pos[a], rdy = p.acc_rdy[a];
            if (!gacco_access<WL>(th, y, L, gid, li, &p.cursor[seg], pos, rdy)) st = ST_ABORT;
        }
        if (tile.any(st != ST_DONE)) return RES_FATAL;
        key_hi = 0;
        key_lo = gid;
        return RES_OK;
    } else {   // GPUTx
        const u32 k = p.rank_of[gid];
        int st = ST_DONE;
        // Early reads (GC_GPUTX_EARLY): an access whose item was last written (in id order)
        // by a K-set before k-1 reads its row before the gate, once that K-set is complete
        // -- nothing writes the item between then and this transaction (later writes of it
        // rank above k).  Only the rows written by K-set k-1 are read after the gate, and
        // those were just installed (L2).  The gate still orders every install.
        bool done_rd = false;
        if (GC_GPUTX_EARLY && act && k > 0) {
            const u32 dep = p.acc_rdy[(u64)gid * p.K + li];
            if (dep < k) {   // K-set dep - 1 <= k - 2 (or no earlier write)
                if (dep > 0) {
                    Spin sp(256);
                    while (ld_acquire32(&p.rank_done[dep - 1]) < p.rank_count[dep - 1])
                        if (!sp.wait(th)) { st = ST_ABORT; break; }
                }
                if (st == ST_DONE) {
                    rd<WL>(th, y, L, gid, li, WL::row(y, L));
                    done_rd = true;
                }
            }
        }
        if (tile.any(st != ST_DONE)) return RES_FATAL;
        if (k > 0) {
            // The rows were prefetched at claim time, often long before the gate opens, and
            // the L2 has turned over since: fetch them again once K-set k-1 is the frontier,
            // so the reads after the gate -- on the K-set chain's critical path -- hit L2.
            if (li == 0 && !kset_near(th, p, k)) st = ST_ABORT;
            if (tile.shfl(st, 0) == ST_DONE && act && !done_rd) WL::prefetch_access(p, y, L);
            if (li == 0 && st == ST_DONE && !kset_wait(th, p, k)) st = ST_ABORT;
            if (li == 0 && st == ST_DONE) kset_trace(p, k, 1);
        }
        tile.sync();          // the leader's acquire orders every lane's accesses (warp barrier)
        if (tile.any(st != ST_DONE)) return RES_FATAL;
        if (act) {
            u64 *row = WL::row(y, L);
#if defined(GC_EXP_NOREAD) && GC_EXP_NOREAD   // timing experiment only (wrong results)
            if (L.w) inst<WL>(th, y, L, row);
#else
            if (!done_rd) rd<WL>(th, y, L, gid, li, row);
            if (L.w) inst<WL>(th, y, L, row);
#endif
        }
        tile.sync();   // every lane's install precedes the K-set release
        if (li == 0) kset_done(p, k);
        key_hi = 0;
        key_lo = gid;
        return RES_OK;
    }
}

// Experiment builds (-DGC_TRACE_COMMIT=1, tools/trace_tail.py): trace[0] = kernel start
// (ns), trace[1] = bucket width (ns), trace[2 + b] = commits, trace[1026 + b] = aborts in
// time bucket b since the start.
#ifndef GC_TRACE_COMMIT
#define GC_TRACE_COMMIT 0
#endif
GC_DEV void trace_event(const ExecParams &p, bool commit) {
#if GC_TRACE_COMMIT
    if (!p.trace) return;
    const u64 t = globaltimer_ns(), t0 = ld_relaxed(&p.trace[0]), w = p.trace[1];
    u64 b = (t > t0 ? t - t0 : 0) / (w ? w : 1000);
    if (b > 1023) b = 1023;
    atomicAdd(&p.trace[(commit ? 2 : 1026) + b], 1ull);
#endif
}

template <int S, class WL, int G>
__global__ void __launch_bounds__(GC_EXEC_MAXT, GC_EXEC_MINB) exec_tile_kernel(ExecParams p, typename WL::Params y) {
    auto tile = cg::tiled_partition<G>(cg::this_thread_block());
    const u32 li = tile.thread_rank();
#if GC_TRACE_COMMIT
    if (p.trace) {
        if (threadIdx.x == 0) atomicCAS(&p.trace[0], 0ull, globaltimer_ns());
        __syncthreads();
    }
#endif
    exec_params_copy(p);
    if (ld_relaxed(&p.ctl->err.v) != 0) return;   // a3 failed (e.g. KEY_NOT_FOUND): nothing runs
    constexpr bool DET = (S == CC_GPUTX || S == CC_GACCO);
    Th &th = reinterpret_cast<Th *>(gc_dyn_smem)[threadIdx.x];   // per-lane context in shared memory
    th.p = exec_params_smem(p);
    th.polls = 0;
    th.cw = nullptr;
    th.cv = 0;
    th.hot = 0;
    th.turn = nullptr;
    th.tq = nullptr;
    stages_init(th, p, li == 0);   // stages are timed by each tile's leader
    th.deadline = globaltimer_ns() + p.watchdog_ns;
    // the lane's access (its read/write-set entry): registers, or -- for workloads whose
    // entry is large (TPC-C: values read, buffered writes, strings) -- shared memory after
    // the contexts, so the tile loop keeps its registers for the row reads
    typename WL::Lane Lr;
    typename WL::Lane *Ls = p.ws ? reinterpret_cast<typename WL::Lane *>(p.ws) + (u64)blockIdx.x * blockDim.x
                                 : reinterpret_cast<typename WL::Lane *>(gc_dyn_smem + (size_t)blockDim.x * sizeof(Th));
    typename WL::Lane &L = WL::STAGE_TILE_LANE ? Ls[threadIdx.x] : Lr;   // (global when it does not fit)
    th.cl = Claim{};
    Claim &cl = th.cl;
    u32 att = 0;   // leader: restarts of the current transaction (fresh ids: 0, not loaded)
    for (;;) {
        u32 gid = NO_TXN;
        bool fresh = false;
        if (li == 0) {
            gid = claim_work<S>(th, cl);
            fresh = cl.fresh;
        }
        gid = tile.shfl(gid, 0);
        fresh = tile.shfl(fresh, 0);
        th.hot = tile.shfl(th.hot, 0);   // from the retry-batch entry (0 for a fresh id)
        if (gid == NO_TXN) break;
        if (li == 0) att = fresh ? 0u : p.restarts[gid];   // fresh ids start at 0 restarts
        if (p.skip && p.skip[gid]) {   // distributed (partitioned TPC-C): phase B handles it
            if (S == CC_GPUTX && li == 0) kset_done(p, p.rank_of[gid]);
            continue;
        }
        bool ok;
        {
            StageClock c(th, STAGE_INDEX);
            ok = WL::load_lane(p, y, gid, li, L);
        }
        if (!tile.all(ok)) {
            if (li == 0) set_err(p.ctl, CC_ERR_KEY_NOT_FOUND);
            break;
        }
        if (!DET && (p.flags & CC_FLAG_WARM)) {
            // the loads' values are consumed here, so no lane issues its first CC step
            // (CAS, pending bit, snapshot) before its lines have arrived in L2
            const u64 v = L.act ? WL::warm(p, y, L) : 0ull;
            if (v == 0x9E3779B97F4A7C15ull) atomicAdd(&p.ctl->warm_hits.v, 1ull);
            tile.sync();
        }
        bool stop = false, next = false;
        while (!stop && !next) {
            u64 kh = 0, kl = 0;
            th.gid = gid;
            th.attempt = tile.shfl(att, 0);   // the leader owns restarts
            AttemptClock ac(th);
            const int r = run_tile<S, WL>(tile, th, gid, L, y, kh, kl);
            if (li == 0) rq_release(th);   // GC_RETRY_FIFO: this attempt used its turn
            ac.done(r == RES_OK);
            if (p.events && r != RES_FATAL) {
                tile.sync();   // every lane's access events precede the commit / abort event
                if (li == 0) log_event(th, 0xFFFFFFFFu, r == RES_OK ? 2u : 3u);
            }
            if (r == RES_OK) {
                {
                    StageClock c(th, STAGE_USEFUL);
                    WL::emit_tile(tile, p, y, gid, L, li);   // outputs + private reserved-slot writes
                }
                if (li == 0) {
                    p.order_hi[gid] = kh;
                    p.order_lo[gid] = kl;
                    p.committed[gid] = 1;
                    trace_event(p, true);
                }
                next = true;
            } else if (r == RES_FATAL || DET) {
                stop = true;
            } else {
                int push = 0;
                if (li == 0) {
                    trace_event(p, false);
                    const u32 nr = ++att;
                    p.restarts[gid] = nr;
                    StageClock c(th, STAGE_ABORT);
                    retry_pace<S>(th, gid, nr);
                    if (dead(th)) push = -1;   // the watchdog also bounds abort-only livelocks
                    else push = !(p.flags & CC_FLAG_IMMEDIATE_RETRY) && !th.turn && try_append_retry(th, gid);   // a6
                }
                push = tile.shfl(push, 0);
                if (push < 0) stop = true;
                next = push > 0;
            }
        }
        if (stop) break;
    }
}

}  // namespace gcctb
