// common.cuh -- device primitives for the sm_100a CC kernels.
//
// Memory-ordering contract ("a memory fence is necessary ... after the
// release of a spin lock"; "the initial read of the integer should use a
// volatile pointer").  On sm_100a we express it with the PTX memory model directly:
//   control words : ld.acquire.gpu / atom.acq_rel.gpu.cas / st.release.gpu
//   row payloads  : ld.global.cg (L2, never a stale L1 line) / st.global.cg
//   seqlock checks: fence.acq_rel.gpu between the payload loads and the re-load.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gcctb {

typedef unsigned long long u64;
typedef uint32_t u32;

#define GC_DEV __device__ __forceinline__

GC_DEV u64 ld_acquire(const u64 *p) {
    u64 v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
GC_DEV u64 ld_relaxed(const u64 *p) {
    u64 v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
GC_DEV u32 ld_acquire32(const u32 *p) {
    u32 v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
GC_DEV u32 ld_relaxed32(const u32 *p) {
    u32 v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
GC_DEV void st_release(u64 *p, u64 v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
GC_DEV void st_release32(u32 *p, u32 v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
GC_DEV void st_relaxed32(u32 *p, u32 v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
GC_DEV void st_relaxed(u64 *p, u64 v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// CAS with acquire+release semantics; returns the old value.
GC_DEV u64 cas_acqrel(u64 *p, u64 expect, u64 desired) {
    u64 old;
    asm volatile("atom.acq_rel.gpu.global.cas.b64 %0, [%1], %2, %3;"
                 : "=l"(old) : "l"(p), "l"(expect), "l"(desired) : "memory");
    return old;
}
// Lock acquisition: acquire ordering only (nothing before it is published by it), so
// ptxas emits no MEMBAR in front of the CAS as it does for acq_rel.
GC_DEV u64 cas_acquire(u64 *p, u64 expect, u64 desired) {
    u64 old;
    asm volatile("atom.acquire.gpu.global.cas.b64 %0, [%1], %2, %3;"
                 : "=l"(old) : "l"(p), "l"(expect), "l"(desired) : "memory");
    return old;
}
GC_DEV u64 atom_add_acqrel(u64 *p, u64 v) {
    u64 old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], %2;"
                 : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}
GC_DEV u64 atom_add_relaxed(u64 *p, u64 v) {
    u64 old;
    asm volatile("atom.relaxed.gpu.global.add.u64 %0, [%1], %2;"
                 : "=l"(old) : "l"(p), "l"(v) : "memory");
    return old;
}
GC_DEV u32 atom_add_release32(u32 *p, u32 v) {
    u32 old;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;"
                 : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
GC_DEV u32 atom_add_acqrel32(u32 *p, u32 v) {
    u32 old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;"
                 : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
GC_DEV void fence_acqrel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
GC_DEV void fence_sc() { asm volatile("fence.sc.gpu;" ::: "memory"); }

// Row payload access through L2 (coherent point), 16 B vectors.
GC_DEV void ld_cg_v2(const u64 *p, u64 &a, u64 &b) {
    asm volatile("ld.global.cg.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
// 32 B vectors (sm_100: one LDG.E.ENL2.256 request instead of two 128-bit ones); p must
// be 32 B aligned
GC_DEV void ld_cg_v4(const u64 *p, u64 &a, u64 &b, u64 &c, u64 &d) {
    asm volatile("ld.global.cg.v4.u64 {%0, %1, %2, %3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p) : "memory");
}
GC_DEV void st_cg_v4(u64 *p, u64 a, u64 b, u64 c, u64 d) {
    asm volatile("st.global.cg.v4.u64 [%0], {%1, %2, %3, %4};" :: "l"(p), "l"(a), "l"(b), "l"(c), "l"(d)
                 : "memory");
}
GC_DEV u64 ld_cg(const u64 *p) {
    u64 a;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(a) : "l"(p) : "memory");
    return a;
}
GC_DEV u32 ld_cg32(const u32 *p) {
    u32 a;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(a) : "l"(p) : "memory");
    return a;
}
GC_DEV void st_cg(u64 *p, u64 v) {
    asm volatile("st.global.cg.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
GC_DEV void st_cg_v2(u64 *p, u64 a, u64 b) {
    asm volatile("st.global.cg.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

GC_DEV u64 globaltimer_ns() {
    u64 t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// L2 prefetch: no memory-ordering effect, so it can run ahead of the acquire loads and
// CASes that must precede the real accesses
GC_DEV void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

GC_DEV u64 clk64() {
    u64 t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
    return t;
}

GC_DEV void backoff(unsigned &ns) {
    __nanosleep(ns);
    ns = ns < 256 ? ns * 2 : 256;
}

// splitmix64 finaliser and the counter-based generator of the a1 batch generator
// (the device copy; the oracle has its own by specification).
__host__ __device__ __forceinline__ u64 mix64(u64 z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ u64 rng3(u64 seed, u64 a, u64 b) {
    return mix64(mix64(seed ^ mix64(a)) ^ b);
}

GC_DEV u64 rotl64(u64 x, unsigned r) { return r ? ((x << r) | (x >> (64u - r))) : x; }

}  // namespace gcctb
