// roof.cu -- the memory-system ceilings the executor is measured against (SURVEY.md
// §8(d) "Which roofline bounds the path"): every access of the hot path is a random
// 128 B line, a control-word atomic, or -- under contention -- a hand-off of one record
// from one transaction to the next.  Three microbenchmarks, each timed with CUDA events
// on the caller's stream:
//   * gather:  random 128 B line reads (4 x 32 B .cg loads, the YCSB row read of
//              exec.cuh) over a buffer larger than L2 -> GB/s of whole lines;
//   * atomics: 64-bit CAS on distinct random words (the control-word CAS of every
//              scheme), once over an L2-resident array and once over an array larger
//              than L2 -> operations / s;
//   * hand-off: a token passed around a ring of one warp per SM; at its turn a warp
//              polls the token (relaxed), acquires, reads the record's 128 B row,
//              installs two words and releases the token (the GaccO / lock hand-off of
//              exec.cuh) -> ns per hop, averaged over every neighbouring SM pair, plus
//              the bare token hop without the row.
#include <cuda_runtime.h>

#include "common.cuh"

namespace gcctb {

GC_DEV u64 roof_hash(u64 x) {   // splitmix64 finaliser
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

constexpr int CAS_ILP = 4;

template <int ROOF_ILP>
__global__ void roof_gather_kernel(const u64 *buf, u64 line_mask, u32 iters, u64 *sink) {   // 2^k lines
    const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    u64 acc = 0;
    for (u32 it = 0; it < iters; it++) {
        u64 v[ROOF_ILP][4];
#pragma unroll
        for (int k = 0; k < ROOF_ILP; k++) {
            const u64 line = roof_hash(t * 0x10001ull + it * ROOF_ILP + k) & line_mask;
            const u64 *p = buf + line * 16;
            u64 a, b, c, d, e, f, g, h;
            ld_cg_v4(p, a, b, c, d);
            ld_cg_v4(p + 4, e, f, g, h);
            v[k][0] = a ^ e;
            v[k][1] = b ^ f;
            ld_cg_v4(p + 8, a, b, c, d);
            ld_cg_v4(p + 12, e, f, g, h);
            v[k][2] = c ^ g ^ a ^ e;
            v[k][3] = d ^ h ^ b ^ f;
        }
#pragma unroll
        for (int k = 0; k < ROOF_ILP; k++) acc += v[k][0] ^ v[k][1] ^ v[k][2] ^ v[k][3];
    }
    if (acc == 0x5A5A5A5A5A5A5A5Aull) sink[0] = acc;   // keeps the loads alive
}

// access-size sweep of the gather ceiling: random BYTES-sized, BYTES-aligned reads (32 B
// .cg vectors), ILP of them in flight per thread
template <int BYTES, int ILP>
__global__ void roof_gather_sweep_kernel(const u64 *buf, u64 unit_mask, u32 iters, u64 *sink) {
    constexpr int V = BYTES / 32;   // 32 B vectors per access
    const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    u64 acc = 0;
    for (u32 it = 0; it < iters; it++) {
        u64 v[ILP];
#pragma unroll
        for (int k = 0; k < ILP; k++) {
            const u64 u = roof_hash(t * 0x10001ull + it * ILP + k) & unit_mask;
            const u64 *p = buf + u * (BYTES / 8);
            u64 x = 0;
#pragma unroll
            for (int j = 0; j < V; j++) {
                u64 a, b, c, d;
                ld_cg_v4(p + 4 * j, a, b, c, d);
                x ^= a ^ b ^ c ^ d;
            }
            v[k] = x;
        }
#pragma unroll
        for (int k = 0; k < ILP; k++) acc += v[k];
    }
    if (acc == 0x5A5A5A5A5A5A5A5Aull) sink[0] = acc;
}

template <int BYTES>
static double sweep_one(cudaStream_t s, int num_sms, const u64 *buf, u64 bytes, u64 *sink, cudaEvent_t a,
                        cudaEvent_t b) {
    const int blk = 256, grid = num_sms * 8;
    const u64 threads = (u64)grid * blk, units = bytes / BYTES;
    double best = 0;
    roof_gather_sweep_kernel<BYTES, 8><<<grid, blk, 0, s>>>(buf, units - 1, 1, sink);   // warm-up
    for (int v = 0; v < 2; v++) {   // 8 or 16 accesses in flight per thread
        const u32 iters = 8;
        cudaEventRecord(a, s);
        if (v == 0) roof_gather_sweep_kernel<BYTES, 8><<<grid, blk, 0, s>>>(buf, units - 1, iters, sink);
        else roof_gather_sweep_kernel<BYTES, 16><<<grid, blk, 0, s>>>(buf, units - 1, iters / 2, sink);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double gbs = (double)threads * 64 * BYTES / (ms * 1e-3) / 1e9;   // 8 x 8 or 16 x 4 accesses
        best = gbs > best ? gbs : best;
    }
    return best;
}

// GB/s of random reads of 32, 64, 128 and 256 B over 1 GiB (larger than L2)
cudaError_t gather_sweep(cudaStream_t s, int num_sms, double out[4]) {
    const u64 bytes = 1ull << 30;
    u64 *buf = nullptr, *sink = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&buf, bytes)) || (e = cudaMalloc(&sink, 64)) || (e = cudaEventCreate(&a)) ||
        (e = cudaEventCreate(&b)))
        goto done;
    cudaMemsetAsync(buf, 0x3C, bytes, s);
    out[0] = sweep_one<32>(s, num_sms, buf, bytes, sink, a, b);
    out[1] = sweep_one<64>(s, num_sms, buf, bytes, sink, a, b);
    out[2] = sweep_one<128>(s, num_sms, buf, bytes, sink, a, b);
    out[3] = sweep_one<256>(s, num_sms, buf, bytes, sink, a, b);
    e = cudaGetLastError();
done:
    cudaStreamSynchronize(s);
    if (buf) cudaFree(buf);
    if (sink) cudaFree(sink);
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    return e;
}

__global__ void roof_cas_kernel(u64 *words, u64 word_mask, u32 iters, u64 *sink) {   // 2^k words
    const u64 t = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    u64 acc = 0;
    for (u32 it = 0; it < iters; it++) {
        u64 r[CAS_ILP];
#pragma unroll
        for (int k = 0; k < CAS_ILP; k++) {
            const u64 w = roof_hash(t * 0x10001ull + it * CAS_ILP + k) & word_mask;
            r[k] = atomicCAS((unsigned long long *)(words + w), 0ull, t + 1);
        }
#pragma unroll
        for (int k = 0; k < CAS_ILP; k++) acc += r[k];
    }
    if (acc == 0x5A5A5A5A5A5A5A5Aull) sink[0] = acc;
}

// one warp per block, one block per SM; lane 0 of block j moves at token values
// j, j + G, j + 2G, ...
// acq_poll: poll with ld.acquire (no separate fence) instead of relaxed polls + fence
__global__ void roof_handoff_kernel(u32 *token, u64 *row, u32 rounds, int with_row, int acq_poll,
                                    u64 timeout_ns, u64 *sink) {
    if (threadIdx.x != 0) return;
    const u64 deadline_ns = globaltimer_ns() + timeout_ns;
    const u32 G = gridDim.x, j = blockIdx.x;
    u64 acc = 0;
    for (u32 r = 0; r < rounds; r++) {
        const u32 turn = r * G + j;
        while ((acq_poll ? ld_acquire32(token) : ld_relaxed32(token)) != turn) {
            if (globaltimer_ns() > deadline_ns) {
                sink[1] = 1;   // timed out (blocks not co-resident)
                return;
            }
        }
        if (!acq_poll) fence_acqrel();
        if (with_row) {
            u64 v[16];
#pragma unroll
            for (int k = 0; k < 4; k++) ld_cg_v4(row + 4 * k, v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
            u64 fp = 0;
#pragma unroll
            for (int k = 0; k < 16; k++) fp += rotl64(v[k], k);
            acc += fp;
            st_cg(row + (turn & 7), v[turn & 7] * 0x9E3779B97F4A7C15ull + turn + 1);
            st_cg(row + 15, v[15] + 1);
        }
        st_release32(token, turn + 1);
    }
    if (acc == 0x5A5A5A5A5A5A5A5Aull) sink[0] = acc;
}

static float time_ms(cudaStream_t s, cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

// out[0] gather GB/s, out[1] CAS/s (L2-resident), out[2] CAS/s (> L2), out[3] hand-off
// ns per hop with the row, out[4] bare token hop ns, out[5] row hop with acquire polls.  Scratch: 1 GiB + 256 MiB.
cudaError_t roofline_probe(cudaStream_t s, int num_sms, double out[6]) {
    const u64 gather_bytes = 1ull << 30, l2_words = 2ull << 20, hbm_words = 32ull << 20;
    u64 *buf = nullptr, *words = nullptr, *sink = nullptr, *row = nullptr;
    u32 *token = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&buf, gather_bytes)) || (e = cudaMalloc(&words, hbm_words * 8)) ||
        (e = cudaMalloc(&sink, 64)) || (e = cudaMalloc(&row, 256)) || (e = cudaMalloc(&token, 256)) ||
        (e = cudaEventCreate(&a)) || (e = cudaEventCreate(&b)))
        goto done;
    cudaMemsetAsync(buf, 0x3C, gather_bytes, s);
    cudaMemsetAsync(words, 0, hbm_words * 8, s);
    cudaMemsetAsync(sink, 0, 64, s);
    cudaMemsetAsync(row, 0, 256, s);
    {
        const int blk = 256, grid = num_sms * 8;
        const u64 threads = (u64)grid * blk;
        const u32 iters = 16;
        const u64 n_lines = gather_bytes / 128;
        roof_gather_kernel<4><<<grid, blk, 0, s>>>(buf, n_lines - 1, 2, sink);   // warm-up
        for (int v = 0; v < 2; v++) {   // 4 or 8 lines in flight per thread: the better one
            cudaEventRecord(a, s);
            if (v == 0) roof_gather_kernel<4><<<grid, blk, 0, s>>>(buf, n_lines - 1, iters, sink);
            else roof_gather_kernel<8><<<grid, blk, 0, s>>>(buf, n_lines - 1, iters / 2, sink);
            cudaEventRecord(b, s);
            const double gbs = (double)threads * iters * 4 * 128.0 / (time_ms(s, a, b) * 1e-3) / 1e9;
            out[0] = gbs > out[0] ? gbs : out[0];
        }
        for (int v = 0; v < 2; v++) {
            const u64 nw = v == 0 ? l2_words : hbm_words;
            roof_cas_kernel<<<grid, blk, 0, s>>>(words, nw - 1, 2, sink);
            cudaEventRecord(a, s);
            roof_cas_kernel<<<grid, blk, 0, s>>>(words, nw - 1, iters, sink);
            cudaEventRecord(b, s);
            out[1 + v] = (double)threads * iters * CAS_ILP / (time_ms(s, a, b) * 1e-3);
        }
        const int idx[3] = {3, 4, 5};
        for (int v = 0; v < 3; v++) {   // row + fence, bare hop, row + acquire polls
            const u32 rounds = 40;
            cudaMemsetAsync(token, 0, 4, s);
            cudaEventRecord(a, s);
            // 2 s bound: the ring needs its blocks co-resident (one warp per SM is)
            roof_handoff_kernel<<<num_sms, 32, 0, s>>>(token, row, rounds, v != 1, v == 2, 2000000000ull, sink);
            cudaEventRecord(b, s);
            out[idx[v]] = time_ms(s, a, b) * 1e6 / ((double)rounds * num_sms);
        }
    }
    e = cudaGetLastError();
    if (e == cudaSuccess) {
        u64 h[2] = {0, 0};
        cudaMemcpyAsync(h, sink, 16, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (h[1]) out[3] = out[4] = out[5] = -1.0;   // ring timed out: no hand-off figure
    }
done:
    cudaStreamSynchronize(s);
    if (buf) cudaFree(buf);
    if (words) cudaFree(words);
    if (sink) cudaFree(sink);
    if (row) cudaFree(row);
    if (token) cudaFree(token);
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    return e;
}

}  // namespace gcctb
