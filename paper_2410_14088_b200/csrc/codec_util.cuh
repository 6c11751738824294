// codec_util.cuh — small device helpers shared by the codec kernels and the
// fused quantisation epilogue of the gate engine.
#pragma once

#include "device_common.cuh"

namespace bmq {

__device__ __forceinline__ uint32_t chunk_len(uint64_t count, uint32_t c) {
    const uint64_t first = static_cast<uint64_t>(c) * kChunk;
    const uint64_t rest = count - first;
    return rest < kChunk ? static_cast<uint32_t>(rest) : kChunk;
}

// valid bits of bitmap word k of a chunk of len scalars
__device__ __forceinline__ uint32_t word_mask(uint32_t len, uint32_t k) {
    const uint32_t first = k * 32;
    if (first >= len) return 0;
    const uint32_t n = len - first;
    return n >= 32 ? 0xffffffffu : ((1u << n) - 1);
}

// CTA (4 warps) reduction of three partial sums, added into dst[0..2]
// (sumsq, sum_re, sum_im are consecutive in BlockPlan and DecInfo).
__device__ __forceinline__ void block_sums3(double a, double b, double c, double (*s_red)[4], double* dst) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (lane == 0) {
        s_red[0][w] = a;
        s_red[1][w] = b;
        s_red[2][w] = c;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        const double v = s_red[threadIdx.x][0] + s_red[threadIdx.x][1] + s_red[threadIdx.x][2] + s_red[threadIdx.x][3];
        if (v != 0.0) atomicAdd(dst + threadIdx.x, v);
    }
}

// Running per-chunk counters of one thread (see ChunkPlan).
struct ChunkAcc {
    uint32_t qmin_inv = 0, qmax_off = 0, nnz = 0, nneg = 0;
    __device__ __forceinline__ void add(uint32_t pk) {
        if (!(pk & 1u)) {
            const uint32_t qo = pk >> 2;
            qmin_inv = max(qmin_inv, kQOffMax - qo);
            qmax_off = max(qmax_off, qo);
            ++nnz;
        }
        nneg += (pk >> 1) & 1u;
    }
};

// Warp-wide reduction of a ChunkAcc and one set of atomics by lane 0 (all 32
// lanes must call it with the same target).
__device__ __forceinline__ void flush_chunk(ChunkPlan* cp, ChunkAcc a) {
    for (int o = 16; o; o >>= 1) {
        a.qmin_inv = max(a.qmin_inv, __shfl_xor_sync(0xffffffffu, a.qmin_inv, o));
        a.qmax_off = max(a.qmax_off, __shfl_xor_sync(0xffffffffu, a.qmax_off, o));
        a.nnz += __shfl_xor_sync(0xffffffffu, a.nnz, o);
        a.nneg += __shfl_xor_sync(0xffffffffu, a.nneg, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (a.nnz) {
            atomicMax(&cp->qmin_inv, a.qmin_inv);
            atomicMax(&cp->qmax_off, a.qmax_off);
            atomicAdd(&cp->nnz, a.nnz);
        }
        if (a.nneg) atomicAdd(&cp->nneg, a.nneg);
    }
}

// Exact quantisation of one scalar into its packed code word.
__device__ __forceinline__ uint32_t quantize_pack(double v, const DevTables& t, bool& bad, bool& oow) {
    if (!isfinite(v)) {
        bad = true;
        return 1u;
    }
    if (v == 0.0) return 1u;
    const int64_t q = quantize(v, t, oow);
    return pack_code(static_cast<uint32_t>(q - t.qlo), v < 0.0, false);
}

// quantize_pack for N scalars at once: every estimate first, then both
// neighbouring thresholds of every estimate as independent loads (2N in
// flight instead of a dependent chain per scalar), then the exact
// settlement; an estimate off by more than one falls back to quantize().
template <int N>
__device__ __forceinline__ void quantize_pack_n(const double* v, uint32_t* pk, const DevTables& t, bool& bad,
                                                bool& oow) {
    uint64_t bits[N];
    int idx[N];  // table index (< 2^25 entries)
    bool live[N], sure[N];
    const double qlo = static_cast<double>(t.qlo);
    const int span = static_cast<int>(t.qhi - t.qlo);
#pragma unroll
    for (int e = 0; e < N; ++e) {
        live[e] = isfinite(v[e]) && v[e] != 0.0;
        if (!isfinite(v[e])) bad = true;
        const double x = live[e] ? quantize_estimate_x(v[e], t, bits[e]) : 0.0;
        const double r = rint(x);
        const int i = __double2int_rz(r - qlo);  // exact (integers below 2^53); saturates
        // the rounding is settled unless x lies within est_eps of a half-integer
        sure[e] = 0.5 - fabs(x - r) > t.est_eps && i >= 0 && i <= span;
        idx[e] = min(max(i, 0), span);
    }
    uint64_t t0[N], t1[N];
#pragma unroll
    for (int e = 0; e < N; ++e) {  // threshold probes only near a tie
        t0[e] = (live[e] && !sure[e]) ? __ldg(t.thresh + idx[e]) : 0;
        t1[e] = (live[e] && !sure[e]) ? __ldg(t.thresh + idx[e] + 1) : ~0ull;
    }
#pragma unroll
    for (int e = 0; e < N; ++e) {
        if (!live[e]) {
            pk[e] = 1u;
            continue;
        }
        uint32_t qoff;
        if (sure[e] || (bits[e] >= t0[e] && bits[e] < t1[e]))
            qoff = static_cast<uint32_t>(idx[e]);
        else
            qoff = static_cast<uint32_t>(quantize(v[e], t, oow) - t.qlo);
        pk[e] = pack_code(qoff, v[e] < 0.0, false);
    }
}

}  // namespace bmq
