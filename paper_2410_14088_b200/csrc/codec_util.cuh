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

// quantize_pack with every step in registers: a scalar whose estimate x
// lies farther than est_eps from a half-integer (inside the table window)
// takes round(x) directly; the others (about 2 est_eps of them) probe both
// neighbouring thresholds and settle exactly, and an estimate off by more
// than one falls back to quantize(). qlo_d = (double) t.qlo, span = qhi - qlo.
__device__ __forceinline__ uint32_t quantize_pack_fast(double v, const DevTables& t, double qlo_d, int span,
                                                       bool& bad, bool& oow) {
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(v)) & 0x7fffffffffffffffull;
    if (bits - 1 >= 0x7fefffffffffffffull) {  // +-0 (wraps), inf or NaN
        if (bits) bad = true;
        return 1u;
    }
    // normal numbers here; a subnormal (ex == 0) is settled by the exact search
    const uint32_t ex = static_cast<uint32_t>(bits >> 52);
    const float m = __int_as_float(0x3f800000 | static_cast<int>((bits >> 29) & 0x7fffffu));  // (see quantize_estimate_x)
    const double x = (static_cast<double>(static_cast<int>(ex) - 1023) + static_cast<double>(__log2f(m))) * t.inv_ba;
    const double r = rint(x);
    const int i = __double2int_rz(r - qlo_d);  // exact (integers below 2^53); saturates
    uint32_t qoff = static_cast<uint32_t>(min(max(i, 0), span));
    if (!(ex != 0 && 0.5 - fabs(x - r) > t.est_eps && static_cast<unsigned>(i) <= static_cast<unsigned>(span))) {
        const uint64_t lo = __ldg(t.thresh + qoff), hi = __ldg(t.thresh + qoff + 1);
        if (!(bits >= lo && bits < hi)) qoff = static_cast<uint32_t>(quantize(v, t, oow) - t.qlo);
    }
    return pack_code(qoff, v < 0.0, false);
}

// The exact settling of quantize_pack_fast for a scalar whose estimate is
// near a half-integer or outside the window (about 2 est_eps of them):
// probe the two neighbouring thresholds, else search.
__device__ __forceinline__ uint32_t quantize_settle(double v, uint64_t bits, int qoff, int span, const DevTables& t,
                                                 bool& oow) {
    uint32_t qo = static_cast<uint32_t>(min(max(qoff, 0), span));
    const uint64_t lo = __ldg(t.thresh + qo), hi = __ldg(t.thresh + qo + 1);
    if (!(bits >= lo && bits < hi)) qo = static_cast<uint32_t>(quantize(v, t, oow) - t.qlo);
    return qo;
}

// quantize_pack_fast with a single-precision estimate (t.f32): with
// v = m 2^e (m in [1, 2)), log2|v| / b_a = e fH + e fL + log2(m) / b_a where
// e fH is exact in float, so q = floor(e fH) + rint(s) for
// s = log2(m) finv + (e fL + frac(e fH)) whenever s lies more than
// 0.5 - ftie from a half-integer (DevTables::ftie, codec_cmp.cu). Zeros,
// subnormals, infinities and NaNs leave through one unsigned range test.
__device__ __forceinline__ float lg2_approx(float m) {
    float r;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(m));
    return r;
}
__device__ __forceinline__ uint32_t quantize_pack_f32(double v, const DevTables& t, int span, bool& bad, bool& oow) {
    const uint32_t hi = static_cast<uint32_t>(__double2hiint(v)), lo = static_cast<uint32_t>(__double2loint(v));
    const uint32_t ahi = hi & 0x7fffffffu;
    if (ahi - 0x00100000u >= 0x7fe00000u) [[unlikely]] {  // not a normal number
        if (ahi >= 0x7ff00000u) {
            bad = true;
            return 1u;
        }
        if ((ahi | lo) == 0u) return 1u;
        return pack_code(static_cast<uint32_t>(quantize(v, t, oow) - t.qlo), (hi >> 31) != 0u, false);
    }
    const float ef = static_cast<float>(static_cast<int>(ahi >> 20) - 1023);
    const float m = __int_as_float(0x3f800000 | (__funnelshift_l(lo, ahi, 3) & 0x7fffffu));
    const float P = __fmul_rn(ef, t.fH);  // exact
    const float Pi = floorf(P);
    const float u = __fmaf_rn(ef, t.fL, __fsub_rn(P, Pi));
    const float s = __fmaf_rn(lg2_approx(m), t.finv, u);
    const float r = rintf(s);
    const int qoff = __float2int_rz(Pi) + __float2int_rz(r) - t.qlo32;
    uint32_t qo = static_cast<uint32_t>(qoff);
    if (!(fabsf(__fsub_rn(s, r)) < t.ftie && qo <= static_cast<uint32_t>(span))) [[unlikely]]
        qo = quantize_settle(v, (static_cast<uint64_t>(ahi) << 32) | lo, qoff, span, t, oow);
    return (qo << 2) | ((hi >> 30) & 2u);
}

// The branch-free part of quantize_pack_f32: the packed word when the
// estimate decides it (a normal number away from a rounding tie, inside the
// window) or when v is +-0; otherwise `need` is set and the caller settles
// the scalar with quantize_pack_fast (zeros, subnormals, infinities, NaNs,
// ties: the exact reference decision). Callers batch several scalars and
// take the (rare) settling path once per batch.
__device__ __forceinline__ uint32_t quant_est_f32(double v, const DevTables& t, int span, bool& need) {
    const uint32_t hi = static_cast<uint32_t>(__double2hiint(v)), lo = static_cast<uint32_t>(__double2loint(v));
    const uint32_t ahi = hi & 0x7fffffffu;
    const bool normal = ahi - 0x00100000u < 0x7fe00000u;
    const float ef = static_cast<float>(static_cast<int>(ahi >> 20) - 1023);
    const float m = __int_as_float(0x3f800000 | (__funnelshift_l(lo, ahi, 3) & 0x7fffffu));
    const float P = __fmul_rn(ef, t.fH);  // exact
    const float Pi = floorf(P);
    const float u = __fmaf_rn(ef, t.fL, __fsub_rn(P, Pi));
    const float s = __fmaf_rn(lg2_approx(m), t.finv, u);
    const float r = rintf(s);
    const uint32_t qo = static_cast<uint32_t>(__float2int_rz(Pi) + __float2int_rz(r) - t.qlo32);
    const bool zero = (ahi | lo) == 0u;
    need = !zero && !(normal && fabsf(__fsub_rn(s, r)) < t.ftie && qo <= static_cast<uint32_t>(span));
    return zero ? 1u : ((qo << 2) | ((hi >> 30) & 2u));
}

// Per-thread counters of one chunk over packed words, reduced per warp with
// REDUX at the flush (ChunkAcc's fields, cheaper per scalar):
//   mn = min over words of (pk ^ 1) - 1  (a zero word 1 -> 0xffffffff, else pk)
//   mx = max over words of pk            (a zero word 1 never exceeds a code)
//   zn = zero words + (negative words << 16)
struct RowAcc {
    uint32_t mn = ~0u, mx = 0, zn = 0;
    __device__ __forceinline__ void add(uint32_t pk) {
        mn = min(mn, (pk ^ 1u) - 1u);
        mx = max(mx, pk);
        zn += (pk & 1u) | ((pk & 2u) << 15);
    }
};

// Warp flush of RowAcc over `scalars` words (all 32 lanes call, same cp).
__device__ __forceinline__ void flush_rows(ChunkPlan* cp, const RowAcc& a, uint32_t scalars) {
    const uint32_t mn = __reduce_min_sync(0xffffffffu, a.mn), mx = __reduce_max_sync(0xffffffffu, a.mx);
    const uint32_t zn = __reduce_add_sync(0xffffffffu, a.zn);
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nnz = scalars - (zn & 0xffffu), nneg = zn >> 16;
    if (lane < 4u && nnz) {
        if (lane == 0) atomicMax(&cp->qmin_inv, kQOffMax - (mn >> 2));
        else if (lane == 1) atomicMax(&cp->qmax_off, mx >> 2);
        else if (lane == 2) atomicAdd(&cp->nnz, nnz);
        else if (nneg) atomicAdd(&cp->nneg, nneg);
    } else if (lane == 3u && nneg) {
        atomicAdd(&cp->nneg, nneg);
    }
}

}  // namespace bmq
