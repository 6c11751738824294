// device_common.cuh — device-side helpers shared by the codec, gate and
// engine kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "bmq_internal.hpp"

namespace bmq {

// ----------------------------------------------------------------- errors
// First device error wins; the host maps the code to the reference message.
enum DevErr : uint32_t {
    DE_NONE = 0,
    DE_NONFINITE = 1,
    DE_WINDOW = 2,
    DE_HDR_TRUNC = 10,
    DE_HDR_BOUND = 11,
    DE_HDR_TRAIL = 12,
    DE_SIGN_TRUNC = 13,
    DE_ZERO_TRUNC = 14,
    DE_TAG = 15,
    DE_PARTIAL = 16,
    DE_WIDTH0 = 17,
    DE_CODES_TRUNC = 18,
    DE_CODES_TRAIL = 19,
    DE_BOUND_MISMATCH = 20,
    DE_COUNT = 21,
    DE_CODE_WINDOW = 22,
    DE_POOL_FULL = 30,
    DE_TOO_LARGE = 31,
};

struct DevError {
    uint32_t code;
    uint32_t pad;
    uint64_t item;  // block index within the launch
};

__device__ __forceinline__ void dev_fail(DevError* e, uint32_t code, uint64_t item) {
    if (atomicCAS(&e->code, 0u, code) == 0u) e->item = item;
}

const char* dev_error_message(uint32_t code);
int dev_error_status(uint32_t code);

// Device allocations come from the device's stream-ordered memory pool with
// an unlimited release threshold, so simulators created back to back reuse
// the same HBM without cudaMalloc/cudaFree round trips.
void* dev_alloc(size_t bytes);
void dev_free(void* p);

// ------------------------------------------------------------ codec tables
struct DevTables {
    const uint64_t* thresh;   // thresh[q - qlo], q in [qlo, qhi + 1]
    const double* dequant;    // dequant[q - qlo], q in [qlo, qhi]
    int64_t qlo, qhi;
    int64_t idem_lo, idem_hi;
    double b_r;               // relative bound written into headers
    double inv_ba;            // 1 / b_a, estimate only
    double est_eps;           // bound on |estimate - log2(v)/b_a| (see quantize_estimate_x)
    // Single-precision estimate (quantize_pack_f32): 1 / b_a = fH + fL with
    // fH carrying 13 significant bits, so e * fH is exact in float for every
    // binary exponent e (|e| < 2^11); ftie = 0.5 - (its error bound).
    float fH, fL, finv, ftie;
    int32_t qlo32;            // qlo (fits: |q| < 2^31 whenever f32 is set)
    uint32_t f32;             // the float estimate is usable for this bound
};

// Device copy of host_tables(b_r) on the current device (cached).
const DevTables& device_tables(double b_r);

constexpr int kChunk = 4096;        // prescan chunk (bits) == scalars per chunk
constexpr int kChunkThreads = 128;  // one thread per bitmap word
constexpr int kWordsPerChunk = kChunk / 32;
constexpr int kHeaderBytes = 26;

// Exact reference quantiser q = llround(log2|v| / b_a) for finite v != 0.
// A float log2 estimate lands within +-1 of the true code; the table
// thresholds then settle it bit-exactly (see codec_tables.cpp).
struct QuantSearch {
    int64_t q;
    bool out_of_window;
};
// Out of line: the settling path of every quantiser variant is rare, and
// inlining its search loops into each call site bloats the hot kernels'
// instruction footprint.
static __device__ __noinline__ QuantSearch quantize_search(double v, const uint64_t* __restrict__ T, int64_t qlo,
                                                    int64_t qhi, double inv_ba) {
    const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(v)) & 0x7fffffffffffffffull;
    const uint32_t ex = static_cast<uint32_t>(bits >> 52);
    uint64_t man = bits & 0xfffffffffffffull;
    int e2;
    if (ex == 0) {  // subnormal: normalise the mantissa
        const int shift = __clzll(static_cast<long long>(man)) - 11;
        man = (man << shift) & 0xfffffffffffffull;
        e2 = -1022 - shift;
    } else {
        e2 = static_cast<int>(ex) - 1023;
    }
    const float m = __int_as_float(0x3f800000 | static_cast<int>(man >> 29));  // mantissa truncated to float
    const double x = (static_cast<double>(e2) + static_cast<double>(__log2f(m))) * inv_ba;
    int64_t q = __double2ll_rn(x);
    q = q < qlo ? qlo : (q > qhi ? qhi : q);
    int64_t i = q - qlo;
    while (bits < __ldg(T + i)) {
        if (i == 0) return QuantSearch{qlo, true};
        --i;
    }
    const int64_t last = qhi - qlo;  // T[last + 1] bounds the window from above
    while (bits >= __ldg(T + i + 1)) {
        if (i == last) return QuantSearch{qhi, true};
        ++i;
    }
    return QuantSearch{qlo + i, false};
}

// Exact reference quantiser q = llround(log2|v| / b_a) for finite v != 0.
// A float log2 estimate lands within +-1 of the true code; the table
// thresholds then settle it bit-exactly (see codec_tables.cpp).
__device__ __forceinline__ int64_t quantize(double v, const DevTables& t, bool& out_of_window) {
    const QuantSearch r = quantize_search(v, t.thresh, t.qlo, t.qhi, t.inv_ba);
    if (r.out_of_window) out_of_window = true;
    return r.q;
}

// x ~ log2|v| / b_a for finite v != 0 from a float log2 of the mantissa.
// __log2f on [1, 2) is within 2^-22.5 of log2, truncating the mantissa
// to float adds at most 2^-23 / ln 2, the double arithmetic a few ulp: the
// estimate is within est_eps = 1e-6 / b_a + 1e-6 of the reference's
// log2(v) / b_a (glibc log2 is within an ulp). Away from a half-integer by
// more than that, llround of the reference value is round(x) itself.
__device__ __forceinline__ double quantize_estimate_x(double v, const DevTables& t, uint64_t& bits) {
    bits = static_cast<uint64_t>(__double_as_longlong(v)) & 0x7fffffffffffffffull;
    const uint32_t ex = static_cast<uint32_t>(bits >> 52);
    uint64_t man = bits & 0xfffffffffffffull;
    int e2;
    if (ex == 0) {
        const int shift = __clzll(static_cast<long long>(man)) - 11;
        man = (man << shift) & 0xfffffffffffffull;
        e2 = -1022 - shift;
    } else {
        e2 = static_cast<int>(ex) - 1023;
    }
    const float m = __int_as_float(0x3f800000 | static_cast<int>(man >> 29));  // mantissa truncated to float
    return (static_cast<double>(e2) + static_cast<double>(__log2f(m))) * t.inv_ba;
}

// The estimate of quantize() for finite v != 0 (table index, not clamped
// against the exact thresholds yet) and |v|'s bit pattern.
__device__ __forceinline__ int64_t quantize_estimate(double v, const DevTables& t, uint64_t& bits) {
    bits = static_cast<uint64_t>(__double_as_longlong(v)) & 0x7fffffffffffffffull;
    const uint32_t ex = static_cast<uint32_t>(bits >> 52);
    uint64_t man = bits & 0xfffffffffffffull;
    int e2;
    if (ex == 0) {
        const int shift = __clzll(static_cast<long long>(man)) - 11;
        man = (man << shift) & 0xfffffffffffffull;
        e2 = -1022 - shift;
    } else {
        e2 = static_cast<int>(ex) - 1023;
    }
    const float m = __int_as_float(0x3f800000 | static_cast<int>(man >> 29));  // mantissa truncated to float
    const double x = (static_cast<double>(e2) + static_cast<double>(__log2f(m))) * t.inv_ba;
    int64_t q = __double2ll_rn(x);
    q = q < t.qlo ? t.qlo : (q > t.qhi ? t.qhi : q);
    return q - t.qlo;
}

// Read `width` (<= 63) bits LSB-first starting at bit `bitpos` of the byte
// stream at `base`. Reads aligned 32-bit words (buffers carry 16 B of slack).
__device__ __forceinline__ uint64_t read_bits(const uint8_t* base, uint64_t bitpos, uint32_t width) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(base) + (bitpos >> 3);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    const uint32_t sh = static_cast<uint32_t>((a & 3) * 8 + (bitpos & 7));
    const uint64_t lo = static_cast<uint64_t>(w[0]) | (static_cast<uint64_t>(w[1]) << 32);
    uint64_t v = lo >> sh;
    if (sh + width > 64) v |= static_cast<uint64_t>(w[2]) << (64 - sh);
    return width >= 64 ? v : (v & ((1ull << width) - 1));
}

__device__ __forceinline__ uint32_t load_u32_unaligned(const uint8_t* p) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    const uint32_t* w = reinterpret_cast<const uint32_t*>(a & ~uintptr_t(3));
    const uint32_t sh = static_cast<uint32_t>(a & 3) * 8;
    return sh ? (__ldg(w) >> sh) | (__ldg(w + 1) << (32 - sh)) : __ldg(w);
}

// Write an LSB-first bit stream src[0..nbits) (words beyond nbits zero) at
// byte dst, starting at bit `bit0` (< 8) of that byte. Interior 32-bit words
// are owned and stored; the first and last words may be shared with
// neighbouring segments of a zero-initialised region and are OR-ed in.
__device__ __forceinline__ void write_bits_block(uint8_t* dst, uint32_t bit0, const uint32_t* src,
                                                 uint64_t nbits, int tid, int nthreads) {
    if (nbits == 0) return;
    const uintptr_t a = reinterpret_cast<uintptr_t>(dst);
    uint32_t* w = reinterpret_cast<uint32_t*>(a & ~uintptr_t(3));
    const uint32_t s = static_cast<uint32_t>(a & 3) * 8 + bit0;
    const uint64_t nsrc = (nbits + 31) / 32;
    const uint64_t nout = (s + nbits + 31) / 32;
    for (uint64_t i = tid; i < nout; i += nthreads) {
        uint32_t v = 0;
        if (i < nsrc) v = src[i] << s;
        if (s && i > 0) v |= src[i - 1] >> (32 - s);
        if (i == 0 || i + 1 == nout)
            atomicOr(w + i, v);
        else
            w[i] = v;
    }
}

// pdep: scatter the low bits of x into the set bits of mask.
__device__ __forceinline__ uint64_t dev_deposit(uint64_t x, uint64_t mask) {
    uint64_t out = 0;
    while (mask) {
        const uint64_t low = mask & (~mask + 1);
        if (x & 1) out |= low;
        x >>= 1;
        mask ^= low;
    }
    return out;
}

// ----------------------------------------------------- codec block records
// Compress: per-block input descriptor and per-chunk / per-block plans.
struct CmpBlock {
    const double* in;   // planar scalars (read by the stats kernel)
    uint32_t* pk;       // packed codes of the block, one word per scalar
    uint64_t count;     // scalars in the block
    uint64_t id;        // engine block id (or index for the API)
};

// Packed per-scalar code word written by the quantiser (stats kernel or the
// fused gate epilogue) and read by emit:
//   pk = (q - qlo) << 2 | negative << 1 | zero      (q meaningful if !zero)
constexpr uint32_t kQOffMax = 0x3fffffffu;

__device__ __forceinline__ uint32_t pack_code(uint32_t qoff, bool neg, bool zero) {
    return (qoff << 2) | (neg ? 2u : 0u) | (zero ? 1u : 0u);
}

// Per-chunk counters, zero-initialised and combined with atomics (max / add)
// by the producers; the plan kernel turns them into tags and offsets.
struct ChunkPlan {
    uint32_t qmin_inv;   // max over nonzero scalars of kQOffMax - (q - qlo)
    uint32_t qmax_off;   // max over nonzero scalars of q - qlo
    uint32_t nnz;        // nonzero scalars
    uint32_t nneg;       // negative scalars
    uint32_t sign_off;   // byte offset of this chunk's raw sign bits in the payload
    uint32_t zero_off;   // byte offset of this chunk's raw zero bits
    uint32_t nz_prefix;  // nonzero scalars before this chunk in the block
    uint8_t stag, ztag, pad0, pad1;
};

struct BlockPlan {
    uint64_t size;          // payload bytes
    uint64_t out_off;       // offset in the output region (~0 = virtual ALL_ZERO)
    int64_t code_min;
    uint64_t code_seg;      // byte offset of the codes segment
    uint64_t nnz;
    uint32_t width;
    uint32_t flags;         // 1 = ALL_ZERO
    int64_t code_max;
    uint64_t ztag_off;      // byte offset of the zero-bitmap tags
    uint32_t ntag;          // tag bytes per bitmap
    uint32_t nch;           // chunks
    double sumsq;           // sum of dequantised squares (norm)
    double sum_re, sum_im;  // sums of dequantised real / imaginary parts
};

// Decompress: per-block descriptor and per-chunk decode plan.
struct DecBlock {
    const uint8_t* in;
    uint64_t size;
    double* out;
    uint64_t expect_count;  // 0 = any
};

struct DecChunk {
    uint32_t sign_off, zero_off;  // raw byte offsets (valid when tag == 2)
    uint32_t nz_prefix;
    uint8_t stag, ztag, pad0, pad1;
};

// Row index of a batch for decoding straight into a gate pass (mode 3 of
// launch_decompress): one record per 32-scalar bitmap word in the planar
// layout of the work buffer (word w covers planar scalars 32 w .. 32 w + 31).
struct DecRow {
    uint32_t nz;    // bit i: scalar i nonzero
    uint32_t sign;  // bit i: scalar i negative
    uint32_t rank;  // codes before this word in its block (the first nonzero's rank)
    uint32_t pad;
};

// Code-domain stages (mode 1 of launch_decompress with a PermSrc array): one
// record per (block slot, chunk). A zero-free full chunk of all-positive or
// all-negative scalars whose codes are at most 16 bits wide and inside the
// idempotent window is not decoded to packed words; the first permutation
// pass reads its codes from the payload through this record instead (meta
// bit 12 set): scalar s of the chunk has rank s, so its code sits at bit
// (meta & 63) + s * width of cw.
struct __align__(16) PermSrc {
    const uint64_t* cw;  // 8-byte aligned base of the chunk's codes
    uint32_t qb;         // packed offset of code 0 (code_min - qlo)
    uint32_t meta;       // bits 0-5: bit offset, 6-10: width, 11: negative, 12: read from the payload,
                         // 13: all-zero chunk (not written; read as zero words)
};

struct DecInfo {
    uint64_t count;
    int64_t code_min;
    uint64_t code_seg;
    uint32_t width;
    uint32_t flags;   // 1 = all zero, 2 = error
    double sumsq;
    double sum_re, sum_im;
};

}  // namespace bmq

#define BMQ_CUDA(call)                                                                        \
    do {                                                                                      \
        cudaError_t err__ = (call);                                                           \
        if (err__ != cudaSuccess)                                                             \
            ::bmq::raise(err__ == cudaErrorMemoryAllocation ? BMQ_ERR_OUT_OF_MEMORY : BMQ_ERR_CUDA, \
                         std::string("CUDA error: ") + cudaGetErrorString(err__) + " at " #call); \
    } while (0)
