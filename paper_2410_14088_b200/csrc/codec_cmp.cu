// codec_cmp.cu — byte-exact device compressor (compress_block,
// codec.hpp:227-295; prescan_encode, bitmap.hpp:109-145) for batches of
// blocks, plus the codec tables, error messages and device allocator.
//
// Work decomposition: one CTA of 128 threads per 4096-scalar chunk, which is
// exactly one prescan chunk of each bitmap (bitmap.hpp:76). Warp w, step j
// handles scalars 128 j + 32 w + lane, so global loads/stores are coalesced
// and a warp ballot yields bitmap word 4 j + w directly (the paper's warp
// ballot pre-scan).
//
// Compress = quantise (k_cmp_stats, or fused into the stage's last gate pass):
//              packed code word per scalar + per-chunk counters
//          -> plan  (per block: code_min, width, tags, segment offsets, size)
//          -> alloc (exclusive scan of sizes into the output region)
//          -> zero  (clear the region so shared edge words can be OR-ed)
//          -> emit  (header, tags, raw mixed chunks, LSB-first codes) from the
//                    packed words — no second quantisation.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <cfloat>
#include <climits>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>

#include "codec.cuh"
#include "codec_util.cuh"

namespace bmq {

// --------------------------------------------------------------- messages
const char* dev_error_message(uint32_t code) {
    switch (code) {
    case DE_NONFINITE: return "input scalars must be finite";
    case DE_WINDOW: return "scalar magnitude outside the quantiser table window of this error bound";
    case DE_HDR_TRUNC: return "header truncated";
    case DE_HDR_BOUND: return "header: invalid relative error bound";
    case DE_HDR_TRAIL: return "header: trailing bytes after payload";
    case DE_SIGN_TRUNC: return "sign bitmap truncated";
    case DE_ZERO_TRUNC: return "zero bitmap truncated";
    case DE_TAG: return "bitmap tag stream corrupt: invalid chunk tag";
    case DE_PARTIAL: return "bitmap final partial chunk must be stored raw";
    case DE_WIDTH0: return "codes: width zero with nonzero scalars present";
    case DE_CODES_TRUNC: return "codes truncated";
    case DE_CODES_TRAIL: return "codes: trailing bytes after payload";
    case DE_BOUND_MISMATCH: return "header: relative bound differs from the decoder tables";
    case DE_COUNT: return "block payload scalar count does not match the layout";
    case DE_CODE_WINDOW: return "codes: decoded code outside the dequantisation table";
    case DE_POOL_FULL: return "device payload pool exhausted";
    case DE_TOO_LARGE: return "payload scalar count exceeds the launch geometry";
    default: return "unknown device error";
    }
}

int dev_error_status(uint32_t code) {
    if (code == DE_COUNT) return BMQ_ERR_ENGINE;
    if (code == DE_POOL_FULL) return BMQ_ERR_STORE;
    return BMQ_ERR_CODEC;
}

// ------------------------------------------------------------- allocation
void* dev_alloc(size_t bytes) {
    int dev = 0;
    BMQ_CUDA(cudaGetDevice(&dev));
    static std::mutex mu;
    static bool configured[64] = {};
    {
        std::lock_guard<std::mutex> lock(mu);
        if (dev < 64 && !configured[dev]) {
            cudaMemPool_t pool;
            BMQ_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
            uint64_t thr = ~0ull;
            BMQ_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
            configured[dev] = true;
        }
    }
    void* p = nullptr;
    BMQ_CUDA(cudaMallocAsync(&p, bytes, cudaStreamPerThread));
    BMQ_CUDA(cudaStreamSynchronize(cudaStreamPerThread));
    return p;
}

void dev_free(void* p) {
    if (!p) return;
    cudaDeviceSynchronize();
    cudaFreeAsync(p, cudaStreamPerThread);
    cudaStreamSynchronize(cudaStreamPerThread);
}

// ------------------------------------------------------------------ tables
const DevTables& device_tables(double b_r) {
    static std::mutex mu;
    static std::map<std::pair<int, uint64_t>, DevTables> cache;
    const CodecTables& h = host_tables(b_r);
    int dev = 0;
    BMQ_CUDA(cudaGetDevice(&dev));
    uint64_t key;
    std::memcpy(&key, &b_r, 8);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({dev, key});
    if (it != cache.end()) return it->second;
    if (static_cast<uint64_t>(h.qhi - h.qlo) >= kQOffMax)
        raise(BMQ_ERR_INVALID_ARGUMENT, "error bound too small for the device code window");
    DevTables t{};
    uint64_t* th = nullptr;
    double* dq = nullptr;
    BMQ_CUDA(cudaMalloc(&th, h.thresh.size() * sizeof(uint64_t)));
    BMQ_CUDA(cudaMalloc(&dq, h.dequant.size() * sizeof(double)));
    BMQ_CUDA(cudaMemcpy(th, h.thresh.data(), h.thresh.size() * sizeof(uint64_t), cudaMemcpyHostToDevice));
    BMQ_CUDA(cudaMemcpy(dq, h.dequant.data(), h.dequant.size() * sizeof(double), cudaMemcpyHostToDevice));
    t.thresh = th;
    t.dequant = dq;
    t.qlo = h.qlo;
    t.qhi = h.qhi;
    t.idem_lo = h.idem_lo;
    t.idem_hi = h.idem_hi;
    t.b_r = h.b_r;
    t.inv_ba = 1.0 / h.b_a;
    t.est_eps = 1e-6 * t.inv_ba + 1e-6;
    {
        // quantize_pack_f32: x = e * inv_ba + lg * inv_ba with e * fH exact,
        // u = e * fL + frac(e * fH), s = lg * finv + u, q = floor(e * fH) + rint(s).
        // Error of s against log2|v| / b_a - floor(e * fH): the double estimate's
        // bound (lg2 approximation, mantissa truncation, reference rounding),
        // finv's rounding (lg < 1), fL's rounding times |e| <= 1074, and one
        // ulp for each of the two float FMAs.
        int ex = 0;
        const double f = std::frexp(t.inv_ba, &ex);
        const double H = std::ldexp(std::nearbyint(std::ldexp(f, 13)), ex - 13);
        const double L = t.inv_ba - H;
        const auto ulp32 = [](double z) { return std::ldexp(1.0, std::ilogb(std::max(z, 1e-30)) - 23); };
        const double umax = 1.0 + 1074.0 * std::fabs(L), smax = umax + t.inv_ba + 1.0;
        const double eps = t.est_eps + t.inv_ba * 0x1p-24 + 1074.0 * std::fabs(L) * 0x1p-24 + ulp32(umax) + ulp32(smax);
        t.fH = static_cast<float>(H);
        t.fL = static_cast<float>(L);
        t.finv = static_cast<float>(t.inv_ba);
        float tie = static_cast<float>(0.5 - eps);
        if (static_cast<double>(tie) > 0.5 - eps) tie = std::nextafter(tie, 0.0f);
        t.ftie = tie;
        t.qlo32 = static_cast<int32_t>(std::max<int64_t>(h.qlo, INT32_MIN));
        t.f32 = (eps < 0.05 && static_cast<double>(t.fH) == H && h.qlo >= -(1ll << 30) && h.qhi <= (1ll << 30)) ? 1u : 0u;
    }
    return cache.emplace(std::make_pair(dev, key), t).first->second;
}

namespace {

// ---------------------------------------------------------------- stats
// Quantise one chunk: packed code words + per-chunk counters.
__global__ void __launch_bounds__(kChunkThreads) k_cmp_stats(const CmpBlock* __restrict__ blks, uint32_t nch_max,
                                                             ChunkPlan* __restrict__ cps, DevTables t,
                                                             DevError* err) {
    const uint32_t bi = blockIdx.x / nch_max, c = blockIdx.x % nch_max;
    const CmpBlock blk = blks[bi];
    const uint64_t nch = (blk.count + kChunk - 1) / kChunk;
    if (c >= nch) return;
    const uint32_t len = chunk_len(blk.count, c);
    const double* src = blk.in + static_cast<uint64_t>(c) * kChunk;
    uint32_t* dst = blk.pk + static_cast<uint64_t>(c) * kChunk;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    RowAcc acc;
    bool bad = false, oow = false;
    const double qlo_d = static_cast<double>(t.qlo);
    const int span = static_cast<int>(t.qhi - t.qlo);
    if (len == kChunk) {  // full chunk: every lane holds a word in every row
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
            const uint32_t s = 128 * j + 32 * w + lane;
            const double v = __ldg(src + s);
            const uint32_t pk = t.f32 ? quantize_pack_f32(v, t, span, bad, oow)
                                      : quantize_pack_fast(v, t, qlo_d, span, bad, oow);
            dst[s] = pk;
            acc.add(pk);
        }
    } else {
        for (int j = 0; j < 32; ++j) {
            const uint32_t s = 128 * j + 32 * w + lane;
            if (s < len) {
                const uint32_t pk = quantize_pack_fast(__ldg(src + s), t, qlo_d, span, bad, oow);
                dst[s] = pk;
                acc.add(pk);
            }
        }
    }
    if (bad) dev_fail(err, DE_NONFINITE, bi);
    if (oow) dev_fail(err, DE_WINDOW, bi);
    // words this warp quantised (a lane past len adds none: RowAcc's identity)
    uint32_t mine = 0;
    for (int j = 0; j < 32; ++j) mine += (128u * j + 32u * w) < len ? min(32u, len - (128u * j + 32u * w)) : 0u;
    flush_rows(cps + static_cast<uint64_t>(bi) * nch_max + c, acc, mine);
}

// ----------------------------------------------------------------- plan
// One CTA per block: reduce chunk counters, derive tags, lay out segments.
constexpr int kPlanThreads = 256;

__device__ __forceinline__ uint8_t tag_of(uint32_t ones, uint32_t len) {
    if (len < kChunk) return 2;  // a partial chunk is always stored raw
    return ones == 0 ? 0 : (ones == len ? 1 : 2);
}

__global__ void __launch_bounds__(kPlanThreads) k_cmp_plan(const CmpBlock* __restrict__ blks, uint32_t nch_max,
                                                           ChunkPlan* __restrict__ cps, BlockPlan* __restrict__ bps,
                                                           int64_t qlo) {
    const uint32_t bi = blockIdx.x;
    const CmpBlock blk = blks[bi];
    const uint32_t nch = static_cast<uint32_t>((blk.count + kChunk - 1) / kChunk);
    ChunkPlan* cp = cps + static_cast<uint64_t>(bi) * nch_max;
    using ReduceU = cub::BlockReduce<unsigned long long, kPlanThreads>;
    using Scan = cub::BlockScan<unsigned long long, kPlanThreads>;
    __shared__ typename ReduceU::TempStorage rs;
    __shared__ typename Scan::TempStorage ss;
    __shared__ unsigned long long s_tot[5];
    // pass 1: totals
    unsigned long long mninv = 0, mx = 0, nnz = 0, sraw = 0, zraw = 0;
    for (uint32_t c = threadIdx.x; c < nch; c += kPlanThreads) {
        const ChunkPlan p = cp[c];
        const uint32_t len = chunk_len(blk.count, c);
        if (p.nnz) {
            mninv = max(mninv, static_cast<unsigned long long>(p.qmin_inv));
            mx = max(mx, static_cast<unsigned long long>(p.qmax_off));
        }
        nnz += p.nnz;
        if (tag_of(p.nneg, len) == 2) sraw += (len + 7) / 8;
        if (tag_of(len - p.nnz, len) == 2) zraw += (len + 7) / 8;
    }
    const unsigned long long r0 = ReduceU(rs).Reduce(mninv, cub::Max());
    __syncthreads();
    const unsigned long long r1 = ReduceU(rs).Reduce(mx, cub::Max());
    __syncthreads();
    const unsigned long long r2 = ReduceU(rs).Sum(nnz);
    __syncthreads();
    const unsigned long long r3 = ReduceU(rs).Sum(sraw);
    __syncthreads();
    const unsigned long long r4 = ReduceU(rs).Sum(zraw);
    if (threadIdx.x == 0) {
        s_tot[0] = r0;
        s_tot[1] = r1;
        s_tot[2] = r2;
        s_tot[3] = r3;
        s_tot[4] = r4;
    }
    __syncthreads();
    const uint64_t qmin_off = kQOffMax - s_tot[0], qmax_off = s_tot[1], total_nnz = s_tot[2];
    const uint32_t ntag = (nch + 3) / 4;
    const uint64_t ztag_off = kHeaderBytes + ntag + s_tot[3];
    const uint64_t code_seg = ztag_off + ntag + s_tot[4];
    uint32_t width = 0;
    if (total_nnz) {
        const uint64_t range = qmax_off - qmin_off;
        width = range ? 64 - __clzll(static_cast<long long>(range)) : 1;
    }
    // pass 2: tags and per-chunk offsets (exclusive scans in chunk order)
    unsigned long long carry_s = 0, carry_z = 0, carry_n = 0;
    for (uint32_t base = 0; base < nch; base += kPlanThreads) {
        const uint32_t c = base + threadIdx.x;
        unsigned long long vs = 0, vz = 0, vn = 0;
        ChunkPlan p{};
        if (c < nch) {
            p = cp[c];
            const uint32_t len = chunk_len(blk.count, c);
            p.stag = tag_of(p.nneg, len);
            p.ztag = tag_of(len - p.nnz, len);
            vs = p.stag == 2 ? (len + 7) / 8 : 0;
            vz = p.ztag == 2 ? (len + 7) / 8 : 0;
            vn = p.nnz;
        }
        unsigned long long ps, pz, pn, ts, tz, tn;
        Scan(ss).ExclusiveSum(vs, ps, ts);
        __syncthreads();
        Scan(ss).ExclusiveSum(vz, pz, tz);
        __syncthreads();
        Scan(ss).ExclusiveSum(vn, pn, tn);
        __syncthreads();
        if (c < nch) {
            p.sign_off = static_cast<uint32_t>(kHeaderBytes + ntag + carry_s + ps);
            p.zero_off = static_cast<uint32_t>(ztag_off + ntag + carry_z + pz);
            p.nz_prefix = static_cast<uint32_t>(carry_n + pn);
            cp[c] = p;
        }
        carry_s += ts;
        carry_z += tz;
        carry_n += tn;
    }
    if (threadIdx.x == 0) {
        BlockPlan bp{};
        bp.nch = nch;
        bp.ntag = ntag;
        bp.nnz = total_nnz;
        if (total_nnz == 0) {
            bp.flags = 1;
            bp.size = kHeaderBytes;
        } else {
            bp.code_min = qlo + static_cast<int64_t>(qmin_off);
            bp.code_max = qlo + static_cast<int64_t>(qmax_off);
            bp.width = width;
            bp.ztag_off = ztag_off;
            bp.code_seg = code_seg;
            bp.size = code_seg + (total_nnz * width + 7) / 8;
        }
        bps[bi] = bp;
    }
}

// ---------------------------------------------------------------- alloc
// Single CTA: exclusive scan of payload sizes into [cursor[0], cursor[0] + total);
// cursor[1] receives total, whether or not it fits.
// virtual_zero: ALL_ZERO payloads take no space (engine pools); they are
// materialised as the canonical 26-byte header on read.
constexpr int kAllocThreads = 1024;

// Payloads are placed at multiples of `align` (16 in engine arenas, so they
// can be moved with 16-byte copies; 1 for back-to-back API output). Nothing
// is written when the region would overflow `cap` (DE_POOL_FULL): the caller
// makes room and launches the allocation again.
__global__ void __launch_bounds__(kAllocThreads) k_cmp_alloc(const CmpBlock* __restrict__ blks, uint64_t nblk,
                                                             BlockPlan* __restrict__ bps, uint64_t* cursor,
                                                             uint64_t cap, uint64_t* range, int virtual_zero,
                                                             uint32_t align, uint64_t* meta_off,
                                                             uint64_t* meta_size, uint64_t meta_base,
                                                             uint64_t meta_tag, DevError* err) {
    using Scan = cub::BlockScan<unsigned long long, kAllocThreads>;
    using Reduce = cub::BlockReduce<unsigned long long, kAllocThreads>;
    __shared__ typename Scan::TempStorage ss;
    __shared__ typename Reduce::TempStorage rs;
    __shared__ bool s_fits;
    const uint64_t start = *cursor;
    const auto placed = [&](uint64_t i) -> unsigned long long {
        const BlockPlan& p = bps[i];
        if (virtual_zero && (p.flags & 1)) return 0;
        return (p.size + align - 1) / align * align;
    };
    unsigned long long part = 0;
    for (uint64_t i = threadIdx.x; i < nblk; i += kAllocThreads) part += placed(i);
    const unsigned long long total = Reduce(rs).Sum(part);
    if (threadIdx.x == 0) {
        cursor[1] = total;  // bytes the batch needs (read back after DE_POOL_FULL)
        s_fits = start + total <= cap;
        if (!s_fits) {
            dev_fail(err, DE_POOL_FULL, 0);
            range[0] = range[1] = start;
        } else {
            range[0] = start;
            range[1] = start + total;
            *cursor = start + total;
        }
    }
    __syncthreads();
    if (!s_fits) return;
    unsigned long long carry = 0;
    for (uint64_t base = 0; base < nblk; base += kAllocThreads) {
        const uint64_t i = base + threadIdx.x;
        const unsigned long long sz = i < nblk ? placed(i) : 0;
        unsigned long long pre, tot;
        Scan(ss).ExclusiveSum(sz, pre, tot);
        __syncthreads();
        if (i < nblk) {
            BlockPlan& p = bps[i];
            const bool virt = virtual_zero && (p.flags & 1);
            p.out_off = virt ? ~0ull : start + carry + pre;
            if (meta_off) {  // metadata may point into another arena (staged host spill)
                const uint64_t id = blks[i].id;
                meta_off[id] = virt ? ~0ull : ((meta_base + p.out_off) | meta_tag);
                meta_size[id] = p.size;
            }
        }
        carry += tot;
    }
}

// ----------------------------------------------------------- edge zeroing
// The emit stores every payload byte outright except the first and last
// 32-bit word of each bit segment it writes (sign / zero raw bitmaps, a
// chunk's code stream): neighbouring segments share those and OR into them
// (write_bits_block). Zeroing just those words before the emit replaces a
// zeroing pass over the whole output. out == nullptr: out_off are addresses.
__device__ __forceinline__ void zero_seg_edges(uint8_t* dst, uint32_t bit0, uint64_t nbits) {
    if (nbits == 0) return;
    const uintptr_t a = reinterpret_cast<uintptr_t>(dst);
    uint32_t* w = reinterpret_cast<uint32_t*>(a & ~uintptr_t(3));
    const uint32_t s = static_cast<uint32_t>(a & 3) * 8 + bit0;
    const uint64_t nout = (s + nbits + 31) / 32;
    w[0] = 0;
    w[nout - 1] = 0;
}

__global__ void k_zero_edges(const CmpBlock* __restrict__ blks, uint32_t nch_max, const ChunkPlan* __restrict__ cps,
                             const BlockPlan* __restrict__ bps, uint8_t* out, uint64_t nblk, const DevError* err) {
    const uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (t >= nblk * nch_max || err->code) return;
    const uint64_t bi = t / nch_max;
    const uint32_t c = static_cast<uint32_t>(t % nch_max);
    const BlockPlan bp = bps[bi];
    if (bp.out_off == ~0ull || (bp.flags & 1) || c >= bp.nch) return;
    const ChunkPlan p = cps[t];
    const uint32_t len = chunk_len(blks[bi].count, c);
    if (p.nnz == 0 && len == kChunk) return;  // tags only
    uint8_t* pay = reinterpret_cast<uint8_t*>(reinterpret_cast<uintptr_t>(out) + bp.out_off);
    const uint32_t raw_bits = ((len + 7) / 8) * 8;
    if (p.stag == 2) zero_seg_edges(pay + p.sign_off, 0, raw_bits);
    if (p.ztag == 2) zero_seg_edges(pay + p.zero_off, 0, raw_bits);
    const uint64_t start_bit = static_cast<uint64_t>(p.nz_prefix) * bp.width;
    zero_seg_edges(pay + bp.code_seg + (start_bit >> 3), static_cast<uint32_t>(start_bit & 7),
                   static_cast<uint64_t>(p.nnz) * bp.width);
}

// ----------------------------------------------------------------- emit
constexpr int kStageWords = (kChunk * 30 + 31) / 32 + 2;  // codes are < 2^30 (kQOffMax)

// The scalar part of emit for one chunk (kFull: all 4096 scalars valid).
struct EmitSmem {
    uint32_t sign[kWordsPerChunk], zero[kWordsPerChunk], pre[kWordsPerChunk], bits[kWordsPerChunk];
    union {                      // cw is read into registers before stage is zeroed and packed
        uint32_t cw[kChunk];     // nonzero codes of word k at cw[32 k + rank in word]
        uint32_t stage[kStageWords];
    };
};

template <bool kFull, bool kW1>
__device__ __forceinline__ void emit_chunk(const ChunkPlan& p, uint32_t len, const uint32_t* __restrict__ src,
                                           const BlockPlan& bp, uint8_t* pay, const DevTables& t, EmitSmem& sm) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t w_bits = bp.width;
    const uint32_t qmin_off = static_cast<uint32_t>(bp.code_min - t.qlo);
    const uint64_t code_bits = static_cast<uint64_t>(p.nnz) * w_bits;
    const uint32_t nstage = static_cast<uint32_t>((code_bits + 31) / 32);
    const uint32_t lt = (1u << lane) - 1;
    if (kW1 && kFull && p.nnz == kChunk) {
        // every code one bit, no zeros: the sign bitmap and the code stream
        // are two ballots per word (no zero bitmap, no prefix)
        uint32_t pkv[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) pkv[j] = __ldcs(src + 128 * j + 32 * w + lane);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t k = 4 * j + w;
            const uint32_t sw = __ballot_sync(0xffffffffu, (pkv[j] >> 1) & 1u);
            const uint32_t bw = __ballot_sync(0xffffffffu, (((pkv[j] >> 2) - qmin_off) & 1u) != 0);
            if (lane == 0) {
                sm.sign[k] = sw;
                sm.bits[k] = bw;
            }
        }
        __syncthreads();
        if (p.stag == 2) write_bits_block(pay + p.sign_off, 0, sm.sign, kChunk, tid, kChunkThreads);
        const uint64_t start_bit = static_cast<uint64_t>(p.nz_prefix);
        write_bits_block(pay + bp.code_seg + (start_bit >> 3), static_cast<uint32_t>(start_bit & 7), sm.bits,
                         kChunk, tid, kChunkThreads);
        return;
    }
    if (!kW1 && kFull && p.nnz == kChunk) {
        // no zero in the chunk: scalar s has rank s, so word k's codes start
        // at stage bit 32 k w (no compaction, no prefix scan, no zero bitmap)
        uint32_t pkv[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) pkv[j] = __ldcs(src + 128 * j + 32 * w + lane);
        for (uint32_t i = tid; i < nstage; i += kChunkThreads) sm.stage[i] = 0;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t k = 4 * j + w;
            const uint32_t pk = pkv[j];
            const uint32_t sw = __ballot_sync(0xffffffffu, (pk >> 1) & 1u);
            if (lane == 0) sm.sign[k] = sw;
            const uint32_t code = (pk >> 2) - qmin_off;
            const uint32_t pbit = (32u * k + lane) * w_bits, wi = pbit >> 5, sh = pbit & 31;
            if (code) {
                atomicOr(&sm.stage[wi], code << sh);
                if (sh + w_bits > 32) atomicOr(&sm.stage[wi + 1], code >> (32 - sh));
            }
        }
        __syncthreads();
        if (p.stag == 2) write_bits_block(pay + p.sign_off, 0, sm.sign, kChunk, tid, kChunkThreads);
        const uint64_t start_bit = static_cast<uint64_t>(p.nz_prefix) * w_bits;
        write_bits_block(pay + bp.code_seg + (start_bit >> 3), static_cast<uint32_t>(start_bit & 7), sm.stage,
                         code_bits, tid, kChunkThreads);
        return;
    }
    // A: all loads in flight; B: ballots -> bitmap words, width-1 code words,
    // or (wider codes) the nonzero codes compacted per word into sm.cw
    {
        uint32_t pkv[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t s = 128 * j + 32 * w + lane;
            pkv[j] = (kFull || s < len) ? __ldcs(src + s) : 1u;
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t k = 4 * j + w;
            const uint32_t pk = pkv[j];
            const uint32_t code = (pk >> 2) - qmin_off;
            const uint32_t sw = __ballot_sync(0xffffffffu, (pk >> 1) & 1u);
            const uint32_t zw = __ballot_sync(0xffffffffu, pk & 1u) & (kFull ? ~0u : word_mask(len, k));
            const uint32_t nzw = ~zw & (kFull ? ~0u : word_mask(len, k));
            if constexpr (kW1) {
                const uint32_t bw = __ballot_sync(0xffffffffu, !(pk & 1u) && (code & 1u));
                if (nzw != ~0u && !(pk & 1u)) sm.cw[32 * k + __popc(nzw & lt)] = code;
                if (lane == 0) sm.bits[k] = bw;
            } else {
                if (!(pk & 1u)) sm.cw[32 * k + __popc(nzw & lt)] = code;
            }
            if (lane == 0) {
                sm.sign[k] = sw;
                sm.zero[k] = zw;
            }
        }
    }
    __syncthreads();
    // nonzero prefix over the 128 words in scalar order
    {
        using Scan = cub::BlockScan<uint32_t, kChunkThreads>;
        __shared__ typename Scan::TempStorage ss;
        const uint32_t cnt = __popc(~sm.zero[tid] & (kFull ? ~0u : word_mask(len, tid)));
        uint32_t pre;
        Scan(ss).ExclusiveSum(cnt, pre);
        sm.pre[tid] = pre;
    }
    __syncthreads();
    // C: each warp packs its words' codes LSB-first into the stage (shared
    // OR: a code spans at most two stage words, edge words are shared). The
    // stage overlays cw: every warp first takes its codes into registers.
    uint32_t cv[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t k = 4 * j + w;
        const uint32_t cnt = __popc(~sm.zero[k] & (kFull ? ~0u : word_mask(len, k)));
        cv[j] = lane < cnt ? sm.cw[32 * k + lane] : 0u;
    }
    __syncthreads();
    for (uint32_t i = tid; i < nstage; i += kChunkThreads) sm.stage[i] = 0;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t k = 4 * j + w;
        const uint32_t nzw = ~sm.zero[k] & (kFull ? ~0u : word_mask(len, k));
        const uint32_t cnt = __popc(nzw);
        if (!cnt) continue;  // warp-uniform
        const uint32_t a0 = sm.pre[k] * w_bits;  // chunk-relative bit of this word's first code
        const uint32_t off0 = a0 & 31, wbase = a0 >> 5;
        if (kW1 && cnt == 32) {  // width 1, all nonzero: the word's code bits are one ballot
            const uint32_t bw = sm.bits[k];
            if (lane == 0 && bw) {
                atomicOr(&sm.stage[wbase], bw << off0);
                if (off0) atomicOr(&sm.stage[wbase + 1], bw >> (32 - off0));
            }
            continue;
        }
        // scatter: the word's code of rank r (lane r) goes to bits
        // [a0 + r w, a0 + (r + 1) w) of the stage, touching at most two words
        if (lane < cnt && cv[j]) {
            const uint32_t pbit = a0 + lane * w_bits, wi = pbit >> 5, sh = pbit & 31;
            atomicOr(&sm.stage[wi], cv[j] << sh);
            if (sh + w_bits > 32) atomicOr(&sm.stage[wi + 1], cv[j] >> (32 - sh));
        }
    }
    __syncthreads();
    const uint32_t raw_bits = ((len + 7) / 8) * 8;
    if (p.stag == 2) write_bits_block(pay + p.sign_off, 0, sm.sign, raw_bits, tid, kChunkThreads);
    if (p.ztag == 2) write_bits_block(pay + p.zero_off, 0, sm.zero, raw_bits, tid, kChunkThreads);
    const uint64_t start_bit = static_cast<uint64_t>(p.nz_prefix) * w_bits;
    write_bits_block(pay + bp.code_seg + (start_bit >> 3), static_cast<uint32_t>(start_bit & 7), sm.stage, code_bits,
                     tid, kChunkThreads);
}

__global__ void __launch_bounds__(kChunkThreads, 9) k_cmp_emit(const CmpBlock* __restrict__ blks, uint32_t nch_max,
                                                            const ChunkPlan* __restrict__ cps,
                                                            BlockPlan* __restrict__ bps, uint8_t* __restrict__ out,
                                                            DevTables t, const DevError* err) {
    // every record this CTA needs, loaded together (one memory round trip)
    const uint32_t bi = blockIdx.x / nch_max, c = blockIdx.x % nch_max;
    const uint32_t failed = err->code;
    const CmpBlock blk = blks[bi];
    const BlockPlan bp = bps[bi];
    const ChunkPlan p = cps[static_cast<uint64_t>(bi) * nch_max + c];
    if (failed) return;
    if (c > 0 && c >= bp.nch) return;  // (an empty block still gets its header from chunk 0)
    if (bp.out_off == ~0ull) return;   // virtual ALL_ZERO
    // (out == nullptr: out_off is the payload's device address, placed by the caller)
    uint8_t* pay = reinterpret_cast<uint8_t*>(reinterpret_cast<uintptr_t>(out) + bp.out_off);
    const int tid = threadIdx.x;
    if (c == 0 && tid == 0) {  // header (codec.hpp:282-286)
        uint64_t v[3];
        v[0] = blk.count;
        v[1] = static_cast<uint64_t>(__double_as_longlong(t.b_r));
        v[2] = static_cast<uint64_t>(bp.code_min);
        for (int f = 0; f < 3; ++f)
            for (int k = 0; k < 8; ++k) pay[8 * f + k] = static_cast<uint8_t>(v[f] >> (8 * k));
        pay[24] = static_cast<uint8_t>(bp.width);
        pay[25] = static_cast<uint8_t>(bp.flags);
    }
    if (bp.flags & 1) return;
    const ChunkPlan* cp = cps + static_cast<uint64_t>(bi) * nch_max;
    if (c == 0) {  // tag bytes of both bitmaps
        for (uint32_t k = tid; k < bp.ntag; k += kChunkThreads) {
            uint32_t sb = 0, zb = 0;
            for (uint32_t i = 0; i < 4; ++i) {
                const uint32_t cc = 4 * k + i;
                if (cc < bp.nch) {
                    sb |= static_cast<uint32_t>(cp[cc].stag) << (2 * i);
                    zb |= static_cast<uint32_t>(cp[cc].ztag) << (2 * i);
                }
            }
            pay[kHeaderBytes + k] = static_cast<uint8_t>(sb);
            pay[bp.ztag_off + k] = static_cast<uint8_t>(zb);
        }
    }
    const uint32_t len = chunk_len(blk.count, c);
    // a full chunk of zeros is tags only (sign tag 0, zero tag 1): no bytes
    if (p.nnz == 0 && len == kChunk) return;
    __shared__ EmitSmem sm;
    const uint32_t* src = blk.pk + static_cast<uint64_t>(c) * kChunk;
    if (bp.width == 1) {
        if (len == kChunk)
            emit_chunk<true, true>(p, len, src, bp, pay, t, sm);
        else
            emit_chunk<false, true>(p, len, src, bp, pay, t, sm);
    } else if (len == kChunk) {
        emit_chunk<true, false>(p, len, src, bp, pay, t, sm);
    } else {
        emit_chunk<false, false>(p, len, src, bp, pay, t, sm);
    }
}

}  // namespace

// ================================================================ launchers

void launch_compress_plan(cudaStream_t st, const CmpBlock* d_blks, uint64_t nblk, uint32_t nch_max,
                          const DevTables& t, BlockPlan* d_bp, ChunkPlan* d_cp, bool have_pk, DevError* d_err,
                          uint64_t* launches) {
    if (nblk == 0) return;
    if (!have_pk) {
        BMQ_CUDA(cudaMemsetAsync(d_cp, 0, nblk * nch_max * sizeof(ChunkPlan), st));
        k_cmp_stats<<<static_cast<uint32_t>(nblk * nch_max), kChunkThreads, 0, st>>>(d_blks, nch_max, d_cp, t,
                                                                                      d_err);
    }
    k_cmp_plan<<<static_cast<uint32_t>(nblk), kPlanThreads, 0, st>>>(d_blks, nch_max, d_cp, d_bp, t.qlo);
    BMQ_CUDA(cudaGetLastError());
    if (launches) *launches += have_pk ? 1 : 2;
}

void launch_compress_emit(cudaStream_t st, const CmpBlock* d_blks, uint64_t nblk, uint32_t nch_max,
                          const DevTables& t, uint8_t* out, uint64_t out_cap, uint64_t* d_cursor, uint64_t* d_range,
                          BlockPlan* d_bp, ChunkPlan* d_cp, uint64_t* meta_off, uint64_t* meta_size,
                          bool virtual_zero, uint32_t align, DevError* d_err, uint64_t* launches,
                          uint64_t meta_base, uint64_t meta_tag) {
    if (nblk == 0) return;
    k_cmp_alloc<<<1, kAllocThreads, 0, st>>>(d_blks, nblk, d_bp, d_cursor, out_cap, d_range, virtual_zero ? 1 : 0,
                                             align, meta_off, meta_size, meta_base, meta_tag, d_err);
    const uint64_t nthr = nblk * nch_max;
    k_zero_edges<<<static_cast<uint32_t>((nthr + 255) / 256), 256, 0, st>>>(d_blks, nch_max, d_cp, d_bp, out, nblk,
                                                                          d_err);
    k_cmp_emit<<<static_cast<uint32_t>(nblk * nch_max), kChunkThreads, 0, st>>>(d_blks, nch_max, d_cp, d_bp, out, t,
                                                                                 d_err);
    BMQ_CUDA(cudaGetLastError());
    if (launches) *launches += 3;
}

void launch_compress_emit_placed(cudaStream_t st, const CmpBlock* d_blks, uint64_t nblk, uint32_t nch_max,
                                 const DevTables& t, BlockPlan* d_bp, ChunkPlan* d_cp, DevError* d_err,
                                 uint64_t* launches) {
    if (nblk == 0) return;
    const uint64_t nthr = nblk * nch_max;
    k_zero_edges<<<static_cast<uint32_t>((nthr + 255) / 256), 256, 0, st>>>(d_blks, nch_max, d_cp, d_bp, nullptr, nblk,
                                                                          d_err);
    k_cmp_emit<<<static_cast<uint32_t>(nblk * nch_max), kChunkThreads, 0, st>>>(d_blks, nch_max, d_cp, d_bp, nullptr,
                                                                                 t, d_err);
    BMQ_CUDA(cudaGetLastError());
    if (launches) *launches += 2;
}

void launch_compress(cudaStream_t st, const CmpBlock* d_blks, uint64_t nblk, uint32_t nch_max, const DevTables& t,
                     uint8_t* out, uint64_t out_cap, uint64_t* d_cursor, uint64_t* d_range, BlockPlan* d_bp,
                     ChunkPlan* d_cp, uint64_t* meta_off, uint64_t* meta_size, bool virtual_zero, bool have_pk,
                     DevError* d_err, uint64_t* launches) {
    launch_compress_plan(st, d_blks, nblk, nch_max, t, d_bp, d_cp, have_pk, d_err, launches);
    launch_compress_emit(st, d_blks, nblk, nch_max, t, out, out_cap, d_cursor, d_range, d_bp, d_cp, meta_off,
                         meta_size, virtual_zero, virtual_zero ? 16 : 1, d_err, launches);
}

}  // namespace bmq
