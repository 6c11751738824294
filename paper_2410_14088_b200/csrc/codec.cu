// codec.cu — byte-exact device implementation of the reference point-wise
// codec (codec.hpp:227-344, bitmap.hpp:109-189) for batches of blocks.
//
// Work decomposition: one CTA of 128 threads per 4096-scalar chunk, which is
// exactly one prescan chunk of each bitmap (bitmap.hpp:76). Warp w, step j
// handles scalars 128 j + 32 w + lane, so global loads/stores are coalesced
// and a warp ballot yields bitmap word 4 j + w directly (the paper's warp
// ballot pre-scan).
//
// Compress = stats (quantise, ballot, per-chunk min/max/nnz/tags)
//          -> plan (per block: code_min, width, segment offsets, size)
//          -> alloc (exclusive scan of sizes into the output region)
//          -> zero (clear the region so shared edge words can be OR-ed)
//          -> emit (header, tags, raw mixed chunks, LSB-first codes).
// Decompress = index (validate header / tags, raw offsets, nonzero prefix)
//            -> decode (bitmaps to SMEM, rank, unpack, exact dequant LUT).
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include <cfloat>
#include <climits>
#include <map>
#include <mutex>

#include "codec.cuh"

namespace bmq {

// --------------------------------------------------------------- messages
const char* dev_error_message(uint32_t code) {
    switch (code) {
    case DE_NONFINITE: return "input scalars must be finite";
    case DE_WINDOW: return "scalar magnitude below the quantiser table window of this error bound";
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
    return cache.emplace(std::make_pair(dev, key), t).first->second;
}

namespace {

__device__ __forceinline__ uint32_t chunk_len(uint64_t count, uint32_t c) {
    const uint64_t first = static_cast<uint64_t>(c) * kChunk;
    const uint64_t rest = count - first;
    return rest < kChunk ? static_cast<uint32_t>(rest) : kChunk;
}

__device__ __forceinline__ uint32_t word_mask(uint32_t len, uint32_t k) {
    // valid bits of bitmap word k of a chunk of len scalars
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

// ============================================================== compress

__global__ void __launch_bounds__(kChunkThreads) k_cmp_stats(const CmpBlock* __restrict__ blks,
                                                             uint32_t nch_max, ChunkPlan* __restrict__ cps,
                                                             DevTables t, DevError* err) {
    const uint32_t bi = blockIdx.x / nch_max, c = blockIdx.x % nch_max;
    const CmpBlock blk = blks[bi];
    const uint64_t nch = (blk.count + kChunk - 1) / kChunk;
    if (c >= nch) return;
    const uint32_t len = chunk_len(blk.count, c);
    const double* src = blk.in + static_cast<uint64_t>(c) * kChunk;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int64_t qmin = LLONG_MAX, qmax = LLONG_MIN;
    uint32_t nnz = 0;
    uint32_t s_or = 0, s_and = ~0u, z_or = 0, z_and = ~0u;
    bool bad = false, oow = false;
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
        const uint32_t s = 128 * j + 32 * w + lane;
        const bool valid = s < len;
        const double v = valid ? __ldg(src + s) : 0.0;
        if (valid && !isfinite(v)) bad = true;
        const bool neg = valid && v < 0.0;
        const bool zero = valid && v == 0.0;
        const uint32_t sw = __ballot_sync(0xffffffffu, neg);
        const uint32_t zw = __ballot_sync(0xffffffffu, zero);
        s_or |= sw;
        s_and &= sw;
        z_or |= zw;
        z_and &= zw;
        if (valid && !zero && isfinite(v)) {
            const int64_t q = quantize(v, t, oow);
            qmin = q < qmin ? q : qmin;
            qmax = q > qmax ? q : qmax;
            ++nnz;
        }
    }
    if (bad) dev_fail(err, DE_NONFINITE, bi);
    if (oow) dev_fail(err, DE_WINDOW, bi);
    using Reduce = cub::BlockReduce<long long, kChunkThreads>;
    using ReduceU = cub::BlockReduce<uint32_t, kChunkThreads>;
    __shared__ typename Reduce::TempStorage r1;
    __shared__ typename ReduceU::TempStorage r2;
    __shared__ uint32_t bits[4][4];
    const long long bmin = Reduce(r1).Reduce(static_cast<long long>(qmin), cub::Min());
    __syncthreads();
    const long long bmax = Reduce(r1).Reduce(static_cast<long long>(qmax), cub::Max());
    const uint32_t bnnz = ReduceU(r2).Sum(nnz);
    if (lane == 0) {
        bits[w][0] = s_or;
        bits[w][1] = s_and;
        bits[w][2] = z_or;
        bits[w][3] = z_and;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t so = 0, sa = ~0u, zo = 0, za = ~0u;
        for (int k = 0; k < 4; ++k) {
            so |= bits[k][0];
            sa &= bits[k][1];
            zo |= bits[k][2];
            za &= bits[k][3];
        }
        ChunkPlan p{};
        p.qmin = bnnz ? static_cast<int32_t>(bmin) : INT_MAX;
        p.qmax = bnnz ? static_cast<int32_t>(bmax) : INT_MIN;
        p.nnz = bnnz;
        const bool full = len == kChunk;
        p.stag = !full ? 2 : (so == 0 ? 0 : (sa == ~0u ? 1 : 2));
        p.ztag = !full ? 2 : (zo == 0 ? 0 : (za == ~0u ? 1 : 2));
        cps[static_cast<uint64_t>(bi) * nch_max + c] = p;
    }
}

// One CTA per block: reduce chunk stats, lay out the payload segments.
constexpr int kPlanThreads = 256;

__global__ void __launch_bounds__(kPlanThreads) k_cmp_plan(const CmpBlock* __restrict__ blks, uint32_t nch_max,
                                                           ChunkPlan* __restrict__ cps, BlockPlan* __restrict__ bps) {
    const uint32_t bi = blockIdx.x;
    const CmpBlock blk = blks[bi];
    const uint32_t nch = static_cast<uint32_t>((blk.count + kChunk - 1) / kChunk);
    ChunkPlan* cp = cps + static_cast<uint64_t>(bi) * nch_max;
    using Reduce = cub::BlockReduce<long long, kPlanThreads>;
    using Scan = cub::BlockScan<unsigned long long, kPlanThreads>;
    __shared__ typename Reduce::TempStorage rs;
    __shared__ typename Scan::TempStorage ss;
    __shared__ long long s_min, s_max;
    __shared__ unsigned long long s_nnz, s_sraw, s_zraw;
    // pass 1: totals
    long long mn = LLONG_MAX, mx = LLONG_MIN;
    unsigned long long nnz = 0, sraw = 0, zraw = 0;
    for (uint32_t c = threadIdx.x; c < nch; c += kPlanThreads) {
        const ChunkPlan p = cp[c];
        const uint32_t len = chunk_len(blk.count, c);
        if (p.nnz) {
            mn = min(mn, static_cast<long long>(p.qmin));
            mx = max(mx, static_cast<long long>(p.qmax));
        }
        nnz += p.nnz;
        if (p.stag == 2) sraw += (len + 7) / 8;
        if (p.ztag == 2) zraw += (len + 7) / 8;
    }
    const long long gmn = Reduce(rs).Reduce(mn, cub::Min());
    __syncthreads();
    const long long gmx = Reduce(rs).Reduce(mx, cub::Max());
    __syncthreads();
    const unsigned long long a = Reduce(rs).Sum(static_cast<long long>(nnz));
    __syncthreads();
    const unsigned long long b = Reduce(rs).Sum(static_cast<long long>(sraw));
    __syncthreads();
    const unsigned long long z = Reduce(rs).Sum(static_cast<long long>(zraw));
    if (threadIdx.x == 0) {
        s_min = gmn;
        s_max = gmx;
        s_nnz = a;
        s_sraw = b;
        s_zraw = z;
    }
    __syncthreads();
    const uint32_t ntag = (nch + 3) / 4;
    const uint64_t ztag_off = kHeaderBytes + ntag + s_sraw;
    const uint64_t code_seg = ztag_off + ntag + s_zraw;
    uint32_t width = 0;
    if (s_nnz) {
        const uint64_t range = static_cast<uint64_t>(s_max - s_min);
        width = range ? 64 - __clzll(static_cast<long long>(range)) : 1;
    }
    // pass 2: per-chunk offsets (exclusive scans in chunk order)
    unsigned long long carry_s = 0, carry_z = 0, carry_n = 0;
    for (uint32_t base = 0; base < nch; base += kPlanThreads) {
        const uint32_t c = base + threadIdx.x;
        unsigned long long vs = 0, vz = 0, vn = 0;
        ChunkPlan p{};
        if (c < nch) {
            p = cp[c];
            const uint32_t len = chunk_len(blk.count, c);
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
        bp.nnz = s_nnz;
        if (s_nnz == 0) {
            bp.flags = 1;
            bp.size = kHeaderBytes;
        } else {
            bp.code_min = s_min;
            bp.code_max = s_max;
            bp.width = width;
            bp.ztag_off = ztag_off;
            bp.code_seg = code_seg;
            bp.size = code_seg + (s_nnz * width + 7) / 8;
        }
        bps[bi] = bp;
    }
}

// Single CTA: exclusive scan of payload sizes into [cursor, cursor + total).
// virtual_zero: ALL_ZERO payloads take no space (engine pools); they are
// materialised as the canonical 26-byte header on read.
constexpr int kAllocThreads = 1024;

__global__ void __launch_bounds__(kAllocThreads) k_cmp_alloc(const CmpBlock* __restrict__ blks, uint64_t nblk,
                                                             BlockPlan* __restrict__ bps, uint64_t* cursor,
                                                             uint64_t cap, uint64_t* range, int virtual_zero,
                                                             uint64_t* meta_off, uint64_t* meta_size,
                                                             DevError* err) {
    using Scan = cub::BlockScan<unsigned long long, kAllocThreads>;
    __shared__ typename Scan::TempStorage ss;
    const uint64_t start = *cursor;
    unsigned long long carry = 0;
    for (uint64_t base = 0; base < nblk; base += kAllocThreads) {
        const uint64_t i = base + threadIdx.x;
        unsigned long long sz = 0;
        if (i < nblk) {
            const BlockPlan& p = bps[i];
            sz = (virtual_zero && (p.flags & 1)) ? 0 : p.size;
        }
        unsigned long long pre, tot;
        Scan(ss).ExclusiveSum(sz, pre, tot);
        __syncthreads();
        if (i < nblk) {
            BlockPlan& p = bps[i];
            const bool virt = virtual_zero && (p.flags & 1);
            p.out_off = virt ? ~0ull : start + carry + pre;
            if (meta_off) {
                const uint64_t id = blks[i].id;
                meta_off[id] = p.out_off;
                meta_size[id] = p.size;
            }
        }
        carry += tot;
    }
    if (threadIdx.x == 0) {
        const uint64_t end = start + carry;
        if (end > cap) {
            dev_fail(err, DE_POOL_FULL, 0);
            range[0] = range[1] = start;
        } else {
            range[0] = start;
            range[1] = end;
            *cursor = end;
        }
    }
}

__global__ void k_zero_range(uint8_t* base, const uint64_t* range) {
    const uint64_t a = range[0], b = range[1];
    if (b <= a) return;
    const uint64_t wa = (a + 3) / 4, wb = b / 4;  // whole words [wa, wb)
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    uint32_t* w = reinterpret_cast<uint32_t*>(base);
    if (wa < wb) {
        for (uint64_t i = wa + tid; i < wb; i += stride) w[i] = 0;
        if (tid < 4) {
            const uint64_t x = a + tid;
            if (x < wa * 4) base[x] = 0;
            const uint64_t y = wb * 4 + tid;
            if (y < b) base[y] = 0;
        }
    } else if (tid < b - a) {
        base[a + tid] = 0;
    }
}

constexpr int kStageWords = (kChunk * 63 + 31) / 32 + 2;

__global__ void __launch_bounds__(kChunkThreads) k_cmp_emit(const CmpBlock* __restrict__ blks, uint32_t nch_max,
                                                            const ChunkPlan* __restrict__ cps,
                                                            BlockPlan* __restrict__ bps, uint8_t* __restrict__ out,
                                                            DevTables t, const DevError* err) {
    if (err->code) return;
    const uint32_t bi = blockIdx.x / nch_max, c = blockIdx.x % nch_max;
    const CmpBlock blk = blks[bi];
    const BlockPlan bp = bps[bi];
    if (c > 0 && c >= bp.nch) return;  // (an empty block still gets its header from chunk 0)
    if (bp.out_off == ~0ull) return;   // virtual ALL_ZERO
    uint8_t* pay = out + bp.out_off;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
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
    const ChunkPlan p = cp[c];
    const uint32_t len = chunk_len(blk.count, c);
    const double* src = blk.in + static_cast<uint64_t>(c) * kChunk;
    __shared__ uint32_t s_sign[kWordsPerChunk], s_zero[kWordsPerChunk], s_pre[kWordsPerChunk];
    __shared__ uint32_t stage[kStageWords];
    __shared__ double s_red[3][4];
    const uint32_t w_bits = bp.width;
    const uint64_t code_bits = static_cast<uint64_t>(p.nnz) * w_bits;
    const uint32_t nstage = static_cast<uint32_t>((code_bits + 31) / 32);
    for (uint32_t i = tid; i < nstage; i += kChunkThreads) stage[i] = 0;
    int32_t qv[32];
    double sq = 0.0, sre = 0.0, sim = 0.0;
    const uint64_t half = blk.count / 2, g0 = static_cast<uint64_t>(c) * kChunk;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t s = 128 * j + 32 * w + lane;
        const bool valid = s < len;
        const double v = valid ? __ldg(src + s) : 0.0;
        const bool neg = valid && v < 0.0;
        const bool zero = !valid || v == 0.0;
        const uint32_t sw = __ballot_sync(0xffffffffu, neg);
        const uint32_t zw = __ballot_sync(0xffffffffu, valid && v == 0.0);
        if (lane == 0) {
            s_sign[4 * j + w] = sw;
            s_zero[4 * j + w] = zw;
        }
        bool oow = false;
        qv[j] = zero ? 0 : static_cast<int32_t>(quantize(v, t, oow));
        if (!zero) {
            const double m = __ldg(t.dequant + (qv[j] - t.qlo));
            sq += m * m;
            if (g0 + s < half)
                sre += neg ? -m : m;
            else
                sim += neg ? -m : m;
        }
    }
    __syncthreads();
    // nonzero prefix over the 128 words in scalar order
    {
        using Scan = cub::BlockScan<uint32_t, kChunkThreads>;
        __shared__ typename Scan::TempStorage ss;
        const uint32_t cnt = __popc(~s_zero[tid] & word_mask(len, tid));
        uint32_t pre;
        Scan(ss).ExclusiveSum(cnt, pre);
        s_pre[tid] = pre;
    }
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t k = 4 * j + w;
        const uint32_t nzw = ~s_zero[k] & word_mask(len, k);
        if ((nzw >> lane) & 1u) {
            const uint32_t rank = s_pre[k] + __popc(nzw & lt);
            const uint64_t code = static_cast<uint64_t>(static_cast<int64_t>(qv[j]) - bp.code_min);
            const uint64_t pos = static_cast<uint64_t>(rank) * w_bits;
            const uint32_t wi = static_cast<uint32_t>(pos >> 5), sh = static_cast<uint32_t>(pos & 31);
            atomicOr(&stage[wi], static_cast<uint32_t>(code << sh));
            if (sh + w_bits > 32) atomicOr(&stage[wi + 1], static_cast<uint32_t>(code >> (32 - sh)));
            if (sh + w_bits > 64) atomicOr(&stage[wi + 2], static_cast<uint32_t>(code >> (64 - sh)));
        }
    }
    __syncthreads();
    const uint32_t raw_bits = ((len + 7) / 8) * 8;
    if (p.stag == 2) write_bits_block(pay + p.sign_off, 0, s_sign, raw_bits, tid, kChunkThreads);
    if (p.ztag == 2) write_bits_block(pay + p.zero_off, 0, s_zero, raw_bits, tid, kChunkThreads);
    const uint64_t start_bit = static_cast<uint64_t>(p.nz_prefix) * w_bits;
    write_bits_block(pay + bp.code_seg + (start_bit >> 3), static_cast<uint32_t>(start_bit & 7), stage, code_bits,
                     tid, kChunkThreads);
    // dequantised sums for norm / analytic fidelity
    block_sums3(sq, sre, sim, s_red, &bps[bi].sumsq);
}

// ============================================================ decompress

__device__ __forceinline__ bool tag_error(uint32_t tag, uint32_t len, uint32_t& code) {
    if (tag > 2) {
        code = DE_TAG;
        return true;
    }
    if (tag != 2 && len < kChunk) {
        code = DE_PARTIAL;
        return true;
    }
    return false;
}

constexpr int kIndexThreads = 256;

__global__ void __launch_bounds__(kIndexThreads) k_dec_index(const DecBlock* __restrict__ blks, uint32_t nch_max,
                                                             DecInfo* __restrict__ infos, DecChunk* __restrict__ dcs,
                                                             DevTables t, int check_bound, DevError* err) {
    const uint32_t bi = blockIdx.x;
    const DecBlock blk = blks[bi];
    const uint8_t* p = blk.in;
    using Scan = cub::BlockScan<unsigned long long, kIndexThreads>;
    using ReduceU = cub::BlockReduce<unsigned long long, kIndexThreads>;
    __shared__ typename Scan::TempStorage ss;
    __shared__ typename ReduceU::TempStorage rs;
    __shared__ uint64_t s_count;
    __shared__ uint32_t s_fail, s_nch, s_ntag, s_width, s_flags;
    __shared__ int64_t s_cmin;
    DecChunk* dc = dcs + static_cast<uint64_t>(bi) * nch_max;
    const int tid = threadIdx.x;
    if (tid == 0) {
        uint32_t fail = 0;
        uint64_t count = 0;
        uint32_t width = 0, flags = 0;
        int64_t cmin = 0;
        if (blk.size < kHeaderBytes) {
            fail = DE_HDR_TRUNC;
        } else {
            uint64_t v[3] = {0, 0, 0};
            for (int f = 0; f < 3; ++f)
                for (int k = 0; k < 8; ++k) v[f] |= static_cast<uint64_t>(p[8 * f + k]) << (8 * k);
            count = v[0];
            const double br = __longlong_as_double(static_cast<long long>(v[1]));
            cmin = static_cast<int64_t>(v[2]);
            width = p[24];
            flags = p[25];
            if (!(br > 0.0) || isnan(br) || isinf(br)) {
                fail = DE_HDR_BOUND;
            } else if (flags & 1) {
                if (blk.size != kHeaderBytes) fail = DE_HDR_TRAIL;
            } else if (check_bound && br != t.b_r) {
                fail = DE_BOUND_MISMATCH;
            } else if ((count + kChunk - 1) / kChunk > nch_max) {
                fail = DE_TOO_LARGE;
            }
        }
        s_fail = fail;
        s_count = count;
        s_width = width;
        s_flags = flags;
        s_cmin = cmin;
        s_nch = static_cast<uint32_t>((count + kChunk - 1) / kChunk);
        s_ntag = (s_nch + 3) / 4;
    }
    __syncthreads();
    const uint64_t count = s_count;
    const uint32_t nch = s_nch, ntag = s_ntag;
    uint32_t fail = s_fail;
    DecInfo info{};
    info.count = count;
    info.code_min = s_cmin;
    info.width = s_width;
    if (!fail && (s_flags & 1)) {
        info.flags = 1;
        if (blk.expect_count && count != blk.expect_count) {
            if (tid == 0) dev_fail(err, DE_COUNT, bi);
            info.flags = 2;
        }
        if (tid == 0) infos[bi] = info;
        return;
    }
    // Both bitmaps: tags, raw offsets; the first bad chunk (in order) reports.
    uint64_t seg = kHeaderBytes;
    for (int bm = 0; bm < 2 && !fail; ++bm) {
        const uint32_t trunc = bm == 0 ? DE_SIGN_TRUNC : DE_ZERO_TRUNC;
        if (blk.size - seg < ntag) {
            fail = trunc;
            break;
        }
        const uint8_t* tags = p + seg;
        const uint64_t raw0 = seg + ntag;
        unsigned long long carry = 0;
        unsigned long long first_bad = ~0ull;
        for (uint32_t base = 0; base < nch; base += kIndexThreads) {
            const uint32_t c = base + tid;
            unsigned long long nb = 0;
            if (c < nch) {
                const uint32_t len = chunk_len(count, c);
                const uint32_t tag = (tags[c / 4] >> (2 * (c % 4))) & 3u;
                uint32_t code;
                if (tag_error(tag, len, code)) first_bad = min(first_bad, (static_cast<unsigned long long>(c) << 8) | code);
                if (tag == 2) nb = (len + 7) / 8;
                if (bm == 0) {
                    dc[c].stag = static_cast<uint8_t>(tag);
                    dc[c].sign_off = static_cast<uint32_t>(raw0 + carry);
                } else {
                    dc[c].ztag = static_cast<uint8_t>(tag);
                    dc[c].zero_off = static_cast<uint32_t>(raw0 + carry);
                }
            }
            unsigned long long pre, tot;
            Scan(ss).ExclusiveSum(nb, pre, tot);
            __syncthreads();
            if (c < nch) {
                if (bm == 0)
                    dc[c].sign_off += static_cast<uint32_t>(pre);
                else
                    dc[c].zero_off += static_cast<uint32_t>(pre);
            }
            carry += tot;
        }
        const unsigned long long fb = ReduceU(rs).Reduce(first_bad, cub::Min());
        __shared__ unsigned long long s_fb;
        if (tid == 0) s_fb = fb;
        __syncthreads();
        if (s_fb != ~0ull) {
            fail = static_cast<uint32_t>(s_fb & 0xff);
            break;
        }
        if (blk.size - raw0 < carry) {
            fail = trunc;
            break;
        }
        seg = raw0 + carry;
    }
    // nonzero scalars per chunk -> prefix
    unsigned long long nnz_total = 0;
    if (!fail) {
        unsigned long long carry = 0;
        for (uint32_t base = 0; base < nch; base += kIndexThreads) {
            const uint32_t c = base + tid;
            unsigned long long nz = 0;
            if (c < nch) {
                const uint32_t len = chunk_len(count, c);
                const uint32_t tag = dc[c].ztag;
                if (tag == 0) {
                    nz = len;
                } else if (tag == 2) {
                    const uint8_t* raw = p + dc[c].zero_off;
                    uint32_t zeros = 0;
                    for (uint32_t k = 0; k * 32 < len; ++k) zeros += __popc(load_u32_unaligned(raw + 4 * k) & word_mask(len, k));
                    nz = len - zeros;
                }
            }
            unsigned long long pre, tot;
            Scan(ss).ExclusiveSum(nz, pre, tot);
            __syncthreads();
            if (c < nch) dc[c].nz_prefix = static_cast<uint32_t>(carry + pre);
            carry += tot;
        }
        nnz_total = carry;
        if (s_width == 0 && nnz_total > 0) {
            fail = DE_WIDTH0;
        } else {
            const uint64_t need = (nnz_total * s_width + 7) / 8;
            if (blk.size - seg < need)
                fail = DE_CODES_TRUNC;
            else if (blk.size - seg != need)
                fail = DE_CODES_TRAIL;
        }
    }
    if (!fail && blk.expect_count && count != blk.expect_count) fail = DE_COUNT;
    if (tid == 0) {
        info.code_seg = seg;
        info.flags = fail ? 2 : 0;
        infos[bi] = info;
        if (fail) dev_fail(err, fail, bi);
    }
}

__global__ void __launch_bounds__(kChunkThreads) k_dec_chunk(const DecBlock* __restrict__ blks, uint32_t nch_max,
                                                             DecInfo* __restrict__ infos,
                                                             const DecChunk* __restrict__ dcs, DevTables t,
                                                             int want_sums, DevError* err) {
    const uint32_t bi = blockIdx.x / nch_max, c = blockIdx.x % nch_max;
    const DecInfo info = infos[bi];
    if (info.flags & 2) return;
    const uint64_t nch = (info.count + kChunk - 1) / kChunk;
    if (c >= nch) return;
    const DecBlock blk = blks[bi];
    const uint32_t len = chunk_len(info.count, c);
    double* dst = blk.out + static_cast<uint64_t>(c) * kChunk;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (info.flags & 1) {
        for (uint32_t s = tid; s < len; s += kChunkThreads) dst[s] = 0.0;
        return;
    }
    const DecChunk d = dcs[static_cast<uint64_t>(bi) * nch_max + c];
    __shared__ uint32_t s_sign[kWordsPerChunk], s_zero[kWordsPerChunk], s_pre[kWordsPerChunk];
    __shared__ double s_red[3][4];
    {
        const uint32_t vm = word_mask(len, tid);
        uint32_t sw = 0, zw = 0;
        if (vm) {
            sw = d.stag == 1 ? vm : (d.stag == 2 ? load_u32_unaligned(blk.in + d.sign_off + 4 * tid) & vm : 0);
            zw = d.ztag == 1 ? vm : (d.ztag == 2 ? load_u32_unaligned(blk.in + d.zero_off + 4 * tid) & vm : 0);
        }
        s_sign[tid] = sw;
        s_zero[tid] = zw;
        using Scan = cub::BlockScan<uint32_t, kChunkThreads>;
        __shared__ typename Scan::TempStorage ss;
        uint32_t pre;
        Scan(ss).ExclusiveSum(static_cast<uint32_t>(__popc(~zw & vm)), pre);
        s_pre[tid] = pre;
    }
    __syncthreads();
    const uint8_t* codes = blk.in + info.code_seg;
    const uint32_t width = info.width;
    const uint32_t lt = (1u << lane) - 1;
    double sq = 0.0, sre = 0.0, sim = 0.0;
    const uint64_t half = info.count / 2, g0 = static_cast<uint64_t>(c) * kChunk;
    bool bad = false;
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
        const uint32_t k = 4 * j + w;
        const uint32_t s = 32 * k + lane;
        if (s >= len) continue;
        const uint32_t vm = word_mask(len, k);
        const uint32_t nzw = ~s_zero[k] & vm;
        double v = 0.0;
        if ((nzw >> lane) & 1u) {
            const uint64_t rank = static_cast<uint64_t>(d.nz_prefix) + s_pre[k] + __popc(nzw & lt);
            const uint64_t code = read_bits(codes, rank * width, width);
            const int64_t q = info.code_min + static_cast<int64_t>(code);
            if (q < t.qlo || q > t.qhi) {
                bad = true;
            } else {
                const double m = __ldg(t.dequant + (q - t.qlo));
                v = ((s_sign[k] >> lane) & 1u) ? -m : m;
                sq += m * m;
                if (g0 + s < half)
                    sre += v;
                else
                    sim += v;
            }
        }
        dst[s] = v;
    }
    if (bad) dev_fail(err, DE_CODE_WINDOW, bi);
    if (want_sums) block_sums3(sq, sre, sim, s_red, &infos[bi].sumsq);
}

}  // namespace

// ================================================================ launchers

void launch_compress(cudaStream_t st, const CmpBlock* d_blks, uint64_t nblk, uint32_t nch_max, const DevTables& t,
                     uint8_t* out, uint64_t out_cap, uint64_t* d_cursor, uint64_t* d_range, BlockPlan* d_bp,
                     ChunkPlan* d_cp, uint64_t* meta_off, uint64_t* meta_size, bool virtual_zero, DevError* d_err,
                     uint64_t* launches) {
    if (nblk == 0) return;
    BMQ_CUDA(cudaMemsetAsync(d_bp, 0, nblk * sizeof(BlockPlan), st));
    const uint32_t grid = static_cast<uint32_t>(nblk * nch_max);
    k_cmp_stats<<<grid, kChunkThreads, 0, st>>>(d_blks, nch_max, d_cp, t, d_err);
    k_cmp_plan<<<static_cast<uint32_t>(nblk), kPlanThreads, 0, st>>>(d_blks, nch_max, d_cp, d_bp);
    k_cmp_alloc<<<1, kAllocThreads, 0, st>>>(d_blks, nblk, d_bp, d_cursor, out_cap, d_range, virtual_zero ? 1 : 0,
                                             meta_off, meta_size, d_err);
    k_zero_range<<<296, 256, 0, st>>>(out, d_range);
    k_cmp_emit<<<grid, kChunkThreads, 0, st>>>(d_blks, nch_max, d_cp, d_bp, out, t, d_err);
    BMQ_CUDA(cudaGetLastError());
    if (launches) *launches += 5;
}

void launch_decompress(cudaStream_t st, const DecBlock* d_blks, uint64_t nblk, uint32_t nch_max, const DevTables& t,
                       DecInfo* d_info, DecChunk* d_dc, bool check_bound, bool want_sums, DevError* d_err,
                       uint64_t* launches) {
    if (nblk == 0) return;
    BMQ_CUDA(cudaMemsetAsync(d_info, 0, nblk * sizeof(DecInfo), st));
    k_dec_index<<<static_cast<uint32_t>(nblk), kIndexThreads, 0, st>>>(d_blks, nch_max, d_info, d_dc, t,
                                                                        check_bound ? 1 : 0, d_err);
    const uint32_t grid = static_cast<uint32_t>(nblk * nch_max);
    k_dec_chunk<<<grid, kChunkThreads, 0, st>>>(d_blks, nch_max, d_info, d_dc, t, want_sums ? 1 : 0, d_err);
    BMQ_CUDA(cudaGetLastError());
    if (launches) *launches += 2;
}

}  // namespace bmq
