// codec_dec.cu — byte-exact device decompressor (decompress_block,
// codec.hpp:299-344; read_prescan / prescan_decode, codec.hpp:190-209,
// bitmap.hpp:147-189) for batches of payloads.
//
// index  (one CTA per block): validate the header and both tag streams in the
//        reference's order, locate each chunk's raw bitmap bytes, and prefix
//        the nonzero counts so every chunk knows where its codes start;
// decode (one CTA per 4096-scalar chunk): bitmaps to SMEM, per-word rank
//        prefix, unpack the LSB-first codes, exact dequantisation by table.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "codec.cuh"
#include "codec_util.cuh"

namespace bmq {

namespace {
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

// zflag (optional): one byte per (block, chunk), 1 when every scalar of the
// chunk is zero (an ALL_ZERO block, or a full chunk with zero tag 1).
__global__ void __launch_bounds__(kIndexThreads) k_dec_index(const DecBlock* __restrict__ blks, uint32_t nch_max,
                                                             DecInfo* __restrict__ infos, DecChunk* __restrict__ dcs,
                                                             DevTables t, int check_bound, DevError* err,
                                                             uint8_t* __restrict__ zflag, uint32_t* imnz,
                                                             uint32_t* wz) {
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
        if (wz && tid == 0) *wz = 1;  // an ALL_ZERO block: its groups are flagged zero
        if (zflag)
            for (uint32_t c = tid; c < nch_max; c += kIndexThreads) zflag[static_cast<uint64_t>(bi) * nch_max + c] = 1;
        return;
    }
    // Both bitmaps: tags, raw offsets; the first bad chunk (in order) reports.
    uint64_t seg = kHeaderBytes;
    bool any_zero = false;
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
                    const bool zc = tag == 1 && len == kChunk;
                    if (zflag) zflag[static_cast<uint64_t>(bi) * nch_max + c] = zc ? 1 : 0;
                    if (imnz && !zc && 2 * c >= nch) *imnz = 1;  // imaginary half (chunks nch/2.. of 2^(lb+1) scalars)
                    if (tag != 0) any_zero = true;  // the chunk has zero scalars (maybe whole zero groups)
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
    // wz: some block may hold an all-zero 32-scalar group (one store per block)
    if (__syncthreads_or(any_zero) && wz && tid == 0) *wz = 1;
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

// Output modes: kDoubles writes the planar scalars; kCodes writes packed
// code words (CmpBlock::pk layout, (q - qlo) << 2 | negative << 1 | zero)
// for code-domain stages — codes must lie in the tables' idempotent window
// so that compress(decompress) reproduces them; kSumsOnly writes nothing and
// only accumulates the dequantised sums (norm / fidelity).
enum DecMode : int { kDoubles = 0, kCodes = 1, kSumsOnly = 2 };

// Warp-cooperative code fetch: the nonzero scalars of one 32-scalar bitmap
// word hold consecutive ranks, so their codes are one contiguous bit range.
// Each lane loads one aligned 32-bit word of that range; lane j's code is
// then two shuffles and a funnel shift away (width <= 30). All 32 lanes call.
__device__ __forceinline__ uint32_t warp_codes(const uint32_t* __restrict__ cs32, uint64_t a0, uint32_t cnt, uint32_t width,
                                               uint32_t rank_in_word, uint32_t lane) {
    const uint32_t off0 = static_cast<uint32_t>(a0 & 31);
    const uint64_t w0 = a0 >> 5;
    const uint32_t nwords = (off0 + cnt * width + 31) >> 5;
    const uint32_t wv = lane < nwords ? __ldg(cs32 + w0 + lane) : 0u;
    const uint32_t a = off0 + rank_in_word * width;
    const uint32_t rel = (a >> 5) & 31, sh = a & 31;
    const uint32_t lo = __shfl_sync(0xffffffffu, wv, rel), hi = __shfl_sync(0xffffffffu, wv, (rel + 1) & 31);
    return __funnelshift_r(lo, hi, sh) & ((1u << width) - 1);
}

// Per-scalar loop of one chunk. kFull: a whole 4096-scalar chunk (no
// partial words). check: some code of the block may fall outside the window
// (block-uniform; decided from code_min and the width).
template <int kMode, bool kFull, bool kCheck>
__device__ __forceinline__ void dec_scalars(const uint32_t* s_sign, const uint32_t* s_nz, const uint32_t* s_pre,
                                            const uint8_t* codes, uint32_t width, uint32_t nz_prefix, uint32_t len,
                                            int64_t qbase, int64_t lo, int64_t hi, const DevTables& t, double* dst,
                                            uint32_t* cdst, uint64_t half, uint64_t g0, bool sums, double& sq,
                                            double& sre, double& sim, bool& bad, uint8_t* gflag) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uintptr_t cs = reinterpret_cast<uintptr_t>(codes);
    const bool coop = width <= 30;  // block-uniform
    // this chunk's codes start at bit cb of the word-aligned segment base
    const uint64_t cb = static_cast<uint64_t>(cs & 3) * 8 + static_cast<uint64_t>(nz_prefix) * width;
    const uint32_t* __restrict__ cw = reinterpret_cast<const uint32_t*>(cs & ~uintptr_t(3)) + (cb >> 5);
    const uint32_t cb0 = static_cast<uint32_t>(cb & 31);
    const uint32_t cmask = width >= 32 ? ~0u : (1u << width) - 1;
    const uint32_t lt = (1u << lane) - 1;
    const uint32_t qb = static_cast<uint32_t>(qbase);  // packed offset of code 0 (in window when !kCheck)
    const auto emit = [&](uint32_t s, bool mine, uint64_t code, uint32_t neg) {
        if (kCheck && mine) {
            const int64_t qo = qbase + static_cast<int64_t>(code);
            if (qo < lo || qo > hi) {
                bad = true;
                mine = false;
            }
        }
        if constexpr (kMode == kCodes) {
            const uint32_t pkw = mine ? ((qb + static_cast<uint32_t>(code)) << 2) | (neg << 1) : 1u;
            if (kFull || s < len) __stcs(cdst + s, pkw);
        } else {
            double v = 0.0;
            if (mine) {
                const double m = __ldg(t.dequant + (qb + static_cast<uint32_t>(code)));
                v = neg ? -m : m;
                if (kMode == kSumsOnly || sums) {
                    sq += m * m;
                    if (g0 + s < half)
                        sre += v;
                    else
                        sim += v;
                }
            }
            if (kMode == kDoubles && (kFull || s < len)) __stcs(dst + s, v);
        }
    };
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
        const uint32_t k = 4 * j + w;
        if (!kFull && k * 32 >= len) break;  // warp-uniform; later words are empty too
        const uint32_t s = 32 * k + lane;
        const uint32_t nzw = s_nz[k];
        const uint32_t neg = (s_sign[k] >> lane) & 1u;
        if (kMode == kDoubles && gflag) {  // 32-scalar group flags: zero groups are not stored
            if (lane == 0) gflag[k] = nzw ? 1 : 0;
            if (!nzw) continue;
        }
        if (coop && nzw == ~0u) {  // every scalar nonzero: rank = lane
            const uint32_t a = cb0 + s_pre[k] * width + lane * width;
            const uint32_t wlo = __ldg(cw + (a >> 5)), whi = __ldg(cw + (a >> 5) + 1);
            emit(s, true, __funnelshift_r(wlo, whi, a & 31) & cmask, neg);
            continue;
        }
        const bool mine = (nzw >> lane) & 1u;
        uint64_t code = 0;
        if (coop) {
            if (nzw) code = warp_codes(cw, cb0 + s_pre[k] * width, __popc(nzw), width, __popc(nzw & lt), lane);
        } else if (mine) {
            code = read_bits(codes, (static_cast<uint64_t>(nz_prefix) + s_pre[k] + __popc(nzw & lt)) * width, width);
        }
        emit(s, mine, code, neg);
    }
}

template <int kMode>
__global__ void __launch_bounds__(kChunkThreads) k_dec_chunk(const DecBlock* __restrict__ blks, uint32_t nch_max,
                                                             DecInfo* __restrict__ infos,
                                                             const DecChunk* __restrict__ dcs, DevTables t,
                                                             int want_sums, DevError* err, int skip_zero_chunks,
                                                             uint8_t* __restrict__ wflag,
                                                             PermSrc* __restrict__ psrc = nullptr) {
    // the CTA's records, loaded together (one memory round trip)
    const uint32_t bi = blockIdx.x / nch_max, c = blockIdx.x % nch_max;
    const DecInfo info = infos[bi];
    const DecBlock blk = blks[bi];
    const DecChunk d = dcs[static_cast<uint64_t>(bi) * nch_max + c];
    const uint64_t nch = (info.count + kChunk - 1) / kChunk;
    if (kMode == kCodes && psrc) {
        // a chunk the first permutation pass can read from the payload (see
        // PermSrc) is not decoded here; every other chunk gets meta 0
        PermSrc r{nullptr, 0u, 0u};
        const bool full = c < nch && chunk_len(info.count, c) == kChunk;
        if ((info.flags & 3) == 1 || (!(info.flags & 3) && full && d.ztag == 1)) r.meta = 1u << 13;  // all zero
        if (!(info.flags & 3) && c < nch && chunk_len(info.count, c) == kChunk && d.ztag == 0 && d.stag != 2 && info.width >= 1 && info.width <= 16) {
            const int64_t qbase = info.code_min - t.qlo;
            const int64_t top = qbase + static_cast<int64_t>((1ull << info.width) - 1);
            if (qbase >= t.idem_lo - t.qlo && top <= t.idem_hi - t.qlo) {
                const uintptr_t cs = reinterpret_cast<uintptr_t>(blk.in + info.code_seg);
                const uint64_t cb = static_cast<uint64_t>(cs & 7) * 8 + static_cast<uint64_t>(d.nz_prefix) * info.width;
                r.cw = reinterpret_cast<const uint64_t*>(cs & ~uintptr_t(7)) + (cb >> 6);
                r.qb = static_cast<uint32_t>(qbase);
                r.meta = static_cast<uint32_t>(cb & 63) | (info.width << 6) | (d.stag == 1 ? 1u << 11 : 0u) | (1u << 12);
            }
        }
        if (threadIdx.x == 0) psrc[blockIdx.x] = r;
        if (r.meta & (1u << 12)) return;
    }
    if (info.flags & 2) return;
    if (c >= nch) return;
    const uint32_t len = chunk_len(info.count, c);
    double* dst = blk.out + static_cast<uint64_t>(c) * kChunk;
    uint32_t* cdst = reinterpret_cast<uint32_t*>(blk.out) + static_cast<uint64_t>(c) * kChunk;
    const int tid = threadIdx.x;
    // codes: chunks flagged all-zero (zflag) are left unwritten and the first
    // permutation pass reads them as zeros; doubles with wflag: one flag per
    // 32-scalar group (1 = stored, 0 = all zero and not stored)
    uint8_t* gflag = (kMode == kDoubles && wflag) ? wflag + (static_cast<uint64_t>(bi) * nch_max + c) * 128 : nullptr;
    const bool skip_zero = (kMode == kCodes && skip_zero_chunks) || gflag;
    if (info.flags & 1) {
        if (gflag && tid < 128) gflag[tid] = 0;
        if (skip_zero) return;
        if constexpr (kMode != kSumsOnly) {
            for (uint32_t s = tid; s < len; s += kChunkThreads) {
                if (kMode == kCodes)
                    cdst[s] = 1u;
                else
                    dst[s] = 0.0;
            }
        }
        return;
    }
    if (skip_zero && d.ztag == 1 && len == kChunk) {
        if (gflag && tid < 128) gflag[tid] = 0;
        return;
    }
    {
        // Warm L1 with the chunk's code bytes (at most len codes from its
        // first rank on): the per-word code fetches below then hit L1 instead
        // of each paying a DRAM round trip.
        const uint8_t* c0 = blk.in + info.code_seg + ((static_cast<uint64_t>(d.nz_prefix) * info.width) >> 3);
        const uint32_t span = (len * info.width + 7) / 8 + 8;
        const uintptr_t line0 = reinterpret_cast<uintptr_t>(c0) & ~uintptr_t(127);
        const uint32_t nlines = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(c0) + span - line0 + 127) >> 7);
        for (uint32_t l = tid; l < nlines; l += kChunkThreads)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(line0 + 128ull * l));
    }
    __shared__ uint32_t s_sign[kWordsPerChunk], s_nz[kWordsPerChunk], s_pre[kWordsPerChunk];
    __shared__ double s_red[3][4];
    {
        const uint32_t vm = word_mask(len, tid);
        uint32_t sw = 0, zw = 0;
        if (vm) {
            sw = d.stag == 1 ? vm : (d.stag == 2 ? load_u32_unaligned(blk.in + d.sign_off + 4 * tid) & vm : 0);
            zw = d.ztag == 1 ? vm : (d.ztag == 2 ? load_u32_unaligned(blk.in + d.zero_off + 4 * tid) & vm : 0);
        }
        s_sign[tid] = sw;
        s_nz[tid] = ~zw & vm;
        using Scan = cub::BlockScan<uint32_t, kChunkThreads>;
        __shared__ typename Scan::TempStorage ss;
        uint32_t pre;
        Scan(ss).ExclusiveSum(static_cast<uint32_t>(__popc(~zw & vm)), pre);
        s_pre[tid] = pre;
    }
    __syncthreads();
    const uint32_t width = info.width;
    // valid packed offsets: the idempotent window (codes) or the dequantisation table
    const int64_t lo = (kMode == kCodes ? t.idem_lo : t.qlo) - t.qlo, hi = (kMode == kCodes ? t.idem_hi : t.qhi) - t.qlo;
    const int64_t qbase = info.code_min - t.qlo;
    const int64_t top = width >= 63 ? INT64_MAX : qbase + static_cast<int64_t>((1ull << width) - 1);
    const bool check = qbase < lo || top > hi || top < qbase;
    double sq = 0.0, sre = 0.0, sim = 0.0;
    bool bad = false;
    const uint64_t half = info.count / 2, g0 = static_cast<uint64_t>(c) * kChunk;
    const uint8_t* codes = blk.in + info.code_seg;
    const bool sums = want_sums != 0;
    const uint32_t nnz_chunk = s_pre[kWordsPerChunk - 1] + __popc(s_nz[kWordsPerChunk - 1]);
    if (kMode == kSumsOnly && len == kChunk && !check && width == 1 && nnz_chunk == kChunk &&
        (half & (kChunk - 1)) == 0) {
        // sums of a zero-free chunk of one-bit codes: every scalar is +-E[qb]
        // or +-E[qb + 1], so each thread counts its 32 codes and signs
        const uintptr_t cs = reinterpret_cast<uintptr_t>(codes);
        const uint64_t cb = static_cast<uint64_t>(cs & 3) * 8 + d.nz_prefix;
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(cs & ~uintptr_t(3)) + (cb >> 5);
        const uint32_t a = static_cast<uint32_t>(cb & 31) + 32u * tid;
        const uint32_t code = __funnelshift_r(__ldg(cw + (a >> 5)), __ldg(cw + (a >> 5) + 1), a & 31);
        const uint32_t sg = s_sign[tid];
        const uint32_t qb = static_cast<uint32_t>(qbase);
        const double m0 = __ldg(t.dequant + qb), m1 = __ldg(t.dequant + qb + 1);
        const int n1 = __popc(code), n0 = 32 - n1;
        const int neg1 = __popc(code & sg), neg0 = __popc(~code & sg);
        sq = n0 * (m0 * m0) + n1 * (m1 * m1);
        const double vs = m0 * (n0 - 2 * neg0) + m1 * (n1 - 2 * neg1);
        if (g0 < half)  // (the chunk lies in one half)
            sre = vs;
        else
            sim = vs;
    } else if (kMode != kSumsOnly && len == kChunk && !check && width <= 16 && nnz_chunk == kChunk) {
        // No zero in the chunk and narrow codes: scalar s has rank s, so each
        // thread decodes four consecutive scalars from one 64-bit window and
        // writes them with 16-byte stores.
        const uintptr_t cs = reinterpret_cast<uintptr_t>(codes);
        const uint64_t cb = static_cast<uint64_t>(cs & 3) * 8 + static_cast<uint64_t>(d.nz_prefix) * width;
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(cs & ~uintptr_t(3)) + (cb >> 5);
        const uint32_t cb0 = static_cast<uint32_t>(cb & 31), cmask = (1u << width) - 1;
        const uint32_t qb = static_cast<uint32_t>(qbase);
        if (gflag && tid < 128) gflag[tid] = 1;  // zero-free chunk
#pragma unroll 4
        for (int i = 0; i < kChunk / (4 * kChunkThreads); ++i) {
            const uint32_t s0 = 4 * tid + 4 * kChunkThreads * i;
            const uint32_t a = cb0 + s0 * width;
            const uint32_t w0 = __ldg(cw + (a >> 5)), w1 = __ldg(cw + (a >> 5) + 1), w2 = __ldg(cw + (a >> 5) + 2);
            const uint64_t win = ((static_cast<uint64_t>(__funnelshift_r(w1, w2, a & 31)) << 32) |
                                  __funnelshift_r(w0, w1, a & 31));
            const uint32_t sg = (s_sign[s0 >> 5] >> (s0 & 31)) & 15u;
            uint32_t c[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) c[e] = static_cast<uint32_t>(win >> (e * width)) & cmask;
            if constexpr (kMode == kCodes) {
                uint4 o;
                o.x = ((qb + c[0]) << 2) | ((sg & 1u) << 1);
                o.y = ((qb + c[1]) << 2) | (sg & 2u);
                o.z = ((qb + c[2]) << 2) | ((sg >> 1) & 2u);
                o.w = ((qb + c[3]) << 2) | ((sg >> 2) & 2u);
                __stcs(reinterpret_cast<uint4*>(cdst + s0), o);
            } else {
                double v[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const double m = __ldg(t.dequant + (qb + c[e]));
                    v[e] = ((sg >> e) & 1u) ? -m : m;
                    if (sums) {
                        sq += m * m;
                        if (g0 + s0 + e < half)
                            sre += v[e];
                        else
                            sim += v[e];
                    }
                }
                __stcs(reinterpret_cast<double2*>(dst + s0), make_double2(v[0], v[1]));
                __stcs(reinterpret_cast<double2*>(dst + s0 + 2), make_double2(v[2], v[3]));
            }
        }
    } else if (kMode == kDoubles && len == kChunk && !check && width <= 30 && nnz_chunk == kChunk) {
        // No zero in the chunk, wider codes: scalar s has rank s, its code at
        // bit cb0 + s w. Eight words per round: all code fetches, then all
        // dequantisation gathers (the latency-bound part) in flight together.
        const uintptr_t cs = reinterpret_cast<uintptr_t>(codes);
        const uint64_t cb = static_cast<uint64_t>(cs & 3) * 8 + static_cast<uint64_t>(d.nz_prefix) * width;
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(cs & ~uintptr_t(3)) + (cb >> 5);
        const uint32_t cb0 = static_cast<uint32_t>(cb & 31), cmask = (1u << width) - 1;
        const uint32_t qb = static_cast<uint32_t>(qbase);
        const int lane = tid & 31, w = tid >> 5;
        if (gflag && tid < 128) gflag[tid] = 1;  // zero-free chunk
#pragma unroll 1
        for (int h = 0; h < 32; h += 8) {
            uint32_t code[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint32_t a = cb0 + (32u * (4u * (h + e) + w) + lane) * width;
                code[e] = __funnelshift_r(__ldg(cw + (a >> 5)), __ldg(cw + (a >> 5) + 1), a & 31) & cmask;
            }
            double m[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) m[e] = __ldg(t.dequant + (qb + code[e]));
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const uint32_t k = 4u * (h + e) + w, sidx = 32u * k + lane;
                const double v = ((s_sign[k] >> lane) & 1u) ? -m[e] : m[e];
                if (sums) {
                    sq += m[e] * m[e];
                    if (g0 + sidx < half)
                        sre += v;
                    else
                        sim += v;
                }
                __stcs(dst + sidx, v);
            }
        }
    } else if (len == kChunk && !check)
        dec_scalars<kMode, true, false>(s_sign, s_nz, s_pre, codes, width, d.nz_prefix, len, qbase, lo, hi, t, dst,
                                        cdst, half, g0, sums, sq, sre, sim, bad, gflag);
    else
        dec_scalars<kMode, false, true>(s_sign, s_nz, s_pre, codes, width, d.nz_prefix, len, qbase, lo, hi, t, dst,
                                        cdst, half, g0, sums, sq, sre, sim, bad, gflag);
    if (bad) dev_fail(err, DE_CODE_WINDOW, bi);
    if (kMode == kSumsOnly || (kMode == kDoubles && want_sums)) block_sums3(sq, sre, sim, s_red, &infos[bi].sumsq);
}

// Mode 3: per-word row records instead of scalars (DecRow): a gate pass
// then decodes each 32-scalar row itself (k_stream_pass, FusedDecode). A
// failed or ALL_ZERO block gets all-zero rows (a failure is reported by the
// index kernel and raised after the stage).
__global__ void __launch_bounds__(kChunkThreads) k_dec_rows(const DecBlock* __restrict__ blks, uint32_t nch_max,
                                                            const DecInfo* __restrict__ infos,
                                                            const DecChunk* __restrict__ dcs,
                                                            DecRow* __restrict__ rows) {
    const uint32_t bi = blockIdx.x / nch_max, c = blockIdx.x % nch_max;
    const DecInfo info = infos[bi];
    const DecBlock blk = blks[bi];
    const DecChunk d = dcs[static_cast<uint64_t>(bi) * nch_max + c];
    const uint32_t tid = threadIdx.x;
    DecRow* out = rows + (static_cast<uint64_t>(bi) * nch_max + c) * kWordsPerChunk;
    const uint64_t nch = (info.count + kChunk - 1) / kChunk;
    if ((info.flags & 3) || c >= nch) {
        out[tid] = DecRow{0u, 0u, 0u, 0u};
        return;
    }
    const uint32_t len = chunk_len(info.count, c);
    const uint32_t vm = word_mask(len, tid);
    uint32_t sw = 0, zw = 0;
    if (vm) {
        sw = d.stag == 1 ? vm : (d.stag == 2 ? load_u32_unaligned(blk.in + d.sign_off + 4 * tid) & vm : 0);
        zw = d.ztag == 1 ? vm : (d.ztag == 2 ? load_u32_unaligned(blk.in + d.zero_off + 4 * tid) & vm : 0);
    }
    const uint32_t nz = ~zw & vm;
    using Scan = cub::BlockScan<uint32_t, kChunkThreads>;
    __shared__ typename Scan::TempStorage ss;
    uint32_t pre;
    Scan(ss).ExclusiveSum(static_cast<uint32_t>(__popc(nz)), pre);
    out[tid] = DecRow{nz, sw & nz, d.nz_prefix + pre, 0u};
}

}  // namespace

void launch_decompress(cudaStream_t st, const DecBlock* d_blks, uint64_t nblk, uint32_t nch_max, const DevTables& t,
                       DecInfo* d_info, DecChunk* d_dc, bool check_bound, bool want_sums, DevError* d_err,
                       uint64_t* launches, int mode, uint8_t* zflag, uint32_t* imnz, DecRow* rows,
                       PermSrc* psrc) {
    if (nblk == 0) return;
    BMQ_CUDA(cudaMemsetAsync(d_info, 0, nblk * sizeof(DecInfo), st));
    // mode 1: zflag = per-chunk zero flags (index kernel); mode 0: zflag =
    // per-32-scalar group flags (decode kernel)
    k_dec_index<<<static_cast<uint32_t>(nblk), kIndexThreads, 0, st>>>(d_blks, nch_max, d_info, d_dc, t,
                                                                        check_bound ? 1 : 0, d_err,
                                                                        mode == 1 ? zflag : nullptr,
                                                                        mode == 1 && zflag ? imnz : nullptr,
                                                                        mode == 0 && zflag ? imnz : nullptr);
    const uint32_t grid = static_cast<uint32_t>(nblk * nch_max);
    if (mode == 3)
        k_dec_rows<<<grid, kChunkThreads, 0, st>>>(d_blks, nch_max, d_info, d_dc, rows);
    else if (mode == 1)
        k_dec_chunk<kCodes><<<grid, kChunkThreads, 0, st>>>(d_blks, nch_max, d_info, d_dc, t, 0, d_err,
                                                             zflag ? 1 : 0, nullptr, psrc);
    else if (mode == 2)
        k_dec_chunk<kSumsOnly><<<grid, kChunkThreads, 0, st>>>(d_blks, nch_max, d_info, d_dc, t, 1, d_err, 0,
                                                               nullptr);
    else
        k_dec_chunk<kDoubles><<<grid, kChunkThreads, 0, st>>>(d_blks, nch_max, d_info, d_dc, t, want_sums ? 1 : 0,
                                                              d_err, 0, zflag);
    BMQ_CUDA(cudaGetLastError());
    if (launches) *launches += 2;
}

}  // namespace bmq
