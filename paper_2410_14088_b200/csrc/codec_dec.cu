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
