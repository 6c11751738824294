// engine.cu — device implementation of cbq::Simulator (engine.hpp:58-250).
//
// State: the compressed payload of every block id lives in an append-only
// device arena (payloads 16-byte aligned); ids whose payload is the
// canonical ALL_ZERO header are virtual (no bytes stored). When the arena
// fills, live payloads are compacted into the second arena.
//
// A stage runs in batches sized to the working set:
//   descriptors -> decompress the batch's blocks into planar buffers
//   -> gate program (last pass quantises in place: packed code words)
//   -> plan -> alloc (append) -> zero -> emit.
// Work skipped without changing a single output byte:
//   * groups whose blocks are all ALL_ZERO (linear gates map 0 to 0 and the
//     codec's ALL_ZERO payload is canonical, codec.hpp:263-271);
//   * with BMQ_FLAG_IDENTITY_SKIP, in stages made only of diagonal gates,
//     blocks on which no gate acts: their payload is left in place, which
//     equals compress(decompress(p)) because the codec is idempotent on every
//     code a finite amplitude can produce (codec_tables.cpp checks this).
// Per-id payload sizes come back to the host once per stage to replay the
// reference BlockStore accounting (peak footprint, spills) in its put order.
#include <cub/block/block_scan.cuh>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "engine.cuh"

namespace bmq {

// ----------------------------------------------------------- StoreModel

void StoreModel::reset(uint64_t num_ids, uint64_t budget) {
    size_.assign(num_ids, 0);
    flags_.assign(num_ids, 4);  // bit2: absent
    budget_ = budget;
    resident_ = spilled_live_ = peak_ = spilled_blocks_ = 0;
    shared_refs_ = shared_size_ = 0;
    shared_spilled_ = false;
}

void StoreModel::detach(uint64_t id) {  // detach_locked (store.hpp:192-212)
    uint8_t& f = flags_[id];
    if (f & 4) return;
    if (f & 2) {
        if (--shared_refs_ == 0) (shared_spilled_ ? spilled_live_ : resident_) -= shared_size_;
    } else {
        ((f & 1) ? spilled_live_ : resident_) -= size_[id];
    }
    f = 4;
}

bool StoreModel::place(uint64_t size) {  // fits_locked (store.hpp:188-190)
    if (size <= budget_ && resident_ <= budget_ - size) {
        resident_ += size;
        return false;
    }
    spilled_live_ += size;
    ++spilled_blocks_;
    return true;
}

void StoreModel::put(uint64_t id, uint64_t size) {  // put (store.hpp:64-83)
    detach(id);
    flags_[id] = place(size) ? 1 : 0;
    size_[id] = size;
    peak_ = std::max(peak_, resident_ + spilled_live_);
}

void StoreModel::put_shared(uint64_t first, uint64_t last, uint64_t size) {  // store.hpp:85-117
    for (uint64_t id = first; id < last; ++id) detach(id);
    shared_spilled_ = place(size);
    shared_size_ = size;
    shared_refs_ = last - first;
    for (uint64_t id = first; id < last; ++id) {
        flags_[id] = 2;
        size_[id] = size;
    }
    peak_ = std::max(peak_, resident_ + spilled_live_);
}

void StoreModel::serialize(std::vector<uint8_t>& out) const {
    const uint64_t n = size_.size();
    const uint64_t head[9] = {n, budget_, resident_, spilled_live_, peak_, spilled_blocks_, shared_refs_,
                              shared_size_, shared_spilled_ ? 1ull : 0ull};
    const size_t at = out.size();
    out.resize(at + sizeof head + n * 8 + n);
    std::memcpy(out.data() + at, head, sizeof head);
    std::memcpy(out.data() + at + sizeof head, size_.data(), n * 8);
    std::memcpy(out.data() + at + sizeof head + n * 8, flags_.data(), n);
}

void StoreModel::deserialize(const uint8_t* p, uint64_t nbytes) {
    uint64_t head[9];
    if (nbytes < sizeof head) raise(BMQ_ERR_STORE, "checkpoint: truncated store accounting");
    std::memcpy(head, p, sizeof head);
    const uint64_t n = head[0];
    if (n != size_.size() || nbytes != sizeof head + n * 9) raise(BMQ_ERR_STORE, "checkpoint: store accounting does not match the layout");
    budget_ = head[1];
    resident_ = head[2];
    spilled_live_ = head[3];
    peak_ = head[4];
    spilled_blocks_ = head[5];
    shared_refs_ = head[6];
    shared_size_ = head[7];
    shared_spilled_ = head[8] != 0;
    std::memcpy(size_.data(), p + sizeof head, n * 8);
    std::memcpy(flags_.data(), p + sizeof head + n * 8, n);
}

// ---------------------------------------------------------------- kernels

namespace {

constexpr uint32_t kArenaAlign = 16;
constexpr uint64_t kHostTag = 1ull << 62;  // payload offset refers to the pinned host arena
constexpr uint64_t kDiskTag = 1ull << 61;  // payload offset refers to the disk level (store_disk.cpp)
constexpr uint64_t kLevelTags = kHostTag | kDiskTag;

__global__ void k_fill_meta(uint64_t* off, uint64_t* size, uint64_t n, uint64_t zero_size) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        off[i] = ~0ull;
        size[i] = zero_size;
    }
}

// pf_off (optional): per batch slot, offset of the payload's prefetched copy
// in pf_base (~0 = not prefetched: device payloads, or host payloads read in
// place through the mapped address)
__global__ void k_build_desc(const uint64_t* __restrict__ ids, uint64_t nblk, const uint64_t* __restrict__ off,
                             const uint64_t* __restrict__ size, const uint8_t* pool, const uint8_t* host_pool,
                             const uint8_t* zero_hdr, double* work, uint32_t* pk, uint32_t b, DecBlock* dec,
                             CmpBlock* cmp, int codes, const uint64_t* __restrict__ pf_off = nullptr,
                             const uint8_t* pf_base = nullptr) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= nblk) return;
    const uint64_t id = ids[i];
    const uint64_t count = 2ull << b;
    double* slot = work + i * count;
    const uint64_t o = off[id];
    const uint64_t pf = pf_off ? pf_off[i] : ~0ull;
    DecBlock d;
    d.in = o == ~0ull ? zero_hdr
                      : (pf != ~0ull ? pf_base + pf : ((o & kHostTag) ? host_pool + (o & ~kHostTag) : pool + o));
    d.size = o == ~0ull ? kHeaderBytes : size[id];
    d.out = codes ? reinterpret_cast<double*>(pk + i * count) : slot;  // codes: decode to packed words
    d.expect_count = count;
    dec[i] = d;
    cmp[i] = CmpBlock{slot, pk + i * count, count, id};
}

__global__ void k_store_dec_sums(const DecInfo* __restrict__ di, const uint64_t* __restrict__ ids, uint64_t nblk,
                                 double* sums) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= nblk) return;
    const uint64_t id = ids[i];
    sums[3 * id] = di[i].sumsq;
    sums[3 * id + 1] = di[i].sum_re;
    sums[3 * id + 2] = di[i].sum_im;
}

// In-place compaction moves (store.hpp): one CTA per payload, 16-byte words
// (arena payloads are 16-byte aligned, sizes rounded up to whole words).
struct Move {
    uint64_t src, dst, words;
};

__global__ void k_move_payloads(const Move* __restrict__ mv, uint64_t n, const uint8_t* src_base, uint8_t* dst_base) {
    for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const Move m = mv[i];
        const uint4* s = reinterpret_cast<const uint4*>(src_base + m.src);
        uint4* d = reinterpret_cast<uint4*>(dst_base + m.dst);
        for (uint64_t w = threadIdx.x; w < m.words; w += blockDim.x) d[w] = s[w];
    }
}

// Heap-mode placement: per block the payload size (~0: virtual ALL_ZERO) for
// the host allocator, then the chosen places back into the plans and metadata
__global__ void k_plan_sizes(const BlockPlan* __restrict__ bps, uint64_t n, uint64_t* out) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = (bps[i].flags & 1) ? ~0ull : bps[i].size;
}

// Stage fusion: the intermediate stage's packed code words back to doubles,
// +-E[q] or +0 — decompress_block(compress_block(.)) scalar by scalar
// (codec.hpp:333-342), which depends on each scalar's code only.
__global__ void k_round(const uint4* __restrict__ pk, double2* __restrict__ out, uint64_t nquads,
                        const double* __restrict__ dequant) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < nquads;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint4 w = __ldcs(pk + i);
        const uint32_t c[4] = {w.x, w.y, w.z, w.w};
        double v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const double m = (c[e] & 1u) ? 0.0 : __ldg(dequant + (c[e] >> 2));
            v[e] = (c[e] & 3u) == 2u ? -m : m;
        }
        __stcs(out + 2 * i, make_double2(v[0], v[1]));
        __stcs(out + 2 * i + 1, make_double2(v[2], v[3]));
    }
}

// place[2i]: the payload's device address (arena or write-back staging),
// place[2i + 1]: its metadata offset (arena offset, or host extent | tag)
__global__ void k_place(BlockPlan* __restrict__ bps, const CmpBlock* __restrict__ blks, uint64_t n,
                        const uint64_t* __restrict__ place, uint64_t* off, uint64_t* size) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    BlockPlan& p = bps[i];
    const uint64_t id = blks[i].id;
    const bool virt = (p.flags & 1) != 0;
    p.out_off = virt ? ~0ull : place[2 * i];
    off[id] = virt ? ~0ull : place[2 * i + 1];
    size[id] = p.size;
}

// (id, off, size) triples -> per-id metadata (host-level batches)
__global__ void k_set_meta(const uint64_t* __restrict__ t, uint64_t n, uint64_t* off, uint64_t* size) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    off[t[3 * i]] = t[3 * i + 1];
    size[t[3 * i]] = t[3 * i + 2];
}

// Shard transfers: one CTA per payload, 16-byte words (arena payloads and
// transfer slots are 16-byte aligned; sizes are rounded up to whole words).
struct Xfer {
    uint64_t id, xoff, size;  // xoff: offset in the transfer buffer
    uint64_t dst;             // import: arena offset (tag included)
    double sums[3];
};

__global__ void k_pack_payloads(const Xfer* __restrict__ xs, uint64_t n, const uint64_t* __restrict__ off,
                                const uint8_t* pool, const uint8_t* host_pool, uint8_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const Xfer x = xs[i];
        if (!x.size) continue;
        const uint64_t o = off[x.id];
        if (o & kDiskTag) continue;  // read from the disk level by the host
        const uint4* s = reinterpret_cast<const uint4*>((o & kHostTag) ? host_pool + (o & ~kHostTag) : pool + o);
        uint4* d = reinterpret_cast<uint4*>(out + x.xoff);
        const uint64_t words = (x.size + 15) / 16;
        for (uint64_t w = threadIdx.x; w < words; w += blockDim.x) d[w] = s[w];
    }
}

// get_payloads: every payload of [first, first + n) back to back (byte
// offsets), ALL_ZERO ids as the canonical header, for one D2H copy.
__global__ void k_gather_payloads(const Xfer* __restrict__ xs, uint64_t n, const uint64_t* __restrict__ off,
                                  const uint8_t* pool, const uint8_t* host_pool, const uint8_t* zero_hdr,
                                  uint8_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const Xfer x = xs[i];
        const uint64_t o = off[x.id];
        if (o != ~0ull && (o & kDiskTag)) continue;  // read from the disk level by the host
        const uint8_t* s = o == ~0ull ? zero_hdr : ((o & kHostTag) ? host_pool + (o & ~kHostTag) : pool + o);
        uint8_t* d = out + x.xoff;
        const uint64_t head = (16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15;  // bytes until d is 16-aligned
        if (head == 0) {  // both ends aligned: 16-byte words, then the tail bytes
            const uint64_t words = x.size / 16;
            for (uint64_t w = threadIdx.x; w < words; w += blockDim.x)
                reinterpret_cast<uint4*>(d)[w] = reinterpret_cast<const uint4*>(s)[w];
            for (uint64_t k = words * 16 + threadIdx.x; k < x.size; k += blockDim.x) d[k] = s[k];
        } else {
            for (uint64_t k = threadIdx.x; k < x.size; k += blockDim.x) d[k] = s[k];
        }
    }
}

__global__ void k_unpack_payloads(const Xfer* __restrict__ xs, uint64_t n, const uint8_t* __restrict__ in,
                                  uint8_t* to, uint64_t tag, uint64_t* off, uint64_t* size, double* sums) {
    for (uint64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const Xfer x = xs[i];
        const bool disk = (x.dst & kDiskTag) != 0;  // written to the disk level by the host
        if (x.size && !disk) {
            const uint4* s = reinterpret_cast<const uint4*>(in + x.xoff);
            uint4* d = reinterpret_cast<uint4*>(to + x.dst);
            const uint64_t words = (x.size + 15) / 16;
            for (uint64_t w = threadIdx.x; w < words; w += blockDim.x) d[w] = s[w];
        }
        if (threadIdx.x == 0) {
            off[x.id] = x.size ? (disk ? x.dst : (x.dst | tag)) : ~0ull;
            size[x.id] = x.size ? x.size : kHeaderBytes;
            for (int k = 0; k < 3; ++k) sums[3 * x.id + k] = x.sums[k];
        }
    }
}

__global__ void k_drop_payloads(const uint64_t* __restrict__ ids, uint64_t n, uint64_t* off, uint64_t* size,
                                double* sums) {
    const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const uint64_t id = ids[i];
    off[id] = ~0ull;
    size[id] = kHeaderBytes;
    sums[3 * id] = sums[3 * id + 1] = sums[3 * id + 2] = 0.0;
}

// planar blocks [re(2^b) | im(2^b)] -> interleaved complex
__global__ void k_interleave(const double* __restrict__ planar, uint64_t nblk, uint32_t b, double* __restrict__ out) {
    const uint64_t total = nblk << b;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < total; p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t blk = p >> b, l = p & ((1ull << b) - 1);
        const double* src = planar + (blk << (b + 1));
        out[2 * p] = src[l];
        out[2 * p + 1] = src[(1ull << b) + l];
    }
}

__device__ __forceinline__ void block_reduce2(double re, double im, double* partial) {
    __shared__ double s[2][256];
    s[0][threadIdx.x] = re;
    s[1][threadIdx.x] = im;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (threadIdx.x < o) {
            s[0][threadIdx.x] += s[0][threadIdx.x + o];
            s[1][threadIdx.x] += s[1][threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        partial[2 * blockIdx.x] = s[0][0];
        partial[2 * blockIdx.x + 1] = s[1][0];
    }
}

// per-CTA partial sums of conj(ideal) * state (planar state, interleaved ideal)
__global__ void k_dot(const double* __restrict__ planar, const double* __restrict__ ideal, uint64_t nblk, uint32_t b,
                      double* __restrict__ partial) {
    const uint64_t total = nblk << b;
    double re = 0.0, im = 0.0;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < total; p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t blk = p >> b, l = p & ((1ull << b) - 1);
        const double* src = planar + (blk << (b + 1));
        const double sr = src[l], si = src[(1ull << b) + l];
        const double ir = ideal[2 * p], ii = -ideal[2 * p + 1];
        re += ir * sr - ii * si;
        im += ir * si + ii * sr;
    }
    block_reduce2(re, im, partial);
}

// per-CTA partial dot of two planar buffers: sum conj(a) * b
__global__ void k_dot2(const double* __restrict__ a, const double* __restrict__ bb, uint64_t nblk, uint32_t b,
                       double* __restrict__ partial) {
    const uint64_t total = nblk << b;
    double re = 0.0, im = 0.0;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < total; p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t blk = p >> b, l = p & ((1ull << b) - 1);
        const uint64_t o = blk << (b + 1);
        const double ar = a[o + l], ai = -a[o + (1ull << b) + l];
        const double br = bb[o + l], bi = bb[o + (1ull << b) + l];
        re += ar * br - ai * bi;
        im += ar * bi + ai * br;
    }
    block_reduce2(re, im, partial);
}

// per-block sums over a dense planar state (raw mode): sumsq, sum_re, sum_im
__global__ void k_block_sums(const double* __restrict__ planar, uint32_t b, double* __restrict__ sums) {
    const uint64_t blk = blockIdx.x;
    const double* src = planar + (blk << (b + 1));
    double sq = 0.0, sr = 0.0, si = 0.0;
    for (uint64_t l = threadIdx.x; l < (1ull << b); l += blockDim.x) {
        const double r = src[l], i = src[(1ull << b) + l];
        sq += r * r + i * i;
        sr += r;
        si += i;
    }
    __shared__ double s[3][256];
    s[0][threadIdx.x] = sq;
    s[1][threadIdx.x] = sr;
    s[2][threadIdx.x] = si;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (threadIdx.x < o)
            for (int k = 0; k < 3; ++k) s[k][threadIdx.x] += s[k][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int k = 0; k < 3; ++k) sums[3 * blk + k] = s[k][0];
}

uint32_t grid_for(uint64_t n, uint32_t threads = 256) {
    const uint64_t g = (n + threads - 1) / threads;
    return static_cast<uint32_t>(std::min<uint64_t>(std::max<uint64_t>(g, 1), 148ull * 64));
}

double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Does any gate of a diagonal-only stage act on a block with inner value v?
// Local condition bits can always be met inside the block.
std::vector<uint8_t> touched_table(const GateProgram& prog, uint32_t b, uint32_t k) {
    std::vector<uint8_t> t(1ull << k, 0);
    for (uint64_t v = 0; v < t.size(); ++v) {
        for (const GateOp& op : prog.ops) {
            const auto bit_ok = [&](uint32_t bit, uint32_t want) {
                return bit < b || ((v >> (bit - b)) & 1) == want;
            };
            bool acts = false;
            if (op.type == OP_DIAG) {
                acts = (op.et[0] != ET_ONE && bit_ok(op.hi, 0)) || (op.et[3] != ET_ONE && bit_ok(op.hi, 1));
            } else if (op.type == OP_CDIAG) {
                acts = op.et[15] != ET_ONE && bit_ok(op.hi, 1) && bit_ok(op.lo, 1);
            } else {
                acts = true;
            }
            if (acts) {
                t[v] = 1;
                break;
            }
        }
    }
    return t;
}

}  // namespace

// ------------------------------------------------------------------ Engine

Engine::Engine(uint32_t n, const bmq_gate* gates, uint64_t ngates, const bmq_config& cfg) : cfg_(cfg) {
    check_circuit(n, gates, ngates);
    if (cfg.disk_dir) disk_dir_ = cfg.disk_dir;  // (the caller's string need not outlive the call)
    cfg_.disk_dir = nullptr;
    if (cfg.disk_pool_bytes && !cfg.host_pool_bytes)
        raise(BMQ_ERR_INVALID_ARGUMENT, "the disk level needs a host level (host_pool_bytes > 0)");
    gates_.assign(gates, gates + ngates);
    L_ = make_layout(n, cfg.block_bits);
    if (cfg.flags & BMQ_FLAG_DEVICE_PLAN) {
        bmq_plan_model pm;
        bmq_plan_model_default(&pm);
        if (cfg.work_bytes) pm.work_bytes = cfg.work_bytes;
        pm.max_inner = cfg.inner_size;
        plan_ = plan_device_aware(n, gates, ngates, cfg.block_bits, pm, &plan_choice_);
    } else {
        plan_ = partition_plan(n, gates, ngates, cfg.block_bits, cfg.inner_size);
    }
    if (!(cfg.error_bound > 0.0) || std::isinf(cfg.error_bound))
        raise(BMQ_ERR_INVALID_ARGUMENT, "relative error bound must be positive and finite");
    if (cfg.workers < 1) raise(BMQ_ERR_INVALID_ARGUMENT, "worker count must be at least 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        raise(BMQ_ERR_NO_DEVICE, "no CUDA device available (the engine has no CPU fallback)");
    }
    if (cfg.device < 0 || cfg.device >= ndev) raise(BMQ_ERR_INVALID_ARGUMENT, "invalid CUDA device ordinal");
    dev_ = cfg.device;
    BMQ_CUDA(cudaSetDevice(dev_));
    BMQ_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    BMQ_CUDA(cudaEventCreate(&ev0_));
    BMQ_CUDA(cudaEventCreate(&ev1_));
    const bool raw = !cfg.compress;
    uint32_t kmax = 0;
    for (const bmq_stage& s : plan_) {
        auto sp = std::make_unique<StagePlan>();
        sp->stage = s;
        sp->gg = group_geometry(L_, s);
        kmax = std::max(kmax, s.inner_count);
        std::vector<GateOp> ops;
        for (uint64_t i = s.gate_begin; i < s.gate_end; ++i) {
            const bmq_gate& g = gates_[i];
            const bool two = gate_is_two_qubit(g.kind);
            if (raw) {
                ops.push_back(make_op(g, g.q0, two ? g.q1 : 0));
            } else {
                const uint32_t hi = buffer_bit(L_, s, g.q0);
                const uint32_t lo = two ? buffer_bit(L_, s, g.q1) : 0;
                ops.push_back(make_op(g, hi, lo));
            }
        }
        build_program(sp->prog, std::move(ops), raw ? L_.n : L_.b + s.inner_count);
        if (!raw && sp->prog.all_diagonal) {
            bool local_tiles = L_.b >= kMaxTileBits;
            for (const GatePass& p : sp->prog.passes) local_tiles = local_tiles && p.fast && !(p.tile_mask >> L_.b);
            if (local_tiles) {
                sp->diag_only = true;
                sp->touched = touched_table(sp->prog, L_.b, s.inner_count);
            }
        }
        stage_plans_.push_back(std::move(sp));
    }
    const uint64_t nid = L_.num_blocks();
    const uint64_t blk_scalars = 2ull << L_.b;
    size_t free_b = 0, total_b = 0;
    BMQ_CUDA(cudaMemGetInfo(&free_b, &total_b));
    off_.alloc(nid);
    size_.alloc(nid);
    sums_.alloc(3 * nid);
    err_.alloc(1);
    cursor_.alloc(8);
    red_.alloc(2 * 148 * 64);
    BMQ_CUDA(cudaMemset(err_.p, 0, sizeof(DevError)));
    BMQ_CUDA(cudaMemset(cursor_.p, 0, 4 * sizeof(uint64_t)));
    // pinned host mirrors: the per-stage metadata copies run at full link
    // speed instead of through pageable staging
    h_off_.assign(nid, ~0ull);
    h_size_.assign(nid, 0);
    if (raw) {
        dense_.alloc(nid * blk_scalars);
        work_scalars_ = 0;
        device_peak_ = dense_.bytes();
        return;
    }
    tabs_ = &device_tables(cfg.error_bound);
    {
        const CodecTables& h = host_tables(cfg.error_bound);
        // every code up to the one of DBL_MAX/(1+b_r) round-trips exactly
        identity_ok_ = h.idem_lo == h.qlo && h.idem_hi >= h.qhi - 1;
    }
    const uint64_t group_bytes = 8ull * (blk_scalars << kmax);
    // Automatic sizes are fractions of the device's total HBM (free memory is
    // misleading once the stream-ordered pool holds released buffers).
    uint64_t want = cfg.work_bytes ? cfg.work_bytes
                                   : std::min<uint64_t>({16ull << 30, total_b / 8, 16ull << L_.n});
    want = std::max<uint64_t>(want, group_bytes);
    work_scalars_ = (want / 8) / blk_scalars * blk_scalars;
    max_blocks_ = work_scalars_ / blk_scalars;
    // bound the per-block scratch for tiny blocks (b small): at most 2^20
    // blocks per batch, but never less than one group
    const uint64_t min_blocks = 1ull << kmax;
    if (max_blocks_ > std::max<uint64_t>(min_blocks, 1ull << 20)) {
        max_blocks_ = std::max<uint64_t>(min_blocks, 1ull << 20);
        work_scalars_ = max_blocks_ * blk_scalars;
    }
    nch_ = static_cast<uint32_t>((blk_scalars + kChunk - 1) / kChunk);
    work_.alloc(work_scalars_);
    cmp_.alloc(max_blocks_);
    dec_.alloc(max_blocks_);
    cplan_.alloc(max_blocks_ * nch_);
    pk_.alloc(work_scalars_);
    bplan_.alloc(max_blocks_);
    dinfo_.alloc(max_blocks_);
    dchunk_.alloc(max_blocks_ * nch_);
    zflag_.alloc(max_blocks_ * nch_);
    psrc_.alloc(max_blocks_ * nch_);
    imnz_.alloc(1);
    wflag_.alloc(work_scalars_ / 32);
    if (L_.b >= 12 && getenv("BMQ_FUSED_DECODE")) rows_.alloc(work_scalars_ / 32);
    // second buffer set (batch k+1's front overlaps batch k's back): when
    // the device has room for it next to a payload arena of the same size
    two_sets_ = cfg.compress && !getenv("BMQ_DBG_ONE_SET") &&
                4 * (work_.bytes() + pk_.bytes() + wflag_.bytes()) < total_b;
    if (two_sets_) {
        work2_.alloc(work_scalars_);
        pk2_.alloc(work_scalars_);
        cmp2_.alloc(max_blocks_);
        dec2_.alloc(max_blocks_);
        cplan2_.alloc(max_blocks_ * nch_);
        bplan2_.alloc(max_blocks_);
        dinfo2_.alloc(max_blocks_);
        dchunk2_.alloc(max_blocks_ * nch_);
        zflag2_.alloc(max_blocks_ * nch_);
        psrc2_.alloc(max_blocks_ * nch_);
        imnz2_.alloc(1);
        wflag2_.alloc(work_scalars_ / 32);
    }
    ids_.alloc(std::max<uint64_t>(nid, max_blocks_));
    vtab_.alloc(std::max<uint64_t>(nid, max_blocks_));
    new_off_.alloc(nid);
    live_ids_.alloc(nid);
    // canonical ALL_ZERO payload (codec.hpp:263-271) + slack
    uint8_t hdr[kHeaderBytes + 16] = {};
    const uint64_t cnt = blk_scalars;
    for (int k = 0; k < 8; ++k) hdr[k] = static_cast<uint8_t>(cnt >> (8 * k));
    std::memcpy(hdr + 8, &cfg.error_bound, 8);
    hdr[25] = 1;
    zero_hdr_.alloc(sizeof hdr);
    BMQ_CUDA(cudaMemcpy(zero_hdr_.p, hdr, sizeof hdr, cudaMemcpyHostToDevice));
    // Device level: one VA range for the whole device, mapped on demand.
    // device_pool_bytes fixes the arena's capacity (unless BMQ_FLAG_POOL_GROW
    // makes it the initial size); automatic arenas start at min(24 GiB,
    // HBM / 8) and grow up to what the device has left.
    const uint64_t worst = nid * (compress_bound(blk_scalars) + kArenaAlign) + 64;
    const uint64_t others = work_.bytes() + pk_.bytes() + cplan_.bytes() + dchunk_.bytes() + zflag_.bytes() +
                            wflag_.bytes() + rows_.bytes() + work2_.bytes() + pk2_.bytes() + cplan2_.bytes() +
                            dchunk2_.bytes() + zflag2_.bytes() + wflag2_.bytes() + psrc_.bytes() + psrc2_.bytes() + 8 * (ids_.n + vtab_.n + new_off_.n + live_ids_.n + off_.n + size_.n) +
                            sums_.bytes();
    const uint64_t headroom = total_b > others + (6ull << 30) ? total_b - others - (6ull << 30) : (1ull << 30);
    arena_grow_ = cfg.device_pool_bytes == 0 || (cfg.flags & BMQ_FLAG_POOL_GROW);
    arena_max_ = arena_grow_ ? std::max<uint64_t>(std::min(worst, headroom), cfg.device_pool_bytes) : cfg.device_pool_bytes;
    arena_.init(dev_, std::min<uint64_t>(total_b, std::max<uint64_t>(arena_max_, 1ull << 30)) + (1ull << 30));
    const uint64_t initial = cfg.device_pool_bytes ? cfg.device_pool_bytes
                                                   : std::min<uint64_t>({24ull << 30, total_b / 8, arena_max_});
    if (!arena_.grow_to(initial + 64)) raise(BMQ_ERR_OUT_OF_MEMORY, "device payload arena: out of memory");
    arena_limit_ = initial;
    heap_mode_ = (cfg.flags & BMQ_FLAG_HEAP_ARENA) != 0;
    arena_auto_ = !(cfg.flags & (BMQ_FLAG_HEAP_ARENA | BMQ_FLAG_BUMP_ARENA)) && nid <= (1ull << 17);
    h_place_.assign(2 * max_blocks_, 0);
    d_place_.alloc(2 * max_blocks_);
    if (two_sets_) {
        h_place2_.assign(2 * max_blocks_, 0);
        d_place2_.alloc(2 * max_blocks_);
        BMQ_CUDA(cudaStreamCreateWithFlags(&st2_, cudaStreamNonBlocking));
        BMQ_CUDA(cudaEventCreateWithFlags(&ev_emitted_, cudaEventDisableTiming));
        BMQ_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    }
    BMQ_CUDA(cudaStreamCreateWithFlags(&cp_in_, cudaStreamNonBlocking));
    BMQ_CUDA(cudaStreamCreateWithFlags(&cp_out_, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        BMQ_CUDA(cudaEventCreateWithFlags(&ev_pf_[k], cudaEventDisableTiming));
        BMQ_CUDA(cudaEventCreateWithFlags(&ev_dec_[k], cudaEventDisableTiming));
    }
    BMQ_CUDA(cudaEventCreateWithFlags(&ev_emit_, cudaEventDisableTiming));
    BMQ_CUDA(cudaEventCreateWithFlags(&ev_wb_, cudaEventDisableTiming));
    device_peak_ = arena_.mapped() + others;
}

Engine::~Engine() {
    cudaSetDevice(dev_);
    use_set(0);
    for (cudaStream_t* q : {&st_, &st2_, &cp_in_, &cp_out_})
        if (*q) {
            cudaStreamSynchronize(*q);
            cudaStreamDestroy(*q);
        }
    for (cudaEvent_t e : {ev_pf_[0], ev_pf_[1], ev_dec_[0], ev_dec_[1], ev_emit_, ev_wb_, ev_emitted_, ev_join_})
        if (e) cudaEventDestroy(e);
    for (auto& [a, b] : link_ev_) {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    if (ev0_) cudaEventDestroy(ev0_);
    if (ev1_) cudaEventDestroy(ev1_);
    for (cudaEvent_t e : phase_ev_) cudaEventDestroy(e);
    if (host_pool_) cudaFreeHost(host_pool_);
}

uint32_t Engine::peek_error() {
    DevError e{};
    BMQ_CUDA(cudaMemcpyAsync(&e, err_.p, sizeof e, cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
    return e.code;
}

void Engine::check_device_error(const char* what) {
    const uint32_t code = peek_error();
    if (code) {
        BMQ_CUDA(cudaMemsetAsync(err_.p, 0, sizeof(DevError), st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
        raise(dev_error_status(code), std::string(what) + dev_error_message(code));
    }
}

void Engine::sync_meta_to_host() {
    BMQ_CUDA(cudaMemcpyAsync(h_off_.data(), off_.p, off_.bytes(), cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaMemcpyAsync(h_size_.data(), size_.p, size_.bytes(), cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
}

uint64_t Engine::arena_used() {
    uint64_t used = 0;
    BMQ_CUDA(cudaMemcpyAsync(&used, cursor_.p, 8, cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
    return used;
}

bool Engine::grow_arena(uint64_t limit) {
    if (limit <= arena_limit_) return true;
    if (!arena_grow_ || limit > arena_max_) return false;
    // grow by at least a quarter, so a run grows O(log) times
    const uint64_t want = std::min(arena_max_, std::max(limit, arena_limit_ + arena_limit_ / 4));
    const uint64_t before = arena_.mapped();
    if (!arena_.grow_to(want + 64) && !arena_.grow_to(limit + 64)) return false;
    arena_limit_ = std::min<uint64_t>(arena_.mapped() - 64, std::max(limit, want));
    device_peak_ += arena_.mapped() > before ? arena_.mapped() - before : 0;
    ++counters_.pool_growths;
    return true;
}

// Compaction in place: the device payloads of every id except `excl` (whose
// payloads the batch in flight has already decoded) slide down to the front
// of the arena in offset order. A window of payloads moves directly when all
// its destinations end before its first source; otherwise (little dead space
// in front of it) the window goes through the dead dense work buffer, packed
// then unpacked. Destinations never pass the sources of later windows, so the
// windows run back to back on st_.
void Engine::compact(const uint64_t* excl, uint64_t nexcl) {
    // the other buffer set's batch may still be decoding payloads this moves
    if (two_sets_) BMQ_CUDA(cudaStreamSynchronize(st2_));
    sync_meta_to_host();
    const uint64_t nid = L_.num_blocks();
    std::vector<uint8_t> dead(nid, 0);
    for (uint64_t i = 0; i < nexcl; ++i) dead[excl[i]] = 1;
    std::vector<uint64_t> live;
    for (uint64_t id = 0; id < nid; ++id) {
        const bool dev = h_off_[id] != ~0ull && !(h_off_[id] & kLevelTags);
        if (dev && dead[id]) h_off_[id] = ~0ull;  // the batch in flight decoded it: gone (its emit rewrites it)
        if (dev && !dead[id]) live.push_back(id);
    }
    std::sort(live.begin(), live.end(), [&](uint64_t x, uint64_t y) { return h_off_[x] < h_off_[y]; });
    const auto bytes_of = [&](uint64_t id) { return (h_size_[id] + kArenaAlign - 1) / kArenaAlign * kArenaAlign; };
    struct Seg {
        size_t first, count;
        int mode;  // 0 arena -> arena, 1 arena -> staging, 2 staging -> arena
    };
    std::vector<Move> mv;
    std::vector<Seg> segs;
    const uint64_t scap = work_.bytes() / kArenaAlign * kArenaAlign;
    uint64_t dst = 0, moved = 0;
    size_t i = 0;
    while (i < live.size()) {
        const uint64_t src0 = h_off_[live[i]];
        if (src0 == dst) {  // already in place
            dst += bytes_of(live[i++]);
            continue;
        }
        size_t j = i;
        for (uint64_t end = dst; j < live.size() && end + bytes_of(live[j]) <= src0; ++j) end += bytes_of(live[j]);
        if (j > i && (j - i >= 32 || j == live.size())) {
            segs.push_back(Seg{mv.size(), j - i, 0});
            for (size_t k = i; k < j; ++k) {
                const uint64_t id = live[k];
                mv.push_back(Move{h_off_[id], dst, bytes_of(id) / kArenaAlign});
                h_off_[id] = dst;
                dst += bytes_of(id);
                moved += bytes_of(id);
            }
        } else {
            j = i;
            uint64_t sp = 0;
            while (j < live.size() && (j == i || sp + bytes_of(live[j]) <= scap)) sp += bytes_of(live[j++]);
            if (sp > scap) raise(BMQ_ERR_STORE, "payload larger than the compaction staging buffer");
            segs.push_back(Seg{mv.size(), j - i, 1});
            sp = 0;
            for (size_t k = i; k < j; ++k) {
                mv.push_back(Move{h_off_[live[k]], sp, bytes_of(live[k]) / kArenaAlign});
                sp += bytes_of(live[k]);
            }
            segs.push_back(Seg{mv.size(), j - i, 2});
            sp = 0;
            for (size_t k = i; k < j; ++k) {
                const uint64_t id = live[k];
                mv.push_back(Move{sp, dst, bytes_of(id) / kArenaAlign});
                sp += bytes_of(id);
                h_off_[id] = dst;
                dst += bytes_of(id);
                moved += 2 * bytes_of(id);
            }
        }
        i = j;
    }
    if (!mv.empty()) {
        DevArray<Move> dm;
        dm.alloc(mv.size());
        BMQ_CUDA(cudaMemcpyAsync(dm.p, mv.data(), mv.size() * sizeof(Move), cudaMemcpyHostToDevice, st_));
        uint8_t* arena = arena_.base();
        uint8_t* staging = reinterpret_cast<uint8_t*>(work_.p);
        for (const Seg& g : segs) {
            const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(g.count, 148 * 16));
            k_move_payloads<<<grid, 256, 0, st_>>>(dm.p + g.first, g.count, g.mode == 2 ? staging : arena,
                                                   g.mode == 1 ? staging : arena);
            ++counters_.kernel_launches;
        }
        BMQ_CUDA(cudaGetLastError());
        BMQ_CUDA(cudaMemcpyAsync(off_.p, h_off_.data(), off_.bytes(), cudaMemcpyHostToDevice, st_));
    }
    BMQ_CUDA(cudaMemcpyAsync(cursor_.p, &dst, 8, cudaMemcpyHostToDevice, st_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
    // automatic policy: a live state that fills a quarter of the arena is
    // rewritten at a cost this compaction just paid; from here on every
    // payload gets its own extent instead (no further compactions)
    if (arena_auto_ && !heap_mode_ && 4 * dst >= arena_limit_) heap_mode_ = true;
    if (heap_mode_) {  // the live payloads now fill [0, dst)
        dev_heap_.reset(arena_limit_, kArenaAlign);
        if (dst) dev_heap_.alloc(dst);
    }
    ++counters_.compactions;
    counters_.compact_bytes += moved;
}

// Room for `need` more bytes at the cursor. Compaction moves the live
// payloads once, so it runs when the garbage is at least the live state
// (amortised: one byte moved per byte written); otherwise the arena grows
// while the device has HBM for it, and compacts as the last resort.
bool Engine::make_room(uint64_t need, const uint64_t* excl, uint64_t nexcl) {
    sync_meta_to_host();
    const uint64_t used = arena_used();
    if (used + need <= arena_limit_) return true;
    std::vector<uint8_t> dead(L_.num_blocks(), 0);
    for (uint64_t i = 0; i < nexcl; ++i) dead[excl[i]] = 1;
    uint64_t live = 0;
    for (uint64_t id = 0; id < L_.num_blocks(); ++id)
        if (!dead[id] && h_off_[id] != ~0ull && !(h_off_[id] & kLevelTags))
            live += (h_size_[id] + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
    const uint64_t garbage = used > live ? used - live : 0;
    if (garbage >= live && live + need <= arena_limit_) {
        compact(excl, nexcl);
        return true;
    }
    if (grow_arena(used + need)) return true;
    if (live + need <= arena_limit_) {
        compact(excl, nexcl);
        return true;
    }
    if (grow_arena(live + need)) {
        compact(excl, nexcl);
        return true;
    }
    return false;
}

void Engine::init_state() {
    if (initialized_) raise(BMQ_ERR_ENGINE, "state already initialized");
    BMQ_CUDA(cudaSetDevice(dev_));
    const uint64_t nid = L_.num_blocks();
    const double one = 1.0;
    store_.reset(nid, cfg_.memory_budget);
    if (host_pool_) {
        sync_copies();
        host_heap_.reset(host_cap_, kArenaAlign);
    }
    if (disk_.is_open()) disk_.heap().reset(cfg_.disk_pool_bytes, kArenaAlign);
    BMQ_CUDA(cudaMemsetAsync(sums_.p, 0, sums_.bytes(), st_));
    if (!cfg_.compress) {
        const uint64_t raw = 16ull << L_.b;
        BMQ_CUDA(cudaMemsetAsync(dense_.p, 0, dense_.bytes(), st_));
        BMQ_CUDA(cudaMemcpyAsync(dense_.p, &one, 8, cudaMemcpyHostToDevice, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
        store_.put(0, raw);
        if (nid > 1) store_.put_shared(1, nid, raw);
        for (uint64_t id = 0; id < nid; ++id) h_size_[id] = raw;
        initialized_ = true;
        next_stage_ = 0;
        return;
    }
    k_fill_meta<<<grid_for(nid), 256, 0, st_>>>(off_.p, size_.p, nid, kHeaderBytes);
    BMQ_CUDA(cudaMemsetAsync(cursor_.p, 0, 2 * sizeof(uint64_t), st_));
    const uint64_t cnt = 2ull << L_.b;
    BMQ_CUDA(cudaMemsetAsync(work_.p, 0, cnt * sizeof(double), st_));
    BMQ_CUDA(cudaMemcpyAsync(work_.p, &one, 8, cudaMemcpyHostToDevice, st_));
    const CmpBlock blk{work_.p, pk_.p, cnt, 0};
    BMQ_CUDA(cudaMemcpyAsync(cmp_.p, &blk, sizeof blk, cudaMemcpyHostToDevice, st_));
    launch_compress(st_, cmp_.p, 1, nch_, *tabs_, arena_.base(), arena_limit_, cursor_.p, cursor_.p + 2, bplan_.p, cplan_.p,
                    off_.p, size_.p, true, false, err_.p, &counters_.kernel_launches);
    check_device_error("init_state: ");
    sums_ok_.assign(nid, 1);
    sums_ok_[0] = 0;
    sync_meta_to_host();
    heap_mode_ = (cfg_.flags & BMQ_FLAG_HEAP_ARENA) != 0;  // each run starts on the configured policy
    if (heap_mode_) {  // block 0's payload sits at offset 0
        dev_heap_.reset(arena_limit_, kArenaAlign);
        if (h_off_[0] != ~0ull) dev_heap_.alloc(h_size_[0]);
    }
    store_.put(0, h_size_[0]);
    if (nid > 1) store_.put_shared(1, nid, kHeaderBytes);  // one zero payload, counted once
    initialized_ = true;
    next_stage_ = 0;
    if (sharded() && owner(0, 0) != shard_rank_) {
        const uint64_t id0 = 0;
        drop_payloads(&id0, 1);
    }
}

void Engine::ensure_init() {
    if (!initialized_) init_state();
}

void Engine::reset() {
    BMQ_CUDA(cudaSetDevice(dev_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
    initialized_ = false;
    next_stage_ = 0;
    stage_compress_calls_ = stage_decompress_calls_ = 0;
    counters_ = bmq_report{};
}

void Engine::phase_event(size_t i) {
    while (phase_ev_.size() <= i) {
        cudaEvent_t e;
        BMQ_CUDA(cudaEventCreate(&e));
        phase_ev_.push_back(e);
    }
    BMQ_CUDA(cudaEventRecord(phase_ev_[i], st_));
}

void Engine::collect_phase_times(size_t nbatches) {
    for (size_t k = 0; k < nbatches; ++k) {
        float a = 0.f, b = 0.f, c = 0.f;
        BMQ_CUDA(cudaEventElapsedTime(&a, phase_ev_[4 * k], phase_ev_[4 * k + 1]));
        BMQ_CUDA(cudaEventElapsedTime(&b, phase_ev_[4 * k + 1], phase_ev_[4 * k + 2]));
        BMQ_CUDA(cudaEventElapsedTime(&c, phase_ev_[4 * k + 2], phase_ev_[4 * k + 3]));
        counters_.decompress_ms += a;
        counters_.gate_ms += b;
        counters_.compress_ms += c;
    }
    counters_.batches += nbatches;
}

void Engine::raw_run_stage(uint64_t s) {
    StagePlan& sp = *stage_plans_[s];
    run_program(st_, sp.prog, dense_.p, L_.b, false, 1, &counters_.kernel_launches);
    counters_.gate_passes += sp.prog.passes.size();
    BMQ_CUDA(cudaStreamSynchronize(st_));
    const uint64_t raw = 16ull << L_.b;
    const GroupGeometry& gg = sp.gg;
    std::vector<uint64_t> inner(gg.per_group());
    for (uint64_t v = 0; v < inner.size(); ++v) inner[v] = deposit_bits(v, gg.inner_mask);
    uint64_t o = 0;
    for (uint64_t g = 0; g < gg.groups(); ++g) {
        for (uint64_t v : inner) store_.put(o | v, raw);
        o = ((o | ~gg.outer_mask) + 1) & gg.outer_mask;
    }
    counters_.groups_processed += gg.groups();
    counters_.blocks_processed += L_.num_blocks();
    counters_.dense_bytes += 32ull << L_.n;
    counters_.model_bytes += 32ull << L_.n;
    counters_.model_groups += gg.groups();
    stage_compress_calls_ += L_.num_blocks();
    stage_decompress_calls_ += L_.num_blocks();
}

// alloc + zero + emit for the batch in flight into the device arena; when it
// does not fit, make room (compaction / growth, the batch's old payloads are
// dead) and try again; a batch that still does not fit goes to the host level.
void Engine::emit_batch(uint64_t nblk, const uint64_t* h_ids) {
    if (heap_mode_) return emit_placed(nblk, h_ids);
    for (int attempt = 0; attempt < 3; ++attempt) {
        launch_compress_emit(st_, cmp_.p, nblk, nch_, *tabs_, arena_.base(), arena_limit_, cursor_.p, cursor_.p + 2,
                             bplan_.p, cplan_.p, off_.p, size_.p, true, kArenaAlign, err_.p,
                             &counters_.kernel_launches);
        if (peek_error() != DE_POOL_FULL) {
            free_extents(h_ids, nblk);
            return;
        }
        BMQ_CUDA(cudaMemsetAsync(err_.p, 0, sizeof(DevError), st_));
        uint64_t need = 0;
        BMQ_CUDA(cudaMemcpyAsync(&need, cursor_.p + 1, 8, cudaMemcpyDeviceToHost, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
        if (!make_room(need, h_ids, nblk)) break;
        if (heap_mode_) return emit_placed(nblk, h_ids);  // the compaction switched the arena policy
    }
    if (!cfg_.host_pool_bytes) raise(BMQ_ERR_STORE, "device payload pool exhausted");
    emit_to_host(nblk, h_ids);
}

// Host level: emit into the write-back staging buffer (the dead work buffer
// when the batch outgrows it), give every payload its own host extent and
// copy the payloads there on cp_out_ while the next batch computes.
void Engine::emit_to_host(uint64_t nblk, const uint64_t* h_ids) {
    ensure_host_pool();
    BMQ_CUDA(cudaStreamWaitEvent(st_, ev_wb_, 0));  // the previous write-back has left wb_
    uint8_t* staging = wb_.p;
    bool in_work = false;
    for (int attempt = 0; attempt < 2; ++attempt) {
        BMQ_CUDA(cudaMemsetAsync(cursor_.p + 4, 0, 8, st_));
        launch_compress_emit(st_, cmp_.p, nblk, nch_, *tabs_, staging, (in_work ? work_.bytes() : wb_.bytes()) - 64,
                             cursor_.p + 4, cursor_.p + 2, bplan_.p, cplan_.p, nullptr, nullptr, true, kArenaAlign,
                             err_.p, &counters_.kernel_launches);
        if (peek_error() != DE_POOL_FULL) break;
        BMQ_CUDA(cudaMemsetAsync(err_.p, 0, sizeof(DevError), st_));
        if (in_work) raise(BMQ_ERR_STORE, "payload batch exceeds the staging buffer");
        staging = reinterpret_cast<uint8_t*>(work_.p);  // dead until the next batch decodes
        in_work = true;
    }
    std::vector<BlockPlan> bp(nblk);
    BMQ_CUDA(cudaMemcpyAsync(bp.data(), bplan_.p, nblk * sizeof(BlockPlan), cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaEventRecord(ev_emit_, st_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
    free_extents(h_ids, nblk);  // the batch's old payloads were decoded
    h_meta_.assign(3 * nblk, 0);
    std::vector<void*> dst, src;
    std::vector<size_t> len;
    uint64_t total = 0;
    for (uint64_t i = 0; i < nblk; ++i) {
        const uint64_t id = h_ids[i];
        uint64_t off = ~0ull, size = kHeaderBytes;
        if (!(bp[i].flags & 1)) {
            size = bp[i].size;
            const uint64_t ext = host_heap_.alloc(size);
            if (ext == ExtentHeap::kNone) {  // host level full: the disk level
                const uint64_t d = disk_alloc(size);
                disk_.write_from_device(staging + bp[i].out_off, size, d);
                off = d | kDiskTag;
                counters_.disk_spill_bytes += size;
            } else {
                off = ext | kHostTag;
                dst.push_back(host_pool_ + ext);
                src.push_back(staging + bp[i].out_off);
                len.push_back(size);
                total += size;
            }
        }
        h_meta_[3 * i] = id;
        h_meta_[3 * i + 1] = off;
        h_meta_[3 * i + 2] = size;
        h_off_[id] = off;
        h_size_[id] = size;
    }
    BMQ_CUDA(cudaStreamWaitEvent(cp_out_, ev_emit_, 0));
    link_event_pair(cp_out_, true);
    copy_batch(dst.data(), src.data(), len.data(), dst.size(), cp_out_);
    link_event_pair(cp_out_, false);
    BMQ_CUDA(cudaEventRecord(ev_wb_, cp_out_));
    if (in_work) BMQ_CUDA(cudaStreamWaitEvent(st_, ev_wb_, 0));  // the next decode overwrites work_
    BMQ_CUDA(cudaMemcpyAsync(d_meta_.p, h_meta_.data(), 3 * nblk * 8, cudaMemcpyHostToDevice, st_));
    k_set_meta<<<grid_for(nblk), 256, 0, st_>>>(d_meta_.p, nblk, off_.p, size_.p);
    ++counters_.kernel_launches;
    BMQ_CUDA(cudaGetLastError());
    counters_.host_spill_bytes += total;
    counters_.link_d2h_bytes += total;
    ++counters_.host_spill_batches;
}

uint64_t Engine::disk_alloc(uint64_t size) {
    if (!disk_.is_open()) raise(BMQ_ERR_STORE, "host payload pool exhausted");
    const uint64_t d = disk_.heap().alloc(size);
    if (d == ExtentHeap::kNone) raise(BMQ_ERR_STORE, "disk payload level exhausted");
    return d;
}

void Engine::free_extents(const uint64_t* ids, uint64_t n) {
    if (!host_pool_ && !heap_mode_) return;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t o = h_off_[ids[i]];
        if (o == ~0ull) continue;
        if (o & kDiskTag)
            disk_.heap().free(o & ~kDiskTag, h_size_[ids[i]]);
        else if (o & kHostTag)
            host_heap_.free(o & ~kHostTag, h_size_[ids[i]]);
        else if (heap_mode_)
            dev_heap_.free(o, h_size_[ids[i]]);
        else
            continue;  // bump mode: garbage until the next compaction
        h_off_[ids[i]] = ~0ull;  // until the next metadata sync
    }
}

uint64_t Engine::dev_alloc(uint64_t size) {
    uint64_t off = dev_heap_.alloc(size);
    if (off != ExtentHeap::kNone) return off;
    if (!grow_arena(arena_limit_ + size + kArenaAlign)) return ExtentHeap::kNone;
    dev_heap_.extend(arena_limit_);
    return dev_heap_.alloc(size);
}

// Heap mode: the batch's payload sizes come back to the host (the batch's old
// payloads, already decoded, are freed first), every payload gets an arena
// extent, or a host extent through the write-back staging buffer when the
// device is full, and the emit writes each payload in place.
void Engine::emit_placed(uint64_t nblk, const uint64_t* h_ids) {
    k_plan_sizes<<<grid_for(nblk), 256, 0, st_>>>(bplan_.p, nblk, d_place_.p);
    ++counters_.kernel_launches;
    BMQ_CUDA(cudaMemcpyAsync(h_place_.data(), d_place_.p, nblk * 8, cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
    std::vector<uint64_t> sz(h_place_.data(), h_place_.data() + nblk);
    free_extents(h_ids, nblk);
    std::vector<uint64_t> dev(nblk, ExtentHeap::kNone);
    std::vector<uint64_t> to_host;
    for (int attempt = 0;; ++attempt) {
        to_host.clear();
        for (uint64_t i = 0; i < nblk; ++i)
            if (sz[i] != ~0ull && (dev[i] = dev_alloc(sz[i])) == ExtentHeap::kNone) to_host.push_back(i);
        if (to_host.empty() || cfg_.host_pool_bytes || attempt > 0) break;
        // no host level: defragment once (the batch's ids hold nothing yet)
        for (uint64_t i = 0; i < nblk; ++i)
            if (dev[i] != ExtentHeap::kNone) dev_heap_.free(dev[i], sz[i]);
        compact(h_ids, nblk);
    }
    if (!to_host.empty() && !cfg_.host_pool_bytes) raise(BMQ_ERR_STORE, "device payload pool exhausted");
    uint8_t* staging = nullptr;
    std::vector<void*> dst, src;
    std::vector<size_t> len;
    uint64_t total = 0;
    if (!to_host.empty()) {
        ensure_host_pool();
        uint64_t need = 0;
        for (uint64_t i : to_host) need += (sz[i] + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
        staging = need <= wb_.bytes() ? wb_.p : reinterpret_cast<uint8_t*>(work_.p);  // work_ is dead until the next decode
        if (need > work_.bytes()) raise(BMQ_ERR_STORE, "payload batch exceeds the staging buffer");
        BMQ_CUDA(cudaStreamWaitEvent(st_, ev_wb_, 0));  // the previous write-back has left the staging buffer
    }
    uint64_t pos = 0;
    size_t th = 0;
    struct DiskWrite {
        const uint8_t* src;
        uint64_t size, off;
    };
    std::vector<DiskWrite> disk_w;
    for (uint64_t i = 0; i < nblk; ++i) {
        const uint64_t id = h_ids[i];
        uint64_t addr = 0, meta = ~0ull;
        if (sz[i] == ~0ull) {
            h_size_[id] = kHeaderBytes;
        } else if (dev[i] != ExtentHeap::kNone) {
            addr = reinterpret_cast<uint64_t>(arena_.base()) + dev[i];
            meta = dev[i];
            h_size_[id] = sz[i];
        } else {
            const uint64_t ext = host_heap_.alloc(sz[i]);
            addr = reinterpret_cast<uint64_t>(staging) + pos;
            if (ext == ExtentHeap::kNone) {  // host level full: the disk level, written after the emit
                const uint64_t d = disk_alloc(sz[i]);
                meta = d | kDiskTag;
                disk_w.push_back({staging + pos, sz[i], d});
            } else {
                meta = ext | kHostTag;
                dst.push_back(host_pool_ + ext);
                src.push_back(staging + pos);
                len.push_back(sz[i]);
                total += sz[i];
                ++th;
            }
            pos += (sz[i] + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
        }
        h_place_[2 * i] = addr;
        h_place_[2 * i + 1] = meta;
        h_off_[id] = meta;
    }
    BMQ_CUDA(cudaMemcpyAsync(d_place_.p, h_place_.data(), 2 * nblk * 8, cudaMemcpyHostToDevice, st_));
    k_place<<<grid_for(nblk), 256, 0, st_>>>(bplan_.p, cmp_.p, nblk, d_place_.p, off_.p, size_.p);
    launch_compress_emit_placed(st_, cmp_.p, nblk, nch_, *tabs_, bplan_.p, cplan_.p, err_.p,
                                &counters_.kernel_launches);
    ++counters_.kernel_launches;
    if (!disk_w.empty()) {  // the staged payloads are final once the emit has run
        BMQ_CUDA(cudaStreamSynchronize(st_));
        for (const DiskWrite& w : disk_w) {
            disk_.write_from_device(w.src, w.size, w.off);
            counters_.disk_spill_bytes += w.size;
        }
    }
    if (th) {
        BMQ_CUDA(cudaEventRecord(ev_emit_, st_));
        BMQ_CUDA(cudaStreamWaitEvent(cp_out_, ev_emit_, 0));
        link_event_pair(cp_out_, true);
        copy_batch(dst.data(), src.data(), len.data(), dst.size(), cp_out_);
        link_event_pair(cp_out_, false);
        BMQ_CUDA(cudaEventRecord(ev_wb_, cp_out_));
        if (staging != wb_.p) BMQ_CUDA(cudaStreamWaitEvent(st_, ev_wb_, 0));  // the next decode overwrites work_
        counters_.host_spill_bytes += total;
        counters_.link_d2h_bytes += total;
        ++counters_.host_spill_batches;
    }
    // (h_place_ is read by the H2D copy above; the next batch's emit only
    // rewrites it after a D2H copy into it on st_ has completed)
}

void Engine::ensure_host_pool() {
    if (host_pool_) return;
    host_cap_ = cfg_.host_pool_bytes;
    BMQ_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&host_pool_), host_cap_ + 64,
                           cudaHostAllocMapped | cudaHostAllocPortable));
    host_heap_.reset(host_cap_, kArenaAlign);
    // staging: write-back buffer and two prefetch slots of a quarter of the
    // dense working set each (at most 4 GiB); batches are cut so their
    // host-level payloads fit one slot
    const uint64_t slot = std::max<uint64_t>(std::min<uint64_t>(work_.bytes() / 4, 4ull << 30), 1ull << 20);
    wb_.alloc(slot + 64);
    for (int k = 0; k < 2; ++k) {
        pf_[k].alloc(slot + 64);  // (+64: decoders read whole words past a payload's last code)
        pf_off_[k].alloc(max_blocks_);
        h_pf_off_[k].assign(max_blocks_, ~0ull);
    }
    d_meta_.alloc(3 * max_blocks_);
    if (two_sets_) d_meta2_.alloc(3 * max_blocks_);
    device_peak_ += wb_.bytes() + 2 * slot + 2 * 8 * max_blocks_ + 24 * max_blocks_;
    if (cfg_.disk_pool_bytes && !disk_.is_open())
        disk_.open(disk_dir_, cfg_.disk_pool_bytes, kArenaAlign);
}

void Engine::copy_batch(void** dst, void** src, size_t* sizes, size_t n, cudaStream_t s) {
    // one cudaMemcpyAsync per run of payloads that are contiguous on both
    // sides (extents are placed in id order, so most batches collapse to a
    // few large copies)
    size_t i = 0;
    while (i < n) {
        char* d = static_cast<char*>(dst[i]);
        char* a = static_cast<char*>(src[i]);
        size_t len = sizes[i++];
        while (i < n && static_cast<char*>(dst[i]) == d + len && static_cast<char*>(src[i]) == a + len) len += sizes[i++];
        if (len) BMQ_CUDA(cudaMemcpyAsync(d, a, len, cudaMemcpyDefault, s));
    }
}

void Engine::link_event_pair(cudaStream_t s, bool start) {
    if (start) {
        if (link_ev_used_ == link_ev_.size()) {
            cudaEvent_t a, b;
            BMQ_CUDA(cudaEventCreate(&a));
            BMQ_CUDA(cudaEventCreate(&b));
            link_ev_.emplace_back(a, b);
        }
        BMQ_CUDA(cudaEventRecord(link_ev_[link_ev_used_].first, s));
    } else {
        BMQ_CUDA(cudaEventRecord(link_ev_[link_ev_used_++].second, s));
    }
}

void Engine::collect_link_times() {
    for (size_t k = 0; k < link_ev_used_; ++k) {
        float ms = 0.f;
        BMQ_CUDA(cudaEventElapsedTime(&ms, link_ev_[k].first, link_ev_[k].second));
        counters_.link_ms += ms;
    }
    link_ev_used_ = 0;
}

// The stage barrier for the copy streams: host-level bytes are final and the
// prefetch slots are free.
void Engine::sync_copies() {
    if (cp_in_) BMQ_CUDA(cudaStreamSynchronize(cp_in_));
    if (cp_out_) BMQ_CUDA(cudaStreamSynchronize(cp_out_));
    collect_link_times();
    pf_live_[0] = pf_live_[1] = false;
}

bool Engine::prefetch(const uint64_t* h_ids, uint64_t nblk, int slot) {
    if (!host_pool_ || (!host_heap_.used() && !(disk_.is_open() && disk_.heap().used()))) return false;
    BMQ_CUDA(cudaStreamWaitEvent(cp_in_, ev_dec_[slot], 0));  // batch k-2 has decoded out of this slot
    uint64_t* tab = h_pf_off_[slot].data();
    std::vector<void*> dst, src;
    std::vector<size_t> len;
    uint64_t pos = 0;
    bool waited = false;
    for (uint64_t i = 0; i < nblk; ++i) {
        const uint64_t o = h_off_[h_ids[i]];
        tab[i] = ~0ull;
        if (o == ~0ull || !(o & kLevelTags)) continue;
        const uint64_t size = h_size_[h_ids[i]];
        if (o & kDiskTag) {  // no mapped address: always through the slot (batches are cut to fit)
            if (pos + size > pf_[slot].bytes()) raise(BMQ_ERR_LOGIC, "disk-level payloads exceed the staging slot");
            if (!waited) BMQ_CUDA(cudaEventSynchronize(ev_dec_[slot]));  // (host-side writes into the slot)
            waited = true;
            disk_.read_to_device(pf_[slot].p + pos, size, o & ~kDiskTag);
            counters_.disk_read_bytes += size;
            tab[i] = pos;
            pos += (size + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
            continue;
        }
        if (pos + size > pf_[slot].bytes()) continue;  // read in place through the mapped address
        tab[i] = pos;
        dst.push_back(pf_[slot].p + pos);
        src.push_back(host_pool_ + (o & ~kHostTag));
        len.push_back(size);
        pos += (size + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
    }
    if (dst.empty() && !waited) return false;
    BMQ_CUDA(cudaMemcpyAsync(pf_off_[slot].p, tab, nblk * 8, cudaMemcpyHostToDevice, cp_in_));
    link_event_pair(cp_in_, true);
    copy_batch(dst.data(), src.data(), len.data(), dst.size(), cp_in_);
    link_event_pair(cp_in_, false);
    BMQ_CUDA(cudaEventRecord(ev_pf_[slot], cp_in_));
    uint64_t bytes = 0;
    for (size_t l : len) bytes += l;
    counters_.link_h2d_bytes += bytes;
    return true;
}

// Swap the current buffer set / stream with the other one (see BatchFront).
void Engine::use_set(int set) {
    if (!two_sets_ || set == cur_set_) return;
    std::swap(st_, st2_);
    work_.swap_with(work2_);
    pk_.swap_with(pk2_);
    cmp_.swap_with(cmp2_);
    dec_.swap_with(dec2_);
    cplan_.swap_with(cplan2_);
    bplan_.swap_with(bplan2_);
    dinfo_.swap_with(dinfo2_);
    dchunk_.swap_with(dchunk2_);
    zflag_.swap_with(zflag2_);
    psrc_.swap_with(psrc2_);
    imnz_.swap_with(imnz2_);
    wflag_.swap_with(wflag2_);
    d_place_.swap_with(d_place2_);
    h_place_.swap_with(h_place2_);
    d_meta_.swap_with(d_meta2_);
    h_meta_.swap_with(h_meta2_);
    cur_set_ = set;
}

// Back on set 0 with everything the other stream queued ordered before
// what st_ runs next.
void Engine::join_sets() {
    use_set(0);
    if (!two_sets_) return;
    BMQ_CUDA(cudaEventRecord(ev_join_, st2_));
    BMQ_CUDA(cudaStreamWaitEvent(st_, ev_join_, 0));
    emitted_live_ = false;
}

Engine::BatchFront Engine::process_front(StagePlan& sp, const uint64_t* d_ids, const uint32_t* d_vtab,
                                         uint64_t nblk, size_t bidx) {
    BatchFront f;
    phase_event(4 * bidx);
    // Code-domain stages (unit-entry monomial gates only) never leave the
    // quantiser codes: decode to packed words, permute them, emit.
    const bool codes = !d_vtab && sp.prog.mono && identity_ok_ && (cfg_.flags & BMQ_FLAG_CODE_DOMAIN);
    f.codes = codes;
    const int slot = static_cast<int>(bidx & 1);
    const bool pf = pf_live_[slot];
    if (pf) BMQ_CUDA(cudaStreamWaitEvent(st_, ev_pf_[slot], 0));  // host-level payloads prefetched
    k_build_desc<<<grid_for(nblk), 256, 0, st_>>>(d_ids, nblk, off_.p, size_.p, arena_.base(), host_pool_,
                                                  zero_hdr_.p, work_.p, pk_.p, L_.b, dec_.p, cmp_.p, codes ? 1 : 0,
                                                  pf ? pf_off_[slot].p : nullptr, pf_[slot].p);
    ++counters_.kernel_launches;
    // code-domain stages: all-zero chunks stay unwritten; the first
    // permutation pass reads them as zero words
    // zero skipping: code-domain stages flag all-zero chunks (zflag_), FP
    // stages all-zero 32-scalar groups (wflag_); neither is stored
    uint8_t* zf = codes ? (mono_zero_skip(sp.prog, L_.b) ? zflag_.p : nullptr)
                        : (program_zero_skip(sp.prog, L_.b, false) ? wflag_.p : nullptr);
    // imnz_: code domain, some imaginary-half chunk nonzero; FP: some group flag 0
    if (zf) BMQ_CUDA(cudaMemsetAsync(imnz_.p, 0, sizeof(uint32_t), st_));
    // Opt-in (BMQ_FUSED_DECODE=1): FP stages whose first pass streams decode
    // the payload rows inside it and the decoder only writes per-word row
    // records (no 16 B per amplitude round trip through HBM). Measured slower
    // on B200 (QAOA-3reg-30 @1e-4: 2.44 s against 1.80 s): the pass's
    // dependent record -> code -> dequantisation loads are latency-bound at
    // its occupancy, where the separate decoder hides them.
    static const bool fused_on = getenv("BMQ_FUSED_DECODE") != nullptr;
    const bool fdec = !codes && rows_.p && fused_on && !two_sets_ &&
                      stream_first_pass(sp.prog, L_.b, false, d_vtab != nullptr);
    // code-domain stages: zero-free narrow chunks stay in the payload and the
    // first permutation pass reads their codes there (PermSrc; BMQ_DBG_NO_PERMSRC=1 decodes every chunk)
    static const bool permsrc_off = getenv("BMQ_DBG_NO_PERMSRC") != nullptr;
    PermSrc* ps = (codes && zf && !permsrc_off) ? psrc_.p : nullptr;
    launch_decompress(st_, dec_.p, nblk, nch_, *tabs_, dinfo_.p, dchunk_.p, true, false, err_.p,
                      &counters_.kernel_launches, fdec ? 3 : (codes ? 1 : 0), fdec ? nullptr : zf,
                      (zf && !fdec) ? imnz_.p : nullptr, rows_.p, ps);
    // the prefetch slot is free again (after the permutation passes when they read payloads)
    if (host_pool_ && !ps) BMQ_CUDA(cudaEventRecord(ev_dec_[slot], st_));
    pf_live_[slot] = false;
    phase_event(4 * bidx + 1);
    // the stage's last gate pass quantises straight into pk_ / cplan_
    BMQ_CUDA(cudaMemsetAsync(cplan_.p, 0, nblk * nch_ * sizeof(ChunkPlan), st_));
    const QuantOut qo{pk_.p, cplan_.p, nch_, *tabs_, err_.p};
    const uint64_t per = sp.gg.per_group();
    if (codes) {
        run_mono_program(st_, sp.prog, pk_.p, L_.b, nblk / per, &counters_.kernel_launches, qo, zf,
                         zf ? imnz_.p : nullptr, ps);
        if (host_pool_ && ps) BMQ_CUDA(cudaEventRecord(ev_dec_[slot], st_));
        ++counters_.code_domain_batches;
    } else {
        FusedDecode fd{};
        if (fdec) {
            fd.blks = dec_.p;
            fd.infos = dinfo_.p;
            fd.rows = rows_.p;
            fd.dequant = tabs_->dequant;
            fd.qlo = tabs_->qlo;
            fd.qhi = tabs_->qhi;
            fd.err = err_.p;
            ++counters_.fused_decode_batches;
        }
        f.fused = run_program(st_, sp.prog, work_.p, L_.b, false, d_vtab ? 0 : nblk / per,
                              &counters_.kernel_launches, &qo, d_vtab, nblk, zf, nch_, zf ? imnz_.p : nullptr,
                              fdec ? &fd : nullptr);
    }
    phase_event(4 * bidx + 2);
    launch_compress_plan(st_, cmp_.p, nblk, nch_, *tabs_, bplan_.p, cplan_.p, f.fused, err_.p,
                         &counters_.kernel_launches);
    return f;
}

void Engine::process_back(StagePlan& sp, const BatchFront& f, const uint64_t* h_ids, uint64_t nblk, size_t bidx) {
    // payload placement stays in batch order (the arena cursor / heap and the
    // reference's put order): wait for the previous batch's emit
    if (emitted_live_) BMQ_CUDA(cudaStreamWaitEvent(st_, ev_emitted_, 0));
    emit_batch(nblk, h_ids);
    if (two_sets_) {
        BMQ_CUDA(cudaEventRecord(ev_emitted_, st_));
        emitted_live_ = true;
    }
    phase_event(4 * bidx + 3);
    if (f.fused) ++counters_.fused_batches;
    if (!f.codes) {
        counters_.lazy_cx += sp.prog.lazy_cx;
        counters_.perm_materialisations += sp.prog.perms;
    }
    counters_.gate_passes += sp.prog.passes.size();
    if (!f.codes)
        for (const GatePass& gp : sp.prog.passes) counters_.stream_passes += gp.sp && !stream_off() ? 1 : 0;
}

void Engine::run_stage(uint64_t s) {
    if (!cfg_.compress) return raw_run_stage(s);
    StagePlan& sp = *stage_plans_[s];
    const GroupGeometry& gg = sp.gg;
    const uint64_t per = gg.per_group(), ngroups = gg.groups();
    const uint64_t nid = L_.num_blocks();
    const bool skip_zero = cfg_.flags & BMQ_FLAG_ZERO_GROUP_SKIP;
    const bool blockwise = sp.diag_only && identity_ok_ && skip_zero && (cfg_.flags & BMQ_FLAG_IDENTITY_SKIP);
    std::vector<uint64_t> inner(per);
    for (uint64_t v = 0; v < per; ++v) inner[v] = deposit_bits(v, gg.inner_mask);
    // the blocks to process, in the reference's group order
    std::vector<uint64_t> work_ids;
    std::vector<uint32_t> work_v;
    std::vector<uint64_t> model_ids;
    work_ids.reserve(nid);
    uint64_t o = 0, groups_done = 0, groups_owned = 0;
    for (uint64_t g = 0; g < ngroups; ++g) {
        if (sharded() && owner(o, s) != shard_rank_) {  // device bits are outer bits: o decides
            o = ((o | ~gg.outer_mask) + 1) & gg.outer_mask;
            continue;
        }
        ++groups_owned;
        {  // SURVEY 8(d) model: every block of a group with a non-ALL_ZERO input
            bool nz = false;
            for (uint64_t v = 0; v < per && !nz; ++v) nz = h_off_[o | inner[v]] != ~0ull;
            if (nz)
                for (uint64_t v = 0; v < per; ++v) model_ids.push_back(o | inner[v]);
        }
        if (blockwise) {
            bool any = false;
            for (uint64_t v = 0; v < per; ++v) {
                const uint64_t id = o | inner[v];
                if (sp.touched[v] && h_off_[id] != ~0ull) {
                    work_ids.push_back(id);
                    work_v.push_back(static_cast<uint32_t>(v));
                    any = true;
                }
            }
            groups_done += any;
        } else {
            bool nonzero = !skip_zero;
            for (uint64_t v = 0; v < per && !nonzero; ++v) nonzero = h_off_[o | inner[v]] != ~0ull;
            if (nonzero) {
                for (uint64_t v = 0; v < per; ++v) work_ids.push_back(o | inner[v]);
                ++groups_done;
            }
        }
        o = ((o | ~gg.outer_mask) + 1) & gg.outer_mask;
    }
    const uint64_t nwork = work_ids.size();
    uint64_t rd = 0;  // payload bytes this stage reads (sizes before it runs)
    for (uint64_t id : work_ids) rd += h_off_[id] == ~0ull ? 0 : h_size_[id];
    uint64_t model_in = 0;
    for (uint64_t id : model_ids) model_in += h_size_[id];
    size_t nbatches = 0;
    if (nwork) {
        BMQ_CUDA(cudaMemcpyAsync(ids_.p, work_ids.data(), nwork * sizeof(uint64_t), cudaMemcpyHostToDevice, st_));
        if (blockwise)
            BMQ_CUDA(cudaMemcpyAsync(vtab_.p, work_v.data(), nwork * sizeof(uint32_t), cudaMemcpyHostToDevice, st_));
        // batches of whole groups, cut so that their host-level payloads fit
        // one prefetch slot
        const uint64_t unit = blockwise ? 1 : per;
        const uint64_t batch_blocks = blockwise ? max_blocks_ : std::max<uint64_t>(1, max_blocks_ / per) * per;
        const uint64_t pf_cap =
            host_pool_ && (host_heap_.used() || (disk_.is_open() && disk_.heap().used())) ? pf_[0].bytes() : ~0ull;
        std::vector<std::pair<uint64_t, uint64_t>> batches;
        uint64_t first = 0, hb = 0;
        for (uint64_t u = 0; u < nwork; u += unit) {
            uint64_t ub = 0;
            if (pf_cap != ~0ull)
                for (uint64_t v = u; v < u + unit; ++v) {
                    const uint64_t o = h_off_[work_ids[v]];
                    if (o != ~0ull && (o & kLevelTags)) ub += (h_size_[work_ids[v]] + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
                }
            if (u > first && (u - first + unit > batch_blocks || hb + ub > pf_cap)) {
                batches.emplace_back(first, u - first);
                first = u;
                hb = 0;
            }
            hb += ub;
        }
        batches.emplace_back(first, nwork - first);
        if (two_sets_) {  // the other stream reads the ids / table just uploaded on st_
            BMQ_CUDA(cudaEventRecord(ev_join_, st_));
            BMQ_CUDA(cudaStreamWaitEvent(st2_, ev_join_, 0));
        }
        const auto front = [&](size_t k) {
            const auto [b0, nblk] = batches[k];
            use_set(static_cast<int>(k & 1));
            return process_front(sp, ids_.p + b0, blockwise ? vtab_.p + b0 : nullptr, nblk, k);
        };
        pf_live_[0] = prefetch(work_ids.data() + batches[0].first, batches[0].second, 0);
        BatchFront cur = front(0), next;
        for (size_t k = 0; k < batches.size(); ++k, ++nbatches) {
            if (k + 1 < batches.size()) {
                // overlaps batch k on the copy engine
                pf_live_[(k + 1) & 1] = prefetch(work_ids.data() + batches[k + 1].first, batches[k + 1].second,
                                                 static_cast<int>((k + 1) & 1));
                if (two_sets_) next = front(k + 1);  // decode of k+1 overlaps the passes of k
            }
            const auto [b0, nblk] = batches[k];
            use_set(static_cast<int>(k & 1));
            process_back(sp, cur, work_ids.data() + b0, nblk, k);
            if (k + 1 < batches.size()) cur = two_sets_ ? next : front(k + 1);
        }
        join_sets();
    }
    check_device_error(("stage " + std::to_string(s) + ": ").c_str());
    sync_copies();
    sync_meta_to_host();
    collect_phase_times(nbatches);
    // accounting replay in the reference put order (groups ascending); a
    // sharded run replays the gathered global sizes in account_stage()
    if (!sharded()) account_stage(s, h_size_.data());
    uint64_t wr = 0;
    for (uint64_t id : work_ids) wr += h_off_[id] == ~0ull ? 0 : h_size_[id];
    uint64_t model_out = 0;
    for (uint64_t id : model_ids) model_out += h_size_[id];
    counters_.model_bytes += model_in + model_out + model_ids.size() * (32ull << L_.b);
    counters_.model_groups += model_ids.size() / per;
    // implementation bytes per phase: FP64 stages move 16 B per amplitude
    // (8 B of packed codes out of the last pass), code-domain stages 8 B
    const bool codes = !blockwise && sp.prog.mono && identity_ok_ && (cfg_.flags & BMQ_FLAG_CODE_DOMAIN);
    const uint64_t half_dense = nwork * (16ull << L_.b), pk_bytes = nwork * (8ull << L_.b);
    const uint64_t work_bytes = codes ? pk_bytes : half_dense;
    counters_.payload_bytes_read += rd;
    counters_.payload_bytes_written += wr;
    counters_.decompress_bytes += rd + work_bytes;
    counters_.gate_bytes += codes ? 2 * pk_bytes * sp.prog.passes.size()
                                  : 2 * half_dense * (sp.prog.passes.size() - 1) + half_dense + pk_bytes;
    counters_.compress_bytes += pk_bytes + wr;
    for (uint64_t id : work_ids) sums_ok_[id] = 0;
    counters_.groups_processed += groups_done;
    counters_.groups_skipped += groups_owned - groups_done;
    counters_.blocks_processed += nwork;
    counters_.dense_bytes += nwork * (32ull << L_.b);
    stage_compress_calls_ += nid;
    stage_decompress_calls_ += nid;
}

// ------------------------------------------------------------ stage fusion
// A stage joins a fused run when it is an FP stage the engine would run on
// the whole working set (not on codes, not block-wise): its programs are
// rebuilt over the union layout, where the same gates act on the same
// amplitudes in the same order (buffer bits are a relabelling).
bool Engine::fusable(uint64_t s) const {
    const StagePlan& sp = *stage_plans_[s];
    const bool skip_zero = cfg_.flags & BMQ_FLAG_ZERO_GROUP_SKIP;
    const bool codes = sp.prog.mono && identity_ok_ && (cfg_.flags & BMQ_FLAG_CODE_DOMAIN);
    const bool blockwise = sp.diag_only && identity_ok_ && skip_zero && (cfg_.flags & BMQ_FLAG_IDENTITY_SKIP);
    // phase-chain stages (QFT) keep their zero-row flags and tile support
    // tracking, which a fused run gives up: QFT-34 (20,6) 0.72 s unfused
    // against 1.42 s with its three chain stages fused
    for (const GatePass& p : sp.prog.passes)
        if (p.fast)
            for (uint32_t i = 0; i < p.fp->nops; ++i)
                if (p.fp->ops[i].type == OP_CHAIN) return false;
    return !codes && !blockwise && !sp.prog.passes.empty();
}

void Engine::plan_fusion() {
    fusion_planned_ = true;
    fused_at_.assign(plan_.size(), -1);
    // (a host level is fine: its payloads are read in place through the
    // mapped pinned arena and written back by emit_to_host; a disk level is
    // not, its payloads must be staged before a batch decodes them)
    if (!(cfg_.flags & BMQ_FLAG_STAGE_FUSION) || !cfg_.compress || sharded() || cfg_.disk_pool_bytes || L_.b < 12)
        return;
    // union inner sets of at most kcap qubits (BMQ_FUSE_INNER, default 8):
    // groups of up to 2^kcap blocks, within one batch; small enough that
    // all-zero union groups of sparse states are still skipped
    static const uint32_t fuse_inner = [] {
        const char* e = getenv("BMQ_FUSE_INNER");
        return e ? static_cast<uint32_t>(std::max(2, std::min(16, atoi(e)))) : 8u;
    }();
    uint32_t kcap = fuse_inner;
    while (kcap > 0 && (1ull << kcap) > max_blocks_) --kcap;
    for (uint64_t s = 0; s < plan_.size();) {
        if (!fusable(s)) {
            ++s;
            continue;
        }
        uint64_t mask = 0, e = s;
        for (; e < plan_.size() && fusable(e); ++e) {
            uint64_t m = mask;
            for (uint32_t i = 0; i < plan_[e].inner_count; ++i) m |= 1ull << plan_[e].inner[i];
            if (static_cast<uint32_t>(__builtin_popcountll(m)) > kcap) break;
            mask = m;
        }
        if (e - s < 2) {
            s = std::max(e, s + 1);
            continue;
        }
        auto fs = std::make_unique<FusedSet>();
        fs->s0 = s;
        fs->s1 = e;
        bmq_stage U{};
        U.gate_begin = plan_[s].gate_begin;
        U.gate_end = plan_[e - 1].gate_end;
        for (uint32_t q = 0; q < 64; ++q)
            if (mask >> q & 1) U.inner[U.inner_count++] = q;
        fs->gg = group_geometry(L_, U);
        for (uint64_t j = s; j < e; ++j) {
            std::vector<GateOp> ops;
            for (uint64_t i = plan_[j].gate_begin; i < plan_[j].gate_end; ++i) {
                const bmq_gate& g = gates_[i];
                const bool two = gate_is_two_qubit(g.kind);
                ops.push_back(make_op(g, buffer_bit(L_, U, g.q0), two ? buffer_bit(L_, U, g.q1) : 0));
            }
            auto prog = std::make_unique<GateProgram>();
            build_program(*prog, std::move(ops), L_.b + U.inner_count);
            fs->progs.push_back(std::move(prog));
        }
        fused_at_[s] = static_cast<int64_t>(fused_sets_.size());
        fused_sets_.push_back(std::move(fs));
        s = e;
    }
    uint64_t nfs = 0;
    for (const auto& fs : fused_sets_) nfs = std::max<uint64_t>(nfs, fs->s1 - fs->s0 - 1);
    if (nfs) fsz_.alloc(nfs * max_blocks_);
}

// Stages [fs.s0, fs.s1) over the union groups: one decode, the stages'
// programs in order with the quantiser round trip between them (the last
// pass's codes -> k_round), one emit; the intermediate stages' payload sizes
// (k_cmp_plan on the same counters the emit would use) are replayed into the
// store model in the reference's put order of each stage.
void Engine::run_fused(const FusedSet& fs) {
    use_set(0);
    const GroupGeometry& gg = fs.gg;
    const uint64_t per = gg.per_group(), ngroups = gg.groups(), nid = L_.num_blocks();
    const uint64_t m = fs.s1 - fs.s0;
    const bool skip_zero = cfg_.flags & BMQ_FLAG_ZERO_GROUP_SKIP;
    std::vector<uint64_t> inner(per);
    for (uint64_t v = 0; v < per; ++v) inner[v] = deposit_bits(v, gg.inner_mask);
    std::vector<uint64_t> work_ids;
    work_ids.reserve(nid);
    uint64_t o = 0;
    for (uint64_t g = 0; g < ngroups; ++g) {
        bool nonzero = !skip_zero;
        for (uint64_t v = 0; v < per && !nonzero; ++v) nonzero = h_off_[o | inner[v]] != ~0ull;
        if (nonzero)
            for (uint64_t v = 0; v < per; ++v) work_ids.push_back(o | inner[v]);
        o = ((o | ~gg.outer_mask) + 1) & gg.outer_mask;
    }
    const uint64_t nwork = work_ids.size();
    // sizes after each stage of the run (the last one is h_size_ after the emit)
    std::vector<std::vector<uint64_t>> sizes(m);
    sizes[0].assign(h_size_.data(), h_size_.data() + nid);  // before the run
    uint64_t rd = 0;
    for (uint64_t id : work_ids) rd += h_off_[id] == ~0ull ? 0 : h_size_[id];
    std::vector<std::vector<uint64_t>> after(m - 1, sizes[0]);
    size_t nbatches = 0;
    if (nwork) {
        BMQ_CUDA(cudaMemcpyAsync(ids_.p, work_ids.data(), nwork * sizeof(uint64_t), cudaMemcpyHostToDevice, st_));
        const uint64_t batch_blocks = std::max<uint64_t>(1, max_blocks_ / per) * per;
        const uint64_t count = 2ull << L_.b;
        std::vector<uint64_t> hsz((m - 1) * max_blocks_);
        for (uint64_t b0 = 0; b0 < nwork; b0 += batch_blocks, ++nbatches) {
            const uint64_t nblk = std::min(batch_blocks, nwork - b0);
            phase_event(4 * nbatches);
            k_build_desc<<<grid_for(nblk), 256, 0, st_>>>(ids_.p + b0, nblk, off_.p, size_.p, arena_.base(), host_pool_,
                                                          zero_hdr_.p, work_.p, pk_.p, L_.b, dec_.p, cmp_.p, 0);
            ++counters_.kernel_launches;
            launch_decompress(st_, dec_.p, nblk, nch_, *tabs_, dinfo_.p, dchunk_.p, true, false, err_.p,
                              &counters_.kernel_launches, 0);
            phase_event(4 * nbatches + 1);
            for (uint64_t j = 0; j < m; ++j) {
                const GateProgram& prog = *fs.progs[j];
                // between stages a streaming last pass writes the dequantised
                // values straight back (no code words, no k_round)
                static const bool kround = getenv("BMQ_DBG_FUSE_KROUND") != nullptr;  // A/B: codes + k_round always
                const bool rnd = j + 1 < m && !kround && last_pass_streams(prog, L_.b);
                QuantOut qo{pk_.p, cplan_.p, nch_, *tabs_, err_.p};
                qo.rnd = rnd ? work_.p : nullptr;
                BMQ_CUDA(cudaMemsetAsync(cplan_.p, 0, nblk * nch_ * sizeof(ChunkPlan), st_));
                const bool fused = run_program(st_, prog, work_.p, L_.b, false, nblk / per, &counters_.kernel_launches,
                                               &qo, nullptr, nblk, nullptr, nch_, nullptr, nullptr);
                if (j + 1 == m) phase_event(4 * nbatches + 2);
                launch_compress_plan(st_, cmp_.p, nblk, nch_, *tabs_, bplan_.p, cplan_.p, fused, err_.p,
                                     &counters_.kernel_launches);
                if (fused) ++counters_.fused_batches;
                counters_.lazy_cx += prog.lazy_cx;
                counters_.perm_materialisations += prog.perms;
                counters_.gate_passes += prog.passes.size();
                for (const GatePass& gp : prog.passes) counters_.stream_passes += gp.sp && !stream_off() ? 1 : 0;
                if (j + 1 == m) break;
                k_plan_sizes<<<grid_for(nblk), 256, 0, st_>>>(bplan_.p, nblk, fsz_.p + j * max_blocks_);
                ++counters_.kernel_launches;
                if (rnd && fused) continue;
                const uint64_t nquads = nblk * count / 4;
                k_round<<<static_cast<uint32_t>(std::min<uint64_t>((nquads + 255) / 256, 148ull * 16)), 256, 0, st_>>>(
                    reinterpret_cast<const uint4*>(pk_.p), reinterpret_cast<double2*>(work_.p), nquads, tabs_->dequant);
                ++counters_.kernel_launches;
            }
            if (m > 1) {
                BMQ_CUDA(cudaMemcpy2DAsync(hsz.data(), nblk * sizeof(uint64_t), fsz_.p, max_blocks_ * sizeof(uint64_t),
                                           nblk * sizeof(uint64_t), m - 1, cudaMemcpyDeviceToHost, st_));
            }
            emit_batch(nblk, work_ids.data() + b0);
            phase_event(4 * nbatches + 3);
            BMQ_CUDA(cudaStreamSynchronize(st_));
            for (uint64_t j = 0; j + 1 < m; ++j)
                for (uint64_t i = 0; i < nblk; ++i) {
                    const uint64_t v = hsz[j * nblk + i];
                    after[j][work_ids[b0 + i]] = v == ~0ull ? kHeaderBytes : v;
                }
        }
    }
    check_device_error(("stages " + std::to_string(fs.s0) + ".." + std::to_string(fs.s1 - 1) + ": ").c_str());
    sync_copies();
    sync_meta_to_host();
    collect_phase_times(nbatches);
    uint64_t wr = 0;
    for (uint64_t id : work_ids) wr += h_off_[id] == ~0ull ? 0 : h_size_[id];
    // per stage: the store model's puts and the SURVEY 8(d) model bytes, each
    // in that stage's own grouping
    for (uint64_t j = 0; j < m; ++j) {
        const uint64_t s = fs.s0 + j;
        const uint64_t* before = j == 0 ? sizes[0].data() : after[j - 1].data();
        const uint64_t* now = j + 1 == m ? h_size_.data() : after[j].data();
        account_stage(s, now);
        const GroupGeometry& sg = stage_plans_[s]->gg;
        const uint64_t sper = sg.per_group();
        std::vector<uint64_t> sin(sper);
        for (uint64_t v = 0; v < sper; ++v) sin[v] = deposit_bits(v, sg.inner_mask);
        uint64_t so = 0, mb = 0, mg = 0;
        for (uint64_t g = 0; g < sg.groups(); ++g) {
            bool nz = false;
            for (uint64_t v = 0; v < sper && !nz; ++v) nz = before[so | sin[v]] > kHeaderBytes;
            if (nz) {
                for (uint64_t v = 0; v < sper; ++v) mb += before[so | sin[v]] + now[so | sin[v]];
                ++mg;
            }
            so = ((so | ~sg.outer_mask) + 1) & sg.outer_mask;
        }
        counters_.model_bytes += mb + mg * sper * (32ull << L_.b);
        counters_.model_groups += mg;
        counters_.groups_processed += nwork / sper;
        counters_.groups_skipped += sg.groups() - nwork / sper;
        stage_compress_calls_ += nid;
        stage_decompress_calls_ += nid;
    }
    // implementation bytes: one decode and one emit for the run, every
    // stage's passes; between stages either a streaming last pass writing
    // doubles (16 B) or code words plus k_round (8 B out, 8 B in, 16 B out)
    const uint64_t half_dense = nwork * (16ull << L_.b), pk_bytes = nwork * (8ull << L_.b);
    counters_.payload_bytes_read += rd;
    counters_.payload_bytes_written += wr;
    counters_.decompress_bytes += rd + half_dense;
    for (uint64_t j = 0; j < m; ++j)
        counters_.gate_bytes += 2 * half_dense * (fs.progs[j]->passes.size() - 1) + half_dense +
                                (j + 1 == m ? pk_bytes
                                            : (last_pass_streams(*fs.progs[j], L_.b) ? half_dense
                                                                                       : 2 * pk_bytes + half_dense));
    counters_.compress_bytes += pk_bytes + wr;
    for (uint64_t id : work_ids) sums_ok_[id] = 0;
    counters_.blocks_processed += nwork * m;
    counters_.dense_bytes += nwork * m * (32ull << L_.b);
    counters_.fused_stages += m;
    counters_.fused_sets += 1;
}

void Engine::run_stages(uint64_t first, uint64_t last) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    if (first != next_stage_ || last < first || last > plan_.size())
        raise(BMQ_ERR_ENGINE, "stages must run in order: next stage is " + std::to_string(next_stage_));
    for (uint64_t s = first; s < last; ++s) {
        run_stage(s);
        next_stage_ = s + 1;
    }
}

void Engine::run(bmq_report* rep, double* stage_ms, uint64_t stage_cap) {
    BMQ_CUDA(cudaSetDevice(dev_));
    if (sharded()) raise(BMQ_ERR_ENGINE, "a sharded simulator is driven stage by stage by its shard driver");
    const double t0 = now_ms();
    ensure_init();
    counters_ = bmq_report{};
    BMQ_CUDA(cudaEventRecord(ev0_, st_));
    if (!fusion_planned_) plan_fusion();
    for (uint64_t s = next_stage_; s < plan_.size(); ++s) {
        const double ts = now_ms();
        const int64_t f = cfg_.compress ? fused_at_[s] : -1;
        if (f >= 0) {  // a fused run: its time goes to its first stage
            const FusedSet& fs = *fused_sets_[f];
            run_fused(fs);
            for (uint64_t j = fs.s0; j < fs.s1; ++j)
                if (stage_ms && j < stage_cap) stage_ms[j] = j == s ? now_ms() - ts : 0.0;
            next_stage_ = fs.s1;
            s = fs.s1 - 1;
            continue;
        }
        run_stage(s);
        next_stage_ = s + 1;
        if (stage_ms && s < stage_cap) stage_ms[s] = now_ms() - ts;
    }
    // The reference's run() ends with state_norm(), a full decompress
    // (engine.hpp:131-132); its device part (per-block sums) is timed here.
    ensure_sums();
    BMQ_CUDA(cudaEventRecord(ev1_, st_));
    BMQ_CUDA(cudaEventSynchronize(ev1_));
    float dms = 0.f;
    BMQ_CUDA(cudaEventElapsedTime(&dms, ev0_, ev1_));
    report(rep, dms);
    rep->final_norm = state_norm();
    rep->wall_ms = now_ms() - t0;
}

// The report of the stages run so far (final_norm / wall_ms left to the caller).
void Engine::report(bmq_report* rep, double device_ms) {
    bmq_report r{};
    r.qubits = L_.n;
    r.gate_count = gates_.size();
    r.stage_count = plan_.size();
    r.device_ms = device_ms;
    r.max_footprint_bytes = store_.peak();
    r.standard_bytes = std::exp2(static_cast<double>(L_.n + 4));
    r.compression_ratio = r.max_footprint_bytes ? r.standard_bytes / static_cast<double>(r.max_footprint_bytes) : 0.0;
    r.spilled_blocks = store_.spilled_blocks();
    r.stage_compress_calls = stage_compress_calls_;
    r.stage_decompress_calls = stage_decompress_calls_;
    r.groups_processed = counters_.groups_processed;
    r.groups_skipped = counters_.groups_skipped;
    r.blocks_processed = counters_.blocks_processed;
    r.payload_bytes_read = counters_.payload_bytes_read;
    r.payload_bytes_written = counters_.payload_bytes_written;
    r.dense_bytes = counters_.dense_bytes;
    r.kernel_launches = counters_.kernel_launches;
    r.gate_passes = counters_.gate_passes;
    r.device_peak_bytes = device_peak_;
    r.decompress_ms = counters_.decompress_ms;
    r.gate_ms = counters_.gate_ms;
    r.compress_ms = counters_.compress_ms;
    r.batches = counters_.batches;
    r.decompress_bytes = counters_.decompress_bytes;
    r.gate_bytes = counters_.gate_bytes;
    r.compress_bytes = counters_.compress_bytes;
    r.fused_batches = counters_.fused_batches;
    r.compactions = counters_.compactions;
    r.host_spill_bytes = counters_.host_spill_bytes;
    r.host_spill_batches = counters_.host_spill_batches;
    r.code_domain_batches = counters_.code_domain_batches;
    r.pool_growths = counters_.pool_growths;
    r.lazy_cx = counters_.lazy_cx;
    r.perm_materialisations = counters_.perm_materialisations;
    r.model_bytes = counters_.model_bytes;
    r.model_groups = counters_.model_groups;
    r.link_h2d_bytes = counters_.link_h2d_bytes;
    r.link_d2h_bytes = counters_.link_d2h_bytes;
    r.link_ms = counters_.link_ms;
    r.compact_bytes = counters_.compact_bytes;
    r.host_peak_bytes = host_heap_.high_water();
    r.arena_bytes = arena_limit_;
    r.fused_decode_batches = counters_.fused_decode_batches;
    r.stream_passes = counters_.stream_passes;
    r.disk_spill_bytes = counters_.disk_spill_bytes;
    r.disk_read_bytes = counters_.disk_read_bytes;
    r.disk_peak_bytes = disk_.is_open() ? disk_.heap().high_water() : 0;
    r.disk_gds = disk_.gds() ? 1 : 0;
    r.fused_stages = counters_.fused_stages;
    r.fused_sets = counters_.fused_sets;
    *rep = r;
}

double Engine::state_norm() {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    const uint64_t nid = L_.num_blocks();
    if (cfg_.compress) ensure_sums();
    if (!cfg_.compress) {
        k_block_sums<<<static_cast<uint32_t>(nid), 256, 0, st_>>>(dense_.p, L_.b, sums_.p);
        BMQ_CUDA(cudaGetLastError());
    }
    std::vector<double> h(3 * nid);
    BMQ_CUDA(cudaMemcpyAsync(h.data(), sums_.p, sums_.bytes(), cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
    double sum = 0.0;
    for (uint64_t id = 0; id < nid; ++id) sum += h[3 * id];
    return std::sqrt(sum);
}

void Engine::host_ids_to_device(const std::vector<uint64_t>& ids) {
    BMQ_CUDA(cudaMemcpyAsync(ids_.p, ids.data(), ids.size() * sizeof(uint64_t), cudaMemcpyHostToDevice, st_));
}

// Disk-level payloads of ids[0..n) (host ids) read into prefetch slot 0 for
// a decode outside the stage loop; the slot table for k_build_desc, or null
// when none of the ids is on disk. n must satisfy disk_fit.
const uint64_t* Engine::stage_disk_reads(const uint64_t* h_ids, uint64_t n) {
    if (!disk_.is_open() || !disk_.heap().used()) return nullptr;
    bool any = false;
    for (uint64_t i = 0; i < n && !any; ++i) any = h_off_[h_ids[i]] != ~0ull && (h_off_[h_ids[i]] & kDiskTag);
    if (!any) return nullptr;
    sync_copies();
    BMQ_CUDA(cudaStreamSynchronize(st_));  // earlier decodes have left the slot
    uint64_t* tab = h_pf_off_[0].data();
    uint64_t pos = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t o = h_off_[h_ids[i]];
        tab[i] = ~0ull;
        if (o == ~0ull || !(o & kDiskTag)) continue;
        const uint64_t size = h_size_[h_ids[i]];
        if (pos + size > pf_[0].bytes()) raise(BMQ_ERR_LOGIC, "disk-level payloads exceed the staging slot");
        disk_.read_to_device(pf_[0].p + pos, size, o & ~kDiskTag);
        counters_.disk_read_bytes += size;
        tab[i] = pos;
        pos += (size + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
    }
    BMQ_CUDA(cudaMemcpyAsync(pf_off_[0].p, tab, n * 8, cudaMemcpyHostToDevice, st_));
    return pf_off_[0].p;
}

// Largest prefix of ids whose disk-level payloads fit one staging slot.
uint64_t Engine::disk_fit(const uint64_t* h_ids, uint64_t n) {
    if (!disk_.is_open() || !disk_.heap().used()) return n;
    uint64_t pos = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t o = h_off_[h_ids[i]];
        if (o == ~0ull || !(o & kDiskTag)) continue;
        pos += (h_size_[h_ids[i]] + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
        if (pos > pf_[0].bytes()) return std::max<uint64_t>(i, 1);
    }
    return n;
}

void Engine::decompress_ids(const uint64_t* d_ids, uint64_t nids, bool want_sums, const uint64_t* h_ids) {
    std::vector<uint64_t> hv;
    if (disk_.is_open() && disk_.heap().used() && !h_ids) {
        hv.resize(nids);
        BMQ_CUDA(cudaMemcpyAsync(hv.data(), d_ids, nids * 8, cudaMemcpyDeviceToHost, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
        h_ids = hv.data();
    }
    const uint64_t count = 2ull << L_.b;
    for (uint64_t k = 0; k < nids;) {
        const uint64_t m = h_ids ? disk_fit(h_ids + k, nids - k) : nids - k;
        const uint64_t* tab = h_ids ? stage_disk_reads(h_ids + k, m) : nullptr;
        k_build_desc<<<grid_for(m), 256, 0, st_>>>(d_ids + k, m, off_.p, size_.p, arena_.base(), host_pool_,
                                                   zero_hdr_.p, work_.p + k * count, pk_.p + k * count, L_.b,
                                                   dec_.p + k, cmp_.p + k, 0, tab, pf_[0].p);
        launch_decompress(st_, dec_.p + k, m, nch_, *tabs_, dinfo_.p + k, dchunk_.p + k * nch_, true, want_sums,
                          err_.p, &counters_.kernel_launches);
        k += m;
        if (k < nids && tab) BMQ_CUDA(cudaStreamSynchronize(st_));  // the slot is reused
    }
}

void Engine::ensure_sums(const uint64_t* ids, uint64_t n) {
    if (!cfg_.compress || !initialized_) return;
    std::vector<uint64_t> stale, zero;
    const auto visit = [&](uint64_t id) {
        if (sums_ok_[id]) return;
        (h_off_[id] == ~0ull ? zero : stale).push_back(id);
        sums_ok_[id] = 1;
    };
    if (ids) {
        for (uint64_t i = 0; i < n; ++i) visit(ids[i]);
    } else {
        for (uint64_t id = 0; id < sums_ok_.size(); ++id) visit(id);
    }
    for (uint64_t id : zero) BMQ_CUDA(cudaMemsetAsync(sums_.p + 3 * id, 0, 3 * sizeof(double), st_));
    for (uint64_t first = 0; first < stale.size();) {
        uint64_t nb = std::min<uint64_t>(max_blocks_, stale.size() - first);
        nb = disk_fit(stale.data() + first, nb);
        BMQ_CUDA(cudaMemcpyAsync(ids_.p, stale.data() + first, nb * sizeof(uint64_t), cudaMemcpyHostToDevice, st_));
        const uint64_t* tab = stage_disk_reads(stale.data() + first, nb);
        k_build_desc<<<grid_for(nb), 256, 0, st_>>>(ids_.p, nb, off_.p, size_.p, arena_.base(), host_pool_,
                                                    zero_hdr_.p, work_.p, pk_.p, L_.b, dec_.p, cmp_.p, 0, tab,
                                                    pf_[0].p);
        launch_decompress(st_, dec_.p, nb, nch_, *tabs_, dinfo_.p, dchunk_.p, true, true, err_.p,
                          &counters_.kernel_launches, 2);
        k_store_dec_sums<<<grid_for(nb), 256, 0, st_>>>(dinfo_.p, ids_.p, nb, sums_.p);
        counters_.kernel_launches += 2;
        BMQ_CUDA(cudaStreamSynchronize(st_));  // ids_ is reused by the next batch
        first += nb;
    }
    if (!stale.empty()) check_device_error("sums: ");
}

void Engine::extract_state(double* amps, uint64_t namps) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    if (L_.n > cfg_.verify_cap_qubits)
        raise(BMQ_ERR_ENGINE, "dense verification refused: " + std::to_string(L_.n) +
                                  " qubits exceeds the cap of " + std::to_string(cfg_.verify_cap_qubits));
    if (namps != (1ull << L_.n)) raise(BMQ_ERR_INVALID_ARGUMENT, "amplitude buffer must hold 2^n amplitudes");
    const uint64_t nid = L_.num_blocks();
    if (!cfg_.compress) {
        DevArray<double> tmp;
        tmp.alloc(2 * namps);
        k_interleave<<<grid_for(namps), 256, 0, st_>>>(dense_.p, nid, L_.b, tmp.p);
        BMQ_CUDA(cudaMemcpyAsync(amps, tmp.p, tmp.bytes(), cudaMemcpyDeviceToHost, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
        return;
    }
    DevArray<double> tmp;
    tmp.alloc(std::min(nid, max_blocks_) * (2ull << L_.b));
    std::vector<uint64_t> ids(nid);
    for (uint64_t i = 0; i < nid; ++i) ids[i] = i;
    host_ids_to_device(ids);
    for (uint64_t first = 0; first < nid; first += max_blocks_) {
        const uint64_t nb = std::min(max_blocks_, nid - first);
        decompress_ids(ids_.p + first, nb, false);
        k_interleave<<<grid_for(nb << L_.b), 256, 0, st_>>>(work_.p, nb, L_.b, tmp.p);
        BMQ_CUDA(cudaMemcpyAsync(amps + 2 * (first << L_.b), tmp.p, (nb << L_.b) * 2 * sizeof(double),
                                 cudaMemcpyDeviceToHost, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
    }
    check_device_error("extract_state: ");
}

void Engine::amplitude(uint64_t index, double* re, double* im) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    if (index >> L_.n) raise(BMQ_ERR_INVALID_ARGUMENT, "amplitude index out of range");
    const uint64_t id = index >> L_.b, l = index & ((1ull << L_.b) - 1);
    const double* src;
    if (!cfg_.compress) {
        src = dense_.p + (id << (L_.b + 1));
    } else {
        host_ids_to_device({id});
        decompress_ids(ids_.p, 1, false);
        src = work_.p;
    }
    BMQ_CUDA(cudaMemcpyAsync(re, src + l, 8, cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaMemcpyAsync(im, src + (1ull << L_.b) + l, 8, cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
    if (cfg_.compress) check_device_error("amplitude: ");
}

uint64_t Engine::zero_payload(uint8_t* out, uint64_t cap) const {
    if (!cfg_.compress) {
        const uint64_t raw = 16ull << L_.b;
        if (out && cap >= raw) std::memset(out, 0, raw);
        return raw;
    }
    if (out && cap >= static_cast<uint64_t>(kHeaderBytes)) {
        std::memset(out, 0, kHeaderBytes);
        const uint64_t cnt = 2ull << L_.b;
        for (int k = 0; k < 8; ++k) out[k] = static_cast<uint8_t>(cnt >> (8 * k));
        std::memcpy(out + 8, &cfg_.error_bound, 8);
        out[25] = 1;
    }
    return kHeaderBytes;
}

uint64_t Engine::get_payload(uint64_t id, uint8_t* out, uint64_t cap) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    if (id >= L_.num_blocks()) raise(BMQ_ERR_STORE, "unknown block id " + std::to_string(id));
    if (!cfg_.compress) {
        const uint64_t raw = 16ull << L_.b;
        if (out && cap >= raw) {
            BMQ_CUDA(cudaMemcpyAsync(out, dense_.p + (id << (L_.b + 1)), raw, cudaMemcpyDeviceToHost, st_));
            BMQ_CUDA(cudaStreamSynchronize(st_));
        }
        return raw;
    }
    if (h_off_[id] == ~0ull) return zero_payload(out, cap);
    const uint64_t size = h_size_[id];
    if (out && cap >= size) {
        if (h_off_[id] & kDiskTag) {
            disk_.read_to_host(out, size, h_off_[id] & ~kDiskTag);
        } else if (h_off_[id] & kHostTag) {
            BMQ_CUDA(cudaStreamSynchronize(st_));
            std::memcpy(out, host_pool_ + (h_off_[id] & ~kHostTag), size);
        } else {
            BMQ_CUDA(cudaMemcpyAsync(out, arena_.base() + h_off_[id], size, cudaMemcpyDeviceToHost, st_));
            BMQ_CUDA(cudaStreamSynchronize(st_));
        }
    }
    return size;
}

void Engine::get_payloads(uint8_t* out, uint64_t cap, uint64_t* sizes, uint64_t* total) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    const uint64_t nid = L_.num_blocks();
    uint64_t t = 0;
    for (uint64_t id = 0; id < nid; ++id) {
        const uint64_t sz = cfg_.compress ? (h_off_[id] == ~0ull ? kHeaderBytes : h_size_[id]) : (16ull << L_.b);
        if (sizes) sizes[id] = sz;
        t += sz;
    }
    *total = t;
    if (!out) return;
    if (cap < t) raise(BMQ_ERR_BUFFER_TOO_SMALL, "payload buffer too small");
    if (!cfg_.compress) {
        BMQ_CUDA(cudaMemcpyAsync(out, dense_.p, t, cudaMemcpyDeviceToHost, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
        return;
    }
    // Gather the payloads of a range of ids back to back on the device (the
    // dead dense work buffer is the staging area), then one D2H copy per range.
    uint8_t* staging = reinterpret_cast<uint8_t*>(work_.p);
    const uint64_t scap = work_.bytes();
    std::vector<Xfer> xs;
    uint64_t pos = 0;
    const auto flush = [&]() {
        if (xs.empty()) return;
        const uint64_t base = xs.front().xoff, len = pos - base;
        for (Xfer& x : xs) x.xoff -= base;
        DevArray<Xfer> dx;
        dx.alloc(xs.size());
        BMQ_CUDA(cudaMemcpyAsync(dx.p, xs.data(), xs.size() * sizeof(Xfer), cudaMemcpyHostToDevice, st_));
        k_gather_payloads<<<static_cast<uint32_t>(std::min<uint64_t>(xs.size(), 148 * 16)), 256, 0, st_>>>(
            dx.p, xs.size(), off_.p, arena_.base(), host_pool_, zero_hdr_.p, staging);
        ++counters_.kernel_launches;
        BMQ_CUDA(cudaGetLastError());
        BMQ_CUDA(cudaMemcpyAsync(out + base, staging, len, cudaMemcpyDeviceToHost, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
        for (const Xfer& x : xs)  // disk-level payloads (skipped by the gather)
            if (h_off_[x.id] != ~0ull && (h_off_[x.id] & kDiskTag))
                disk_.read_to_host(out + base + x.xoff, x.size, h_off_[x.id] & ~kDiskTag);
        xs.clear();
    };
    for (uint64_t id = 0; id < nid; ++id) {
        const uint64_t sz = h_off_[id] == ~0ull ? kHeaderBytes : h_size_[id];
        if (!xs.empty() && pos + sz - xs.front().xoff > scap) flush();
        xs.push_back(Xfer{id, pos, sz, 0, {}});
        pos += sz;
    }
    flush();
}

void Engine::put_payload(uint64_t id, const uint8_t* data, uint64_t size) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    if (id >= L_.num_blocks()) raise(BMQ_ERR_STORE, "unknown block id " + std::to_string(id));
    if (!cfg_.compress) {
        const uint64_t raw = 16ull << L_.b;
        if (size != raw) raise(BMQ_ERR_ENGINE, "raw block payload has invalid length");
        BMQ_CUDA(cudaMemcpyAsync(dense_.p + (id << (L_.b + 1)), data, raw, cudaMemcpyHostToDevice, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
        store_.put(id, raw);
        return;
    }
    // device arena first (its previous payload stays live until the new one
    // decodes), else a host-level extent
    const uint64_t prev_off = h_off_[id], prev_size = h_size_[id];
    uint64_t off = ~0ull;
    if (heap_mode_) {
        sync_copies();
        off = dev_alloc(size);
        if (off != ExtentHeap::kNone)
            BMQ_CUDA(cudaMemcpyAsync(arena_.base() + off, data, size, cudaMemcpyHostToDevice, st_));
    }
    if (heap_mode_ && off != ExtentHeap::kNone) {
        BMQ_CUDA(cudaStreamSynchronize(st_));
    } else if (!heap_mode_ && make_room(size + kArenaAlign, nullptr, 0)) {
        const uint64_t used = arena_used();
        off = used;
        BMQ_CUDA(cudaMemcpyAsync(arena_.base() + used, data, size, cudaMemcpyHostToDevice, st_));
        const uint64_t end = (used + size + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
        BMQ_CUDA(cudaMemcpyAsync(cursor_.p, &end, 8, cudaMemcpyHostToDevice, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));  // `end` and `off` live on this frame
    } else {
        if (!cfg_.host_pool_bytes) raise(BMQ_ERR_STORE, "device payload pool exhausted");
        ensure_host_pool();
        sync_copies();
        const uint64_t ext = host_heap_.alloc(size);
        if (ext != ExtentHeap::kNone) {
            std::memcpy(host_pool_ + ext, data, size);
            off = ext | kHostTag;
        } else {  // host level full: the disk level
            const uint64_t d = disk_alloc(size);
            disk_.write_from_host(data, size, d);
            off = d | kDiskTag;
        }
    }
    BMQ_CUDA(cudaMemcpyAsync(off_.p + id, &off, 8, cudaMemcpyHostToDevice, st_));
    BMQ_CUDA(cudaMemcpyAsync(size_.p + id, &size, 8, cudaMemcpyHostToDevice, st_));
    host_ids_to_device({id});
    decompress_ids(ids_.p, 1, true);
    k_store_dec_sums<<<1, 32, 0, st_>>>(dinfo_.p, ids_.p, 1, sums_.p);
    try {
        check_device_error("");
    } catch (...) {  // restore the previous payload
        BMQ_CUDA(cudaMemcpyAsync(off_.p + id, &prev_off, 8, cudaMemcpyHostToDevice, st_));
        BMQ_CUDA(cudaMemcpyAsync(size_.p + id, &prev_size, 8, cudaMemcpyHostToDevice, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
        if (off & kDiskTag)
            disk_.heap().free(off & ~kDiskTag, size);
        else if (off & kHostTag)
            host_heap_.free(off & ~kHostTag, size);
        else if (heap_mode_)
            dev_heap_.free(off, size);
        throw;
    }
    free_extents(&id, 1);  // the replaced payload, if it was on the host
    h_off_[id] = off;
    h_size_[id] = size;
    sums_ok_[id] = 1;
    store_.put(id, size);
}

double Engine::fidelity_dense(const double* ideal, uint64_t namps) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    if (namps != (1ull << L_.n)) raise(BMQ_ERR_INVALID_ARGUMENT, "fidelity requires equal-length states");
    const uint64_t nid = L_.num_blocks();
    const uint64_t step = cfg_.compress ? max_blocks_ : nid;
    DevArray<double> dideal;
    dideal.alloc(std::min(step, nid) * (2ull << L_.b));
    std::vector<uint64_t> ids(nid);
    for (uint64_t i = 0; i < nid; ++i) ids[i] = i;
    if (cfg_.compress) host_ids_to_device(ids);
    double re = 0.0, im = 0.0;
    std::vector<double> part(2 * 148 * 64);
    for (uint64_t first = 0; first < nid; first += step) {
        const uint64_t nb = std::min(step, nid - first);
        const double* planar = dense_.p ? dense_.p + (first << (L_.b + 1)) : nullptr;
        if (cfg_.compress) {
            decompress_ids(ids_.p + first, nb, false);
            planar = work_.p;
        }
        BMQ_CUDA(cudaMemcpyAsync(dideal.p, ideal + 2 * (first << L_.b), (nb << L_.b) * 16, cudaMemcpyHostToDevice, st_));
        const uint32_t g = grid_for(nb << L_.b);
        k_dot<<<g, 256, 0, st_>>>(planar, dideal.p, nb, L_.b, red_.p);
        BMQ_CUDA(cudaMemcpyAsync(part.data(), red_.p, 2 * g * sizeof(double), cudaMemcpyDeviceToHost, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
        for (uint32_t k = 0; k < g; ++k) {
            re += part[2 * k];
            im += part[2 * k + 1];
        }
    }
    if (cfg_.compress) check_device_error("fidelity: ");
    return std::hypot(re, im);
}

double Engine::fidelity_analytic(int kind) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    if (kind == 0) {  // uniform 2^(-n/2): |<u|psi>| = 2^(-n/2) |sum psi_i|
        const uint64_t nid = L_.num_blocks();
        if (cfg_.compress) ensure_sums();
        if (!cfg_.compress) {
            k_block_sums<<<static_cast<uint32_t>(nid), 256, 0, st_>>>(dense_.p, L_.b, sums_.p);
            BMQ_CUDA(cudaGetLastError());
        }
        std::vector<double> h(3 * nid);
        BMQ_CUDA(cudaMemcpyAsync(h.data(), sums_.p, sums_.bytes(), cudaMemcpyDeviceToHost, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
        double re = 0.0, im = 0.0;
        for (uint64_t id = 0; id < nid; ++id) {
            re += h[3 * id + 1];
            im += h[3 * id + 2];
        }
        return std::hypot(re, im) * std::exp2(-0.5 * static_cast<double>(L_.n));
    }
    if (kind == 1) {  // GHZ (|0..0> + |1..1>) / sqrt 2
        double r0, i0, r1, i1;
        amplitude(0, &r0, &i0);
        amplitude((1ull << L_.n) - 1, &r1, &i1);
        return std::hypot(r0 + r1, i0 + i1) / std::sqrt(2.0);
    }
    raise(BMQ_ERR_INVALID_ARGUMENT, "unknown analytic ideal state kind");
}

double Engine::fidelity_pair(Engine& a, Engine& b) {
    if (a.L_.n != b.L_.n || a.L_.b != b.L_.b) raise(BMQ_ERR_INVALID_ARGUMENT, "fidelity requires equal-length states");
    if (a.dev_ != b.dev_) raise(BMQ_ERR_INVALID_ARGUMENT, "fidelity requires both simulators on one device");
    BMQ_CUDA(cudaSetDevice(a.dev_));
    a.ensure_init();
    b.ensure_init();
    const uint64_t nid = a.L_.num_blocks();
    uint64_t step = nid;
    if (a.cfg_.compress) step = std::min(step, a.max_blocks_);
    if (b.cfg_.compress) step = std::min(step, b.max_blocks_);
    std::vector<uint64_t> ids(nid);
    for (uint64_t i = 0; i < nid; ++i) ids[i] = i;
    if (a.cfg_.compress) a.host_ids_to_device(ids);
    if (b.cfg_.compress) b.host_ids_to_device(ids);
    BMQ_CUDA(cudaStreamSynchronize(a.st_));
    BMQ_CUDA(cudaStreamSynchronize(b.st_));
    double re = 0.0, im = 0.0;
    std::vector<double> part(2 * 148 * 64);
    for (uint64_t first = 0; first < nid; first += step) {
        const uint64_t nb = std::min(step, nid - first);
        const double* pa = a.cfg_.compress ? a.work_.p : a.dense_.p + (first << (a.L_.b + 1));
        const double* pb = b.cfg_.compress ? b.work_.p : b.dense_.p + (first << (b.L_.b + 1));
        if (a.cfg_.compress) a.decompress_ids(a.ids_.p + first, nb, false);
        if (b.cfg_.compress) b.decompress_ids(b.ids_.p + first, nb, false);
        BMQ_CUDA(cudaStreamSynchronize(a.st_));
        BMQ_CUDA(cudaStreamSynchronize(b.st_));
        const uint32_t g = grid_for(nb << a.L_.b);
        k_dot2<<<g, 256, 0, a.st_>>>(pa, pb, nb, a.L_.b, a.red_.p);
        BMQ_CUDA(cudaMemcpyAsync(part.data(), a.red_.p, 2 * g * sizeof(double), cudaMemcpyDeviceToHost, a.st_));
        BMQ_CUDA(cudaStreamSynchronize(a.st_));
        for (uint32_t k = 0; k < g; ++k) {
            re += part[2 * k];
            im += part[2 * k + 1];
        }
    }
    if (a.cfg_.compress) a.check_device_error("fidelity: ");
    if (b.cfg_.compress) b.check_device_error("fidelity: ");
    return std::hypot(re, im);
}

// ------------------------------------------------------------ sharded runs

void Engine::shard(uint32_t rank, uint32_t world) {
    if (initialized_) raise(BMQ_ERR_ENGINE, "shard() must be called before the state is initialized");
    if (!cfg_.compress) raise(BMQ_ERR_INVALID_ARGUMENT, "sharded runs require compression");
    dev_bits_ = shard_plan(L_, plan_, world);
    if (rank >= world) raise(BMQ_ERR_INVALID_ARGUMENT, "shard rank out of range");
    shard_rank_ = rank;
    shard_world_ = world;
    shard_m_ = 0;
    while ((1u << shard_m_) < world) ++shard_m_;
}

void Engine::export_payloads(const uint64_t* ids, uint64_t n, uint64_t* meta, void* dst, uint64_t cap) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    if (!cfg_.compress) raise(BMQ_ERR_INVALID_ARGUMENT, "payload export requires compression");
    const uint64_t nid = L_.num_blocks();
    for (uint64_t i = 0; i < n; ++i)
        if (ids[i] >= nid) raise(BMQ_ERR_STORE, "unknown block id " + std::to_string(ids[i]));
    ensure_sums(ids, n);
    std::vector<double> sums(3 * nid);
    BMQ_CUDA(cudaMemcpyAsync(sums.data(), sums_.p, sums_.bytes(), cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
    std::vector<Xfer> xs(n);
    uint64_t pos = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t id = ids[i];
        if (id >= nid) raise(BMQ_ERR_STORE, "unknown block id " + std::to_string(id));
        const uint64_t size = h_off_[id] == ~0ull ? 0 : h_size_[id];
        xs[i] = Xfer{id, pos, size, 0, {sums[3 * id], sums[3 * id + 1], sums[3 * id + 2]}};
        meta[4 * i] = size;
        std::memcpy(meta + 4 * i + 1, &sums[3 * id], 24);
        pos += (size + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
    }
    if (!dst || !n) return;
    if (reinterpret_cast<uintptr_t>(dst) % kArenaAlign) raise(BMQ_ERR_INVALID_ARGUMENT, "transfer buffer must be 16-byte aligned");
    if (cap < pos) raise(BMQ_ERR_BUFFER_TOO_SMALL, "transfer buffer too small");
    DevArray<Xfer> dx;
    dx.alloc(n);
    BMQ_CUDA(cudaMemcpyAsync(dx.p, xs.data(), n * sizeof(Xfer), cudaMemcpyHostToDevice, st_));
    k_pack_payloads<<<static_cast<uint32_t>(std::min<uint64_t>(n, 148 * 16)), 256, 0, st_>>>(
        dx.p, n, off_.p, arena_.base(), host_pool_, static_cast<uint8_t*>(dst));
    ++counters_.kernel_launches;
    BMQ_CUDA(cudaGetLastError());
    BMQ_CUDA(cudaStreamSynchronize(st_));
    cudaPointerAttributes pa{};
    const bool dst_dev = cudaPointerGetAttributes(&pa, dst) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    for (uint64_t i = 0; i < n; ++i) {  // disk-level payloads (skipped by the pack)
        const uint64_t o = h_off_[ids[i]];
        if (o == ~0ull || !(o & kDiskTag)) continue;
        uint8_t* d = static_cast<uint8_t*>(dst) + xs[i].xoff;
        if (dst_dev)
            disk_.read_to_device(d, xs[i].size, o & ~kDiskTag);
        else
            disk_.read_to_host(d, xs[i].size, o & ~kDiskTag);
    }
}

void Engine::import_payloads(const uint64_t* ids, uint64_t n, const uint64_t* meta, const void* src) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    if (!cfg_.compress) raise(BMQ_ERR_INVALID_ARGUMENT, "payload import requires compression");
    if (!n) return;
    const uint64_t nid = L_.num_blocks();
    if (src && reinterpret_cast<uintptr_t>(src) % kArenaAlign)
        raise(BMQ_ERR_INVALID_ARGUMENT, "transfer buffer must be 16-byte aligned");
    std::vector<Xfer> xs(n);
    uint64_t pos = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (ids[i] >= nid) raise(BMQ_ERR_STORE, "unknown block id " + std::to_string(ids[i]));
        Xfer x{ids[i], pos, meta[4 * i], pos, {}};
        std::memcpy(x.sums, meta + 4 * i + 1, 24);
        if (x.size && !src) raise(BMQ_ERR_INVALID_ARGUMENT, "payload bytes missing");
        xs[i] = x;
        pos += (x.size + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
    }
    // the ids' previous payloads are replaced: host extents go back first
    sync_meta_to_host();
    sync_copies();
    free_extents(ids, n);
    // the batch back to back in the device arena (after compaction or growth
    // if needed), else one host-level extent per payload
    uint8_t* to = arena_.base();
    uint64_t tag = 0, base = 0;
    const uint64_t ext = heap_mode_ && pos ? dev_alloc(pos) : ExtentHeap::kNone;
    if (heap_mode_ && (ext != ExtentHeap::kNone || !pos)) {
        base = pos ? ext : 0;
    } else if (!heap_mode_ && make_room(pos, ids, n)) {
        base = arena_used();
        const uint64_t end = base + pos;
        BMQ_CUDA(cudaMemcpyAsync(cursor_.p, &end, 8, cudaMemcpyHostToDevice, st_));
        BMQ_CUDA(cudaStreamSynchronize(st_));
    } else {
        if (!cfg_.host_pool_bytes) raise(BMQ_ERR_STORE, "device payload pool exhausted");
        ensure_host_pool();
        to = host_pool_;
        tag = kHostTag;
        for (Xfer& x : xs) {
            if (!x.size) continue;
            const uint64_t ext = host_heap_.alloc(x.size);
            x.dst = ext != ExtentHeap::kNone ? ext : (disk_alloc(x.size) | kDiskTag);  // host level full: disk
        }
        counters_.host_spill_bytes += pos;
        ++counters_.host_spill_batches;
    }
    if (!tag)
        for (Xfer& x : xs) x.dst = base + x.dst;
    DevArray<Xfer> dx;
    dx.alloc(n);
    BMQ_CUDA(cudaMemcpyAsync(dx.p, xs.data(), n * sizeof(Xfer), cudaMemcpyHostToDevice, st_));
    k_unpack_payloads<<<static_cast<uint32_t>(std::min<uint64_t>(n, 148 * 16)), 256, 0, st_>>>(
        dx.p, n, static_cast<const uint8_t*>(src), to, tag, off_.p, size_.p, sums_.p);
    ++counters_.kernel_launches;
    BMQ_CUDA(cudaGetLastError());
    BMQ_CUDA(cudaStreamSynchronize(st_));
    cudaPointerAttributes pa{};
    const bool src_dev = src && cudaPointerGetAttributes(&pa, src) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    for (const Xfer& x : xs) {
        const bool disk = x.size && (x.dst & kDiskTag);
        if (disk) {
            const uint8_t* from = static_cast<const uint8_t*>(src) + x.xoff;
            if (src_dev)
                disk_.write_from_device(from, x.size, x.dst & ~kDiskTag);
            else
                disk_.write_from_host(from, x.size, x.dst & ~kDiskTag);
            counters_.disk_spill_bytes += x.size;
        }
        h_off_[x.id] = x.size ? (disk ? x.dst : (x.dst | tag)) : ~0ull;
        h_size_[x.id] = x.size ? x.size : kHeaderBytes;
        sums_ok_[x.id] = 1;  // the sums travelled with the payload
    }
}

void Engine::drop_payloads(const uint64_t* ids, uint64_t n) {
    BMQ_CUDA(cudaSetDevice(dev_));
    if (!cfg_.compress) raise(BMQ_ERR_INVALID_ARGUMENT, "payload drop requires compression");
    if (!n) return;
    const uint64_t nid = L_.num_blocks();
    for (uint64_t i = 0; i < n; ++i)
        if (ids[i] >= nid) raise(BMQ_ERR_STORE, "unknown block id " + std::to_string(ids[i]));
    sync_copies();
    free_extents(ids, n);
    DevArray<uint64_t> d;
    d.alloc(n);
    BMQ_CUDA(cudaMemcpyAsync(d.p, ids, n * 8, cudaMemcpyHostToDevice, st_));
    k_drop_payloads<<<grid_for(n), 256, 0, st_>>>(d.p, n, off_.p, size_.p, sums_.p);
    ++counters_.kernel_launches;
    BMQ_CUDA(cudaGetLastError());
    BMQ_CUDA(cudaStreamSynchronize(st_));
    for (uint64_t i = 0; i < n; ++i) {
        h_off_[ids[i]] = ~0ull;
        h_size_[ids[i]] = kHeaderBytes;
        if (!sums_ok_.empty()) sums_ok_[ids[i]] = 1;
    }
}

// Sizes of the ids this rank owns under stage s (0 elsewhere), so a sum over
// ranks yields every id's size.
void Engine::stage_sizes(uint64_t s, uint64_t* sizes) {
    if (s >= plan_.size()) raise(BMQ_ERR_INVALID_ARGUMENT, "stage index out of range");
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    for (uint64_t id = 0; id < L_.num_blocks(); ++id)
        sizes[id] = owner(id, s) == shard_rank_ ? (cfg_.compress ? h_size_[id] : 16ull << L_.b) : 0;
}

// BlockStore puts of stage s in the reference order (groups ascending,
// block_ids order; engine.hpp:114-115, store.hpp:64-83).
void Engine::account_stage(uint64_t s, const uint64_t* sizes) {
    if (s >= plan_.size()) raise(BMQ_ERR_INVALID_ARGUMENT, "stage index out of range");
    const GroupGeometry& gg = stage_plans_[s]->gg;
    std::vector<uint64_t> inner(gg.per_group());
    for (uint64_t v = 0; v < inner.size(); ++v) inner[v] = deposit_bits(v, gg.inner_mask);
    uint64_t o = 0;
    for (uint64_t g = 0; g < gg.groups(); ++g) {
        for (uint64_t v : inner) store_.put(o | v, sizes[o | v]);
        o = ((o | ~gg.outer_mask) + 1) & gg.outer_mask;
    }
}

void Engine::partial_sums(double* out3) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    const uint64_t nid = L_.num_blocks();
    if (cfg_.compress) ensure_sums();
    if (!cfg_.compress) {
        k_block_sums<<<static_cast<uint32_t>(nid), 256, 0, st_>>>(dense_.p, L_.b, sums_.p);
        BMQ_CUDA(cudaGetLastError());
    }
    std::vector<double> h(3 * nid);
    BMQ_CUDA(cudaMemcpyAsync(h.data(), sums_.p, sums_.bytes(), cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
    out3[0] = out3[1] = out3[2] = 0.0;
    for (uint64_t id = 0; id < nid; ++id)
        for (int k = 0; k < 3; ++k) out3[k] += h[3 * id + k];
}

// ------------------------------------------------------- checkpoint / resume
// File: "BMQCKPT1" | u32 n, b, version, pad | f64 b_r | u64 fnv(gates),
// fnv(plan), next_stage, stage_compress_calls, stage_decompress_calls,
// store-accounting bytes A, payload bytes P | accounting[A] |
// meta[4 * 2^c] (size, sumsq, sum_re, sum_im as bits) | payloads[P] packed
// 16-byte aligned in id order (bmq_simulator_export layout).
namespace {
constexpr char kCkptMagic[8] = {'B', 'M', 'Q', 'C', 'K', 'P', 'T', '1'};
uint64_t fnv1a(const void* data, size_t n, uint64_t h = 1469598103934665603ull) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 1099511628211ull;
    return h;
}
struct PinnedBuf {
    void* p = nullptr;
    explicit PinnedBuf(uint64_t n) { BMQ_CUDA(cudaMallocHost(&p, std::max<uint64_t>(n, 16))); }
    ~PinnedBuf() { cudaFreeHost(p); }
};
struct File {
    FILE* f;
    File(const char* path, const char* mode) : f(std::fopen(path, mode)) {
        if (!f) raise(BMQ_ERR_STORE, std::string("checkpoint: cannot open ") + path);
    }
    ~File() { if (f) std::fclose(f); }
    void write(const void* p, size_t n) {
        if (n && std::fwrite(p, 1, n, f) != n) raise(BMQ_ERR_STORE, "checkpoint: write failed");
    }
    void read(void* p, size_t n) {
        if (n && std::fread(p, 1, n, f) != n) raise(BMQ_ERR_STORE, "checkpoint: truncated file");
    }
};
}  // namespace

void Engine::save_checkpoint(const char* path) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    if (sharded()) raise(BMQ_ERR_ENGINE, "checkpoint: save each rank's payloads through export instead");
    if (!cfg_.compress) raise(BMQ_ERR_INVALID_ARGUMENT, "checkpoint requires compression");
    const uint64_t nid = L_.num_blocks();
    std::vector<uint64_t> ids(nid), meta(4 * nid);
    for (uint64_t i = 0; i < nid; ++i) ids[i] = i;
    export_payloads(ids.data(), nid, meta.data(), nullptr, 0);  // sizes and sums first
    uint64_t total = 0;
    for (uint64_t i = 0; i < nid; ++i) total += (meta[4 * i] + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
    PinnedBuf buf(total);
    export_payloads(ids.data(), nid, meta.data(), buf.p, std::max<uint64_t>(total, 16));
    std::vector<uint8_t> acct;
    store_.serialize(acct);
    const uint32_t head32[4] = {L_.n, L_.b, 1u, 0u};
    const double br = cfg_.error_bound;
    const uint64_t head64[7] = {fnv1a(gates_.data(), gates_.size() * sizeof(bmq_gate)),
                                fnv1a(plan_.data(), plan_.size() * sizeof(bmq_stage)),
                                next_stage_, stage_compress_calls_, stage_decompress_calls_, acct.size(), total};
    File f(path, "wb");
    f.write(kCkptMagic, 8);
    f.write(head32, sizeof head32);
    f.write(&br, 8);
    f.write(head64, sizeof head64);
    f.write(acct.data(), acct.size());
    f.write(meta.data(), meta.size() * 8);
    f.write(buf.p, total);
}

uint64_t Engine::load_checkpoint(const char* path) {
    BMQ_CUDA(cudaSetDevice(dev_));
    if (sharded()) raise(BMQ_ERR_ENGINE, "checkpoint: load each rank's payloads through import instead");
    if (!cfg_.compress) raise(BMQ_ERR_INVALID_ARGUMENT, "checkpoint requires compression");
    File f(path, "rb");
    char magic[8];
    f.read(magic, 8);
    if (std::memcmp(magic, kCkptMagic, 8)) raise(BMQ_ERR_STORE, "checkpoint: not a checkpoint file");
    uint32_t head32[4];
    double br;
    uint64_t head64[7];
    f.read(head32, sizeof head32);
    f.read(&br, 8);
    f.read(head64, sizeof head64);
    if (head32[2] != 1u) raise(BMQ_ERR_STORE, "checkpoint: unsupported version");
    if (head32[0] != L_.n || head32[1] != L_.b || br != cfg_.error_bound)
        raise(BMQ_ERR_STORE, "checkpoint: qubits, block bits or error bound differ from this simulator");
    if (head64[0] != fnv1a(gates_.data(), gates_.size() * sizeof(bmq_gate)) ||
        head64[1] != fnv1a(plan_.data(), plan_.size() * sizeof(bmq_stage)))
        raise(BMQ_ERR_STORE, "checkpoint: circuit or stage plan differs from this simulator");
    const uint64_t next = head64[2];
    if (next > plan_.size()) raise(BMQ_ERR_STORE, "checkpoint: stage cursor out of range");
    const uint64_t nid = L_.num_blocks();
    std::vector<uint8_t> acct(head64[5]);
    f.read(acct.data(), acct.size());
    std::vector<uint64_t> ids(nid), meta(4 * nid);
    f.read(meta.data(), meta.size() * 8);
    uint64_t total = 0;
    for (uint64_t i = 0; i < nid; ++i) {
        ids[i] = i;
        total += (meta[4 * i] + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
    }
    if (total != head64[6]) raise(BMQ_ERR_STORE, "checkpoint: payload index does not match the payload bytes");
    PinnedBuf buf(total);
    f.read(buf.p, total);
    // fresh arena: the previous payloads are dropped, then every id imported
    reset();
    init_state();
    StoreModel model = store_;
    model.deserialize(acct.data(), acct.size());
    import_payloads(ids.data(), nid, meta.data(), buf.p);
    store_ = model;
    next_stage_ = next;
    stage_compress_calls_ = head64[3];
    stage_decompress_calls_ = head64[4];
    return next;
}

}  // namespace bmq

