// gates.cu — bit-exact gate-stage engine (apply_stage / apply_unitary2/4,
// kernel.hpp:24-122) on device buffers.
//
// Gates are applied one by one in program order — their arithmetic is never
// fused, so every amplitude sees exactly the reference's rounding sequence —
// but their MEMORY traffic is fused: a pass loads one tile of 2^tb
// amplitudes into shared memory, applies a run of gates whose mixing bits
// all lie inside the tile, and writes the tile back once. Diagonal gates
// (Z, S, T, RZ, P, CZ, CP, ...) and CX controls never mix amplitudes, so
// they add no tile bits; a QFT stage of dozens of controlled phases is one
// pass. Tiles always contain buffer bits 0..4 so global accesses coalesce.
#include <algorithm>

#include "gates.cuh"

namespace bmq {

namespace {

EntryType classify(const Cx& z) {
    if (z.re == 0.0 && z.im == 0.0) return ET_ZERO;
    if (z.im == 0.0 && z.re == 1.0) return ET_ONE;
    if (z.im == 0.0 && z.re == -1.0) return ET_NEG;
    if (z.im == 0.0) return ET_REAL;
    if (z.re == 0.0) return ET_IMAG;
    return ET_CPLX;
}

void fill_matrix(GateOp& op, const Cx* u, int n) {
    for (int i = 0; i < n; ++i) {
        op.m[2 * i] = u[i].re;
        op.m[2 * i + 1] = u[i].im;
        op.et[i] = classify(u[i]);
    }
}

}  // namespace

GateOp make_op(const bmq_gate& g, uint32_t hi_bit, uint32_t lo_bit) {
    GateOp op{};
    Cx u[16];
    const int dim = gate_matrix(g, u);
    op.hi = static_cast<uint8_t>(hi_bit);
    op.lo = static_cast<uint8_t>(dim == 4 ? lo_bit : 0);
    if (dim == 2) {
        fill_matrix(op, u, 4);
        op.type = (op.et[1] == ET_ZERO && op.et[2] == ET_ZERO) ? OP_DIAG : OP_U2;
    } else {
        fill_matrix(op, u, 16);
        op.type = g.kind == BMQ_GATE_CX ? OP_CX : OP_CDIAG;
    }
    return op;
}

GateOp make_matrix_op(const Cx* u, bool two_qubit, uint32_t hi_bit, uint32_t lo_bit) {
    GateOp op{};
    op.hi = static_cast<uint8_t>(hi_bit);
    op.lo = static_cast<uint8_t>(two_qubit ? lo_bit : 0);
    fill_matrix(op, u, two_qubit ? 16 : 4);
    if (two_qubit)
        op.type = OP_U4;
    else
        op.type = (op.et[1] == ET_ZERO && op.et[2] == ET_ZERO) ? OP_DIAG : OP_U2;
    return op;
}

GateProgram::~GateProgram() {
    if (d_ops) cudaFree(d_ops);
}

namespace {

uint64_t mixing_bits(const GateOp& op) {
    switch (op.type) {
    case OP_U2: return 1ull << op.hi;
    case OP_CX: return 1ull << op.lo;
    case OP_U4: return (1ull << op.hi) | (1ull << op.lo);
    default: return 0;
    }
}

uint8_t rank_in(uint64_t mask, uint32_t bit) {
    return static_cast<uint8_t>(__builtin_popcountll(mask & ((1ull << bit) - 1)));
}

}  // namespace

void build_program(GateProgram& prog, std::vector<GateOp> ops, uint32_t total_bits) {
    prog.total_bits = total_bits;
    prog.passes.clear();
    const uint64_t all = total_bits >= 64 ? ~0ull : (1ull << total_bits) - 1;
    const uint32_t tb = std::min(total_bits, kMaxTileBits);
    const uint64_t coalesce = (1ull << std::min(5u, total_bits)) - 1;
    prog.all_diagonal = true;
    prog.diag_cond_mask = 0;
    for (const GateOp& op : ops) {
        if (mixing_bits(op)) prog.all_diagonal = false;
        if (op.type == OP_DIAG) prog.diag_cond_mask |= 1ull << op.hi;
        if (op.type == OP_CDIAG) prog.diag_cond_mask |= (1ull << op.hi) | (1ull << op.lo);
    }
    const auto close = [&](uint64_t mix, uint32_t begin, uint32_t end) {
        uint64_t mask = (mix | coalesce) & all;
        for (uint32_t b = 0; __builtin_popcountll(mask) < static_cast<int>(tb); ++b) mask |= (1ull << b) & all;
        GatePass p{mask, tb, begin, end - begin};
        for (uint32_t i = begin; i < end; ++i) {
            GateOp& op = ops[i];
            op.in_hi = (mask >> op.hi) & 1;
            op.in_lo = (mask >> op.lo) & 1;
            op.tp_hi = op.in_hi ? rank_in(mask, op.hi) : 0;
            op.tp_lo = op.in_lo ? rank_in(mask, op.lo) : 0;
        }
        prog.passes.push_back(p);
    };
    uint64_t mix = 0;
    uint32_t begin = 0;
    for (uint32_t i = 0; i < ops.size(); ++i) {
        const uint64_t m = mixing_bits(ops[i]);
        if (__builtin_popcountll((mix | m | coalesce) & all) > static_cast<int>(tb) && i > begin) {
            close(mix, begin, i);
            begin = i;
            mix = 0;
        }
        mix |= m;
    }
    if (begin < ops.size()) close(mix, begin, static_cast<uint32_t>(ops.size()));
    prog.ops = std::move(ops);
    if (prog.d_ops) {
        cudaFree(prog.d_ops);
        prog.d_ops = nullptr;
    }
    if (!prog.ops.empty()) {
        BMQ_CUDA(cudaMalloc(&prog.d_ops, prog.ops.size() * sizeof(GateOp)));
        BMQ_CUDA(cudaMemcpy(prog.d_ops, prog.ops.data(), prog.ops.size() * sizeof(GateOp), cudaMemcpyHostToDevice));
    }
}

namespace {

struct C2 {
    double re, im;
};

// u * a for one classified entry, with the reference's rounding (no FMA).
__device__ __forceinline__ C2 entry_mul(uint8_t et, double ur, double ui, C2 a) {
    switch (et) {
    case ET_ONE: return a;
    case ET_NEG: return C2{-a.re, -a.im};
    case ET_REAL: return C2{__dmul_rn(ur, a.re), __dmul_rn(ur, a.im)};
    case ET_IMAG: return C2{-__dmul_rn(ui, a.im), __dmul_rn(ui, a.re)};
    default:
        return C2{__dsub_rn(__dmul_rn(ur, a.re), __dmul_rn(ui, a.im)),
                  __dadd_rn(__dmul_rn(ur, a.im), __dmul_rn(ui, a.re))};
    }
}

// sum_c u[r][c] * a[c], left to right over the nonzero entries.
template <int N>
__device__ __forceinline__ C2 mat_row(const GateOp* __restrict__ g, int r, const C2* a) {
    C2 acc{0.0, 0.0};
    bool any = false;
#pragma unroll
    for (int c = 0; c < N; ++c) {
        const int e = r * N + c;
        const uint8_t et = g->et[e];
        if (et == ET_ZERO) continue;
        const C2 t = entry_mul(et, g->m[2 * e], g->m[2 * e + 1], a[c]);
        acc = any ? C2{__dadd_rn(acc.re, t.re), __dadd_rn(acc.im, t.im)} : t;
        any = true;
    }
    return acc;
}

__device__ __forceinline__ uint32_t insert0(uint32_t x, uint32_t pos) {
    const uint32_t low = (1u << pos) - 1;
    return ((x & ~low) << 1) | (x & low);
}

__device__ __forceinline__ uint64_t deposit_x(uint64_t x, uint64_t mask) {
    uint64_t out = 0;
    while (x) {
        const uint64_t low = mask & (~mask + 1);
        if (x & 1) out |= low;
        x >>= 1;
        mask ^= low;
    }
    return out;
}

constexpr int kPassThreads = 256;

__global__ void __launch_bounds__(kPassThreads) k_gate_pass(double* __restrict__ buf, uint32_t lb, int interleaved,
                                                            uint64_t tile_mask, uint32_t tb,
                                                            const GateOp* __restrict__ ops, uint32_t nops) {
    extern __shared__ double sm[];
    const uint32_t tsz = 1u << tb;
    double* sre = sm;
    double* sim = sm + tsz;
    const uint32_t nth = blockDim.x, tid = threadIdx.x;
    const uint32_t per = tsz / nth;
    const uint64_t base = deposit_x(blockIdx.x, ~tile_mask);
    const uint64_t toff = deposit_x(tid, tile_mask);
    const uint64_t lmask = (1ull << lb) - 1;
    const auto addr = [&](uint64_t p) -> uint64_t {
        return interleaved ? 2 * p : (((p >> lb) << (lb + 1)) | (p & lmask));
    };
    const uint64_t im_off = interleaved ? 1 : (1ull << lb);
#pragma unroll 4
    for (uint32_t j = 0; j < per; ++j) {
        const uint32_t k = tid + j * nth;
        const uint64_t a = addr(base | toff | deposit_x(static_cast<uint64_t>(j) * nth, tile_mask));
        sre[k] = buf[a];
        sim[k] = buf[a + im_off];
    }
    bool owners_only = true;  // smem entries touched since the last barrier were written by their owners
    for (uint32_t i = 0; i < nops; ++i) {
        const GateOp* g = ops + i;
        const uint8_t type = g->type;
        if (type == OP_DIAG || type == OP_CDIAG) {
            if (!owners_only) {
                __syncthreads();
                owners_only = true;
            }
            const uint64_t bhi = (base >> g->hi) & 1, blo = (base >> g->lo) & 1;
            const uint8_t et = type == OP_DIAG ? 0 : 15;
            for (uint32_t j = 0; j < per; ++j) {
                const uint32_t k = tid + j * nth;
                const uint32_t hv = g->in_hi ? (k >> g->tp_hi) & 1 : static_cast<uint32_t>(bhi);
                uint8_t e;
                if (type == OP_DIAG) {
                    e = hv ? 3 : 0;
                } else {
                    const uint32_t lv = g->in_lo ? (k >> g->tp_lo) & 1 : static_cast<uint32_t>(blo);
                    if (!(hv && lv)) continue;
                    e = et;
                }
                const uint8_t ty = g->et[e];
                if (ty == ET_ONE) continue;
                const C2 r = ty == ET_ZERO ? C2{0.0, 0.0} : entry_mul(ty, g->m[2 * e], g->m[2 * e + 1], C2{sre[k], sim[k]});
                sre[k] = r.re;
                sim[k] = r.im;
            }
            continue;
        }
        __syncthreads();
        owners_only = false;
        if (type == OP_U2) {
            const uint32_t tp = g->tp_hi, m = 1u << tp;
            for (uint32_t r = tid; r < tsz / 2; r += nth) {
                const uint32_t i0 = insert0(r, tp), i1 = i0 | m;
                const C2 a[2] = {{sre[i0], sim[i0]}, {sre[i1], sim[i1]}};
                const C2 o0 = mat_row<2>(g, 0, a), o1 = mat_row<2>(g, 1, a);
                sre[i0] = o0.re;
                sim[i0] = o0.im;
                sre[i1] = o1.re;
                sim[i1] = o1.im;
            }
        } else if (type == OP_CX) {
            const uint32_t tp = g->tp_lo, m = 1u << tp;
            const uint32_t bctl = static_cast<uint32_t>((base >> g->hi) & 1);
            for (uint32_t r = tid; r < tsz / 2; r += nth) {
                const uint32_t i0 = insert0(r, tp), i1 = i0 | m;
                const uint32_t ctl = g->in_hi ? (i0 >> g->tp_hi) & 1 : bctl;
                if (!ctl) continue;
                const double r0 = sre[i0], m0 = sim[i0];
                sre[i0] = sre[i1];
                sim[i0] = sim[i1];
                sre[i1] = r0;
                sim[i1] = m0;
            }
        } else {  // OP_U4
            const uint32_t ph = g->tp_hi, pl = g->tp_lo;
            const uint32_t p0 = ph < pl ? ph : pl, p1 = ph < pl ? pl : ph;
            const uint32_t mh = 1u << ph, ml = 1u << pl;
            for (uint32_t r = tid; r < tsz / 4; r += nth) {
                const uint32_t i = insert0(insert0(r, p0), p1);
                const uint32_t idx[4] = {i, i | ml, i | mh, i | mh | ml};
                C2 a[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) a[q] = C2{sre[idx[q]], sim[idx[q]]};
                C2 o[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) o[q] = mat_row<4>(g, q, a);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    sre[idx[q]] = o[q].re;
                    sim[idx[q]] = o[q].im;
                }
            }
        }
    }
    __syncthreads();
#pragma unroll 4
    for (uint32_t j = 0; j < per; ++j) {
        const uint32_t k = tid + j * nth;
        const uint64_t a = addr(base | toff | deposit_x(static_cast<uint64_t>(j) * nth, tile_mask));
        buf[a] = sre[k];
        buf[a + im_off] = sim[k];
    }
}

}  // namespace

void run_program(cudaStream_t st, const GateProgram& prog, double* buf, uint32_t lb, bool interleaved,
                 uint64_t nreps, uint64_t* launches) {
    static thread_local int attr_dev = -1;
    int dev = 0;
    BMQ_CUDA(cudaGetDevice(&dev));
    if (attr_dev != dev) {
        BMQ_CUDA(cudaFuncSetAttribute(k_gate_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      2 * (1 << kMaxTileBits) * static_cast<int>(sizeof(double))));
        attr_dev = dev;
    }
    for (const GatePass& p : prog.passes) {
        const uint64_t tiles = nreps << (prog.total_bits - p.tb);
        const uint32_t nth = std::min<uint32_t>(kPassThreads, 1u << p.tb);
        const size_t smem = 2 * (size_t(1) << p.tb) * sizeof(double);
        k_gate_pass<<<static_cast<uint32_t>(tiles), nth, smem, st>>>(buf, lb, interleaved ? 1 : 0, p.tile_mask, p.tb,
                                                                    prog.d_ops + p.begin, p.count);
        BMQ_CUDA(cudaGetLastError());
        if (launches) ++*launches;
    }
}

}  // namespace bmq
