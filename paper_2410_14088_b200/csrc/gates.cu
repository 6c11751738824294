// gates.cu — bit-exact gate-stage engine (apply_stage / apply_unitary2/4,
// kernel.hpp:24-122) on device buffers.
//
// Gates are applied one by one in program order — their arithmetic is never
// fused, so every amplitude sees exactly the reference's rounding sequence —
// but their MEMORY traffic is fused: a pass loads one tile of 2^12
// amplitudes into shared memory, applies a run of gates whose mixing bits
// all lie inside the tile, and writes the tile back once. Diagonal gates
// (Z, S, T, RZ, P, CZ, CP, ...) and CX controls never mix amplitudes, so
// they add no tile bits; a QFT stage of dozens of controlled phases is one
// pass. Tiles always contain buffer bits 0..4 so global accesses coalesce.
//
// Diagonal runs are applied amplitude by amplitude (no barriers). A run of
// controlled phases sharing one control bit (a QFT "phase chain") is one
// OP_CHAIN: the amplitude walks the set bits of (index & R) in program order
// and multiplies by each bit's phase, so the cost is the number of phases
// that actually apply, not the number of gates.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <functional>

#include "codec_util.cuh"
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
    if (d_ops) dev_free(d_ops);
    if (d_chain_tab) dev_free(d_chain_tab);
    if (d_perm_tab) dev_free(d_perm_tab);
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

// Runs of `mask` restricted to [0, limit); when tail_to is set, the source
// bits past the mask's runs are appended as one run landing at tail_to.
BitRuns make_runs(uint64_t mask, uint32_t limit, int tail_to) {
    BitRuns r{};
    uint32_t src = 0;
    for (uint32_t b = 0; b < limit;) {
        if (!((mask >> b) & 1)) {
            ++b;
            continue;
        }
        uint32_t e = b;
        while (e < limit && ((mask >> e) & 1)) ++e;
        r.src[r.n] = static_cast<uint8_t>(src);
        r.dst[r.n] = static_cast<uint8_t>(b);
        r.width[r.n] = static_cast<uint8_t>(e - b);
        ++r.n;
        src += e - b;
        b = e;
    }
    if (tail_to >= 0) {
        r.src[r.n] = static_cast<uint8_t>(src);
        r.dst[r.n] = static_cast<uint8_t>(tail_to);
        r.width[r.n] = static_cast<uint8_t>(64 - std::max<uint32_t>(src, tail_to));
        ++r.n;
    }
    return r;
}

FastOp to_fast(const GateOp& g) {
    FastOp f{};
    f.type = g.type;
    f.tp_hi = g.tp_hi;
    f.tp_lo = g.tp_lo;
    f.in_hi = g.in_hi;
    f.in_lo = g.in_lo;
    f.hi = g.hi;
    f.lo = g.lo;
    const auto take = [&](int slot, int e) {
        f.et[slot] = g.et[e];
        f.m[2 * slot] = g.m[2 * e];
        f.m[2 * slot + 1] = g.m[2 * e + 1];
    };
    if (g.type == OP_U2) {
        for (int e = 0; e < 4; ++e) take(e, e);
        // real 2x2 (H, RY, X, Z): the real product form is exact for every
        // entry class incl. 0 and +-1 (up to the sign of an exact zero)
        bool real = true;
        for (int e = 0; e < 4; ++e) real = real && g.m[2 * e + 1] == 0.0;
        f.pad = real ? 1 : 0;
        // real diagonal, imaginary off-diagonal (RX): one specialised form too
        if (!real && g.m[1] == 0.0 && g.m[7] == 0.0 && g.m[2] == 0.0 && g.m[4] == 0.0) f.pad = 2;
    } else if (g.type == OP_DIAG) {
        take(0, 0);
        take(1, 3);
    } else if (g.type == OP_CDIAG) {
        take(0, 15);
    }
    return f;
}

// Tile positions of a lone chain's walk (4 bits each, packed): five lane
// positions (the lowest, so SMEM accesses stay dense), three warp positions,
// three per-thread positions and (control outside the tile) one round
// position. The per-thread positions prefer tile bits outside R, where the
// thread's amplitudes have identical masks and every product is useful.
uint64_t chain_positions(uint64_t tile_mask, int pc, uint64_t R) {
    std::vector<int> rest, lanes;
    for (int p = 0; p < static_cast<int>(kMaxTileBits); ++p)
        if (p != pc) rest.push_back(p);
    lanes.assign(rest.begin(), rest.begin() + 5);
    rest.erase(rest.begin(), rest.begin() + 5);
    const auto in_r = [&](int p) {
        uint64_t m = tile_mask;
        for (int k = 0; k < p; ++k) m &= m - 1;  // drop the p lowest set bits
        const int bit = __builtin_ctzll(m);
        return ((R >> bit) & 1) != 0;
    };
    std::stable_sort(rest.begin(), rest.end(), [&](int a, int b) { return !in_r(a) && in_r(b); });
    const int qb = kChainQBits;
    std::vector<int> q(rest.begin(), rest.begin() + qb);     // per-thread
    std::vector<int> other(rest.begin() + qb, rest.end());   // warps, then rounds
    std::vector<int> order = lanes;                           // [0, 5): lanes
    order.insert(order.end(), other.begin(), other.begin() + 3);  // [5, 8): warps
    order.insert(order.end(), q.begin(), q.end());                // [8, 8 + qb): per thread
    order.insert(order.end(), other.begin() + 3, other.end());    // rounds
    uint64_t plan = 0;
    for (size_t i = 0; i < order.size(); ++i) plan |= static_cast<uint64_t>(order[i]) << (4 * i);
    return plan;
}

// Fast ops for [begin, end): consecutive CP-like ops (OP_CDIAG with a
// complex entry) that share one bit and whose other bits are distinct and
// monotone become one OP_CHAIN with a 64-entry phase table.
std::vector<FastOp> fuse_chains(const std::vector<GateOp>& ops, uint32_t begin, uint32_t end,
                                std::vector<double>& tab, uint64_t tile_mask) {
    std::vector<FastOp> out;
    const size_t pass_base = tab.size();  // chain offsets are relative to the pass
    const auto chainable = [](const GateOp& o) {
        return o.type == OP_CDIAG && o.et[15] == ET_CPLX && o.hi < 32 && o.lo < 32;
    };
    uint32_t i = begin;
    while (i < end) {
        const GateOp& a = ops[i];
        if (chainable(a) && i + 1 < end && chainable(ops[i + 1])) {
            const GateOp& b = ops[i + 1];
            int c = -1;
            if (b.hi == a.hi || b.lo == a.hi)
                c = a.hi;
            else if (b.hi == a.lo || b.lo == a.lo)
                c = a.lo;
            if (c >= 0) {
                const auto other = [c](const GateOp& o) { return static_cast<int>(o.hi == c ? o.lo : o.hi); };
                const int oa = other(a), ob = other(b);
                if (oa != ob) {
                    const bool desc = ob < oa;
                    uint64_t R = (1ull << oa) | (1ull << ob);
                    int last = ob;
                    uint32_t j = i + 2;
                    while (j < end && chainable(ops[j]) && (ops[j].hi == c || ops[j].lo == c)) {
                        const int oj = other(ops[j]);
                        if ((R >> oj) & 1) break;
                        if (desc ? !(oj < last) : !(oj > last)) break;
                        R |= 1ull << oj;
                        last = oj;
                        ++j;
                    }
                    const size_t off = tab.size();
                    tab.resize(off + 64, 0.0);  // 32 entries (re, im)
                    for (uint32_t k = i; k < j; ++k) {
                        const int o = other(ops[k]);
                        tab[off + 2 * o] = ops[k].m[30];
                        tab[off + 2 * o + 1] = ops[k].m[31];
                    }
                    FastOp f{};
                    f.type = OP_CHAIN;
                    f.hi = static_cast<uint8_t>(c);
                    f.in_hi = static_cast<uint8_t>((tile_mask >> c) & 1);
                    f.tp_hi = f.in_hi ? rank_in(tile_mask, c) : 0;
                    const uint64_t plan = chain_positions(tile_mask, f.in_hi ? f.tp_hi : -1, R);
                    std::memcpy(&f.m[1], &plan, 8);
                    f.et[0] = desc ? 1 : 0;
                    f.pad2 = static_cast<uint32_t>((off - pass_base) / 2);
                    std::memcpy(&f.m[0], &R, 8);
                    out.push_back(f);
                    i = j;
                    continue;
                }
            }
        }
        out.push_back(to_fast(a));
        ++i;
    }
    return out;
}

// Unit index of an exact matrix entry: 1 -> 0, i -> 1, -1 -> 2, -i -> 3.
int unit_of(double re, double im) {
    if (im == 0.0 && re == 1.0) return 0;
    if (re == 0.0 && im == 1.0) return 1;
    if (im == 0.0 && re == -1.0) return 2;
    if (re == 0.0 && im == -1.0) return 3;
    return -1;
}

bool to_mono(const GateOp& g, MonoOp& o) {
    o = MonoOp{};
    o.hi = g.hi;
    o.lo = g.lo;
    const auto unit = [&](int e) { return unit_of(g.m[2 * e], g.m[2 * e + 1]); };
    switch (g.type) {
    case OP_DIAG: {
        const int a = unit(0), b = unit(3);
        if (a < 0 || b < 0) return false;
        o.kind = MK_DIAG;
        o.u0 = static_cast<uint8_t>(a);
        o.u1 = static_cast<uint8_t>(b);
        return true;
    }
    case OP_CDIAG: {
        const int d = unit(15);
        if (unit(0) != 0 || unit(5) != 0 || unit(10) != 0 || d < 0) return false;
        o.kind = MK_CDIAG;
        o.u1 = static_cast<uint8_t>(d);
        return true;
    }
    case OP_CX:
        o.kind = MK_MIX;
        o.tp = g.tp_lo;
        o.ctl = g.in_hi ? 1 : 2;
        o.ctl_tp = g.tp_hi;
        return true;
    case OP_U2: {
        if (g.et[0] != ET_ZERO || g.et[3] != ET_ZERO) return false;
        const int a = unit(1), b = unit(2);
        if (a < 0 || b < 0) return false;
        o.kind = MK_MIX;
        o.tp = g.tp_hi;
        o.u0 = static_cast<uint8_t>(a);
        o.u1 = static_cast<uint8_t>(b);
        return true;
    }
    default: return false;
    }
}

// A program is code-domain when every op is monomial with unit entries and
// every pass tiles 2^12 amplitudes.
void build_mono(GateProgram& prog) {
    prog.mono = false;
    if (prog.d_perm_tab) {
        dev_free(prog.d_perm_tab);
        prog.d_perm_tab = nullptr;
    }
    if (prog.ops.empty() || prog.total_bits < kMaxTileBits) return;
    std::vector<std::shared_ptr<MonoPass>> mps;
    const uint64_t all = prog.total_bits >= 64 ? ~0ull : (1ull << prog.total_bits) - 1;
    for (const GatePass& p : prog.passes) {
        if (p.tb != kMaxTileBits || p.count > static_cast<uint32_t>(kMaxMonoOps)) return;
        auto mp = std::make_shared<MonoPass>();
        std::memset(mp.get(), 0, sizeof(MonoPass));
        mp->tile = make_runs(p.tile_mask, prog.total_bits, -1);
        mp->base = make_runs(~p.tile_mask & all, prog.total_bits, static_cast<int>(prog.total_bits));
        mp->nops = p.count;
        for (uint32_t i = 0; i < p.count; ++i)
            if (!to_mono(prog.ops[p.begin + i], mp->ops[i])) return;
        mps.push_back(mp);
    }
    for (size_t i = 0; i < mps.size(); ++i) prog.passes[i].mp = mps[i];
    prog.mono = true;
    // Table form of each pass (composite signed permutation per pattern).
    if (prog.total_bits + 1 > 32) return;  // planar tile offsets are 32-bit
    std::vector<uint16_t> tabs;
    std::vector<std::pair<size_t, std::shared_ptr<PermPass>>> pps;
    for (size_t pi = 0; pi < prog.passes.size(); ++pi) {
        const GatePass& p = prog.passes[pi];
        const MonoPass& mp = *p.mp;
        const auto in_tile = [&](uint32_t bit) { return ((p.tile_mask >> bit) & 1) != 0; };
        std::vector<uint8_t> pat;
        const auto need = [&](uint32_t bit) {
            if (!in_tile(bit) && std::find(pat.begin(), pat.end(), bit) == pat.end()) pat.push_back(static_cast<uint8_t>(bit));
        };
        for (uint32_t i = 0; i < mp.nops; ++i) {
            const MonoOp& o = mp.ops[i];
            if (o.kind == MK_DIAG) need(o.hi);
            if (o.kind == MK_CDIAG) {
                need(o.hi);
                need(o.lo);
            }
            if (o.kind == MK_MIX && o.ctl == 2) need(o.hi);
        }
        if (pat.size() > static_cast<size_t>(kMaxPatBits)) continue;
        auto pp = std::make_shared<PermPass>();
        std::memset(pp.get(), 0, sizeof(PermPass));
        pp->tile = mp.tile;
        pp->base = mp.base;
        pp->npat_bits = static_cast<uint32_t>(pat.size());
        for (uint32_t b = 0, k = 0; b < 64; ++b) {  // buffer bits of tile positions 2..6 and 10..11
            if (!((p.tile_mask >> b) & 1)) continue;
            if (k >= 2 && k <= 6) pp->lane_bits |= 1ull << b;
            if (k >= 10) pp->group_bits |= 1ull << b;
            ++k;
        }
        for (size_t i = 0; i < pat.size(); ++i) pp->pat_bits[i] = pat[i];
        const size_t off = tabs.size();
        for (uint32_t P = 0; P < (1u << pat.size()); ++P) {
            const auto bitval = [&](uint32_t bit, uint32_t k) -> uint32_t {
                if (in_tile(bit)) return (k >> rank_in(p.tile_mask, bit)) & 1;
                const size_t i = std::find(pat.begin(), pat.end(), bit) - pat.begin();
                return (P >> i) & 1;
            };
            std::vector<uint16_t> src(4096);
            std::vector<uint8_t> U(4096, 0);
            for (uint32_t k = 0; k < 4096; ++k) src[k] = static_cast<uint16_t>(k);
            for (uint32_t i = 0; i < mp.nops; ++i) {
                const MonoOp& o = mp.ops[i];
                if (o.kind == MK_DIAG) {
                    for (uint32_t k = 0; k < 4096; ++k) U[k] = (U[k] + (bitval(o.hi, k) ? o.u1 : o.u0)) & 3;
                } else if (o.kind == MK_CDIAG) {
                    for (uint32_t k = 0; k < 4096; ++k)
                        if (bitval(o.hi, k) && bitval(o.lo, k)) U[k] = (U[k] + o.u1) & 3;
                } else {
                    const uint32_t m = 1u << o.tp;
                    for (uint32_t k = 0; k < 4096; ++k) {
                        if (k & m) continue;
                        const uint32_t i0 = k, i1 = k | m;
                        const uint32_t ctl = o.ctl == 0 ? 1u : (o.ctl == 1 ? (i0 >> o.ctl_tp) & 1 : bitval(o.hi, k));
                        if (!ctl) continue;
                        const uint16_t s0 = src[i1], s1 = src[i0];
                        const uint8_t v0 = (U[i1] + o.u0) & 3, v1 = (U[i0] + o.u1) & 3;
                        src[i0] = s0;
                        U[i0] = v0;
                        src[i1] = s1;
                        U[i1] = v1;
                    }
                }
            }
            for (uint32_t k = 0; k < 4096; ++k) {
                const uint32_t u = U[k];
                if (u & 1) pp->reim_swap = 1;
                tabs.push_back(static_cast<uint16_t>(src[k] | (u & 1) << 12 | ((u ^ (u >> 1)) & 1) << 13 | (u >> 1) << 14));
            }
        }
        pps.push_back({pi, pp});
        pp->table = reinterpret_cast<const uint16_t*>(off);  // fixed up after upload
    }
    if (pps.empty()) return;
    prog.d_perm_tab = static_cast<uint16_t*>(dev_alloc(tabs.size() * sizeof(uint16_t)));
    BMQ_CUDA(cudaMemcpy(prog.d_perm_tab, tabs.data(), tabs.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    for (auto& [pi, pp] : pps) {
        pp->table = prog.d_perm_tab + reinterpret_cast<uintptr_t>(pp->table);
        prog.passes[pi].pp = pp;
    }
}

// Lazy CX (see FastOp): fold every CX of a fast pass into the pass's GF(2)
// map y = M x ^ c, annotate the other ops with the rows / columns of M they
// need, and materialise the map before phase chains (which address
// amplitudes by their full index).
void lazify(std::vector<FastOp>& fops, FastPass& fp, uint32_t& ncx, uint32_t& nperm) {
    uint16_t rows[kMaxTileBits], cols[kMaxTileBits];
    const auto reset = [&]() {
        for (uint32_t i = 0; i < kMaxTileBits; ++i) rows[i] = cols[i] = static_cast<uint16_t>(1u << i);
    };
    const auto identity = [&]() {
        for (uint32_t i = 0; i < kMaxTileBits; ++i)
            if (rows[i] != (1u << i)) return false;
        return true;
    };
    reset();
    bool affine = false;  // some CX has its control outside the tile: c may be nonzero
    std::vector<FastOp> out;
    for (FastOp f : fops) {
        switch (f.type) {
        case OP_CX:
            ++ncx;
            if (f.in_hi) {
                rows[f.tp_lo] ^= rows[f.tp_hi];
                cols[f.tp_hi] ^= cols[f.tp_lo];
            } else {
                affine = true;
            }
            break;
        case OP_U2:
            f.mrow = rows[f.tp_hi];
            f.dvec = cols[f.tp_hi];
            break;
        case OP_DIAG:
            f.mrow = f.in_hi ? rows[f.tp_hi] : 0;
            break;
        case OP_CDIAG:
            f.mrow = f.in_hi ? rows[f.tp_hi] : 0;
            f.mrow2 = f.in_lo ? rows[f.tp_lo] : 0;
            break;
        case OP_CHAIN:
            if (!identity() || affine) {
                FastOp m{};
                m.type = OP_PERM;
                ++nperm;
                std::memcpy(&m.m[0], cols, sizeof cols);
                out.push_back(m);
                reset();
                affine = false;
            }
            break;
        default: break;
        }
        out.push_back(f);
    }
    std::memcpy(fp.minv, cols, sizeof cols);
    fp.final_perm = (!identity() || affine) ? 1u : 0u;
    fops = std::move(out);
}

}  // namespace

// Register-streaming form of a pass (see StreamPass), or null when the pass
// needs the tiled kernel: other op types (U4), partners outside the lane
// bits and two more bits, a CX map that is not the identity at the end, or
// too many ops for per-amplitude application to beat the tile's phase chains.
static std::shared_ptr<StreamPass> make_stream(const std::vector<GateOp>& ops, uint32_t begin, uint32_t end,
                                               uint32_t total_bits) {
    if (total_bits < 12 || total_bits > 63) return nullptr;
    // lazy CX: rows of M (logical bit t = parity(row[t] & x)) and columns of M^-1
    uint64_t row[64], col[64];
    for (uint32_t t = 0; t < total_bits; ++t) row[t] = col[t] = 1ull << t;
    uint64_t R = 0;
    uint32_t nops = 0;
    for (uint32_t i = begin; i < end; ++i) {
        const GateOp& g = ops[i];
        if (g.type == OP_CX) {
            row[g.lo] ^= row[g.hi];
            col[g.hi] ^= col[g.lo];
        } else if (g.type == OP_U2) {
            R |= col[g.hi] & ~31ull;
            ++nops;
        } else if (g.type == OP_DIAG || g.type == OP_CDIAG) {
            ++nops;
        } else {
            return nullptr;
        }
    }
    for (uint32_t t = 0; t < total_bits; ++t)
        if (row[t] != 1ull << t) return nullptr;  // the pass would end permuted
    if (__builtin_popcountll(R) > kStreamNQ || nops > static_cast<uint32_t>(kMaxStreamOps)) return nullptr;
    uint64_t Q = R;
    for (uint32_t b = 5; __builtin_popcountll(Q) < kStreamNQ; ++b) Q |= 1ull << b;
    auto sp = std::make_shared<StreamPass>();
    std::memset(sp.get(), 0, sizeof(StreamPass));
    uint32_t qi = 0;
    uint64_t dep[1 << kStreamNQ] = {};
    for (uint32_t b = 0; b < 64; ++b)
        if (Q >> b & 1) sp->qbit[qi++] = static_cast<uint8_t>(b);
    for (uint32_t r = 0; r < (1u << kStreamNQ); ++r)
        for (uint32_t k = 0; k < kStreamNQ; ++k)
            if (r >> k & 1) dep[r] |= 1ull << sp->qbit[k];
    const uint64_t all = (1ull << total_bits) - 1;
    sp->base = make_runs(~(Q | 31ull) & all, total_bits, static_cast<int>(total_bits));
    const auto pat = [&](uint64_t rw) {
        uint8_t p = 0;
        for (uint32_t r = 0; r < (1u << kStreamNQ); ++r) p |= static_cast<uint8_t>((__builtin_popcountll(rw & dep[r]) & 1) << r);
        return p;
    };
    for (uint32_t t = 0; t < total_bits; ++t) row[t] = col[t] = 1ull << t;
    for (uint32_t i = begin; i < end; ++i) {
        const GateOp& g = ops[i];
        if (g.type == OP_CX) {
            row[g.lo] ^= row[g.hi];
            col[g.hi] ^= col[g.lo];
            continue;
        }
        StreamOp& o = sp->ops[sp->nops++];
        o.type = g.type;
        o.row = row[g.hi] & ~Q;
        o.rpat = pat(row[g.hi]);
        const auto take = [&](int slot, int e) {
            o.et[slot] = g.et[e];
            o.m[2 * slot] = g.m[2 * e];
            o.m[2 * slot + 1] = g.m[2 * e + 1];
        };
        if (g.type == OP_U2) {
            for (int e = 0; e < 4; ++e) take(e, e);
            // specialised forms (k_stream_pass): real diagonal entries with real
            // or imaginary off-diagonal ones, no zero among them (row2 skips
            // zero products, the specialised form adds +-0: equal up to the
            // sign of a zero)
            const auto cls = [&](int e) { return g.et[e] == ET_ONE || g.et[e] == ET_NEG ? ET_REAL : g.et[e]; };
            if (cls(0) == ET_REAL && cls(3) == ET_REAL && cls(1) == ET_REAL && cls(2) == ET_REAL) o.pad = 1;
            if (cls(0) == ET_REAL && cls(3) == ET_REAL && cls(1) == ET_IMAG && cls(2) == ET_IMAG) o.pad = 2;
            const uint64_t d = col[g.hi];
            o.dl = static_cast<uint32_t>(d & 31);
            for (uint32_t k = 0; k < kStreamNQ; ++k)
                if (d >> sp->qbit[k] & 1) o.dq |= static_cast<uint8_t>(1u << k);
        } else if (g.type == OP_DIAG) {
            take(0, 0);
            take(1, 3);
        } else {
            take(0, 15);
            o.row2 = row[g.lo] & ~Q;
            o.rpat2 = pat(row[g.lo]);
        }
    }
    return sp;
}

void build_program(GateProgram& prog, std::vector<GateOp> ops, uint32_t total_bits) {
    prog.total_bits = total_bits;
    prog.passes.clear();
    prog.lazy_cx = prog.perms = 0;
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
    prog.chain_tab.clear();
    std::function<void(uint32_t, uint32_t)> close = [&](uint32_t begin, uint32_t end) {
        uint64_t mix = 0;
        for (uint32_t i = begin; i < end; ++i) mix |= mixing_bits(ops[i]);
        uint64_t mask = (mix | coalesce) & all;
        for (uint32_t b = 0; __builtin_popcountll(mask) < static_cast<int>(tb); ++b) mask |= (1ull << b) & all;
        GatePass p{mask, tb, begin, end - begin};
        bool fast = tb == kMaxTileBits;
        for (uint32_t i = begin; i < end; ++i) {
            GateOp& op = ops[i];
            op.in_hi = (mask >> op.hi) & 1;
            op.in_lo = (mask >> op.lo) & 1;
            op.tp_hi = op.in_hi ? rank_in(mask, op.hi) : 0;
            op.tp_lo = op.in_lo ? rank_in(mask, op.lo) : 0;
            if (op.type == OP_U4) fast = false;
        }
        if (fast) {
            const size_t tab_mark = prog.chain_tab.size();
            std::vector<FastOp> fops = fuse_chains(ops, begin, end, prog.chain_tab, mask);
            FastPass lazy{};
            uint32_t ncx = 0, nperm = 0;
            lazify(fops, lazy, ncx, nperm);
            if (fops.size() > static_cast<size_t>(kMaxFastOps) && end - begin > 1) {
                prog.chain_tab.resize(tab_mark);
                const uint32_t mid = begin + (end - begin) / 2;
                close(begin, mid);
                close(mid, end);
                return;
            }
            if (fops.size() <= static_cast<size_t>(kMaxFastOps)) {
                auto fp = std::make_shared<FastPass>();
                std::memset(fp.get(), 0, sizeof(FastPass));
                fp->tile = make_runs(mask, total_bits, -1);
                fp->base = make_runs(~mask & all, total_bits, static_cast<int>(total_bits));
                fp->nops = static_cast<uint32_t>(fops.size());
                std::memcpy(fp->minv, lazy.minv, sizeof fp->minv);
                prog.lazy_cx += ncx;
                prog.perms += nperm;
                fp->final_perm = lazy.final_perm;
                fp->tab_base = tab_mark / 2;
                fp->tab_entries = static_cast<uint32_t>((prog.chain_tab.size() - tab_mark) / 2);
                std::copy(fops.begin(), fops.end(), fp->ops);
                if (getenv("BMQ_DBG_PASSES")) {  // development aid: the pass's ops
                    fprintf(stderr, "pass %zu mask %llx ops %zu:", prog.passes.size(),
                            static_cast<unsigned long long>(mask), fops.size());
                    for (const FastOp& o : fops) fprintf(stderr, " %u/%u", o.type, o.tp_hi);
                    fprintf(stderr, "\n");
                }
                p.fast = true;
                p.fp = fp;
                // phase chains (QFT) walk only the set bits of each amplitude and the
                // tiled kernel tracks sparse tile support: those passes stay tiled
                bool chains = false;
                for (const FastOp& o : fops) chains = chains || o.type == OP_CHAIN;
                if (!chains) p.sp = make_stream(ops, begin, end, total_bits);
            }
        }
        prog.passes.push_back(p);
    };
    uint64_t mix = 0;
    uint32_t begin = 0;
    for (uint32_t i = 0; i < ops.size(); ++i) {
        const uint64_t m = mixing_bits(ops[i]);
        const bool too_wide = __builtin_popcountll((mix | m | coalesce) & all) > static_cast<int>(tb);
        const bool too_long = i - begin >= 4096u;
        if ((too_wide || too_long) && i > begin) {
            close(begin, i);
            begin = i;
            mix = 0;
        }
        mix |= m;
    }
    if (begin < ops.size()) close(begin, static_cast<uint32_t>(ops.size()));
    prog.ops = std::move(ops);
    build_mono(prog);
    if (prog.d_ops) {
        dev_free(prog.d_ops);
        prog.d_ops = nullptr;
    }
    if (prog.d_chain_tab) {
        dev_free(prog.d_chain_tab);
        prog.d_chain_tab = nullptr;
    }
    if (!prog.ops.empty()) {
        prog.d_ops = static_cast<GateOp*>(dev_alloc(prog.ops.size() * sizeof(GateOp)));
        BMQ_CUDA(cudaMemcpy(prog.d_ops, prog.ops.data(), prog.ops.size() * sizeof(GateOp), cudaMemcpyHostToDevice));
    }
    if (!prog.chain_tab.empty()) {
        prog.d_chain_tab = static_cast<double*>(dev_alloc(prog.chain_tab.size() * sizeof(double)));
        BMQ_CUDA(cudaMemcpy(prog.d_chain_tab, prog.chain_tab.data(), prog.chain_tab.size() * sizeof(double),
                            cudaMemcpyHostToDevice));
    }
    for (GatePass& p : prog.passes)
        if (p.fast) p.fp->chain_tab = prog.d_chain_tab;
}

namespace {

struct C2 {
    double re, im;
};

// u * a with the reference's rounding: (ur*ar - ui*ai, ur*ai + ui*ar), each
// product rounded, no FMA. For u = 1, -1, real or imaginary this equals the
// cheaper special forms except for the sign of an exact zero, so the
// specialised cases below are exact too.
__device__ __forceinline__ C2 cmul(double ur, double ui, C2 a) {
    return C2{__dsub_rn(__dmul_rn(ur, a.re), __dmul_rn(ui, a.im)), __dadd_rn(__dmul_rn(ur, a.im), __dmul_rn(ui, a.re))};
}

__device__ __forceinline__ C2 entry_mul(uint8_t et, double ur, double ui, C2 a) {
    switch (et) {
    case ET_ZERO: return C2{0.0, 0.0};
    case ET_ONE: return a;
    case ET_NEG: return C2{-a.re, -a.im};
    case ET_REAL: return C2{__dmul_rn(ur, a.re), __dmul_rn(ur, a.im)};
    case ET_IMAG: return C2{-__dmul_rn(ui, a.im), __dmul_rn(ui, a.re)};
    default: return cmul(ur, ui, a);
    }
}

__device__ __forceinline__ C2 cadd(C2 a, C2 b) { return C2{__dadd_rn(a.re, b.re), __dadd_rn(a.im, b.im)}; }

// Row r of a 2x2 (entries 2r, 2r+1): sum over nonzero entries, left to right.
__device__ __forceinline__ C2 row2(const uint8_t* et, const double* m, int r, C2 a0, C2 a1) {
    const uint8_t e0 = et[2 * r], e1 = et[2 * r + 1];
    if (e0 == ET_ZERO) return entry_mul(e1, m[4 * r + 2], m[4 * r + 3], a1);
    const C2 t0 = entry_mul(e0, m[4 * r], m[4 * r + 1], a0);
    if (e1 == ET_ZERO) return t0;
    return cadd(t0, entry_mul(e1, m[4 * r + 2], m[4 * r + 3], a1));
}

// sum_c u[r][c] * a[c], left to right over the nonzero entries (general 4x4).
__device__ __forceinline__ C2 row4(const GateOp* __restrict__ g, int r, const C2* a) {
    C2 acc{0.0, 0.0};
    bool any = false;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int e = r * 4 + c;
        const uint8_t et = g->et[e];
        if (et == ET_ZERO) continue;
        const C2 t = entry_mul(et, g->m[2 * e], g->m[2 * e + 1], a[c]);
        acc = any ? cadd(acc, t) : t;
        any = true;
    }
    return acc;
}

__device__ __forceinline__ uint32_t insert0(uint32_t x, uint32_t pos) {
    const uint32_t low = (1u << pos) - 1;
    return ((x & ~low) << 1) | (x & low);
}

__device__ __forceinline__ uint64_t runs_deposit(uint64_t x, const BitRuns& r) {
    uint64_t out = 0;
    for (uint32_t i = 0; i < r.n; ++i) {
        const uint32_t w = r.width[i];
        const uint64_t m = w >= 64 ? ~0ull : ((1ull << w) - 1);
        out |= ((x >> r.src[i]) & m) << r.dst[i];
    }
    return out;
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

__device__ __forceinline__ uint64_t planar_addr(uint64_t p, uint32_t lb, uint64_t lmask, int interleaved) {
    return interleaved ? 2 * p : (((p >> lb) << (lb + 1)) | (p & lmask));
}

// ------------------------------------------------------- fast tiled pass

constexpr int kFastThreads = 256;
constexpr int kPer = 16;  // tile positions per thread: k = tid + 256 j

// kParMask[m] bit j = parity(m & j), j < 16: the parity of a tile row's bits
// 8..11 (m) over the row index j of k = tid + 256 j
__constant__ uint32_t kParMask[16] = {0x0000, 0xaaaa, 0xcccc, 0x6666, 0xf0f0, 0x5a5a, 0x3c3c, 0x9696,
                                      0xff00, 0x55aa, 0x33cc, 0x9966, 0x0ff0, 0xa55a, 0xc33c, 0x6996};

// Diagonal ops [q0, q1) on one amplitude with full buffer index x; chain
// phase tables live in shared memory (stab).
// Walk the set bits of s in the chain's program order, multiplying by the
// phase of each (exact reference product per phase).
__device__ __forceinline__ C2 chain_walk(uint32_t s, bool desc, const double2* tab, C2 a) {
    if (a.re == 0.0 && a.im == 0.0) return a;  // zero stays zero (see chain_walk8)
    if (desc) {
        while (s) {
            const int r = 31 - __clz(s);
            s &= ~(1u << r);
            const double2 u = tab[r];
            a = cmul(u.x, u.y, a);
        }
    } else {
        while (s) {
            const int r = __ffs(s) - 1;
            s &= s - 1;
            const double2 u = tab[r];
            a = cmul(u.x, u.y, a);
        }
    }
    return a;
}

constexpr int kLanesPerStep = 1 << kChainQBits;

// pdep over a <= 12-bit tile mask: the low bits of r into the set bits of m.
__device__ __forceinline__ uint32_t deposit12(uint32_t r, uint32_t m) {
    if (__popc(m) > 6) {  // dense mask: insert a zero at each hole, lowest first
        for (uint32_t h = ~m & 0xfffu; h; h &= h - 1) r = insert0(r, __ffs(h) - 1);
        return r;
    }
    uint32_t out = 0;
    for (; m; m &= m - 1, r >>= 1)
        if (r & 1u) out |= m & (0u - m);
    return out;
}

template <bool kDesc>
__device__ __forceinline__ int next_bit(uint32_t s) {
    return kDesc ? 31 - __clz(s) : __ffs(s) - 1;
}

// A lone phase chain (control c, other bits R, phases in program order).
// Only amplitudes with bit c set are touched, so when c lies in the tile
// the thread takes eight of the 2048 positions with that bit set (bit c
// inserted into t + 256 i); when c is a base bit, the whole tile (or none of
// it) qualifies.
template <bool kDesc>
__device__ __forceinline__ void chain_walk8(double2* tile_s, const double2* tab, uint32_t tid, uint32_t xlo,
                                            const uint32_t* lut_lo, const uint32_t* lut_hi, int pc, uint32_t R,
                                            uint64_t plan, uint32_t round) {
    uint32_t pos[kLanesPerStep], sb[kLanesPerStep];
    C2 a[kLanesPerStep];
    uint32_t tb = pc >= 0 ? (1u << pc) : 0u;
#pragma unroll
    for (int b = 0; b < 8; ++b) tb |= ((tid >> b) & 1u) << ((plan >> (4 * b)) & 15);
#pragma unroll
    for (int b = 0; b < 4; ++b)  // round bits follow the per-thread bits
        if (8 + kChainQBits + b < 12 - (pc >= 0 ? 1 : 0)) tb |= ((round >> b) & 1u) << ((plan >> (4 * (8 + kChainQBits + b))) & 15);
    uint32_t qo[kChainQBits];
#pragma unroll
    for (int b = 0; b < kChainQBits; ++b) qo[b] = 1u << ((plan >> (4 * (8 + b))) & 15);
    uint32_t any = 0, all = ~0u;
#pragma unroll
    for (int q = 0; q < kLanesPerStep; ++q) {
        uint32_t p = tb;
#pragma unroll
        for (int b = 0; b < kChainQBits; ++b)
            if ((q >> b) & 1) p |= qo[b];
        pos[q] = p;
        sb[q] = (xlo | lut_lo[p & 63] | lut_hi[p >> 6]) & R;
        any |= sb[q];
        all &= sb[q];
    }
#pragma unroll
    for (int q = 0; q < kLanesPerStep; ++q) {
        const double2 v = tile_s[pos[q]];
        a[q] = C2{v.x, v.y};
        // an exact zero stays zero under any phase (the product is +-0,
        // which the codec stores as zero): no walk for it
        if (v.x == 0.0 && v.y == 0.0) sb[q] = 0;
    }
    any = 0;
    all = ~0u;
#pragma unroll
    for (int q = 0; q < kLanesPerStep; ++q) {
        any |= sb[q];
        all &= sb[q];
    }
    // Walk the union of the eight masks in program order; bits set in all
    // eight multiply unconditionally (independent products, full ILP), the
    // others under each amplitude's own bit. One bit scan and one phase load
    // serve all eight amplitudes.
    uint32_t rem = any;
    while (rem) {
        const int r = next_bit<kDesc>(rem);
        rem &= ~(1u << r);
        const double2 u = tab[r];
        if ((all >> r) & 1u) {
#pragma unroll
            for (int q = 0; q < kLanesPerStep; ++q) a[q] = cmul(u.x, u.y, a[q]);
        } else {
#pragma unroll
            for (int q = 0; q < kLanesPerStep; ++q)
                if ((sb[q] >> r) & 1u) a[q] = cmul(u.x, u.y, a[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < kLanesPerStep; ++q)
        if (sb[q]) tile_s[pos[q]] = make_double2(a[q].re, a[q].im);  // untouched amplitudes stay as they are
}

// Lazy CX on the affine part of a tile's index map (see FastOp).
__device__ __forceinline__ uint32_t cx_update(const FastOp& g, uint32_t cvec, uint64_t base) {
    const uint32_t ctl = g.in_hi ? (cvec >> g.tp_hi) & 1u : static_cast<uint32_t>((base >> g.hi) & 1);
    return cvec ^ (ctl << g.tp_lo);
}

// Diagonal ops [q0, q1) on the amplitude at physical tile position k (x:
// its buffer index). DIAG / CDIAG read logical bits through the pass's lazy
// CX map (FastOp::mrow, cvec); phase chains only run where the map is the
// identity (lazify), so they use x directly.
__device__ __forceinline__ C2 apply_diag_run(const FastOp* ops, const double2* stab, uint32_t q0, uint32_t q1,
                                             uint64_t x, C2 a, uint32_t cvec, uint32_t k) {
    const auto bit = [&](bool in, uint16_t row, uint8_t tp, uint8_t b) -> uint32_t {
        return in ? ((__popc(row & k) ^ (cvec >> tp)) & 1u) : static_cast<uint32_t>((x >> b) & 1);
    };
    for (uint32_t q = q0; q < q1; ++q) {
        const FastOp& o = ops[q];
        if (o.type == OP_CX) {  // (chain-free runs only: the map's affine part moves on)
            cvec = cx_update(o, cvec, x);
            continue;
        }
        if (o.type == OP_CHAIN) {
            if (!((x >> o.hi) & 1)) continue;
            uint32_t R;
            memcpy(&R, &o.m[0], 4);
            a = chain_walk(static_cast<uint32_t>(x) & R, o.et[0] != 0, stab + o.pad2, a);
        } else if (o.type == OP_CDIAG) {
            if (bit(o.in_hi, o.mrow, o.tp_hi, o.hi) & bit(o.in_lo, o.mrow2, o.tp_lo, o.lo) && o.et[0] != ET_ONE)
                a = entry_mul(o.et[0], o.m[0], o.m[1], a);
        } else {  // OP_DIAG
            const int e = static_cast<int>(bit(o.in_hi, o.mrow, o.tp_hi, o.hi));
            if (o.et[e] != ET_ONE) a = entry_mul(o.et[e], o.m[2 * e], o.m[2 * e + 1], a);
        }
    }
    return a;
}

__device__ __forceinline__ bool is_diag(uint8_t t) { return t == OP_DIAG || t == OP_CDIAG || t == OP_CHAIN; }

__device__ __forceinline__ bool has_chain(const FastOp* ops, uint32_t q0, uint32_t q1) {
    for (uint32_t q = q0; q < q1; ++q)
        if (ops[q].type == OP_CHAIN) return true;
    return false;
}

// Quantisation epilogue: amplitudes j of this thread -> packed words and
// per-chunk counters. Lanes of a warp hold 32 consecutive locals (tile
// positions 0..4 are buffer bits 0..4), so (block slot, chunk) is
// warp-uniform: each thread keeps RowAcc counters for the current chunk and
// the warp reduces them with REDUX when the chunk changes (rows in jnew).
template <bool kF32>
__device__ __forceinline__ void quant_rows(const QuantOut& q, const double2* tile_s, uint32_t tid, uint64_t pbt,
                                           const uint64_t* pjoff, uint32_t jnew, uint32_t lb, bool gather,
                                           uint32_t cvec, const uint16_t* gat_lo, const uint16_t* gat_hi) {
    // pbt: planar index of (tile base | thread offset); pjoff[j]: of row j
    const uint64_t im_off = 1ull << lb;
    const double qlo_d = static_cast<double>(q.t.qlo);
    const int span = static_cast<int>(q.t.qhi - q.t.qlo);
    uint32_t* const pk = q.pk + pbt;
    RowAcc acc_re, acc_im;
    // chunks are 4096 scalars and 2^(lb+1) / 4096 = nch per block (lb >= 12),
    // so the chunk of a scalar is its planar index >> 12; the bits of pbt and
    // pjoff[j] are disjoint, so row j's chunk is (pbt >> 12) | (pjoff[j] >> 12)
    // and it changes only at the rows set in jnew (the same for every tile)
    const uint64_t kb = pbt >> 12, kim = im_off >> 12;
    uint64_t key = kb | (pjoff[0] >> 12);
    uint32_t rows = 0;
    bool bad = false, oow = false;
#pragma unroll 1
    for (int j = 0; j < kPer; ++j) {
        uint32_t y = tid + 256 * j;
        if (gather) y = gat_lo[(y ^ cvec) & 63] ^ gat_hi[(y ^ cvec) >> 6];
        const double2 a = tile_s[y];
        uint32_t pr, pi;
        if constexpr (kF32) {
            pr = quantize_pack_f32(a.x, q.t, span, bad, oow);
            pi = quantize_pack_f32(a.y, q.t, span, bad, oow);
        } else {
            pr = quantize_pack_fast(a.x, q.t, qlo_d, span, bad, oow);
            pi = quantize_pack_fast(a.y, q.t, qlo_d, span, bad, oow);
        }
        const uint64_t o = pjoff[j];
        if ((jnew >> j) & 1u) {  // warp-uniform
            flush_rows(q.cps + key, acc_re, 32u * rows);
            flush_rows(q.cps + key + kim, acc_im, 32u * rows);
            acc_re = RowAcc{};
            acc_im = RowAcc{};
            rows = 0;
            key = kb | (o >> 12);
        }
        pk[o] = pr;
        pk[o + im_off] = pi;
        acc_re.add(pr);
        acc_im.add(pi);
        ++rows;
    }
    flush_rows(q.cps + key, acc_re, 32u * rows);
    flush_rows(q.cps + key + kim, acc_im, 32u * rows);
    if (bad) dev_fail(q.err, DE_NONFINITE, 0);
    if (oow) dev_fail(q.err, DE_WINDOW, 0);
}

__device__ __forceinline__ void quant_epilogue(const QuantOut& q, const double2* tile_s, uint32_t tid, uint64_t pbt,
                                               const uint64_t* pjoff, uint32_t jnew, uint32_t lb, bool gather,
                                               uint32_t cvec, const uint16_t* gat_lo, const uint16_t* gat_hi) {
    if (q.t.f32)
        quant_rows<true>(q, tile_s, tid, pbt, pjoff, jnew, lb, gather, cvec, gat_lo, gat_hi);
    else
        quant_rows<false>(q, tile_s, tid, pbt, pjoff, jnew, lb, gather, cvec, gat_lo, gat_hi);
}

__global__ void __launch_bounds__(kFastThreads, 3) k_gate_pass_fast(double* __restrict__ buf, uint32_t lb,
                                                                 int interleaved, uint64_t ntiles,
                                                                 const __grid_constant__ FastPass pass,
                                                                 const __grid_constant__ QuantOut quant,
                                                                 const uint32_t* __restrict__ vtab,
                                                                 int dbg_full_support,
                                                                 uint8_t* __restrict__ wf, uint32_t* wz) {
    // dynamic SMEM: 4096 amplitudes (tile position k) | chain tables | ops
    extern __shared__ double2 tile_s[];
    __shared__ uint64_t joff[kPer];
    __shared__ uint64_t pjoff[kPer];             // planar index of joff[j] (planar_addr is OR-linear)
    __shared__ uint32_t lut_lo[64], lut_hi[64];  // tile position -> buffer bits (low 32)
    __shared__ uint16_t gat_lo[64], gat_hi[64];  // final M^-1 on a 12-bit tile index (lazy CX)
    double2* stab = tile_s + 4096;
    FastOp* sops = reinterpret_cast<FastOp*>(stab + pass.tab_entries);
    const uint32_t tid = threadIdx.x;
    const uint64_t lmask = (1ull << lb) - 1;
    const uint64_t im_off = interleaved ? 1 : (1ull << lb);
    const uint64_t toff = runs_deposit(tid, pass.tile);
    const uint64_t ptoff = planar_addr(toff, lb, lmask, interleaved);
    if (tid < kPer) {
        joff[tid] = runs_deposit(static_cast<uint64_t>(tid) << 8, pass.tile);
        pjoff[tid] = planar_addr(joff[tid], lb, lmask, interleaved);
    }
    if (tid < 64) lut_lo[tid] = static_cast<uint32_t>(runs_deposit(tid, pass.tile));
    else if (tid < 128) lut_hi[tid - 64] = static_cast<uint32_t>(runs_deposit(static_cast<uint64_t>(tid - 64) << 6, pass.tile));
    else if (tid < 256) {
        const uint32_t v = tid & 63, sh = tid < 192 ? 0 : 6;
        uint32_t x = 0;
        for (uint32_t b = 0; b < 6; ++b)
            if ((v >> b) & 1) x ^= pass.minv[b + sh];
        (tid < 192 ? gat_lo : gat_hi)[v] = static_cast<uint16_t>(x);
    }
    for (uint32_t e = tid; e < pass.tab_entries; e += kFastThreads)
        stab[e] = __ldg(reinterpret_cast<const double2*>(pass.chain_tab) + pass.tab_base + e);
    {
        const uint32_t* src = reinterpret_cast<const uint32_t*>(pass.ops);
        uint32_t* dst = reinterpret_cast<uint32_t*>(sops);
        const uint32_t words = pass.nops * static_cast<uint32_t>(sizeof(FastOp) / 4);
        for (uint32_t e = tid; e < words; e += kFastThreads) dst[e] = src[e];
    }
    __shared__ uint32_t s_supp[2];
    if (tid < 2) s_supp[tid] = 0;
    // *wz == 0: no group of the buffer is flagged zero (every flag is 1), so
    // loads need not test flags; a pass that flags a group zero sets it
    const bool wf_read = wf && *reinterpret_cast<volatile uint32_t*>(wz) != 0;
    bool set_wz = false;  // this thread flagged a group zero (one store per CTA at the end)
    __syncthreads();
    // rows j > 0 whose chunk differs from row j - 1's (quant epilogue)
    uint32_t jnew = 0;
    for (int j = 1; j < kPer; ++j)
        if ((pjoff[j] >> 12) != (pjoff[j - 1] >> 12)) jnew |= 1u << j;
    __syncthreads();
    // Sweeps are the same for every tile: a run of diagonal ops, extended
    // over CX / DIAG / CDIAG when it holds no phase chain (lazy CX).
    if (tid < pass.nops && is_diag(sops[tid].type)) {
        uint32_t i2 = tid + 1;
        while (i2 < pass.nops && is_diag(sops[i2].type)) ++i2;
        const bool chain = has_chain(sops, tid, i2);
        if (!chain)
            while (i2 < pass.nops && (sops[i2].type == OP_CX || sops[i2].type == OP_DIAG || sops[i2].type == OP_CDIAG))
                ++i2;
        sops[tid].run = static_cast<uint16_t>(i2 | (chain ? 0x8000u : 0u));
    }
    __syncthreads();
    uint32_t parity = 0;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, parity ^= 1) {
        const uint64_t base = runs_deposit(tile, pass.base);
        const uint64_t pbt = planar_addr(base, lb, lmask, interleaved) + ptoff;  // planar index of base | toff
        // Index used by diagonal conditions. Block-wise batches (vtab) hold
        // single blocks of a diagonal stage: the bits above lb are the
        // block's inner value, not its slot in the batch.
        const uint64_t xbase = vtab ? ((static_cast<uint64_t>(vtab[base >> lb]) << lb) | (base & lmask)) : base;
        // Group flags of the warp's 32 groups (lane 2j + c: scalar c of row j).
        uint32_t fl = 1;
        if (wf_read) {
            const uint32_t lane = tid & 31;
            const uint64_t a = pbt + pjoff[lane >> 1];
            fl = wf[(a + ((lane & 1) ? im_off : 0)) >> 5];
        }
        // Barrier: the previous tile's stores have read tile_s.
        const int any_group = __syncthreads_or(fl);
        if (tid == 0) s_supp[parity ^ 1] = 0;  // the next tile's slot (last read two tiles ago)
        // All groups flagged zero: the tile stays zero in place (flags stay 0).
        if (!any_group && !quant.pk) continue;
        {
            double re[kPer], im[kPer];
            uint32_t nzpos = 0;
            const uint32_t fmask = __ballot_sync(0xffffffffu, fl != 0);  // bit 2j + c: group (row j, part c) stored
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const uint64_t a = pbt + pjoff[j];
                if (wf_read) {  // 32-scalar groups flagged zero were not stored (warp-uniform test)
                    re[j] = ((fmask >> (2 * j)) & 1u) ? buf[a] : 0.0;
                    im[j] = ((fmask >> (2 * j + 1)) & 1u) ? buf[a + im_off] : 0.0;
                    continue;
                }
                re[j] = buf[a];
                im[j] = buf[a + im_off];
            }
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                tile_s[tid + 256 * j] = make_double2(re[j], im[j]);
                if (re[j] != 0.0 || im[j] != 0.0) nzpos |= 0x80000000u | (tid + 256u * j);  // bit 31: some nonzero
            }
            nzpos = __reduce_or_sync(0xffffffffu, nzpos);
            if ((tid & 31) == 0 && nzpos) atomicOr(&s_supp[parity], nzpos);
        }
        __syncthreads();
        // Support: every nonzero amplitude of the tile sits at a position
        // inside S (x & ~S == 0). Diagonal gates keep S, a mixing gate adds
        // its partner offset; ops below only visit positions inside S (a zero
        // stays zero under every gate, up to the sign the codec ignores).
        uint32_t S = dbg_full_support ? 0x80000fffu : s_supp[parity];  // bit 31 set unless the tile is all zero
        if (S == 0 && wf && !quant.pk) {  // an all-zero tile stays zero: flag its groups, store nothing
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const uint64_t a = pbt + pjoff[j];
                if ((tid & 31) == 0) {
                    wf[a >> 5] = 0;
                    wf[(a + im_off) >> 5] = 0;
                    set_wz = true;
                }
            }
            continue;
        }
        // barrier scope owed by the ops since the last barrier: 0 = every
        // thread touched only its own positions (tid + 256 j), 1 = positions
        // of its warp, 2 = any position of the tile
        uint32_t scope = 0;
        uint32_t cvec = 0;  // lazy CX: affine part of the tile's index map
        for (uint32_t i = 0; i < pass.nops;) {
            const FastOp& g = sops[i];
            if (g.type == OP_CX) {  // no data moves: only the map changes
                cvec = cx_update(g, cvec, base);
                ++i;
                continue;
            }
            if (g.type == OP_PERM) {  // materialise: logical y takes the amplitude at M^-1 (y ^ c)
                uint16_t cols[kMaxTileBits];
                memcpy(cols, &g.m[0], sizeof cols);
                __syncthreads();
                double2 v[kPer];
#pragma unroll
                for (int j = 0; j < kPer; ++j) {
                    const uint32_t y = (tid + 256u * j) ^ cvec;
                    uint32_t x = 0;
                    for (uint32_t b = 0; b < kMaxTileBits; ++b)
                        if ((y >> b) & 1) x ^= cols[b];
                    v[j] = tile_s[x];
                }
                __syncthreads();
#pragma unroll
                for (int j = 0; j < kPer; ++j) tile_s[tid + 256u * j] = v[j];
                cvec = 0;
                if (S) S = 0x80000fffu;  // (conservative: the map moved the support)
                scope = 0;
                ++i;
                continue;
            }
            if (is_diag(g.type)) {
                // a chain-free run also absorbs CX ops (lazy: they only change
                // the index map), so CX-RZ-CX sequences are one sweep
                const uint32_t i2 = g.run & 0x7fffu;
                const bool run_chain = (g.run & 0x8000u) != 0;
                const uint32_t cvec_in = cvec;  // the map's affine part at the start of the run
                for (uint32_t q = i; q < i2; ++q)
                    if (sops[q].type == OP_CX) cvec = cx_update(sops[q], cvec, base);
                if (!run_chain && S != 0) {
                    // a chain-free run is the identity on this tile when each op's
                    // entry is 1 for every value its condition bits take on the
                    // support (an in-tile logical bit is constant when its row of
                    // M misses S; an outer bit is the tile base's)
                    const uint32_t Sp = S & 0xfffu;
                    bool act = false;
                    uint32_t cv = cvec_in;
                    const auto vals = [&](uint8_t in, uint16_t row, uint8_t tp, uint8_t b) -> uint32_t {
                        if (!in) return ((xbase >> b) & 1) ? 2u : 1u;  // bit 0: can be 0, bit 1: can be 1
                        if (row & Sp) return 3u;
                        return ((cv >> tp) & 1u) ? 2u : 1u;
                    };
                    for (uint32_t q = i; q < i2 && !act; ++q) {
                        const FastOp& o = sops[q];
                        if (o.type == OP_CX) {
                            cv = cx_update(o, cv, base);
                            continue;
                        }
                        const uint32_t vh = vals(o.in_hi, o.mrow, o.tp_hi, o.hi);
                        if (o.type == OP_DIAG)
                            act = ((vh & 1u) && o.et[0] != ET_ONE) || ((vh & 2u) && o.et[1] != ET_ONE);
                        else
                            act = (vh & 2u) && (vals(o.in_lo, o.mrow2, o.tp_lo, o.lo) & 2u) && o.et[0] != ET_ONE;
                    }
                    if (!act) {
                        i = i2;
                        continue;
                    }
                }
                if (run_chain && i2 == i + 1 && g.type == OP_CHAIN && S != 0) {
                    // a lone chain with nothing to act on (see below): no sweep, no barrier
                    uint32_t R;
                    memcpy(&R, &g.m[0], 4);
                    const uint32_t rs = (static_cast<uint32_t>(xbase) | lut_lo[S & 63u] | lut_hi[(S >> 6) & 63u]) & R;
                    if (!(rs && (g.in_hi ? ((S >> g.tp_hi) & 1) : ((xbase >> g.hi) & 1)))) {
                        i = i2;
                        continue;
                    }
                }
                if (scope == 2) __syncthreads();
                else if (scope == 1) __syncwarp();
                scope = 0;
                if (S == 0) {  // an all-zero tile: nothing to do
                    i = i2;
                    continue;
                }
                const uint32_t Sp = S & 0xfffu;  // positions
                const bool lone_chain = i2 == i + 1 && g.type == OP_CHAIN;
                if (!lone_chain && __popc(Sp) < 11) {  // sparse tile: only the 2^|S| positions of the support
                    __syncthreads();
                    const uint32_t np = 1u << __popc(Sp);
                    for (uint32_t r = tid; r < np; r += kFastThreads) {
                        const uint32_t k = deposit12(r, Sp);
                        const double2 v = tile_s[k];
                        const uint64_t xb = xbase | lut_lo[k & 63] | lut_hi[k >> 6];
                        const C2 o = apply_diag_run(sops, stab, i, i2, xb, C2{v.x, v.y}, cvec_in, k);
                        tile_s[k] = make_double2(o.re, o.im);
                    }
                    scope = 2;
                    i = i2;
                    continue;
                }
                if (lone_chain) {  // a lone phase chain: parameters in registers
                    uint32_t R;
                    uint64_t plan;
                    memcpy(&R, &g.m[0], 4);
                    memcpy(&plan, &g.m[1], 8);
                    const bool desc = g.et[0] != 0;
                    const double2* tab = stab + g.pad2;
                    const int pc = g.in_hi ? g.tp_hi : -1;
                    const uint32_t xlo = static_cast<uint32_t>(xbase);
                    // support: no nonzero amplitude with bit c, or none with a bit of R
                    const uint32_t rs = (xlo | lut_lo[S & 63u] | lut_hi[(S >> 6) & 63u]) & R;
                    const bool active = rs && (pc >= 0 ? ((S >> pc) & 1) : ((xbase >> g.hi) & 1));
                    if (active && __popc(S & 0xfffu) < 11) {  // sparse tile: the support positions with bit c
                        __syncthreads();
                        const uint32_t Sp = S & 0xfffu;
                        const uint32_t cm = pc >= 0 ? (Sp & ~(1u << pc)) : Sp, cb = pc >= 0 ? (1u << pc) : 0u;
                        const uint32_t np = 1u << __popc(cm);
                        for (uint32_t r = tid; r < np; r += kFastThreads) {
                            const uint32_t k = deposit12(r, cm) | cb;
                            const double2 v = tile_s[k];
                            const uint32_t x = xlo | lut_lo[k & 63] | lut_hi[k >> 6];
                            const C2 o = chain_walk(x & R, desc, tab, C2{v.x, v.y});
                            tile_s[k] = make_double2(o.re, o.im);
                        }
                        scope = 2;
                    } else if (active) {
                        __syncthreads();  // positions cross thread ownership
                        const uint32_t rounds = (pc >= 0 ? 2048u : 4096u) / (256u * kLanesPerStep);
                        for (uint32_t rd = 0; rd < rounds; ++rd) {
                            if (desc)
                                chain_walk8<true>(tile_s, tab, tid, xlo, lut_lo, lut_hi, pc, R, plan, rd);
                            else
                                chain_walk8<false>(tile_s, tab, tid, xlo, lut_lo, lut_hi, pc, R, plan, rd);
                        }
                        scope = 2;
                    }
                } else if (!run_chain) {
                    // plain diagonal gates: op by op, each a branch-free
                    // product with the entry its amplitude selects (an entry 1
                    // multiplies exactly: 1*x - 0*y == x up to a zero's sign)
                    for (int h = 0; h < kPer; h += 8) {  // eight amplitudes in registers at a time
                        C2 a[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const double2 v = tile_s[tid + 256u * (h + j)];
                            a[j] = C2{v.x, v.y};
                        }
                        uint32_t cv = cvec_in;
                        for (uint32_t q = i; q < i2; ++q) {
                            const FastOp& o = sops[q];
                            if (o.type == OP_CX) {
                                cv = cx_update(o, cv, base);
                                continue;
                            }
                            const bool cd = o.type == OP_CDIAG;
                            const double r0 = cd ? 1.0 : o.m[0], i0 = cd ? 0.0 : o.m[1];
                            const double r1 = cd ? o.m[0] : o.m[2], i1 = cd ? o.m[1] : o.m[3];
                            // logical bit = parity(row of M & physical position) ^ c (in the
                            // tile) or the base bit; a missing second bit reads as 1
                            const uint32_t rh = o.in_hi ? o.mrow : 0u, rl = cd && o.in_lo ? o.mrow2 : 0u;
                            const uint32_t ch = o.in_hi ? (cv >> o.tp_hi) & 1u : static_cast<uint32_t>((xbase >> o.hi) & 1);
                            const uint32_t cl = !cd ? 1u
                                                    : (o.in_lo ? (cv >> o.tp_lo) & 1u
                                                               : static_cast<uint32_t>((xbase >> o.lo) & 1));
                            // bit j of `on`: amplitude k = tid + 256 j takes entry u1. A
                            // row's parity over k splits into the thread's bits (tid)
                            // and the row index j (kParMask), so the per-amplitude
                            // test is one bit of a per-op mask
                            const uint32_t ph = (__popc(rh & tid) ^ ch) & 1u, pl = (__popc(rl & tid) ^ cl) & 1u;
                            const uint32_t on = ((kParMask[(rh >> 8) & 15u] ^ (0u - ph)) &
                                                 (kParMask[(rl >> 8) & 15u] ^ (0u - pl))) >> h;
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const bool b = (on >> j) & 1u;
                                a[j] = cmul(b ? r1 : r0, b ? i1 : i0, a[j]);
                            }
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j) tile_s[tid + 256u * (h + j)] = make_double2(a[j].re, a[j].im);
                    }
                } else {
                    for (int j = 0; j < kPer; ++j) {
                        const uint32_t k = tid + 256u * j;
                        const double2 v = tile_s[k];
                        const C2 r = apply_diag_run(sops, stab, i, i2, xbase | toff | joff[j], C2{v.x, v.y}, cvec_in, k);
                        tile_s[k] = make_double2(r.re, r.im);
                    }
                }
                i = i2;
                continue;
            }
            ++i;
            if (S == 0) continue;  // zeros map to zeros (tile-uniform)
            // U2 on logical tile bit t: physical pairs (x, x ^ dvec); x is
            // the |0> side when parity(mrow & x) ^ c_t is 0
            const uint32_t dv = g.dvec, piv = __ffs(dv) - 1, ct = (cvec >> g.tp_hi) & 1u;
            const uint32_t S2 = (S | dv) & 0xfffu;
            const bool dense = __popc(S2) == 12;  // (11 support bits: 1024 pairs, none all-zero by construction)
            const uint32_t npairs = dense ? 2048u : (1u << (__popc(S2) - 1)), pm = S2 & ~(1u << piv);
            S = S2 | 0x80000000u;
            // Dense sweeps pair positions inside the smallest owner set that
            // holds both partners: a thread's own 16 positions (dvec in tile
            // bits 8..11), its warp's 512 (bits 0..4 and 8..11), else the
            // tile; the barrier before the sweep only spans that set and what
            // earlier ops touched since the last one.
            const uint32_t lvl = !dense ? 2u : (!(dv & 0xffu) ? 0u : (!(dv & 0xe0u) ? 1u : 2u));
            const uint32_t need = scope > lvl ? scope : lvl;
            if (need == 2) __syncthreads();
            else if (need == 1) __syncwarp();
            scope = lvl;
            const uint32_t lane = tid & 31u, wbase = tid & ~31u;
            // (op fields are read into registers once: tile_s stores could alias sops)
            const uint32_t mrow = g.mrow;
            // visit every pair of this thread: sparse, tile-, warp- or thread-local enumeration
            const auto sweep = [&](auto&& body) {
                if (!dense) {
                    for (uint32_t r = tid; r < npairs; r += kFastThreads) body(deposit12(r, pm));
                } else if (lvl == 2) {
#pragma unroll 2
                    for (uint32_t m = 0; m < 8; ++m) body(insert0(tid + kFastThreads * m, piv));
                } else if (lvl == 1) {  // warp-local index: bits 0..4 lanes, 5..8 rows (tile bits 8..11)
#pragma unroll 2
                    for (uint32_t m = 0; m < 8; ++m) {
                        const uint32_t u = insert0(lane + 32u * m, piv);
                        body((u & 31u) | wbase | ((u >> 5) << 8));
                    }
                } else {
#pragma unroll 2
                    for (uint32_t m = 0; m < 8; ++m) body(tid + 256u * insert0(m, piv - 8));
                }
            };
            if (g.pad == 1) {  // all entries real: u*a = (u*ar, u*ai) exactly
                const double u00 = g.m[0], u01 = g.m[2], u10 = g.m[4], u11 = g.m[6];
                sweep([&](uint32_t x0) {
                    const uint32_t x1 = x0 ^ dv;
                    const bool sw = (__popc(mrow & x0) ^ ct) & 1u;
                    const uint32_t i0 = sw ? x1 : x0, i1 = sw ? x0 : x1;
                    const double2 v0 = tile_s[i0], v1 = tile_s[i1];
                    // a pair of exact zeros maps to zeros (+-0 for the codec); only
                    // worth testing in full sweeps, where S may be a loose superset
                    if (dense && v0.x == 0.0 && v0.y == 0.0 && v1.x == 0.0 && v1.y == 0.0) return;
                    tile_s[i0] = make_double2(__dadd_rn(__dmul_rn(u00, v0.x), __dmul_rn(u01, v1.x)),
                                              __dadd_rn(__dmul_rn(u00, v0.y), __dmul_rn(u01, v1.y)));
                    tile_s[i1] = make_double2(__dadd_rn(__dmul_rn(u10, v0.x), __dmul_rn(u11, v1.x)),
                                              __dadd_rn(__dmul_rn(u10, v0.y), __dmul_rn(u11, v1.y)));
                });
            } else if (g.pad == 2) {  // u00, u11 real, u01, u10 imaginary (RX): row2's products, fixed classes
                const double u00 = g.m[0], u01i = g.m[3], u10i = g.m[5], u11 = g.m[6];
                sweep([&](uint32_t x0) {
                    const uint32_t x1 = x0 ^ dv;
                    const bool sw = (__popc(mrow & x0) ^ ct) & 1u;
                    const uint32_t i0 = sw ? x1 : x0, i1 = sw ? x0 : x1;
                    const double2 v0 = tile_s[i0], v1 = tile_s[i1];
                    if (dense && v0.x == 0.0 && v0.y == 0.0 && v1.x == 0.0 && v1.y == 0.0) return;
                    tile_s[i0] = make_double2(__dadd_rn(__dmul_rn(u00, v0.x), -__dmul_rn(u01i, v1.y)),
                                              __dadd_rn(__dmul_rn(u00, v0.y), __dmul_rn(u01i, v1.x)));
                    tile_s[i1] = make_double2(__dadd_rn(-__dmul_rn(u10i, v0.y), __dmul_rn(u11, v1.x)),
                                              __dadd_rn(__dmul_rn(u10i, v0.x), __dmul_rn(u11, v1.y)));
                });
            } else {
                uint8_t et[4];
                double m[8];
                memcpy(et, g.et, sizeof et);
                memcpy(m, g.m, sizeof m);
                sweep([&](uint32_t x0) {
                    const uint32_t x1 = x0 ^ dv;
                    const bool sw = (__popc(mrow & x0) ^ ct) & 1u;
                    const uint32_t i0 = sw ? x1 : x0, i1 = sw ? x0 : x1;
                    const double2 v0 = tile_s[i0], v1 = tile_s[i1];
                    if (v0.x == 0.0 && v0.y == 0.0 && v1.x == 0.0 && v1.y == 0.0) return;
                    const C2 a0{v0.x, v0.y}, a1{v1.x, v1.y};
                    const C2 o0 = row2(et, m, 0, a0, a1), o1 = row2(et, m, 1, a0, a1);
                    tile_s[i0] = make_double2(o0.re, o0.im);
                    tile_s[i1] = make_double2(o1.re, o1.im);
                });
            }
        }
        const bool gather = pass.final_perm || cvec;  // logical y lives at M^-1 (y ^ c)
        if (scope == 2 || gather) __syncthreads();
        else if (scope == 1) __syncwarp();
        if (quant.pk) {
            quant_epilogue(quant, tile_s, tid, pbt, pjoff, jnew, lb, gather, cvec, gat_lo, gat_hi);
            continue;
        }
        {
            double re[kPer], im[kPer];
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                uint32_t y = tid + 256 * j;
                if (gather) y = gat_lo[(y ^ cvec) & 63] ^ gat_hi[(y ^ cvec) >> 6];
                const double2 v = tile_s[y];
                re[j] = v.x;
                im[j] = v.y;
            }
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const uint64_t a = pbt + pjoff[j];
                if (wf) {  // an all-zero 32-scalar group is flagged instead of stored
                    const bool nr = __any_sync(0xffffffffu, re[j] != 0.0), ni = __any_sync(0xffffffffu, im[j] != 0.0);
                    if ((threadIdx.x & 31) == 0) {
                        wf[a >> 5] = nr;
                        wf[(a + im_off) >> 5] = ni;
                        if (!(nr && ni)) set_wz = true;
                    }
                    if (nr) buf[a] = re[j];
                    if (ni) buf[a + im_off] = im[j];
                    continue;
                }
                buf[a] = re[j];
                buf[a + im_off] = im[j];
            }
        }
    }
    if (wf && __syncthreads_or(set_wz) && tid == 0) *wz = 1;
}

// ------------------------------------------------ register-streaming pass
// See StreamPass (gates.cuh). Lane l, value r of unit u holds buffer index
// base(u) | l | dep(r); ops run in program order on registers with the
// tiled kernel's arithmetic (cmul / row2: the reference's products, exact
// up to the sign of an exact zero, which the codec never stores).
constexpr int kStreamThreads = 256;
constexpr int kNV = 1 << kStreamNQ;

__device__ __forceinline__ C2 shfl_c2(C2 a, uint32_t m) {
    return C2{__shfl_xor_sync(0xffffffffu, a.re, m), __shfl_xor_sync(0xffffffffu, a.im, m)};
}

// kSame: every register row of a unit lies in the unit's 4096-scalar chunk
// (the register bits are below bit 12), so one accumulator pair serves them.
// kRound (stage fusion): the quantised scalars are stored back as their
// dequantised values (QuantOut::rnd) instead of code words.
template <bool kQuant, bool kDecode, bool kSame = false, bool kRound = false>
__global__ void __launch_bounds__(kStreamThreads, kQuant ? 2 : 3) k_stream_pass(double* __restrict__ buf, uint32_t lb, uint64_t nunits,
                                                                const __grid_constant__ StreamPass pass,
                                                                const __grid_constant__ QuantOut q,
                                                                const uint32_t* __restrict__ vtab,
                                                                uint8_t* __restrict__ wf, uint32_t* wz,
                                                                const __grid_constant__ FusedDecode dec) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * kStreamThreads + threadIdx.x) >> 5;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * kStreamThreads) >> 5;
    // a contiguous range of units per warp: consecutive units mostly share
    // their chunks, so the epilogue's counters flush once per run
    const uint64_t per = (nunits + nwarps - 1) / nwarps;
    const uint64_t u0 = warp * per, u1 = min(nunits, u0 + per);
    if (u0 >= u1) return;
    const uint64_t lmask = (1ull << lb) - 1, im_off = 1ull << lb;
    uint64_t pdep[kNV];  // planar offsets of the register rows (planar_addr is OR-linear)
#pragma unroll
    for (int r = 0; r < kNV; ++r) {
        uint64_t d = 0;
#pragma unroll
        for (int i = 0; i < kStreamNQ; ++i) d |= static_cast<uint64_t>((r >> i) & 1) << pass.qbit[i];
        pdep[r] = planar_addr(d, lb, lmask, 0);
    }
    // *wz == 0: every 32-scalar group of the input is stored (flags all 1)
    const bool wf_read = wf && *reinterpret_cast<volatile uint32_t*>(wz) != 0;
    bool set_wz = false;
    bool bad = false, oow = false;
    const int span = static_cast<int>(q.t.qhi - q.t.qlo);
    const double qlo_d = static_cast<double>(q.t.qlo);
    // Per-chunk counters of the current run, reduced per row with REDUX as it
    // is quantised: warp-uniform values (uniform registers, not 24 per-lane
    // ones), fields as RowAcc's.
    constexpr int kAcc = kSame ? 1 : kNV;
    uint32_t amn[kAcc][2], amx[kAcc][2], azn[kAcc][2];
#pragma unroll
    for (int r = 0; r < kAcc; ++r)
#pragma unroll
        for (int h = 0; h < 2; ++h) amn[r][h] = ~0u, amx[r][h] = 0u, azn[r][h] = 0u;
    uint64_t run_pb = 0;  // planar base of the current counter run
    uint32_t run_len = 0;
    const auto flush = [&]() {
#pragma unroll
        for (int r = 0; r < kAcc; ++r) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                ChunkPlan* cp = q.cps + (((run_pb | pdep[r]) >> 12) + (h ? (im_off >> 12) : 0));
                const uint32_t nnz = 32u * (kNV / kAcc) * run_len - (azn[r][h] & 0xffffu), nneg = azn[r][h] >> 16;
                if (lane == 0 && nnz) atomicMax(&cp->qmin_inv, kQOffMax - (amn[r][h] >> 2));
                if (lane == 1 && nnz) atomicMax(&cp->qmax_off, amx[r][h] >> 2);
                if (lane == 2 && nnz) atomicAdd(&cp->nnz, nnz);
                if (lane == 3 && nneg) atomicAdd(&cp->nneg, nneg);
                amn[r][h] = ~0u;
                amx[r][h] = 0u;
                azn[r][h] = 0u;
            }
        }
        run_len = 0;
    };
    // one unit's values in flight ahead of the one being processed; returns
    // true when every row of the unit is zero (nothing was loaded)
    constexpr bool decode = kDecode;
    const int dspan = static_cast<int>(dec.qhi - dec.qlo);
    bool dbad = false;
    const uint32_t lt = (1u << lane) - 1;
    // one 32-scalar row straight from its payload (decompress_block,
    // codec.hpp:333-342): rank of this lane's code from the row record
    const auto decode_row = [&](uint64_t p, bool& any) -> double {
        const DecRow rec = dec.rows[p >> 5];
        if (!rec.nz) return 0.0;  // warp-uniform
        any = true;
        const uint64_t slot = p >> (lb + 1);
        const uint8_t* codes = dec.blks[slot].in;
        const DecInfo& di = dec.infos[slot];
        const uint32_t width = di.width;
        const uintptr_t cs = reinterpret_cast<uintptr_t>(codes + di.code_seg);
        const uint32_t* cw = reinterpret_cast<const uint32_t*>(cs & ~uintptr_t(3));
        const uint64_t bit = static_cast<uint64_t>(cs & 3) * 8 +
                             static_cast<uint64_t>(rec.rank + __popc(rec.nz & lt)) * width;
        if (!((rec.nz >> lane) & 1u)) return 0.0;
        const uint32_t code = __funnelshift_r(__ldg(cw + (bit >> 5)), __ldg(cw + (bit >> 5) + 1), bit & 31) &
                              (width >= 32 ? ~0u : (1u << width) - 1);
        const int qi = static_cast<int>(di.code_min - dec.qlo) + static_cast<int>(code);
        if (static_cast<unsigned>(qi) > static_cast<unsigned>(dspan)) {
            dbad = true;
            return 0.0;
        }
        const double m = __ldg(dec.dequant + qi);
        return ((rec.sign >> lane) & 1u) ? -m : m;
    };
    const auto load_unit = [&](uint64_t pbu, C2* v) {
        bool any = !wf_read && !decode;
#pragma unroll
        for (int r = 0; r < kNV; ++r) {
            const uint64_t p = pbu + pdep[r];
            if (decode) {
                v[r].re = decode_row(p, any);
                v[r].im = decode_row(p + im_off, any);
            } else if (wf_read) {  // rows flagged zero were not stored (warp-uniform tests)
                const bool fr = wf[p >> 5] != 0, fi = wf[(p + im_off) >> 5] != 0;
                v[r].re = fr ? __ldcs(buf + p + lane) : 0.0;
                v[r].im = fi ? __ldcs(buf + p + im_off + lane) : 0.0;
                any = any || fr || fi;
            } else {
                v[r].re = __ldcs(buf + p + lane);
                v[r].im = __ldcs(buf + p + im_off + lane);
            }
        }
        return !any;
    };
    C2 nxt[kNV];
    uint64_t nbase = runs_deposit(u0, pass.base);
    bool nzero = load_unit(planar_addr(nbase, lb, lmask, 0), nxt);
    for (uint64_t u = u0; u < u1; ++u) {
        const uint64_t base = nbase;
        const uint64_t pb = planar_addr(base, lb, lmask, 0);
        const uint64_t xb = vtab ? ((static_cast<uint64_t>(vtab[base >> lb]) << lb) | (base & lmask)) : base;
        const bool zunit = nzero;  // all zero: gates keep it zero (partners lie inside the unit)
        C2 a[kNV];
#pragma unroll
        for (int r = 0; r < kNV; ++r) a[r] = nxt[r];
        if (u + 1 < u1) {
            nbase = runs_deposit(u + 1, pass.base);
            nzero = load_unit(planar_addr(nbase, lb, lmask, 0), nxt);
        }
        if (zunit && !kQuant) {  // nothing stored: the flags say so (already, unless decoding)
            if (decode && wf && lane == 0) {
#pragma unroll
                for (int r = 0; r < kNV; ++r) {
                    wf[(pb + pdep[r]) >> 5] = 0;
                    wf[(pb + pdep[r] + im_off) >> 5] = 0;
                }
                set_wz = true;
            }
            continue;
        }
        const uint64_t xl = xb | lane;  // condition index without the register bits
        for (uint32_t i = 0; i < (zunit ? 0u : pass.nops); ++i) {
            const StreamOp& o = pass.ops[i];
            const uint32_t lp = __popcll(o.row & xl) & 1u;
            if (o.type == OP_DIAG) {
                // entries of logical bit 0 / 1 for this lane; register r takes B where rpat says so
                const double Ar = lp ? o.m[2] : o.m[0], Ai = lp ? o.m[3] : o.m[1];
                const double Br = lp ? o.m[0] : o.m[2], Bi = lp ? o.m[1] : o.m[3];
#pragma unroll
                for (int r = 0; r < kNV; ++r) {
                    if ((o.rpat >> r) & 1u)  // uniform
                        a[r] = cmul(Br, Bi, a[r]);
                    else
                        a[r] = cmul(Ar, Ai, a[r]);
                }
            } else if (o.type == OP_CDIAG) {
                const uint32_t lp2 = __popcll(o.row2 & xl) & 1u;
                const uint32_t on = (o.rpat ^ (0u - lp)) & (o.rpat2 ^ (0u - lp2));
#pragma unroll
                for (int r = 0; r < kNV; ++r)
                    if ((on >> r) & 1u) a[r] = cmul(o.m[0], o.m[1], a[r]);
            } else {  // OP_U2: partner x ^ d; this value is the |1> side where its logical bit is 1
                // partner register r ^ dq (dq uniform: one branch, constant indices,
                // so the values stay in registers)
                C2 pv[kNV];
                switch (o.dq & (kNV - 1)) {
                case 0:
#pragma unroll
                    for (int r = 0; r < kNV; ++r) pv[r] = a[r];
                    break;
                case 1:
#pragma unroll
                    for (int r = 0; r < kNV; ++r) pv[r] = a[r ^ 1];
                    break;
                case 2:
#pragma unroll
                    for (int r = 0; r < kNV; ++r) pv[r] = a[r ^ 2];
                    break;
                default:
#pragma unroll
                    for (int r = 0; r < kNV; ++r) pv[r] = a[r ^ 3];
                    break;
                }
                if (o.dl) {
#pragma unroll
                    for (int r = 0; r < kNV; ++r) pv[r] = shfl_c2(pv[r], o.dl);
                }
                const uint32_t side = o.rpat ^ (0u - lp);
                // out = u[b][b] mine + u[b][!b] partner for logical bit b of this
                // value: row 0 = u00 a0 + u01 a1, row 1 = u10 a0 + u11 a1 (the sum
                // commutes exactly). When u00, u11 and u01, u10 share their entry
                // classes (H, X, Y, RX, RY, ...) one specialised product serves
                // both rows (o.pad: 1 real / imaginary pair, see make_stream).
                if (o.pad == 1) {  // cm real, cp real
#pragma unroll
                    for (int r = 0; r < kNV; ++r) {
                        const uint32_t me = (side >> r) & 1u;
                        const double cm = me ? o.m[6] : o.m[0], cp = me ? o.m[4] : o.m[2];
                        a[r] = C2{__dadd_rn(__dmul_rn(cm, a[r].re), __dmul_rn(cp, pv[r].re)),
                                  __dadd_rn(__dmul_rn(cm, a[r].im), __dmul_rn(cp, pv[r].im))};
                    }
                } else if (o.pad == 2) {  // cm real, cp imaginary: cp * z = (-ci zi, ci zr)
#pragma unroll
                    for (int r = 0; r < kNV; ++r) {
                        const uint32_t me = (side >> r) & 1u;
                        const double cm = me ? o.m[6] : o.m[0], ci = me ? o.m[5] : o.m[3];
                        a[r] = C2{__dadd_rn(__dmul_rn(cm, a[r].re), -__dmul_rn(ci, pv[r].im)),
                                  __dadd_rn(__dmul_rn(cm, a[r].im), __dmul_rn(ci, pv[r].re))};
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < kNV; ++r) {
                        const uint32_t me = (side >> r) & 1u;
                        const C2 a0 = me ? pv[r] : a[r], a1 = me ? a[r] : pv[r];
                        const double w0r = me ? o.m[4] : o.m[0], w0i = me ? o.m[5] : o.m[1];
                        const double w1r = me ? o.m[6] : o.m[2], w1i = me ? o.m[7] : o.m[3];
                        pv[r] = cadd(cmul(w0r, w0i, a0), cmul(w1r, w1i, a1));
                    }
#pragma unroll
                    for (int r = 0; r < kNV; ++r) a[r] = pv[r];
                }
            }
        }
        if constexpr (kQuant) {
            if (run_len && ((pb ^ run_pb) >> 12)) flush();
            if (!run_len) run_pb = pb;
            uint32_t pk[2 * kNV];
            if (zunit) {
#pragma unroll
                for (int k = 0; k < 2 * kNV; ++k) pk[k] = 1u;
            } else if (q.t.f32) {
                uint32_t need = 0;
#pragma unroll
                for (int r = 0; r < kNV; ++r) {
                    bool n0, n1;
                    pk[2 * r] = quant_est_f32(a[r].re, q.t, span, n0);
                    pk[2 * r + 1] = quant_est_f32(a[r].im, q.t, span, n1);
                    need |= (n0 ? 1u : 0u) << (2 * r);
                    need |= (n1 ? 1u : 0u) << (2 * r + 1);
                }
                if (need) [[unlikely]] {  // ties, subnormals, non-finite: the exact decision
#pragma unroll
                    for (int r = 0; r < kNV; ++r) {
                        if (need >> (2 * r) & 1u) pk[2 * r] = quantize_pack_fast(a[r].re, q.t, qlo_d, span, bad, oow);
                        if (need >> (2 * r + 1) & 1u)
                            pk[2 * r + 1] = quantize_pack_fast(a[r].im, q.t, qlo_d, span, bad, oow);
                    }
                }
            } else {
#pragma unroll
                for (int r = 0; r < kNV; ++r) {
                    pk[2 * r] = quantize_pack_fast(a[r].re, q.t, qlo_d, span, bad, oow);
                    pk[2 * r + 1] = quantize_pack_fast(a[r].im, q.t, qlo_d, span, bad, oow);
                }
            }
            // round trip in place (stage fusion): the table gathers are issued
            // here and land while the counters below are reduced
            double ev[2 * kNV];
            if constexpr (kRound) {
#pragma unroll
                for (int k = 0; k < 2 * kNV; ++k)
                    ev[k] = (pk[k] & 1u) ? 0.0 : __ldg(q.t.dequant + (pk[k] >> 2));
            }
#pragma unroll
            for (int r = 0; r < kNV; ++r) {
                const uint64_t p = pb + pdep[r] + lane;
                if constexpr (!kRound) {
                    __stcs(q.pk + p, pk[2 * r]);
                    __stcs(q.pk + p + im_off, pk[2 * r + 1]);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t w = pk[2 * r + h];
                    const int ra = kSame ? 0 : r;
                    amn[ra][h] = min(amn[ra][h], __reduce_min_sync(0xffffffffu, (w ^ 1u) - 1u));
                    amx[ra][h] = max(amx[ra][h], __reduce_max_sync(0xffffffffu, w));
                    azn[ra][h] += __reduce_add_sync(0xffffffffu, (w & 1u) | ((w & 2u) << 15));
                }
            }
            if constexpr (kRound) {
#pragma unroll
                for (int k = 0; k < 2 * kNV; ++k)
                    q.rnd[pb + pdep[k >> 1] + lane + ((k & 1) ? im_off : 0)] = (pk[k] & 3u) == 2u ? -ev[k] : ev[k];
            }
            ++run_len;
        } else {
#pragma unroll
            for (int r = 0; r < kNV; ++r) {
                const uint64_t p = pb + pdep[r];
                if (wf) {  // an all-zero 32-scalar group is flagged instead of stored
                    const bool nr = __any_sync(0xffffffffu, a[r].re != 0.0), ni = __any_sync(0xffffffffu, a[r].im != 0.0);
                    if (lane == 0) {
                        wf[p >> 5] = nr;
                        wf[(p + im_off) >> 5] = ni;
                    }
                    set_wz = set_wz || !(nr && ni);
                    if (nr) buf[p + lane] = a[r].re;
                    if (ni) buf[p + im_off + lane] = a[r].im;
                } else {
                    buf[p + lane] = a[r].re;
                    buf[p + im_off + lane] = a[r].im;
                }
            }
        }
    }
    if (dbad) dev_fail(dec.err, DE_CODE_WINDOW, 0);
    if constexpr (kQuant) {
        if (run_len) flush();
        if (bad) dev_fail(q.err, DE_NONFINITE, 0);
        if (oow) dev_fail(q.err, DE_WINDOW, 0);
    } else {
        if (set_wz && lane == 0) *wz = 1;
    }
}

// ------------------------------------------------------ general pass (SMEM)
// Any tile size and general 4x4 matrices; used for small buffers and U4.

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
    const uint64_t im_off = interleaved ? 1 : (1ull << lb);
    for (uint32_t j = 0; j < per; ++j) {
        const uint32_t k = tid + j * nth;
        const uint64_t a = planar_addr(base | toff | deposit_x(static_cast<uint64_t>(j) * nth, tile_mask), lb, lmask,
                                       interleaved);
        sre[k] = buf[a];
        sim[k] = buf[a + im_off];
    }
    bool owners_only = true;
    for (uint32_t i = 0; i < nops; ++i) {
        const GateOp* g = ops + i;
        const uint8_t type = g->type;
        if (type == OP_DIAG || type == OP_CDIAG) {
            if (!owners_only) {
                __syncthreads();
                owners_only = true;
            }
            const uint64_t bhi = (base >> g->hi) & 1, blo = (base >> g->lo) & 1;
            for (uint32_t j = 0; j < per; ++j) {
                const uint32_t k = tid + j * nth;
                const uint32_t hv = g->in_hi ? (k >> g->tp_hi) & 1 : static_cast<uint32_t>(bhi);
                uint8_t e;
                if (type == OP_DIAG) {
                    e = hv ? 3 : 0;
                } else {
                    const uint32_t lv = g->in_lo ? (k >> g->tp_lo) & 1 : static_cast<uint32_t>(blo);
                    if (!(hv && lv)) continue;
                    e = 15;
                }
                const uint8_t ty = g->et[e];
                if (ty == ET_ONE) continue;
                const C2 r = entry_mul(ty, g->m[2 * e], g->m[2 * e + 1], C2{sre[k], sim[k]});
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
                const C2 a0{sre[i0], sim[i0]}, a1{sre[i1], sim[i1]};
                const C2 o0 = row2(g->et, g->m, 0, a0, a1), o1 = row2(g->et, g->m, 1, a0, a1);
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
                for (int q = 0; q < 4; ++q) o[q] = row4(g, q, a);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    sre[idx[q]] = o[q].re;
                    sim[idx[q]] = o[q].im;
                }
            }
        }
    }
    __syncthreads();
    for (uint32_t j = 0; j < per; ++j) {
        const uint32_t k = tid + j * nth;
        const uint64_t a = planar_addr(base | toff | deposit_x(static_cast<uint64_t>(j) * nth, tile_mask), lb, lmask,
                                       interleaved);
        buf[a] = sre[k];
        buf[a + im_off] = sim[k];
    }
}

// ------------------------------------------------- code-domain pass (mono)
// Packed code words: (q - qlo) << 2 | negative << 1 | zero. Negation flips
// the sign bit of a nonzero scalar; -0 is a zero with sign bit 0.
__device__ __forceinline__ uint32_t code_neg(uint32_t c) { return (c & 1u) ? c : c ^ 2u; }

// (re, im) * unit: 1 -> (re, im); i -> (-im, re); -1 -> (-re, -im); -i -> (im, -re)
__device__ __forceinline__ uint2 code_unit(uint32_t u, uint2 a) {
    switch (u & 3u) {
    case 0: return a;
    case 1: return make_uint2(code_neg(a.y), a.x);
    case 2: return make_uint2(code_neg(a.x), code_neg(a.y));
    default: return make_uint2(a.y, code_neg(a.x));
    }
}

__global__ void __launch_bounds__(kFastThreads) k_code_pass(uint32_t* __restrict__ pk, uint32_t lb, uint64_t ntiles,
                                                            const __grid_constant__ MonoPass pass,
                                                            ChunkPlan* __restrict__ cps, uint32_t nch) {
    __shared__ uint2 tile_s[1 << kMaxTileBits];
    __shared__ uint64_t joff[kPer];
    __shared__ MonoOp sops[kMaxMonoOps];
    const uint32_t tid = threadIdx.x;
    const uint64_t lmask = (1ull << lb) - 1;
    const uint64_t im_off = 1ull << lb;
    const uint64_t toff = runs_deposit(tid, pass.tile);
    if (tid < kPer) joff[tid] = runs_deposit(static_cast<uint64_t>(tid) << 8, pass.tile);
    for (uint32_t e = tid; e < pass.nops; e += kFastThreads) sops[e] = pass.ops[e];
    __syncthreads();
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t base = runs_deposit(tile, pass.base);
        __syncthreads();  // previous tile's stores have read tile_s
        {
            uint32_t re[kPer], im[kPer];
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const uint64_t a = planar_addr(base | toff | joff[j], lb, lmask, 0);
                re[j] = __ldcs(pk + a);
                im[j] = __ldcs(pk + a + im_off);
            }
#pragma unroll
            for (int j = 0; j < kPer; ++j) tile_s[tid + 256 * j] = make_uint2(re[j], im[j]);
        }
        bool owners_only = true;
        for (uint32_t i = 0; i < pass.nops; ++i) {
            const MonoOp g = sops[i];
            if (g.kind != MK_MIX) {
                if (!owners_only) __syncthreads();
                owners_only = true;
#pragma unroll 4
                for (int j = 0; j < kPer; ++j) {
                    const uint64_t x = base | toff | joff[j];
                    uint32_t u;
                    if (g.kind == MK_DIAG) {
                        u = ((x >> g.hi) & 1) ? g.u1 : g.u0;
                    } else {
                        if (!((x >> g.hi) & (x >> g.lo) & 1)) continue;
                        u = g.u1;
                    }
                    if (u) {
                        const uint32_t k = tid + 256u * j;
                        tile_s[k] = code_unit(u, tile_s[k]);
                    }
                }
                continue;
            }
            __syncthreads();
            owners_only = false;
            const uint32_t m = 1u << g.tp;
            const uint32_t bctl = static_cast<uint32_t>((base >> g.hi) & 1);
            for (uint32_t r = tid; r < 2048; r += kFastThreads) {
                const uint32_t i0 = insert0(r, g.tp), i1 = i0 | m;
                const uint32_t ctl = g.ctl == 0 ? 1u : (g.ctl == 1 ? (i0 >> g.ctl_tp) & 1 : bctl);
                if (!ctl) continue;
                const uint2 a0 = tile_s[i0], a1 = tile_s[i1];
                tile_s[i0] = code_unit(g.u0, a1);
                tile_s[i1] = code_unit(g.u1, a0);
            }
        }
        if (!owners_only) __syncthreads();
        if (cps) {  // last pass: codes + per-chunk counters (see quant_epilogue)
            ChunkAcc acc_re, acc_im;
            uint64_t key_re = ~0ull, key_im = ~0ull;
            for (int j = 0; j < kPer; ++j) {
                const uint2 v = tile_s[tid + 256 * j];
                const uint64_t p = base | toff | joff[j];
                const uint64_t slot = p >> lb, l = p & lmask;
                const uint64_t s_im = im_off + l;
                const uint64_t kre = slot * nch + (l >> 12), kim = slot * nch + (s_im >> 12);
                if (kre != key_re) {  // warp-uniform
                    if (key_re != ~0ull) flush_chunk(cps + key_re, acc_re);
                    acc_re = ChunkAcc{};
                    key_re = kre;
                }
                if (kim != key_im) {
                    if (key_im != ~0ull) flush_chunk(cps + key_im, acc_im);
                    acc_im = ChunkAcc{};
                    key_im = kim;
                }
                uint32_t* dst = pk + (slot << (lb + 1));
                __stcs(dst + l, v.x);
                __stcs(dst + s_im, v.y);
                acc_re.add(v.x);
                acc_im.add(v.y);
            }
            flush_chunk(cps + key_re, acc_re);
            flush_chunk(cps + key_im, acc_im);
            continue;
        }
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint2 v = tile_s[tid + 256 * j];
            const uint64_t a = planar_addr(base | toff | joff[j], lb, lmask, 0);
            __stcs(pk + a, v.x);
            __stcs(pk + a + im_off, v.y);
        }
    }
}

// Table-driven code pass. Thread t owns tile positions 4t + e + 1024 g
// (e, g in 0..3): positions 0..1 are buffer bits 0..1, so each (t, g) is four
// consecutive code words of the real half and of the imaginary half (one
// 16-byte load / store each). The tile is gathered once through the pass's
// (src, unit) table. The last pass also accumulates per-chunk counters:
// lanes are grouped by chunk (__match_any_sync) and reduced with REDUX.
struct CodeAcc4 {
    uint32_t mn = ~0u, mx = 0, nnz = 0, nneg = 0;  // min / max over nonzero packed words
    __device__ __forceinline__ void add(uint32_t c) {
        const uint32_t z = c & 1u;
        mn = min(mn, z ? ~0u : c);
        mx = max(mx, z ? 0u : c);
        nnz += z ^ 1u;
        nneg += (c >> 1) & 1u;
    }
    // all 32 lanes call; lanes with the same key reduce together
    __device__ __forceinline__ void flush(ChunkPlan* cps, uint64_t key) {
        const uint32_t grp = __match_any_sync(0xffffffffu, key);
        const uint32_t a = __reduce_min_sync(grp, mn), b = __reduce_max_sync(grp, mx);
        const uint32_t n = __reduce_add_sync(grp, nnz), g = __reduce_add_sync(grp, nneg);
        if ((threadIdx.x & 31) == static_cast<uint32_t>(__ffs(grp) - 1)) {
            ChunkPlan* cp = cps + key;
            if (n) {
                atomicMax(&cp->qmin_inv, kQOffMax - (a >> 2));
                atomicMax(&cp->qmax_off, b >> 2);
                atomicAdd(&cp->nnz, n);
            }
            if (g) atomicAdd(&cp->nneg, g);
        }
        *this = CodeAcc4{};
    }
    // all 32 lanes call with the same key
    __device__ __forceinline__ void flush_uniform(ChunkPlan* cps, uint64_t key) {
        const uint32_t a = __reduce_min_sync(0xffffffffu, mn), b = __reduce_max_sync(0xffffffffu, mx);
        const uint32_t n = __reduce_add_sync(0xffffffffu, nnz), g = __reduce_add_sync(0xffffffffu, nneg);
        if ((threadIdx.x & 31) == 0) {
            ChunkPlan* cp = cps + key;
            if (n) {
                atomicMax(&cp->qmin_inv, kQOffMax - (a >> 2));
                atomicMax(&cp->qmax_off, b >> 2);
                atomicAdd(&cp->nnz, n);
            }
            if (g) atomicAdd(&cp->nneg, g);
        }
        *this = CodeAcc4{};
    }
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ uint32_t neg_if(uint32_t c, uint32_t n) { return c ^ ((~c & n & 1u) << 1); }

__device__ __forceinline__ void apply_ent(uint32_t e, const uint2* tile_s, uint32_t& x, uint32_t& y) {
    const uint2 a = tile_s[e & 0xfffu];
    const bool sw = (e >> 12) & 1u;
    x = neg_if(sw ? a.y : a.x, e >> 13);
    y = neg_if(sw ? a.x : a.y, e >> 14);
}

constexpr int kPermGroups = 4;  // 4 x 4 positions per thread

// Four consecutive code words (chunk positions s .. s + 3, s a multiple of
// 4) of a chunk read from its payload through a PermSrc record (meta bit 12):
// fetch the two aligned 64-bit words holding their 4 w <= 64 bits, then unpack.
struct PayloadWords {
    uint64_t lo, hi;
    uint32_t sh;
};
__device__ __forceinline__ PayloadWords psrc_fetch(const PermSrc& r, uint32_t s) {
    const uint32_t a = (r.meta & 63u) + s * ((r.meta >> 6) & 31u);
    const uint64_t* p = r.cw + (a >> 6);
    return PayloadWords{__ldg(p), __ldg(p + 1), a & 63u};
}
__device__ __forceinline__ uint4 psrc_unpack(const PayloadWords& f, uint32_t qb, uint32_t meta) {
    const uint32_t w = (meta >> 6) & 31u, mask = (1u << w) - 1, ng = ((meta >> 11) & 1u) << 1;
    const uint64_t win = (f.lo >> f.sh) | ((f.hi << 1) << (63u - f.sh));
    uint4 o;
    o.x = ((qb + (static_cast<uint32_t>(win) & mask)) << 2) | ng;
    o.y = ((qb + (static_cast<uint32_t>(win >> w) & mask)) << 2) | ng;
    o.z = ((qb + (static_cast<uint32_t>(win >> (2 * w)) & mask)) << 2) | ng;
    o.w = ((qb + (static_cast<uint32_t>(win >> (3 * w)) & mask)) << 2) | ng;
    return o;
}

template <bool kLast, bool kPsrc>
__global__ void __launch_bounds__(kFastThreads) k_perm_pass(uint32_t* __restrict__ pk, uint32_t lb, uint64_t ntiles,
                                                            const __grid_constant__ PermPass pass,
                                                            ChunkPlan* __restrict__ cps, const uint8_t* __restrict__ zf,
                                                            uint32_t nch, const uint32_t* __restrict__ imnz,
                                                            const PermSrc* __restrict__ psrc) {
    // kPsrc: the input chunks are described by PermSrc records (psrc; first
    // pass of a code-domain stage): zero chunks and chunks left in the
    // payload were not decoded to pk, the latter are read from the payload
    __shared__ __align__(16) uint2 tile_s[1 << kMaxTileBits];
    const uint32_t tid = threadIdx.x;
    const uint64_t lmask = (1ull << lb) - 1;
    const uint64_t im_off = 1ull << lb;
    uint32_t toffp[kPermGroups];
#pragma unroll
    for (int g = 0; g < kPermGroups; ++g) {
        const uint64_t t = runs_deposit(4u * tid + 1024u * g, pass.tile);
        toffp[g] = static_cast<uint32_t>(((t >> lb) << (lb + 1)) | (t & lmask));
    }
    const uint32_t kshift = lb >= 12 ? 12 : lb + 1;
    const uint64_t kim = lb >= 12 ? (1ull << (lb - 12)) : 0;
    // (slot, chunk) index of a planar address: slots are 2^(lb+1) scalars and
    // chunks 4096 (kPsrc needs lb >= 12), so it is the address >> 12
    const auto chunk_of = [&](uint64_t addr) -> uint64_t {
        return kPsrc ? addr >> 12 : (addr >> (lb + 1)) * nch + ((addr & ((2ull << lb) - 1)) >> 12);
    };
    // imaginary halves all zero (and no pass swaps re / im): they stay zero,
    // and the real halves permute alone (no entry has the swap bit)
    const bool im_zero = imnz && *imnz == 0;
    if (im_zero) {
        // Real halves only, double-buffered: the next tile's words stream
        // into SMEM (cp.async) while this tile is gathered and stored.
        uint32_t* tile_w = reinterpret_cast<uint32_t*>(tile_s);  // two 4096-word buffers
        // The copies are issued unconditionally (an all-zero chunk the decoder
        // left unwritten is read stale); its flag, loaded with the copies and
        // used one tile later, has the thread overwrite its own slots with
        // zero words once they have landed. kPsrc: groups of chunks left in
        // the payload fetch their payload words instead, unpacked into the
        // buffer at the start of the tile's iteration.
        PayloadWords pw[kPermGroups];
        uint32_t pqb[kPermGroups], pmeta[kPermGroups];
        uint32_t pend = 0;  // groups of the next tile held in pw
        const auto issue = [&](uint64_t base, uint32_t* dst) -> uint32_t {
            const uint64_t pb = ((base >> lb) << (lb + 1)) | (base & lmask);
            uint32_t zm = 0;
            if constexpr (kPsrc) {
                PermSrc r[kPermGroups];
#pragma unroll
                for (int g = 0; g < kPermGroups; ++g) r[g] = psrc[chunk_of(pb + toffp[g])];
#pragma unroll
                for (int g = 0; g < kPermGroups; ++g) {
                    const uint64_t addr = pb + toffp[g];
                    if (r[g].meta & (1u << 12)) {
                        pw[g] = psrc_fetch(r[g], static_cast<uint32_t>(addr & 4095u));
                        pqb[g] = r[g].qb;
                        pmeta[g] = r[g].meta;
                        pend |= 1u << g;
                    } else if (r[g].meta & (1u << 13)) {
                        zm |= 1u << g;
                    } else {
                        cp_async16(dst + 4u * tid + 1024u * g, pk + addr);
                    }
                }
            } else {
#pragma unroll
                for (int g = 0; g < kPermGroups; ++g) {
                    const uint64_t addr = pb + toffp[g];
                    cp_async16(dst + 4u * tid + 1024u * g, pk + addr);
                    if (zf && zf[chunk_of(addr)]) zm |= 1u << g;
                }
            }
            cp_async_commit();
            return zm;
        };
        uint64_t tile = blockIdx.x;
        uint64_t base_next = tile < ntiles ? runs_deposit(tile, pass.base) : 0;
        uint32_t zcur = tile < ntiles ? issue(base_next, tile_w) : 0u;
        // one table (no pattern bits): its entries stay in registers
        const bool one_tab = pass.npat_bits == 0;
        uint2 ent[kPermGroups];
        if (one_tab) {
#pragma unroll
            for (int g = 0; g < kPermGroups; ++g)
                ent[g] = __ldg(reinterpret_cast<const uint2*>(pass.table + 4u * tid + 1024u * g));
        }
        CodeAcc4 acc;  // last pass: counters of the real halves (see PermPass::chunk_mode)
        for (uint32_t k = 0; tile < ntiles; tile += gridDim.x, ++k) {
            uint32_t* cur = tile_w + ((k & 1u) << kMaxTileBits);
            if (kPsrc && pend) {  // this tile's payload-read groups
#pragma unroll
                for (int g = 0; g < kPermGroups; ++g)
                    if ((pend >> g) & 1u)
                        *reinterpret_cast<uint4*>(cur + 4u * tid + 1024u * g) = psrc_unpack(pw[g], pqb[g], pmeta[g]);
                pend = 0;
            }
            const uint64_t base = base_next;
            uint32_t znext = 0;
            if (tile + gridDim.x < ntiles) {
                base_next = runs_deposit(tile + gridDim.x, pass.base);
                znext = issue(base_next, tile_w + (((k + 1) & 1u) << kMaxTileBits));
            } else {
                cp_async_commit();  // (an empty group keeps the wait count uniform)
            }
            const uint64_t pb = ((base >> lb) << (lb + 1)) | (base & lmask);
            if (!one_tab) {
                uint32_t pat = 0;
                for (uint32_t i = 0; i < pass.npat_bits; ++i)
                    pat |= static_cast<uint32_t>((base >> pass.pat_bits[i]) & 1) << i;
                const uint16_t* tab = pass.table + (static_cast<uint64_t>(pat) << kMaxTileBits);
#pragma unroll
                for (int g = 0; g < kPermGroups; ++g)
                    ent[g] = __ldg(reinterpret_cast<const uint2*>(tab + 4u * tid + 1024u * g));
            }
            cp_async_wait<1>();  // this tile's group has landed
            if (zcur) {
#pragma unroll
                for (int g = 0; g < kPermGroups; ++g)
                    if ((zcur >> g) & 1u) *reinterpret_cast<uint4*>(cur + 4u * tid + 1024u * g) = make_uint4(1u, 1u, 1u, 1u);
            }
            zcur = znext;
            __syncthreads();
#pragma unroll
            for (int g = 0; g < kPermGroups; ++g) {
                uint4 xo;
                const uint32_t e0 = ent[g].x & 0xffffu, e1 = ent[g].x >> 16, e2 = ent[g].y & 0xffffu, e3 = ent[g].y >> 16;
                xo.x = neg_if(cur[e0 & 0xfffu], e0 >> 13);
                xo.y = neg_if(cur[e1 & 0xfffu], e1 >> 13);
                xo.z = neg_if(cur[e2 & 0xfffu], e2 >> 13);
                xo.w = neg_if(cur[e3 & 0xfffu], e3 >> 13);
                const uint64_t addr = pb + toffp[g];
                __stcs(reinterpret_cast<uint4*>(pk + addr), xo);
                if (kLast) {
                    acc.add(xo.x);
                    acc.add(xo.y);
                    acc.add(xo.z);
                    acc.add(xo.w);
                    if (pass.chunk_mode == 0)
                        acc.flush(cps, addr >> kshift);
                    else if (pass.chunk_mode == 1 || g == kPermGroups - 1)
                        acc.flush_uniform(cps, addr >> kshift);
                }
            }
            __syncthreads();  // this buffer is refilled two tiles on
        }
        return;
    }
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint64_t base = runs_deposit(tile, pass.base);
        const uint64_t pb = ((base >> lb) << (lb + 1)) | (base & lmask);
        uint4 re[kPermGroups], im[kPermGroups];
        if constexpr (kPsrc) {
            PermSrc rr[kPermGroups], ri[kPermGroups];
#pragma unroll
            for (int g = 0; g < kPermGroups; ++g) {
                rr[g] = psrc[chunk_of(pb + toffp[g])];
                ri[g] = psrc[chunk_of(pb + toffp[g] + im_off)];
            }
            const auto load = [&](const PermSrc& r, uint64_t addr) -> uint4 {
                if (r.meta & (1u << 12)) return psrc_unpack(psrc_fetch(r, static_cast<uint32_t>(addr & 4095u)), r.qb, r.meta);
                if (r.meta & (1u << 13)) return make_uint4(1u, 1u, 1u, 1u);
                return __ldcs(reinterpret_cast<const uint4*>(pk + addr));
            };
#pragma unroll
            for (int g = 0; g < kPermGroups; ++g) {
                const uint64_t addr = pb + toffp[g];
                re[g] = load(rr[g], addr);
                im[g] = im_zero ? make_uint4(1u, 1u, 1u, 1u) : load(ri[g], addr + im_off);
            }
        } else {
#pragma unroll
            for (int g = 0; g < kPermGroups; ++g) {
                const uint64_t addr = pb + toffp[g];
                if (zf) {  // all-zero input chunks were not written: read them as zero words
                    const uint64_t slot = addr >> (lb + 1), off = addr & ((2ull << lb) - 1);
                    const uint8_t* zs = zf + slot * nch;
                    re[g] = zs[off >> 12] ? make_uint4(1u, 1u, 1u, 1u) : __ldcs(reinterpret_cast<const uint4*>(pk + addr));
                    im[g] = im_zero || zs[(off + im_off) >> 12] ? make_uint4(1u, 1u, 1u, 1u)
                                                                 : __ldcs(reinterpret_cast<const uint4*>(pk + addr + im_off));
                    continue;
                }
                re[g] = __ldcs(reinterpret_cast<const uint4*>(pk + addr));
                im[g] = im_zero ? make_uint4(1u, 1u, 1u, 1u) : __ldcs(reinterpret_cast<const uint4*>(pk + addr + im_off));
            }
        }
        uint32_t pat = 0;
        for (uint32_t i = 0; i < pass.npat_bits; ++i) pat |= static_cast<uint32_t>((base >> pass.pat_bits[i]) & 1) << i;
        const uint16_t* tab = pass.table + (static_cast<uint64_t>(pat) << kMaxTileBits);
        uint2 ent[kPermGroups];
#pragma unroll
        for (int g = 0; g < kPermGroups; ++g) ent[g] = __ldg(reinterpret_cast<const uint2*>(tab + 4u * tid + 1024u * g));
        __syncthreads();  // previous tile's gathers are done
#pragma unroll
        for (int g = 0; g < kPermGroups; ++g) {
            uint4* d = reinterpret_cast<uint4*>(tile_s + 4u * tid + 1024u * g);
            d[0] = make_uint4(re[g].x, im[g].x, re[g].y, im[g].y);
            d[1] = make_uint4(re[g].z, im[g].z, re[g].w, im[g].w);
        }
        __syncthreads();
#pragma unroll
        for (int g = 0; g < kPermGroups; ++g) {
            uint4 xo, yo;
            apply_ent(ent[g].x & 0xffffu, tile_s, xo.x, yo.x);
            apply_ent(ent[g].x >> 16, tile_s, xo.y, yo.y);
            apply_ent(ent[g].y & 0xffffu, tile_s, xo.z, yo.z);
            apply_ent(ent[g].y >> 16, tile_s, xo.w, yo.w);
            const uint64_t addr = pb + toffp[g];
            __stcs(reinterpret_cast<uint4*>(pk + addr), xo);
            if (!im_zero) __stcs(reinterpret_cast<uint4*>(pk + addr + im_off), yo);
            if (kLast) {
                CodeAcc4 ar;
                ar.add(xo.x);
                ar.add(xo.y);
                ar.add(xo.z);
                ar.add(xo.w);
                const uint64_t key = addr >> kshift;  // chunk of the real half
                ar.flush(cps, key);
                if (!im_zero) {  // (zero codes add nothing to the counters)
                    CodeAcc4 ai;
                    ai.add(yo.x);
                    ai.add(yo.y);
                    ai.add(yo.z);
                    ai.add(yo.w);
                    ai.flush(cps, key + kim);
                }
            }
        }
    }
}

}  // namespace

bool mono_zero_skip(const GateProgram& prog, uint32_t lb) {
    return prog.mono && !prog.passes.empty() && prog.passes[0].pp && lb >= 12;
}

void run_mono_program(cudaStream_t st, const GateProgram& prog, uint32_t* pk, uint32_t lb, uint64_t nreps,
                      uint64_t* launches, const QuantOut& quant, const uint8_t* zflag, const uint32_t* imnz,
                      const PermSrc* psrc) {
    if ((zflag || psrc) && !mono_zero_skip(prog, lb))
        raise(BMQ_ERR_LOGIC, "zero-chunk skipping needs a table first pass");
    if (!prog.mono) raise(BMQ_ERR_LOGIC, "stage is not a code-domain program");
    // imaginary halves can stay untouched only if every pass is a table pass that never swaps re / im
    if (!zflag) imnz = nullptr;
    for (const GatePass& p : prog.passes)
        if (!p.pp || p.pp->reim_swap) imnz = nullptr;
    for (size_t pi = 0; pi < prog.passes.size(); ++pi) {
        const GatePass& p = prog.passes[pi];
        const uint64_t tiles = nreps << (prog.total_bits - p.tb);
        const uint64_t grid = std::min<uint64_t>(tiles, 148ull * 6 * 8);
        const bool last = pi + 1 == prog.passes.size();
        if (p.pp && lb >= 4) {  // 16-byte groups of four code words stay inside a block half
            const uint64_t g2 = std::min<uint64_t>(tiles, 148ull * 4 * 16);
            const uint8_t* zf = pi == 0 ? zflag : nullptr;
            const PermSrc* ps = pi == 0 ? psrc : nullptr;
            PermPass pp = *p.pp;
            pp.chunk_mode = 0;
            if (lb >= 12 && !(pp.lane_bits >> 12)) pp.chunk_mode = (pp.group_bits >> 12) ? 1u : 2u;
            const auto launch = [&](auto kern, ChunkPlan* cps) {
                kern<<<static_cast<uint32_t>(g2), kFastThreads, 0, st>>>(pk, lb, tiles, pp, cps, zf, quant.nch, imnz, ps);
            };
            if (last)
                ps ? launch(k_perm_pass<true, true>, quant.cps) : launch(k_perm_pass<true, false>, quant.cps);
            else
                ps ? launch(k_perm_pass<false, true>, nullptr) : launch(k_perm_pass<false, false>, nullptr);
        } else {
            k_code_pass<<<static_cast<uint32_t>(grid), kFastThreads, 0, st>>>(pk, lb, tiles, *p.mp,
                                                                              last ? quant.cps : nullptr, quant.nch);
        }
        BMQ_CUDA(cudaGetLastError());
        if (launches) ++*launches;
    }
}

// BMQ_DBG_FULL_SUPPORT=1 disables tile support tracking (every position is
// visited), for bisecting; read once.
bool full_support_debug() {
    static const bool on = getenv("BMQ_DBG_FULL_SUPPORT") != nullptr;
    return on;
}

// BMQ_DBG_NO_STREAM=1 keeps every pass on the tiled kernel (A/B and
// bisecting); read once.
bool stream_off() {
    static const bool on = getenv("BMQ_DBG_NO_STREAM") != nullptr;
    return on;
}

bool stream_first_pass(const GateProgram& prog, uint32_t lb, bool interleaved, bool blockwise) {
    if (prog.passes.empty() || interleaved || lb < 12 || stream_off()) return false;
    const GatePass& p = prog.passes[0];
    return p.sp && (!blockwise || !((1ull << p.sp->qbit[kStreamNQ - 1]) >> lb));
}

bool program_zero_skip(const GateProgram& prog, uint32_t lb, bool interleaved) {
    if (interleaved || lb < 12 || prog.passes.empty()) return false;
    for (const GatePass& p : prog.passes)
        if (!p.fast) return false;
    return true;
}

bool last_pass_streams(const GateProgram& prog, uint32_t lb) {
    return !prog.passes.empty() && prog.passes.back().fast && prog.passes.back().sp && lb >= 12 && !stream_off();
}

bool run_program(cudaStream_t st, const GateProgram& prog, double* buf, uint32_t lb, bool interleaved,
                 uint64_t nreps, uint64_t* launches, const QuantOut* quant, const uint32_t* vtab,
                 uint64_t nblocks, const uint8_t* zflag, uint32_t nch, uint32_t* wz, const FusedDecode* dec) {
    if (zflag && !wz) raise(BMQ_ERR_LOGIC, "zero-group flags need their summary word");
    if (zflag && !program_zero_skip(prog, lb, interleaved))
        raise(BMQ_ERR_LOGIC, "zero-group skipping needs fast passes only");
    const bool fuse = quant && !interleaved && lb >= 12 && !prog.passes.empty() && prog.passes.back().fast;
    if (vtab) {  // block-wise batch: every pass must be fast and its tile local
        for (const GatePass& p : prog.passes)
            if (!p.fast || (p.tile_mask >> lb) || lb < p.tb)
                raise(BMQ_ERR_LOGIC, "block-wise gate batch needs local fast passes");
    }
    const QuantOut none{};
    static thread_local int attr_dev = -1;
    int dev = 0;
    BMQ_CUDA(cudaGetDevice(&dev));
    const int tile_bytes = (1 << kMaxTileBits) * static_cast<int>(sizeof(double2));
    if (attr_dev != dev) {
        BMQ_CUDA(cudaFuncSetAttribute(k_gate_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, tile_bytes));
        BMQ_CUDA(cudaFuncSetAttribute(k_gate_pass_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr_dev = dev;
    }
    for (size_t pi = 0; pi < prog.passes.size(); ++pi) {
        const GatePass& p = prog.passes[pi];
        const uint64_t tiles = vtab ? nblocks << (lb - p.tb) : nreps << (prog.total_bits - p.tb);
        const bool last = pi + 1 == prog.passes.size();
        const FusedDecode fd = (pi == 0 && dec) ? *dec : FusedDecode{};
        if (pi == 0 && dec && !stream_first_pass(prog, lb, interleaved, vtab != nullptr))
            raise(BMQ_ERR_LOGIC, "fused decoding needs a streaming first pass");
        if (p.sp && !interleaved && lb >= 12 && !stream_off() &&
            (!vtab || !((1ull << p.sp->qbit[kStreamNQ - 1]) >> lb))) {
            const uint64_t units = (vtab ? nblocks << lb : nreps << prog.total_bits) >> (5 + kStreamNQ);
            const uint64_t warps_per_cta = kStreamThreads / 32;
            const uint64_t grid = std::min<uint64_t>((units + warps_per_cta - 1) / warps_per_cta, 148ull * 8);
            uint8_t* zf = const_cast<uint8_t*>(zflag);
            const dim3 g(static_cast<uint32_t>(grid)), b(kStreamThreads);
            if (fuse && last) {
                if (fd.rows)
                    k_stream_pass<true, true><<<g, b, 0, st>>>(buf, lb, units, *p.sp, *quant, vtab, zf, wz, fd);
                else if (quant->rnd && p.sp->qbit[kStreamNQ - 1] < 12)
                    k_stream_pass<true, false, true, true><<<g, b, 0, st>>>(buf, lb, units, *p.sp, *quant, vtab, zf, wz, fd);
                else if (quant->rnd)
                    k_stream_pass<true, false, false, true><<<g, b, 0, st>>>(buf, lb, units, *p.sp, *quant, vtab, zf, wz, fd);
                else if (p.sp->qbit[kStreamNQ - 1] < 12)
                    k_stream_pass<true, false, true><<<g, b, 0, st>>>(buf, lb, units, *p.sp, *quant, vtab, zf, wz, fd);
                else
                    k_stream_pass<true, false><<<g, b, 0, st>>>(buf, lb, units, *p.sp, *quant, vtab, zf, wz, fd);
            } else {
                if (fd.rows)
                    k_stream_pass<false, true><<<g, b, 0, st>>>(buf, lb, units, *p.sp, none, vtab, zf, wz, fd);
                else
                    k_stream_pass<false, false><<<g, b, 0, st>>>(buf, lb, units, *p.sp, none, vtab, zf, wz, fd);
            }
        } else if (p.fast) {
            const size_t smem = tile_bytes + p.fp->tab_entries * sizeof(double2) + p.fp->nops * sizeof(FastOp);
            const uint64_t per_sm = std::max<uint64_t>(1, (227ull * 1024) / (smem + 2048));
            const uint64_t grid = std::min<uint64_t>(tiles, 148ull * per_sm * 8);
            k_gate_pass_fast<<<static_cast<uint32_t>(grid), kFastThreads, smem, st>>>(
                buf, lb, interleaved ? 1 : 0, tiles, *p.fp, (fuse && last) ? *quant : none, vtab,
                full_support_debug() ? 1 : 0, const_cast<uint8_t*>(zflag), wz);
        } else {
            const uint32_t nth = std::min<uint32_t>(kPassThreads, 1u << p.tb);
            const size_t smem = 2 * (size_t(1) << p.tb) * sizeof(double);
            k_gate_pass<<<static_cast<uint32_t>(tiles), nth, smem, st>>>(buf, lb, interleaved ? 1 : 0, p.tile_mask,
                                                                        p.tb, prog.d_ops + p.begin, p.count);
        }
        BMQ_CUDA(cudaGetLastError());
        if (launches) ++*launches;
    }
    return fuse;
}

}  // namespace bmq
