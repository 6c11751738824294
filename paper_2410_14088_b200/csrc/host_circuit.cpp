// host_circuit.cpp — host-side descriptors of the drop-in surface: gate
// validation and unitaries (circuit.hpp), the benchmark generators
// (benchmarks.hpp), layout / greedy staging / group geometry (partition.hpp).
// These are the inputs the device path consumes; they run once per circuit.
#include <algorithm>
#include <cmath>
#include <complex>
#include <numbers>
#include <random>

#include "bmq_internal.hpp"

namespace bmq {

bool gate_is_two_qubit(uint32_t kind) {
    return kind == BMQ_GATE_CX || kind == BMQ_GATE_CZ || kind == BMQ_GATE_CP;
}

// Circuit(n) and Circuit::add (circuit.hpp:103-127).
void check_circuit(uint32_t n, const bmq_gate* gates, uint64_t count) {
    if (n < 1 || n > 62)
        raise(BMQ_ERR_INVALID_ARGUMENT, "qubit count must be in [1, 62], got " + std::to_string(n));
    for (uint64_t i = 0; i < count; ++i) {
        const bmq_gate& g = gates[i];
        if (g.kind > BMQ_GATE_CP) raise(BMQ_ERR_INVALID_ARGUMENT, "unknown gate kind " + std::to_string(g.kind));
        const auto out_of_range = [n](uint32_t q) {
            return "gate operand " + std::to_string(q) + " out of range for " + std::to_string(n) + " qubits";
        };
        if (g.q0 >= n) raise(BMQ_ERR_INVALID_ARGUMENT, out_of_range(g.q0));
        if (gate_is_two_qubit(g.kind)) {
            if (g.q1 >= n) raise(BMQ_ERR_INVALID_ARGUMENT, out_of_range(g.q1));
            if (g.q0 == g.q1) raise(BMQ_ERR_INVALID_ARGUMENT, "two-qubit gate operands must be distinct");
        }
    }
}

namespace {
Cx from_std(std::complex<double> z) { return Cx{z.real(), z.imag()}; }
}  // namespace

// Entries use the same libm calls as the reference (sqrt, cos, sin,
// std::polar), so every matrix entry is bit-identical to unitary2/unitary4.
int gate_matrix(const bmq_gate& g, Cx* u) {
    constexpr double pi = std::numbers::pi;
    const double a = g.angle;
    const Cx zero{0.0, 0.0}, one{1.0, 0.0};
    if (gate_is_two_qubit(g.kind)) {
        for (int i = 0; i < 16; ++i) u[i] = zero;
        u[0] = one;   // |00> -> |00>
        u[5] = one;   // |01> -> |01>
        switch (g.kind) {
        case BMQ_GATE_CX: u[11] = one; u[14] = one; break;          // swap |10>,|11>
        case BMQ_GATE_CZ: u[10] = one; u[15] = Cx{-1.0, 0.0}; break;
        default: u[10] = one; u[15] = from_std(std::polar(1.0, a)); break;  // CP
        }
        return 4;
    }
    for (int i = 0; i < 4; ++i) u[i] = zero;
    switch (g.kind) {
    case BMQ_GATE_H: {
        const double h = 1.0 / std::sqrt(2.0);
        u[0] = Cx{h, 0}; u[1] = Cx{h, 0}; u[2] = Cx{h, 0}; u[3] = Cx{-h, 0};
        break;
    }
    case BMQ_GATE_X: u[1] = one; u[2] = one; break;
    case BMQ_GATE_Y: u[1] = Cx{0, -1}; u[2] = Cx{0, 1}; break;
    case BMQ_GATE_Z: u[0] = one; u[3] = Cx{-1, 0}; break;
    case BMQ_GATE_S: u[0] = one; u[3] = Cx{0, 1}; break;
    case BMQ_GATE_SDG: u[0] = one; u[3] = Cx{0, -1}; break;
    case BMQ_GATE_T: u[0] = one; u[3] = from_std(std::polar(1.0, pi / 4)); break;
    case BMQ_GATE_TDG: u[0] = one; u[3] = from_std(std::polar(1.0, -pi / 4)); break;
    case BMQ_GATE_RX: {
        const double c = std::cos(a / 2), s = std::sin(a / 2);
        u[0] = Cx{c, 0}; u[1] = Cx{0, -s}; u[2] = Cx{0, -s}; u[3] = Cx{c, 0};
        break;
    }
    case BMQ_GATE_RY: {
        const double c = std::cos(a / 2), s = std::sin(a / 2);
        u[0] = Cx{c, 0}; u[1] = Cx{-s, 0}; u[2] = Cx{s, 0}; u[3] = Cx{c, 0};
        break;
    }
    case BMQ_GATE_RZ:
        u[0] = from_std(std::polar(1.0, -a / 2));
        u[3] = from_std(std::polar(1.0, a / 2));
        break;
    case BMQ_GATE_P: u[0] = one; u[3] = from_std(std::polar(1.0, a)); break;
    default: raise(BMQ_ERR_LOGIC, "unitary2 called on a two-qubit gate");
    }
    return 2;
}

// Benchmark generators (benchmarks.hpp:44-166).
// ---- BASELINE.json workloads outside the reference's generator set. They
// use only the reference gate set, so the reference consumes the same gate
// lists (or their QASM text, bmq_emit_qasm -> parse_qasm) unchanged.

// Random 3-regular graph on n nodes (n even, n >= 4) by the pairing model:
// 3n points, Fisher-Yates shuffle driven by mt19937_64(seed), consecutive
// points paired; a pairing with a loop or a repeated edge is redrawn.
// Edges are returned sorted (i < j, lexicographic).
std::vector<std::pair<uint32_t, uint32_t>> random_3regular(uint32_t n, uint64_t seed) {
    if (n < 4 || n % 2) raise(BMQ_ERR_INVALID_ARGUMENT, "a 3-regular graph needs an even node count >= 4");
    std::mt19937_64 rng(seed);
    std::vector<uint32_t> pts(3 * n);
    for (;;) {
        for (uint32_t i = 0; i < 3 * n; ++i) pts[i] = i / 3;
        for (uint32_t i = 3 * n - 1; i > 0; --i) std::swap(pts[i], pts[rng() % (i + 1)]);
        std::vector<std::pair<uint32_t, uint32_t>> e;
        bool ok = true;
        for (uint32_t i = 0; i < 3 * n && ok; i += 2) {
            const uint32_t a = std::min(pts[i], pts[i + 1]), b = std::max(pts[i], pts[i + 1]);
            ok = a != b;
            e.push_back({a, b});
        }
        if (!ok) continue;
        std::sort(e.begin(), e.end());
        if (std::adjacent_find(e.begin(), e.end()) != e.end()) continue;
        return e;
    }
}

// QAOA MaxCut: p layers of CX-RZ(gamma)-CX per
// edge of a random 3-regular graph, then RX(beta) on every qubit; gamma and
// beta drawn per layer exactly like make_qaoa (benchmarks.hpp:118-143); no
// initial H layer, mirroring the reference's QAOA.
std::vector<bmq_gate> make_qaoa_3regular(uint32_t n, uint32_t layers, uint64_t seed) {
    if (layers < 1) raise(BMQ_ERR_INVALID_ARGUMENT, "qaoa requires at least one layer");
    const auto edges = random_3regular(n, seed);
    std::mt19937_64 rng(seed);
    const double two_pi = 2.0 * std::numbers::pi;
    std::vector<bmq_gate> c;
    for (uint32_t l = 0; l < layers; ++l) {
        const double gamma = static_cast<double>(rng() >> 11) * 0x1.0p-53 * two_pi;
        const double beta = static_cast<double>(rng() >> 11) * 0x1.0p-53 * two_pi;
        for (const auto& [i, j] : edges) {
            c.push_back({BMQ_GATE_CX, i, j, 0, 0.0});
            c.push_back({BMQ_GATE_RZ, j, 0, 0, gamma});
            c.push_back({BMQ_GATE_CX, i, j, 0, 0.0});
        }
        for (uint32_t q = 0; q < n; ++q) c.push_back({BMQ_GATE_RX, q, 0, 0, beta});
    }
    return c;
}

// Random circuit on an r x c grid (r = largest
// divisor of n not above sqrt(n)): per cycle a random sqrt(X) / sqrt(Y) /
// sqrt(W) on every qubit, never the same gate twice in a row on one qubit,
// then CZ on one of four nearest-neighbour patterns cycled A B C D
// (horizontal even / odd columns, vertical even / odd rows). In the
// reference gate set sqrt(X) = RX(pi/2), sqrt(Y) = RY(pi/2) and
// sqrt(W) = RZ(-pi/4) RX(pi/2) RZ(pi/4) (up to a global phase).
std::vector<bmq_gate> make_random_circuit(uint32_t n, uint32_t cycles, uint64_t seed) {
    if (cycles < 1) raise(BMQ_ERR_INVALID_ARGUMENT, "random circuit requires at least one cycle");
    uint32_t rows = 1;
    for (uint32_t r = 1; r * r <= n; ++r)
        if (n % r == 0) rows = r;
    const uint32_t cols = n / rows;
    std::mt19937_64 rng(seed);
    const double h = std::numbers::pi / 2, qtr = std::numbers::pi / 4;
    std::vector<bmq_gate> c;
    std::vector<int> prev(n, -1);
    for (uint32_t cy = 0; cy < cycles; ++cy) {
        for (uint32_t q = 0; q < n; ++q) {
            int g = static_cast<int>(rng() % 3);
            if (prev[q] >= 0) {  // one of the two gates other than the previous one
                const int k = static_cast<int>(rng() % 2);
                g = (prev[q] + 1 + k) % 3;
            }
            prev[q] = g;
            if (g == 0) {
                c.push_back({BMQ_GATE_RX, q, 0, 0, h});
            } else if (g == 1) {
                c.push_back({BMQ_GATE_RY, q, 0, 0, h});
            } else {
                c.push_back({BMQ_GATE_RZ, q, 0, 0, -qtr});
                c.push_back({BMQ_GATE_RX, q, 0, 0, h});
                c.push_back({BMQ_GATE_RZ, q, 0, 0, qtr});
            }
        }
        const uint32_t pat = cy % 4;
        for (uint32_t r = 0; r < rows; ++r)
            for (uint32_t k = 0; k < cols; ++k) {
                const uint32_t q = r * cols + k;
                if (pat < 2 && k % 2 == pat && k + 1 < cols) c.push_back({BMQ_GATE_CZ, q, q + 1, 0, 0.0});
                if (pat >= 2 && r % 2 == pat - 2 && r + 1 < rows) c.push_back({BMQ_GATE_CZ, q, q + cols, 0, 0.0});
            }
    }
    return c;
}

std::vector<bmq_gate> make_benchmark(const std::string& name, uint32_t n, uint32_t layers,
                                     uint64_t seed, const char* secret) {
    const bool ghz = name == "ghz" || name == "cat_state";
    if (name == "qaoa3reg") return make_qaoa_3regular(n, layers, seed);
    if (name == "random") return make_random_circuit(n, layers, seed);
    if (!ghz && name != "bv" && name != "qft" && name != "qaoa")
        raise(BMQ_ERR_INVALID_ARGUMENT, "unknown benchmark '" + name + "'");
    if (n < 2) raise(BMQ_ERR_INVALID_ARGUMENT, name + " requires at least 2 qubits");
    if (n > 62) raise(BMQ_ERR_INVALID_ARGUMENT, "qubit count must be in [1, 62], got " + std::to_string(n));
    std::vector<bmq_gate> c;
    const auto one = [&c](uint32_t k, uint32_t q, double ang = 0.0) { c.push_back({k, q, 0, 0, ang}); };
    const auto two = [&c](uint32_t k, uint32_t q0, uint32_t q1, double ang = 0.0) {
        c.push_back({k, q0, q1, 0, ang});
    };
    if (ghz) {  // H(0) then a CX ladder
        one(BMQ_GATE_H, 0);
        for (uint32_t q = 1; q < n; ++q) two(BMQ_GATE_CX, q - 1, q);
    } else if (name == "bv") {
        std::string s;
        if (secret && *secret) {
            s = secret;
        } else {
            for (uint32_t i = 0; i + 1 < n; ++i) s.push_back(i % 2 ? '0' : '1');
        }
        if (s.size() > n - 1)
            raise(BMQ_ERR_INVALID_ARGUMENT, "bv secret longer than the " + std::to_string(n - 1) + " data qubits");
        if (s.find_first_not_of("01") != std::string::npos)
            raise(BMQ_ERR_INVALID_ARGUMENT, "bv secret must contain only '0' and '1'");
        const uint32_t anc = n - 1;
        one(BMQ_GATE_X, anc);
        for (uint32_t q = 0; q < n; ++q) one(BMQ_GATE_H, q);
        for (uint32_t i = 0; i < s.size(); ++i)
            if (s[i] == '1') two(BMQ_GATE_CX, i, anc);
        for (uint32_t q = 0; q < n; ++q) one(BMQ_GATE_H, q);
    } else if (name == "qft") {
        for (uint32_t t = n; t-- > 0;) {
            one(BMQ_GATE_H, t);
            for (uint32_t ctl = t; ctl-- > 0;)
                two(BMQ_GATE_CP, ctl, t, std::numbers::pi / static_cast<double>(1ull << (t - ctl)));
        }
        for (uint32_t lo = 0; lo < n / 2; ++lo) {  // bit reversal, swaps as CX triples
            const uint32_t hi = n - 1 - lo;
            two(BMQ_GATE_CX, lo, hi);
            two(BMQ_GATE_CX, hi, lo);
            two(BMQ_GATE_CX, lo, hi);
        }
    } else {  // qaoa: ring ZZ via CX-RZ-CX, RX mixer, angles from mt19937_64
        if (layers < 1) raise(BMQ_ERR_INVALID_ARGUMENT, "qaoa requires at least one layer");
        std::mt19937_64 rng(seed);
        const double two_pi = 2.0 * std::numbers::pi;
        for (uint32_t l = 0; l < layers; ++l) {
            const double gamma = static_cast<double>(rng() >> 11) * 0x1.0p-53 * two_pi;
            const double beta = static_cast<double>(rng() >> 11) * 0x1.0p-53 * two_pi;
            for (uint32_t q = 0; q < n; ++q) {
                const uint32_t nxt = q + 1 == n ? 0 : q + 1;
                two(BMQ_GATE_CX, q, nxt);
                one(BMQ_GATE_RZ, nxt, gamma);
                two(BMQ_GATE_CX, q, nxt);
            }
            for (uint32_t q = 0; q < n; ++q) one(BMQ_GATE_RX, q, beta);
        }
    }
    return c;
}

Layout make_layout(uint32_t n, uint32_t b) {
    if (n < 1 || n > 62) raise(BMQ_ERR_INVALID_ARGUMENT, "layout qubit count must be in [1, 62]");
    if (b < 1 || b > n) raise(BMQ_ERR_INVALID_ARGUMENT, "local index bits must be in [1, n]");
    return Layout{n, b, n - b};
}

// Greedy Alg. 1 staging (partition.hpp:59-101). The open stage's distinct
// global operands are tracked as a bit mask; a gate that would push the
// count past max(inner_size, 2) closes the stage (unless it is the stage's
// first gate) and opens the next one with its own globals.
std::vector<bmq_stage> partition_plan(uint32_t n, const bmq_gate* gates, uint64_t count,
                                      uint32_t block_bits, uint32_t inner_size) {
    check_circuit(n, gates, count);
    const Layout L = make_layout(n, block_bits);
    const uint32_t limit = std::max(inner_size, 2u);
    const auto globals_of = [&](const bmq_gate& g) {
        uint64_t m = 0;
        if (g.q0 >= L.b) m |= 1ull << g.q0;
        if (gate_is_two_qubit(g.kind) && g.q1 >= L.b) m |= 1ull << g.q1;
        return m;
    };
    const auto close = [](std::vector<bmq_stage>& out, uint64_t begin, uint64_t end, uint64_t mask) {
        bmq_stage st{};
        st.gate_begin = begin;
        st.gate_end = end;
        for (uint32_t q = 0; q < 64; ++q)
            if (mask >> q & 1) st.inner[st.inner_count++] = q;
        out.push_back(st);
    };
    std::vector<bmq_stage> stages;
    uint64_t open_mask = 0, begin = 0;
    for (uint64_t i = 0; i < count; ++i) {
        const uint64_t g = globals_of(gates[i]);
        const uint64_t merged = open_mask | g;
        if (static_cast<uint32_t>(__builtin_popcountll(merged)) > limit && i > begin) {
            close(stages, begin, i, open_mask);
            begin = i;
            open_mask = g;
        } else {
            open_mask = merged;
        }
    }
    if (begin < count) close(stages, begin, count, open_mask);
    return stages;
}

// ------------------------------------------------ device-aware planning
// An optional alternative to the fixed inner_size of
// partition_circuit: every greedy plan partition_plan(n, b, k) is a legal
// staging, and on this engine a stage costs about one trip of the state
// through HBM per tile pass (decode -> passes -> quantise -> emit), so fewer
// stages (larger k) win until the extra tile passes of wider stages, the
// group buffer (2^(b+k) complex doubles must fit the work budget) or, for
// world > 1, the device bits (k <= c - log2 world) and the payload remaps
// between stages take over. The chosen plan is partition_plan at the best k,
// so it can be replayed by the reference (partition.hpp:59-101) with
// inner_size = k.

namespace {

bool gate_mixes(uint32_t kind) {
    switch (kind) {
    case BMQ_GATE_H: case BMQ_GATE_X: case BMQ_GATE_Y: case BMQ_GATE_RX: case BMQ_GATE_RY: case BMQ_GATE_CX:
        return true;
    default:
        return false;
    }
}

// Tile passes of one stage (gates.cu build_program): a pass holds buffer
// bits 0..4 plus the mixing bits of its gates, at most 12.
uint32_t stage_passes(const Layout& L, const bmq_stage& st, const bmq_gate* gates) {
    const uint32_t total = L.b + st.inner_count;
    const uint32_t tb = std::min<uint32_t>(total, 12);
    const uint64_t coalesce = (1ull << std::min<uint32_t>(5, total)) - 1;
    uint32_t passes = 1;
    uint64_t mix = 0;
    for (uint64_t i = st.gate_begin; i < st.gate_end; ++i) {
        const bmq_gate& g = gates[i];
        if (!gate_mixes(g.kind)) continue;
        const uint32_t q = g.kind == BMQ_GATE_CX ? g.q1 : g.q0;
        const uint64_t m = 1ull << buffer_bit(L, st, q);
        if (static_cast<uint32_t>(__builtin_popcountll(mix | m | coalesce)) > tb && mix) {
            ++passes;
            mix = 0;
        }
        mix |= m;
    }
    return passes;
}

}  // namespace

std::vector<bmq_stage> plan_device_aware(uint32_t n, const bmq_gate* gates, uint64_t count, uint32_t block_bits,
                                         const bmq_plan_model& model, bmq_plan_choice* choice) {
    check_circuit(n, gates, count);
    const Layout L = make_layout(n, block_bits);
    if (model.world == 0 || (model.world & (model.world - 1)))
        raise(BMQ_ERR_INVALID_ARGUMENT, "shard count must be a power of two");
    if (!(model.hbm_gbs > 0.0) || (model.world > 1 && !(model.link_gbs > 0.0)) || !(model.ratio > 0.0) ||
        !(model.codec_eff > 0.0) || !(model.pass_eff > 0.0))
        raise(BMQ_ERR_INVALID_ARGUMENT, "plan model needs positive bandwidths, efficiencies and compression ratio");
    uint32_t m = 0;
    while ((1u << m) < model.world) ++m;
    if (m > L.c) raise(BMQ_ERR_INVALID_ARGUMENT, "more shards than blocks");
    // largest inner size: outer bits left for the device bits, group buffer within the work budget
    uint32_t kmax = std::min<uint32_t>(L.c - m, model.max_inner ? model.max_inner : 64);
    while (kmax > 2 && (16ull << (L.b + kmax)) > model.work_bytes) --kmax;
    kmax = std::max<uint32_t>(kmax, std::min<uint32_t>(2, L.c - m));
    const double amps = std::ldexp(1.0, static_cast<int>(n)) / model.world;  // per GPU
    const double cbytes = 16.0 / model.ratio;                               // payload bytes per amplitude
    std::vector<bmq_stage> best;
    double best_s = 0.0;
    bmq_plan_choice ch{};
    ch.candidates = 0;
    for (uint32_t k = 2; k <= std::max<uint32_t>(kmax, 2); ++k) {
        std::vector<bmq_stage> plan = partition_plan(n, gates, count, block_bits, k);
        double bytes = 0.0;
        uint64_t passes = 0;
        double secs = 0.0;
        for (const bmq_stage& st : plan) {
            const uint32_t p = stage_passes(L, st, gates);
            passes += p;
            // codec trip: payloads read and written, decode's 16 B write and
            // emit's 8 B read of codes; gate passes: 16 B in + 8 B of codes out
            // for the first / last, 32 B for each further pass. Each at the
            // fraction of HBM its kernels reach
            const double codec = amps * (2.0 * cbytes + 24.0), gate = amps * (24.0 + 32.0 * (p - 1));
            bytes += codec + gate;
            secs += codec / (model.codec_eff * model.hbm_gbs * 1e9) + gate / (model.pass_eff * model.hbm_gbs * 1e9);
        }
        secs += plan.size() * model.stage_overhead_s;
        uint32_t remaps = 0;
        if (m && !plan.empty()) {
            // a remap moves the payloads whose owner changes: 1 - 2^-s of this
            // GPU's share for s re-chosen device bits, over the peer link
            const std::vector<uint32_t> dev = shard_plan(L, plan, model.world);
            for (size_t s = 1; s < plan.size(); ++s) {
                uint32_t moved = 0;
                for (uint32_t j = 0; j < m; ++j) moved += dev[s * m + j] != dev[(s - 1) * m + j];
                if (moved) {
                    ++remaps;
                    secs += amps * cbytes * (1.0 - std::ldexp(1.0, -static_cast<int>(moved))) / (model.link_gbs * 1e9);
                }
            }
        }
        if (ch.candidates < 16) {
            ch.inner[ch.candidates] = k;
            ch.model_s[ch.candidates] = secs;
            ++ch.candidates;
        }
        if (best.empty() || secs < best_s) {
            best = std::move(plan);
            best_s = secs;
            ch.inner_size = k;
            ch.stages = best.size();
            ch.passes = passes;
            ch.remaps = remaps;
            ch.model_s_best = secs;
        }
    }
    if (choice) *choice = ch;
    return best;
}

uint64_t GroupGeometry::block_id(uint64_t outer, uint64_t v) const {
    return deposit_bits(outer, outer_mask) | deposit_bits(v, inner_mask);
}

// enumerate_groups geometry (partition.hpp:120-153): inner offsets q - b.
GroupGeometry group_geometry(const Layout& L, const bmq_stage& st) {
    GroupGeometry gg;
    for (uint32_t i = 0; i < st.inner_count; ++i) {
        const uint32_t q = st.inner[i];
        if (q < L.b || q >= L.n)
            raise(BMQ_ERR_INVALID_ARGUMENT,
                  "stage inner index " + std::to_string(q) + " outside the global index range");
        gg.inner_mask |= 1ull << (q - L.b);
    }
    gg.inner_bits = static_cast<uint32_t>(__builtin_popcountll(gg.inner_mask));
    const uint64_t all = L.c >= 64 ? ~0ull : (1ull << L.c) - 1;
    gg.outer_mask = all & ~gg.inner_mask;
    gg.outer_bits = L.c - gg.inner_bits;
    return gg;
}

// buffer_bit_of_qubit (partition.hpp:158-169).
uint32_t buffer_bit(const Layout& L, const bmq_stage& st, uint32_t q) {
    if (q < L.b) return q;
    for (uint32_t i = 0; i < st.inner_count; ++i)
        if (st.inner[i] == q) return L.b + i;
    raise(BMQ_ERR_LOGIC, "qubit " + std::to_string(q) + " is an outer index for this stage");
}

// Device-bit plan for `world` shards. The reference is
// single-node; its stage loop (engine.hpp:109-120) only needs every group of a
// stage on one worker, which holds iff the device bits are outer bits of that
// stage. Slot j of stage s holds the id bit whose value is bit j of the owning
// rank. A slot is only re-chosen when the stage needs its bit as an inner
// bit, and then gets the free bit used furthest in the future (Belady);
// ties go to the highest bit, so the plan is deterministic on every rank.
std::vector<uint32_t> shard_plan(const Layout& L, const std::vector<bmq_stage>& plan, uint32_t world) {
    if (world == 0 || (world & (world - 1))) raise(BMQ_ERR_INVALID_ARGUMENT, "shard count must be a power of two");
    uint32_t m = 0;
    while ((1u << m) < world) ++m;
    const uint64_t ns = plan.size();
    std::vector<uint32_t> out(ns * m);
    if (!m) return out;
    std::vector<uint64_t> inner_mask(ns, 0);
    for (uint64_t s = 0; s < ns; ++s) {
        for (uint32_t i = 0; i < plan[s].inner_count; ++i) inner_mask[s] |= 1ull << (plan[s].inner[i] - L.b);
        if (L.c - plan[s].inner_count < m)
            raise(BMQ_ERR_INVALID_ARGUMENT, "stage " + std::to_string(s) + " leaves " +
                                                std::to_string(L.c - plan[s].inner_count) +
                                                " outer bits, too few for " + std::to_string(world) + " shards");
    }
    const auto next_use = [&](uint32_t bit, uint64_t from) {
        for (uint64_t s = from; s < ns; ++s)
            if (inner_mask[s] >> bit & 1) return s;
        return ns;
    };
    std::vector<uint32_t> slots;
    uint64_t held = 0;
    const auto pick = [&](uint64_t s) {
        uint32_t best = ~0u;
        uint64_t best_use = 0;
        for (uint32_t bit = L.c; bit-- > 0;) {
            if ((inner_mask[s] >> bit & 1) || (held >> bit & 1)) continue;
            const uint64_t u = next_use(bit, s);
            if (best == ~0u || u > best_use) best = bit, best_use = u;
        }
        held |= 1ull << best;
        return best;
    };
    for (uint32_t j = 0; j < m; ++j) slots.push_back(pick(0));
    std::sort(slots.begin(), slots.end());
    for (uint64_t s = 0; s < ns; ++s) {
        for (uint32_t j = 0; j < m; ++j) {
            if (!(inner_mask[s] >> slots[j] & 1)) continue;
            held &= ~(1ull << slots[j]);
            slots[j] = pick(s);
        }
        for (uint32_t j = 0; j < m; ++j) out[s * m + j] = slots[j];
    }
    return out;
}

uint64_t compress_bound(uint64_t n) {
    const uint64_t chunks = (n + 4095) / 4096;
    return 26 + 2 * ((chunks + 3) / 4 + (n + 7) / 8) + (n * 63 + 7) / 8 + 16;
}

}  // namespace bmq
