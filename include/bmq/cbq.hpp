// bmq/cbq.hpp — C++ drop-in surface for the reference's `namespace cbq`
// (/root/reference/proj/include/cbq), backed by libbmq.so (include/bmq.h).
//
// A reference user replaces
//     #include "cbq/engine.hpp"   (and codec.hpp, partition.hpp, ...)
// with
//     #include "bmq/cbq.hpp"
// and links -lbmq. Types, function names, argument meaning and exception
// types follow the reference; Simulator::run executes on the B200.
#pragma once

#include <algorithm>
#include <array>
#include <bit>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

#include "bmq.h"

namespace cbq {

using Complex = std::complex<double>;
using Mat2 = std::array<Complex, 4>;
using Mat4 = std::array<Complex, 16>;

// -------------------------------------------------------------- exceptions
class CodecError : public std::runtime_error {  // bitmap.hpp:14-17
public:
    using std::runtime_error::runtime_error;
};
class StoreError : public std::runtime_error {  // store.hpp:23-26
public:
    using std::runtime_error::runtime_error;
};
class EngineError : public std::runtime_error {  // engine.hpp:18-21
public:
    using std::runtime_error::runtime_error;
};
class DeviceError : public std::runtime_error {  // CUDA / no device (new)
public:
    using std::runtime_error::runtime_error;
};
class QasmError : public std::runtime_error {  // qasm.hpp:17-31
public:
    QasmError(int line, int col, const std::string& msg)
        : std::runtime_error("line " + std::to_string(line) + ", col " + std::to_string(col) + ": " + msg),
          line_(line),
          col_(col) {}
    int line() const { return line_; }
    int col() const { return col_; }

private:
    int line_;
    int col_;
};

namespace detail {
[[noreturn]] inline void rethrow(int rc) {
    const std::string msg = bmq_last_error();
    switch (rc) {
    case BMQ_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case BMQ_ERR_LOGIC: throw std::logic_error(msg);
    case BMQ_ERR_CODEC: throw CodecError(msg);
    case BMQ_ERR_STORE: throw StoreError(msg);
    case BMQ_ERR_ENGINE: throw EngineError(msg);
    case BMQ_ERR_QASM: {  // "line L, col C: what" (qasm.hpp:20-22)
        int line = 0, col = 0, used = 0;
        if (std::sscanf(msg.c_str(), "line %d, col %d: %n", &line, &col, &used) == 2 && used > 0)
            throw QasmError(line, col, msg.substr(static_cast<std::size_t>(used)));
        throw QasmError(0, 0, msg);
    }
    default: throw DeviceError(msg);
    }
}
inline void check(int rc) {
    if (rc != BMQ_OK) rethrow(rc);
}
}  // namespace detail

// ----------------------------------------------------------------- circuit
enum class GateKind : std::uint8_t { H, X, Y, Z, S, Sdg, T, Tdg, RX, RY, RZ, P, CX, CZ, CP };

constexpr bool is_two_qubit(GateKind k) { return k == GateKind::CX || k == GateKind::CZ || k == GateKind::CP; }

struct Gate {  // circuit.hpp:65-72
    GateKind kind{};
    std::uint32_t q0 = 0;
    std::uint32_t q1 = 0;
    double angle = 0.0;
    bool operator==(const Gate&) const = default;
    bmq_gate c() const { return bmq_gate{static_cast<uint32_t>(kind), q0, is_two_qubit(kind) ? q1 : 0u, 0u, angle}; }
};

struct Circuit {  // circuit.hpp:97-130
    std::uint32_t num_qubits = 1;
    std::vector<Gate> gates;
    Circuit() = default;
    explicit Circuit(std::uint32_t n) : num_qubits(n) { detail::check(bmq_circuit_validate(n, nullptr, 0)); }
    void add(const Gate& g) {
        const bmq_gate cg = g.c();
        detail::check(bmq_circuit_validate(num_qubits, &cg, 1));
        gates.push_back(g);
    }
    std::vector<bmq_gate> c_gates() const {
        std::vector<bmq_gate> v;
        v.reserve(gates.size());
        for (const Gate& g : gates) v.push_back(g.c());
        return v;
    }
    bool operator==(const Circuit&) const = default;
};

inline Mat2 unitary2(const Gate& g) {  // circuit.hpp:133-170
    if (is_two_qubit(g.kind)) throw std::logic_error("unitary2 called on a two-qubit gate");
    const bmq_gate cg = g.c();
    double m[32];
    detail::check(bmq_gate_unitary(&cg, m));
    Mat2 u;
    for (int i = 0; i < 4; ++i) u[i] = Complex(m[2 * i], m[2 * i + 1]);
    return u;
}

inline Mat4 unitary4(const Gate& g) {  // circuit.hpp:174-198
    if (!is_two_qubit(g.kind)) throw std::logic_error("unitary4 called on a single-qubit gate");
    const bmq_gate cg = g.c();
    double m[32];
    detail::check(bmq_gate_unitary(&cg, m));
    Mat4 u;
    for (int i = 0; i < 16; ++i) u[i] = Complex(m[2 * i], m[2 * i + 1]);
    return u;
}

enum class Benchmark { Ghz, CatState, Bv, Qft, Qaoa };

struct BenchmarkParams {  // benchmarks.hpp:24-28
    std::uint32_t layers = 1;
    std::optional<std::string> secret;
    std::uint64_t seed = 1;
};

inline Circuit generate_benchmark(Benchmark b, std::uint32_t n, const BenchmarkParams& p = {}) {
    static const char* names[] = {"ghz", "cat_state", "bv", "qft", "qaoa"};
    const char* name = names[static_cast<int>(b)];
    const std::string secret = p.secret.value_or("");
    std::uint64_t count = 0;
    int rc = bmq_generate_benchmark(name, n, p.layers, p.seed, secret.c_str(), nullptr, 0, &count);
    if (rc != BMQ_OK && rc != BMQ_ERR_BUFFER_TOO_SMALL) detail::rethrow(rc);
    std::vector<bmq_gate> v(count);
    detail::check(bmq_generate_benchmark(name, n, p.layers, p.seed, secret.c_str(), v.data(), count, &count));
    Circuit c(n);
    for (const bmq_gate& g : v) c.gates.push_back(Gate{static_cast<GateKind>(g.kind), g.q0, g.q1, g.angle});
    return c;
}

// -------------------------------------------------------------------- qasm
// parse_qasm (qasm.hpp:387-389): OPENQASM 2.0 subset; warnings (ignored
// measure) are appended to *warnings. Errors throw QasmError(line, col).
inline Circuit parse_qasm(std::string_view text, std::vector<std::string>* warnings = nullptr) {
    const std::string t(text);
    std::uint32_t n = 0;
    std::uint64_t count = 0, nw = 0;
    int rc = bmq_parse_qasm(t.c_str(), &n, nullptr, 0, &count, nullptr, 0, &nw);
    if (rc != BMQ_OK && rc != BMQ_ERR_BUFFER_TOO_SMALL) detail::rethrow(rc);
    std::vector<bmq_gate> v(std::max<std::uint64_t>(count, 1));
    std::string w(4096 + 256 * nw, '\0');
    detail::check(bmq_parse_qasm(t.c_str(), &n, v.data(), v.size(), &count, w.data(), w.size(), &nw));
    Circuit c(n);
    for (std::uint64_t i = 0; i < count; ++i)
        c.gates.push_back(Gate{static_cast<GateKind>(v[i].kind), v[i].q0, v[i].q1, v[i].angle});
    if (warnings && nw) {
        w.resize(std::strlen(w.c_str()));
        std::size_t pos = 0;
        for (std::uint64_t k = 0; k < nw; ++k) {
            const std::size_t e = w.find('\n', pos);
            warnings->push_back(w.substr(pos, e == std::string::npos ? std::string::npos : e - pos));
            if (e == std::string::npos) break;
            pos = e + 1;
        }
    }
    return c;
}

// emit_qasm (qasm.hpp:392-411): parse_qasm(emit_qasm(c)) == c.
inline std::string emit_qasm(const Circuit& circuit) {
    const auto g = circuit.c_gates();
    std::uint64_t size = 0;
    int rc = bmq_emit_qasm(circuit.num_qubits, g.data(), g.size(), nullptr, 0, &size);
    if (rc != BMQ_OK && rc != BMQ_ERR_BUFFER_TOO_SMALL) detail::rethrow(rc);
    std::string out(size + 1, '\0');
    detail::check(bmq_emit_qasm(circuit.num_qubits, g.data(), g.size(), out.data(), out.size(), &size));
    out.resize(size);
    return out;
}

// --------------------------------------------------------------- partition
struct Layout {  // partition.hpp:14-21
    std::uint32_t n = 1, b = 1, c = 0;
    std::uint64_t num_blocks() const { return 1ull << c; }
    std::uint64_t block_size() const { return 1ull << b; }
};

inline Layout make_layout(std::uint32_t n, std::uint32_t b) {
    if (n < 1 || n > 62) throw std::invalid_argument("layout qubit count must be in [1, 62]");
    if (b < 1 || b > n) throw std::invalid_argument("local index bits must be in [1, n]");
    return Layout{n, b, n - b};
}

struct Stage {  // partition.hpp:36-40
    std::size_t gate_begin = 0, gate_end = 0;
    std::vector<std::uint32_t> inner;
    bmq_stage c() const {
        bmq_stage s{};
        s.gate_begin = gate_begin;
        s.gate_end = gate_end;
        s.inner_count = static_cast<uint32_t>(inner.size());
        for (std::size_t i = 0; i < inner.size(); ++i) s.inner[i] = inner[i];
        return s;
    }
};

struct PartitionPlan {  // partition.hpp:42-46
    Layout layout;
    std::uint32_t inner_size = 0;
    std::vector<Stage> stages;
};

struct SVGroup {  // partition.hpp:50-53
    std::uint64_t outer_value = 0;
    std::vector<std::uint64_t> block_ids;
};

inline PartitionPlan partition_circuit(const Circuit& c, std::uint32_t block_bits, std::uint32_t inner_size) {
    const auto g = c.c_gates();
    std::vector<bmq_stage> out(std::max<std::size_t>(1, g.size()));
    std::uint64_t ns = 0;
    detail::check(bmq_partition(c.num_qubits, g.data(), g.size(), block_bits, inner_size, out.data(), out.size(), &ns));
    PartitionPlan plan{make_layout(c.num_qubits, block_bits), inner_size, {}};
    for (std::uint64_t i = 0; i < ns; ++i)
        plan.stages.push_back(Stage{out[i].gate_begin, out[i].gate_end,
                                    std::vector<std::uint32_t>(out[i].inner, out[i].inner + out[i].inner_count)});
    return plan;
}

inline std::vector<SVGroup> enumerate_groups(const Stage& stage, const Layout& layout) {
    const bmq_stage s = stage.c();
    std::vector<std::uint64_t> ids(layout.num_blocks());
    std::uint64_t count = 0;
    detail::check(bmq_enumerate_groups(layout.n, layout.b, &s, ids.data(), ids.size(), &count));
    const std::uint64_t per = 1ull << stage.inner.size();
    std::vector<SVGroup> groups(count / per);
    for (std::uint64_t o = 0; o < groups.size(); ++o) {
        groups[o].outer_value = o;
        groups[o].block_ids.assign(ids.begin() + o * per, ids.begin() + (o + 1) * per);
    }
    return groups;
}

inline std::uint32_t buffer_bit_of_qubit(const Stage& stage, const Layout& layout, std::uint32_t q) {
    const bmq_stage s = stage.c();
    std::uint32_t bit = 0;
    detail::check(bmq_buffer_bit_of_qubit(layout.n, layout.b, &s, q, &bit));
    return bit;
}

// ------------------------------------------------------------------ kernel
// kernel.hpp:14-122. Gate application runs on the B200 (bmq_apply_gate /
// bmq_apply_stage copy the caller's buffer to the device and back) with the
// reference's arithmetic, so results are bit-identical to the CPU kernels.
using SVBlock = std::vector<Complex>;

struct GroupBuffer {  // kernel.hpp:16-19
    SVGroup group;
    std::vector<Complex> amps;
};

inline void apply_unitary2(std::span<Complex> amps, std::uint32_t bit, const Mat2& u) {  // kernel.hpp:24-38
    double m[8];
    for (int i = 0; i < 4; ++i) {
        m[2 * i] = u[i].real();
        m[2 * i + 1] = u[i].imag();
    }
    detail::check(bmq_apply_gate(reinterpret_cast<double*>(amps.data()), amps.size(), m, 0, bit, 0));
}

inline void apply_unitary4(std::span<Complex> amps, std::uint32_t hi_bit, std::uint32_t lo_bit,
                           const Mat4& u) {  // kernel.hpp:42-64
    double m[32];
    for (int i = 0; i < 16; ++i) {
        m[2 * i] = u[i].real();
        m[2 * i + 1] = u[i].imag();
    }
    detail::check(bmq_apply_gate(reinterpret_cast<double*>(amps.data()), amps.size(), m, 1, hi_bit, lo_bit));
}

inline GroupBuffer assemble_group_buffer(SVGroup group, const std::vector<SVBlock>& blocks) {  // kernel.hpp:66-84
    if (blocks.empty() || !std::has_single_bit(blocks.size()))
        throw std::invalid_argument("group block count must be a nonzero power of two");
    if (blocks.size() != group.block_ids.size()) throw std::invalid_argument("block list does not match the group");
    const std::size_t block_size = blocks.front().size();
    GroupBuffer buf;
    buf.amps.reserve(block_size * blocks.size());
    for (const SVBlock& blk : blocks) {
        if (blk.size() != block_size) throw std::invalid_argument("group blocks must have equal length");
        buf.amps.insert(buf.amps.end(), blk.begin(), blk.end());
    }
    buf.group = std::move(group);
    return buf;
}

inline std::vector<SVBlock> split_buffer(const GroupBuffer& buf, std::uint32_t block_bits) {  // kernel.hpp:87-98
    const std::uint64_t block_size = 1ull << block_bits;
    if (buf.amps.size() % block_size != 0)
        throw std::invalid_argument("buffer length not divisible by the block size");
    std::vector<SVBlock> blocks;
    blocks.reserve(buf.amps.size() / block_size);
    for (std::size_t off = 0; off < buf.amps.size(); off += block_size)
        blocks.emplace_back(buf.amps.begin() + static_cast<std::ptrdiff_t>(off),
                            buf.amps.begin() + static_cast<std::ptrdiff_t>(off + block_size));
    return blocks;
}

inline void apply_gate(GroupBuffer& buf, const Mat2& u, std::uint32_t bit) { apply_unitary2(buf.amps, bit, u); }
inline void apply_gate(GroupBuffer& buf, const Mat4& u, std::uint32_t hi_bit, std::uint32_t lo_bit) {
    apply_unitary4(buf.amps, hi_bit, lo_bit, u);
}

// apply_stage (kernel.hpp:111-122): the stage's gates in program order, outer
// operands refused with the reference's logic_error.
inline void apply_stage(GroupBuffer& buf, const Stage& stage, const Circuit& circuit, const Layout& layout) {
    const auto g = circuit.c_gates();
    const bmq_stage s = stage.c();
    detail::check(bmq_apply_stage(reinterpret_cast<double*>(buf.amps.data()), buf.amps.size(), circuit.num_qubits,
                                  g.data(), g.size(), &s, layout.b));
}

// ------------------------------------------------------------------- codec
struct ErrorBound {  // codec.hpp:19-29
    double relative;
    double log2_abs;
    explicit ErrorBound(double b_r) : relative(b_r), log2_abs(0.0) { detail::check(bmq_error_bound(b_r, &log2_abs)); }
};

inline std::vector<std::uint8_t> compress_block(std::span<const double> scalars, const ErrorBound& bound) {
    std::vector<std::uint8_t> out(bmq_compress_bound(scalars.size()));
    std::uint64_t size = 0;
    detail::check(bmq_compress_blocks(scalars.data(), 1, scalars.size(), bound.relative, out.data(), out.size(), &size));
    out.resize(size);
    return out;
}

inline std::vector<double> decompress_block(std::span<const std::uint8_t> payload) {
    const std::uint64_t off = 0, size = payload.size();
    std::uint64_t count = 0;
    double dummy = 0.0;
    int rc = bmq_decompress_blocks(payload.data(), &off, &size, 1, &dummy, 0, &count);
    if (rc != BMQ_OK && rc != BMQ_ERR_BUFFER_TOO_SMALL) detail::rethrow(rc);
    std::vector<double> out(count);
    if (count) detail::check(bmq_decompress_blocks(payload.data(), &off, &size, 1, out.data(), count, &count));
    return out;
}

// ------------------------------------------------------------------ engine
inline constexpr std::uint64_t kUnlimitedBudget = std::numeric_limits<std::uint64_t>::max();

struct Config {  // engine.hpp:23-37 (+ device knobs)
    std::uint32_t block_bits = 1;
    std::uint32_t inner_size = 2;
    double error_bound = 1e-3;
    std::uint64_t memory_budget = kUnlimitedBudget;
    unsigned workers = 1;
    bool compress = true;
    std::uint32_t verify_cap_qubits = 24;
    int device = 0;
    // device-side knobs (bmq_config)
    bool identity_skip = false;
    bool zero_group_skip = true;
    bool code_domain = true;
    bool pool_grow = false;
    bool fuse_stages = true;  // BMQ_FLAG_STAGE_FUSION (same payloads, fewer codec trips)
    enum class Arena { Auto, Heap, Bump } arena = Arena::Auto;  // device arena placement (BMQ_FLAG_*_ARENA)
    std::uint64_t device_pool_bytes = 0;  // 0 = automatic
    std::uint64_t work_bytes = 0;         // 0 = automatic
    std::uint64_t host_pool_bytes = 0;    // pinned host level of the store; 0 = none
    std::uint64_t disk_pool_bytes = 0;    // disk level beneath it (spill file); 0 = none
    std::string disk_dir;                 // spill file directory ("" = /tmp)
    bmq_config c() const {
        bmq_config k;
        bmq_config_default(&k);
        k.block_bits = block_bits;
        k.inner_size = inner_size;
        k.error_bound = error_bound;
        k.memory_budget = memory_budget;
        k.workers = workers;
        k.compress = compress ? 1u : 0u;
        k.verify_cap_qubits = verify_cap_qubits;
        k.device = device;
        k.device_pool_bytes = device_pool_bytes;
        k.work_bytes = work_bytes;
        k.host_pool_bytes = host_pool_bytes;
        k.disk_pool_bytes = disk_pool_bytes;
        k.disk_dir = disk_dir.empty() ? nullptr : disk_dir.c_str();
        k.flags = (zero_group_skip ? BMQ_FLAG_ZERO_GROUP_SKIP : 0u) | (identity_skip ? BMQ_FLAG_IDENTITY_SKIP : 0u) |
                  (code_domain ? BMQ_FLAG_CODE_DOMAIN : 0u) | (pool_grow ? BMQ_FLAG_POOL_GROW : 0u) |
                  (arena == Arena::Heap ? BMQ_FLAG_HEAP_ARENA : 0u) | (arena == Arena::Bump ? BMQ_FLAG_BUMP_ARENA : 0u) |
                  (fuse_stages ? BMQ_FLAG_STAGE_FUSION : 0u);
        return k;
    }
};

struct Footprint {  // store.hpp:30-35
    std::uint64_t resident_bytes = 0;
    std::uint64_t spilled_live_bytes = 0;
    std::uint64_t peak_bytes = 0;
};

struct SimulationReport {  // engine.hpp:39-53
    std::uint64_t qubits = 0, gate_count = 0, stage_count = 0, max_footprint_bytes = 0;
    double standard_bytes = 0.0, compression_ratio = 0.0;
    std::uint64_t spilled_blocks = 0;
    double wall_ms = 0.0;
    std::vector<double> stage_ms;
    std::optional<double> fidelity;
    double final_norm = 0.0;
    std::uint64_t stage_compress_calls = 0, stage_decompress_calls = 0;
    bmq_report device{};
};

class Simulator {  // engine.hpp:58-250
public:
    // BlockStore view (store.hpp:47-300): exact payload bytes per id and the
    // replayed footprint; the payloads themselves live in the device pool.
    class StoreView {
    public:
        explicit StoreView(bmq_simulator* s) : s_(s) {}
        std::vector<std::uint8_t> get(std::uint64_t id) const {
            std::uint64_t size = 0;
            detail::check(bmq_simulator_get_payload(s_, id, nullptr, 0, &size));
            std::vector<std::uint8_t> out(size);
            detail::check(bmq_simulator_get_payload(s_, id, out.data(), out.size(), &size));
            return out;
        }
        Footprint footprint() const {
            Footprint f;
            detail::check(bmq_simulator_footprint(s_, &f.resident_bytes, &f.spilled_live_bytes, &f.peak_bytes));
            return f;
        }

    private:
        bmq_simulator* s_;
    };

    Simulator(Circuit circuit, Config config) : circuit_(std::move(circuit)), config_(config) {
        const bmq_config c = config_.c();
        const auto g = circuit_.c_gates();
        detail::check(bmq_simulator_create(circuit_.num_qubits, g.data(), g.size(), &c, &sim_));
    }
    Simulator(const Simulator&) = delete;
    Simulator& operator=(const Simulator&) = delete;
    ~Simulator() { bmq_simulator_destroy(sim_); }

    void init_state() { detail::check(bmq_simulator_init_state(sim_)); }

    SimulationReport run() { return run_on(nullptr); }

    // One rank of a sharded run (bmq_simulator_run_sharded): every rank
    // calls it with its own simulator; norm, counters and peak are global.
    SimulationReport run_sharded(bmq_collective* col) { return run_on(col); }

private:
    SimulationReport run_on(bmq_collective* col) {
        bmq_report r{};
        std::vector<double> stage_ms(std::max<std::size_t>(1, circuit_.gates.size()));
        if (col)
            detail::check(bmq_simulator_run_sharded(sim_, col, &r, stage_ms.data(), stage_ms.size()));
        else
            detail::check(bmq_simulator_run(sim_, &r, stage_ms.data(), stage_ms.size()));
        SimulationReport out;
        out.qubits = r.qubits;
        out.gate_count = r.gate_count;
        out.stage_count = r.stage_count;
        out.max_footprint_bytes = r.max_footprint_bytes;
        out.standard_bytes = r.standard_bytes;
        out.compression_ratio = r.compression_ratio;
        out.spilled_blocks = r.spilled_blocks;
        out.wall_ms = r.wall_ms;
        out.stage_ms.assign(stage_ms.begin(), stage_ms.begin() + static_cast<std::ptrdiff_t>(r.stage_count));
        out.final_norm = r.final_norm;
        out.stage_compress_calls = r.stage_compress_calls;
        out.stage_decompress_calls = r.stage_decompress_calls;
        out.device = r;
        return out;
    }

public:
    std::vector<Complex> extract_state() const {
        std::vector<Complex> st(1ull << circuit_.num_qubits);
        detail::check(bmq_simulator_extract_state(sim_, reinterpret_cast<double*>(st.data()), st.size()));
        return st;
    }

    double state_norm() const {
        double n = 0.0;
        detail::check(bmq_simulator_state_norm(sim_, &n));
        return n;
    }

    Complex amplitude(std::uint64_t index) const {
        double re = 0.0, im = 0.0;
        detail::check(bmq_simulator_amplitude(sim_, index, &re, &im));
        return {re, im};
    }
    // Sampling / top-k queries (bmq_simulator_sample / _top_k; beyond the
    // reference, whose only state query is the dense extract_state).
    std::vector<std::uint64_t> sample(std::uint64_t shots, std::uint64_t seed = 1) {
        std::vector<std::uint64_t> out(shots);
        detail::check(bmq_simulator_sample(sim_, shots, seed, out.data()));
        return out;
    }
    std::vector<std::pair<std::uint64_t, Complex>> top_k(std::uint64_t k) {
        std::vector<std::uint64_t> idx(k);
        std::vector<double> re(k), im(k);
        std::uint64_t n = 0;
        detail::check(bmq_simulator_top_k(sim_, k, idx.data(), re.data(), im.data(), &n));
        std::vector<std::pair<std::uint64_t, Complex>> out;
        for (std::uint64_t i = 0; i < n; ++i) out.emplace_back(idx[i], Complex(re[i], im[i]));
        return out;
    }

    std::vector<std::uint8_t> get_payload(std::uint64_t id) const {  // store().get(id)
        std::uint64_t size = 0;
        detail::check(bmq_simulator_get_payload(sim_, id, nullptr, 0, &size));
        std::vector<std::uint8_t> out(size);
        detail::check(bmq_simulator_get_payload(sim_, id, out.data(), out.size(), &size));
        return out;
    }

    void put_payload(std::uint64_t id, std::span<const std::uint8_t> p) {  // store().put(id, p)
        detail::check(bmq_simulator_put_payload(sim_, id, p.data(), p.size()));
    }

    // Stage-level driving and checkpoint / resume (new: the reference keeps
    // no persisted index, store.hpp:36-46).
    void run_stages(std::uint64_t first, std::uint64_t last) {
        detail::check(bmq_simulator_run_stages(sim_, first, last));
    }
    void save(const std::string& path) const { detail::check(bmq_simulator_save(sim_, path.c_str())); }
    std::uint64_t load(const std::string& path) {  // returns the next stage to run
        std::uint64_t next = 0;
        detail::check(bmq_simulator_load(sim_, path.c_str(), &next));
        return next;
    }

    StoreView store() const { return StoreView(sim_); }
    Layout layout() const { return make_layout(circuit_.num_qubits, config_.block_bits); }
    PartitionPlan plan() const { return partition_circuit(circuit_, config_.block_bits, config_.inner_size); }

private:
    mutable bmq_simulator* sim_ = nullptr;
    Circuit circuit_;
    Config config_;
};

inline std::vector<Complex> dense_reference(const Circuit& c, std::uint32_t verify_cap_qubits = 24) {
    if (c.num_qubits > verify_cap_qubits)
        throw EngineError("dense reference refused: " + std::to_string(c.num_qubits) +
                          " qubits exceeds the cap of " + std::to_string(verify_cap_qubits));
    std::vector<Complex> st(1ull << c.num_qubits);
    const auto g = c.c_gates();
    detail::check(bmq_dense_reference(c.num_qubits, g.data(), g.size(), reinterpret_cast<double*>(st.data()),
                                      verify_cap_qubits));
    return st;
}

// fidelity (engine.hpp:299-308): |<a|b>|, conjugate-linear in a.
inline double fidelity(std::span<const Complex> a, std::span<const Complex> b) {
    if (a.size() != b.size()) throw std::invalid_argument("fidelity requires equal-length states");
    double f = 0.0;
    detail::check(bmq_fidelity(reinterpret_cast<const double*>(a.data()), reinterpret_cast<const double*>(b.data()),
                               a.size(), &f));
    return f;
}

}  // namespace cbq
