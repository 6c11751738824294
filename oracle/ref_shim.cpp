// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Exposes the UNMODIFIED reference implementation (header-only C++20 under
// /root/reference/proj/include/cbq, compiled where it lies by oracle/Makefile)
// behind a plain C ABI so the parity tests, smoke() and bench.py's
// cpu_baseline / --impl reference legs can drive it through ctypes.
// Output goes to oracle/_ref/libcbqref.so (git-ignored, travels to the GPU box).
//
// Every entry point below is a thin adapter around a reference symbol:
//   cbqref_compress_block     -> cbq::compress_block        codec.hpp:227-295
//   cbqref_decompress_block   -> cbq::decompress_block      codec.hpp:299-344
//   cbqref_log2_abs           -> cbq::ErrorBound            codec.hpp:19-29
//   cbqref_prescan_encode     -> cbq::prescan_encode        bitmap.hpp:109-145
//   cbqref_unitary            -> cbq::unitary2 / unitary4   circuit.hpp:133-198
//   cbqref_generate_benchmark -> cbq::generate_benchmark    benchmarks.hpp:148-166
//   cbqref_parse_qasm         -> cbq::parse_qasm            qasm.hpp:387-389
//   cbqref_partition          -> cbq::partition_circuit     partition.hpp:59-101
//   cbqref_enumerate_groups   -> cbq::enumerate_groups      partition.hpp:120-153
//   cbqref_apply_stage        -> cbq::apply_stage           kernel.hpp:111-122
//   cbqref_apply_gate         -> cbq::apply_unitary2/4      kernel.hpp:24-64
//   cbqref_simulate           -> cbq::Simulator::run        engine.hpp:97-134
//   cbqref_dense_reference    -> cbq::dense_reference       engine.hpp:254-296
//   cbqref_fidelity           -> cbq::fidelity              engine.hpp:299-308
//   cbqref_group_pipeline     -> the body of Simulator::process_group
//                                (engine.hpp:203-225) rebuilt from the public
//                                BlockStore/codec/kernel API, for bounded
//                                CPU-baseline samples.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "cbq/benchmarks.hpp"
#include "cbq/engine.hpp"
#include "cbq/qasm.hpp"

namespace {

thread_local std::string g_err;

enum : int {
    kOk = 0,
    kInvalidArgument = 1,
    kLogic = 2,
    kCodec = 3,
    kStore = 4,
    kEngine = 5,
    kQasm = 6,
    kBufferTooSmall = 10,
    kOther = 99,
};

struct BufferTooSmall : std::runtime_error {
    using std::runtime_error::runtime_error;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return kOk;
    } catch (const BufferTooSmall& e) {
        g_err = e.what();
        return kBufferTooSmall;
    } catch (const cbq::CodecError& e) {
        g_err = e.what();
        return kCodec;
    } catch (const cbq::StoreError& e) {
        g_err = e.what();
        return kStore;
    } catch (const cbq::EngineError& e) {
        g_err = e.what();
        return kEngine;
    } catch (const cbq::QasmError& e) {
        g_err = e.what();
        return kQasm;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return kInvalidArgument;
    } catch (const std::logic_error& e) {
        g_err = e.what();
        return kLogic;
    } catch (const std::exception& e) {
        g_err = e.what();
        return kOther;
    }
}

}  // namespace

extern "C" {

struct cbqref_gate {
    uint32_t kind, q0, q1, pad;
    double angle;
};

struct cbqref_stage {
    uint64_t gate_begin, gate_end;
    uint32_t inner_count, pad;
    uint32_t inner[64];
};

struct cbqref_report {
    uint64_t qubits, gate_count, stage_count, max_footprint_bytes;
    double standard_bytes, compression_ratio;
    uint64_t spilled_blocks;
    double wall_ms;
    int32_t has_fidelity, pad;
    double fidelity, final_norm;
    uint64_t stage_compress_calls, stage_decompress_calls;
};

}  // extern "C"

namespace {

cbq::Gate to_gate(const cbqref_gate& g) {
    return cbq::Gate{static_cast<cbq::GateKind>(g.kind), g.q0, g.q1, g.angle};
}

cbqref_gate from_gate(const cbq::Gate& g) {
    return cbqref_gate{static_cast<uint32_t>(g.kind), g.q0, g.q1, 0u, g.angle};
}

cbq::Circuit to_circuit(uint32_t n, const cbqref_gate* gates, uint64_t count) {
    cbq::Circuit c(n);
    for (uint64_t i = 0; i < count; ++i) c.add(to_gate(gates[i]));
    return c;
}

cbq::Stage to_stage(const cbqref_stage& s) {
    cbq::Stage st;
    st.gate_begin = s.gate_begin;
    st.gate_end = s.gate_end;
    st.inner.assign(s.inner, s.inner + s.inner_count);
    return st;
}

void put_gates(const cbq::Circuit& c, cbqref_gate* out, uint64_t cap, uint64_t* count) {
    *count = c.gates.size();
    if (c.gates.size() > cap) throw BufferTooSmall("gate buffer too small");
    for (std::size_t i = 0; i < c.gates.size(); ++i) out[i] = from_gate(c.gates[i]);
}

}  // namespace

extern "C" {

const char* cbqref_last_error(void) { return g_err.c_str(); }

int cbqref_log2_abs(double b_r, double* out) {
    return guarded([&] { *out = cbq::ErrorBound(b_r).log2_abs; });
}

int cbqref_compress_block(const double* scalars, uint64_t n, double b_r, uint8_t* out,
                          uint64_t cap, uint64_t* size) {
    return guarded([&] {
        const auto p = cbq::compress_block(std::span<const double>(scalars, n), cbq::ErrorBound(b_r));
        *size = p.size();
        if (p.size() > cap) throw BufferTooSmall("payload buffer too small");
        std::memcpy(out, p.data(), p.size());
    });
}

int cbqref_decompress_block(const uint8_t* payload, uint64_t size, double* out, uint64_t cap,
                            uint64_t* count) {
    return guarded([&] {
        const auto v = cbq::decompress_block(std::span<const uint8_t>(payload, size));
        *count = v.size();
        if (v.size() > cap) throw BufferTooSmall("scalar buffer too small");
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

int cbqref_prescan_encode(const uint64_t* words, uint64_t bit_count, uint8_t* out, uint64_t cap,
                          uint64_t* size) {
    return guarded([&] {
        cbq::Bitmap bm(bit_count);
        for (std::size_t w = 0; w < bm.words().size(); ++w) bm.words()[w] = words[w];
        if (bit_count % 64 && !bm.words().empty())
            bm.words().back() &= (1ull << (bit_count % 64)) - 1;
        const auto pb = cbq::prescan_encode(bm);
        *size = pb.tags.size() + pb.raw.size();
        if (*size > cap) throw BufferTooSmall("prescan buffer too small");
        std::memcpy(out, pb.tags.data(), pb.tags.size());
        std::memcpy(out + pb.tags.size(), pb.raw.data(), pb.raw.size());
    });
}

int cbqref_unitary(const cbqref_gate* g, double* out) {
    return guarded([&] {
        const cbq::Gate gate = to_gate(*g);
        if (cbq::is_two_qubit(gate.kind)) {
            const auto u = cbq::unitary4(gate);
            for (int i = 0; i < 16; ++i) {
                out[2 * i] = u[i].real();
                out[2 * i + 1] = u[i].imag();
            }
        } else {
            const auto u = cbq::unitary2(gate);
            for (int i = 0; i < 4; ++i) {
                out[2 * i] = u[i].real();
                out[2 * i + 1] = u[i].imag();
            }
        }
    });
}

int cbqref_generate_benchmark(const char* name, uint32_t n, uint32_t layers, uint64_t seed,
                              const char* secret, cbqref_gate* out, uint64_t cap,
                              uint64_t* count) {
    return guarded([&] {
        cbq::BenchmarkParams p;
        p.layers = layers;
        p.seed = seed;
        if (secret && *secret) p.secret = std::string(secret);
        const cbq::Circuit c = cbq::generate_benchmark(cbq::benchmark_from_name(name), n, p);
        put_gates(c, out, cap, count);
    });
}

int cbqref_parse_qasm(const char* text, uint32_t* num_qubits, cbqref_gate* out, uint64_t cap,
                      uint64_t* count, uint64_t* warning_count) {
    return guarded([&] {
        std::vector<std::string> warnings;
        const cbq::Circuit c = cbq::parse_qasm(text, &warnings);
        *num_qubits = c.num_qubits;
        if (warning_count) *warning_count = warnings.size();
        put_gates(c, out, cap, count);
    });
}

int cbqref_emit_qasm(uint32_t n, const cbqref_gate* gates, uint64_t ngates, char* out,
                     uint64_t cap, uint64_t* size) {
    return guarded([&] {
        const std::string s = cbq::emit_qasm(to_circuit(n, gates, ngates));
        *size = s.size();
        if (s.size() + 1 > cap) throw BufferTooSmall("text buffer too small");
        std::memcpy(out, s.c_str(), s.size() + 1);
    });
}

int cbqref_partition(uint32_t n, const cbqref_gate* gates, uint64_t ngates, uint32_t block_bits,
                     uint32_t inner_size, cbqref_stage* out, uint64_t cap, uint64_t* nstages) {
    return guarded([&] {
        const auto plan = cbq::partition_circuit(to_circuit(n, gates, ngates), block_bits, inner_size);
        *nstages = plan.stages.size();
        if (plan.stages.size() > cap) throw BufferTooSmall("stage buffer too small");
        for (std::size_t s = 0; s < plan.stages.size(); ++s) {
            const auto& st = plan.stages[s];
            cbqref_stage o{};
            o.gate_begin = st.gate_begin;
            o.gate_end = st.gate_end;
            o.inner_count = static_cast<uint32_t>(st.inner.size());
            for (std::size_t i = 0; i < st.inner.size(); ++i) o.inner[i] = st.inner[i];
            out[s] = o;
        }
    });
}

int cbqref_enumerate_groups(uint32_t n, uint32_t block_bits, const cbqref_stage* stage,
                            uint64_t* ids, uint64_t cap, uint64_t* count) {
    return guarded([&] {
        const auto groups = cbq::enumerate_groups(to_stage(*stage), cbq::make_layout(n, block_bits));
        uint64_t k = 0;
        for (const auto& g : groups) k += g.block_ids.size();
        *count = k;
        if (k > cap) throw BufferTooSmall("id buffer too small");
        k = 0;
        for (const auto& g : groups)
            for (uint64_t id : g.block_ids) ids[k++] = id;
    });
}

int cbqref_buffer_bit_of_qubit(uint32_t n, uint32_t block_bits, const cbqref_stage* stage,
                               uint32_t q, uint32_t* out) {
    return guarded([&] {
        *out = cbq::buffer_bit_of_qubit(to_stage(*stage), cbq::make_layout(n, block_bits), q);
    });
}

int cbqref_apply_stage(double* amps, uint64_t namps, uint32_t n, const cbqref_gate* gates,
                       uint64_t ngates, const cbqref_stage* stage, uint32_t block_bits) {
    return guarded([&] {
        const cbq::Circuit c = to_circuit(n, gates, ngates);
        cbq::GroupBuffer buf;
        buf.amps.resize(namps);
        std::memcpy(buf.amps.data(), amps, namps * sizeof(cbq::Complex));
        cbq::apply_stage(buf, to_stage(*stage), c, cbq::make_layout(n, block_bits));
        std::memcpy(amps, buf.amps.data(), namps * sizeof(cbq::Complex));
    });
}

int cbqref_apply_gate(double* amps, uint64_t namps, const double* u, int two_qubit,
                      uint32_t hi_bit, uint32_t lo_bit) {
    return guarded([&] {
        std::span<cbq::Complex> s(reinterpret_cast<cbq::Complex*>(amps), namps);
        if (two_qubit) {
            cbq::Mat4 m;
            for (int i = 0; i < 16; ++i) m[i] = cbq::Complex(u[2 * i], u[2 * i + 1]);
            cbq::apply_unitary4(s, hi_bit, lo_bit, m);
        } else {
            cbq::Mat2 m;
            for (int i = 0; i < 4; ++i) m[i] = cbq::Complex(u[2 * i], u[2 * i + 1]);
            cbq::apply_unitary2(s, hi_bit, m);
        }
    });
}

// Full Simulator::run. Optional outputs: per-stage wall ms, the final
// payload of every block id (concatenated in id order, sizes in pay_sizes),
// and the dense final state (interleaved re/im) plus dense-reference fidelity.
int cbqref_simulate(uint32_t n, const cbqref_gate* gates, uint64_t ngates, uint32_t block_bits,
                    uint32_t inner_size, double error_bound, uint64_t memory_budget,
                    uint32_t workers, int compress, const char* spill_dir, cbqref_report* rep,
                    double* stage_ms, uint64_t stage_cap, uint8_t* payloads, uint64_t pay_cap,
                    uint64_t* pay_sizes, double* state, int with_fidelity) {
    return guarded([&] {
        const cbq::Circuit c = to_circuit(n, gates, ngates);
        cbq::Config cfg;
        cfg.block_bits = block_bits;
        cfg.inner_size = inner_size;
        cfg.error_bound = error_bound;
        cfg.memory_budget = memory_budget;
        if (workers) cfg.workers = workers;
        cfg.compress = compress != 0;
        if (spill_dir && *spill_dir) cfg.spill_dir = spill_dir;
        cbq::Simulator sim(c, cfg);
        cbq::SimulationReport r = sim.run();
        if (with_fidelity) {
            const auto ideal = cbq::dense_reference(c, cfg.verify_cap_qubits);
            const auto got = sim.extract_state();
            r.fidelity = cbq::fidelity(ideal, got);
        }
        cbqref_report o{};
        o.qubits = r.qubits;
        o.gate_count = r.gate_count;
        o.stage_count = r.stage_count;
        o.max_footprint_bytes = r.max_footprint_bytes;
        o.standard_bytes = r.standard_bytes;
        o.compression_ratio = r.compression_ratio;
        o.spilled_blocks = r.spilled_blocks;
        o.wall_ms = r.wall_ms;
        o.has_fidelity = r.fidelity.has_value();
        o.fidelity = r.fidelity.value_or(0.0);
        o.final_norm = r.final_norm;
        o.stage_compress_calls = r.stage_compress_calls;
        o.stage_decompress_calls = r.stage_decompress_calls;
        *rep = o;
        if (stage_ms)
            for (std::size_t s = 0; s < r.stage_ms.size() && s < stage_cap; ++s) stage_ms[s] = r.stage_ms[s];
        if (pay_sizes) {
            uint64_t off = 0;
            for (uint64_t id = 0; id < sim.layout().num_blocks(); ++id) {
                const auto p = sim.store().get(id);
                pay_sizes[id] = p.size();
                if (payloads) {
                    if (off + p.size() > pay_cap) throw BufferTooSmall("payload buffer too small");
                    std::memcpy(payloads + off, p.data(), p.size());
                }
                off += p.size();
            }
        }
        if (state) {
            const auto st = sim.extract_state();
            std::memcpy(state, st.data(), st.size() * sizeof(cbq::Complex));
        }
    });
}

int cbqref_dense_reference(uint32_t n, const cbqref_gate* gates, uint64_t ngates, double* out) {
    return guarded([&] {
        const auto st = cbq::dense_reference(to_circuit(n, gates, ngates), 30);
        std::memcpy(out, st.data(), st.size() * sizeof(cbq::Complex));
    });
}

int cbqref_fidelity(const double* a, const double* b, uint64_t namps, double* out) {
    return guarded([&] {
        *out = cbq::fidelity(std::span<const cbq::Complex>(reinterpret_cast<const cbq::Complex*>(a), namps),
                             std::span<const cbq::Complex>(reinterpret_cast<const cbq::Complex*>(b), namps));
    });
}

// One bounded CPU-baseline sample: the reference's per-group pipeline
// (BlockStore::get -> decompress_block -> assemble_group_buffer -> apply_stage
// -> split_buffer -> compress_block -> BlockStore::put, engine.hpp:203-225) for
// `ngroups` groups of one stage, run on `workers` threads with the reference's
// own parallel_for (parallel.hpp:16-64). Input payloads are supplied by the
// caller (one per block id of the sampled groups, `group_ids` row-major:
// ngroups x 2^|inner|). Returns the wall milliseconds of the parallel region.
int cbqref_group_pipeline(uint32_t n, const cbqref_gate* gates, uint64_t ngates,
                          const cbqref_stage* stage, uint32_t block_bits, double error_bound,
                          uint32_t workers, const uint64_t* group_ids, uint64_t ngroups,
                          const uint8_t* payloads, const uint64_t* pay_offsets,
                          const uint64_t* pay_sizes, double* wall_ms, uint64_t* out_bytes) {
    return guarded([&] {
        const cbq::Circuit c = to_circuit(n, gates, ngates);
        const cbq::Layout layout = cbq::make_layout(n, block_bits);
        const cbq::Stage st = to_stage(*stage);
        const cbq::ErrorBound bound(error_bound);
        const uint64_t per = 1ull << st.inner.size();
        cbq::BlockStore store;
        for (uint64_t g = 0; g < ngroups; ++g)
            for (uint64_t v = 0; v < per; ++v) {
                const uint64_t k = g * per + v;
                store.put(group_ids[k], std::vector<uint8_t>(payloads + pay_offsets[k],
                                                             payloads + pay_offsets[k] + pay_sizes[k]));
            }
        const uint64_t bs = layout.block_size();
        const auto t0 = std::chrono::steady_clock::now();
        cbq::parallel_for(workers, ngroups, [&](std::size_t gi) {
            cbq::SVGroup grp;
            grp.outer_value = gi;
            std::vector<cbq::SVBlock> blocks;
            for (uint64_t v = 0; v < per; ++v) {
                const uint64_t id = group_ids[gi * per + v];
                grp.block_ids.push_back(id);
                const auto scal = cbq::decompress_block(store.get(id));
                cbq::SVBlock b(bs);
                for (uint64_t i = 0; i < bs; ++i) b[i] = cbq::Complex(scal[i], scal[bs + i]);
                blocks.push_back(std::move(b));
            }
            cbq::GroupBuffer buf = cbq::assemble_group_buffer(grp, blocks);
            cbq::apply_stage(buf, st, c, layout);
            const auto out = cbq::split_buffer(buf, layout.b);
            for (std::size_t j = 0; j < out.size(); ++j) {
                std::vector<double> scal(2 * bs);
                for (uint64_t i = 0; i < bs; ++i) {
                    scal[i] = out[j][i].real();
                    scal[bs + i] = out[j][i].imag();
                }
                store.put(grp.block_ids[j], cbq::compress_block(scal, bound));
            }
        });
        *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (out_bytes) *out_bytes = store.footprint().resident_bytes;
    });
}


// Stratified CPU-baseline sample across a whole plan: group gi runs the
// reference per-group pipeline (as cbqref_group_pipeline) for stage
// stages[group_stage[gi]], on `workers` threads of the reference's own
// parallel_for. group_ids / payloads are row-major over the sampled groups,
// each group holding 2^|inner| ids of its own stage (offsets in id_first).
// group_ms[gi] receives the thread time of group gi, *wall_ms the wall time
// of the whole parallel region.
int cbqref_stage_groups(uint32_t n, const cbqref_gate* gates, uint64_t ngates, const cbqref_stage* stages,
                        uint64_t nstages, uint32_t block_bits, double error_bound, uint32_t workers,
                        const uint64_t* group_stage, const uint64_t* id_first, uint64_t ngroups,
                        const uint64_t* group_ids, const uint8_t* payloads, const uint64_t* pay_offsets,
                        const uint64_t* pay_sizes, double* group_ms, double* wall_ms) {
    return guarded([&] {
        const cbq::Circuit c = to_circuit(n, gates, ngates);
        const cbq::Layout layout = cbq::make_layout(n, block_bits);
        const cbq::ErrorBound bound(error_bound);
        std::vector<cbq::Stage> st(nstages);
        for (uint64_t s = 0; s < nstages; ++s) st[s] = to_stage(stages[s]);
        // one store per group: sampled groups of different stages may share ids
        std::vector<cbq::BlockStore> stores(ngroups);
        for (uint64_t g = 0; g < ngroups; ++g) {
            const uint64_t per = 1ull << st[group_stage[g]].inner.size();
            for (uint64_t v = 0; v < per; ++v) {
                const uint64_t k = id_first[g] + v;
                stores[g].put(group_ids[k], std::vector<uint8_t>(payloads + pay_offsets[k],
                                                                 payloads + pay_offsets[k] + pay_sizes[k]));
            }
        }
        const uint64_t bs = layout.block_size();
        const auto t0 = std::chrono::steady_clock::now();
        cbq::parallel_for(workers, ngroups, [&](std::size_t gi) {
            const auto g0 = std::chrono::steady_clock::now();
            const cbq::Stage& stage = st[group_stage[gi]];
            const uint64_t per = 1ull << stage.inner.size();
            cbq::BlockStore& store = stores[gi];
            cbq::SVGroup grp;
            grp.outer_value = gi;
            std::vector<cbq::SVBlock> blocks;
            for (uint64_t v = 0; v < per; ++v) {
                const uint64_t id = group_ids[id_first[gi] + v];
                grp.block_ids.push_back(id);
                const auto scal = cbq::decompress_block(store.get(id));
                cbq::SVBlock b(bs);
                for (uint64_t i = 0; i < bs; ++i) b[i] = cbq::Complex(scal[i], scal[bs + i]);
                blocks.push_back(std::move(b));
            }
            cbq::GroupBuffer buf = cbq::assemble_group_buffer(grp, blocks);
            cbq::apply_stage(buf, stage, c, layout);
            const auto out = cbq::split_buffer(buf, layout.b);
            for (std::size_t j = 0; j < out.size(); ++j) {
                std::vector<double> scal(2 * bs);
                for (uint64_t i = 0; i < bs; ++i) {
                    scal[i] = out[j][i].real();
                    scal[bs + i] = out[j][i].imag();
                }
                store.put(grp.block_ids[j], cbq::compress_block(scal, bound));
            }
            group_ms[gi] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - g0).count();
        });
        *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    });
}

}  // extern "C"
