// capi.cpp — the extern "C" boundary (include/bmq.h). Every entry point
// converts exceptions into a bmq_status plus a thread-local message carrying
// the reference's exception text.
#include <cuda_runtime.h>

#include <cstring>
#include <limits>
#include <new>
#include <string>

#include "api_ops.hpp"
#include "bmq.h"
#include "bmq_internal.hpp"
#include "engine.cuh"
#include "shard_run.hpp"

struct bmq_simulator {
    std::unique_ptr<bmq::Engine> engine;
};

struct bmq_collective {
    std::unique_ptr<bmq::Collective> col;
};

namespace {

thread_local std::string g_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return BMQ_OK;
    } catch (const bmq::Error& e) {
        g_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_error = "host allocation failed";
        return BMQ_ERR_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        g_error = e.what();
        return BMQ_ERR_LOGIC;
    }
}

void null_check(const void* p, const char* what) {
    if (!p) bmq::raise(BMQ_ERR_INVALID_ARGUMENT, std::string(what) + " must not be null");
}

}  // namespace

extern "C" {

const char* bmq_last_error(void) { return g_error.c_str(); }

const char* bmq_version(void) { return "bmq-b200 0.1 (sm_100a)"; }

int bmq_device_count(int* count) {
    return guarded([&] {
        null_check(count, "count");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        *count = n;
    });
}

int bmq_error_bound(double b_r, double* log2_abs) {
    return guarded([&] {
        if (!(b_r > 0.0) || std::isinf(b_r))
            bmq::raise(BMQ_ERR_INVALID_ARGUMENT, "relative error bound must be positive and finite");
        *log2_abs = std::log2(1.0 + b_r);
    });
}

int bmq_gate_unitary(const bmq_gate* gate, double* out) {
    return guarded([&] {
        null_check(gate, "gate");
        if (gate->kind > BMQ_GATE_CP) bmq::raise(BMQ_ERR_INVALID_ARGUMENT, "unknown gate kind");
        bmq::Cx u[16];
        const int dim = bmq::gate_matrix(*gate, u);
        for (int i = 0; i < dim * dim; ++i) {
            out[2 * i] = u[i].re;
            out[2 * i + 1] = u[i].im;
        }
    });
}

int bmq_circuit_validate(uint32_t num_qubits, const bmq_gate* gates, uint64_t count) {
    return guarded([&] { bmq::check_circuit(num_qubits, gates, count); });
}

int bmq_generate_benchmark(const char* name, uint32_t num_qubits, uint32_t layers, uint64_t seed, const char* secret,
                           bmq_gate* out, uint64_t cap, uint64_t* count) {
    return guarded([&] {
        null_check(name, "name");
        const auto c = bmq::make_benchmark(name, num_qubits, layers, seed, secret);
        *count = c.size();
        if (c.size() > cap) bmq::raise(BMQ_ERR_BUFFER_TOO_SMALL, "gate buffer too small");
        std::memcpy(out, c.data(), c.size() * sizeof(bmq_gate));
    });
}

int bmq_partition(uint32_t num_qubits, const bmq_gate* gates, uint64_t count, uint32_t block_bits,
                  uint32_t inner_size, bmq_stage* out, uint64_t cap, uint64_t* num_stages) {
    return guarded([&] {
        const auto plan = bmq::partition_plan(num_qubits, gates, count, block_bits, inner_size);
        *num_stages = plan.size();
        if (plan.size() > cap) bmq::raise(BMQ_ERR_BUFFER_TOO_SMALL, "stage buffer too small");
        std::memcpy(out, plan.data(), plan.size() * sizeof(bmq_stage));
    });
}

void bmq_plan_model_default(bmq_plan_model* model) {
    if (!model) return;
    *model = bmq_plan_model{};
    model->work_bytes = 16ull << 30;  // the engine's automatic work buffer on a B200
    model->hbm_gbs = 6500.0;          // measured copy bandwidth (MEASURED_PEAKS.json)
    model->link_gbs = 700.0;          // NVLink 5 per GPU and direction, after protocol
    model->ratio = 4.0;
    model->stage_overhead_s = 100e-6;
    model->world = 1;
    model->codec_eff = 0.4;  // decode / emit ~2.6 TB/s of 6.5 (profiles/r2b_ncu_qaoa28.txt)
    model->pass_eff = 0.5;   // streaming 5.4 TB/s, tiled 1.8-2.2 TB/s
}

int bmq_plan_device_aware(uint32_t num_qubits, const bmq_gate* gates, uint64_t count, uint32_t block_bits,
                          const bmq_plan_model* model, bmq_stage* out, uint64_t cap, uint64_t* num_stages,
                          bmq_plan_choice* choice) {
    return guarded([&] {
        null_check(model, "model");
        const auto plan = bmq::plan_device_aware(num_qubits, gates, count, block_bits, *model, choice);
        *num_stages = plan.size();
        if (plan.size() > cap) bmq::raise(BMQ_ERR_BUFFER_TOO_SMALL, "stage buffer too small");
        std::memcpy(out, plan.data(), plan.size() * sizeof(bmq_stage));
    });
}

int bmq_enumerate_groups(uint32_t num_qubits, uint32_t block_bits, const bmq_stage* stage, uint64_t* ids,
                         uint64_t cap, uint64_t* count) {
    return guarded([&] {
        null_check(stage, "stage");
        const bmq::Layout L = bmq::make_layout(num_qubits, block_bits);
        const bmq::GroupGeometry gg = bmq::group_geometry(L, *stage);
        *count = gg.groups() * gg.per_group();
        if (*count > cap) bmq::raise(BMQ_ERR_BUFFER_TOO_SMALL, "id buffer too small");
        uint64_t k = 0;
        for (uint64_t o = 0; o < gg.groups(); ++o)
            for (uint64_t v = 0; v < gg.per_group(); ++v) ids[k++] = gg.block_id(o, v);
    });
}

int bmq_buffer_bit_of_qubit(uint32_t num_qubits, uint32_t block_bits, const bmq_stage* stage, uint32_t qubit,
                            uint32_t* bit) {
    return guarded([&] {
        null_check(stage, "stage");
        *bit = bmq::buffer_bit(bmq::make_layout(num_qubits, block_bits), *stage, qubit);
    });
}

int bmq_parse_qasm(const char* text, uint32_t* num_qubits, bmq_gate* out, uint64_t cap, uint64_t* count,
                   char* warnings, uint64_t warnings_cap, uint64_t* num_warnings) {
    return guarded([&] {
        null_check(text, "text");
        const bmq::QasmCircuit c = bmq::parse_qasm_text(text);
        *num_qubits = c.num_qubits;
        *count = c.gates.size();
        if (num_warnings) *num_warnings = c.warnings.size();
        if (warnings && warnings_cap) {
            std::string joined;
            for (size_t i = 0; i < c.warnings.size(); ++i) joined += (i ? "\n" : "") + c.warnings[i];
            const size_t n = std::min<size_t>(joined.size(), warnings_cap - 1);
            std::memcpy(warnings, joined.data(), n);
            warnings[n] = 0;
        }
        if (c.gates.size() > cap) bmq::raise(BMQ_ERR_BUFFER_TOO_SMALL, "gate buffer too small");
        std::memcpy(out, c.gates.data(), c.gates.size() * sizeof(bmq_gate));
    });
}

int bmq_emit_qasm(uint32_t num_qubits, const bmq_gate* gates, uint64_t count, char* out, uint64_t cap,
                  uint64_t* size) {
    return guarded([&] {
        const std::string s = bmq::emit_qasm_text(num_qubits, gates, count);
        *size = s.size();
        if (s.size() + 1 > cap) bmq::raise(BMQ_ERR_BUFFER_TOO_SMALL, "text buffer too small");
        std::memcpy(out, s.c_str(), s.size() + 1);
    });
}

uint64_t bmq_compress_bound(uint64_t scalar_count) { return bmq::compress_bound(scalar_count); }

int bmq_compress_blocks(const double* scalars, uint64_t nblocks, uint64_t scalars_per_block, double error_bound,
                        uint8_t* out, uint64_t out_cap, uint64_t* sizes) {
    return guarded([&] {
        bmq::api_compress_blocks(scalars, nblocks, scalars_per_block, error_bound, out, out_cap, sizes);
    });
}

int bmq_decompress_blocks(const uint8_t* payloads, const uint64_t* offsets, const uint64_t* sizes, uint64_t nblocks,
                          double* out, uint64_t out_cap, uint64_t* counts) {
    return guarded([&] { bmq::api_decompress_blocks(payloads, offsets, sizes, nblocks, out, out_cap, counts); });
}

int bmq_apply_gate(double* amps, uint64_t namps, const double* u, int two_qubit, uint32_t hi_bit, uint32_t lo_bit) {
    return guarded([&] { bmq::api_apply_gate(amps, namps, u, two_qubit, hi_bit, lo_bit); });
}

int bmq_apply_stage(double* amps, uint64_t namps, uint32_t num_qubits, const bmq_gate* gates, uint64_t ngates,
                    const bmq_stage* stage, uint32_t block_bits) {
    return guarded([&] {
        null_check(stage, "stage");
        bmq::api_apply_stage(amps, namps, num_qubits, gates, ngates, *stage, block_bits);
    });
}

int bmq_dense_reference(uint32_t num_qubits, const bmq_gate* gates, uint64_t ngates, double* state,
                        uint32_t verify_cap_qubits) {
    return guarded([&] { bmq::api_dense_reference(num_qubits, gates, ngates, state, verify_cap_qubits); });
}

int bmq_fidelity(const double* a, const double* b, uint64_t namps, double* fidelity) {
    return guarded([&] {
        null_check(fidelity, "fidelity");
        if (namps) {
            null_check(a, "state a");
            null_check(b, "state b");
        }
        *fidelity = bmq::api_fidelity(a, b, namps);
    });
}

int bmq_simulator_footprint(bmq_simulator* sim, uint64_t* resident_bytes, uint64_t* spilled_live_bytes,
                            uint64_t* peak_bytes) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->footprint(resident_bytes, spilled_live_bytes, peak_bytes);
    });
}

void bmq_config_default(bmq_config* cfg) {
    if (!cfg) return;
    std::memset(cfg, 0, sizeof *cfg);
    cfg->block_bits = 1;
    cfg->inner_size = 2;
    cfg->error_bound = 1e-3;
    cfg->memory_budget = std::numeric_limits<uint64_t>::max();
    cfg->workers = 1;
    cfg->compress = 1;
    cfg->verify_cap_qubits = 24;
    cfg->device = 0;
    cfg->flags = BMQ_FLAG_ZERO_GROUP_SKIP | BMQ_FLAG_CODE_DOMAIN | BMQ_FLAG_STAGE_FUSION;
}

int bmq_simulator_create(uint32_t num_qubits, const bmq_gate* gates, uint64_t ngates, const bmq_config* cfg,
                         bmq_simulator** out) {
    return guarded([&] {
        null_check(cfg, "config");
        null_check(out, "out");
        *out = nullptr;
        auto s = std::make_unique<bmq_simulator>();
        s->engine = std::make_unique<bmq::Engine>(num_qubits, gates, ngates, *cfg);
        *out = s.release();
    });
}

int bmq_simulator_destroy(bmq_simulator* sim) {
    return guarded([&] { delete sim; });
}

int bmq_simulator_plan(const bmq_simulator* sim, bmq_stage* out, uint64_t cap, uint64_t* count) {
    return guarded([&] {
        null_check(sim, "simulator");
        const auto& p = sim->engine->plan();
        *count = p.size();
        if (p.size() > cap) bmq::raise(BMQ_ERR_BUFFER_TOO_SMALL, "stage buffer too small");
        std::memcpy(out, p.data(), p.size() * sizeof(bmq_stage));
    });
}

int bmq_simulator_init_state(bmq_simulator* sim) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->init_state();
    });
}

int bmq_simulator_run(bmq_simulator* sim, bmq_report* report, double* stage_ms, uint64_t stage_cap) {
    return guarded([&] {
        null_check(sim, "simulator");
        null_check(report, "report");
        sim->engine->run(report, stage_ms, stage_cap);
    });
}

int bmq_simulator_reset(bmq_simulator* sim) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->reset();
    });
}

int bmq_simulator_run_stages(bmq_simulator* sim, uint64_t first, uint64_t last) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->run_stages(first, last);
    });
}

int bmq_simulator_state_norm(bmq_simulator* sim, double* norm) {
    return guarded([&] {
        null_check(sim, "simulator");
        *norm = sim->engine->state_norm();
    });
}

int bmq_simulator_extract_state(bmq_simulator* sim, double* amps, uint64_t namps) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->extract_state(amps, namps);
    });
}

int bmq_simulator_amplitude(bmq_simulator* sim, uint64_t index, double* re, double* im) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->amplitude(index, re, im);
    });
}

int bmq_simulator_sample(bmq_simulator* sim, uint64_t nshots, uint64_t seed, uint64_t* out) {
    return guarded([&] {
        null_check(sim, "simulator");
        if (nshots) null_check(out, "out");
        sim->engine->sample(nshots, seed, out);
    });
}

int bmq_simulator_top_k(bmq_simulator* sim, uint64_t k, uint64_t* idx, double* re, double* im, uint64_t* count) {
    return guarded([&] {
        null_check(sim, "simulator");
        null_check(count, "count");
        if (k) {
            null_check(idx, "idx");
            null_check(re, "re");
            null_check(im, "im");
        }
        *count = sim->engine->top_k(k, idx, re, im);
    });
}

int bmq_simulator_get_payload(bmq_simulator* sim, uint64_t id, uint8_t* out, uint64_t cap, uint64_t* size) {
    return guarded([&] {
        null_check(sim, "simulator");
        *size = sim->engine->get_payload(id, out, cap);
        if (out && *size > cap) bmq::raise(BMQ_ERR_BUFFER_TOO_SMALL, "payload buffer too small");
    });
}

int bmq_simulator_get_payloads(bmq_simulator* sim, uint8_t* out, uint64_t cap, uint64_t* sizes, uint64_t* total) {
    return guarded([&] {
        null_check(sim, "simulator");
        null_check(total, "total");
        sim->engine->get_payloads(out, cap, sizes, total);
    });
}

int bmq_simulator_put_payload(bmq_simulator* sim, uint64_t id, const uint8_t* payload, uint64_t size) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->put_payload(id, payload, size);
    });
}

int bmq_simulator_fidelity_dense(bmq_simulator* sim, const double* ideal, uint64_t namps, double* fidelity) {
    return guarded([&] {
        null_check(sim, "simulator");
        *fidelity = sim->engine->fidelity_dense(ideal, namps);
    });
}

int bmq_simulator_fidelity(bmq_simulator* a, bmq_simulator* b, double* fidelity) {
    return guarded([&] {
        null_check(a, "simulator");
        null_check(b, "simulator");
        *fidelity = bmq::Engine::fidelity_pair(*a->engine, *b->engine);
    });
}

int bmq_simulator_fidelity_analytic(bmq_simulator* sim, int ideal_kind, double* fidelity) {
    return guarded([&] {
        null_check(sim, "simulator");
        *fidelity = sim->engine->fidelity_analytic(ideal_kind);
    });
}

int bmq_shard_plan(uint32_t num_qubits, uint32_t block_bits, const bmq_stage* stages, uint64_t num_stages,
                   uint32_t world, uint32_t* device_qubits) {
    return guarded([&] {
        const bmq::Layout L = bmq::make_layout(num_qubits, block_bits);
        std::vector<bmq_stage> plan(stages, stages + num_stages);
        for (const bmq_stage& st : plan) {
            if (st.inner_count > 64) bmq::raise(BMQ_ERR_INVALID_ARGUMENT, "stage has too many inner qubits");
            for (uint32_t i = 0; i < st.inner_count; ++i)
                if (st.inner[i] < L.b || st.inner[i] >= L.n)
                    bmq::raise(BMQ_ERR_INVALID_ARGUMENT, "inner qubit is not a global qubit");
        }
        const auto bits = bmq::shard_plan(L, plan, world);
        for (size_t i = 0; i < bits.size(); ++i) device_qubits[i] = bits[i] + L.b;
    });
}

int bmq_nccl_unique_id(uint8_t id[128]) {
    return guarded([&] {
        null_check(id, "id");
        bmq::nccl_unique_id(id);
    });
}

int bmq_collective_nccl_create(const uint8_t id[128], uint32_t rank, uint32_t world, int32_t device,
                               bmq_collective** out) {
    return guarded([&] {
        null_check(id, "id");
        null_check(out, "out");
        auto c = std::make_unique<bmq_collective>();
        c->col = bmq::make_nccl_collective(id, rank, world, device);
        *out = c.release();
    });
}

int bmq_collective_local_create(uint32_t world, bmq_collective** ranks) {
    return guarded([&] {
        null_check(ranks, "ranks");
        auto cols = bmq::make_local_collectives(world);
        for (uint32_t r = 0; r < world; ++r) {
            ranks[r] = new bmq_collective;
            ranks[r]->col = std::move(cols[r]);
        }
    });
}

int bmq_collective_destroy(bmq_collective* col) {
    delete col;
    return BMQ_OK;
}

int bmq_simulator_run_sharded(bmq_simulator* sim, bmq_collective* col, bmq_report* report, double* stage_ms,
                              uint64_t stage_cap) {
    return guarded([&] {
        null_check(sim, "simulator");
        null_check(col, "collective");
        bmq::run_sharded(*sim->engine, *col->col, report, stage_ms, stage_cap);
    });
}

int bmq_simulator_shard(bmq_simulator* sim, uint32_t rank, uint32_t world) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->shard(rank, world);
    });
}

int bmq_simulator_export(bmq_simulator* sim, const uint64_t* ids, uint64_t n, uint64_t* meta, void* dst,
                         uint64_t cap) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->export_payloads(ids, n, meta, dst, cap);
    });
}

int bmq_simulator_import(bmq_simulator* sim, const uint64_t* ids, uint64_t n, const uint64_t* meta,
                         const void* src) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->import_payloads(ids, n, meta, src);
    });
}

int bmq_simulator_drop(bmq_simulator* sim, const uint64_t* ids, uint64_t n) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->drop_payloads(ids, n);
    });
}

int bmq_simulator_stage_sizes(bmq_simulator* sim, uint64_t stage, uint64_t* sizes) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->stage_sizes(stage, sizes);
    });
}

int bmq_simulator_account_stage(bmq_simulator* sim, uint64_t stage, const uint64_t* sizes) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->account_stage(stage, sizes);
    });
}

int bmq_simulator_partial_sums(bmq_simulator* sim, double* sums3) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->partial_sums(sums3);
    });
}

int bmq_simulator_report(bmq_simulator* sim, bmq_report* report) {
    return guarded([&] {
        null_check(sim, "simulator");
        sim->engine->report(report, 0.0);
    });
}

int bmq_simulator_save(bmq_simulator* sim, const char* path) {
    return guarded([&] {
        null_check(sim, "simulator");
        null_check(path, "path");
        sim->engine->save_checkpoint(path);
    });
}

int bmq_simulator_load(bmq_simulator* sim, const char* path, uint64_t* next_stage) {
    return guarded([&] {
        null_check(sim, "simulator");
        null_check(path, "path");
        const uint64_t next = sim->engine->load_checkpoint(path);
        if (next_stage) *next_stage = next;
    });
}

}  // extern "C"
