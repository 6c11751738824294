// A reference user's program, compiled against the C++ drop-in header
// (include/bmq/cbq.hpp) instead of /root/reference/proj/include/cbq, run on
// the B200. It exercises the surface north_star names and writes what the
// test compares with the oracle:
//   * Simulator::run on QFT-16 (b = 12, inner = 2) and QAOA-3reg-16 (p = 1,
//     1e-4) -> report fields, FNV-1a-64 of store().get(id) over all ids,
//     store().footprint(), fidelity(dense_reference, extract_state);
//   * parse_qasm(emit_qasm(c)) == c, and a QasmError's line / col;
//   * assemble_group_buffer -> apply_stage -> split_buffer on a 4-block group
//     of QAOA-3reg-10 whose input and output are written to argv[1] for the
//     test to replay through the reference kernels;
//   * apply_unitary2 / apply_unitary4 out-of-range errors.
#include <cmath>
#include <cstdint>
#include <cstdio>

#include "bmq/cbq.hpp"

namespace {

std::uint64_t fnv(const std::vector<std::uint8_t>& p, std::uint64_t h) {
    for (std::uint8_t c : p) h = (h ^ c) * 1099511628211ull;
    return h;
}

void run_case(const char* tag, const cbq::Circuit& c, std::uint32_t b, double br) {
    cbq::Config cfg;
    cfg.block_bits = b;
    cfg.inner_size = 2;
    cfg.error_bound = br;
    cfg.identity_skip = true;
    cbq::Simulator sim(c, cfg);
    const cbq::SimulationReport rep = sim.run();
    std::uint64_t h = 0xCBF29CE484222325ull;
    for (std::uint64_t id = 0; id < sim.layout().num_blocks(); ++id) h = fnv(sim.store().get(id), h);
    const cbq::Footprint f = sim.store().footprint();
    const double fid = cbq::fidelity(cbq::dense_reference(c), sim.extract_state());
    std::printf("%s stages %llu peak %llu ratio %.17g norm %.17g fnv %016llx fp_peak %llu fidelity %.17g\n", tag,
                static_cast<unsigned long long>(rep.stage_count),
                static_cast<unsigned long long>(rep.max_footprint_bytes), rep.compression_ratio, rep.final_norm,
                static_cast<unsigned long long>(h), static_cast<unsigned long long>(f.peak_bytes), fid);
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    run_case("qft16", cbq::generate_benchmark(cbq::Benchmark::Qft, 16), 12, 1e-3);
    const cbq::Circuit qaoa = cbq::parse_qasm(std::string(argv[2] ? argv[2] : ""));
    run_case("qaoa3reg16", qaoa, 12, 1e-4);

    // QASM round trip and error positions (qasm.hpp:17-31,387-411)
    const cbq::Circuit qft5 = cbq::generate_benchmark(cbq::Benchmark::Qft, 5);
    std::printf("qasm_roundtrip %d\n", cbq::parse_qasm(cbq::emit_qasm(qft5)) == qft5 ? 1 : 0);
    std::vector<std::string> warnings;
    cbq::parse_qasm("OPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg q[2];\nh q[0];\nmeasure q[0] -> c[0];\n",
                    &warnings);
    std::printf("qasm_warnings %zu\n", warnings.size());
    try {
        cbq::parse_qasm("OPENQASM 2.0;\nqreg q[2];\nh q[5];\n");
    } catch (const cbq::QasmError& e) {
        std::printf("qasm_error %d %d %s\n", e.line(), e.col(), e.what());
    }

    // kernel.hpp surface on one group of QAOA-3reg-10 at b = 4 (inner = 1; a CX pair makes it 4 blocks)
    const cbq::Circuit small = cbq::parse_qasm(std::string(argv[3] ? argv[3] : ""));
    const cbq::Layout L = cbq::make_layout(small.num_qubits, 4);
    const cbq::PartitionPlan plan = cbq::partition_circuit(small, 4, 1);
    const cbq::Stage& st = plan.stages.at(plan.stages.size() / 2);
    const auto groups = cbq::enumerate_groups(st, L);
    std::vector<cbq::SVBlock> blocks;
    for (std::size_t j = 0; j < groups[1].block_ids.size(); ++j) {
        cbq::SVBlock blk(L.block_size());
        for (std::size_t i = 0; i < blk.size(); ++i)
            blk[i] = cbq::Complex(std::ldexp(static_cast<double>((i * 7 + j * 3) % 11) - 5.0, -4),
                                  std::ldexp(static_cast<double>((i * 5 + j) % 13) - 6.0, -5));
        blocks.push_back(std::move(blk));
    }
    cbq::GroupBuffer buf = cbq::assemble_group_buffer(groups[1], blocks);
    const std::vector<cbq::Complex> input = buf.amps;
    cbq::apply_stage(buf, st, small, L);
    const auto out = cbq::split_buffer(buf, L.b);
    std::FILE* fp = std::fopen(argv[1], "wb");
    const std::uint64_t head[4] = {plan.stages.size() / 2, input.size(), out.size(), groups[1].block_ids.size()};
    std::fwrite(head, 8, 4, fp);
    std::fwrite(input.data(), sizeof(cbq::Complex), input.size(), fp);
    for (const auto& blk : out) std::fwrite(blk.data(), sizeof(cbq::Complex), blk.size(), fp);
    std::fclose(fp);
    std::printf("apply_stage_written %zu\n", out.size());

    std::vector<cbq::Complex> amps(8, cbq::Complex(1.0, 0.0));
    try {
        cbq::apply_unitary2(amps, 3, cbq::unitary2(cbq::Gate{cbq::GateKind::H, 0, 0, 0.0}));
    } catch (const std::invalid_argument& e) {
        std::printf("invalid_argument %s\n", e.what());
    }
    try {
        cbq::apply_unitary4(amps, 1, 1, cbq::unitary4(cbq::Gate{cbq::GateKind::CX, 0, 1, 0.0}));
    } catch (const std::invalid_argument& e) {
        std::printf("invalid_argument %s\n", e.what());
    }
    try {
        cbq::GroupBuffer bad = cbq::assemble_group_buffer(cbq::SVGroup{0, {0, 1, 2}}, {{}, {}, {}});
    } catch (const std::invalid_argument& e) {
        std::printf("invalid_argument %s\n", e.what());
    }
    return 0;
}
