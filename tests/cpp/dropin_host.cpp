// Compiles against the C++ drop-in header (include/bmq/cbq.hpp) exactly as a
// reference user would, and prints host-side descriptors for the test to
// compare with the oracle: QFT-34 stage counts, the partition_test.cc group
// golden {0,2,8,10}, and the error types of bad input.
#include <cstdio>

#include "bmq/cbq.hpp"

int main() {
    const cbq::Circuit qft = cbq::generate_benchmark(cbq::Benchmark::Qft, 34);
    std::printf("qft34_gates %zu\n", qft.gates.size());
    for (auto [b, i] : {std::pair{14u, 2u}, {20u, 2u}, {20u, 6u}})
        std::printf("stages %u %u %zu\n", b, i, cbq::partition_circuit(qft, b, i).stages.size());
    const auto groups = cbq::enumerate_groups(cbq::Stage{0, 0, {3, 5}}, cbq::make_layout(6, 2));
    std::printf("group0");
    for (auto id : groups[0].block_ids) std::printf(" %llu", static_cast<unsigned long long>(id));
    std::printf("\n");
    const auto u = cbq::unitary2(cbq::Gate{cbq::GateKind::H, 0, 0, 0.0});
    std::printf("h00 %.17g\n", u[0].real());
    try {
        cbq::Circuit c(3);
        c.add(cbq::Gate{cbq::GateKind::CX, 1, 1, 0.0});
    } catch (const std::invalid_argument& e) {
        std::printf("invalid_argument %s\n", e.what());
    }
    try {
        cbq::buffer_bit_of_qubit(cbq::Stage{0, 0, {3, 5}}, cbq::make_layout(6, 2), 4);
    } catch (const std::logic_error& e) {
        std::printf("logic_error %s\n", e.what());
    }
    return 0;
}
