// bmq_internal.hpp — shared declarations of libbmq (host C++ + sm_100a CUDA).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "bmq.h"

namespace bmq {

// Error carrying a bmq_status; the C ABI converts it to (status, message).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error(code, msg); }

// ------------------------------------------------------------------ circuit
struct Cx {
    double re, im;
};

bool gate_is_two_qubit(uint32_t kind);
void check_circuit(uint32_t n, const bmq_gate* gates, uint64_t count);
// Reference unitary (circuit.hpp:133-198) built with the host libm so the
// matrix entries are bit-identical to the reference's.
int gate_matrix(const bmq_gate& g, Cx* out);  // returns dimension (2 or 4)
std::vector<bmq_gate> make_benchmark(const std::string& name, uint32_t n, uint32_t layers,
                                     uint64_t seed, const char* secret);

struct Layout {
    uint32_t n = 1, b = 1, c = 0;
    uint64_t num_blocks() const { return 1ull << c; }
    uint64_t block_size() const { return 1ull << b; }
};
Layout make_layout(uint32_t n, uint32_t b);

std::vector<bmq_stage> partition_plan(uint32_t n, const bmq_gate* gates, uint64_t count,
                                      uint32_t block_bits, uint32_t inner_size);

// Device-aware plan: partition_plan at the inner size the
// engine's cost model prefers for this device (bmq_plan_device_aware).
std::vector<bmq_stage> plan_device_aware(uint32_t n, const bmq_gate* gates, uint64_t count, uint32_t block_bits,
                                         const bmq_plan_model& model, bmq_plan_choice* choice);

// Group geometry of one stage: block id of (outer value o, inner value v) is
// pdep(o, outer_mask) | pdep(v, inner_mask) over the c global-index bits.
struct GroupGeometry {
    uint64_t inner_mask = 0, outer_mask = 0;
    uint32_t inner_bits = 0, outer_bits = 0;
    uint64_t groups() const { return 1ull << outer_bits; }
    uint64_t per_group() const { return 1ull << inner_bits; }
    uint64_t block_id(uint64_t outer, uint64_t v) const;
};
GroupGeometry group_geometry(const Layout& L, const bmq_stage& st);

// Device bits (block-id bit positions, log2(world) per stage) of a sharded run.
std::vector<uint32_t> shard_plan(const Layout& L, const std::vector<bmq_stage>& plan, uint32_t world);
inline uint32_t shard_owner(uint64_t id, const uint32_t* bits, uint32_t m) {
    uint32_t r = 0;
    for (uint32_t j = 0; j < m; ++j) r |= static_cast<uint32_t>(id >> bits[j] & 1) << j;
    return r;
}
uint32_t buffer_bit(const Layout& L, const bmq_stage& st, uint32_t q);

inline uint64_t deposit_bits(uint64_t x, uint64_t mask) {
    uint64_t out = 0;
    for (uint64_t bit = 1; mask; bit <<= 1) {
        const uint64_t low = mask & (~mask + 1);
        if (x & bit) out |= low;
        mask ^= low;
    }
    return out;
}

// ------------------------------------------------------------- codec tables
// Exact quantiser tables for one relative bound (built with the host libm):
//   thresh[q - qlo] = bit pattern of the smallest positive double v with
//                     llround(log2(v) / b_a) >= q      (q in [qlo, qhi+1])
//   dequant[q - qlo] = exp2((double)q * b_a)           (q in [qlo, qhi])
// f(v) = llround(log2(v)/b_a) is monotone, so f(v) = max{q : thresh[q] <= v}:
// the device computes q exactly with a float log2 estimate plus two integer
// compares against thresh, and decodes exactly with one dequant lookup.
struct CodecTables {
    double b_r = 0.0, b_a = 0.0;
    int64_t qlo = 0, qhi = 0;
    std::vector<uint64_t> thresh;
    std::vector<double> dequant;
    // Every code q in [idem_lo, idem_hi] that compress can emit satisfies
    // f(exp2(q b_a)) == q, so a payload whose codes all lie in that range is
    // a fixed point of decompress -> compress.
    int64_t idem_lo = 0, idem_hi = 0;
};
const CodecTables& host_tables(double b_r);

// ------------------------------------------------------------------- stats
uint64_t compress_bound(uint64_t n);

// -------------------------------------------------------------------- qasm
struct QasmCircuit {
    uint32_t num_qubits = 0;
    std::vector<bmq_gate> gates;
    std::vector<std::string> warnings;
};
QasmCircuit parse_qasm_text(std::string_view text);
std::string emit_qasm_text(uint32_t n, const bmq_gate* gates, uint64_t count);

}  // namespace bmq
