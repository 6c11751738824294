// api_ops.hpp — stateless device entry points behind the C ABI.
#pragma once

#include "bmq_internal.hpp"

namespace bmq {

void require_device();
void api_compress_blocks(const double* scalars, uint64_t nblocks, uint64_t n, double b_r, uint8_t* out,
                         uint64_t out_cap, uint64_t* sizes);
void api_decompress_blocks(const uint8_t* payloads, const uint64_t* offsets, const uint64_t* sizes, uint64_t nblocks,
                           double* out, uint64_t out_cap, uint64_t* counts);
void api_apply_gate(double* amps, uint64_t namps, const double* u, int two_qubit, uint32_t hi, uint32_t lo);
void api_apply_stage(double* amps, uint64_t namps, uint32_t n, const bmq_gate* gates, uint64_t ngates,
                     const bmq_stage& stage, uint32_t b);
double api_fidelity(const double* a, const double* b, uint64_t namps);
void api_dense_reference(uint32_t n, const bmq_gate* gates, uint64_t ngates, double* state, uint32_t cap);

}  // namespace bmq
