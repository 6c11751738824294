// gates.cuh — gate-stage engine: compiles a stage's gates (in program
// order) into tiled passes and applies them on device buffers.
#pragma once

#include <vector>

#include "device_common.cuh"

namespace bmq {

enum OpType : uint8_t { OP_U2 = 0, OP_DIAG = 1, OP_CX = 2, OP_CDIAG = 3, OP_U4 = 4 };
// Matrix entry classes. Each class evaluates the reference product u * a
// (libstdc++ (ur*ar - ui*ai, ur*ai + ui*ar), every product rounded) exactly,
// up to the sign of an exact zero, which the codec maps to the same bytes.
enum EntryType : uint8_t { ET_ZERO = 0, ET_ONE = 1, ET_NEG = 2, ET_REAL = 3, ET_IMAG = 4, ET_CPLX = 5 };

struct GateOp {
    uint8_t type;
    uint8_t hi, lo;       // buffer bits: hi = q0 (CX control), lo = q1 (CX target); 1q: hi
    uint8_t tp_hi, tp_lo; // tile positions (valid for the bits a pass mixes)
    uint8_t in_hi, in_lo; // condition bit lies inside the tile (1) or in the tile base (0)
    uint8_t pad;
    uint8_t et[16];
    double m[32];         // row-major entries, interleaved re/im
};

struct GatePass {
    uint64_t tile_mask;   // buffer bits spanned by one CTA tile
    uint32_t tb;          // popcount(tile_mask)
    uint32_t begin, count;
};

constexpr uint32_t kMaxTileBits = 12;  // 4096 amplitudes = 64 KiB of SMEM per tile

struct GateProgram {
    std::vector<GateOp> ops;
    std::vector<GatePass> passes;
    GateOp* d_ops = nullptr;
    uint32_t total_bits = 0;
    bool all_diagonal = true;     // no op mixes amplitudes
    uint64_t diag_cond_mask = 0;  // bits whose values decide whether any op acts
    ~GateProgram();
    GateProgram() = default;
    GateProgram(const GateProgram&) = delete;
    GateProgram& operator=(const GateProgram&) = delete;
};

// Classify one reference gate (already mapped to buffer bits).
GateOp make_op(const bmq_gate& g, uint32_t hi_bit, uint32_t lo_bit);
// General matrix on buffer bits (bmq_apply_gate).
GateOp make_matrix_op(const Cx* u, bool two_qubit, uint32_t hi_bit, uint32_t lo_bit);

// Split ops into passes over a buffer of 2^total_bits amplitudes and upload.
void build_program(GateProgram& prog, std::vector<GateOp> ops, uint32_t total_bits);

// Apply every pass in place to nreps consecutive buffers of
// 2^total_bits amplitudes (e.g. the groups of a batch). Layout: interleaved
// complex (lb ignored) or planar per block of 2^lb amplitudes.
void run_program(cudaStream_t st, const GateProgram& prog, double* buf, uint32_t lb, bool interleaved,
                 uint64_t nreps, uint64_t* launches);

}  // namespace bmq
