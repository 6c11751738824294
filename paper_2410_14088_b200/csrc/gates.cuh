// gates.cuh — gate-stage engine: compiles a stage's gates (in program
// order) into tiled passes and applies them on device buffers.
#pragma once

#include <memory>
#include <vector>

#include "device_common.cuh"

namespace bmq {

// OP_CHAIN (fast kernel only): consecutive CP-like ops sharing one control
// bit c whose other bits are distinct and monotone in program order; an
// amplitude with bit c set is multiplied, in program order, by the phase of
// every set bit of (index & R), found by scanning set bits instead of ops.
enum OpType : uint8_t { OP_U2 = 0, OP_DIAG = 1, OP_CX = 2, OP_CDIAG = 3, OP_U4 = 4, OP_CHAIN = 5 };
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

// pdep(x, mask) as a short list of contiguous runs:
//   out = OR_i ((x >> src[i]) & (2^width[i] - 1)) << dst[i]
struct BitRuns {
    uint32_t n;
    uint8_t src[16], dst[16], width[16];
};

// Compact op for the register-tiled kernel (kernel parameter space).
struct FastOp {
    uint8_t type, tp_hi, tp_lo, in_hi, in_lo, hi, lo, pad;
    uint8_t et[4];    // CHAIN: et[0] = 1 when the other bits descend in program order
    uint32_t pad2;    // CHAIN: offset of the 64-entry phase table (double2 units)
    double m[8];      // U2: u00 u01 u10 u11; DIAG: u00 u11; CDIAG: u33 (interleaved re/im)
                      // CHAIN: m[0] holds the mask R of other bits (bit pattern)
};

constexpr uint32_t kMaxTileBits = 12;  // 4096 amplitudes per tile
constexpr int kMaxFastOps = 96;

struct FastPass {
    BitRuns tile;   // tile position k (12 bits) -> buffer offset
    BitRuns base;   // tile index -> buffer bits outside the tile
    uint32_t nops;
    uint32_t tab_entries;     // phase-table entries (double2) of this pass's chains
    uint64_t tab_base;        // first entry of this pass in chain_tab
    const double* chain_tab;  // phase tables of OP_CHAIN ops (re, im pairs), 32 per chain
    FastOp ops[kMaxFastOps];
};

struct GatePass {
    uint64_t tile_mask;   // buffer bits spanned by one CTA tile
    uint32_t tb;          // popcount(tile_mask)
    uint32_t begin, count;
    bool fast = false;
    std::shared_ptr<FastPass> fp;
};

struct GateProgram {
    std::vector<GateOp> ops;
    std::vector<GatePass> passes;
    GateOp* d_ops = nullptr;
    std::vector<double> chain_tab;   // host copy of the chain phase tables
    double* d_chain_tab = nullptr;
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

// Fused quantisation epilogue for the last pass of a stage: instead of
// storing the tile's doubles, the pass quantises them (exact reference
// quantiser) into packed code words (CmpBlock::pk layout: per block of 2^lb
// amplitudes, 2^(lb+1) words) and accumulates the per-chunk counters that
// the compressor's plan kernel consumes.
struct QuantOut {
    uint32_t* pk;      // packed words, block slot s at pk + s * 2^(lb+1)
    ChunkPlan* cps;    // counters, block slot s at cps + s * nch (zeroed)
    uint32_t nch;      // chunks per block
    DevTables t;
    DevError* err;
};

// Apply every pass in place to nreps consecutive buffers of
// 2^total_bits amplitudes (e.g. the groups of a batch). Layout: interleaved
// complex (lb ignored) or planar per block of 2^lb amplitudes. With quant
// given (planar layout only), the last pass runs the quantisation epilogue
// when it can (returns true); otherwise the doubles are stored as usual and
// the caller quantises them separately (returns false).
// With vtab (block-wise batches of a diagonal-only stage) the buffer holds
// nblocks independent blocks; vtab[slot] is the inner value of the block in
// that slot, used for the ops' inner-bit conditions.
bool run_program(cudaStream_t st, const GateProgram& prog, double* buf, uint32_t lb, bool interleaved,
                 uint64_t nreps, uint64_t* launches, const QuantOut* quant = nullptr,
                 const uint32_t* vtab = nullptr, uint64_t nblocks = 0);

}  // namespace bmq
