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
// OP_PERM (fast kernel only): materialise the pass's pending CX permutation
// (see FastOp::mrow) before an op that needs physical = logical positions.
enum OpType : uint8_t { OP_U2 = 0, OP_DIAG = 1, OP_CX = 2, OP_CDIAG = 3, OP_U4 = 4, OP_CHAIN = 5, OP_PERM = 6 };
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
// Lazy CX: within a fast pass a CX moves no data. The tile keeps a GF(2)
// affine map from physical tile position x to logical tile index
// y = M x ^ c (M: pass-constant, tracked on the host; c: per tile, on the
// device). Ops then address amplitudes through it:
//   DIAG / CDIAG: logical bit at tile position p = parity(mrow & x) ^ c_p
//                 (mrow = row p of M; mrow2 for CDIAG's second bit);
//   U2 on tile position t: pairs (x, x ^ dvec) with dvec = M^-1 e_t, the
//                 logical bit t of x being parity(mrow & x) ^ c_t.
// The pass ends (and a phase chain starts) with a gather through M^-1.
struct FastOp {
    uint8_t type, tp_hi, tp_lo, in_hi, in_lo, hi, lo, pad;
    uint8_t et[4];    // CHAIN: et[0] = 1 when the other bits descend in program order
    uint32_t pad2;    // CHAIN: offset of the 64-entry phase table (double2 units)
    double m[8];      // U2: u00 u01 u10 u11; DIAG: u00 u11; CDIAG: u33 (interleaved re/im)
                      // CHAIN: m[0] holds the mask R of other bits (bit pattern)
                      // PERM: m[0..2] hold the 12 columns of M^-1 (uint16 each)
    uint16_t mrow, mrow2, dvec;
    uint16_t run;     // diagonal ops (set on device): end of the sweep starting here | has-chain << 15
};

constexpr uint32_t kMaxTileBits = 12;  // 4096 amplitudes per tile
constexpr int kChainQBits = 3;         // a lone chain walks 2^kChainQBits amplitudes per thread together
constexpr int kMaxFastOps = 96;

struct FastPass {
    BitRuns tile;   // tile position k (12 bits) -> buffer offset
    BitRuns base;   // tile index -> buffer bits outside the tile
    uint32_t nops;
    uint16_t minv[kMaxTileBits];  // columns of M^-1 at the end of the pass (lazy CX)
    uint32_t final_perm;          // the pass ends with a non-identity M (gather on store)
    uint32_t tab_entries;     // phase-table entries (double2) of this pass's chains
    uint64_t tab_base;        // first entry of this pass in chain_tab
    const double* chain_tab;  // phase tables of OP_CHAIN ops (re, im pairs), 32 per chain
    FastOp ops[kMaxFastOps];
};

// Code-domain ("monomial") ops. Every entry of X, Y, Z, S, Sdg, CX and CZ
// is 0 or a unit in {1, i, -1, -i}, so the reference product u * a only moves
// real / imaginary parts and flips signs (up to the sign of an exact zero).
// A stage made only of such gates maps each decompressed scalar +-E[q] to
// another +-E[q] of the same code, so it runs on the packed code words
// (quantiser codes, sign and zero bits) with no floating point at all.
// Units: 0 = 1, 1 = i, 2 = -1, 3 = -i.
enum MonoKind : uint8_t { MK_DIAG = 0, MK_CDIAG = 1, MK_MIX = 2 };
struct MonoOp {
    uint8_t kind;
    uint8_t tp;            // MIX: tile position of the mixing bit
    uint8_t ctl;           // MIX: 0 none, 1 control bit in the tile (ctl_tp), 2 control bit in the base (hi)
    uint8_t ctl_tp;
    uint8_t hi, lo;        // buffer bits (DIAG: hi; CDIAG: hi and lo; MIX control: hi)
    uint8_t u0, u1;        // DIAG: units of |0>, |1>; CDIAG: u1 on |11>; MIX: out0 = u0 a1, out1 = u1 a0
};
constexpr int kMaxMonoOps = 512;
struct MonoPass {
    BitRuns tile, base;
    uint32_t nops;
    MonoOp ops[kMaxMonoOps];
};

// The composite of a pass's monomial ops on one tile is a signed
// permutation: out[k] = i^U(k) * in[src(k)], where (src, U) depends on the
// tile position k and on the few base bits the ops test outside the tile
// (their values form the "pattern"). Table entry per (pattern, k):
//   src (12 bits) | swap re/im << 12 | negate re << 13 | negate im << 14
constexpr int kMaxPatBits = 4;
struct PermPass {
    BitRuns tile, base;
    uint32_t npat_bits;
    uint32_t reim_swap;             // some entry swaps re / im (an odd unit)
    // buffer bits of tile positions 2..6 (a warp's lanes) and 10..11 (a
    // thread's four groups): below bit 12 (and lb >= 12) the chunk of a
    // lane's words is warp-uniform / also group-uniform, so the last pass's
    // counters reduce without matching (run_mono_program sets chunk_mode)
    uint64_t lane_bits, group_bits;
    uint32_t chunk_mode;            // 0: match lanes by chunk, 1: warp-uniform, 2: tile-uniform per warp
    uint8_t pat_bits[kMaxPatBits];  // buffer bits outside the tile, pattern bit i
    const uint16_t* table;          // [1 << npat_bits][4096] (device)
};

// Register-streaming pass (k_stream_pass): for passes of U2 / DIAG / CDIAG /
// CX gates whose partners stay within the lane bits 0..4 and two more bits Q.
// A warp owns "units" of 128 amplitudes: lane l, register value r of unit u
// holds buffer index x = base(u) | l | dep(r), dep(r) spreading r over Q.
// CX moves no data (as the tiled kernel's lazy CX): the host folds every CX
// into a GF(2) map y = M x from physical to logical index, so a diagonal gate
// on logical bit t multiplies by the entry of parity(row_t & x), and a U2 on
// logical bit t pairs x with x ^ d, d = column t of M^-1 (lane bits through a
// shuffle, Q bits as another register). A pass qualifies only if M is the
// identity again at its end (QAOA's CX-RZ-CX is). The parity over the
// register bits is a host-made 4-bit pattern per op (rpat), the rest one
// popcount per lane. Arithmetic is the tiled kernel's (cmul / row2: the
// reference's products, exact up to the sign of an exact zero). No shared
// memory, no barriers; units are dealt to warps in contiguous ranges so the
// quantising epilogue's per-chunk counters reduce once per run.
constexpr int kStreamNQ = 2;  // register bits per lane (4 values)
constexpr int kMaxStreamOps = 48;
struct StreamOp {
    uint8_t type;             // OP_DIAG, OP_CDIAG or OP_U2 (CX folded into the rows)
    uint8_t rpat, rpat2;      // bit r: parity(row & dep(r)) (row2: CDIAG's second bit)
    uint8_t dq;               // U2: partner register = r ^ dq
    uint32_t dl;              // U2: partner lane = lane ^ dl
    uint64_t row, row2;       // logical bit(s) = parity(row & x) over the non-register bits of x
    double m[8];              // U2: u00 u01 u10 u11; DIAG: u00 u11; CDIAG: u33 (interleaved re/im)
    uint8_t et[4];            // entry classes (U2: row-major; DIAG: u00 u11; CDIAG: u33)
    uint32_t pad;             // U2: 1 = real 2x2, 2 = real diagonal + imaginary off-diagonal, 0 = general
};
struct StreamPass {
    BitRuns base;             // unit index -> buffer bits outside {0..4} and Q
    uint8_t qbit[kStreamNQ];  // register bit i -> buffer bit
    uint8_t pad[6];
    uint32_t nops;
    uint32_t pad2;
    StreamOp ops[kMaxStreamOps];
};

struct GatePass {
    uint64_t tile_mask;   // buffer bits spanned by one CTA tile
    uint32_t tb;          // popcount(tile_mask)
    uint32_t begin, count;
    bool fast = false;
    std::shared_ptr<FastPass> fp;
    std::shared_ptr<MonoPass> mp;  // set on every pass when GateProgram::mono
    std::shared_ptr<PermPass> pp;  // table form of mp (when the pattern bits fit)
    std::shared_ptr<StreamPass> sp;  // register-streaming form (set when the pass qualifies)
};

struct GateProgram {
    std::vector<GateOp> ops;
    std::vector<GatePass> passes;
    GateOp* d_ops = nullptr;
    std::vector<double> chain_tab;   // host copy of the chain phase tables
    double* d_chain_tab = nullptr;
    uint16_t* d_perm_tab = nullptr;  // PermPass tables of all passes
    uint32_t total_bits = 0;
    bool all_diagonal = true;     // no op mixes amplitudes
    bool mono = false;            // every op is monomial with unit entries (code-domain stage)
    uint32_t lazy_cx = 0, perms = 0;  // CX folded into index maps / materialisations (fast passes)
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
    // stage fusion: the streaming pass stores each quantised scalar back as
    // its dequantised value (+-E[q], zero -> +0) at the same planar index of
    // rnd instead of its code word in pk (counters as usual)
    double* rnd = nullptr;
};

// First pass decodes its input rows itself (mode 3 of launch_decompress):
// the payload of block slot s is blks[s].in, its code segment, width and
// code_min in infos[s]; rows[w] describes planar word w of the batch.
struct FusedDecode {
    const DecBlock* blks = nullptr;
    const DecInfo* infos = nullptr;
    const DecRow* rows = nullptr;
    const double* dequant = nullptr;
    int64_t qlo = 0, qhi = 0;
    DevError* err = nullptr;
};
bool stream_first_pass(const GateProgram& prog, uint32_t lb, bool interleaved, bool blockwise);
bool stream_off();  // BMQ_DBG_NO_STREAM

// Apply every pass in place to nreps consecutive buffers of
// 2^total_bits amplitudes (e.g. the groups of a batch). Layout: interleaved
// complex (lb ignored) or planar per block of 2^lb amplitudes. With quant
// given (planar layout only), the last pass runs the quantisation epilogue
// when it can (returns true); otherwise the doubles are stored as usual and
// the caller quantises them separately (returns false).
// With vtab (block-wise batches of a diagonal-only stage) the buffer holds
// nblocks independent blocks; vtab[slot] is the inner value of the block in
// that slot, used for the ops' inner-bit conditions.
// zflag (optional; needs program_zero_skip): one flag byte per 32-scalar
// group of buf (index = planar address / 32), 0 for an all-zero group that
// was not stored; every pass reads and (except the quantising last pass)
// maintains them. nch is unused. wz (with zflag): device word, nonzero when
// some flag may be 0; launch_decompress and the passes set it.
bool program_zero_skip(const GateProgram& prog, uint32_t lb, bool interleaved);
// The program's last pass runs as a (quantising) streaming pass on a
// planar buffer of 2^lb-amplitude blocks, so QuantOut::rnd applies to it.
bool last_pass_streams(const GateProgram& prog, uint32_t lb);
bool run_program(cudaStream_t st, const GateProgram& prog, double* buf, uint32_t lb, bool interleaved,
                 uint64_t nreps, uint64_t* launches, const QuantOut* quant = nullptr,
                 const uint32_t* vtab = nullptr, uint64_t nblocks = 0, const uint8_t* zflag = nullptr,
                 uint32_t nch = 0, uint32_t* wz = nullptr, const FusedDecode* dec = nullptr);

// Code-domain program (prog.mono): the passes permute packed code words in
// place (planar per block of 2^lb amplitudes, CmpBlock::pk layout); the last
// pass also accumulates the per-chunk counters into quant->cps (zeroed).
// zflag (optional; needs mono_zero_skip): all-zero input chunks (launch_decompress)
// that the decoder left unwritten; the first pass reads them as zero words.
// imnz (optional, with zflag): device word, 0 when every imaginary-half chunk
// of the input is all zero (launch_decompress); if no pass swaps re / im the
// imaginary halves then stay zero and are neither read nor written.
// psrc (optional, with zflag): per (slot, chunk) PermSrc records (mode 1 of
// launch_decompress); chunks with meta != 0 were not decoded and the first
// pass reads their codes from the payload.
bool mono_zero_skip(const GateProgram& prog, uint32_t lb);
void run_mono_program(cudaStream_t st, const GateProgram& prog, uint32_t* pk, uint32_t lb, uint64_t nreps,
                      uint64_t* launches, const QuantOut& quant, const uint8_t* zflag = nullptr,
                      const uint32_t* imnz = nullptr, const PermSrc* psrc = nullptr);

}  // namespace bmq
