/* bmq.h — C ABI of the B200-native compressed-block state-vector engine
 * (libbmq.so, built from paper_2410_14088_b200/csrc).
 *
 * This is the drop-in boundary for the hot path of the BMQSim reference
 * (/root/reference/proj/include/cbq, header-only C++20). The reference has no
 * FFI of its own; each entry point below replaces the reference C++ symbol it
 * cites, with plain pointers and sizes so that ctypes / cgo / JNI / N-API can
 * bind it directly. The C++ drop-in surface in
 * include/bmq/cbq.hpp wraps these calls back into the reference's types
 * (Circuit, PartitionPlan, Simulator, compress_block, ...).
 *
 * Conventions
 *  - Every function returns a bmq_status; on failure bmq_last_error() holds a
 *    thread-local message with the same text the reference exception carries
 *    (e.g. "sign bitmap truncated", "stage 3: group with outer value 1: ...").
 *  - Host pointers everywhere; device memory is owned by the library.
 *  - Amplitude arrays are interleaved complex128 (re, im), block scalar
 *    arrays are the reference's planar layout (2^b real parts, then 2^b
 *    imaginary parts, engine.hpp:166-180).
 *  - Compute entry points run on the CUDA device (sm_100a). There is no CPU
 *    fallback: without a device they return BMQ_ERR_NO_DEVICE.
 */
#ifndef BMQ_H
#define BMQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum bmq_status {
    BMQ_OK = 0,
    BMQ_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument            */
    BMQ_ERR_LOGIC = 2,            /* std::logic_error                 */
    BMQ_ERR_CODEC = 3,            /* cbq::CodecError  (bitmap.hpp:14) */
    BMQ_ERR_STORE = 4,            /* cbq::StoreError  (store.hpp:23)  */
    BMQ_ERR_ENGINE = 5,           /* cbq::EngineError (engine.hpp:18) */
    BMQ_ERR_QASM = 6,             /* cbq::QasmError   (qasm.hpp:17)   */
    BMQ_ERR_CUDA = 7,
    BMQ_ERR_NO_DEVICE = 8,
    BMQ_ERR_OUT_OF_MEMORY = 9,
    BMQ_ERR_BUFFER_TOO_SMALL = 10
} bmq_status;

/* Gate kinds in the reference order (circuit.hpp:20-22). */
typedef enum bmq_gate_kind {
    BMQ_GATE_H = 0, BMQ_GATE_X, BMQ_GATE_Y, BMQ_GATE_Z, BMQ_GATE_S, BMQ_GATE_SDG,
    BMQ_GATE_T, BMQ_GATE_TDG, BMQ_GATE_RX, BMQ_GATE_RY, BMQ_GATE_RZ, BMQ_GATE_P,
    BMQ_GATE_CX, BMQ_GATE_CZ, BMQ_GATE_CP
} bmq_gate_kind;

/* cbq::Gate (circuit.hpp:65-72). For two-qubit kinds q0 is the HIGH bit of
 * the 2-bit sub-index (CX: q0 = control). 24 bytes. */
typedef struct bmq_gate {
    uint32_t kind;
    uint32_t q0;
    uint32_t q1;
    uint32_t reserved;
    double angle;
} bmq_gate;

/* cbq::Stage (partition.hpp:36-40): gates [gate_begin, gate_end) whose global
 * operands lie in inner[0..inner_count) (sorted ascending, each >= b). */
typedef struct bmq_stage {
    uint64_t gate_begin;
    uint64_t gate_end;
    uint32_t inner_count;
    uint32_t reserved;
    uint32_t inner[64];
} bmq_stage;

/* cbq::Config (engine.hpp:23-37) plus device-side knobs. */
typedef struct bmq_config {
    uint32_t block_bits;         /* b; reference default 1 */
    uint32_t inner_size;         /* reference default 2 */
    double error_bound;          /* point-wise relative bound b_r; default 1e-3 */
    uint64_t memory_budget;      /* store budget for the reference's accounting; UINT64_MAX = unlimited */
    uint32_t workers;            /* accepted for API parity; device concurrency is streams */
    uint32_t compress;           /* 1 = compressed payloads, 0 = raw little-endian doubles */
    uint32_t verify_cap_qubits;  /* default 24 */
    int32_t device;              /* CUDA ordinal, default 0 */
    uint64_t device_pool_bytes;  /* device payload arena capacity; 0 = automatic (grows) */
    uint64_t work_bytes;         /* dense group working set; 0 = automatic */
    uint32_t flags;              /* BMQ_FLAG_* */
    uint32_t reserved;
    /* Second level of the two-level store (store.hpp:47-300): pinned host
     * memory that receives payloads when the device arena is full (0 = no
     * host level: a full device arena is a StoreError). Device kernels read
     * and write it directly through the mapped address. */
    uint64_t host_pool_bytes;
    /* Third level (the reference's spill file, store.hpp:234-283):
     * payloads that fit neither the device arena nor the host level go to an
     * anonymous spill file in disk_dir (NULL: /tmp) of disk_pool_bytes,
     * moved device <-> file through a pinned bounce buffer (pread/pwrite),
     * or by GPUDirect Storage (cuFile) with BMQ_GDS=1 in the environment.
     * Needs host_pool_bytes > 0. */
    uint64_t disk_pool_bytes;
    const char* disk_dir;
} bmq_config;

/* Skip groups whose blocks are all ALL_ZERO (bit-exact: linear gates map
 * 0 -> 0 and the ALL_ZERO payload is canonical, codec.hpp:263-271). */
#define BMQ_FLAG_ZERO_GROUP_SKIP 0x1u
/* Skip blocks on which every gate of the stage acts as the identity
 * (diagonal-only stages whose controls are not all set for the block);
 * bit-exact because compress(decompress(p)) == p for every payload p the
 * device codec emits (checked per error bound when the tables are built). */
#define BMQ_FLAG_IDENTITY_SKIP 0x2u
/* Run stages made only of gates whose matrix entries are 0 or units
 * (X, Y, Z, S, Sdg, CX, CZ) on the quantiser codes: such gates only move
 * real/imaginary parts and flip signs, so every decompressed scalar +-E[q]
 * lands on another scalar with the same code. Bit-exact under the same
 * idempotence check as BMQ_FLAG_IDENTITY_SKIP; default on. */
#define BMQ_FLAG_CODE_DOMAIN 0x4u
/* device_pool_bytes is only the initial arena size: arenas double when the
 * live state fills more than half of one after a compaction (always the case
 * for automatic sizing, device_pool_bytes == 0). */
#define BMQ_FLAG_POOL_GROW 0x8u
/* Device arena placement. Default: one extent per payload from a host-side
 * best-fit heap when the layout has at most 2^17 blocks (freed when the block
 * is rewritten: dense stages reuse the space they decode, no compaction), a
 * bump cursor with in-place compaction for more, smaller blocks. These flags
 * force either policy (payload bytes are identical). */
#define BMQ_FLAG_HEAP_ARENA 0x10u
#define BMQ_FLAG_BUMP_ARENA 0x20u
/* Plan with bmq_plan_device_aware (this device's work buffer and HBM, world
 * 1, inner_size as the cap) instead of partition_circuit(inner_size). */
#define BMQ_FLAG_DEVICE_PLAN 0x40u
/* Stage fusion: runs of consecutive FP stages of the plan run over the groups
 * of the union of their inner qubits, decoded once and emitted once. Between
 * two fused stages every amplitude is quantised and dequantised in place
 * (v -> +-E[q(v)], zero -> 0: exactly decompress_block(compress_block(.)),
 * whose result depends on each scalar's code only, not on the block's
 * code_min / width), and the intermediate stage's payload sizes come from the
 * same per-chunk counters the emit would use, so the payloads, the peak and
 * every reported size equal the unfused run's (codec.hpp:227-344). Not used
 * with a disk level, on code-domain, identity-skipped (diagonal block-wise)
 * or phase-chain stages, or in sharded runs. Default on (bmq_config_default). */
#define BMQ_FLAG_STAGE_FUSION 0x80u

/* cbq::SimulationReport (engine.hpp:39-53) plus device-side counters. */
typedef struct bmq_report {
    uint64_t qubits;
    uint64_t gate_count;
    uint64_t stage_count;
    uint64_t max_footprint_bytes;   /* replayed in the reference's sequential put order */
    double standard_bytes;          /* 2^(n+4) */
    double compression_ratio;       /* standard_bytes / max_footprint_bytes */
    uint64_t spilled_blocks;
    double wall_ms;                 /* host wall clock of run(), as the reference */
    int32_t has_fidelity;
    int32_t reserved;
    double fidelity;
    double final_norm;
    uint64_t stage_compress_calls;
    uint64_t stage_decompress_calls;
    /* device-side extras */
    double device_ms;               /* CUDA-event time of the stage loop */
    uint64_t groups_processed;      /* groups that went through decompress/gates/compress */
    uint64_t groups_skipped;        /* zero / identity groups */
    uint64_t blocks_processed;
    uint64_t payload_bytes_read;    /* compressed bytes consumed by processed groups */
    uint64_t payload_bytes_written;
    uint64_t dense_bytes;           /* 32 B x amplitudes of processed groups (roofline model) */
    uint64_t kernel_launches;
    uint64_t device_peak_bytes;     /* pools + working set high-water */
    uint64_t gate_passes;
    /* CUDA-event time per phase of the stage loop (engine stream) */
    double decompress_ms;           /* descriptor build + index + decode */
    double gate_ms;                 /* gate-program passes */
    double compress_ms;             /* stats + plan + alloc + zero + emit + sums */
    uint64_t batches;
    /* algorithmic HBM bytes per phase (roofline numerators) */
    uint64_t decompress_bytes;      /* payload bytes read + 16 B per amplitude written */
    uint64_t gate_bytes;            /* 32 B per amplitude per gate pass */
    uint64_t compress_bytes;        /* 16 B per amplitude read + payload bytes written */
    uint64_t fused_batches;         /* batches whose last gate pass quantised in place */
    uint64_t compactions;           /* payload arena compactions */
    uint64_t host_spill_bytes;      /* payload bytes placed in the pinned host arena */
    uint64_t host_spill_batches;    /* batches whose payloads went to the host arena */
    uint64_t code_domain_batches;   /* batches run on quantiser codes (BMQ_FLAG_CODE_DOMAIN) */
    uint64_t pool_growths;          /* device arena growths (more HBM mapped in place) */
    uint64_t lazy_cx;               /* CX gates folded into a pass's index map (per batch) */
    uint64_t perm_materialisations; /* index maps materialised before a phase chain (per batch) */
    /* SURVEY 8(d) roofline numerator: for every group with at least one
     * non-ALL_ZERO input block, the reference-exact payload bytes of ALL its
     * blocks read and written (identity-skipped blocks included, ALL_ZERO
     * blocks as their 26-byte header) plus 32 B per amplitude of the group */
    uint64_t model_bytes;
    uint64_t model_groups;          /* the groups model_bytes counts */
    uint64_t link_h2d_bytes;        /* host-tier payload bytes moved host -> device */
    uint64_t link_d2h_bytes;        /* host-tier payload bytes moved device -> host */
    double link_ms;                 /* CUDA-event time of the host-tier copies (copy streams) */
    uint64_t compact_bytes;         /* payload bytes moved by in-place arena compactions */
    uint64_t host_peak_bytes;       /* high-water of live payload bytes in the pinned host level */
    uint64_t arena_bytes;           /* device arena capacity at the end of the run */
    uint64_t fused_decode_batches;  /* batches whose first gate pass decoded the payload rows itself */
    uint64_t stream_passes;         /* gate passes with a register-streaming form (k_stream_pass; blocks of >= 2^12) */
    uint64_t disk_spill_bytes;      /* payload bytes written to the disk level */
    uint64_t disk_read_bytes;       /* payload bytes read back from the disk level */
    uint64_t disk_peak_bytes;       /* high-water of live payload bytes on the disk level */
    uint64_t disk_gds;              /* 1 when the disk level moves data with GPUDirect Storage (cuFile) */
    uint64_t fused_stages;          /* stages run inside a fused run (BMQ_FLAG_STAGE_FUSION) */
    uint64_t fused_sets;            /* fused runs of consecutive stages */
} bmq_report;

/* ------------------------------------------------------------ host-only
 * (descriptor logic; callable without a GPU) */

const char* bmq_last_error(void);
const char* bmq_version(void);
int bmq_device_count(int* count);

/* ErrorBound (codec.hpp:19-29): log2_abs = log2(1 + b_r). */
int bmq_error_bound(double b_r, double* log2_abs);

/* unitary2 / unitary4 (circuit.hpp:133-198): row-major, interleaved re/im;
 * writes 8 doubles (1-qubit) or 32 doubles (2-qubit). */
int bmq_gate_unitary(const bmq_gate* gate, double* out);

/* Circuit(n) + Circuit::add validation (circuit.hpp:103-127). */
int bmq_circuit_validate(uint32_t num_qubits, const bmq_gate* gates, uint64_t count);

/* generate_benchmark (benchmarks.hpp:148-166); name in {ghz, cat_state, bv,
 * qft, qaoa}, plus the BASELINE.json workloads built from the reference gate
 * set: "qaoa3reg" (QAOA MaxCut on a random 3-regular graph, `layers` = p) and
 * "random" (sqrt-X/Y/W + CZ grid circuit, `layers` = cycles).
 * *count receives the full gate count even when cap is short. */
int bmq_generate_benchmark(const char* name, uint32_t num_qubits, uint32_t layers, uint64_t seed,
                           const char* secret, bmq_gate* out, uint64_t cap, uint64_t* count);

/* partition_circuit (partition.hpp:59-101). */
int bmq_partition(uint32_t num_qubits, const bmq_gate* gates, uint64_t count, uint32_t block_bits,
                  uint32_t inner_size, bmq_stage* out, uint64_t cap, uint64_t* num_stages);

/* Device-aware planning (optional). partition_circuit's
 * inner_size is a fixed user knob; this picks it for the device: it builds
 * partition_circuit(circuit, block_bits, k) for every feasible k (group
 * buffer 2^(b+k) complex doubles <= work_bytes, k <= c - log2(world),
 * k <= max_inner when nonzero) and keeps the plan whose modelled time is
 * least: per stage, the HBM bytes of this engine's decode -> tile passes ->
 * quantise -> emit trip (passes counted as gates.cu splits them) at the
 * fractions codec_eff / pass_eff of hbm_gbs, plus stage_overhead_s, plus
 * (world > 1) the payload remaps of the shard plan at link_gbs. The result is always a partition_circuit plan, so the
 * reference replays it with inner_size = choice->inner_size. */
typedef struct bmq_plan_model {
    uint64_t work_bytes;      /* group buffer budget (bytes) */
    double hbm_gbs;           /* per-GPU HBM bandwidth */
    double link_gbs;          /* per-GPU peer bandwidth for remaps (world > 1) */
    double ratio;             /* expected compression ratio (payload bytes = 16 / ratio per amplitude) */
    double stage_overhead_s;  /* fixed cost per stage (launches, syncs) */
    uint32_t world;           /* GPUs (power of two) */
    uint32_t max_inner;       /* 0 = no cap */
    double codec_eff;         /* fraction of hbm_gbs the decode / emit kernels reach (measured ~0.4) */
    double pass_eff;          /* fraction of hbm_gbs the gate passes reach (measured ~0.5) */
} bmq_plan_model;
typedef struct bmq_plan_choice {
    uint32_t inner_size;      /* chosen k */
    uint32_t candidates;      /* entries of inner / model_s */
    uint64_t stages, passes;  /* of the chosen plan */
    uint32_t remaps, reserved;
    double model_s_best;
    uint32_t inner[16];
    double model_s[16];
} bmq_plan_choice;
void bmq_plan_model_default(bmq_plan_model* model);
int bmq_plan_device_aware(uint32_t num_qubits, const bmq_gate* gates, uint64_t count, uint32_t block_bits,
                          const bmq_plan_model* model, bmq_stage* out, uint64_t cap, uint64_t* num_stages,
                          bmq_plan_choice* choice);

/* enumerate_groups (partition.hpp:120-153): block ids row-major
 * (group o, inner value v) -> ids[o * 2^|inner| + v]. */
int bmq_enumerate_groups(uint32_t num_qubits, uint32_t block_bits, const bmq_stage* stage,
                         uint64_t* ids, uint64_t cap, uint64_t* count);

/* buffer_bit_of_qubit (partition.hpp:158-169). */
int bmq_buffer_bit_of_qubit(uint32_t num_qubits, uint32_t block_bits, const bmq_stage* stage,
                            uint32_t qubit, uint32_t* bit);

/* parse_qasm (qasm.hpp:387-389): OPENQASM 2.0 subset. On BMQ_ERR_QASM the
 * message is "line L, col C: ..." (cbq::QasmError). *count receives the full
 * gate count even when cap is short; warnings (e.g. ignored measure) are
 * written '\n'-separated into `warnings` (may be NULL). */
int bmq_parse_qasm(const char* text, uint32_t* num_qubits, bmq_gate* out, uint64_t cap, uint64_t* count,
                   char* warnings, uint64_t warnings_cap, uint64_t* num_warnings);

/* emit_qasm (qasm.hpp:392-411): parse_qasm(emit_qasm(c)) == c. *size gets the
 * text length (without the terminating NUL, which is written when it fits). */
int bmq_emit_qasm(uint32_t num_qubits, const bmq_gate* gates, uint64_t count, char* out, uint64_t cap,
                  uint64_t* size);

/* Upper bound on compress output bytes for one block of n scalars. */
uint64_t bmq_compress_bound(uint64_t scalar_count);

/* ------------------------------------------------------- device compute */

/* compress_block (codec.hpp:227-295) for nblocks blocks of n scalars each
 * (scalars[k*n .. k*n+n)). Payloads are written back to back into out;
 * sizes[k] receives each payload's length. Byte-identical to the reference. */
int bmq_compress_blocks(const double* scalars, uint64_t nblocks, uint64_t scalars_per_block,
                        double error_bound, uint8_t* out, uint64_t out_cap, uint64_t* sizes);

/* decompress_block (codec.hpp:299-344) for nblocks payloads (payloads +
 * offsets[k], sizes[k] bytes). Scalars are written back to back into out;
 * counts[k] receives each block's scalar count. Bit-identical values. */
int bmq_decompress_blocks(const uint8_t* payloads, const uint64_t* offsets, const uint64_t* sizes,
                          uint64_t nblocks, double* out, uint64_t out_cap, uint64_t* counts);

/* apply_unitary2 / apply_unitary4 (kernel.hpp:24-64) on an interleaved
 * complex buffer of namps amplitudes; u is row-major interleaved (8 or 32
 * doubles). Bit-identical to the reference arithmetic. */
int bmq_apply_gate(double* amps, uint64_t namps, const double* u, int two_qubit, uint32_t hi_bit,
                   uint32_t lo_bit);

/* apply_stage (kernel.hpp:111-122) on one assembled group buffer. */
int bmq_apply_stage(double* amps, uint64_t namps, uint32_t num_qubits, const bmq_gate* gates,
                    uint64_t ngates, const bmq_stage* stage, uint32_t block_bits);

/* dense_reference (engine.hpp:254-296), full FP64 vector on the device. */
int bmq_dense_reference(uint32_t num_qubits, const bmq_gate* gates, uint64_t ngates,
                        double* state, uint32_t verify_cap_qubits);

/* fidelity (engine.hpp:299-308): |sum_i conj(a_i) b_i| of two interleaved
 * complex host states of namps amplitudes, reduced on the device. */
int bmq_fidelity(const double* a, const double* b, uint64_t namps, double* fidelity);

/* ------------------------------------------------------------ simulator
 * cbq::Simulator (engine.hpp:58-250). */

typedef struct bmq_simulator bmq_simulator;

void bmq_config_default(bmq_config* cfg);
int bmq_simulator_create(uint32_t num_qubits, const bmq_gate* gates, uint64_t ngates,
                         const bmq_config* cfg, bmq_simulator** out);
int bmq_simulator_destroy(bmq_simulator* sim);
/* plan() (engine.hpp:161) */
int bmq_simulator_plan(const bmq_simulator* sim, bmq_stage* out, uint64_t cap, uint64_t* count);
/* init_state() (engine.hpp:74-95) */
int bmq_simulator_init_state(bmq_simulator* sim);
/* run() (engine.hpp:97-134); stage_ms may be NULL. */
int bmq_simulator_run(bmq_simulator* sim, bmq_report* report, double* stage_ms, uint64_t stage_cap);
/* Discard the state so init_state()/run() can start over (plan, tables and
 * device buffers are kept). */
int bmq_simulator_reset(bmq_simulator* sim);
/* run stages [first, last) only (stage-level driver for pipelined callers). */
int bmq_simulator_run_stages(bmq_simulator* sim, uint64_t first, uint64_t last);
/* state_norm() (engine.hpp:150-158) */
int bmq_simulator_state_norm(bmq_simulator* sim, double* norm);
/* extract_state() (engine.hpp:138-147); refuses above verify_cap_qubits. */
int bmq_simulator_extract_state(bmq_simulator* sim, double* amps, uint64_t namps);
/* single amplitude query (new: the reference only has the dense extract). */
int bmq_simulator_amplitude(bmq_simulator* sim, uint64_t index, double* re, double* im);
/* Sampling (the reference has only the dense extract_state,
 * engine.hpp:138-147): nshots basis-state indices drawn from |a_i|^2 / norm^2
 * of the stored (decompressed) state, deterministic for a seed (mt19937_64).
 * Only blocks that receive shots are decoded. */
int bmq_simulator_sample(bmq_simulator* sim, uint64_t nshots, uint64_t seed, uint64_t* out);
/* The k amplitudes of largest |a|^2 (ties to the lower index), largest
 * first; *count = min(k, number of nonzero amplitudes). */
int bmq_simulator_top_k(bmq_simulator* sim, uint64_t k, uint64_t* idx, double* re, double* im, uint64_t* count);
/* store().get(id) (store.hpp:120-136): exact payload bytes of block id. */
int bmq_simulator_get_payload(bmq_simulator* sim, uint64_t id, uint8_t* out, uint64_t cap,
                              uint64_t* size);
/* All payloads in id order, back to back; sizes[2^c]. */
int bmq_simulator_get_payloads(bmq_simulator* sim, uint8_t* out, uint64_t cap, uint64_t* sizes,
                               uint64_t* total);
/* store().put(id, payload) (store.hpp:64-83). */
int bmq_simulator_put_payload(bmq_simulator* sim, uint64_t id, const uint8_t* payload,
                              uint64_t size);
/* fidelity(dense_reference, extract_state) (engine.hpp:299-308) against a
 * caller-supplied ideal state (interleaved, 2^n amplitudes). */
int bmq_simulator_fidelity_dense(bmq_simulator* sim, const double* ideal, uint64_t namps,
                                 double* fidelity);
/* |<a|b>| between two simulators of the same layout, streamed block-wise. */
int bmq_simulator_fidelity(bmq_simulator* a, bmq_simulator* b, double* fidelity);
/* |<ideal|state>| for closed-form ideal states: 0 = uniform 2^(-n/2)
 * (QFT of |0>), 1 = GHZ (|0..0> + |1..1>)/sqrt 2. */
int bmq_simulator_fidelity_analytic(bmq_simulator* sim, int ideal_kind, double* fidelity);

/* ---- sharded runs (one simulator per rank) ----
 * The reference runs one process (engine.hpp:97-134); these entry points let a
 * shard driver (paper_2410_14088_b200/shard.py) spread its stage loop over
 * `world` ranks. Stage s's groups belong to the rank whose bits are the values
 * of log2(world) "device qubits" (outer qubits of s); payloads whose owner
 * changes between stages move through the driver's collective. */

/* Device qubits of every stage: device_qubits[s * log2(world) + j] is the
 * qubit whose value is bit j of the owning rank. Host-only. */
int bmq_shard_plan(uint32_t num_qubits, uint32_t block_bits, const bmq_stage* stages, uint64_t num_stages,
                   uint32_t world, uint32_t* device_qubits);
/* Make `sim` rank `rank` of `world` (before the state is initialized).
 * run() is then refused: drive stages with run_stages + export/import. */
int bmq_simulator_shard(bmq_simulator* sim, uint32_t rank, uint32_t world);
/* meta[4 i .. 4 i + 3] = {payload size (0 = ALL_ZERO, no bytes), then the
 * block's sum |a|^2, sum re, sum im as f64 bit patterns}. With dst != NULL
 * (device or host memory, 16-byte aligned) the payloads are packed at
 * 16-byte aligned offsets in id-list order; cap >= sum of rounded sizes. */
int bmq_simulator_export(bmq_simulator* sim, const uint64_t* ids, uint64_t n, uint64_t* meta, void* dst,
                         uint64_t cap);
/* Store payloads packed as by export (src device or host memory). */
int bmq_simulator_import(bmq_simulator* sim, const uint64_t* ids, uint64_t n, const uint64_t* meta,
                         const void* src);
/* Forget payloads (the ids become ALL_ZERO with zero sums). */
int bmq_simulator_drop(bmq_simulator* sim, const uint64_t* ids, uint64_t n);
/* sizes[id] = payload size of every id this rank owns under stage s, else 0. */
int bmq_simulator_stage_sizes(bmq_simulator* sim, uint64_t stage, uint64_t* sizes);
/* Replay BlockStore::put of stage s (store.hpp:64-83) with global sizes. */
int bmq_simulator_account_stage(bmq_simulator* sim, uint64_t stage, const uint64_t* sizes);
/* {sum |a|^2, sum re, sum im} over the blocks this rank holds. */
int bmq_simulator_partial_sums(bmq_simulator* sim, double* sums3);
/* store().footprint() (store.hpp:30-35): the replayed BlockStore accounting
 * of the reference's sequential put order. Any pointer may be NULL. */
int bmq_simulator_footprint(bmq_simulator* sim, uint64_t* resident_bytes, uint64_t* spilled_live_bytes,
                            uint64_t* peak_bytes);
/* Report of the stages run so far (final_norm, wall_ms, device_ms = 0). */
int bmq_simulator_report(bmq_simulator* sim, bmq_report* report);

/* ---- multi-GPU stage loop behind the C ABI ----
 * A collective names this rank of a sharded run. NCCL: one process per GPU;
 * rank 0 gets a 128-byte id from bmq_nccl_unique_id and hands it to every
 * rank by the caller's own means (libnccl.so.2 is loaded at run time).
 * Local: `world` collectives for `world` simulators driven by `world`
 * threads of one process (any devices, e.g. several ranks on one GPU).
 * bmq_simulator_run_sharded is Simulator::run (engine.hpp:97-134) for one
 * rank: every rank calls it (SPMD) with its own simulator of the same
 * circuit and config; device qubits (bmq_shard_plan) keep every stage's
 * groups on one rank, payloads whose owner changes between stages move over
 * the collective, the BlockStore accounting is replayed from all-reduced
 * sizes, and the report's norm and counters are global. Final payloads equal
 * the single-GPU run's; each rank holds the blocks it owns under the last
 * stage (the others read ALL_ZERO). */
typedef struct bmq_collective bmq_collective;
int bmq_nccl_unique_id(uint8_t id[128]);
int bmq_collective_nccl_create(const uint8_t id[128], uint32_t rank, uint32_t world, int32_t device,
                               bmq_collective** out);
int bmq_collective_local_create(uint32_t world, bmq_collective** ranks);
int bmq_collective_destroy(bmq_collective* col);
int bmq_simulator_run_sharded(bmq_simulator* sim, bmq_collective* col, bmq_report* report, double* stage_ms,
                              uint64_t stage_cap);

/* ---- checkpoint / resume (the reference keeps no persisted
 * index, store.hpp:36-46) ----
 * save: every payload (exact bytes, codec.hpp:33-54) with its block sums,
 * the BlockStore accounting replay and the stage cursor, to one file.
 * load: into a simulator of the same circuit, layout, plan and error bound
 * (validated); *next_stage = the first stage still to run (continue with
 * bmq_simulator_run_stages / bmq_simulator_run). Payloads, max_footprint and
 * the final state equal those of an uninterrupted run. */
int bmq_simulator_save(bmq_simulator* sim, const char* path);
int bmq_simulator_load(bmq_simulator* sim, const char* path, uint64_t* next_stage);

#ifdef __cplusplus
}
#endif
#endif /* BMQ_H */
