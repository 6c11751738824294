/* oracle/cbq_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's hot path (BMQSim CPU reference,
 * /root/reference/proj/include/cbq). Used exclusively as the checker by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg; never
 * linked into or called by the product (paper_2410_14088_b200/).
 *
 * Parity status: PINNED. tests/test_oracle.py checks this port byte-for-byte
 * against the unmodified reference compiled into oracle/_ref/libcbqref.so
 * (payload bytes, plans, group ids, gate results, simulator reports) and
 * against the SPEC known answers / golden fixtures in tests/golden/.
 */
#ifndef CBQ_ORACLE_H
#define CBQ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (same numbering as include/bmq.h) */
enum {
    CBQO_OK = 0,
    CBQO_INVALID_ARGUMENT = 1,
    CBQO_LOGIC = 2,
    CBQO_CODEC = 3,
    CBQO_STORE = 4,
    CBQO_ENGINE = 5,
    CBQO_BUFFER_TOO_SMALL = 10
};

/* gate kinds in reference order (circuit.hpp:20-22) */
enum {
    CBQO_H, CBQO_X, CBQO_Y, CBQO_Z, CBQO_S, CBQO_SDG, CBQO_T, CBQO_TDG,
    CBQO_RX, CBQO_RY, CBQO_RZ, CBQO_P, CBQO_CX, CBQO_CZ, CBQO_CP
};

typedef struct {
    uint32_t kind, q0, q1, pad;
    double angle;
} cbqo_gate;

typedef struct {
    uint64_t gate_begin, gate_end;
    uint32_t inner_count, pad;
    uint32_t inner[64];
} cbqo_stage;

typedef struct {
    uint64_t qubits, gate_count, stage_count, max_footprint_bytes;
    double standard_bytes, compression_ratio;
    uint64_t spilled_blocks;
    double wall_ms;
    int32_t has_fidelity, pad;
    double fidelity, final_norm;
    uint64_t stage_compress_calls, stage_decompress_calls;
} cbqo_report;

const char* cbqo_last_error(void);

int cbqo_log2_abs(double b_r, double* out);
uint64_t cbqo_compress_bound(uint64_t scalar_count);
int cbqo_compress_block(const double* scalars, uint64_t n, double b_r, uint8_t* out,
                        uint64_t cap, uint64_t* size);
int cbqo_decompress_block(const uint8_t* payload, uint64_t size, double* out, uint64_t cap,
                          uint64_t* count);
int cbqo_prescan_encode(const uint64_t* words, uint64_t bit_count, uint8_t* out, uint64_t cap,
                        uint64_t* size);

int cbqo_unitary(const cbqo_gate* g, double* out);
int cbqo_generate_benchmark(const char* name, uint32_t n, uint32_t layers, uint64_t seed,
                            const char* secret, cbqo_gate* out, uint64_t cap, uint64_t* count);
int cbqo_partition(uint32_t n, const cbqo_gate* gates, uint64_t ngates, uint32_t block_bits,
                   uint32_t inner_size, cbqo_stage* out, uint64_t cap, uint64_t* nstages);
int cbqo_enumerate_groups(uint32_t n, uint32_t block_bits, const cbqo_stage* stage,
                          uint64_t* ids, uint64_t cap, uint64_t* count);
int cbqo_buffer_bit_of_qubit(uint32_t n, uint32_t block_bits, const cbqo_stage* stage,
                             uint32_t q, uint32_t* out);
int cbqo_apply_gate(double* amps, uint64_t namps, const double* u, int two_qubit,
                    uint32_t hi_bit, uint32_t lo_bit);
int cbqo_apply_stage(double* amps, uint64_t namps, uint32_t n, const cbqo_gate* gates,
                     uint64_t ngates, const cbqo_stage* stage, uint32_t block_bits);
int cbqo_simulate(uint32_t n, const cbqo_gate* gates, uint64_t ngates, uint32_t block_bits,
                  uint32_t inner_size, double error_bound, uint64_t memory_budget, int compress,
                  cbqo_report* rep, uint8_t* payloads, uint64_t pay_cap, uint64_t* pay_sizes,
                  double* state);
int cbqo_dense_reference(uint32_t n, const cbqo_gate* gates, uint64_t ngates, double* out);
int cbqo_fidelity(const double* a, const double* b, uint64_t namps, double* out);
uint64_t cbqo_fnv1a64(const uint8_t* data, uint64_t len, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif
