/* oracle/cbq_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * A from-scratch C11 restatement of the BMQSim CPU reference hot path. Each
 * function names the reference file:line it restates (paths relative to
 * /root/reference/proj/include/cbq). Arithmetic follows the reference's
 * rounding exactly: complex products are (ar*br - ai*bi, ar*bi + ai*br) with
 * every product rounded (build with -ffp-contract=off), sums are evaluated
 * left to right, and quantisation uses the same libm log2/llround/exp2 calls.
 * Pinned byte-for-byte against oracle/_ref (the reference itself) by
 * tests/test_oracle.py.
 */
#define _GNU_SOURCE
#include "cbq_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* cbqo_last_error(void) { return g_err; }

uint64_t cbqo_fnv1a64(const uint8_t* data, uint64_t len, uint64_t h) {
    if (h == 0) h = 0xcbf29ce484222325ull;
    for (uint64_t i = 0; i < len; ++i) {
        h ^= data[i];
        h *= 0x100000001b3ull;
    }
    return h;
}

/* ---------------------------------------------------------------- complex */

typedef struct {
    double re, im;
} cx;

static inline cx cx_mul(cx a, cx b) { /* libstdc++ operator* without -ffast-math */
    cx r;
    r.re = a.re * b.re - a.im * b.im;
    r.im = a.re * b.im + a.im * b.re;
    return r;
}
static inline cx cx_add(cx a, cx b) {
    cx r = {a.re + b.re, a.im + b.im};
    return r;
}

/* ------------------------------------------------------------ error bound */

/* ErrorBound (codec.hpp:19-29): b_a = log2(1 + b_r), b_r > 0 and finite. */
int cbqo_log2_abs(double b_r, double* out) {
    if (!(b_r > 0.0) || isinf(b_r))
        return fail(CBQO_INVALID_ARGUMENT, "relative error bound must be positive and finite");
    *out = log2(1.0 + b_r);
    return CBQO_OK;
}

/* ----------------------------------------------------------------- prescan */

enum { CHUNK_BITS = 4096, CHUNK_WORDS = 64, CHUNK_BYTES = 512 };

static uint64_t chunk_count(uint64_t bits) { return (bits + CHUNK_BITS - 1) / CHUNK_BITS; }
static uint64_t tag_bytes(uint64_t bits) { return (chunk_count(bits) + 3) / 4; }

/* prescan_encode (bitmap.hpp:109-145): 2-bit tag per 4096-bit chunk
 * (0 all-zero, 1 all-one, 2 mixed), raw bytes for mixed chunks only; a final
 * partial chunk is always mixed. Writes tags then raw; returns bytes written. */
static uint64_t prescan_write(const uint64_t* words, uint64_t bits, uint8_t* out) {
    const uint64_t nch = chunk_count(bits), ntag = tag_bytes(bits);
    memset(out, 0, ntag);
    uint64_t pos = ntag;
    for (uint64_t c = 0; c < nch; ++c) {
        const uint64_t first = c * CHUNK_BITS;
        const uint64_t len = bits - first < CHUNK_BITS ? bits - first : CHUNK_BITS;
        const uint64_t* w = words + c * CHUNK_WORDS;
        unsigned tag = 2;
        if (len == CHUNK_BITS) {
            int zeros = 1, ones = 1;
            for (int k = 0; k < CHUNK_WORDS; ++k) {
                zeros &= w[k] == 0;
                ones &= w[k] == ~0ull;
            }
            tag = zeros ? 0u : (ones ? 1u : 2u);
        }
        out[c / 4] |= (uint8_t)(tag << (2 * (c % 4)));
        if (tag == 2) {
            const uint64_t nb = (len + 7) / 8;
            memcpy(out + pos, w, nb); /* little-endian words -> bytes */
            pos += nb;
        }
    }
    return pos;
}

static uint64_t prescan_size(const uint64_t* words, uint64_t bits) {
    uint64_t size = tag_bytes(bits);
    for (uint64_t c = 0; c < chunk_count(bits); ++c) {
        const uint64_t first = c * CHUNK_BITS;
        const uint64_t len = bits - first < CHUNK_BITS ? bits - first : CHUNK_BITS;
        int mixed = len < CHUNK_BITS;
        if (!mixed) {
            const uint64_t* w = words + c * CHUNK_WORDS;
            int zeros = 1, ones = 1;
            for (int k = 0; k < CHUNK_WORDS; ++k) {
                zeros &= w[k] == 0;
                ones &= w[k] == ~0ull;
            }
            mixed = !zeros && !ones;
        }
        if (mixed) size += (len + 7) / 8;
    }
    return size;
}

int cbqo_prescan_encode(const uint64_t* words, uint64_t bits, uint8_t* out, uint64_t cap,
                        uint64_t* size) {
    const uint64_t nw = (bits + 63) / 64;
    uint64_t* tmp = calloc(nw ? nw : 1, sizeof(uint64_t));
    if (nw) memcpy(tmp, words, nw * 8);
    if (bits % 64 && nw) tmp[nw - 1] &= (1ull << (bits % 64)) - 1;
    *size = prescan_size(tmp, bits);
    if (*size > cap) {
        free(tmp);
        return fail(CBQO_BUFFER_TOO_SMALL, "prescan buffer too small");
    }
    prescan_write(tmp, bits, out);
    free(tmp);
    return CBQO_OK;
}

/* read_prescan + prescan_decode (codec.hpp:190-209, bitmap.hpp:147-189). */
static int prescan_read(const uint8_t* p, uint64_t size, uint64_t* pos, uint64_t bits,
                        uint64_t* words, const char* seg) {
    const uint64_t nch = chunk_count(bits), ntag = tag_bytes(bits);
    if (size - *pos < ntag) return fail(CBQO_CODEC, "%s truncated", seg);
    const uint8_t* tags = p + *pos;
    *pos += ntag;
    uint64_t raw = 0;
    for (uint64_t c = 0; c < nch; ++c) {
        const uint64_t first = c * CHUNK_BITS;
        const uint64_t len = bits - first < CHUNK_BITS ? bits - first : CHUNK_BITS;
        const unsigned tag = (tags[c / 4] >> (2 * (c % 4))) & 3u;
        if (tag > 2) return fail(CBQO_CODEC, "bitmap tag stream corrupt: invalid chunk tag");
        if (tag == 2)
            raw += (len + 7) / 8;
        else if (len < CHUNK_BITS)
            return fail(CBQO_CODEC, "bitmap final partial chunk must be stored raw");
    }
    if (size - *pos < raw) return fail(CBQO_CODEC, "%s truncated", seg);
    const uint8_t* src = p + *pos;
    *pos += raw;
    uint64_t off = 0;
    for (uint64_t c = 0; c < nch; ++c) {
        const uint64_t first = c * CHUNK_BITS;
        const uint64_t len = bits - first < CHUNK_BITS ? bits - first : CHUNK_BITS;
        const unsigned tag = (tags[c / 4] >> (2 * (c % 4))) & 3u;
        uint64_t* w = words + c * CHUNK_WORDS;
        if (tag == 1) {
            for (int k = 0; k < CHUNK_WORDS; ++k) w[k] = ~0ull;
        } else if (tag == 2) {
            const uint64_t nb = (len + 7) / 8;
            memcpy(w, src + off, nb);
            off += nb;
            if (len % 64) w[len / 64] &= (1ull << (len % 64)) - 1;
        }
    }
    return CBQO_OK;
}

/* ------------------------------------------------------------------ codec */

enum { HEADER_BYTES = 26 };

static void put_u64(uint8_t* p, uint64_t v) {
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static uint64_t get_u64(const uint8_t* p) {
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

static unsigned bit_width_u64(uint64_t x) { return x ? 64u - (unsigned)__builtin_clzll(x) : 0u; }

uint64_t cbqo_compress_bound(uint64_t n) {
    return HEADER_BYTES + 2 * (tag_bytes(n) + (n + 7) / 8 + 8) + n * 8 + 8;
}

/* compress_block (codec.hpp:227-295). */
int cbqo_compress_block(const double* s, uint64_t n, double b_r, uint8_t* out, uint64_t cap,
                        uint64_t* size) {
    double b_a;
    int rc = cbqo_log2_abs(b_r, &b_a);
    if (rc) return rc;
    const uint64_t nw = (n + 63) / 64 + CHUNK_WORDS;
    uint64_t* signs = calloc(nw, 8);
    uint64_t* zeros = calloc(nw, 8);
    int64_t* q = malloc((n ? n : 1) * sizeof(int64_t));
    uint64_t nnz = 0;
    rc = CBQO_OK;
    for (uint64_t i = 0; i < n && !rc; ++i) {
        const double v = s[i];
        if (isnan(v) || isinf(v)) {
            rc = fail(CBQO_CODEC, "input scalars must be finite");
            break;
        }
        if (v < 0.0) signs[i / 64] |= 1ull << (i % 64);
        if (v == 0.0) {
            zeros[i / 64] |= 1ull << (i % 64);
        } else {
            const double x = log2(fabs(v)) / b_a;
            if (fabs(x) > 0x1.0p62) {
                rc = fail(CBQO_CODEC, "quantized magnitude exceeds the 63-bit code range");
                break;
            }
            q[nnz++] = llround(x);
        }
    }
    if (!rc) {
        int64_t qmin = 0, qmax = 0;
        uint8_t width = 0, flags = 0;
        if (nnz == 0) {
            flags = 1;
        } else {
            qmin = qmax = q[0];
            for (uint64_t k = 1; k < nnz; ++k) {
                if (q[k] < qmin) qmin = q[k];
                if (q[k] > qmax) qmax = q[k];
            }
            const unsigned bw = bit_width_u64((uint64_t)(qmax - qmin));
            width = (uint8_t)(bw > 1 ? bw : 1);
        }
        uint64_t need = HEADER_BYTES;
        if (!flags) need += prescan_size(signs, n) + prescan_size(zeros, n) + (nnz * width + 7) / 8;
        *size = need;
        if (need > cap) {
            rc = fail(CBQO_BUFFER_TOO_SMALL, "payload buffer too small");
        } else {
            put_u64(out, n);
            uint64_t bits;
            memcpy(&bits, &b_r, 8);
            put_u64(out + 8, bits);
            put_u64(out + 16, (uint64_t)qmin);
            out[24] = width;
            out[25] = flags;
            if (!flags) {
                uint64_t pos = HEADER_BYTES;
                pos += prescan_write(signs, n, out + pos);
                pos += prescan_write(zeros, n, out + pos);
                /* BitWriter (codec.hpp:144-161): LSB-first fixed-width codes */
                const uint64_t nbytes = (nnz * width + 7) / 8;
                memset(out + pos, 0, nbytes);
                uint64_t bit = 0;
                for (uint64_t k = 0; k < nnz; ++k) {
                    const uint64_t code = (uint64_t)(q[k] - qmin);
                    for (unsigned j = 0; j < width; ++j, ++bit)
                        out[pos + bit / 8] |= (uint8_t)(((code >> j) & 1u) << (bit % 8));
                }
            }
        }
    }
    free(signs);
    free(zeros);
    free(q);
    return rc;
}

/* decompress_block (codec.hpp:299-344). */
int cbqo_decompress_block(const uint8_t* p, uint64_t size, double* out, uint64_t cap,
                          uint64_t* count) {
    if (size < HEADER_BYTES) return fail(CBQO_CODEC, "header truncated");
    const uint64_t n = get_u64(p);
    double b_r;
    const uint64_t bb = get_u64(p + 8);
    memcpy(&b_r, &bb, 8);
    const int64_t code_min = (int64_t)get_u64(p + 16);
    const unsigned width = p[24], flags = p[25];
    if (!(b_r > 0.0) || isnan(b_r) || isinf(b_r))
        return fail(CBQO_CODEC, "header: invalid relative error bound");
    *count = n;
    if (flags & 1u) {
        if (size != HEADER_BYTES) return fail(CBQO_CODEC, "header: trailing bytes after payload");
        if (n > cap) return fail(CBQO_BUFFER_TOO_SMALL, "scalar buffer too small");
        for (uint64_t i = 0; i < n; ++i) out[i] = 0.0;
        return CBQO_OK;
    }
    const uint64_t nw = (n + 63) / 64 + CHUNK_WORDS;
    uint64_t* signs = calloc(nw, 8);
    uint64_t* zeros = calloc(nw, 8);
    uint64_t pos = HEADER_BYTES;
    int rc = prescan_read(p, size, &pos, n, signs, "sign bitmap");
    if (!rc) rc = prescan_read(p, size, &pos, n, zeros, "zero bitmap");
    if (!rc) {
        uint64_t pc = 0;
        for (uint64_t w = 0; w < (n + 63) / 64; ++w) pc += (uint64_t)__builtin_popcountll(zeros[w]);
        const uint64_t nnz = n - pc;
        if (width == 0 && nnz > 0) {
            rc = fail(CBQO_CODEC, "codes: width zero with nonzero scalars present");
        } else {
            const uint64_t nbytes = (nnz * width + 7) / 8;
            if (size - pos < nbytes) {
                rc = fail(CBQO_CODEC, "codes truncated");
            } else if (size - pos != nbytes) {
                rc = fail(CBQO_CODEC, "codes: trailing bytes after payload");
            } else if (n > cap) {
                rc = fail(CBQO_BUFFER_TOO_SMALL, "scalar buffer too small");
            } else {
                const uint8_t* codes = p + pos;
                const double b_a = log2(1.0 + b_r);
                uint64_t bit = 0;
                for (uint64_t i = 0; i < n; ++i) {
                    if ((zeros[i / 64] >> (i % 64)) & 1u) {
                        out[i] = 0.0;
                        continue;
                    }
                    uint64_t code = 0;
                    for (unsigned j = 0; j < width; ++j, ++bit)
                        code |= (uint64_t)((codes[bit / 8] >> (bit % 8)) & 1u) << j;
                    const int64_t qq = (int64_t)code + code_min;
                    const double mag = exp2((double)qq * b_a);
                    out[i] = ((signs[i / 64] >> (i % 64)) & 1u) ? -mag : mag;
                }
            }
        }
    }
    free(signs);
    free(zeros);
    return rc;
}

/* ---------------------------------------------------------------- circuit */

static int is_two(uint32_t k) { return k == CBQO_CX || k == CBQO_CZ || k == CBQO_CP; }

static cx polar1(double t) {
    cx r = {cos(t), sin(t)};
    return r;
}

/* unitary2 / unitary4 (circuit.hpp:133-198); row-major, interleaved re/im. */
int cbqo_unitary(const cbqo_gate* g, double* out) {
    const double pi = 3.14159265358979323846;
    const double a = g->angle;
    cx u[16];
    memset(u, 0, sizeof u);
    const cx one = {1, 0}, zero = {0, 0};
    switch (g->kind) {
    case CBQO_H: {
        const double r = 1.0 / sqrt(2.0);
        u[0].re = r; u[1].re = r; u[2].re = r; u[3].re = -r;
        break;
    }
    case CBQO_X: u[1] = one; u[2] = one; break;
    case CBQO_Y: u[1].im = -1; u[2].im = 1; break;
    case CBQO_Z: u[0] = one; u[3].re = -1; break;
    case CBQO_S: u[0] = one; u[3].im = 1; break;
    case CBQO_SDG: u[0] = one; u[3].im = -1; break;
    case CBQO_T: u[0] = one; u[3] = polar1(pi / 4); break;
    case CBQO_TDG: u[0] = one; u[3] = polar1(-pi / 4); break;
    case CBQO_RX: {
        const double c = cos(a / 2), s = sin(a / 2);
        u[0].re = c; u[1].im = -s; u[2].im = -s; u[3].re = c;
        break;
    }
    case CBQO_RY: {
        const double c = cos(a / 2), s = sin(a / 2);
        u[0].re = c; u[1].re = -s; u[2].re = s; u[3].re = c;
        break;
    }
    case CBQO_RZ: u[0] = polar1(-a / 2); u[3] = polar1(a / 2); break;
    case CBQO_P: u[0] = one; u[3] = polar1(a); break;
    case CBQO_CX: u[0] = one; u[5] = one; u[11] = one; u[14] = one; break;
    case CBQO_CZ: u[0] = one; u[5] = one; u[10] = one; u[15].re = -1; break;
    case CBQO_CP: u[0] = one; u[5] = one; u[10] = one; u[15] = polar1(a); break;
    default: return fail(CBQO_LOGIC, "unknown gate kind %u", g->kind);
    }
    (void)zero;
    const int m = is_two(g->kind) ? 16 : 4;
    for (int i = 0; i < m; ++i) {
        out[2 * i] = u[i].re;
        out[2 * i + 1] = u[i].im;
    }
    return CBQO_OK;
}

static int validate_circuit(uint32_t n, const cbqo_gate* g, uint64_t ng) {
    if (n < 1 || n > 62) return fail(CBQO_INVALID_ARGUMENT, "qubit count must be in [1, 62], got %u", n);
    for (uint64_t i = 0; i < ng; ++i) { /* Circuit::add (circuit.hpp:110-127) */
        if (g[i].kind > CBQO_CP) return fail(CBQO_INVALID_ARGUMENT, "unknown gate kind");
        if (g[i].q0 >= n)
            return fail(CBQO_INVALID_ARGUMENT, "gate operand %u out of range for %u qubits", g[i].q0, n);
        if (is_two(g[i].kind)) {
            if (g[i].q1 >= n)
                return fail(CBQO_INVALID_ARGUMENT, "gate operand %u out of range for %u qubits", g[i].q1, n);
            if (g[i].q0 == g[i].q1)
                return fail(CBQO_INVALID_ARGUMENT, "two-qubit gate operands must be distinct");
        }
    }
    return CBQO_OK;
}

/* ------------------------------------------------------------- generators */

typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ull * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

static uint64_t mt64_next(mt64* r) {
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ull) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFull);
            uint64_t xa = x >> 1;
            if (x & 1u) xa ^= 0xB5026F5AA96619E9ull;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

typedef struct {
    cbqo_gate* out;
    uint64_t cap, n;
} gate_sink;

static void emit(gate_sink* s, uint32_t kind, uint32_t q0, uint32_t q1, double angle) {
    if (s->n < s->cap) {
        cbqo_gate g = {kind, q0, is_two(kind) ? q1 : 0u, 0u, angle};
        s->out[s->n] = g;
    }
    s->n++;
}

/* generate_benchmark (benchmarks.hpp:148-166) and make_* (:44-143). */
int cbqo_generate_benchmark(const char* name, uint32_t n, uint32_t layers, uint64_t seed,
                            const char* secret, cbqo_gate* out, uint64_t cap, uint64_t* count) {
    const double pi = 3.14159265358979323846;
    gate_sink s = {out, cap, 0};
    const int ghz = !strcmp(name, "ghz") || !strcmp(name, "cat_state");
    const int bv = !strcmp(name, "bv"), qft = !strcmp(name, "qft"), qaoa = !strcmp(name, "qaoa");
    if (!ghz && !bv && !qft && !qaoa) return fail(CBQO_INVALID_ARGUMENT, "unknown benchmark '%s'", name);
    if (n < 2) return fail(CBQO_INVALID_ARGUMENT, "%s requires at least 2 qubits", name);
    if (n > 62) return fail(CBQO_INVALID_ARGUMENT, "qubit count must be in [1, 62], got %u", n);
    if (ghz) {
        emit(&s, CBQO_H, 0, 0, 0);
        for (uint32_t i = 0; i + 1 < n; ++i) emit(&s, CBQO_CX, i, i + 1, 0);
    } else if (bv) {
        char buf[64];
        const char* sec = secret;
        if (!sec || !*sec) {
            uint32_t k = 0;
            for (; k + 1 < n; ++k) buf[k] = (k % 2 == 0) ? '1' : '0';
            buf[k] = 0;
            sec = buf;
        }
        const size_t len = strlen(sec);
        if (len > n - 1) return fail(CBQO_INVALID_ARGUMENT, "bv secret longer than the %u data qubits", n - 1);
        for (size_t i = 0; i < len; ++i)
            if (sec[i] != '0' && sec[i] != '1')
                return fail(CBQO_INVALID_ARGUMENT, "bv secret must contain only '0' and '1'");
        const uint32_t anc = n - 1;
        emit(&s, CBQO_X, anc, 0, 0);
        for (uint32_t q = 0; q < n; ++q) emit(&s, CBQO_H, q, 0, 0);
        for (uint32_t i = 0; i < len; ++i)
            if (sec[i] == '1') emit(&s, CBQO_CX, i, anc, 0);
        for (uint32_t q = 0; q < n; ++q) emit(&s, CBQO_H, q, 0, 0);
    } else if (qft) {
        for (uint32_t i = n; i-- > 0;) {
            emit(&s, CBQO_H, i, 0, 0);
            for (uint32_t j = i; j-- > 0;) emit(&s, CBQO_CP, j, i, pi / (double)(1ull << (i - j)));
        }
        for (uint32_t i = 0; i < n / 2; ++i) {
            const uint32_t j = n - 1 - i;
            emit(&s, CBQO_CX, i, j, 0);
            emit(&s, CBQO_CX, j, i, 0);
            emit(&s, CBQO_CX, i, j, 0);
        }
    } else {
        if (layers < 1) return fail(CBQO_INVALID_ARGUMENT, "qaoa requires at least one layer");
        const double two_pi = 2.0 * pi;
        mt64 r;
        mt64_seed(&r, seed);
        for (uint32_t l = 0; l < layers; ++l) {
            const double gamma = (double)(mt64_next(&r) >> 11) * 0x1.0p-53 * two_pi;
            const double beta = (double)(mt64_next(&r) >> 11) * 0x1.0p-53 * two_pi;
            for (uint32_t i = 0; i < n; ++i) {
                const uint32_t j = (i + 1) % n;
                emit(&s, CBQO_CX, i, j, 0);
                emit(&s, CBQO_RZ, j, 0, gamma);
                emit(&s, CBQO_CX, i, j, 0);
            }
            for (uint32_t q = 0; q < n; ++q) emit(&s, CBQO_RX, q, 0, beta);
        }
    }
    *count = s.n;
    if (s.n > cap) return fail(CBQO_BUFFER_TOO_SMALL, "gate buffer too small");
    return CBQO_OK;
}

/* -------------------------------------------------------------- partition */

static int check_layout(uint32_t n, uint32_t b) { /* make_layout (partition.hpp:23-31) */
    if (n < 1 || n > 62) return fail(CBQO_INVALID_ARGUMENT, "layout qubit count must be in [1, 62]");
    if (b < 1 || b > n) return fail(CBQO_INVALID_ARGUMENT, "local index bits must be in [1, n]");
    return CBQO_OK;
}

static void set_insert(uint32_t* set, uint32_t* len, uint32_t q, uint32_t b) {
    if (q < b) return;
    uint32_t i = 0;
    while (i < *len && set[i] < q) ++i;
    if (i < *len && set[i] == q) return;
    memmove(set + i + 1, set + i, (*len - i) * sizeof(uint32_t));
    set[i] = q;
    ++*len;
}

/* partition_circuit (partition.hpp:59-101): greedy staging with threshold
 * max(inner_size, 2) on the distinct global operands of the open stage. */
int cbqo_partition(uint32_t n, const cbqo_gate* g, uint64_t ng, uint32_t b, uint32_t inner_size,
                   cbqo_stage* out, uint64_t cap, uint64_t* nstages) {
    int rc = validate_circuit(n, g, ng);
    if (!rc) rc = check_layout(n, b);
    if (rc) return rc;
    const uint32_t thr = inner_size > 2 ? inner_size : 2;
    uint32_t cur[64], cand[64], nc = 0, nd;
    uint64_t begin = 0, ns = 0;
    for (uint64_t i = 0; i < ng; ++i) {
        memcpy(cand, cur, nc * sizeof(uint32_t));
        nd = nc;
        set_insert(cand, &nd, g[i].q0, b);
        if (is_two(g[i].kind)) set_insert(cand, &nd, g[i].q1, b);
        if (nd > thr && i > begin) {
            if (ns < cap) {
                cbqo_stage st;
                memset(&st, 0, sizeof st);
                st.gate_begin = begin;
                st.gate_end = i;
                st.inner_count = nc;
                memcpy(st.inner, cur, nc * sizeof(uint32_t));
                out[ns] = st;
            }
            ++ns;
            begin = i;
            nc = 0;
            set_insert(cur, &nc, g[i].q0, b);
            if (is_two(g[i].kind)) set_insert(cur, &nc, g[i].q1, b);
        } else {
            memcpy(cur, cand, nd * sizeof(uint32_t));
            nc = nd;
        }
    }
    if (begin < ng) {
        if (ns < cap) {
            cbqo_stage st;
            memset(&st, 0, sizeof st);
            st.gate_begin = begin;
            st.gate_end = ng;
            st.inner_count = nc;
            memcpy(st.inner, cur, nc * sizeof(uint32_t));
            out[ns] = st;
        }
        ++ns;
    }
    *nstages = ns;
    if (ns > cap) return fail(CBQO_BUFFER_TOO_SMALL, "stage buffer too small");
    return CBQO_OK;
}

static uint64_t scatter(uint64_t packed, const uint32_t* offs, uint32_t k) {
    uint64_t out = 0;
    for (uint32_t j = 0; j < k; ++j) out |= ((packed >> j) & 1ull) << offs[j];
    return out;
}

typedef struct {
    uint32_t inner_offs[64], outer_offs[64], ni, no;
} group_map;

static int make_group_map(uint32_t n, uint32_t b, const cbqo_stage* st, group_map* m) {
    int rc = check_layout(n, b);
    if (rc) return rc;
    const uint32_t c = n - b;
    m->ni = m->no = 0;
    for (uint32_t i = 0; i < st->inner_count; ++i) {
        const uint32_t q = st->inner[i];
        if (q < b || q >= n)
            return fail(CBQO_INVALID_ARGUMENT, "stage inner index %u outside the global index range", q);
        m->inner_offs[m->ni++] = q - b;
    }
    for (uint32_t off = 0; off < c; ++off) {
        int in = 0;
        for (uint32_t i = 0; i < m->ni; ++i) in |= m->inner_offs[i] == off;
        if (!in) m->outer_offs[m->no++] = off;
    }
    return CBQO_OK;
}

/* enumerate_groups (partition.hpp:120-153): ids row-major, group by group. */
int cbqo_enumerate_groups(uint32_t n, uint32_t b, const cbqo_stage* st, uint64_t* ids,
                          uint64_t cap, uint64_t* count) {
    group_map m;
    int rc = make_group_map(n, b, st, &m);
    if (rc) return rc;
    const uint64_t ng = 1ull << m.no, per = 1ull << m.ni;
    *count = ng * per;
    if (*count > cap) return fail(CBQO_BUFFER_TOO_SMALL, "id buffer too small");
    for (uint64_t o = 0; o < ng; ++o) {
        const uint64_t base = scatter(o, m.outer_offs, m.no);
        for (uint64_t v = 0; v < per; ++v) ids[o * per + v] = base | scatter(v, m.inner_offs, m.ni);
    }
    return CBQO_OK;
}

/* buffer_bit_of_qubit (partition.hpp:158-169). */
int cbqo_buffer_bit_of_qubit(uint32_t n, uint32_t b, const cbqo_stage* st, uint32_t q,
                             uint32_t* out) {
    (void)n;
    if (q < b) {
        *out = q;
        return CBQO_OK;
    }
    for (uint32_t i = 0; i < st->inner_count; ++i)
        if (st->inner[i] == q) {
            *out = b + i;
            return CBQO_OK;
        }
    return fail(CBQO_LOGIC, "qubit %u is an outer index for this stage", q);
}

/* ------------------------------------------------------------------ gates */

/* apply_unitary2 / apply_unitary4 (kernel.hpp:24-64), in place. */
static int apply2(cx* a, uint64_t size, uint32_t bit, const cx* u) {
    if (bit >= 64 || (1ull << bit) >= size) return fail(CBQO_INVALID_ARGUMENT, "gate bit out of range for buffer");
    const uint64_t m = 1ull << bit;
    for (uint64_t base = 0; base < size; base += m << 1)
        for (uint64_t i = base; i < base + m; ++i) {
            const cx a0 = a[i], a1 = a[i | m];
            a[i] = cx_add(cx_mul(u[0], a0), cx_mul(u[1], a1));
            a[i | m] = cx_add(cx_mul(u[2], a0), cx_mul(u[3], a1));
        }
    return CBQO_OK;
}

static int apply4(cx* a, uint64_t size, uint32_t hi, uint32_t lo, const cx* u) {
    if (hi >= 64 || lo >= 64 || (1ull << hi) >= size || (1ull << lo) >= size || hi == lo)
        return fail(CBQO_INVALID_ARGUMENT, "gate bits invalid for buffer");
    const uint64_t mh = 1ull << hi, ml = 1ull << lo;
    const uint64_t low0 = (1ull << (hi < lo ? hi : lo)) - 1, low1 = (1ull << (hi < lo ? lo : hi)) - 1;
    for (uint64_t k = 0; k < size >> 2; ++k) {
        uint64_t i = ((k & ~low0) << 1) | (k & low0);
        i = ((i & ~low1) << 1) | (i & low1);
        const cx a0 = a[i], a1 = a[i | ml], a2 = a[i | mh], a3 = a[i | mh | ml];
        cx r[4];
        for (int row = 0; row < 4; ++row) {
            const cx* ur = u + 4 * row;
            r[row] = cx_add(cx_add(cx_add(cx_mul(ur[0], a0), cx_mul(ur[1], a1)), cx_mul(ur[2], a2)),
                            cx_mul(ur[3], a3));
        }
        a[i] = r[0];
        a[i | ml] = r[1];
        a[i | mh] = r[2];
        a[i | mh | ml] = r[3];
    }
    return CBQO_OK;
}

int cbqo_apply_gate(double* amps, uint64_t namps, const double* u, int two, uint32_t hi, uint32_t lo) {
    cx m[16];
    for (int i = 0; i < (two ? 16 : 4); ++i) {
        m[i].re = u[2 * i];
        m[i].im = u[2 * i + 1];
    }
    return two ? apply4((cx*)amps, namps, hi, lo, m) : apply2((cx*)amps, namps, hi, m);
}

static int apply_stage_cx(cx* a, uint64_t namps, uint32_t n, const cbqo_gate* g,
                          const cbqo_stage* st, uint32_t b) {
    for (uint64_t i = st->gate_begin; i < st->gate_end; ++i) {
        double ud[32];
        cx u[16];
        int rc = cbqo_unitary(&g[i], ud);
        if (rc) return rc;
        const int two = is_two(g[i].kind);
        for (int k = 0; k < (two ? 16 : 4); ++k) {
            u[k].re = ud[2 * k];
            u[k].im = ud[2 * k + 1];
        }
        uint32_t b0, b1 = 0;
        rc = cbqo_buffer_bit_of_qubit(n, b, st, g[i].q0, &b0);
        if (!rc && two) rc = cbqo_buffer_bit_of_qubit(n, b, st, g[i].q1, &b1);
        if (!rc) rc = two ? apply4(a, namps, b0, b1, u) : apply2(a, namps, b0, u);
        if (rc) return rc;
    }
    return CBQO_OK;
}

/* apply_stage (kernel.hpp:111-122). */
int cbqo_apply_stage(double* amps, uint64_t namps, uint32_t n, const cbqo_gate* g, uint64_t ng,
                     const cbqo_stage* st, uint32_t b) {
    int rc = validate_circuit(n, g, ng);
    if (!rc) rc = check_layout(n, b);
    if (rc) return rc;
    if (st->gate_end > ng || st->gate_begin > st->gate_end)
        return fail(CBQO_INVALID_ARGUMENT, "stage gate range out of bounds");
    return apply_stage_cx((cx*)amps, namps, n, g, st, b);
}

/* -------------------------------------------------------------- simulator */

/* Payload objects with reference counts: the store's memory/spill accounting
 * (store.hpp:64-117,188-232) replayed sequentially (worker count 1). */
typedef struct {
    uint8_t* data;
    uint64_t size;
    uint64_t refs;
    int spilled;
} pobj;

typedef struct {
    pobj** by_id;
    uint64_t budget, resident, spilled_live, peak, spilled_blocks;
} store_t;

static void store_detach(store_t* s, uint64_t id) {
    pobj* o = s->by_id[id];
    if (!o) return;
    s->by_id[id] = NULL;
    if (--o->refs == 0) {
        if (o->spilled)
            s->spilled_live -= o->size;
        else
            s->resident -= o->size;
        free(o->data);
        free(o);
    }
}

static pobj* store_place(store_t* s, uint8_t* data, uint64_t size) {
    pobj* o = calloc(1, sizeof *o);
    o->data = data;
    o->size = size;
    const int fits = size <= s->budget && s->resident <= s->budget - size;
    if (fits) {
        s->resident += size;
    } else {
        o->spilled = 1;
        s->spilled_live += size;
        s->spilled_blocks++;
    }
    return o;
}

static void store_finish(store_t* s) {
    const uint64_t t = s->resident + s->spilled_live;
    if (t > s->peak) s->peak = t;
}

static void store_put(store_t* s, uint64_t id, uint8_t* data, uint64_t size) {
    store_detach(s, id);
    pobj* o = store_place(s, data, size);
    o->refs = 1;
    s->by_id[id] = o;
    store_finish(s);
}

static int pack_block(const cx* blk, uint64_t bs, int compress, double b_r, uint8_t** out,
                      uint64_t* size) {
    double* sc = malloc(2 * bs * sizeof(double));
    for (uint64_t i = 0; i < bs; ++i) {
        sc[i] = blk[i].re;
        sc[bs + i] = blk[i].im;
    }
    int rc = CBQO_OK;
    if (compress) {
        const uint64_t cap = cbqo_compress_bound(2 * bs);
        *out = malloc(cap);
        rc = cbqo_compress_block(sc, 2 * bs, b_r, *out, cap, size);
    } else {
        *size = 2 * bs * sizeof(double);
        *out = malloc(*size);
        memcpy(*out, sc, *size);
    }
    free(sc);
    return rc;
}

static int unpack_block(const pobj* o, uint64_t bs, int compress, cx* blk, double* scratch) {
    uint64_t cnt;
    if (compress) {
        int rc = cbqo_decompress_block(o->data, o->size, scratch, 2 * bs + 1, &cnt);
        if (rc == CBQO_BUFFER_TOO_SMALL) cnt = 2 * bs + 1;
        else if (rc) return rc;
    } else {
        if (o->size % 16) return fail(CBQO_ENGINE, "raw block payload has invalid length");
        cnt = o->size / 8;
        if (cnt == 2 * bs) memcpy(scratch, o->data, o->size);
    }
    if (cnt != 2 * bs) return fail(CBQO_ENGINE, "block payload scalar count does not match the layout");
    for (uint64_t i = 0; i < bs; ++i) {
        blk[i].re = scratch[i];
        blk[i].im = scratch[bs + i];
    }
    return CBQO_OK;
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

/* Simulator::init_state + run + state_norm (engine.hpp:74-158), sequential
 * group order (parallel_for with one worker). */
int cbqo_simulate(uint32_t n, const cbqo_gate* g, uint64_t ng, uint32_t b, uint32_t inner_size,
                  double b_r, uint64_t budget, int compress, cbqo_report* rep, uint8_t* payloads,
                  uint64_t pay_cap, uint64_t* pay_sizes, double* state) {
    const double t0 = now_ms();
    int rc = validate_circuit(n, g, ng);
    if (!rc) rc = check_layout(n, b);
    double b_a;
    if (!rc) rc = cbqo_log2_abs(b_r, &b_a);
    if (rc) return rc;
    const uint32_t c = n - b;
    const uint64_t nblk = 1ull << c, bs = 1ull << b;
    uint64_t nst;
    rc = cbqo_partition(n, g, ng, b, inner_size, NULL, 0, &nst);
    if (rc && rc != CBQO_BUFFER_TOO_SMALL) return rc;
    cbqo_stage* stages = calloc(nst ? nst : 1, sizeof *stages);
    cbqo_partition(n, g, ng, b, inner_size, stages, nst, &nst);

    store_t s;
    memset(&s, 0, sizeof s);
    s.budget = budget;
    s.by_id = calloc(nblk, sizeof(pobj*));
    cx* blk = calloc(bs, sizeof(cx));
    double* scratch = malloc((2 * bs + 1) * sizeof(double));
    uint8_t* pd;
    uint64_t psz;
    blk[0].re = 1.0;
    rc = pack_block(blk, bs, compress, b_r, &pd, &psz);
    if (!rc) store_put(&s, 0, pd, psz);
    if (!rc && c > 0) {
        blk[0].re = 0.0;
        rc = pack_block(blk, bs, compress, b_r, &pd, &psz);
        if (!rc) { /* put_shared (store.hpp:85-117) */
            for (uint64_t id = 1; id < nblk; ++id) store_detach(&s, id);
            pobj* o = store_place(&s, pd, psz);
            o->refs = nblk - 1;
            for (uint64_t id = 1; id < nblk; ++id) s.by_id[id] = o;
            store_finish(&s);
        }
    }
    uint64_t comp_calls = 0, decomp_calls = 0;
    uint64_t* ids = NULL;
    cx* buf = NULL;
    for (uint64_t si = 0; si < nst && !rc; ++si) {
        const cbqo_stage* st = &stages[si];
        uint64_t nid;
        rc = cbqo_enumerate_groups(n, b, st, NULL, 0, &nid);
        if (rc != CBQO_BUFFER_TOO_SMALL && rc) break;
        rc = CBQO_OK;
        ids = realloc(ids, nid * sizeof(uint64_t));
        cbqo_enumerate_groups(n, b, st, ids, nid, &nid);
        const uint64_t per = 1ull << st->inner_count, ngr = nid / per;
        buf = realloc(buf, per * bs * sizeof(cx));
        for (uint64_t gi = 0; gi < ngr && !rc; ++gi) {
            const uint64_t* gid = ids + gi * per;
            for (uint64_t v = 0; v < per && !rc; ++v)
                rc = unpack_block(s.by_id[gid[v]], bs, compress, buf + v * bs, scratch);
            decomp_calls += per;
            if (!rc) rc = apply_stage_cx(buf, per * bs, n, g, st, b);
            for (uint64_t v = 0; v < per && !rc; ++v) {
                rc = pack_block(buf + v * bs, bs, compress, b_r, &pd, &psz);
                if (!rc) store_put(&s, gid[v], pd, psz);
            }
            if (!rc) comp_calls += per;
            if (rc) {
                char msg[640];
                snprintf(msg, sizeof msg, "stage %llu: group with outer value %llu: %s",
                         (unsigned long long)si, (unsigned long long)gi, g_err);
                rc = fail(CBQO_ENGINE, "%s", msg);
            }
        }
    }
    double sum = 0.0;
    for (uint64_t id = 0; id < nblk && !rc; ++id) {
        rc = unpack_block(s.by_id[id], bs, compress, blk, scratch);
        for (uint64_t i = 0; i < bs && !rc; ++i) {
            sum += blk[i].re * blk[i].re + blk[i].im * blk[i].im;
            if (state) {
                state[2 * (id * bs + i)] = blk[i].re;
                state[2 * (id * bs + i) + 1] = blk[i].im;
            }
        }
    }
    if (!rc && rep) {
        memset(rep, 0, sizeof *rep);
        rep->qubits = n;
        rep->gate_count = ng;
        rep->stage_count = nst;
        rep->max_footprint_bytes = s.peak;
        rep->standard_bytes = exp2((double)(n + 4));
        rep->compression_ratio = s.peak ? rep->standard_bytes / (double)s.peak : 0.0;
        rep->spilled_blocks = s.spilled_blocks;
        rep->final_norm = sqrt(sum);
        rep->stage_compress_calls = comp_calls;
        rep->stage_decompress_calls = decomp_calls;
        rep->wall_ms = now_ms() - t0;
    }
    if (!rc && pay_sizes) {
        uint64_t off = 0;
        for (uint64_t id = 0; id < nblk && !rc; ++id) {
            const pobj* o = s.by_id[id];
            pay_sizes[id] = o->size;
            if (payloads) {
                if (off + o->size > pay_cap) rc = fail(CBQO_BUFFER_TOO_SMALL, "payload buffer too small");
                else memcpy(payloads + off, o->data, o->size);
            }
            off += o->size;
        }
    }
    for (uint64_t id = 0; id < nblk; ++id) store_detach(&s, id);
    free(s.by_id);
    free(blk);
    free(scratch);
    free(ids);
    free(buf);
    free(stages);
    return rc;
}

/* dense_reference (engine.hpp:254-296): full-vector FP64 from e0. */
int cbqo_dense_reference(uint32_t n, const cbqo_gate* g, uint64_t ng, double* out) {
    int rc = validate_circuit(n, g, ng);
    if (rc) return rc;
    if (n > 30) return fail(CBQO_ENGINE, "dense reference refused: %u qubits exceeds the cap of 30", n);
    const uint64_t N = 1ull << n;
    cx* a = (cx*)out;
    memset(a, 0, N * sizeof(cx));
    a[0].re = 1.0;
    for (uint64_t i = 0; i < ng; ++i) {
        double ud[32];
        cx u[16];
        cbqo_unitary(&g[i], ud);
        const int two = is_two(g[i].kind);
        for (int k = 0; k < (two ? 16 : 4); ++k) {
            u[k].re = ud[2 * k];
            u[k].im = ud[2 * k + 1];
        }
        if (two) {
            const uint64_t mh = 1ull << g[i].q0, ml = 1ull << g[i].q1;
            for (uint64_t x = 0; x < N; ++x) {
                if ((x & mh) || (x & ml)) continue;
                const cx a0 = a[x], a1 = a[x | ml], a2 = a[x | mh], a3 = a[x | mh | ml];
                cx r[4];
                for (int row = 0; row < 4; ++row) {
                    const cx* ur = u + 4 * row;
                    r[row] = cx_add(cx_add(cx_add(cx_mul(ur[0], a0), cx_mul(ur[1], a1)), cx_mul(ur[2], a2)),
                                    cx_mul(ur[3], a3));
                }
                a[x] = r[0];
                a[x | ml] = r[1];
                a[x | mh] = r[2];
                a[x | mh | ml] = r[3];
            }
        } else {
            const uint64_t m = 1ull << g[i].q0;
            for (uint64_t x = 0; x < N; ++x) {
                if (x & m) continue;
                const cx a0 = a[x], a1 = a[x | m];
                a[x] = cx_add(cx_mul(u[0], a0), cx_mul(u[1], a1));
                a[x | m] = cx_add(cx_mul(u[2], a0), cx_mul(u[3], a1));
            }
        }
    }
    return CBQO_OK;
}

/* fidelity (engine.hpp:299-308): |sum conj(a_i) b_i|, unnormalised. */
int cbqo_fidelity(const double* a, const double* b, uint64_t namps, double* out) {
    cx acc = {0, 0};
    for (uint64_t i = 0; i < namps; ++i) {
        const cx ca = {a[2 * i], -a[2 * i + 1]}, bb = {b[2 * i], b[2 * i + 1]};
        acc = cx_add(acc, cx_mul(ca, bb));
    }
    *out = hypot(acc.re, acc.im);
    return CBQO_OK;
}
