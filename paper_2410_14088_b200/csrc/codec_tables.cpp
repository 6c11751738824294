// codec_tables.cpp — exact quantiser / dequantiser tables (host, built once
// per relative bound with the same libm the reference links).
//
// The reference quantises a nonzero scalar v as
//     q = llround(log2(|v|) / b_a),   b_a = log2(1 + b_r)      (codec.hpp:249-253)
// and reconstructs exp2(q * b_a)                                   (codec.hpp:340).
// CUDA's log2/exp2 are not bit-identical to glibc's, so the device never
// evaluates them on the hot path. Because f(v) = llround(log2 v / b_a) is
// monotone in v, it is fully described by its thresholds
//     T[q] = min { v > 0 : f(v) >= q },
// found here by bisection on the IEEE bit pattern using std::log2 itself.
// The device estimates q with a float log2 and corrects it with two integer
// compares against T, which reproduces glibc's f bit-for-bit; exp2 becomes a
// table lookup E[q]. Entries span every positive finite double when the
// table fits (b_r >= ~2e-5); narrower bounds get a window anchored at the
// top of the range and values below it are rejected loudly by the kernels.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>

#include "bmq_internal.hpp"

namespace bmq {
namespace {

constexpr uint64_t kMaxEntries = 1ull << 25;
constexpr uint64_t kInfBits = 0x7ff0000000000000ull;

inline double from_bits(uint64_t b) {
    double d;
    std::memcpy(&d, &b, 8);
    return d;
}
inline uint64_t to_bits(double d) {
    uint64_t b;
    std::memcpy(&b, &d, 8);
    return b;
}

struct Quantiser {
    double b_a;
    // The reference expression, evaluated exactly as compress_block does.
    int64_t operator()(uint64_t bits) const {
        return std::llround(std::log2(std::fabs(from_bits(bits))) / b_a);
    }
};

// Smallest positive bit pattern v with f(v) >= q, given f(lo) < q <= f(hi).
uint64_t bisect(const Quantiser& f, int64_t q, uint64_t lo, uint64_t hi) {
    while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (f(mid) >= q)
            hi = mid;
        else
            lo = mid;
    }
    return hi;
}

uint64_t threshold(const Quantiser& f, int64_t q, uint64_t max_bits) {
    const double guess = std::exp2((static_cast<double>(q) - 0.5) * f.b_a);
    uint64_t g = to_bits(std::min(std::max(guess, DBL_TRUE_MIN), DBL_MAX));
    uint64_t span = 1ull << 10;  // ulps; the guess is within ~400 ulps
    for (;;) {
        const uint64_t lo = g > span ? g - span : 1;
        const uint64_t hi = std::min(g + span, max_bits);
        const bool lo_ok = lo == 1 ? f(1) < q : f(lo) < q;
        const bool hi_ok = f(hi) >= q;
        if (lo == 1 && !lo_ok) return 1;  // q at/below the bottom of the range
        if (lo_ok && hi_ok) return bisect(f, q, lo, hi);
        if (hi == max_bits && !hi_ok) return kInfBits;
        span <<= 2;
    }
}

std::unique_ptr<CodecTables> build(double b_r) {
    if (!(b_r > 0.0) || std::isinf(b_r))
        raise(BMQ_ERR_INVALID_ARGUMENT, "relative error bound must be positive and finite");
    auto t = std::make_unique<CodecTables>();
    t->b_r = b_r;
    t->b_a = std::log2(1.0 + b_r);
    const Quantiser f{t->b_a};
    const uint64_t max_bits = to_bits(DBL_MAX);
    const int64_t qtop = f(max_bits);
    t->qhi = qtop;
    t->qlo = f(1);  // DBL_TRUE_MIN
    if (static_cast<uint64_t>(t->qhi - t->qlo) + 2 > kMaxEntries) {
        // Tiny bounds: keep a window of kMaxEntries codes for magnitudes up
        // to 2^32 and down from there (amplitudes are at most 1); scalars
        // outside it are rejected as out of window.
        t->qhi = std::min(qtop, f(to_bits(0x1p32)));
        t->qlo = t->qhi - static_cast<int64_t>(kMaxEntries) + 2;
    }
    const uint64_t count = static_cast<uint64_t>(t->qhi - t->qlo) + 1;
    t->thresh.assign(count + 1, kInfBits);
    if (t->qhi < qtop) t->thresh[count] = threshold(f, t->qhi + 1, max_bits);  // top of the window
    t->dequant.assign(count, 0.0);
    unsigned nthreads = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    std::vector<int64_t> worst_lo(nthreads, INT64_MIN), worst_hi(nthreads, INT64_MAX);
    for (unsigned w = 0; w < nthreads; ++w) {
        pool.emplace_back([&, w] {
            const uint64_t begin = count * w / nthreads, end = count * (w + 1) / nthreads;
            for (uint64_t i = begin; i < end; ++i) {
                const int64_t q = t->qlo + static_cast<int64_t>(i);
                t->thresh[i] = (i == 0 && f(1) >= q) ? 1 : threshold(f, q, max_bits);
                const double e = std::exp2(static_cast<double>(q) * t->b_a);
                t->dequant[i] = e;
                // Idempotence of the codec on this code: decompress -> compress
                // must give q back. Only codes compress can emit matter
                // (f(T[q]) == q); failures sit in the coarse subnormal range.
                const bool reachable = t->thresh[i] != kInfBits && f(t->thresh[i]) == q;
                if (reachable && (!(e > 0.0) || !(e <= DBL_MAX) || f(to_bits(e)) != q)) {
                    if (q < 0)
                        worst_lo[w] = std::max(worst_lo[w], q);
                    else
                        worst_hi[w] = std::min(worst_hi[w], q);
                }
            }
        });
    }
    for (auto& th : pool) th.join();
    int64_t lo = INT64_MIN, hi = INT64_MAX;
    for (unsigned w = 0; w < nthreads; ++w) {
        lo = std::max(lo, worst_lo[w]);
        hi = std::min(hi, worst_hi[w]);
    }
    t->idem_lo = lo == INT64_MIN ? t->qlo : lo + 1;
    t->idem_hi = hi == INT64_MAX ? t->qhi : hi - 1;
    // thresh must be non-decreasing for the device search to be exact.
    for (uint64_t i = 1; i <= count; ++i)
        if (t->thresh[i] < t->thresh[i - 1])
            raise(BMQ_ERR_LOGIC, "quantiser threshold table is not monotone");
    return t;
}

}  // namespace

const CodecTables& host_tables(double b_r) {
    static std::mutex mu;
    static std::map<uint64_t, std::unique_ptr<CodecTables>> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto& slot = cache[to_bits(b_r)];
    if (!slot) slot = build(b_r);
    return *slot;
}

}  // namespace bmq
