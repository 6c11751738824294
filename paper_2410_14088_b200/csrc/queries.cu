// queries.cu — measurement-style queries on the compressed state (SURVEY §8
// f3). The reference only offers the dense extract_state, capped at 24
// qubits (engine.hpp:138-147); these answer the questions a caller of a
// 34-36 qubit state asks without ever materialising it:
//
//  sample(): basis-state indices drawn from |a_i|^2 / sum |a|^2. A block is
//    chosen by its probability mass (the per-block sums the engine keeps,
//    k_dec_chunk<kSumsOnly>), then only the blocks that received shots are
//    decoded and each shot is resolved inside its block by a fixed-order
//    prefix of |a|^2 (deterministic for a given seed).
//  top_k(): the k amplitudes of largest |a|^2 (ties to the lower index), by
//    a radix select on the IEEE bits of |a|^2 (order-preserving for
//    non-negative doubles): histogram passes over the decoded blocks fix the
//    k-th key 12 bits at a time (at most six), a count pass and a collect
//    pass take the keys above it and, in index order, the ties needed to
//    make k.
#include <cub/block/block_scan.cuh>

#include <algorithm>
#include <numeric>
#include <random>

#include "engine.cuh"
#include "codec.cuh"

namespace bmq {

namespace {

constexpr int kQThreads = 256;

__device__ __forceinline__ double prob_at(const double* blk, uint64_t half, uint64_t i) {
    const double re = blk[i], im = blk[half + i];
    return __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
}

// One CTA per block with shots: thread t owns amplitudes [t * per, (t+1) * per)
// of the block; inclusive prefix of the thread totals, then every shot finds
// its thread by bisection and walks that thread's range.
__global__ void __launch_bounds__(kQThreads) k_sample_blocks(const double* __restrict__ work, uint32_t b,
                                                              const uint32_t* __restrict__ slot_of,
                                                              const uint64_t* __restrict__ shot_off,
                                                              const double* __restrict__ shot_u,
                                                              uint64_t* __restrict__ local) {
    const uint32_t k = blockIdx.x;
    const uint64_t half = 1ull << b;
    const double* blk = work + static_cast<uint64_t>(slot_of[k]) * (2ull << b);
    const uint64_t per = half >= kQThreads ? half / kQThreads : 1;
    const uint32_t tid = threadIdx.x;
    double tot = 0.0;
    uint64_t last_nz = 0;
    bool any = false;
    if (tid * per < half) {
        for (uint64_t i = tid * per; i < (tid + 1) * per; ++i) {
            const double p = prob_at(blk, half, i);
            tot = __dadd_rn(tot, p);
            if (p > 0.0) last_nz = i, any = true;
        }
    }
    using Scan = cub::BlockScan<double, kQThreads>;
    __shared__ typename Scan::TempStorage ss;
    __shared__ double incl[kQThreads];
    __shared__ unsigned long long s_last;
    if (tid == 0) s_last = 0;
    __syncthreads();
    double pre;
    Scan(ss).InclusiveScan(tot, pre, [](double a, double c) { return __dadd_rn(a, c); });
    incl[tid] = pre;
    if (any) atomicMax(&s_last, static_cast<unsigned long long>(last_nz));
    __syncthreads();
    for (uint64_t s = shot_off[k] + tid; s < shot_off[k + 1]; s += kQThreads) {
        const double u = shot_u[s];
        // first thread whose inclusive prefix exceeds u
        int lo = 0, hi = kQThreads - 1;
        while (lo < hi) {
            const int mid = (lo + hi) / 2;
            if (incl[mid] > u) hi = mid; else lo = mid + 1;
        }
        uint64_t pick = s_last;  // u at or past the block's total: its last nonzero amplitude
        if (incl[lo] > u && static_cast<uint64_t>(lo) * per < half) {
            double c = lo ? incl[lo - 1] : 0.0;
            for (uint64_t i = lo * per; i < (lo + 1) * per; ++i) {
                const double p = prob_at(blk, half, i);
                c = __dadd_rn(c, p);
                if (p > 0.0 && c > u) {
                    pick = i;
                    break;
                }
            }
        }
        local[s] = pick;
    }
}

__device__ __forceinline__ uint64_t key_at(const double* blk, uint64_t half, uint64_t i) {
    return static_cast<uint64_t>(__double_as_longlong(prob_at(blk, half, i)));
}

// Histogram of key bits [shift, shift + width) (width <= 12) over the keys
// whose bits above shift + width equal `prefix` (one radix-select level);
// per-CTA shared bins, flushed once.
constexpr int kDigitBits = 12;
__global__ void __launch_bounds__(kQThreads) k_topk_hist(const double* __restrict__ work, uint32_t b, uint64_t nblk,
                                                          uint64_t prefix, uint32_t shift, uint32_t width,
                                                          unsigned long long* __restrict__ hist) {
    __shared__ unsigned int h[1 << kDigitBits];
    for (uint32_t i = threadIdx.x; i < (1u << width); i += kQThreads) h[i] = 0;
    __syncthreads();
    const uint64_t half = 1ull << b, total = nblk << b;
    const uint64_t hi_mask = shift + width >= 64 ? 0ull : ~0ull << (shift + width);
    const uint64_t dmask = (1ull << width) - 1;
    for (uint64_t g = blockIdx.x * uint64_t(kQThreads) + threadIdx.x; g < total; g += uint64_t(gridDim.x) * kQThreads) {
        const uint64_t key = key_at(work + (g >> b) * (2ull << b), half, g & (half - 1));
        if ((key & hi_mask) != prefix || key == 0) continue;
        atomicAdd(&h[(key >> shift) & dmask], 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < (1u << width); i += kQThreads)
        if (h[i]) atomicAdd(&hist[i], static_cast<unsigned long long>(h[i]));
}

// Per block: keys above tau and keys equal to tau (counts).
__global__ void __launch_bounds__(kQThreads) k_topk_count(const double* __restrict__ work, uint32_t b, uint64_t tau,
                                                           unsigned long long* __restrict__ above,
                                                           unsigned long long* __restrict__ equal) {
    const uint64_t half = 1ull << b;
    const double* blk = work + blockIdx.x * (2ull << b);
    unsigned long long a = 0, e = 0;
    for (uint64_t i = threadIdx.x; i < half; i += kQThreads) {
        const uint64_t key = key_at(blk, half, i);
        a += key > tau;
        e += key == tau && tau != 0;
    }
    using Scan = cub::BlockScan<unsigned long long, kQThreads>;
    __shared__ typename Scan::TempStorage ss;
    unsigned long long ta, te, pa, pe;
    Scan(ss).ExclusiveSum(a, pa, ta);
    __syncthreads();
    Scan(ss).ExclusiveSum(e, pe, te);
    if (threadIdx.x == 0) {
        above[blockIdx.x] = ta;
        equal[blockIdx.x] = te;
    }
}

// Collect, per block in index order: every key above tau, and the first
// take_eq[blk] keys equal to tau, at out offsets out_a[blk] / out_e[blk].
__global__ void __launch_bounds__(kQThreads) k_topk_collect(const double* __restrict__ work, uint32_t b,
                                                             const uint64_t* __restrict__ ids, uint64_t tau,
                                                             const unsigned long long* __restrict__ out_a,
                                                             const unsigned long long* __restrict__ out_e,
                                                             const unsigned long long* __restrict__ take_eq,
                                                             uint64_t* __restrict__ idx, double* __restrict__ re,
                                                             double* __restrict__ im) {
    const uint64_t half = 1ull << b;
    const double* blk = work + blockIdx.x * (2ull << b);
    const uint64_t base = ids[blockIdx.x] << b;
    using Scan = cub::BlockScan<unsigned int, kQThreads>;
    __shared__ typename Scan::TempStorage ss;
    __shared__ unsigned long long s_a, s_e;
    if (threadIdx.x == 0) s_a = out_a[blockIdx.x], s_e = 0;
    __syncthreads();
    const unsigned long long want_e = take_eq[blockIdx.x];
    for (uint64_t i0 = 0; i0 < half; i0 += kQThreads) {
        const uint64_t i = i0 + threadIdx.x;
        const uint64_t key = i < half ? key_at(blk, half, i) : 0;
        const unsigned fa = i < half && key > tau, fe = i < half && key == tau && tau != 0;
        unsigned pa, pe, ta, te;
        Scan(ss).ExclusiveSum(fa, pa, ta);
        __syncthreads();
        Scan(ss).ExclusiveSum(fe, pe, te);
        if (fa) {
            const unsigned long long o = s_a + pa;
            idx[o] = base | i;
            re[o] = blk[i];
            im[o] = blk[half + i];
        }
        if (fe && s_e + pe < want_e) {
            const unsigned long long o = out_e[blockIdx.x] + s_e + pe;
            idx[o] = base | i;
            re[o] = blk[i];
            im[o] = blk[half + i];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_a += ta;
            s_e += te;
        }
        __syncthreads();
    }
}

}  // namespace

// Decoded planar doubles of blocks ids[0..n) (n <= max_blocks_): work_ for
// compressed states, the dense array itself for raw ones (ids consecutive).
const double* Engine::decoded_batch(const uint64_t* h_ids, uint64_t n) {
    if (!cfg_.compress) {
        for (uint64_t i = 1; i < n; ++i)
            if (h_ids[i] != h_ids[0] + i) raise(BMQ_ERR_LOGIC, "raw batches must be consecutive ids");
        return dense_.p + h_ids[0] * (2ull << L_.b);
    }
    BMQ_CUDA(cudaMemcpyAsync(ids_.p, h_ids, n * sizeof(uint64_t), cudaMemcpyHostToDevice, st_));
    decompress_ids(ids_.p, n, false);
    return work_.p;
}

void Engine::sample(uint64_t nshots, uint64_t seed, uint64_t* out) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    if (!nshots) return;
    const uint64_t nid = L_.num_blocks();
    state_norm();  // fills the per-block sums (sums_) for either state form
    std::vector<double> h(3 * nid);
    BMQ_CUDA(cudaMemcpyAsync(h.data(), sums_.p, sums_.bytes(), cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
    std::vector<double> cdf(nid);
    double acc = 0.0;
    for (uint64_t id = 0; id < nid; ++id) cdf[id] = acc = acc + h[3 * id];
    if (!(acc > 0.0)) raise(BMQ_ERR_ENGINE, "cannot sample a zero state");
    // shots -> (block, target within the block's mass), grouped by block
    std::mt19937_64 gen(seed);
    std::vector<uint64_t> blk(nshots);
    std::vector<double> u(nshots);
    for (uint64_t s = 0; s < nshots; ++s) {
        const double x = static_cast<double>(gen() >> 11) * 0x1p-53 * acc;
        // first block whose cumulative mass exceeds x (it has a positive mass)
        const uint64_t id = std::min<uint64_t>(
            static_cast<uint64_t>(std::upper_bound(cdf.begin(), cdf.end(), x) - cdf.begin()), nid - 1);
        blk[s] = id;
        u[s] = x - (id ? cdf[id - 1] : 0.0);
    }
    std::vector<uint64_t> order(nshots);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t c) { return blk[a] < blk[c]; });
    std::vector<uint64_t> ids;          // blocks with shots, ascending
    std::vector<uint64_t> off;          // CSR over order
    for (uint64_t i = 0; i < nshots; ++i) {
        if (ids.empty() || ids.back() != blk[order[i]]) {
            ids.push_back(blk[order[i]]);
            off.push_back(i);
        }
    }
    off.push_back(nshots);
    std::vector<double> us(nshots);
    for (uint64_t i = 0; i < nshots; ++i) us[i] = u[order[i]];
    DevArray<double> d_u;
    DevArray<uint64_t> d_off, d_local;
    DevArray<uint32_t> d_slot;
    d_u.alloc(nshots);
    d_local.alloc(nshots);
    const uint64_t batch = cfg_.compress ? std::min<uint64_t>(max_blocks_, ids.size()) : 1;  // raw: per block
    d_off.alloc(batch + 1);
    d_slot.alloc(batch);
    std::vector<uint64_t> local(nshots);
    std::vector<uint32_t> slot(batch);
    std::iota(slot.begin(), slot.end(), 0u);
    BMQ_CUDA(cudaMemcpyAsync(d_slot.p, slot.data(), batch * sizeof(uint32_t), cudaMemcpyHostToDevice, st_));
    BMQ_CUDA(cudaMemcpyAsync(d_u.p, us.data(), nshots * sizeof(double), cudaMemcpyHostToDevice, st_));
    for (uint64_t first = 0; first < ids.size(); first += batch) {
        const uint64_t nb = std::min(batch, ids.size() - first);
        const double* w = decoded_batch(ids.data() + first, nb);
        std::vector<uint64_t> o(nb + 1);
        for (uint64_t k = 0; k <= nb; ++k) o[k] = off[first + k] - off[first];
        BMQ_CUDA(cudaMemcpyAsync(d_off.p, o.data(), (nb + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st_));
        k_sample_blocks<<<static_cast<uint32_t>(nb), kQThreads, 0, st_>>>(w, L_.b, d_slot.p, d_off.p,
                                                                         d_u.p + off[first], d_local.p + off[first]);
        BMQ_CUDA(cudaGetLastError());
        BMQ_CUDA(cudaStreamSynchronize(st_));  // ids_ / work_ / d_off are reused by the next batch
    }
    counters_.kernel_launches += ids.size();
    BMQ_CUDA(cudaMemcpyAsync(local.data(), d_local.p, nshots * sizeof(uint64_t), cudaMemcpyDeviceToHost, st_));
    BMQ_CUDA(cudaStreamSynchronize(st_));
    check_device_error("sample: ");
    for (uint64_t i = 0; i < nshots; ++i) out[order[i]] = (blk[order[i]] << L_.b) | local[i];
}

uint64_t Engine::top_k(uint64_t k, uint64_t* idx, double* re, double* im) {
    BMQ_CUDA(cudaSetDevice(dev_));
    ensure_init();
    if (k == 0) return 0;
    const uint64_t nid = L_.num_blocks();
    // blocks that can hold a nonzero amplitude, ascending
    std::vector<uint64_t> ids;
    for (uint64_t id = 0; id < nid; ++id)
        if (!cfg_.compress || h_off_[id] != ~0ull) ids.push_back(id);
    const uint64_t batch = cfg_.compress ? max_blocks_ : 1;
    const auto for_batches = [&](auto&& fn) {
        for (uint64_t first = 0; first < ids.size(); first += batch) {
            const uint64_t nb = std::min(batch, ids.size() - first);
            fn(decoded_batch(ids.data() + first, nb), first, nb);
            BMQ_CUDA(cudaStreamSynchronize(st_));
        }
    };
    // radix select of the k-th largest nonzero key, 16 bits per level
    DevArray<unsigned long long> hist;
    hist.alloc(1 << kDigitBits);
    uint64_t prefix = 0, need = k;  // need: keys still to take at or below the prefix
    uint64_t tau = 0;
    bool found = k > 0;
    for (uint32_t covered = 0; covered < 64 && found;) {
        const uint32_t width = std::min<uint32_t>(kDigitBits, 64 - covered), shift = 64 - covered - width;
        BMQ_CUDA(cudaMemsetAsync(hist.p, 0, hist.bytes(), st_));
        for_batches([&](const double* w, uint64_t, uint64_t nb) {
            k_topk_hist<<<148 * 8, kQThreads, 0, st_>>>(w, L_.b, nb, prefix, shift, width, hist.p);
            BMQ_CUDA(cudaGetLastError());
        });
        std::vector<unsigned long long> hh(1u << width);
        BMQ_CUDA(cudaMemcpy(hh.data(), hist.p, hh.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
        uint64_t seen = 0;
        int64_t digit = -1;
        for (int64_t d = static_cast<int64_t>(hh.size()) - 1; d >= 0; --d) {
            if (seen + hh[d] >= need) {
                digit = d;
                break;
            }
            seen += hh[d];
        }
        if (digit < 0) {  // fewer than k nonzero amplitudes: every nonzero one
            found = false;
            break;
        }
        need -= seen;
        prefix |= static_cast<uint64_t>(digit) << shift;
        covered += width;
    }
    tau = found ? prefix : 0;  // keys > tau all taken, `need` of the keys == tau (lowest indices)
    // per block counts, then ordered collection
    std::vector<unsigned long long> above(ids.size()), equal(ids.size());
    {
        DevArray<unsigned long long> da, de;
        da.alloc(batch);
        de.alloc(batch);
        for_batches([&](const double* w, uint64_t first, uint64_t nb) {
            k_topk_count<<<static_cast<uint32_t>(nb), kQThreads, 0, st_>>>(w, L_.b, tau, da.p, de.p);
            BMQ_CUDA(cudaMemcpyAsync(above.data() + first, da.p, nb * sizeof(unsigned long long),
                                     cudaMemcpyDeviceToHost, st_));
            BMQ_CUDA(cudaMemcpyAsync(equal.data() + first, de.p, nb * sizeof(unsigned long long),
                                     cudaMemcpyDeviceToHost, st_));
        });
    }
    uint64_t n_above = 0;
    for (auto a : above) n_above += a;
    if (!found) need = 0;
    std::vector<unsigned long long> out_a(ids.size()), out_e(ids.size()), take(ids.size());
    uint64_t ca = 0, ce = n_above, left = need;
    for (size_t i = 0; i < ids.size(); ++i) {
        out_a[i] = ca;
        ca += above[i];
        take[i] = std::min<unsigned long long>(equal[i], left);
        out_e[i] = ce;
        ce += take[i];
        left -= take[i];
    }
    const uint64_t count = n_above + need;
    if (count > k) raise(BMQ_ERR_LOGIC, "top_k selection overflow");
    DevArray<uint64_t> d_idx;
    DevArray<double> d_re, d_im;
    DevArray<unsigned long long> d_oa, d_oe, d_take;
    d_idx.alloc(std::max<uint64_t>(count, 1));
    d_re.alloc(std::max<uint64_t>(count, 1));
    d_im.alloc(std::max<uint64_t>(count, 1));
    d_oa.alloc(batch);
    d_oe.alloc(batch);
    d_take.alloc(batch);
    if (count)
        for_batches([&](const double* w, uint64_t first, uint64_t nb) {
            BMQ_CUDA(cudaMemcpyAsync(d_oa.p, out_a.data() + first, nb * 8, cudaMemcpyHostToDevice, st_));
            BMQ_CUDA(cudaMemcpyAsync(d_oe.p, out_e.data() + first, nb * 8, cudaMemcpyHostToDevice, st_));
            BMQ_CUDA(cudaMemcpyAsync(d_take.p, take.data() + first, nb * 8, cudaMemcpyHostToDevice, st_));
            const uint64_t* dids = ids_.p;
            if (!cfg_.compress)  // raw: decoded_batch did not upload the id
                BMQ_CUDA(cudaMemcpyAsync(ids_.p, ids.data() + first, 8, cudaMemcpyHostToDevice, st_));
            k_topk_collect<<<static_cast<uint32_t>(nb), kQThreads, 0, st_>>>(w, L_.b, dids, tau, d_oa.p, d_oe.p,
                                                                            d_take.p, d_idx.p, d_re.p, d_im.p);
            BMQ_CUDA(cudaGetLastError());
            BMQ_CUDA(cudaStreamSynchronize(st_));
        });
    check_device_error("top_k: ");
    std::vector<uint64_t> hi(count);
    std::vector<double> hr(count), him(count);
    if (count) {
        BMQ_CUDA(cudaMemcpy(hi.data(), d_idx.p, count * 8, cudaMemcpyDeviceToHost));
        BMQ_CUDA(cudaMemcpy(hr.data(), d_re.p, count * 8, cudaMemcpyDeviceToHost));
        BMQ_CUDA(cudaMemcpy(him.data(), d_im.p, count * 8, cudaMemcpyDeviceToHost));
    }
    // largest |a|^2 first, ties by index (keys recomputed exactly as on the device)
    std::vector<uint64_t> ord(count);
    std::iota(ord.begin(), ord.end(), 0);
    const auto keyh = [&](uint64_t i) {
        volatile double p = hr[i] * hr[i];
        volatile double q = him[i] * him[i];
        return static_cast<double>(p) + static_cast<double>(q);
    };
    std::sort(ord.begin(), ord.end(), [&](uint64_t a, uint64_t c) {
        const double ka = keyh(a), kc = keyh(c);
        return ka != kc ? ka > kc : hi[a] < hi[c];
    });
    for (uint64_t i = 0; i < count; ++i) {
        idx[i] = hi[ord[i]];
        re[i] = hr[ord[i]];
        im[i] = him[ord[i]];
    }
    return count;
}

}  // namespace bmq
