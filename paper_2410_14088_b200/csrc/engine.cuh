// engine.cuh — the device Simulator (cbq::Simulator, engine.hpp:58-250).
#pragma once

#include <memory>
#include <utility>
#include <vector>

#include "codec.cuh"
#include "gates.cuh"
#include "store.hpp"
#include "store_disk.hpp"

namespace bmq {

template <class T>
struct DevArray {
    T* p = nullptr;
    size_t n = 0;
    DevArray() = default;
    DevArray(const DevArray&) = delete;
    DevArray& operator=(const DevArray&) = delete;
    ~DevArray() { release(); }
    void alloc(size_t count) {
        release();
        if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T)));
        n = count;
    }
    void release() {
        if (p) dev_free(p);
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
    void swap_with(DevArray& o) {
        std::swap(p, o.p);
        std::swap(n, o.n);
    }
};

// Page-locked host array (cudaMallocHost), owned RAII: the engine's host
// mirrors of per-id metadata are copied every stage.
template <class T>
class PinnedVec {
public:
    PinnedVec() = default;
    PinnedVec(const PinnedVec&) = delete;
    PinnedVec& operator=(const PinnedVec&) = delete;
    ~PinnedVec() { release(); }
    void assign(size_t count, T value) {
        if (count != n_) {
            release();
            if (count) {
                void* q = nullptr;
                if (cudaMallocHost(&q, count * sizeof(T)) != cudaSuccess) {
                    cudaGetLastError();
                    raise(BMQ_ERR_CUDA, "cudaMallocHost failed for host metadata");
                }
                p_ = static_cast<T*>(q);
            }
            n_ = count;
        }
        for (size_t i = 0; i < n_; ++i) p_[i] = value;
    }
    T* data() { return p_; }
    const T* data() const { return p_; }
    size_t size() const { return n_; }
    T& operator[](size_t i) { return p_[i]; }
    const T& operator[](size_t i) const { return p_[i]; }
    T* begin() { return p_; }
    T* end() { return p_ + n_; }
    void swap_with(PinnedVec& o) {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
    }

private:
    void release() {
        if (p_) cudaFreeHost(p_);
        p_ = nullptr;
        n_ = 0;
    }
    T* p_ = nullptr;
    size_t n_ = 0;
};

// Host replay of BlockStore's accounting (store.hpp:64-117,188-232) in the
// reference's sequential put order, so max_footprint_bytes and
// spilled_blocks match the reference run with one worker.
class StoreModel {
public:
    void reset(uint64_t num_ids, uint64_t budget);
    void put(uint64_t id, uint64_t size);
    void put_shared(uint64_t first_id, uint64_t last_id, uint64_t size);  // ids [first, last)
    uint64_t peak() const { return peak_; }
    uint64_t resident() const { return resident_; }
    uint64_t spilled_live() const { return spilled_live_; }
    uint64_t spilled_blocks() const { return spilled_blocks_; }
    // checkpoint image of the whole accounting state
    void serialize(std::vector<uint8_t>& out) const;
    void deserialize(const uint8_t* p, uint64_t n);

private:
    void detach(uint64_t id);
    bool place(uint64_t size);  // returns spilled
    std::vector<uint64_t> size_;
    std::vector<uint8_t> flags_;  // bit0 spilled, bit1 shared, bit2 absent
    uint64_t budget_ = ~0ull, resident_ = 0, spilled_live_ = 0, peak_ = 0, spilled_blocks_ = 0;
    uint64_t shared_refs_ = 0, shared_size_ = 0;
    bool shared_spilled_ = false;
};

struct StagePlan {
    bmq_stage stage;
    GroupGeometry gg;
    GateProgram prog;            // over the 2^(b + |inner|) group buffer
    bool diag_only = false;      // no gate mixes amplitudes: blocks are independent
    std::vector<uint8_t> touched;  // diag_only: inner value v -> some gate acts on the block
};

// BMQ_FLAG_STAGE_FUSION: stages [s0, s1) run over the groups of the union of
// their inner qubits; progs[j] is stage s0 + j's program on that layout.
struct FusedSet {
    uint64_t s0 = 0, s1 = 0;
    GroupGeometry gg;
    std::vector<std::unique_ptr<GateProgram>> progs;
};

class Engine {
public:
    Engine(uint32_t n, const bmq_gate* gates, uint64_t ngates, const bmq_config& cfg);
    ~Engine();

    void init_state();
    void reset();
    void run(bmq_report* rep, double* stage_ms, uint64_t stage_cap);
    void run_stages(uint64_t first, uint64_t last);
    double state_norm();
    void extract_state(double* amps, uint64_t namps);
    void amplitude(uint64_t index, double* re, double* im);
    // queries.cu: shots in basis-index form; top-k by |a|^2
    void sample(uint64_t nshots, uint64_t seed, uint64_t* out);
    uint64_t top_k(uint64_t k, uint64_t* idx, double* re, double* im);
    uint64_t get_payload(uint64_t id, uint8_t* out, uint64_t cap);
    void get_payloads(uint8_t* out, uint64_t cap, uint64_t* sizes, uint64_t* total);
    void put_payload(uint64_t id, const uint8_t* data, uint64_t size);
    double fidelity_dense(const double* ideal, uint64_t namps);
    double fidelity_analytic(int kind);
    static double fidelity_pair(Engine& a, Engine& b);

    // Sharded runs (one engine per rank). A sharded engine only
    // processes the groups of its rank under each stage's device bits; ids it
    // does not own hold ALL_ZERO with zero sums, so local reductions are
    // partial sums. The host driver moves payloads between stages.
    void shard(uint32_t rank, uint32_t world);
    const std::vector<uint32_t>& device_bits() const { return dev_bits_; }
    uint32_t shard_world() const { return shard_world_; }
    bool initialized() const { return initialized_; }
    uint32_t owner_of(uint64_t id, uint64_t s) const { return owner(id, s); }
    // the device bits of stage s differ from those of stage s - 1
    bool owners_changed(uint64_t s) const {
        for (uint32_t j = 0; j < shard_m_; ++j)
            if (dev_bits_[s * shard_m_ + j] != dev_bits_[(s - 1) * shard_m_ + j]) return true;
        return false;
    }
    // meta per id: {size (0 = ALL_ZERO), sumsq, sum_re, sum_im (f64 bits)}
    void export_payloads(const uint64_t* ids, uint64_t n, uint64_t* meta, void* dst, uint64_t cap);
    void import_payloads(const uint64_t* ids, uint64_t n, const uint64_t* meta, const void* src);
    void drop_payloads(const uint64_t* ids, uint64_t n);
    void stage_sizes(uint64_t s, uint64_t* sizes);
    void account_stage(uint64_t s, const uint64_t* sizes);
    void partial_sums(double* out3);
    void report(bmq_report* rep, double device_ms);
    // BlockStore::footprint() (store.hpp:30-35,138-142) of the replayed accounting
    void footprint(uint64_t* resident, uint64_t* spilled_live, uint64_t* peak) const {
        if (resident) *resident = store_.resident();
        if (spilled_live) *spilled_live = store_.spilled_live();
        if (peak) *peak = store_.peak();
    }

    // Checkpoint / resume: every payload with its sums, the
    // store accounting and the stage cursor, in one file. load_checkpoint
    // needs an engine of the same circuit, layout, plan and bound and returns
    // the next stage to run.
    void save_checkpoint(const char* path);
    uint64_t load_checkpoint(const char* path);

    const Layout& layout() const { return L_; }
    const std::vector<bmq_stage>& plan() const { return plan_; }

private:
    bool sharded() const { return shard_world_ > 1; }
    uint32_t owner(uint64_t id, uint64_t s) const {
        return shard_m_ ? shard_owner(id, dev_bits_.data() + s * shard_m_, shard_m_) : 0;
    }
    uint32_t shard_rank_ = 0, shard_world_ = 1, shard_m_ = 0;
    std::vector<uint32_t> dev_bits_;  // shard_m_ block-id bits per stage

    void ensure_init();
    void run_stage(uint64_t s);
    // stage fusion (BMQ_FLAG_STAGE_FUSION)
    bool fusable(uint64_t s) const;
    void plan_fusion();
    void run_fused(const FusedSet& fs);
    bool fusion_planned_ = false;
    std::vector<std::unique_ptr<FusedSet>> fused_sets_;
    std::vector<int64_t> fused_at_;  // stage -> index of the fused set starting there, else -1
    void raw_run_stage(uint64_t s);
    // Batches alternate between two buffer sets and two streams: the front
    // of batch k+1 (descriptors, decode, gate passes, plan) is queued before
    // the back of batch k (allocation + emit, with its host synchronisation),
    // so the decode of one batch overlaps the passes of the other. Emits stay
    // in batch order (ev_emitted_), and compaction waits for the other set.
    struct BatchFront {
        bool codes = false, fused = true;
    };
    BatchFront process_front(StagePlan& sp, const uint64_t* d_ids, const uint32_t* d_vtab, uint64_t nblk,
                             size_t bidx);
    void process_back(StagePlan& sp, const BatchFront& f, const uint64_t* h_ids, uint64_t nblk, size_t bidx);
    void use_set(int s);
    void join_sets();
    int cur_set_ = 0;
    bool two_sets_ = false;
    cudaStream_t st2_ = nullptr;
    cudaEvent_t ev_emitted_ = nullptr, ev_join_ = nullptr;
    bool emitted_live_ = false;
    void emit_batch(uint64_t nblk, const uint64_t* h_ids);
    void emit_to_host(uint64_t nblk, const uint64_t* h_ids);

    // ---- device level (store.hpp DeviceArena): bump cursor cursor_[0],
    // logical capacity arena_limit_ (mapped >= limit), in-place compaction
    uint64_t arena_used();
    // make `need` more bytes available at the cursor: compaction (payloads
    // of the `excl` ids are dead) and / or growth; false = the device is full
    bool make_room(uint64_t need, const uint64_t* excl, uint64_t nexcl);
    void compact(const uint64_t* excl, uint64_t nexcl);
    bool grow_arena(uint64_t limit);
    DeviceArena arena_;
    uint64_t arena_limit_ = 0, arena_max_ = 0;
    bool arena_grow_ = false;
    // Heap mode (large blocks, few ids): every payload gets its own arena
    // extent from dev_heap_, freed when the block is rewritten, so dense
    // stages reuse the space of the payloads they decoded (no compaction);
    // a batch whose payloads do not all fit sends the rest to the host level.
    // Bump mode (many small payloads): cursor_[0] + in-place compaction.
    bool heap_mode_ = false, arena_auto_ = false;  // auto: bump until a compaction finds a dense state
    ExtentHeap dev_heap_;
    uint64_t dev_alloc(uint64_t size);  // heap mode; ExtentHeap::kNone when the device is full
    void emit_placed(uint64_t nblk, const uint64_t* h_ids);
    PinnedVec<uint64_t> h_place_;
    DevArray<uint64_t> d_place_;
    void sync_meta_to_host();
    void decompress_ids(const uint64_t* d_ids, uint64_t nids, bool want_sums, const uint64_t* h_ids = nullptr);
    const uint64_t* stage_disk_reads(const uint64_t* h_ids, uint64_t n);
    uint64_t disk_fit(const uint64_t* h_ids, uint64_t n);
    uint64_t disk_alloc(uint64_t size);
    DiskLevel disk_;
    std::string disk_dir_;
    const double* decoded_batch(const uint64_t* h_ids, uint64_t n);
    void host_ids_to_device(const std::vector<uint64_t>& ids);
    // Per-id dequantised sums are computed lazily (the emit kernel does not
    // produce them): ensure_sums decodes the payloads of stale ids, all ids
    // or the n given ones.
    void ensure_sums(const uint64_t* ids = nullptr, uint64_t n = 0);
    std::vector<uint8_t> sums_ok_;
    uint64_t zero_payload(uint8_t* out, uint64_t cap) const;
    uint32_t peek_error();
    void check_device_error(const char* what);
    void phase_event(size_t i);
    void collect_phase_times(size_t nbatches);

    Layout L_;
    bmq_config cfg_;
    std::vector<bmq_gate> gates_;
    std::vector<bmq_stage> plan_;
    bmq_plan_choice plan_choice_{};  // BMQ_FLAG_DEVICE_PLAN: the planner's choice
    std::vector<std::unique_ptr<StagePlan>> stage_plans_;
    const DevTables* tabs_ = nullptr;
    int dev_ = 0;
    cudaStream_t st_ = nullptr;
    cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
    std::vector<cudaEvent_t> phase_ev_;  // 4 per batch: start, decoded, gated, compressed
    bool initialized_ = false;
    bool identity_ok_ = false;  // codec idempotent on every representable amplitude
    uint64_t next_stage_ = 0;

    // compressed state: payloads in the device arena (16-byte aligned) or in
    // the pinned host level, per-id metadata (off ~0 = canonical ALL_ZERO,
    // bit 62 = host-level extent)
    DevArray<uint64_t> cursor_;  // [0] arena cursor, [1] batch total, [2..3] range, [4] staging cursor, [5] total
    // ---- host level (store.hpp ExtentHeap): pinned, mapped host arena with
    // one extent per payload, freed when the block is rewritten
    uint8_t* host_pool_ = nullptr;
    uint64_t host_cap_ = 0;
    ExtentHeap host_heap_;
    void ensure_host_pool();
    // the payload extents of rewritten / dropped ids: host level, and the
    // device arena in heap mode
    void free_extents(const uint64_t* ids, uint64_t n);
    // ---- copy streams ("2 streams"): host-level payloads of
    // batch k+1 are prefetched H2D on cp_in_ while batch k computes on st_,
    // and payloads of batch k-1 bound for the host are written back D2H from
    // wb_ on cp_out_
    cudaStream_t cp_in_ = nullptr, cp_out_ = nullptr;
    cudaEvent_t ev_pf_[2] = {}, ev_dec_[2] = {}, ev_emit_ = nullptr, ev_wb_ = nullptr;
    DevArray<uint8_t> pf_[2], wb_;
    DevArray<uint64_t> pf_off_[2];
    PinnedVec<uint64_t> h_pf_off_[2];
    PinnedVec<uint64_t> h_meta_;  // (id, off, size) triples of a host-bound batch
    DevArray<uint64_t> d_meta_;
    bool pf_live_[2] = {false, false};
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> link_ev_;
    size_t link_ev_used_ = 0;
    void link_event_pair(cudaStream_t s, bool start);
    void collect_link_times();
    // queue the H2D copies of the host-level payloads of one batch into
    // prefetch slot `slot`; false = nothing to prefetch
    bool prefetch(const uint64_t* h_ids, uint64_t nblk, int slot);
    void copy_batch(void** dst, void** src, size_t* sizes, size_t n, cudaStream_t s);
    void sync_copies();
    DevArray<uint64_t> off_, size_, new_off_, live_ids_;
    DevArray<double> sums_;       // per id: sumsq, sum_re, sum_im (3 doubles)
    DevArray<uint8_t> zero_hdr_;  // canonical ALL_ZERO payload (+ slack)
    // raw mode (compress == false): dense planar state
    DevArray<double> dense_;
    // working set
    DevArray<double> work_;
    uint64_t work_scalars_ = 0;
    uint64_t max_blocks_ = 0;
    uint32_t nch_ = 1;
    DevArray<CmpBlock> cmp_;
    DevArray<DecBlock> dec_;
    DevArray<ChunkPlan> cplan_;
    DevArray<uint32_t> pk_;  // packed code words of the batch (4 B per scalar)
    DevArray<BlockPlan> bplan_;
    DevArray<DecInfo> dinfo_;
    DevArray<DecChunk> dchunk_;
    DevArray<uint8_t> zflag_;  // per (batch slot, chunk): all-zero input chunk (code-domain stages)
    DevArray<PermSrc> psrc_;   // per (batch slot, chunk): chunk read from the payload by the first permutation pass
    DevArray<uint32_t> imnz_;  // 1 word: code domain, some imaginary-half input chunk is nonzero; FP, some group flag is 0
    DevArray<DecRow> rows_;    // per 32 scalars of work_: decode rows of a streaming first pass (fused decode)
    DevArray<uint8_t> wflag_;  // per 32 scalars of work_: group stored (1) or all zero (0), FP stages
    // the second buffer set (use_set swaps it with the members above)
    DevArray<double> work2_;
    DevArray<uint32_t> pk2_, imnz2_;
    DevArray<CmpBlock> cmp2_;
    DevArray<DecBlock> dec2_;
    DevArray<ChunkPlan> cplan2_;
    DevArray<BlockPlan> bplan2_;
    DevArray<DecInfo> dinfo2_;
    DevArray<DecChunk> dchunk2_;
    DevArray<uint8_t> zflag2_, wflag2_;
    DevArray<PermSrc> psrc2_;
    DevArray<uint64_t> d_place2_, d_meta2_;
    PinnedVec<uint64_t> h_place2_, h_meta2_;
    DevArray<uint64_t> ids_;
    DevArray<uint64_t> fsz_;  // stage fusion: payload sizes of the intermediate stages of a batch
    DevArray<uint32_t> vtab_;
    DevArray<DevError> err_;
    DevArray<double> red_;

    // host mirrors
    PinnedVec<uint64_t> h_off_, h_size_;
    StoreModel store_;
    uint64_t stage_compress_calls_ = 0, stage_decompress_calls_ = 0;
    bmq_report counters_{};
    uint64_t device_peak_ = 0;
};

}  // namespace bmq
