// shard_run.cpp — cbq::Simulator::run (engine.hpp:97-134) over several GPUs
// behind the C ABI (bmq_simulator_run_sharded), the host C++
// twin of paper_2410_14088_b200/shard.py for callers without Python.
//
// One engine per rank. log2(world) device qubits among each stage's outer
// qubits (shard_plan, furthest-next-use) decide which rank owns a group, so
// a stage runs with no communication. When the device qubits change, the
// compressed payloads whose owner changes move: their meta (size + block
// sums, 32 B per id), then their bytes (16-byte aligned slots), as two
// all-to-all-v exchanges of device buffers. One sum all-reduce of the per-id
// sizes per stage lets every rank replay the reference BlockStore
// accounting (store.hpp:64-83) in put order; norm and counters are
// all-reduced at the end.
//
// Collectives: NCCL (one process per GPU; libnccl.so.2 loaded at run time,
// so libbmq has no link-time NCCL dependency) or an in-process hub for
// several engines driven by threads of one process (any devices; used to
// run world > 1 on a single GPU).
#include "shard_run.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>

namespace bmq {

namespace {

uint64_t aligned16(uint64_t x) { return (x + 15) / 16 * 16; }

// ------------------------------------------------------------ in-process hub
struct Hub {
    uint32_t world;
    std::mutex mu;
    std::condition_variable cv;
    uint32_t arrived = 0;
    uint64_t generation = 0;
    std::vector<const void*> send;
    std::vector<const uint64_t*> counts;
    std::vector<std::vector<double>> red;
    explicit Hub(uint32_t w) : world(w), send(w), counts(w), red(w) {}
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t gen = generation;
        if (++arrived == world) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return generation != gen; });
        }
    }
};

class LocalCollective final : public Collective {
public:
    LocalCollective(std::shared_ptr<Hub> hub, uint32_t rank) : hub_(std::move(hub)), rank_(rank) {}
    uint32_t rank() const override { return rank_; }
    uint32_t world() const override { return hub_->world; }
    void all_to_all_v(const void* send, const uint64_t* send_bytes, void* recv, const uint64_t* recv_bytes) override {
        hub_->send[rank_] = send;
        hub_->counts[rank_] = send_bytes;
        hub_->barrier();
        uint64_t at = 0;
        for (uint32_t p = 0; p < hub_->world; ++p) {
            uint64_t from = 0;
            for (uint32_t q = 0; q < rank_; ++q) from += hub_->counts[p][q];
            if (hub_->counts[p][rank_] != recv_bytes[p])
                raise(BMQ_ERR_LOGIC, "sharded exchange: peers disagree on a transfer size");
            if (recv_bytes[p])
                BMQ_CUDA(cudaMemcpy(static_cast<uint8_t*>(recv) + at, static_cast<const uint8_t*>(hub_->send[p]) + from,
                                    recv_bytes[p], cudaMemcpyDefault));
            at += recv_bytes[p];
        }
        hub_->barrier();  // every peer has read our send buffer
    }
    void all_reduce_sum(double* dev, uint64_t n) override {
        std::vector<double>& mine = hub_->red[rank_];
        mine.resize(n);
        BMQ_CUDA(cudaMemcpy(mine.data(), dev, n * sizeof(double), cudaMemcpyDeviceToHost));
        hub_->barrier();
        std::vector<double> tot(n, 0.0);
        for (uint32_t p = 0; p < hub_->world; ++p)  // fixed rank order: identical on every rank
            for (uint64_t i = 0; i < n; ++i) tot[i] += hub_->red[p][i];
        hub_->barrier();
        BMQ_CUDA(cudaMemcpy(dev, tot.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    }
    void all_reduce_sum(uint64_t* dev, uint64_t n) override {
        std::vector<double>& mine = hub_->red[rank_];  // (u64 carried bit-exactly in 8-byte slots)
        mine.resize(n);
        BMQ_CUDA(cudaMemcpy(mine.data(), dev, n * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        hub_->barrier();
        std::vector<uint64_t> tot(n, 0);
        for (uint32_t p = 0; p < hub_->world; ++p) {
            const uint64_t* v = reinterpret_cast<const uint64_t*>(hub_->red[p].data());
            for (uint64_t i = 0; i < n; ++i) tot[i] += v[i];
        }
        hub_->barrier();
        BMQ_CUDA(cudaMemcpy(dev, tot.data(), n * sizeof(uint64_t), cudaMemcpyHostToDevice));
    }

private:
    std::shared_ptr<Hub> hub_;
    uint32_t rank_;
};

// ------------------------------------------------------------------ NCCL
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!a.h) return a;
        const auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::decay_t<decltype(f)>>(dlsym(a.h, name)); };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.AllReduce, "ncclAllReduce");
        sym(a.Send, "ncclSend");
        sym(a.Recv, "ncclRecv");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.GetErrorString, "ncclGetErrorString");
        return a;
    }();
    if (!api.h || !api.CommInitRank || !api.Send || !api.GroupEnd)
        raise(BMQ_ERR_INVALID_ARGUMENT, "NCCL (libnccl.so.2) is not available");
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        raise(BMQ_ERR_CUDA, std::string("NCCL ") + what + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "error"));
}

class NcclCollective final : public Collective {
public:
    NcclCollective(const uint8_t id[128], uint32_t rank, uint32_t world, int device) : rank_(rank), world_(world) {
        const NcclApi& a = nccl();
        BMQ_CUDA(cudaSetDevice(device));
        ncclUniqueId uid;
        static_assert(sizeof uid == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(&uid, id, sizeof uid);
        nccl_check(a.CommInitRank(&comm_, static_cast<int>(world), uid, static_cast<int>(rank)), "CommInitRank");
        BMQ_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    }
    ~NcclCollective() override {
        if (st_) cudaStreamDestroy(st_);
        if (comm_) nccl().CommDestroy(comm_);
    }
    uint32_t rank() const override { return rank_; }
    uint32_t world() const override { return world_; }
    void all_to_all_v(const void* send, const uint64_t* send_bytes, void* recv, const uint64_t* recv_bytes) override {
        const NcclApi& a = nccl();
        nccl_check(a.GroupStart(), "GroupStart");
        uint64_t so = 0, ro = 0;
        for (uint32_t p = 0; p < world_; ++p) {
            if (send_bytes[p])
                nccl_check(a.Send(static_cast<const uint8_t*>(send) + so, send_bytes[p], ncclUint8, static_cast<int>(p),
                                  comm_, st_), "Send");
            if (recv_bytes[p])
                nccl_check(a.Recv(static_cast<uint8_t*>(recv) + ro, recv_bytes[p], ncclUint8, static_cast<int>(p), comm_,
                                  st_), "Recv");
            so += send_bytes[p];
            ro += recv_bytes[p];
        }
        nccl_check(a.GroupEnd(), "GroupEnd");
        BMQ_CUDA(cudaStreamSynchronize(st_));
    }
    void all_reduce_sum(double* dev, uint64_t n) override {
        nccl_check(nccl().AllReduce(dev, dev, n, ncclFloat64, ncclSum, comm_, st_), "AllReduce");
        BMQ_CUDA(cudaStreamSynchronize(st_));
    }
    void all_reduce_sum(uint64_t* dev, uint64_t n) override {
        nccl_check(nccl().AllReduce(dev, dev, n, ncclUint64, ncclSum, comm_, st_), "AllReduce");
        BMQ_CUDA(cudaStreamSynchronize(st_));
    }

private:
    uint32_t rank_, world_;
    ncclComm_t comm_ = nullptr;
    cudaStream_t st_ = nullptr;
};

// device scratch that grows and is freed with the driver
struct Scratch {
    void* p = nullptr;
    uint64_t n = 0;
    void* get(uint64_t bytes) {
        if (bytes > n) {
            if (p) dev_free(p);
            n = std::max<uint64_t>(bytes, 2 * n);
            p = dev_alloc(n);
        }
        return p;
    }
    ~Scratch() {
        if (p) dev_free(p);
    }
};

}  // namespace

std::vector<std::unique_ptr<Collective>> make_local_collectives(uint32_t world) {
    if (world == 0) raise(BMQ_ERR_INVALID_ARGUMENT, "world must be at least 1");
    auto hub = std::make_shared<Hub>(world);
    std::vector<std::unique_ptr<Collective>> out;
    for (uint32_t r = 0; r < world; ++r) out.push_back(std::make_unique<LocalCollective>(hub, r));
    return out;
}

std::unique_ptr<Collective> make_nccl_collective(const uint8_t id[128], uint32_t rank, uint32_t world, int device) {
    if (rank >= world) raise(BMQ_ERR_INVALID_ARGUMENT, "shard rank out of range");
    return std::make_unique<NcclCollective>(id, rank, world, device);
}

void nccl_unique_id(uint8_t id[128]) {
    ncclUniqueId uid;
    nccl_check(nccl().GetUniqueId(&uid), "GetUniqueId");
    std::memcpy(id, &uid, sizeof uid);
}

void run_sharded(Engine& e, Collective& col, bmq_report* rep, double* stage_ms, uint64_t stage_cap,
                 ShardStats* stats) {
    const uint32_t world = col.world(), rank = col.rank();
    if (world & (world - 1)) raise(BMQ_ERR_INVALID_ARGUMENT, "shard count must be a power of two");
    const auto t_start = std::chrono::steady_clock::now();
    if (e.initialized()) e.reset();  // (shard() needs an uninitialised state)
    if (world > 1 && e.shard_world() != world) e.shard(rank, world);
    e.init_state();
    const Layout& L = e.layout();
    const uint64_t nid = L.num_blocks(), ns = e.plan().size();
    ShardStats st{};
    Scratch s_meta, r_meta, s_buf, r_buf, s_sizes;
    std::vector<uint64_t> ids_send, ids_recv, meta, rmeta, sb(world), rb(world), smc(world), rmc(world);
    for (uint64_t s = 0; s < ns; ++s) {
        const auto ts = std::chrono::steady_clock::now();
        if (s && world > 1 && e.owners_changed(s)) {
            const auto tx = std::chrono::steady_clock::now();
            // ids leaving / arriving, grouped by peer in ascending id order
            std::vector<std::vector<uint64_t>> sends(world), recvs(world);
            for (uint64_t id = 0; id < nid; ++id) {
                const uint32_t a = e.owner_of(id, s - 1), b = e.owner_of(id, s);
                if (a == b) continue;
                if (a == rank) sends[b].push_back(id);
                if (b == rank) recvs[a].push_back(id);
            }
            ids_send.clear();
            ids_recv.clear();
            for (uint32_t p = 0; p < world; ++p) {
                ids_send.insert(ids_send.end(), sends[p].begin(), sends[p].end());
                ids_recv.insert(ids_recv.end(), recvs[p].begin(), recvs[p].end());
                smc[p] = 32 * sends[p].size();
                rmc[p] = 32 * recvs[p].size();
            }
            meta.assign(4 * ids_send.size(), 0);
            e.export_payloads(ids_send.data(), ids_send.size(), meta.data(), nullptr, 0);
            void* dm = s_meta.get(std::max<uint64_t>(8, meta.size() * 8));
            void* drm = r_meta.get(std::max<uint64_t>(8, 32 * ids_recv.size()));
            BMQ_CUDA(cudaMemcpy(dm, meta.data(), meta.size() * 8, cudaMemcpyHostToDevice));
            col.all_to_all_v(dm, smc.data(), drm, rmc.data());
            rmeta.assign(4 * ids_recv.size(), 0);
            BMQ_CUDA(cudaMemcpy(rmeta.data(), drm, rmeta.size() * 8, cudaMemcpyDeviceToHost));
            uint64_t stot = 0, rtot = 0, k = 0;
            for (uint32_t p = 0; p < world; ++p) {
                sb[p] = 0;
                for (size_t i = 0; i < sends[p].size(); ++i, ++k) sb[p] += aligned16(meta[4 * k]);
                stot += sb[p];
            }
            k = 0;
            for (uint32_t p = 0; p < world; ++p) {
                rb[p] = 0;
                for (size_t i = 0; i < recvs[p].size(); ++i, ++k) rb[p] += aligned16(rmeta[4 * k]);
                rtot += rb[p];
            }
            void* dsend = s_buf.get(std::max<uint64_t>(16, stot));
            void* drecv = r_buf.get(std::max<uint64_t>(16, rtot));
            e.export_payloads(ids_send.data(), ids_send.size(), meta.data(), dsend, stot);
            col.all_to_all_v(dsend, sb.data(), drecv, rb.data());
            e.import_payloads(ids_recv.data(), ids_recv.size(), rmeta.data(), drecv);
            e.drop_payloads(ids_send.data(), ids_send.size());
            ++st.remaps;
            st.moved_bytes += stot;
            st.exchange_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tx).count();
        }
        e.run_stages(s, s + 1);
        if (world > 1) {
            const auto ta = std::chrono::steady_clock::now();
            std::vector<uint64_t> sizes(nid);
            e.stage_sizes(s, sizes.data());
            uint64_t* ds = static_cast<uint64_t*>(s_sizes.get(nid * 8));
            BMQ_CUDA(cudaMemcpy(ds, sizes.data(), nid * 8, cudaMemcpyHostToDevice));
            col.all_reduce_sum(ds, nid);
            BMQ_CUDA(cudaMemcpy(sizes.data(), ds, nid * 8, cudaMemcpyDeviceToHost));
            e.account_stage(s, sizes.data());
            st.account_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta).count();
        }
        if (stage_ms && s < stage_cap)
            stage_ms[s] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts).count();
    }
    // report: this rank's counters, global norm and summed counters
    bmq_report r{};
    e.report(&r, 0.0);
    double sums[3];
    e.partial_sums(sums);
    double* dsum = static_cast<double*>(s_sizes.get(std::max<uint64_t>(nid, 64) * 8));
    BMQ_CUDA(cudaMemcpy(dsum, sums, sizeof sums, cudaMemcpyHostToDevice));
    col.all_reduce_sum(dsum, 3);
    BMQ_CUDA(cudaMemcpy(sums, dsum, sizeof sums, cudaMemcpyDeviceToHost));
    r.final_norm = std::sqrt(sums[0]);
    uint64_t* fields[] = {&r.groups_processed, &r.groups_skipped, &r.blocks_processed, &r.payload_bytes_read,
                          &r.payload_bytes_written, &r.dense_bytes, &r.kernel_launches, &r.gate_passes, &r.batches,
                          &r.decompress_bytes, &r.gate_bytes, &r.compress_bytes, &r.fused_batches, &r.compactions,
                          &r.host_spill_bytes, &r.host_spill_batches, &r.code_domain_batches, &r.pool_growths,
                          &r.lazy_cx, &r.perm_materialisations, &r.model_bytes, &r.model_groups, &r.link_h2d_bytes,
                          &r.link_d2h_bytes, &r.compact_bytes, &r.stream_passes, &r.fused_decode_batches};
    constexpr uint64_t nf = sizeof fields / sizeof fields[0];
    uint64_t vals[nf];
    for (uint64_t i = 0; i < nf; ++i) vals[i] = *fields[i];
    uint64_t* dv = static_cast<uint64_t*>(s_sizes.get(std::max<uint64_t>(nid, 64) * 8));
    BMQ_CUDA(cudaMemcpy(dv, vals, sizeof vals, cudaMemcpyHostToDevice));
    col.all_reduce_sum(dv, nf);
    BMQ_CUDA(cudaMemcpy(vals, dv, sizeof vals, cudaMemcpyDeviceToHost));
    for (uint64_t i = 0; i < nf; ++i) *fields[i] = vals[i];
    r.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    if (rep) *rep = r;
    if (stats) *stats = st;
}

}  // namespace bmq
