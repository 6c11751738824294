// shard_run.hpp — multi-GPU driver of the stage loop behind the C ABI
// (bmq_simulator_run_sharded); see shard_run.cpp.
#pragma once

#include <chrono>
#include <cmath>
#include <memory>
#include <vector>

#include "engine.cuh"

namespace bmq {

// Collective over the ranks of a sharded run; buffers are device memory.
class Collective {
public:
    virtual ~Collective() = default;
    virtual uint32_t rank() const = 0;
    virtual uint32_t world() const = 0;
    // send_bytes[p] bytes to peer p from consecutive slices of `send`;
    // recv_bytes[p] bytes from peer p into consecutive slices of `recv`
    virtual void all_to_all_v(const void* send, const uint64_t* send_bytes, void* recv, const uint64_t* recv_bytes) = 0;
    virtual void all_reduce_sum(double* dev, uint64_t n) = 0;
    virtual void all_reduce_sum(uint64_t* dev, uint64_t n) = 0;
};

struct ShardStats {
    uint64_t remaps = 0, moved_bytes = 0;
    double exchange_ms = 0.0, account_ms = 0.0;
};

// world collectives of one process, for world engines driven by world threads
std::vector<std::unique_ptr<Collective>> make_local_collectives(uint32_t world);
// one rank of an NCCL communicator (libnccl.so.2 loaded at run time)
std::unique_ptr<Collective> make_nccl_collective(const uint8_t id[128], uint32_t rank, uint32_t world, int device);
void nccl_unique_id(uint8_t id[128]);

// Simulator::run over col.world() ranks; every rank calls it with its engine.
void run_sharded(Engine& e, Collective& col, bmq_report* rep, double* stage_ms, uint64_t stage_cap,
                 ShardStats* stats = nullptr);

}  // namespace bmq
