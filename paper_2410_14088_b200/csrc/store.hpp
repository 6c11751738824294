// store.hpp — the two memory levels behind the engine's payload store
// (BlockStore, store.hpp:47-300 of the reference: RAM budget + spill file;
// here HBM arena + pinned host arena).
//
//   DeviceArena  one virtual-address range reserved for the whole device and
//                backed by physical HBM chunks on demand (cuMemCreate /
//                cuMemMap), so the arena grows in place with no copy and no
//                second arena. Payloads are appended at a bump cursor and
//                compacted in place when the garbage outweighs the live state.
//   ExtentHeap   host-side best-fit allocator of byte extents with
//                coalescing: the pinned host level places every payload in
//                its own extent and frees it when the block is rewritten, so
//                a state that is rewritten every stage reuses the same host
//                memory (the reference's spill file leaves dead extents
//                behind, store.hpp:40-41,266-270; pinned RAM cannot).
#pragma once

#include <cstdint>
#include <map>

#include "bmq_internal.hpp"

namespace bmq {

class ExtentHeap {
public:
    static constexpr uint64_t kNone = ~0ull;
    void reset(uint64_t capacity, uint64_t align);
    // best fit (smallest free extent that holds `size`, lowest offset among
    // equals); kNone when no extent is large enough
    uint64_t alloc(uint64_t size);
    void free(uint64_t off, uint64_t size);
    // grow the capacity to `capacity` (the new tail is free)
    void extend(uint64_t capacity);
    uint64_t capacity() const { return cap_; }
    uint64_t used() const { return used_; }
    uint64_t high_water() const { return high_; }
    uint64_t largest_free() const { return by_size_.empty() ? 0 : by_size_.rbegin()->first; }
    size_t extents() const { return by_off_.size(); }
    // consistency check (tests): free extents disjoint, coalesced, summing to cap - used
    bool check() const;

private:
    uint64_t round(uint64_t n) const { return (n + align_ - 1) / align_ * align_; }
    void insert(uint64_t off, uint64_t size);
    void erase_free(std::map<uint64_t, uint64_t>::iterator it);
    std::map<uint64_t, uint64_t> by_off_;            // free extents: offset -> size
    std::multimap<uint64_t, uint64_t> by_size_;      // size -> offset
    uint64_t cap_ = 0, align_ = 16, used_ = 0, high_ = 0;
};

// Physically backed prefix [0, mapped) of a reserved device VA range
// [0, reserved). Growth maps more chunks at the end; nothing moves.
class DeviceArena {
public:
    DeviceArena() = default;
    DeviceArena(const DeviceArena&) = delete;
    DeviceArena& operator=(const DeviceArena&) = delete;
    ~DeviceArena() { release(); }
    void init(int device, uint64_t reserve_bytes);
    // map chunks until mapped() >= bytes (bytes <= reserved()); false when
    // the device has no HBM left for it (the arena is unchanged then)
    bool grow_to(uint64_t bytes);
    void release();
    uint8_t* base() const { return base_; }
    uint64_t mapped() const { return mapped_; }
    uint64_t reserved() const { return reserved_; }
    uint64_t granularity() const { return gran_; }

private:
    struct Chunk {
        unsigned long long handle;
        uint64_t size;
    };
    int dev_ = 0;
    uint8_t* base_ = nullptr;
    uint64_t reserved_ = 0, mapped_ = 0, gran_ = 0;
    std::map<uint64_t, Chunk> chunks_;  // offset -> physical allocation
};

}  // namespace bmq
