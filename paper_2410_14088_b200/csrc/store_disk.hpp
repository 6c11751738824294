// store_disk.hpp — the disk level beneath the pinned host level (see
// store_disk.cpp).
#pragma once

#include <string>

#include "store.hpp"

namespace bmq {

class DiskLevel {
public:
    DiskLevel() = default;
    DiskLevel(const DiskLevel&) = delete;
    DiskLevel& operator=(const DiskLevel&) = delete;
    ~DiskLevel();
    // an anonymous spill file in `dir` (default /tmp) with `capacity` bytes of extents
    void open(const std::string& dir, uint64_t capacity, uint64_t align);
    void close();
    bool is_open() const { return fd_ >= 0; }
    bool gds() const { return gds_; }
    ExtentHeap& heap() { return heap_; }
    const ExtentHeap& heap() const { return heap_; }
    // synchronous transfers (the caller orders them against its streams)
    void write_from_device(const void* dev, uint64_t size, uint64_t off);
    void read_to_device(void* dev, uint64_t size, uint64_t off);
    void read_to_host(void* host, uint64_t size, uint64_t off);
    void write_from_host(const void* host, uint64_t size, uint64_t off);
    uint64_t bytes_written() const { return bytes_written_; }
    uint64_t bytes_read() const { return bytes_read_; }

private:
    int fd_ = -1;
    std::string path_;
    void* fh_ = nullptr;  // CUfileHandle_t
    bool gds_ = false;
    void* bounce_ = nullptr;
    uint64_t bounce_bytes_ = 0;
    ExtentHeap heap_;
    uint64_t bytes_written_ = 0, bytes_read_ = 0;
};

}  // namespace bmq
