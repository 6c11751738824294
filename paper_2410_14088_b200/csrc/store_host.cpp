// store_host.cpp — ExtentHeap, the allocator of the pinned host level
// (store.hpp). Host-only: built with g++ and also linked into the CPU test
// tests/cpp/extent_heap_test.cpp.
#include <algorithm>

#include "store.hpp"

namespace bmq {

// ------------------------------------------------------------- ExtentHeap

void ExtentHeap::reset(uint64_t capacity, uint64_t align) {
    align_ = std::max<uint64_t>(align, 1);
    cap_ = capacity / align_ * align_;
    by_off_.clear();
    by_size_.clear();
    used_ = high_ = 0;
    if (cap_) insert(0, cap_);
}

void ExtentHeap::insert(uint64_t off, uint64_t size) {
    by_off_.emplace(off, size);
    by_size_.emplace(size, off);
}

void ExtentHeap::erase_free(std::map<uint64_t, uint64_t>::iterator it) {
    auto [lo, hi] = by_size_.equal_range(it->second);
    for (auto s = lo; s != hi; ++s)
        if (s->second == it->first) {
            by_size_.erase(s);
            break;
        }
    by_off_.erase(it);
}

uint64_t ExtentHeap::alloc(uint64_t size) {
    const uint64_t need = round(std::max<uint64_t>(size, 1));
    auto s = by_size_.lower_bound(need);
    if (s == by_size_.end()) return kNone;
    const uint64_t off = s->second, have = s->first;
    erase_free(by_off_.find(off));
    if (have > need) insert(off + need, have - need);
    used_ += need;
    high_ = std::max(high_, used_);
    return off;
}

void ExtentHeap::free(uint64_t off, uint64_t size) {
    uint64_t len = round(std::max<uint64_t>(size, 1));
    if (off % align_ || off + len > cap_ || len > used_) raise(BMQ_ERR_STORE, "host extent freed twice or out of range");
    // every check before any change: a rejected free leaves the heap intact
    auto next = by_off_.lower_bound(off);
    if (next != by_off_.end() && next->first < off + len) raise(BMQ_ERR_STORE, "host extent freed twice");
    auto prev = next == by_off_.begin() ? by_off_.end() : std::prev(next);
    if (prev != by_off_.end() && prev->first + prev->second > off) raise(BMQ_ERR_STORE, "host extent freed twice");
    used_ -= len;
    if (next != by_off_.end() && next->first == off + len) {  // merge with the following free extent
        len += next->second;
        erase_free(next);
    }
    if (prev != by_off_.end() && prev->first + prev->second == off) {  // and with the preceding one
        off = prev->first;
        len += prev->second;
        erase_free(prev);
    }
    insert(off, len);
}

void ExtentHeap::extend(uint64_t capacity) {
    const uint64_t cap = capacity / align_ * align_;
    if (cap <= cap_) return;
    const uint64_t old = cap_;
    cap_ = cap;
    used_ += cap - old;  // the new tail enters as one allocated extent and is freed (coalescing)
    free(old, cap - old);
}

bool ExtentHeap::check() const {
    uint64_t end = 0, free_total = 0;
    bool first = true;
    for (const auto& [off, size] : by_off_) {
        if (!first && off <= end) return false;  // overlapping or not coalesced
        if (size == 0 || off % align_ || size % align_) return false;
        end = off + size;
        free_total += size;
        first = false;
    }
    return end <= cap_ && free_total + used_ == cap_ && by_size_.size() == by_off_.size();
}

}  // namespace bmq
