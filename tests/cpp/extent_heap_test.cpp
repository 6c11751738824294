// CPU test of ExtentHeap, the pinned host level's allocator (store.hpp):
// random alloc / free sequences against a brute-force model of the arena.
// Checks that live extents never overlap and stay inside the capacity, that
// the free list stays coalesced and sums to capacity - used, that alloc fails
// only when no free extent is large enough (best fit), that a double free is
// rejected, that growth adds a free tail, and that freeing everything
// coalesces back to one extent.
#include <cstdio>
#include <map>
#include <random>
#include <vector>

#include "store.hpp"

#define CHECK(c)                                                      \
    do {                                                              \
        if (!(c)) {                                                   \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);  \
            return 1;                                                 \
        }                                                             \
    } while (0)

int main() {
    for (uint64_t seed = 1; seed <= 20; ++seed) {
        std::mt19937_64 rng(seed);
        const uint64_t cap = (1ull << 20) + 16 * (rng() % 1000);
        bmq::ExtentHeap h;
        h.reset(cap, 16);
        std::map<uint64_t, uint64_t> live;  // off -> rounded size
        for (int op = 0; op < 20000; ++op) {
            const bool do_alloc = live.empty() || rng() % 100 < 55;
            if (do_alloc) {
                const uint64_t size = 1 + rng() % ((rng() % 8 == 0) ? 65536 : 2048);
                const uint64_t need = (size + 15) / 16 * 16;
                const uint64_t largest = h.largest_free();
                const uint64_t off = h.alloc(size);
                if (off == bmq::ExtentHeap::kNone) {
                    CHECK(largest < need);
                    continue;
                }
                CHECK(off % 16 == 0 && off + need <= cap);
                auto nx = live.lower_bound(off);
                CHECK(nx == live.end() || nx->first >= off + need);
                if (nx != live.begin()) {
                    auto pv = std::prev(nx);
                    CHECK(pv->first + pv->second <= off);
                }
                live.emplace(off, need);
            } else {
                auto it = live.begin();
                std::advance(it, rng() % live.size());
                h.free(it->first, it->second);
                live.erase(it);
            }
            if (op % 97 == 0) CHECK(h.check());
        }
        uint64_t used = 0;
        for (auto& [o, s] : live) used += s;
        CHECK(h.used() == used && h.check());
        if (!live.empty()) {  // a double free is an error, and leaves the heap intact
            bool threw = false;
            try {
                h.free(live.begin()->first, live.begin()->second);
                h.free(live.begin()->first, live.begin()->second);
            } catch (const bmq::Error&) {
                threw = true;
            }
            CHECK(threw);
            live.erase(live.begin());
        }
        const uint64_t before = h.capacity(), grown = before + 16 * (1 + rng() % 4096);  // the new tail is free
        h.extend(grown);
        CHECK(h.capacity() == grown && h.check() && h.largest_free() >= grown - before);
        for (auto& [o, s] : live) h.free(o, s);
        CHECK(h.used() == 0 && h.extents() == 1 && h.largest_free() == h.capacity() && h.check());
    }
    std::printf("extent_heap ok\n");
    return 0;
}
