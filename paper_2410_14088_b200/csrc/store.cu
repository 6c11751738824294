// store.cu — ExtentHeap (pinned host level) and DeviceArena (HBM level on
// CUDA virtual memory). See store.hpp.
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "device_common.cuh"
#include "store.hpp"

namespace bmq {

// ------------------------------------------------------------ DeviceArena
// Driver VMM entry points come from the runtime (cudaGetDriverEntryPoint*),
// so libbmq has no link-time dependency on libcuda.

namespace {

struct Vmm {
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemAddressFree) addr_free = nullptr;
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemRelease) mem_release = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) set_access = nullptr;
    decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
};

template <class F>
void entry(const char* name, F& fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPointByVersion(name, &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p) {
        cudaGetLastError();
        raise(BMQ_ERR_CUDA, std::string("CUDA driver entry point unavailable: ") + name);
    }
    fn = reinterpret_cast<F>(p);
}

const Vmm& vmm() {
    static std::once_flag once;
    static Vmm v;
    std::call_once(once, [] {
        entry("cuMemAddressReserve", v.reserve);
        entry("cuMemAddressFree", v.addr_free);
        entry("cuMemCreate", v.create);
        entry("cuMemRelease", v.mem_release);
        entry("cuMemMap", v.map);
        entry("cuMemUnmap", v.unmap);
        entry("cuMemSetAccess", v.set_access);
        entry("cuMemGetAllocationGranularity", v.granularity);
    });
    return v;
}

void drv(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS)
        raise(r == CUDA_ERROR_OUT_OF_MEMORY ? BMQ_ERR_OUT_OF_MEMORY : BMQ_ERR_CUDA,
              std::string(what) + " failed (CUresult " + std::to_string(static_cast<int>(r)) + ")");
}

CUmemAllocationProp prop_for(int dev) {
    CUmemAllocationProp p{};
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = dev;
    return p;
}

// Released arenas stay mapped for the next simulator on the device (one per
// device), like the stream-ordered pool keeps released buffers: creating a
// simulator then costs no cuMemCreate / cuMemMap round trips.
struct Cached {
    int dev;
    uint8_t* base;
    uint64_t reserved, mapped, gran;
    std::map<uint64_t, std::pair<unsigned long long, uint64_t>> chunks;
};
std::mutex g_cache_mu;
std::vector<Cached> g_cache;

void unmap_all(const Cached& c) {
    const Vmm& v = vmm();
    for (auto& [off, ch] : c.chunks) {
        v.unmap(reinterpret_cast<CUdeviceptr>(c.base) + off, ch.second);
        v.mem_release(ch.first);
    }
    v.addr_free(reinterpret_cast<CUdeviceptr>(c.base), c.reserved);
}

// hand cached arenas of `dev` back to the driver (before an allocation fails)
bool trim_cache(int dev) {
    std::vector<Cached> drop;
    {
        std::lock_guard<std::mutex> lock(g_cache_mu);
        for (size_t i = 0; i < g_cache.size();)
            if (g_cache[i].dev == dev) {
                drop.push_back(std::move(g_cache[i]));
                g_cache.erase(g_cache.begin() + i);
            } else {
                ++i;
            }
    }
    for (const Cached& c : drop) unmap_all(c);
    return !drop.empty();
}

}  // namespace

void DeviceArena::init(int device, uint64_t reserve_bytes) {
    release();
    dev_ = device;
    {
        std::lock_guard<std::mutex> lock(g_cache_mu);
        for (size_t i = 0; i < g_cache.size(); ++i)
            if (g_cache[i].dev == device && g_cache[i].reserved >= reserve_bytes) {
                Cached c = std::move(g_cache[i]);
                g_cache.erase(g_cache.begin() + i);
                base_ = c.base;
                reserved_ = c.reserved;
                mapped_ = c.mapped;
                gran_ = c.gran;
                for (auto& [off, ch] : c.chunks) chunks_.emplace(off, Chunk{ch.first, ch.second});
                return;
            }
    }
    trim_cache(device);  // a cached arena too small for this one: release it
    BMQ_CUDA(cudaFree(nullptr));  // the primary context exists before driver calls
    const Vmm& v = vmm();
    const CUmemAllocationProp p = prop_for(dev_);
    size_t g = 0;
    drv(v.granularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
    // chunks of at least 512 MiB keep the mapping count small
    gran_ = std::max<uint64_t>(g, 512ull << 20) / g * g;
    reserved_ = (std::max<uint64_t>(reserve_bytes, gran_) + gran_ - 1) / gran_ * gran_;
    CUdeviceptr va = 0;
    drv(v.reserve(&va, reserved_, gran_, 0, 0), "cuMemAddressReserve");
    base_ = reinterpret_cast<uint8_t*>(va);
    mapped_ = 0;
}

bool DeviceArena::grow_to(uint64_t bytes) {
    if (bytes <= mapped_) return true;
    if (bytes > reserved_) return false;
    const Vmm& v = vmm();
    const CUmemAllocationProp p = prop_for(dev_);
    CUmemAccessDesc acc{};
    acc.location = p.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    while (mapped_ < bytes) {
        const uint64_t size = gran_;
        CUmemGenericAllocationHandle h = 0;
        CUresult r = v.create(&h, size, &p, 0);
        if (r == CUDA_ERROR_OUT_OF_MEMORY) {
            // released stream-ordered allocations stay cached in the default
            // pool (dev_alloc), released arenas in the arena cache; hand them
            // back to the device and retry once
            trim_cache(dev_);
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, dev_) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
            cudaGetLastError();
            r = v.create(&h, size, &p, 0);
        }
        if (r == CUDA_ERROR_OUT_OF_MEMORY) return false;
        drv(r, "cuMemCreate");
        const CUdeviceptr at = reinterpret_cast<CUdeviceptr>(base_) + mapped_;
        r = v.map(at, size, 0, h, 0);
        if (r != CUDA_SUCCESS) {
            v.mem_release(h);
            drv(r, "cuMemMap");
        }
        r = v.set_access(at, size, &acc, 1);
        if (r != CUDA_SUCCESS) {
            v.unmap(at, size);
            v.mem_release(h);
            drv(r, "cuMemSetAccess");
        }
        chunks_.emplace(mapped_, Chunk{h, size});
        mapped_ += size;
    }
    return true;
}

void DeviceArena::release() {
    if (!base_) return;
    cudaSetDevice(dev_);
    cudaDeviceSynchronize();  // no kernel may still touch the range
    Cached c{dev_, base_, reserved_, mapped_, gran_, {}};
    for (auto& [off, ch] : chunks_) c.chunks.emplace(off, std::make_pair(ch.handle, ch.size));
    chunks_.clear();
    base_ = nullptr;
    reserved_ = mapped_ = 0;
    bool keep = false;
    {
        std::lock_guard<std::mutex> lock(g_cache_mu);
        size_t mine = 0;
        for (const Cached& x : g_cache) mine += x.dev == c.dev;
        if (mine == 0) {
            g_cache.push_back(std::move(c));
            keep = true;
        }
    }
    if (!keep) unmap_all(c);
}

}  // namespace bmq
