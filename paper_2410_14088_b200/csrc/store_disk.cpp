// store_disk.cpp — third memory level of the payload store:
// a file on local storage beneath the pinned host level, the B200 form of the
// reference's spill file (store.hpp:234-283) and of the paper's SSD level
// (PAPER.md:361-371). Payload extents come from an ExtentHeap over the file,
// so a block rewritten every stage reuses its bytes (the reference's spill
// file only appends). Transfers go device <-> file through a pinned bounce
// buffer and pread / pwrite (what cuFile's compatibility mode does without
// the nvidia-fs module), or through GPUDirect Storage (cuFile,
// libcufile.so.0 loaded at run time) when BMQ_GDS=1 and the driver opens:
// opt-in, because on the measured B200 boxes (containers without nvidia-fs)
// cuFile's driver open / first I/O did not return within 90 s.
#include "store_disk.hpp"

#include <cuda_runtime.h>
#include <cufile.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <unistd.h>

#include <cstring>

namespace bmq {

namespace {

struct CuFileApi {
    void* h = nullptr;
    CUfileError_t (*DriverOpen)() = nullptr;
    CUfileError_t (*HandleRegister)(CUfileHandle_t*, CUfileDescr_t*) = nullptr;
    void (*HandleDeregister)(CUfileHandle_t) = nullptr;
    ssize_t (*Read)(CUfileHandle_t, void*, size_t, off_t, off_t) = nullptr;
    ssize_t (*Write)(CUfileHandle_t, const void*, size_t, off_t, off_t) = nullptr;
    bool ok = false;
};

const CuFileApi& cufile() {
    static CuFileApi api = [] {
        CuFileApi a;
        if (!getenv("BMQ_GDS") || getenv("BMQ_NO_GDS")) return a;
        a.h = dlopen("libcufile.so.0", RTLD_NOW);
        if (!a.h) a.h = dlopen("libcufile.so", RTLD_NOW);
        if (!a.h) return a;
        const auto sym = [&](auto& f, const char* n) { f = reinterpret_cast<std::decay_t<decltype(f)>>(dlsym(a.h, n)); };
        sym(a.DriverOpen, "cuFileDriverOpen");
        sym(a.HandleRegister, "cuFileHandleRegister");
        sym(a.HandleDeregister, "cuFileHandleDeregister");
        sym(a.Read, "cuFileRead");
        sym(a.Write, "cuFileWrite");
        a.ok = a.DriverOpen && a.HandleRegister && a.Read && a.Write && a.DriverOpen().err == CU_FILE_SUCCESS;
        return a;
    }();
    return api;
}

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise(BMQ_ERR_CUDA, std::string("CUDA error: ") + cudaGetErrorString(e) + " at " + what);
}

}  // namespace

DiskLevel::~DiskLevel() { close(); }

void DiskLevel::open(const std::string& dir, uint64_t capacity, uint64_t align) {
    close();
    std::string base = dir.empty() ? std::string("/tmp") : dir;
    path_ = base + "/bmq_spill_XXXXXX";
    std::vector<char> tmpl(path_.begin(), path_.end());
    tmpl.push_back('\0');
    fd_ = mkstemp(tmpl.data());
    if (fd_ < 0) raise(BMQ_ERR_STORE, "disk level: cannot create a spill file in " + base);
    path_ = tmpl.data();
    unlink(path_.c_str());  // anonymous: gone with the descriptor
    heap_.reset(capacity, align);
    const CuFileApi& a = cufile();
    gds_ = false;
    if (a.ok) {
        CUfileDescr_t d{};
        d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
        d.handle.fd = fd_;
        CUfileHandle_t fh = nullptr;
        if (a.HandleRegister(&fh, &d).err == CU_FILE_SUCCESS) {
            fh_ = fh;
            gds_ = true;
        }
    }
    if (!gds_) {
        bounce_bytes_ = 64ull << 20;
        cuda_ok(cudaHostAlloc(&bounce_, bounce_bytes_, cudaHostAllocDefault), "disk bounce buffer");
    }
}

void DiskLevel::close() {
    if (fh_ && cufile().HandleDeregister) cufile().HandleDeregister(fh_);
    fh_ = nullptr;
    if (bounce_) cudaFreeHost(bounce_);
    bounce_ = nullptr;
    if (fd_ >= 0) ::close(fd_);
    fd_ = -1;
    gds_ = false;
}

void DiskLevel::write_from_device(const void* dev, uint64_t size, uint64_t off) {
    if (!size) return;
    if (gds_) {
        const ssize_t n = cufile().Write(fh_, dev, size, static_cast<off_t>(off), 0);
        if (n != static_cast<ssize_t>(size)) raise(BMQ_ERR_STORE, "disk level: cuFileWrite failed");
    } else {
        for (uint64_t done = 0; done < size;) {
            const uint64_t n = std::min(bounce_bytes_, size - done);
            cuda_ok(cudaMemcpy(bounce_, static_cast<const uint8_t*>(dev) + done, n, cudaMemcpyDeviceToHost), "disk write");
            if (pwrite(fd_, bounce_, n, static_cast<off_t>(off + done)) != static_cast<ssize_t>(n))
                raise(BMQ_ERR_STORE, "disk level: write failed");
            done += n;
        }
    }
    bytes_written_ += size;
}

void DiskLevel::read_to_device(void* dev, uint64_t size, uint64_t off) {
    if (!size) return;
    if (gds_) {
        const ssize_t n = cufile().Read(fh_, dev, size, static_cast<off_t>(off), 0);
        if (n != static_cast<ssize_t>(size)) raise(BMQ_ERR_STORE, "disk level: cuFileRead failed");
    } else {
        for (uint64_t done = 0; done < size;) {
            const uint64_t n = std::min(bounce_bytes_, size - done);
            if (pread(fd_, bounce_, n, static_cast<off_t>(off + done)) != static_cast<ssize_t>(n))
                raise(BMQ_ERR_STORE, "disk level: read failed");
            cuda_ok(cudaMemcpy(static_cast<uint8_t*>(dev) + done, bounce_, n, cudaMemcpyHostToDevice), "disk read");
            done += n;
        }
    }
    bytes_read_ += size;
}

void DiskLevel::write_from_host(const void* host, uint64_t size, uint64_t off) {
    for (uint64_t done = 0; done < size;) {
        const ssize_t n = pwrite(fd_, static_cast<const uint8_t*>(host) + done, size - done, static_cast<off_t>(off + done));
        if (n <= 0) raise(BMQ_ERR_STORE, "disk level: write failed");
        done += static_cast<uint64_t>(n);
    }
    bytes_written_ += size;
}

void DiskLevel::read_to_host(void* host, uint64_t size, uint64_t off) {
    for (uint64_t done = 0; done < size;) {
        const ssize_t n = pread(fd_, static_cast<uint8_t*>(host) + done, size - done, static_cast<off_t>(off + done));
        if (n <= 0) raise(BMQ_ERR_STORE, "disk level: read failed");
        done += static_cast<uint64_t>(n);
    }
    bytes_read_ += size;
}

}  // namespace bmq
