// fsld_nvls.cu -- the data-parallel gradient exchange through NVSwitch multicast (NVLS).
//
// The loss is a sum over images (optim.py:186-189), so ranks holding disjoint image shards add
// their partial adjoints into one gradient.  Instead of a brick pass followed by an all-reduce,
// every rank maps the SAME multicast object over its own copy of the accumulator and the brick
// kernel's per-item flush issues `multimem.red.add.v2.f32` on the multicast address: NVSwitch
// applies each flush to every rank's copy, so when all ranks have passed the barrier that follows
// the pass, each copy holds the full sum -- the exchange overlaps the compute item by item and no
// separate collective runs.
//
// Set-up (driver API through cudaGetDriverEntryPoint, so the library needs no libcuda at link time):
//   rank 0: fsld_nvls_create (cuMulticastCreate, exported as a POSIX fd when n_ranks > 1)
//   rank r: fsld_nvls_import (the fd, received from rank 0 with fsld_fd_send / fsld_fd_recv:
//           SCM_RIGHTS over an abstract unix socket of the node)
//   all:    fsld_nvls_add_device, then (after every rank added its device) fsld_nvls_bind -- local
//           physical memory bound to the object, mapped twice: the unicast view (read / zero the
//           local copy) and the multicast view (the kernels' reduction target).
// Layout of the bound range: [0, data_bytes) the accumulator; at kCtlOff(data_bytes) the barrier
// word (u32) and, 64 bytes on, one f64 slot per rank (the ranks' |r|^2 sums, summed in rank order
// after the barrier: the loss is the same on every rank and independent of arrival order).
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <cerrno>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <thread>

#include "fsld_b200.h"

namespace {

template <typename F>
F entry(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
    return reinterpret_cast<F>(p);
}

struct Driver {
    decltype(&cuDeviceGet) DeviceGet = nullptr;
    decltype(&cuDeviceGetAttribute) DeviceGetAttribute = nullptr;
    decltype(&cuMulticastGetGranularity) McGranularity = nullptr;
    decltype(&cuMulticastCreate) McCreate = nullptr;
    decltype(&cuMulticastAddDevice) McAddDevice = nullptr;
    decltype(&cuMulticastBindMem) McBindMem = nullptr;
    decltype(&cuMulticastUnbind) McUnbind = nullptr;
    decltype(&cuMemCreate) MemCreate = nullptr;
    decltype(&cuMemRelease) MemRelease = nullptr;
    decltype(&cuMemAddressReserve) AddressReserve = nullptr;
    decltype(&cuMemAddressFree) AddressFree = nullptr;
    decltype(&cuMemMap) Map = nullptr;
    decltype(&cuMemUnmap) Unmap = nullptr;
    decltype(&cuMemSetAccess) SetAccess = nullptr;
    decltype(&cuMemExportToShareableHandle) Export = nullptr;
    decltype(&cuMemImportFromShareableHandle) Import = nullptr;
    bool ok = false;
};

const Driver& drv() {
    static Driver d = [] {
        Driver r;
        r.DeviceGet = entry<decltype(&cuDeviceGet)>("cuDeviceGet");
        r.DeviceGetAttribute = entry<decltype(&cuDeviceGetAttribute)>("cuDeviceGetAttribute");
        r.McGranularity = entry<decltype(&cuMulticastGetGranularity)>("cuMulticastGetGranularity");
        r.McCreate = entry<decltype(&cuMulticastCreate)>("cuMulticastCreate");
        r.McAddDevice = entry<decltype(&cuMulticastAddDevice)>("cuMulticastAddDevice");
        r.McBindMem = entry<decltype(&cuMulticastBindMem)>("cuMulticastBindMem");
        r.McUnbind = entry<decltype(&cuMulticastUnbind)>("cuMulticastUnbind");
        r.MemCreate = entry<decltype(&cuMemCreate)>("cuMemCreate");
        r.MemRelease = entry<decltype(&cuMemRelease)>("cuMemRelease");
        r.AddressReserve = entry<decltype(&cuMemAddressReserve)>("cuMemAddressReserve");
        r.AddressFree = entry<decltype(&cuMemAddressFree)>("cuMemAddressFree");
        r.Map = entry<decltype(&cuMemMap)>("cuMemMap");
        r.Unmap = entry<decltype(&cuMemUnmap)>("cuMemUnmap");
        r.SetAccess = entry<decltype(&cuMemSetAccess)>("cuMemSetAccess");
        r.Export = entry<decltype(&cuMemExportToShareableHandle)>("cuMemExportToShareableHandle");
        r.Import = entry<decltype(&cuMemImportFromShareableHandle)>("cuMemImportFromShareableHandle");
        r.ok = r.DeviceGet && r.DeviceGetAttribute && r.McGranularity && r.McCreate && r.McAddDevice &&
               r.McBindMem && r.McUnbind && r.MemCreate && r.MemRelease && r.AddressReserve && r.AddressFree &&
               r.Map && r.Unmap && r.SetAccess && r.Export && r.Import;
        return r;
    }();
    return d;
}

constexpr size_t kCtlBytes = 4096;  // barrier word + per-rank f64 slots (<= 256 ranks)
constexpr int kMaxRanks = 256;

size_t ctl_off(size_t data_bytes) { return (data_bytes + 255) & ~(size_t)255; }

size_t round_up(size_t x, size_t g) { return (x + g - 1) / g * g; }

}  // namespace

struct fsld_nvls {
    int n_ranks = 0, rank = 0, ordinal = -1;
    size_t data_bytes = 0, size = 0, gran = 0;
    CUmemGenericAllocationHandle mc = 0, mem = 0;
    CUdeviceptr mc_va = 0, uc_va = 0;
    bool have_mc = false, have_mem = false, bound = false, uc_mapped = false, mc_mapped = false;
    int fd = -1;
    unsigned* epoch = nullptr;  // this rank's barrier count (device memory, not shared)
    int* err = nullptr;         // set by a barrier that timed out waiting for a peer
};

namespace {

__global__ void nvls_barrier_kernel(unsigned* mc_flag, const unsigned* uc_flag, unsigned* epoch, int* err, int n,
                                    int rank, double* mc_sq, const double* uc_sq, const double* sq_in,
                                    double* sq_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (sq_in) {
        const double s = *sq_in;
        asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(mc_sq + rank), "d"(s) : "memory");
    }
    // the stream's earlier kernels (the pass and its multicast flushes) are complete; order them
    // and the slot store before the arrival
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    const unsigned e = *epoch + 1u;
    *epoch = e;
    asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" ::"l"(mc_flag), "r"(1u) : "memory");
    const unsigned target = e * (unsigned)n;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned f;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(f) : "l"(uc_flag) : "memory");
        if ((int)(f - target) >= 0) break;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20000000000ull) {  // 20 s without every peer: give up (a peer died), flag it
            atomicExch(err, 1);
            return;
        }
        __nanosleep(256);
    }
    if (sq_out) {  // the ranks' sums in rank order: the same loss on every rank
        double s = 0.0;
        for (int r = 0; r < n; ++r) s += reinterpret_cast<const volatile double*>(uc_sq)[r];
        *sq_out = s;
    }
}

int fail(fsld_nvls* g) {
    fsld_nvls_destroy(g);
    return FSLD_ECUDA;
}

}  // namespace

extern "C" {

int fsld_nvls_supported(int device) {
    const Driver& d = drv();
    if (!d.ok) return 0;
    CUdevice dev;
    if (d.DeviceGet(&dev, device) != CUDA_SUCCESS) return 0;
    int v = 0;
    if (d.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS || !v) return 0;
    // the attribute alone is not enough (a container without the fabric's multicast service reports
    // it and still refuses the object): create and release a minimal one-device team
    CUmulticastObjectProp prop{};
    prop.numDevices = 1;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
    size_t g = 0;
    if (d.McGranularity(&g, &prop, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS || g == 0) return 0;
    prop.size = g;
    CUmemGenericAllocationHandle h = 0;
    if (d.McCreate(&h, &prop) != CUDA_SUCCESS) return 0;
    d.MemRelease(h);
    return 1;
}

size_t fsld_nvls_ctl_offset(size_t data_bytes) { return ctl_off(data_bytes); }

int fsld_nvls_create(int n_ranks, size_t data_bytes, size_t* size_out, int* fd_out, fsld_nvls** out) {
    if (n_ranks < 1 || n_ranks > kMaxRanks || data_bytes == 0 || !size_out || !fd_out || !out) return FSLD_EINVAL;
    const Driver& d = drv();
    if (!d.ok) return FSLD_ENODEV;
    fsld_nvls* g = new fsld_nvls;
    g->n_ranks = n_ranks;
    g->data_bytes = data_bytes;
    CUmulticastObjectProp prop{};
    prop.numDevices = (unsigned)n_ranks;
    prop.size = ctl_off(data_bytes) + kCtlBytes;
    prop.handleTypes = n_ranks > 1 ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
    size_t gmin = 0, grec = 0;
    if (d.McGranularity(&gmin, &prop, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS) return fail(g);
    if (d.McGranularity(&grec, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) grec = gmin;
    g->gran = (grec && grec <= 2 * prop.size) ? grec : gmin;
    g->size = round_up(prop.size, g->gran);
    prop.size = g->size;
    if (d.McCreate(&g->mc, &prop) != CUDA_SUCCESS) return fail(g);
    g->have_mc = true;
    if (n_ranks > 1) {
        int fd = -1;
        if (d.Export(&fd, g->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) != CUDA_SUCCESS) return fail(g);
        g->fd = fd;
    }
    *size_out = g->size;
    *fd_out = g->fd;
    *out = g;
    return FSLD_OK;
}

int fsld_nvls_import(int fd, int n_ranks, int rank, size_t data_bytes, size_t size, fsld_nvls** out) {
    if (fd < 0 || n_ranks < 2 || n_ranks > kMaxRanks || rank < 1 || rank >= n_ranks || !out || data_bytes == 0 ||
        size < ctl_off(data_bytes) + kCtlBytes)
        return FSLD_EINVAL;
    const Driver& d = drv();
    if (!d.ok) return FSLD_ENODEV;
    fsld_nvls* g = new fsld_nvls;
    g->n_ranks = n_ranks;
    g->rank = rank;
    g->data_bytes = data_bytes;
    g->size = size;
    if (d.Import(&g->mc, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) !=
        CUDA_SUCCESS)
        return fail(g);
    g->have_mc = true;
    g->fd = fd;
    CUmulticastObjectProp prop{};
    prop.numDevices = (unsigned)n_ranks;
    prop.size = size;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    if (d.McGranularity(&g->gran, &prop, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS) return fail(g);
    *out = g;
    return FSLD_OK;
}

int fsld_nvls_add_device(fsld_nvls* g) {
    if (!g || !g->have_mc || g->ordinal >= 0) return FSLD_EINVAL;
    const Driver& d = drv();
    int ord = 0;
    if (cudaGetDevice(&ord) != cudaSuccess) return FSLD_ECUDA;
    CUdevice dev;
    if (d.DeviceGet(&dev, ord) != CUDA_SUCCESS) return FSLD_ECUDA;
    if (d.McAddDevice(g->mc, dev) != CUDA_SUCCESS) return FSLD_ECUDA;
    g->ordinal = ord;
    return FSLD_OK;
}

int fsld_nvls_bind(fsld_nvls* g, void** uc_ptr, void** mc_ptr) {
    if (!g || g->ordinal < 0 || g->bound || !uc_ptr || !mc_ptr) return FSLD_EINVAL;
    const Driver& d = drv();
    CUmemAllocationProp mp{};
    mp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    mp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    mp.location.id = g->ordinal;
    if (d.MemCreate(&g->mem, g->size, &mp, 0) != CUDA_SUCCESS) return FSLD_ECUDA;
    g->have_mem = true;
    if (d.McBindMem(g->mc, 0, g->mem, 0, g->size, 0) != CUDA_SUCCESS) return FSLD_ECUDA;
    g->bound = true;
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = g->ordinal;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (d.AddressReserve(&g->uc_va, g->size, g->gran, 0, 0) != CUDA_SUCCESS) return FSLD_ECUDA;
    if (d.Map(g->uc_va, g->size, 0, g->mem, 0) != CUDA_SUCCESS) return FSLD_ECUDA;
    g->uc_mapped = true;
    if (d.SetAccess(g->uc_va, g->size, &acc, 1) != CUDA_SUCCESS) return FSLD_ECUDA;
    if (d.AddressReserve(&g->mc_va, g->size, g->gran, 0, 0) != CUDA_SUCCESS) return FSLD_ECUDA;
    if (d.Map(g->mc_va, g->size, 0, g->mc, 0) != CUDA_SUCCESS) return FSLD_ECUDA;
    g->mc_mapped = true;
    if (d.SetAccess(g->mc_va, g->size, &acc, 1) != CUDA_SUCCESS) return FSLD_ECUDA;
    if (cudaMemset(reinterpret_cast<void*>(g->uc_va), 0, g->size) != cudaSuccess) return FSLD_ECUDA;
    if (cudaMalloc(&g->epoch, 64) != cudaSuccess) return FSLD_ECUDA;
    if (cudaMemset(g->epoch, 0, 64) != cudaSuccess) return FSLD_ECUDA;
    g->err = reinterpret_cast<int*>(g->epoch + 4);
    if (cudaDeviceSynchronize() != cudaSuccess) return FSLD_ECUDA;
    *uc_ptr = reinterpret_cast<void*>(g->uc_va);
    *mc_ptr = reinterpret_cast<void*>(g->mc_va);
    return FSLD_OK;
}

int fsld_nvls_barrier(fsld_nvls* g, const double* sq_in, double* sq_out, void* stream) {
    if (!g || !g->mc_mapped || (sq_out && !sq_in)) return FSLD_EINVAL;
    const size_t co = ctl_off(g->data_bytes);
    unsigned* mc_flag = reinterpret_cast<unsigned*>(g->mc_va + co);
    const unsigned* uc_flag = reinterpret_cast<const unsigned*>(g->uc_va + co);
    double* mc_sq = reinterpret_cast<double*>(g->mc_va + co + 64);
    const double* uc_sq = reinterpret_cast<const double*>(g->uc_va + co + 64);
    nvls_barrier_kernel<<<1, 32, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        mc_flag, uc_flag, g->epoch, g->err, g->n_ranks, g->rank, mc_sq, uc_sq, sq_in, sq_out);
    return cudaGetLastError() == cudaSuccess ? FSLD_OK : FSLD_ECUDA;
}

int fsld_nvls_status(fsld_nvls* g) {
    if (!g || !g->err) return FSLD_EINVAL;
    int e = 0;
    if (cudaMemcpy(&e, g->err, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return FSLD_ECUDA;
    return e ? FSLD_ECUDA : FSLD_OK;
}

int fsld_nvls_destroy(fsld_nvls* g) {
    if (!g) return FSLD_EINVAL;
    const Driver& d = drv();
    cudaDeviceSynchronize();
    if (g->epoch) cudaFree(g->epoch);
    if (g->mc_mapped) d.Unmap(g->mc_va, g->size);
    if (g->mc_va) d.AddressFree(g->mc_va, g->size);
    if (g->uc_mapped) d.Unmap(g->uc_va, g->size);
    if (g->uc_va) d.AddressFree(g->uc_va, g->size);
    if (g->bound) {
        CUdevice dev;
        if (d.DeviceGet(&dev, g->ordinal) == CUDA_SUCCESS) d.McUnbind(g->mc, dev, 0, g->size);
    }
    if (g->have_mem) d.MemRelease(g->mem);
    if (g->have_mc) d.MemRelease(g->mc);
    if (g->fd >= 0) close(g->fd);
    delete g;
    return FSLD_OK;
}

// ---- fd passing between the ranks of one node (SCM_RIGHTS over abstract unix sockets)

static int abstract_addr(const char* name, sockaddr_un& a, socklen_t& len) {
    const size_t n = strlen(name);
    if (n == 0 || n + 1 > sizeof(a.sun_path)) return -1;
    memset(&a, 0, sizeof(a));
    a.sun_family = AF_UNIX;
    memcpy(a.sun_path + 1, name, n);  // sun_path[0] = 0: the abstract namespace (no file)
    len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
    return 0;
}

int fsld_fd_listen(const char* name, int* sock_out) {
    if (!name || !sock_out) return FSLD_EINVAL;
    sockaddr_un a;
    socklen_t len;
    if (abstract_addr(name, a, len) != 0) return FSLD_EINVAL;
    const int s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
    if (s < 0) return FSLD_ECUDA;
    if (bind(s, reinterpret_cast<sockaddr*>(&a), len) != 0 || listen(s, 16) != 0) {
        close(s);
        return FSLD_ECUDA;
    }
    *sock_out = s;
    return FSLD_OK;
}

int fsld_fd_recv(int sock, int* fd_out) {
    if (sock < 0 || !fd_out) return FSLD_EINVAL;
    const int c = accept(sock, nullptr, nullptr);
    close(sock);
    if (c < 0) return FSLD_ECUDA;
    char byte = 0;
    iovec io{&byte, 1};
    alignas(cmsghdr) char ctrl[CMSG_SPACE(sizeof(int))];
    msghdr m{};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    m.msg_control = ctrl;
    m.msg_controllen = sizeof(ctrl);
    const ssize_t r = recvmsg(c, &m, 0);
    close(c);
    cmsghdr* h = CMSG_FIRSTHDR(&m);
    if (r != 1 || !h || h->cmsg_level != SOL_SOCKET || h->cmsg_type != SCM_RIGHTS) return FSLD_ECUDA;
    int fd;
    memcpy(&fd, CMSG_DATA(h), sizeof(int));
    *fd_out = fd;
    return FSLD_OK;
}

int fsld_fd_send(const char* name, int fd) {
    if (!name || fd < 0) return FSLD_EINVAL;
    sockaddr_un a;
    socklen_t len;
    if (abstract_addr(name, a, len) != 0) return FSLD_EINVAL;
    int s = -1;
    for (int attempt = 0; attempt < 200; ++attempt) {  // the receiver listens before the sender is told to send
        s = socket(AF_UNIX, SOCK_STREAM | SOCK_CLOEXEC, 0);
        if (s < 0) return FSLD_ECUDA;
        if (connect(s, reinterpret_cast<sockaddr*>(&a), len) == 0) break;
        close(s);
        s = -1;
        std::this_thread::sleep_for(std::chrono::milliseconds(50));
    }
    if (s < 0) return FSLD_ECUDA;
    char byte = 'F';
    iovec io{&byte, 1};
    alignas(cmsghdr) char ctrl[CMSG_SPACE(sizeof(int))];
    memset(ctrl, 0, sizeof(ctrl));
    msghdr m{};
    m.msg_iov = &io;
    m.msg_iovlen = 1;
    m.msg_control = ctrl;
    m.msg_controllen = sizeof(ctrl);
    cmsghdr* h = CMSG_FIRSTHDR(&m);
    h->cmsg_level = SOL_SOCKET;
    h->cmsg_type = SCM_RIGHTS;
    h->cmsg_len = CMSG_LEN(sizeof(int));
    memcpy(CMSG_DATA(h), &fd, sizeof(int));
    const ssize_t w = sendmsg(s, &m, 0);
    close(s);
    return w == 1 ? FSLD_OK : FSLD_ECUDA;
}

}  // extern "C"
