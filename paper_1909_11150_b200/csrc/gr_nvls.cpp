// gr_nvls.cpp — NVLink SHARP (NVLS) multicast fusion buffer.
//
// One multicast object spanning the N GPUs, one physical allocation per GPU bound to it:
// a multimem.ld_reduce through the multicast address makes the NVSwitch read every GPU's
// copy and return the sum; a multimem.st writes one value into every GPU's copy. Per rank
// and direction this moves S(1+1/N) bytes for an allreduce of S, against 2S(N-1)/N for the
// two-shot peer-memory path — fewer bytes from N >= 4 on.
//
// Bootstrap (collective, inside gr_init): rank 0 creates the multicast object with a POSIX
// file-descriptor handle (FABRIC handles are refused without an IMEX channel on these boxes),
// passes the fd to every other rank over an abstract AF_UNIX datagram socket (SCM_RIGHTS),
// every rank adds its device, then binds and maps its own physical memory. Every step ends
// with an allgathered vote, so all ranks agree on enabling NVLS; any failure cleans up and
// leaves the context on the peer-memory path. Driver entry points come from
// cudaGetDriverEntryPoint (no link-time dependency on libcuda).
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/time.h>
#include <sys/un.h>
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "gr_nvls.h"

namespace gr {
namespace {

template <typename F>
bool entry(const char *name, F &fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return false;
    fn = reinterpret_cast<F>(p);
    return true;
}

struct Api {
    CUresult (*DeviceGet)(CUdevice *, int);
    CUresult (*DeviceGetAttribute)(int *, CUdevice_attribute, CUdevice);
    CUresult (*DeviceGetUuid)(CUuuid *, CUdevice);
    CUresult (*MulticastGetGranularity)(size_t *, const CUmulticastObjectProp *, CUmulticastGranularity_flags);
    CUresult (*MulticastCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *);
    CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice);
    CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                                 unsigned long long);
    CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
    CUresult (*MemCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *, unsigned long long);
    CUresult (*MemRelease)(CUmemGenericAllocationHandle);
    CUresult (*MemExportToShareableHandle)(void *, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                           unsigned long long);
    CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle *, void *, CUmemAllocationHandleType);
    CUresult (*MemAddressReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long);
    CUresult (*MemAddressFree)(CUdeviceptr, size_t);
    CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    CUresult (*MemUnmap)(CUdeviceptr, size_t);
    CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t);

    bool load() {
        return entry("cuDeviceGet", DeviceGet) && entry("cuDeviceGetAttribute", DeviceGetAttribute) &&
               entry("cuDeviceGetUuid", DeviceGetUuid) &&
               entry("cuMulticastGetGranularity", MulticastGetGranularity) &&
               entry("cuMulticastCreate", MulticastCreate) && entry("cuMulticastAddDevice", MulticastAddDevice) &&
               entry("cuMulticastBindMem", MulticastBindMem) && entry("cuMulticastUnbind", MulticastUnbind) &&
               entry("cuMemCreate", MemCreate) && entry("cuMemRelease", MemRelease) &&
               entry("cuMemExportToShareableHandle", MemExportToShareableHandle) &&
               entry("cuMemImportFromShareableHandle", MemImportFromShareableHandle) &&
               entry("cuMemAddressReserve", MemAddressReserve) && entry("cuMemAddressFree", MemAddressFree) &&
               entry("cuMemMap", MemMap) && entry("cuMemUnmap", MemUnmap) && entry("cuMemSetAccess", MemSetAccess);
    }
};

Api g_api;

std::string sock_name(uint64_t job, int rank) {
    char b[96];
    snprintf(b, sizeof b, "gr-nvls-%016llx-%d", (unsigned long long)job, rank);
    return b;
}

int bind_abstract(const std::string &name) {
    int s = socket(AF_UNIX, SOCK_DGRAM, 0);
    if (s < 0) return -1;
    sockaddr_un a{};
    a.sun_family = AF_UNIX;
    a.sun_path[0] = '\0';
    memcpy(a.sun_path + 1, name.data(), name.size());
    if (bind(s, reinterpret_cast<sockaddr *>(&a), (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + name.size())) != 0) {
        close(s);
        return -1;
    }
    timeval tv{20, 0};
    setsockopt(s, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof tv);
    return s;
}

bool send_fd(const std::string &name, int fd) {
    int s = socket(AF_UNIX, SOCK_DGRAM, 0);
    if (s < 0) return false;
    sockaddr_un a{};
    a.sun_family = AF_UNIX;
    a.sun_path[0] = '\0';
    memcpy(a.sun_path + 1, name.data(), name.size());
    char byte = 'g';
    iovec iov{&byte, 1};
    char cbuf[CMSG_SPACE(sizeof(int))];
    memset(cbuf, 0, sizeof cbuf);
    msghdr m{};
    m.msg_name = &a;
    m.msg_namelen = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + name.size());
    m.msg_iov = &iov;
    m.msg_iovlen = 1;
    m.msg_control = cbuf;
    m.msg_controllen = sizeof cbuf;
    cmsghdr *c = CMSG_FIRSTHDR(&m);
    c->cmsg_level = SOL_SOCKET;
    c->cmsg_type = SCM_RIGHTS;
    c->cmsg_len = CMSG_LEN(sizeof(int));
    memcpy(CMSG_DATA(c), &fd, sizeof(int));
    const bool ok = sendmsg(s, &m, 0) == 1;
    close(s);
    return ok;
}

int recv_fd(int s) {
    char byte;
    iovec iov{&byte, 1};
    char cbuf[CMSG_SPACE(sizeof(int))];
    msghdr m{};
    m.msg_iov = &iov;
    m.msg_iovlen = 1;
    m.msg_control = cbuf;
    m.msg_controllen = sizeof cbuf;
    if (recvmsg(s, &m, 0) != 1) return -1;
    cmsghdr *c = CMSG_FIRSTHDR(&m);
    if (!c || c->cmsg_type != SCM_RIGHTS) return -1;
    int fd;
    memcpy(&fd, CMSG_DATA(c), sizeof(int));
    return fd;
}

}  // namespace

// every rank contributes ok; returns true only if all ranks are ok
static bool vote(const std::function<int(const void *, void *, size_t)> &ag, int N, bool ok) {
    int32_t mine = ok ? 1 : 0;
    std::vector<int32_t> all(N);
    if (ag(&mine, all.data(), sizeof mine) != 0) return false;
    for (int v : all)
        if (!v) return false;
    return true;
}

void nvls_free(Nvls &s) {
    if (s.mcva) {
        g_api.MemUnmap(s.mcva, s.size);
        g_api.MemAddressFree(s.mcva, s.size);
    }
    if (s.ucva) {
        g_api.MemUnmap(s.ucva, s.size);
        g_api.MemAddressFree(s.ucva, s.size);
    }
    if (s.bound) g_api.MulticastUnbind(s.mc, s.cudev, 0, s.size);
    if (s.phys) g_api.MemRelease(s.phys);
    if (s.mc) g_api.MemRelease(s.mc);
    s = Nvls{};
}

int nvls_setup(Nvls &s, int rank, int N, int dev, size_t bytes,
               const std::function<int(const void *, void *, size_t)> &ag, std::string &why) {
    s = Nvls{};
    bool ok = N >= 2 && g_api.load();
    CUdevice cudev = 0;
    int mcsup = 0;
    if (ok) ok = g_api.DeviceGet(&cudev, dev) == CUDA_SUCCESS &&
                 g_api.DeviceGetAttribute(&mcsup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cudev) == CUDA_SUCCESS &&
                 mcsup;
    if (!vote(ag, N, ok)) {
        why = "multicast not supported on every rank";
        return 1;
    }
    {   // one multicast member per device: ranks sharing a GPU (oversubscribed tests) cannot use it
        CUuuid id{};
        ok = g_api.DeviceGetUuid(&id, cudev) == CUDA_SUCCESS;
        std::vector<CUuuid> ids(N);
        if (ag(&id, ids.data(), sizeof(CUuuid)) != 0) ok = false;
        for (int i = 0; ok && i < N; ++i)
            for (int j = i + 1; ok && j < N; ++j)
                if (memcmp(&ids[i], &ids[j], sizeof(CUuuid)) == 0) ok = false;
        if (!vote(ag, N, ok)) {
            why = "ranks share a device (or no device UUID)";
            return 1;
        }
    }
    s.cudev = cudev;
    CUmulticastObjectProp mp{};
    mp.numDevices = (unsigned)N;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = 2u << 20;
    size_t gran = 0;
    ok = g_api.MulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS && gran;
    if (!vote(ag, N, ok)) {
        why = "cuMulticastGetGranularity failed";
        return 1;
    }
    s.size = (bytes + gran - 1) / gran * gran;
    mp.size = s.size;
    // physical memory first (creating it after cuMulticastAddDevice failed on this driver)
    CUmemAllocationProp pp{};
    pp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    pp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    pp.location.id = dev;
    pp.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // must match the multicast object
    CUresult cr = g_api.MemCreate(&s.phys, s.size, &pp, 0);
    if (!vote(ag, N, cr == CUDA_SUCCESS)) {
        why = "cuMemCreate failed (" + std::to_string((int)cr) + ")";
        nvls_free(s);
        return 1;
    }
    // rank 0 creates + exports; a random job id names the sockets
    struct Hdr {
        uint64_t job;
        int32_t ok;
    } mine{0, 1}, r0{};
    int fd = -1;
    if (rank == 0) {
        std::random_device rd;
        mine.job = ((uint64_t)rd() << 32) ^ rd() ^ (uint64_t)getpid();
        mine.ok = g_api.MulticastCreate(&s.mc, &mp) == CUDA_SUCCESS &&
                  g_api.MemExportToShareableHandle(&fd, s.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0) == CUDA_SUCCESS;
    }
    std::vector<Hdr> hs(N);
    if (ag(&mine, hs.data(), sizeof(Hdr)) != 0 || !hs[0].ok) {
        why = "rank 0 could not create/export the multicast object";
        if (fd >= 0) close(fd);
        nvls_free(s);
        return 1;
    }
    r0 = hs[0];
    // fd passing: ranks > 0 bind, vote, rank 0 sends, ranks receive + import
    int sock = -1;
    if (rank > 0) sock = bind_abstract(sock_name(r0.job, rank));
    if (!vote(ag, N, rank == 0 || sock >= 0)) {
        why = "could not bind the fd-passing socket";
        if (sock >= 0) close(sock);
        if (fd >= 0) close(fd);
        nvls_free(s);
        return 1;
    }
    ok = true;
    if (rank == 0) {
        for (int r = 1; r < N; ++r) ok = ok && send_fd(sock_name(r0.job, r), fd);
        close(fd);
    } else {
        const int got = recv_fd(sock);
        ok = got >= 0 && g_api.MemImportFromShareableHandle(&s.mc, (void *)(uintptr_t)got,
                                                            CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR) == CUDA_SUCCESS;
        if (got >= 0) close(got);
        close(sock);
    }
    if (!vote(ag, N, ok)) {
        why = "multicast handle exchange failed";
        nvls_free(s);
        return 1;
    }
    if (!vote(ag, N, g_api.MulticastAddDevice(s.mc, cudev) == CUDA_SUCCESS)) {
        why = "cuMulticastAddDevice failed";
        nvls_free(s);
        return 1;
    }
    CUmemAccessDesc ad{};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = dev;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    int step = 0;
    cr = g_api.MulticastBindMem(s.mc, 0, s.phys, 0, s.size, 0);
    s.bound = cr == CUDA_SUCCESS;
    if (cr == CUDA_SUCCESS && ++step) cr = g_api.MemAddressReserve(&s.ucva, s.size, gran, 0, 0);
    if (cr == CUDA_SUCCESS && ++step) cr = g_api.MemMap(s.ucva, s.size, 0, s.phys, 0);
    if (cr == CUDA_SUCCESS && ++step) cr = g_api.MemSetAccess(s.ucva, s.size, &ad, 1);
    if (cr == CUDA_SUCCESS && ++step) cr = g_api.MemAddressReserve(&s.mcva, s.size, gran, 0, 0);
    if (cr == CUDA_SUCCESS && ++step) cr = g_api.MemMap(s.mcva, s.size, 0, s.mc, 0);
    if (cr == CUDA_SUCCESS && ++step) cr = g_api.MemSetAccess(s.mcva, s.size, &ad, 1);
    ok = cr == CUDA_SUCCESS;
    if (!vote(ag, N, ok)) {
        why = "binding / mapping the multicast memory failed (step " + std::to_string(step) + ", error " +
              std::to_string((int)cr) + ")";
        nvls_free(s);
        return 1;
    }
    s.enabled = true;
    return 0;
}

}  // namespace gr
