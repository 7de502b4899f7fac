// gr_nvls.h — NVLS multicast fusion buffer setup (see gr_nvls.cpp). Internal.
#pragma once
#include <cuda.h>

#include <cstddef>
#include <functional>
#include <string>

namespace gr {

struct Nvls {
    bool enabled = false, bound = false;
    size_t size = 0;
    CUdevice cudev = 0;
    CUmemGenericAllocationHandle mc = 0, phys = 0;
    CUdeviceptr ucva = 0;  // this GPU's copy (unicast view)
    CUdeviceptr mcva = 0;  // the multicast view (multimem.* instructions)
};

// Collective. 0: enabled; 1: unsupported / failed on some rank (every rank returns 1 and
// `why` says why); the allgather callback follows gr_allgather_fn's contract.
int nvls_setup(Nvls &s, int rank, int N, int dev, size_t bytes,
               const std::function<int(const void *, void *, size_t)> &allgather, std::string &why);
void nvls_free(Nvls &s);

}  // namespace gr
