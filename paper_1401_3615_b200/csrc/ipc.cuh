// ipc.cuh -- plumbing for one-process-per-GPU drivers that let a kernel read
// another process's device buffer directly (fused transfer + compute):
// CUDA IPC buffers and stream-ordered 32-bit flags (cuStreamWriteValue32 /
// cuStreamWaitValue32, fetched through cudaGetDriverEntryPoint so the library
// does not link libcuda).
// Internal part of libconebeam_b200.so: included by cbb_runtime.cu after
// runtime_common.cuh.
#pragma once

#include <cuda.h>

namespace cbb {

using PfnWriteValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using PfnWaitValue32 = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

struct StreamMemOps {
    PfnWriteValue32 write = nullptr;
    PfnWaitValue32 wait = nullptr;
    static const StreamMemOps& get() {
        static StreamMemOps ops = [] {
            StreamMemOps o;
            cudaDriverEntryPointQueryResult q;
            void* f = nullptr;
            if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) ==
                    cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                o.write = reinterpret_cast<PfnWriteValue32>(f);
            f = nullptr;
            if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) ==
                    cudaSuccess &&
                q == cudaDriverEntryPointSuccess)
                o.wait = reinterpret_cast<PfnWaitValue32>(f);
            cudaGetLastError();
            return o;
        }();
        return ops;
    }
};

inline void check_cu(CUresult r, const char* what) {
    if (r != CUDA_SUCCESS)
        fail(CBB_ERR_INTERNAL, "%s failed (CUresult %d)", what, (int)r);
}

} // namespace cbb
