// nccl_window.cu -- NCCL 2.28 symmetric-memory windows as the peer-memory transport of NCCL plans.
//
// A workspace allocated with ncclMemAlloc and registered collectively with ncclCommWindowRegister
// (NCCL_WIN_COLL_SYMMETRIC) is mapped by NCCL into every rank of the NVLink domain (LSA team).  NCCL's device API
// gives the address of rank r's copy (ncclGetLsaPointer); the library resolves every rank's base once per plan and
// then runs the same peer-memory exchange as the CUDA-IPC transport on those addresses: copy-engine copies into the
// receivers' regions or direct stores from the pack / attention kernels, ordered by epoch flags in each workspace
// (PAPER.md:95 / :110's per-stage All_to_All, done as peer stores over NVLink / NVSwitch instead of a collective).
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstdint>

#include "spa_internal.h"

namespace spa {

namespace {

__global__ void lsa_bases_kernel(ncclWindow_t w, int n, uint8_t **out) {
    const int i = threadIdx.x;
    if (i < n) out[i] = static_cast<uint8_t *>(ncclGetLsaPointer(w, 0, i));
}

// self-test: every word of the window written through this rank's own LSA address, read back locally
__global__ void lsa_pattern_kernel(uint32_t *lsa_self, long long n_words, uint32_t seed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_words; i += (long long)gridDim.x * blockDim.x)
        lsa_self[i] = (uint32_t)(i * 2654435761u) ^ seed;
}

}  // namespace

// bases[r] = rank r's address of the window's byte 0 (r < n <= 1024), resolved on the device.
cudaError_t nccl_window_bases(ncclWindow_t w, int n, uint8_t **bases, cudaStream_t st) {
    if (n <= 0 || n > 1024) return cudaErrorInvalidValue;
    uint8_t **d = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&d), sizeof(uint8_t *) * n, st);
    if (e != cudaSuccess) return e;
    lsa_bases_kernel<<<1, 1024, 0, st>>>(w, n, d);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(bases, d, sizeof(uint8_t *) * n, cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(d, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e;
}

// The communicator's LSA team (the ranks NCCL maps into each other's address space -- one NVLink domain): size and
// this rank's index in it, from a device communicator with no resource requirements (collective).
ncclResult_t nccl_lsa_team(ncclComm_t comm, int *lsa_size, int *lsa_rank) {
    ncclDevCommRequirements_t reqs = {};
    ncclDevComm_t dc = {};
    ncclResult_t r = ncclDevCommCreate(comm, &reqs, &dc);
    if (r != ncclSuccess) return r;
    *lsa_size = dc.lsaSize;
    *lsa_rank = dc.lsaRank;
    return ncclDevCommDestroy(comm, &dc);
}

cudaError_t nccl_window_fill_pattern(uint32_t *lsa_self, long long n_words, uint32_t seed, cudaStream_t st) {
    lsa_pattern_kernel<<<148, 256, 0, st>>>(lsa_self, n_words, seed);
    return cudaGetLastError();
}

}  // namespace spa
