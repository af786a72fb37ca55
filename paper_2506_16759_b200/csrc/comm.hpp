// In-library NCCL communicator (comm.cpp): run-time loaded libnccl.so.2; failures throw
// h2::Error(H2_ERR_NCCL).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstring>

namespace h2 {
void nccl_unique_id(void* id128);
void* nccl_comm_init(const void* id128, int rank, int nranks);
void nccl_comm_free(void* comm);
// in-place all-gather of byte segments: one NCCL group of broadcasts (segment r rooted at rank r)
void nccl_allgatherv(void* comm, int nranks, void* buf, const int64_t* counts, const int64_t* displs, cudaStream_t st);
// all-to-all of byte segments: one NCCL group of ncclSend / ncclRecv (own segment: device copy)
void nccl_alltoallv(void* comm, int rank, int nranks, const void* send, const int64_t* scounts, const int64_t* sdispls,
                    void* recv, const int64_t* rcounts, const int64_t* rdispls, cudaStream_t st);
}  // namespace h2
