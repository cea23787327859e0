// comm.h -- allreduce over NCCL (see comm.cpp).
#pragma once
#include <cuda_runtime.h>
#include <string.h>

namespace enmf {

struct Comm;
enum class CommType { F64, F32 };
enum class CommOp { Sum, Min, Max };

int comm_init(Comm** out, const void* uid128, int world, int rank);
// In-place allreduce on `st`; no-op when c == nullptr or world == 1.
int comm_allreduce(Comm* c, void* buf, size_t count, CommType t, CommOp op, cudaStream_t st);
// In-place reduce-scatter (sum): buf holds world x count elements; on return this rank's
// block buf[rank * count, (rank + 1) * count) is the sum over ranks (the others are unchanged
// or scratch).  In-place all-gather: this rank's block of buf is sent, every block is filled.
int comm_reduce_scatter(Comm* c, void* buf, size_t count, CommType t, cudaStream_t st);
int comm_allgather(Comm* c, void* buf, size_t count, CommType t, cudaStream_t st);
// In-place sum to `root` (buf holds count elements on every rank; the result on root).
int comm_reduce(Comm* c, void* buf, size_t count, CommType t, int root, cudaStream_t st);
void comm_destroy(Comm* c);
// ncclGetUniqueId into 128 bytes (rank 0 of a job); 0 on success.
int comm_unique_id(void* out128);

}  // namespace enmf
