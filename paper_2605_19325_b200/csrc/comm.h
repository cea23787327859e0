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
void comm_destroy(Comm* c);
// ncclGetUniqueId into 128 bytes (rank 0 of a job); 0 on success.
int comm_unique_id(void* out128);

}  // namespace enmf
