// comm.cpp -- NCCL over NVLink/NVSwitch for the row-sharded path.
// NCCL is resolved at run time with dlopen("libnccl.so.2") so the process uses the NCCL
// already loaded by torch (or the system one when used from plain C).  ncclAllReduce for the
// r x r Grams, the PBCD stopping partials and scalars; in a sweep the n x r partial X^T U is
// reduce-scattered (each rank updates its V slice) -- on the tensor-core path one ncclReduce
// per slice, each overlapping the pass's next band range -- and the V slices are all-gathered
// (fp32).
#include <dlfcn.h>
#include <nccl.h>
#include <stdio.h>

#include "comm.h"

namespace enmf {
namespace {

struct Api {
  bool loaded = false;
  void* so = nullptr;
  decltype(&ncclCommInitRank) init = nullptr;
  decltype(&ncclAllReduce) allreduce = nullptr;
  decltype(&ncclReduceScatter) reduce_scatter = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclReduce) reduce = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
};

Api& api() {
  static Api a;
  if (!a.loaded) {
    a.loaded = true;
    a.so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.so) a.so = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (a.so) {
      a.init = (decltype(a.init))dlsym(a.so, "ncclCommInitRank");
      a.allreduce = (decltype(a.allreduce))dlsym(a.so, "ncclAllReduce");
      a.reduce_scatter = (decltype(a.reduce_scatter))dlsym(a.so, "ncclReduceScatter");
      a.allgather = (decltype(a.allgather))dlsym(a.so, "ncclAllGather");
      a.reduce = (decltype(a.reduce))dlsym(a.so, "ncclReduce");
      a.destroy = (decltype(a.destroy))dlsym(a.so, "ncclCommDestroy");
      a.errstr = (decltype(a.errstr))dlsym(a.so, "ncclGetErrorString");
    }
  }
  return a;
}

}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
};

int comm_init(Comm** out, const void* uid128, int world, int rank) {
  *out = nullptr;
  Api& a = api();
  if (!a.init || !a.allreduce || !a.reduce_scatter || !a.allgather || !a.reduce) return -1;
  ncclUniqueId id;
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(&id, uid128, sizeof(id));
  Comm* c = new Comm();
  c->world = world;
  c->rank = rank;
  ncclResult_t rc = a.init(&c->comm, world, id, rank);
  if (rc != ncclSuccess) {
    fprintf(stderr, "enmf: ncclCommInitRank failed: %s\n", a.errstr ? a.errstr(rc) : "?");
    delete c;
    return -1;
  }
  *out = c;
  return 0;
}

int comm_allreduce(Comm* c, void* buf, size_t count, CommType t, CommOp op, cudaStream_t st) {
  if (!c || count == 0) return 0;
  ncclDataType_t dt = t == CommType::F64 ? ncclFloat64 : ncclFloat32;
  ncclRedOp_t o = op == CommOp::Sum ? ncclSum : (op == CommOp::Min ? ncclMin : ncclMax);
  ncclResult_t rc = api().allreduce(buf, buf, count, dt, o, c->comm, st);
  return rc == ncclSuccess ? 0 : -1;
}

int comm_reduce_scatter(Comm* c, void* buf, size_t count, CommType t, cudaStream_t st) {
  if (!c || count == 0) return 0;
  const ncclDataType_t dt = t == CommType::F64 ? ncclFloat64 : ncclFloat32;
  const size_t esz = t == CommType::F64 ? 8 : 4;
  char* b = static_cast<char*>(buf);
  // in place: recvbuff = sendbuff + rank * recvcount (NCCL's in-place convention)
  ncclResult_t rc = api().reduce_scatter(b, b + (size_t)c->rank * count * esz, count, dt, ncclSum,
                                         c->comm, st);
  return rc == ncclSuccess ? 0 : -1;
}

int comm_reduce(Comm* c, void* buf, size_t count, CommType t, int root, cudaStream_t st) {
  if (!c || count == 0) return 0;
  const ncclDataType_t dt = t == CommType::F64 ? ncclFloat64 : ncclFloat32;
  // in place on the root (sendbuff == recvbuff); the other ranks only send
  ncclResult_t rc = api().reduce(buf, buf, count, dt, ncclSum, root, c->comm, st);
  return rc == ncclSuccess ? 0 : -1;
}

int comm_allgather(Comm* c, void* buf, size_t count, CommType t, cudaStream_t st) {
  if (!c || count == 0) return 0;
  const ncclDataType_t dt = t == CommType::F64 ? ncclFloat64 : ncclFloat32;
  const size_t esz = t == CommType::F64 ? 8 : 4;
  char* b = static_cast<char*>(buf);
  // in place: sendbuff = recvbuff + rank * sendcount
  ncclResult_t rc = api().allgather(b + (size_t)c->rank * count * esz, b, count, dt, c->comm, st);
  return rc == ncclSuccess ? 0 : -1;
}

int comm_unique_id(void* out128) {
  Api& a = api();
  if (!a.so) return -1;
  auto get = (decltype(&ncclGetUniqueId))dlsym(a.so, "ncclGetUniqueId");
  if (!get) return -1;
  ncclUniqueId id;
  if (get(&id) != ncclSuccess) return -1;
  memcpy(out128, &id, sizeof(id));
  return 0;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  if (c->comm && api().destroy) api().destroy(c->comm);
  delete c;
}

}  // namespace enmf
