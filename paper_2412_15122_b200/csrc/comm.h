// comm.h — the collectives the row-sharded path needs, behind
// one interface with two transports (internal):
//
//   * NcclComm  — one process per GPU; NCCL over NVLink 5 / NVSwitch, with a
//                 communicator built from the caller's ncclUniqueId (the
//                 production path; libnccl is dlopen()ed only when world > 1).
//   * LocalComm — an in-process group: every rank is a host thread of ONE
//                 process driving its own handle and stream, all on the same
//                 device.  A collective is a host rendezvous followed by
//                 device-to-device copies / one reduction kernel issued on a
//                 single stream, ordered against every rank's stream with CUDA
//                 events.  No kernel ever waits on another kernel, so it is
//                 safe on one GPU (B200_PROFILING.md: never run spinning
//                 ranks as separate launches on one device).  It exists so the
//                 sharded code path — partition, owners, panel broadcasts,
//                 swap-with-last across ranks, reductions — is exercised
//                 bit-for-bit on a single B200 (tests/test_gpu_sharded.py).
//
// Every call is in place where NCCL's is, enqueued on the caller's stream,
// and returns 0 on success or a nonzero code (errstr() names it).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stddef.h>
#include <stdint.h>

namespace apsp {

struct P2POp {
  int send;          // 1 send, 0 receive
  void* buf;         // send: source (read), receive: destination
  size_t count;
  ncclDataType_t dt;
  int peer;
};

struct Comm {
  virtual ~Comm() {}
  virtual int bcast(void* buf, size_t count, ncclDataType_t dt, int root, cudaStream_t st) = 0;
  virtual int allreduce(void* buf, size_t count, ncclDataType_t dt, ncclRedOp_t op,
                        cudaStream_t st) = 0;
  // recv[r*count ...] = rank r's send[0 .. count)
  virtual int allgather(const void* send, void* recv, size_t count, ncclDataType_t dt,
                        cudaStream_t st) = 0;
  // a group of point-to-point transfers posted together (no deadlock when two
  // ranks exchange in both directions)
  virtual int sendrecv(const P2POp* ops, int nops, cudaStream_t st) = 0;
  virtual const char* errstr(int code) = 0;
};

size_t dtype_size(ncclDataType_t dt);

// NCCL transport.  Returns nullptr (and sets *err) if libnccl cannot be
// loaded or the communicator cannot be created.
Comm* make_nccl_comm(const void* unique_id128, int world, int rank, int* err);
bool nccl_unique_id(void* out128);

// In-process group (LocalComm): create once, then one handle per rank.
struct LocalGroup;
LocalGroup* local_group_create(int world);
void local_group_destroy(LocalGroup* g);
int local_group_world(const LocalGroup* g);
Comm* make_local_comm(LocalGroup* g, int rank);

// out[i] = op over the g inputs ins[0..g)[i] (device pointers on the same device)
cudaError_t reduce_multi(const void* const* ins, int g, void* out, size_t count, ncclDataType_t dt,
                         ncclRedOp_t op, cudaStream_t st);

}  // namespace apsp
