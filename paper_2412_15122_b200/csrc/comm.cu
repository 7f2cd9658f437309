// comm.cu — transports of the row-sharded path (see comm.h).
#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <vector>

#include "comm.h"

namespace apsp {

size_t dtype_size(ncclDataType_t dt) {
  switch (dt) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;   // ncclInt64, ncclUint64, ncclFloat64
  }
}

// ============================================================================ NCCL
namespace {

struct Nccl {
  bool tried = false, ok = false;
  std::mutex mu;
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool load() {
    std::lock_guard<std::mutex> lk(mu);
    if (tried) return ok;
    tried = true;
    // RTLD_LOCAL: the library's NCCL symbols never interpose on the copy the
    // host framework (torch) may have loaded; APSP_NCCL_LIB overrides the path.
    const char* path = getenv("APSP_NCCL_LIB");
    h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) return false;
#define SYM(name, field)                                            \
  field = reinterpret_cast<decltype(field)>(dlsym(h, "nccl" name)); \
  if (!field) return false;
    SYM("GetUniqueId", GetUniqueId)
    SYM("CommInitRank", CommInitRank)
    SYM("CommDestroy", CommDestroy)
    SYM("Broadcast", Broadcast)
    SYM("AllReduce", AllReduce)
    SYM("AllGather", AllGather)
    SYM("Send", Send)
    SYM("Recv", Recv)
    SYM("GroupStart", GroupStart)
    SYM("GroupEnd", GroupEnd)
    SYM("GetErrorString", GetErrorString)
#undef SYM
    ok = true;
    return true;
  }
};
Nccl g_nccl;

struct NcclComm final : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) g_nccl.CommDestroy(c);
  }
  int bcast(void* buf, size_t count, ncclDataType_t dt, int root, cudaStream_t st) override {
    return (int)g_nccl.Broadcast(buf, buf, count, dt, root, c, st);
  }
  int allreduce(void* buf, size_t count, ncclDataType_t dt, ncclRedOp_t op, cudaStream_t st) override {
    return (int)g_nccl.AllReduce(buf, buf, count, dt, op, c, st);
  }
  int allgather(const void* send, void* recv, size_t count, ncclDataType_t dt, cudaStream_t st) override {
    return (int)g_nccl.AllGather(send, recv, count, dt, c, st);
  }
  int sendrecv(const P2POp* ops, int nops, cudaStream_t st) override {
    ncclResult_t r = g_nccl.GroupStart();
    if (r != ncclSuccess) return (int)r;
    for (int i = 0; i < nops && r == ncclSuccess; ++i)
      r = ops[i].send ? g_nccl.Send(ops[i].buf, ops[i].count, ops[i].dt, ops[i].peer, c, st)
                      : g_nccl.Recv(ops[i].buf, ops[i].count, ops[i].dt, ops[i].peer, c, st);
    ncclResult_t e = g_nccl.GroupEnd();
    return (int)(r != ncclSuccess ? r : e);
  }
  const char* errstr(int code) override { return g_nccl.GetErrorString((ncclResult_t)code); }
};

}  // namespace

bool nccl_unique_id(void* out128) {
  if (!g_nccl.load()) return false;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return false;
  std::memcpy(out128, &id, sizeof id);
  return true;
}

Comm* make_nccl_comm(const void* unique_id128, int world, int rank, int* err) {
  *err = 0;
  if (!g_nccl.load()) {
    *err = (int)ncclSystemError;
    return nullptr;
  }
  ncclUniqueId id;
  std::memcpy(&id, unique_id128, sizeof id);
  auto* c = new NcclComm();
  ncclResult_t r = g_nccl.CommInitRank(&c->c, world, id, rank);
  if (r != ncclSuccess) {
    c->c = nullptr;
    delete c;
    *err = (int)r;
    return nullptr;
  }
  return c;
}

// ============================================================================ reduction kernel
namespace {

constexpr int kMaxLocalWorld = 16;
struct Ptrs {
  const void* p[kMaxLocalWorld];
};

template <typename T>
__device__ __forceinline__ T red(T a, T b, int op) {
  if (op == ncclSum) return a + b;
  if (op == ncclMax) return a > b ? a : b;
  return a < b ? a : b;   // ncclMin
}
template <>
__device__ __forceinline__ float red<float>(float a, float b, int op) {
  if (op == ncclSum) return a + b;
  if (op == ncclMax) return fmaxf(a, b);
  return fminf(a, b);
}

template <typename T>
__global__ void k_reduce_multi(Ptrs in, int g, T* __restrict__ out, size_t count, int op) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x) {
    T a = reinterpret_cast<const T*>(in.p[0])[i];
    for (int r = 1; r < g; ++r) a = red<T>(a, reinterpret_cast<const T*>(in.p[r])[i], op);
    out[i] = a;
  }
}

}  // namespace

cudaError_t reduce_multi(const void* const* ins, int g, void* out, size_t count, ncclDataType_t dt,
                         ncclRedOp_t op, cudaStream_t st) {
  if (g < 1 || g > kMaxLocalWorld || (op != ncclSum && op != ncclMax && op != ncclMin))
    return cudaErrorInvalidValue;
  if (count == 0) return cudaSuccess;
  Ptrs p{};
  for (int r = 0; r < g; ++r) p.p[r] = ins[r];
  const int threads = 256;
  const int blocks = (int)std::min<size_t>((count + threads - 1) / threads, 4096);
  switch (dt) {
    case ncclInt32: k_reduce_multi<int32_t><<<blocks, threads, 0, st>>>(p, g, (int32_t*)out, count, op); break;
    case ncclUint32: k_reduce_multi<uint32_t><<<blocks, threads, 0, st>>>(p, g, (uint32_t*)out, count, op); break;
    case ncclInt64: k_reduce_multi<long long><<<blocks, threads, 0, st>>>(p, g, (long long*)out, count, op); break;
    case ncclUint64:
      k_reduce_multi<unsigned long long><<<blocks, threads, 0, st>>>(p, g, (unsigned long long*)out, count, op);
      break;
    case ncclFloat32: k_reduce_multi<float><<<blocks, threads, 0, st>>>(p, g, (float*)out, count, op); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ============================================================================ in-process group
enum LocalErr { kLocalOk = 0, kLocalCuda = 1001, kLocalMismatch = 1002, kLocalArg = 1003, kLocalTimeout = 1004 };

// A rank that never arrives (its thread failed before the collective) must not
// hang the others forever: every host wait gives up after this long.
std::chrono::seconds local_timeout() {
  const char* e = getenv("APSP_LOCAL_TIMEOUT_S");
  return std::chrono::seconds(e && *e ? atoi(e) : 120);
}

struct LocalGroup {
  enum Kind { kBcast = 1, kAllReduce = 2, kAllGather = 3 };
  struct Post {
    int kind;
    void* buf;          // bcast / allreduce buffer; allgather receive buffer
    const void* sbuf;   // allgather send buffer
    size_t count;
    ncclDataType_t dt;
    ncclRedOp_t op;
    int root;
  };
  struct Msg {
    const void* buf = nullptr;
    size_t bytes = 0;
    cudaEvent_t ready = nullptr, done = nullptr;
    bool acked = false;
  };

  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  int status = 0;
  std::vector<Post> post;
  std::vector<cudaEvent_t> ev_in;
  cudaEvent_t ev_done = nullptr;
  void* tmp = nullptr;                 // reduction scratch (owned by the group)
  size_t tmp_bytes = 8u << 20;
  std::vector<std::deque<std::shared_ptr<Msg>>> box;   // box[src * world + dst]

  // Runs on the last rank to arrive, on its stream `st`, under `mu`.
  int execute(cudaStream_t st) {
    const Post& p0 = post[0];
    for (int r = 1; r < world; ++r)
      if (post[r].kind != p0.kind || post[r].count != p0.count || post[r].dt != p0.dt ||
          post[r].op != p0.op || post[r].root != p0.root)
        return kLocalMismatch;
    for (int r = 0; r < world; ++r)
      if (cudaStreamWaitEvent(st, ev_in[r], 0) != cudaSuccess) return kLocalCuda;
    const size_t es = dtype_size(p0.dt), bytes = p0.count * es;
    cudaError_t e = cudaSuccess;
    if (p0.kind == kBcast) {
      if (p0.root < 0 || p0.root >= world) return kLocalArg;
      for (int r = 0; r < world && e == cudaSuccess; ++r)
        if (r != p0.root && bytes)
          e = cudaMemcpyAsync(post[r].buf, post[p0.root].buf, bytes, cudaMemcpyDeviceToDevice, st);
    } else if (p0.kind == kAllReduce) {
      const size_t chunk = tmp_bytes / es;
      std::vector<const void*> ins(world);
      for (size_t off = 0; off < p0.count && e == cudaSuccess; off += chunk) {
        const size_t c = std::min(chunk, p0.count - off);
        for (int r = 0; r < world; ++r) ins[r] = (const char*)post[r].buf + off * es;
        e = reduce_multi(ins.data(), world, tmp, c, p0.dt, p0.op, st);
        for (int r = 0; r < world && e == cudaSuccess; ++r)
          e = cudaMemcpyAsync((char*)post[r].buf + off * es, tmp, c * es, cudaMemcpyDeviceToDevice, st);
      }
    } else if (p0.kind == kAllGather) {
      for (int src = 0; src < world && e == cudaSuccess; ++src)
        for (int dst = 0; dst < world && e == cudaSuccess; ++dst) {
          void* to = (char*)post[dst].buf + (size_t)src * bytes;
          if (to != post[src].sbuf && bytes)
            e = cudaMemcpyAsync(to, post[src].sbuf, bytes, cudaMemcpyDeviceToDevice, st);
        }
    }
    if (e == cudaSuccess) e = cudaEventRecord(ev_done, st);
    return e == cudaSuccess ? kLocalOk : kLocalCuda;
  }

  int collective(int rank, const Post& p, cudaStream_t st) {
    std::unique_lock<std::mutex> lk(mu);
    if (cudaEventRecord(ev_in[rank], st) != cudaSuccess) return kLocalCuda;
    post[rank] = p;
    const uint64_t my = gen;
    if (++arrived == world) {
      status = execute(st);
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      if (!cv.wait_for(lk, local_timeout(), [&] { return gen != my; })) {
        --arrived;   // withdraw: the group is unusable after a timeout
        return kLocalTimeout;
      }
    }
    if (status != kLocalOk) return status;
    return cudaStreamWaitEvent(st, ev_done, 0) == cudaSuccess ? kLocalOk : kLocalCuda;
  }

  int sendrecv(int rank, const P2POp* ops, int nops, cudaStream_t st) {
    std::unique_lock<std::mutex> lk(mu);
    std::vector<std::shared_ptr<Msg>> mine;
    for (int i = 0; i < nops; ++i) {
      if (!ops[i].send) continue;
      if (ops[i].peer < 0 || ops[i].peer >= world) return kLocalArg;
      auto m = std::make_shared<Msg>();
      m->buf = ops[i].buf;
      m->bytes = ops[i].count * dtype_size(ops[i].dt);
      if (cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming) != cudaSuccess ||
          cudaEventRecord(m->ready, st) != cudaSuccess)
        return kLocalCuda;
      box[(size_t)rank * world + ops[i].peer].push_back(m);
      mine.push_back(m);
    }
    cv.notify_all();
    int status_out = kLocalOk;
    for (int i = 0; i < nops; ++i) {
      if (ops[i].send) continue;
      if (ops[i].peer < 0 || ops[i].peer >= world) return kLocalArg;
      auto& q = box[(size_t)ops[i].peer * world + rank];
      if (!cv.wait_for(lk, local_timeout(), [&] { return !q.empty(); })) return kLocalTimeout;
      std::shared_ptr<Msg> m = q.front();
      q.pop_front();
      const size_t bytes = ops[i].count * dtype_size(ops[i].dt);
      if (bytes != m->bytes) status_out = kLocalMismatch;
      cudaError_t e = cudaStreamWaitEvent(st, m->ready, 0);
      if (e == cudaSuccess && bytes && status_out == kLocalOk)
        e = cudaMemcpyAsync(ops[i].buf, m->buf, bytes, cudaMemcpyDeviceToDevice, st);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&m->done, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventRecord(m->done, st);
      if (e != cudaSuccess) status_out = kLocalCuda;
      m->acked = true;   // acknowledged even on failure: the sender must not hang
      cv.notify_all();
    }
    for (auto& m : mine) {
      if (!cv.wait_for(lk, local_timeout(), [&] { return m->acked; })) return kLocalTimeout;
      if (m->done && cudaStreamWaitEvent(st, m->done, 0) != cudaSuccess) status_out = kLocalCuda;
      cudaEventDestroy(m->ready);
      if (m->done) cudaEventDestroy(m->done);
    }
    return status_out;
  }
};

LocalGroup* local_group_create(int world) {
  if (world < 1 || world > kMaxLocalWorld) return nullptr;
  auto* g = new LocalGroup();
  g->world = world;
  g->post.resize(world);
  g->ev_in.resize(world);
  g->box.resize((size_t)world * world);
  bool ok = cudaMalloc(&g->tmp, g->tmp_bytes) == cudaSuccess &&
            cudaEventCreateWithFlags(&g->ev_done, cudaEventDisableTiming) == cudaSuccess;
  for (int r = 0; r < world && ok; ++r)
    ok = cudaEventCreateWithFlags(&g->ev_in[r], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    local_group_destroy(g);
    return nullptr;
  }
  return g;
}

void local_group_destroy(LocalGroup* g) {
  if (!g) return;
  cudaDeviceSynchronize();
  for (auto e : g->ev_in)
    if (e) cudaEventDestroy(e);
  if (g->ev_done) cudaEventDestroy(g->ev_done);
  if (g->tmp) cudaFree(g->tmp);
  delete g;
}

int local_group_world(const LocalGroup* g) { return g ? g->world : 0; }

namespace {

struct LocalComm final : Comm {
  LocalGroup* g;
  int rank;
  LocalComm(LocalGroup* g_, int r) : g(g_), rank(r) {}
  int bcast(void* buf, size_t count, ncclDataType_t dt, int root, cudaStream_t st) override {
    return g->collective(rank, {LocalGroup::kBcast, buf, nullptr, count, dt, ncclSum, root}, st);
  }
  int allreduce(void* buf, size_t count, ncclDataType_t dt, ncclRedOp_t op, cudaStream_t st) override {
    return g->collective(rank, {LocalGroup::kAllReduce, buf, nullptr, count, dt, op, 0}, st);
  }
  int allgather(const void* send, void* recv, size_t count, ncclDataType_t dt, cudaStream_t st) override {
    return g->collective(rank, {LocalGroup::kAllGather, recv, send, count, dt, ncclSum, 0}, st);
  }
  int sendrecv(const P2POp* ops, int nops, cudaStream_t st) override {
    return g->sendrecv(rank, ops, nops, st);
  }
  const char* errstr(int code) override {
    switch (code) {
      case kLocalCuda: return "local group: CUDA error in a collective";
      case kLocalMismatch: return "local group: ranks called mismatched collectives";
      case kLocalArg: return "local group: bad root/peer";
      case kLocalTimeout: return "local group: timed out waiting for the other ranks";
    }
    return "local group: error";
  }
};

}  // namespace

Comm* make_local_comm(LocalGroup* g, int rank) {
  if (!g || rank < 0 || rank >= g->world) return nullptr;
  return new LocalComm(g, rank);
}

}  // namespace apsp
