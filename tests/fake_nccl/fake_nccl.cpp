// fake_nccl.cpp -- TEST INFRASTRUCTURE: an in-process stand-in for the NCCL calls
// pbit_sort_list_mg makes, so that G ranks can run the REAL mg.cu kernels and host code on
// ONE GPU, one host thread per rank (NCCL itself refuses two ranks on one device).
//
// Every collective is emulated synchronously: the rank waits for its stream, publishes its
// buffers, meets the other ranks at a barrier, copies what it receives with stream-ordered
// device-to-device copies (all ranks share the device), waits for them, and meets the
// others again before its buffers may change.  Grouped ncclSend/ncclRecv are queued until
// ncclGroupEnd; the k-th send from p to r matches the k-th receive of r from p (NCCL's
// ordering).  Only what mg.cu uses is implemented.  Linked with -Bsymbolic into a test
// build of the library (tests/fake_nccl/build_fake.py); the product links real NCCL.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <atomic>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace {

struct P2P {
  int peer;
  void* ptr;
  size_t bytes;
};

struct World {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> src;           // per rank: published send buffer
  std::vector<size_t> bytes;              // per rank: its byte count
  std::vector<std::vector<P2P>> sends;    // per rank: queued sends of the current group
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

std::mutex g_mu;
std::map<std::string, std::shared_ptr<World>> g_worlds;

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

struct Group {
  int depth = 0;
  ncclComm_t comm = nullptr;
  cudaStream_t stream = nullptr;
  std::vector<P2P> sends, recvs;
};
thread_local Group t_group;
// the communicator and stream of this thread's last call: a group with no operations on
// this rank still has to meet the ranks that do have some
thread_local ncclComm_t t_last_comm = nullptr;
thread_local cudaStream_t t_last_stream = nullptr;

ncclResult_t cuda_ok(cudaError_t e) { return e == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError; }

template <typename T>
void reduce(T* acc, const T* x, size_t count, ncclRedOp_t op) {
  for (size_t i = 0; i < count; ++i) {
    if (op == ncclSum) acc[i] += x[i];
    else if (op == ncclMax) acc[i] = acc[i] < x[i] ? x[i] : acc[i];
    else if (op == ncclMin) acc[i] = x[i] < acc[i] ? x[i] : acc[i];
    else if (op == ncclProd) acc[i] *= x[i];
  }
}

}  // namespace

struct ncclComm {
  int rank = 0, n = 1;
  std::shared_ptr<World> w;
};

extern "C" {

const char* ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "no error (fake NCCL)" : "fake NCCL error"; }

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  static std::atomic<uint64_t> ctr{1};
  memset(id, 0, sizeof *id);
  const uint64_t c = ctr.fetch_add(1) ^ ((uint64_t)(uintptr_t)&ctr << 16);
  memcpy(id->internal, &c, sizeof c);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (!comm || nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  const std::string key(id.internal, sizeof id.internal);
  std::shared_ptr<World> w;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& slot = g_worlds[key];
    if (!slot) {
      slot = std::make_shared<World>();
      slot->n = nranks;
      slot->src.resize(nranks);
      slot->bytes.resize(nranks);
      slot->sends.resize(nranks);
    }
    w = slot;
  }
  if (w->n != nranks) return ncclInvalidUsage;
  auto* c = new ncclComm;
  c->rank = rank;
  c->n = nranks;
  c->w = w;
  w->barrier();  // like ncclCommInitRank: returns once every rank has joined
  *comm = c;
  t_last_comm = c;
  return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  if (t_last_comm == comm) t_last_comm = nullptr;
  delete comm;
  return ncclSuccess;
}
ncclResult_t ncclCommAbort(ncclComm_t comm) { return ncclCommDestroy(comm); }
ncclResult_t ncclCommCount(const ncclComm_t comm, int* count) { *count = comm->n; return ncclSuccess; }
ncclResult_t ncclCommUserRank(const ncclComm_t comm, int* rank) { *rank = comm->rank; return ncclSuccess; }
ncclResult_t ncclCommGetAsyncError(ncclComm_t, ncclResult_t* err) { *err = ncclSuccess; return ncclSuccess; }

ncclResult_t ncclAllGather(const void* sendbuff, void* recvbuff, size_t sendcount, ncclDataType_t dt,
                           ncclComm_t comm, cudaStream_t st) {
  World& w = *comm->w;
  const size_t b = sendcount * type_size(dt);
  t_last_comm = comm;
  t_last_stream = st;
  if (cudaStreamSynchronize(st) != cudaSuccess) return ncclUnhandledCudaError;
  w.src[comm->rank] = sendbuff;
  w.barrier();
  for (int s = 0; s < w.n; ++s) {
    char* dst = (char*)recvbuff + (size_t)s * b;
    if (b && dst != w.src[s] && cudaMemcpyAsync(dst, w.src[s], b, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return ncclUnhandledCudaError;
  }
  const ncclResult_t r = cuda_ok(cudaStreamSynchronize(st));
  w.barrier();
  return r;
}

ncclResult_t ncclAllReduce(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t dt, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t st) {
  World& w = *comm->w;
  const size_t b = count * type_size(dt);
  t_last_comm = comm;
  t_last_stream = st;
  if (cudaStreamSynchronize(st) != cudaSuccess) return ncclUnhandledCudaError;
  w.src[comm->rank] = sendbuff;
  w.barrier();
  std::vector<char> acc(b), x(b);
  ncclResult_t r = ncclSuccess;
  for (int s = 0; s < w.n && r == ncclSuccess; ++s) {
    if (cudaMemcpyAsync(s ? x.data() : acc.data(), w.src[s], b, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      r = ncclUnhandledCudaError;
      break;
    }
    if (!s) continue;
    switch (dt) {
      case ncclInt32: reduce((int32_t*)acc.data(), (const int32_t*)x.data(), count, op); break;
      case ncclUint32: reduce((uint32_t*)acc.data(), (const uint32_t*)x.data(), count, op); break;
      case ncclInt64: reduce((int64_t*)acc.data(), (const int64_t*)x.data(), count, op); break;
      case ncclUint64: reduce((uint64_t*)acc.data(), (const uint64_t*)x.data(), count, op); break;
      default: r = ncclInvalidArgument;
    }
  }
  w.barrier();  // every rank has read every send buffer before any recv buffer changes
  if (r == ncclSuccess && b) {
    r = cuda_ok(cudaMemcpyAsync(recvbuff, acc.data(), b, cudaMemcpyHostToDevice, st));
    if (r == ncclSuccess) r = cuda_ok(cudaStreamSynchronize(st));  // acc is pageable and local
  }
  return r;
}

ncclResult_t ncclGroupStart() {
  ++t_group.depth;
  return ncclSuccess;
}

static ncclResult_t run_p2p(ncclComm_t comm, cudaStream_t st, std::vector<P2P>& sends, std::vector<P2P>& recvs) {
  World& w = *comm->w;
  const int me = comm->rank;
  if (cudaStreamSynchronize(st) != cudaSuccess) return ncclUnhandledCudaError;
  w.sends[me] = sends;
  w.barrier();
  ncclResult_t r = ncclSuccess;
  std::vector<int> taken(w.n, 0);  // sends from each peer to me already matched
  for (const P2P& rv : recvs) {
    const std::vector<P2P>& from = w.sends[rv.peer];
    int k = 0;
    const P2P* hit = nullptr;
    for (const P2P& sd : from)
      if (sd.peer == me && k++ == taken[rv.peer]) { hit = &sd; break; }
    if (!hit || hit->bytes != rv.bytes) { r = ncclInvalidUsage; break; }
    ++taken[rv.peer];
    if (rv.bytes && cudaMemcpyAsync(rv.ptr, hit->ptr, rv.bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess) {
      r = ncclUnhandledCudaError;
      break;
    }
  }
  if (cudaStreamSynchronize(st) != cudaSuccess && r == ncclSuccess) r = ncclUnhandledCudaError;
  w.barrier();
  sends.clear();
  recvs.clear();
  return r;
}

ncclResult_t ncclGroupEnd() {
  if (t_group.depth <= 0) return ncclInvalidUsage;
  if (--t_group.depth) return ncclSuccess;
  ncclComm_t c = t_group.comm ? t_group.comm : t_last_comm;
  cudaStream_t st = t_group.comm ? t_group.stream : t_last_stream;
  t_group.comm = nullptr;
  if (!c) return ncclSuccess;
  return run_p2p(c, st, t_group.sends, t_group.recvs);
}

static ncclResult_t queue(bool send, void* buf, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm,
                          cudaStream_t st) {
  if (peer < 0 || peer >= comm->n) return ncclInvalidArgument;
  if (t_group.comm && (t_group.comm != comm || t_group.stream != st)) return ncclInvalidUsage;
  t_group.comm = comm;
  t_group.stream = st;
  t_last_comm = comm;
  t_last_stream = st;
  (send ? t_group.sends : t_group.recvs).push_back(P2P{peer, buf, count * type_size(dt)});
  if (t_group.depth == 0) {  // outside a group: one operation on its own
    ncclComm_t c = t_group.comm;
    t_group.comm = nullptr;
    return run_p2p(c, st, t_group.sends, t_group.recvs);
  }
  return ncclSuccess;
}

ncclResult_t ncclSend(const void* sendbuff, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm,
                      cudaStream_t st) {
  return queue(true, const_cast<void*>(sendbuff), count, dt, peer, comm, st);
}

ncclResult_t ncclRecv(void* recvbuff, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm, cudaStream_t st) {
  return queue(false, recvbuff, count, dt, peer, comm, st);
}

}  // extern "C"
