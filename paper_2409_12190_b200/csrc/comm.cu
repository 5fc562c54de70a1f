// Collective backends of the landmark-sharded solver (see comm.hpp).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "bae_internal.hpp"
#include "comm.hpp"

namespace {
constexpr int kMaxGroup = 16;
}

// In-process rank group: a generation barrier plus, per rank, the buffer it
// contributes to the current collective and two events (data ready, peers
// done reading). Owned by the caller (bae_group_create / bae_group_destroy).
struct bae_group {
  int world = 0;
  // owners: the caller's handle (bae_group_destroy) and every rank's
  // communicator; the last one to let go frees the group, so a problem may
  // outlive the caller's handle
  std::atomic<int> refs{1};
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool broken = false;
  std::vector<const void*> src;
  std::vector<cudaEvent_t> ready, done;
  std::vector<int> dev;

  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (broken) throw bae::Error(BAE_ERR_CUDA, "rank group: a peer rank failed");
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    // a peer that dies must not hang the others forever
    if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      throw bae::Error(BAE_ERR_CUDA, "rank group: barrier timed out or a peer rank failed");
    }
  }
};

namespace bae {
namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(BAE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// NCCL, resolved at run time.
// ---------------------------------------------------------------------------
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                         cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(dlsym(h, "ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(dlsym(h, "ncclAllGather"));
    api.Reduce = reinterpret_cast<decltype(api.Reduce)>(dlsym(h, "ncclReduce"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(dlsym(h, "ncclBroadcast"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllReduce || !api.AllGather ||
        !api.Reduce || !api.Broadcast || !api.GetErrorString) {
      err = "libnccl.so.2 lacks an expected symbol";
      api = NcclApi{};
    }
  });
  if (!api.AllReduce) throw Error(BAE_ERR_NCCL, err);
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw Error(BAE_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

class NcclComm final : public Comm {
 public:
  NcclComm(const void* id128, int rank, int world, int device) : Comm(rank, world) {
    const NcclApi& api = nccl();
    ncclUniqueId id;
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(&id, id128, sizeof(id));
    ck(cudaSetDevice(device), "cudaSetDevice");
    nck(api.CommInitRank(&comm_, world, id, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  void allreduce_sum(double* buf, std::size_t n, cudaStream_t s) override {
    nck(nccl().AllReduce(buf, buf, n, ncclFloat64, ncclSum, comm_, s), "ncclAllReduce(sum)");
  }
  void allreduce_min(int* buf, std::size_t n, cudaStream_t s) override {
    nck(nccl().AllReduce(buf, buf, n, ncclInt32, ncclMin, comm_, s), "ncclAllReduce(min)");
  }
  void reduce_sum(double* buf, std::size_t n, int root, cudaStream_t s) override {
    nck(nccl().Reduce(buf, buf, n, ncclFloat64, ncclSum, root, comm_, s), "ncclReduce(sum)");
  }
  void broadcast(void* buf, std::size_t bytes, int root, cudaStream_t s) override {
    nck(nccl().Broadcast(buf, buf, bytes, ncclUint8, root, comm_, s), "ncclBroadcast");
  }
  void allgather(const void* send, void* recv, std::size_t bytes, cudaStream_t s) override {
    nck(nccl().AllGather(send, recv, bytes, ncclUint8, comm_, s), "ncclAllGather");
  }
  bool capturable() const override { return true; }
  const char* kind() const override { return "nccl"; }

 private:
  ncclComm_t comm_ = nullptr;
};

// ---------------------------------------------------------------------------
// In-process group: fixed-rank-order sums over peer buffers.
// ---------------------------------------------------------------------------
template <class T>
struct PtrPack {
  const T* p[kMaxGroup];
};

__global__ void k_group_sum(PtrPack<double> src, int world, long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double a = src.p[0][i];
    for (int r = 1; r < world; ++r) a += src.p[r][i];
    out[i] = a;
  }
}

__global__ void k_group_min(PtrPack<int> src, int world, long long n, int* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    int a = src.p[0][i];
    for (int r = 1; r < world; ++r) a = min(a, src.p[r][i]);
    out[i] = a;
  }
}

void group_release(bae_group* g) {
  if (g && g->refs.fetch_sub(1) == 1) delete g;
}

class GroupComm final : public Comm {
 public:
  GroupComm(bae_group* g, int rank, int device) : Comm(rank, g->world), g_(g), device_(device) {
    g->refs.fetch_add(1);
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaEventCreateWithFlags(&g->ready[rank], cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&g->done[rank], cudaEventDisableTiming), "event");
    g->dev[rank] = device;
    g->barrier();  // every rank's events and device are registered
    for (int q = 0; q < world(); ++q)
      if (g->dev[q] != device) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(g->dev[q], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          throw Error(BAE_ERR_CUDA, "rank group: peer access between devices is unavailable");
        cudaGetLastError();
      }
  }
  ~GroupComm() override {
    cudaSetDevice(device_);
    if (scratch_) cudaFree(scratch_);
    cudaEventDestroy(g_->ready[rank()]);
    cudaEventDestroy(g_->done[rank()]);
    g_->ready[rank()] = nullptr;
    g_->done[rank()] = nullptr;
    group_release(g_);
  }

  void allreduce_sum(double* buf, std::size_t n, cudaStream_t s) override {
    reduce<double>(buf, n, s, [&](const PtrPack<double>& pk, int blocks, void* out) {
      k_group_sum<<<blocks, 256, 0, s>>>(pk, world(), static_cast<long long>(n), static_cast<double*>(out));
    });
  }
  void allreduce_min(int* buf, std::size_t n, cudaStream_t s) override {
    reduce<int>(buf, n, s, [&](const PtrPack<int>& pk, int blocks, void* out) {
      k_group_min<<<blocks, 256, 0, s>>>(pk, world(), static_cast<long long>(n), static_cast<int*>(out));
    });
  }
  void reduce_sum(double* buf, std::size_t n, int root, cudaStream_t s) override {
    reduce<double>(
        buf, n, s,
        [&](const PtrPack<double>& pk, int blocks, void* out) {
          k_group_sum<<<blocks, 256, 0, s>>>(pk, world(), static_cast<long long>(n), static_cast<double*>(out));
        },
        root);
  }
  void broadcast(void* buf, std::size_t bytes, int root, cudaStream_t s) override {
    if (bytes == 0) return;
    publish(buf, s);
    if (rank() != root) ck(cudaMemcpyAsync(buf, g_->src[root], bytes, cudaMemcpyDefault, s), "group broadcast");
    retire(s);
  }
  void allgather(const void* send, void* recv, std::size_t bytes, cudaStream_t s) override {
    publish(send, s);
    for (int q = 0; q < world(); ++q)
      ck(cudaMemcpyAsync(static_cast<char*>(recv) + q * bytes, g_->src[q], bytes, cudaMemcpyDefault, s),
         "group allgather");
    retire(s);
  }
  bool capturable() const override { return false; }
  const char* kind() const override { return "group"; }

 private:
  // Phase 1: make this rank's buffer visible once its producer finished.
  void publish(const void* buf, cudaStream_t s) {
    ck(cudaEventRecord(g_->ready[rank()], s), "event record");
    g_->src[rank()] = buf;
    g_->barrier();
    for (int q = 0; q < world(); ++q) ck(cudaStreamWaitEvent(s, g_->ready[q], 0), "stream wait");
  }
  // Phase 2: no rank touches its buffer again before every peer read it.
  void retire(cudaStream_t s) {
    ck(cudaEventRecord(g_->done[rank()], s), "event record");
    g_->barrier();
    for (int q = 0; q < world(); ++q)
      if (q != rank()) ck(cudaStreamWaitEvent(s, g_->done[q], 0), "stream wait");
  }
  // Element-wise reduction of every rank's buf (fixed rank order) into buf
  // of every rank, or of `root` only (root >= 0).
  template <class T, class Launch>
  void reduce(T* buf, std::size_t n, cudaStream_t s, Launch launch, int root = -1) {
    if (n == 0) return;
    const bool mine = root < 0 || root == rank();
    if (mine && scratch_bytes_ < n * sizeof(T)) {
      if (scratch_) ck(cudaFree(scratch_), "cudaFree");
      scratch_ = nullptr;
      ck(cudaMalloc(&scratch_, n * sizeof(T)), "cudaMalloc");
      scratch_bytes_ = n * sizeof(T);
    }
    publish(buf, s);
    PtrPack<T> pk{};
    for (int q = 0; q < world(); ++q) pk.p[q] = static_cast<const T*>(g_->src[q]);
    const int blocks = static_cast<int>(std::min<std::size_t>((n + 255) / 256, 1184));
    if (mine) {
      launch(pk, blocks, scratch_);
      ck(cudaGetLastError(), "group reduce launch");
    }
    retire(s);
    if (mine) ck(cudaMemcpyAsync(buf, scratch_, n * sizeof(T), cudaMemcpyDeviceToDevice, s), "group result");
  }

  bae_group* g_;
  int device_;
  void* scratch_ = nullptr;
  std::size_t scratch_bytes_ = 0;
};

}  // namespace

void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  nck(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

std::unique_ptr<Comm> make_nccl_comm(const void* id128, int rank, int world, int device) {
  if (world < 1 || rank < 0 || rank >= world) throw Error(BAE_ERR_INVALID_ARGUMENT, "bad rank / world");
  return std::unique_ptr<Comm>(new NcclComm(id128, rank, world, device));
}

std::unique_ptr<Comm> make_group_comm(bae_group* g, int rank, int device) {
  if (!g || rank < 0 || rank >= g->world) throw Error(BAE_ERR_INVALID_ARGUMENT, "bad rank for the rank group");
  return std::unique_ptr<Comm>(new GroupComm(g, rank, device));
}

bae_group* group_create(int world) {
  if (world < 1 || world > kMaxGroup) throw Error(BAE_ERR_INVALID_ARGUMENT, "rank group: world must be in [1, 16]");
  auto* g = new bae_group;
  g->world = world;
  g->src.assign(static_cast<std::size_t>(world), nullptr);
  g->ready.assign(static_cast<std::size_t>(world), nullptr);
  g->done.assign(static_cast<std::size_t>(world), nullptr);
  g->dev.assign(static_cast<std::size_t>(world), -1);
  return g;
}

void group_destroy(bae_group* g) { group_release(g); }

}  // namespace bae

