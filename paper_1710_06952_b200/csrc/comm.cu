// comm.cu -- NCCL and in-process implementations of adp::Comm (comm.h).
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <iterator>
#include <set>

#include <nccl.h>

#include "../../include/adpsgd.h"
#include "comm.h"

namespace adp {

namespace {

// ------------------------------------------------------------------ NCCL ----
ncclDataType_t nccl_type(DType t) {
  switch (t) {
    case DType::F32: return ncclFloat32;
    case DType::F64: return ncclFloat64;
    case DType::U64: return ncclUint64;
    default: return ncclInt32;
  }
}

ncclRedOp_t nccl_op(ROp op) { return op == ROp::Sum ? ncclSum : (op == ROp::Min ? ncclMin : ncclMax); }

int nccl_fail(ncclResult_t r, const char* what, std::string& err) {
  err = std::string(what) + ": " + ncclGetErrorString(r);
  return ADPSGD_E_NCCL;
}

class NcclComm final : public Comm {
 public:
  NcclComm(ncclComm_t c, int rank, int size) : c_(c) { rank_ = rank; size_ = size; }
  ~NcclComm() override { if (c_) ncclCommDestroy(c_); }
  int allreduce(const void* send, void* recv, size_t count, DType t, ROp op, cudaStream_t s,
                std::string& err) override {
    ncclResult_t r = ncclAllReduce(send, recv, count, nccl_type(t), nccl_op(op), c_, s);
    return r == ncclSuccess ? 0 : nccl_fail(r, "ncclAllReduce", err);
  }
  int broadcast(void* buf, size_t count, DType t, int root, cudaStream_t s, std::string& err) override {
    ncclResult_t r = ncclBroadcast(buf, buf, count, nccl_type(t), root, c_, s);
    return r == ncclSuccess ? 0 : nccl_fail(r, "ncclBroadcast", err);
  }
  int exchange(const std::vector<P2POp>& sends, const std::vector<P2POp>& recvs, cudaStream_t s,
               std::string& err) override {
    ncclResult_t r = ncclGroupStart();
    for (const P2POp& o : recvs)
      if (r == ncclSuccess) r = ncclRecv(o.buf, o.count, ncclFloat32, o.peer, c_, s);
    for (const P2POp& o : sends)
      if (r == ncclSuccess) r = ncclSend(o.buf, o.count, ncclFloat32, o.peer, c_, s);
    ncclResult_t r2 = ncclGroupEnd();
    if (r == ncclSuccess) r = r2;
    return r == ncclSuccess ? 0 : nccl_fail(r, "ncclSend/Recv", err);
  }
  int split(int color, int key, Comm** out, std::string& err) override {
    ncclComm_t sub = nullptr;
    ncclResult_t r = ncclCommSplit(c_, color, key, &sub, nullptr);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommSplit", err);
    int sr = 0, ss = 0;
    ncclCommUserRank(sub, &sr);
    ncclCommCount(sub, &ss);
    *out = new NcclComm(sub, sr, ss);
    return 0;
  }

 private:
  ncclComm_t c_ = nullptr;
};

// ------------------------------------------------------------ in-process ----
// A group of ranks driven by host threads of one process.  Collectives follow
// the NCCL calling convention (every rank calls, same order); each is
//   arrive (publish buffers, record `ready` on the rank's stream) -> barrier ->
//   wait for every rank's `ready`, do this rank's part on its stream, record
//   `done` -> barrier -> wait for every `done` (nobody's inputs are overwritten
//   before all ranks have read them).
// The reductions run over the ranks in rank order (fixed; NCCL's order is its
// own, so results agree bitwise with NCCL for two ranks and within rounding
// otherwise).
constexpr int kMaxRanks = 64;
constexpr double kBarrierTimeoutS = 120.0;

struct Arrival {
  const void* send = nullptr;
  void* recv = nullptr;
  cudaEvent_t ready = nullptr, done = nullptr;
  int device = 0;
  std::vector<P2POp> sends, recvs;
  int color = 0, key = 0;
};

struct LocalGroup {
  std::string id;
  int size = 0;
  std::mutex mu;
  std::condition_variable cv;
  unsigned long long gen = 0;
  int arrived = 0;
  std::vector<Arrival> a;

  bool barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long g = gen;
    if (++arrived == size) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(lk, std::chrono::duration<double>(kBarrierTimeoutS), [&] { return gen != g; });
  }
};

std::mutex g_reg_mu;
std::map<std::string, std::weak_ptr<LocalGroup>> g_groups;

std::shared_ptr<LocalGroup> lookup_group(const std::string& id, int size) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  for (auto e = g_groups.begin(); e != g_groups.end();)        // forget groups whose ranks are gone
    e = e->second.expired() ? g_groups.erase(e) : std::next(e);
  auto it = g_groups.find(id);
  if (it != g_groups.end())
    if (auto g = it->second.lock()) return g->size == size ? g : nullptr;
  auto g = std::make_shared<LocalGroup>();
  g->id = id;
  g->size = size;
  g->a.resize(size);
  g_groups[id] = g;
  return g;
}

struct InPtrs {
  const void* p[kMaxRanks];
};

template <typename T, int kOp>
__global__ void k_reduce_ranks(InPtrs in, int n_in, T* out, size_t count) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    T acc = static_cast<const T*>(in.p[0])[i];
    for (int q = 1; q < n_in; ++q) {
      const T v = static_cast<const T*>(in.p[q])[i];
      if (kOp == 0) acc = acc + v;                     // rank order 0, 1, ..., n-1
      else if (kOp == 1) acc = v < acc ? v : acc;
      else acc = v > acc ? v : acc;
    }
    out[i] = acc;
  }
}

template <typename T>
cudaError_t launch_reduce(const InPtrs& in, int n, void* out, size_t count, ROp op, cudaStream_t s) {
  const int threads = 256;
  const int blocks = (int)std::min<size_t>((count + threads - 1) / threads, 148 * 8);
  if (count == 0) return cudaSuccess;
  if (op == ROp::Sum) k_reduce_ranks<T, 0><<<blocks, threads, 0, s>>>(in, n, static_cast<T*>(out), count);
  else if (op == ROp::Min) k_reduce_ranks<T, 1><<<blocks, threads, 0, s>>>(in, n, static_cast<T*>(out), count);
  else k_reduce_ranks<T, 2><<<blocks, threads, 0, s>>>(in, n, static_cast<T*>(out), count);
  return cudaGetLastError();
}

size_t type_size(DType t) { return t == DType::F32 || t == DType::I32 ? 4 : 8; }

int cuda_fail(cudaError_t e, const char* what, std::string& err) {
  err = std::string(what) + ": " + cudaGetErrorString(e);
  return ADPSGD_E_CUDA;
}

#define LC(x)                                                   \
  do {                                                          \
    cudaError_t e_ = (x);                                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x, err);       \
  } while (0)

class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalGroup> g, int rank, int device) : g_(std::move(g)), device_(device) {
    rank_ = rank;
    size_ = g_->size;
  }
  ~LocalComm() override {
    cudaSetDevice(device_);
    if (ready_) cudaEventDestroy(ready_);
    if (done_) cudaEventDestroy(done_);
    if (tmp_) cudaFree(tmp_);
    for (void* p : old_) cudaFree(p);
  }
  int init(std::string& err) {
    LC(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming));
    LC(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
    return 0;
  }

  int allreduce(const void* send, void* recv, size_t count, DType t, ROp op, cudaStream_t s,
                std::string& err) override {
    const size_t bytes = count * type_size(t);
    if (size_ > kMaxRanks) { err = "in-process group larger than 64 ranks"; return ADPSGD_E_UNSUPPORTED; }
    int rc = ensure_tmp(bytes, err);
    if (rc) return rc;
    Arrival& me = g_->a[rank_];
    me.send = send;
    me.device = device_;
    LC(cudaEventRecord(ready_, s));
    me.ready = ready_;
    me.done = done_;
    if ((rc = sync(err))) return rc;
    InPtrs in{};
    for (int q = 0; q < size_; ++q) {
      in.p[q] = g_->a[q].send;
      if ((rc = peer(g_->a[q].device, err))) return rc;
      LC(cudaStreamWaitEvent(s, g_->a[q].ready, 0));
    }
    cudaError_t e = cudaSuccess;
    switch (t) {
      case DType::F32: e = launch_reduce<float>(in, size_, tmp_, count, op, s); break;
      case DType::F64: e = launch_reduce<double>(in, size_, tmp_, count, op, s); break;
      case DType::U64: e = launch_reduce<unsigned long long>(in, size_, tmp_, count, op, s); break;
      case DType::I32: e = launch_reduce<int>(in, size_, tmp_, count, op, s); break;
    }
    LC(e);
    LC(cudaEventRecord(done_, s));
    if ((rc = sync(err))) return rc;
    for (int q = 0; q < size_; ++q) LC(cudaStreamWaitEvent(s, g_->a[q].done, 0));
    if (bytes) LC(cudaMemcpyAsync(recv, tmp_, bytes, cudaMemcpyDeviceToDevice, s));
    return 0;
  }

  int broadcast(void* buf, size_t count, DType t, int root, cudaStream_t s, std::string& err) override {
    const size_t bytes = count * type_size(t);
    if (root < 0 || root >= size_) { err = "broadcast root"; return ADPSGD_E_INVALID; }
    Arrival& me = g_->a[rank_];
    me.recv = buf;
    me.device = device_;
    LC(cudaEventRecord(ready_, s));
    me.ready = ready_;
    me.done = done_;
    int rc = sync(err);
    if (rc) return rc;
    const Arrival& src = g_->a[root];
    if (rank_ != root && bytes) {
      if ((rc = peer(src.device, err))) return rc;
      LC(cudaStreamWaitEvent(s, src.ready, 0));
      LC(cudaMemcpyAsync(buf, src.recv, bytes, cudaMemcpyDefault, s));
    }
    LC(cudaEventRecord(done_, s));
    if ((rc = sync(err))) return rc;
    if (rank_ == root)
      for (int q = 0; q < size_; ++q) LC(cudaStreamWaitEvent(s, g_->a[q].done, 0));
    return 0;
  }

  int exchange(const std::vector<P2POp>& sends, const std::vector<P2POp>& recvs, cudaStream_t s,
               std::string& err) override {
    Arrival& me = g_->a[rank_];
    me.sends = sends;
    me.recvs = recvs;
    me.device = device_;
    LC(cudaEventRecord(ready_, s));
    me.ready = ready_;
    me.done = done_;
    int rc = sync(err);
    if (rc) return rc;
    std::vector<int> nth(size_, 0);      // receives from each source matched so far
    for (const P2POp& rv : recvs) {
      if (rv.peer < 0 || rv.peer >= size_) { err = "exchange peer"; return ADPSGD_E_INVALID; }
      const Arrival& src = g_->a[rv.peer];
      int seen = 0;
      const P2POp* match = nullptr;
      for (const P2POp& sd : src.sends)
        if (sd.peer == rank_ && seen++ == nth[rv.peer]) { match = &sd; break; }
      if (!match || match->count != rv.count) { err = "exchange: unmatched send/recv"; return ADPSGD_E_INVALID; }
      ++nth[rv.peer];
      if ((rc = peer(src.device, err))) return rc;
      LC(cudaStreamWaitEvent(s, src.ready, 0));
      if (rv.count) LC(cudaMemcpyAsync(rv.buf, match->buf, rv.count * sizeof(float), cudaMemcpyDefault, s));
    }
    LC(cudaEventRecord(done_, s));
    if ((rc = sync(err))) return rc;
    for (int q = 0; q < size_; ++q) LC(cudaStreamWaitEvent(s, g_->a[q].done, 0));
    return 0;
  }

  int split(int color, int key, Comm** out, std::string& err) override {
    Arrival& me = g_->a[rank_];
    me.color = color;
    me.key = key;
    int rc = sync(err);
    if (rc) return rc;
    std::vector<std::pair<int, int>> mem;     // (key, parent rank) of my color
    for (int q = 0; q < size_; ++q)
      if (g_->a[q].color == color) mem.emplace_back(g_->a[q].key, q);
    std::sort(mem.begin(), mem.end());
    int nr = 0;
    while (mem[nr].second != rank_) ++nr;
    const std::string cid = g_->id + "/split" + std::to_string(splits_++) + "/" + std::to_string(color);
    auto child = lookup_group(cid, (int)mem.size());
    if ((rc = sync(err))) return rc;          // everyone read the colors before they are reused
    if (!child) { err = "split: group size mismatch"; return ADPSGD_E_INVALID; }
    auto* c = new LocalComm(child, nr, device_);
    if ((rc = c->init(err))) { delete c; return rc; }
    *out = c;
    return 0;
  }

 private:
  int sync(std::string& err) {
    if (!g_->barrier()) {
      err = "in-process collective: a peer rank did not arrive (barrier timeout)";
      return ADPSGD_E_TIMEOUT;
    }
    return 0;
  }
  int peer(int dev, std::string& err) {
    if (dev == device_ || peers_.count(dev)) return 0;
    cudaError_t e = cudaDeviceEnablePeerAccess(dev, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    else if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess", err);
    peers_.insert(dev);
    return 0;
  }
  int ensure_tmp(size_t bytes, std::string& err) {
    if (bytes <= tmp_bytes_) return 0;
    // the old buffer may still be read by queued work: retire it until destroy
    // (a cudaFree here could wait for peer ranks' persistent engines)
    if (tmp_) old_.push_back(tmp_);
    tmp_ = nullptr;
    LC(cudaMalloc(&tmp_, bytes));
    tmp_bytes_ = bytes;
    return 0;
  }

  std::shared_ptr<LocalGroup> g_;
  int device_ = 0;
  cudaEvent_t ready_ = nullptr, done_ = nullptr;
  void* tmp_ = nullptr;
  size_t tmp_bytes_ = 0;
  std::vector<void*> old_;
  std::set<int> peers_;
  int splits_ = 0;
};

}  // namespace

int make_nccl_comm(const void* id128, int size, int rank, Comm** out, std::string& err) {
  ncclUniqueId id;
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommInitRank(&c, size, id, rank);
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank", err);
  *out = new NcclComm(c, rank, size);
  return 0;
}

int make_local_comm(const void* id128, int size, int rank, int device, Comm** out, std::string& err) {
  if (size < 1 || rank < 0 || rank >= size) { err = "local comm rank/size"; return ADPSGD_E_INVALID; }
  const std::string id(static_cast<const char*>(id128), 128);
  auto g = lookup_group(id, size);
  if (!g) { err = "in-process group exists with another size"; return ADPSGD_E_INVALID; }
  auto* c = new LocalComm(g, rank, device);
  int rc = c->init(err);
  if (rc) { delete c; return rc; }
  *out = c;
  return 0;
}

const void* comm_module_anchor() { return (const void*)k_reduce_ranks<float, 0>; }

}  // namespace adp
