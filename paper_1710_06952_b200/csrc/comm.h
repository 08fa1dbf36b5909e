// comm.h -- the collectives the runtime needs (consensus sum, AllReduce-SGD,
// D-PSGD halo, super-learner groups, ticket agreement) behind one interface,
// with two transports:
//   * NcclComm  -- one process per GPU, NCCL over NVLink (the production path);
//   * LocalComm -- several ranks driven by host threads of ONE process (any
//     device mix, including several virtual ranks on one GPU).  Every rank's
//     buffers are directly addressable, so a collective is a fixed-order device
//     reduction / copy between host barriers, ordered with CUDA events.  This
//     is how the cross-rank engine protocol is exercised on a single B200
//     ("multi-GPU on 1 GPU is the same kernel with local pointers").
// Not part of the ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

namespace adp {

enum class DType { F32, F64, U64, I32 };
enum class ROp { Sum, Min, Max };

struct P2POp {            // one send or receive of a grouped exchange
  void* buf;
  size_t count;           // elements of DType::F32
  int peer;
};

class Comm {
 public:
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int size() const { return size_; }
  // Every call is collective over the communicator, enqueued on `s`, and
  // returns 0 or an adpsgd_status code with `err` set.  recv may alias send.
  virtual int allreduce(const void* send, void* recv, size_t count, DType t, ROp op, cudaStream_t s,
                        std::string& err) = 0;
  virtual int broadcast(void* buf, size_t count, DType t, int root, cudaStream_t s, std::string& err) = 0;
  // grouped point-to-point: the n-th send from a to b matches the n-th receive of b from a
  virtual int exchange(const std::vector<P2POp>& sends, const std::vector<P2POp>& recvs, cudaStream_t s,
                       std::string& err) = 0;
  // sub-communicator of the ranks with the same color, ordered by (key, rank)
  virtual int split(int color, int key, Comm** out, std::string& err) = 0;

 protected:
  int rank_ = 0, size_ = 1;
};

// NCCL: id = the 128-byte ncclUniqueId of rank 0
int make_nccl_comm(const void* id128, int size, int rank, Comm** out, std::string& err);
// In-process: id = any 128-byte token shared by the ranks of one group (threads)
int make_local_comm(const void* id128, int size, int rank, int device, Comm** out, std::string& err);

}  // namespace adp
