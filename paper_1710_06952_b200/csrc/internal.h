// internal.h -- host-side declarations shared by the runtime (runtime.cu) and
// the kernel translation units (kernels.cu, engine.cu).  Not part of the ABI.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include "device.cuh"

namespace adp {

// --------------------------------------------------------------- engine ----
struct Slot {                      // per local worker, in the peer-mapped control arena
  unsigned int tag;                // (seq << 2) | state
  unsigned int rem;                // tiles of the running event not yet credited (both GPUs' for a
                                   // coop event): the CTA whose credit brings it to 0 commits
  unsigned long long next;         // claim word of this GPU's share (claim_word, device.cuh)
  unsigned int nwork;              // CTAs of this GPU that tried to join (cross events are capped)
  unsigned int ntiles;             // tiles of the event
  int i, j;
  int tau;
  unsigned int flags;
  long long k;
  float* xi;
  float* xj;
  WorkerCtl* ctl_i;
  WorkerCtl* ctl_j;                // partner's control (local or peer), null if none
  unsigned int* lock;              // lock word held by the running event (free-running)
  unsigned long long ready_ns;     // compute phase ends (free-running)
  unsigned long long t0;
  unsigned int nb_ctr;             // neighbour-choice counter (free-running)
  int pending_j;                   // chosen partner awaiting its lock; -2 none
  long long ev_cur, ev_end;        // replay cursor into ReplayEv list
  int cross;                       // partner lives on another rank
  // App. A (wait_free) and flush-first events; replay reads (stale reads)
  int kind;                        // kKindEvent (ticketed), kKindPull (App. A computation thread),
                                   // kKindRead (replay: gradient at X_{k - tau} into a row)
  unsigned long long key;          // random-draw key of an inline / pulled / read gradient
  float* g;                        // event: gradient row to apply; pull: g_p to compensate with
  float* gout;                     // pull / read: gradient row written
  // slow-link emulation (R21): the passive's lock is released at unlock_at
  unsigned int* held_lock;
  unsigned long long unlock_at;
  int absorb;                      // slot of a passive whose local step (event k-1) is fused into this pair, -1 none
  int coop;                        // cross event processed by both GPUs (the partner claims the odd tiles)
  unsigned int commit_ready;       // mailbox seq of a coop event whose last leave was on the partner GPU
  unsigned int gseq;               // the partner mailbox's sequence for this coop event
};
constexpr int kKindEvent = 0, kKindPull = 1, kKindRead = 2;

struct ReplayEv {                  // one op of a local worker's replay list, in order
  long long k;                     // event index (kKindRead: the event whose gradient is read)
  int j;                           // partner or -1
  unsigned int flags;
  unsigned int e_i, e_j;           // required epochs of i and j before the op
  int kind;                        // kKindEvent or kKindRead
  int grow;                        // gradient row of a stale-read event (-1: inline, tau = 0)
};

struct EngineParams {
  const WorkerDesc* workers;
  const int* nbrs;
  int n;
  int n_local;
  Slot* slots;
  const int* local_ids;            // n_local global ids
  GlobalCtl* gctl0;                // rank 0's GlobalCtl (ticket, log owner)
  GlobalCtl* gctl;                 // this rank's GlobalCtl (error, stats)
  LogEntry* log;                   // rank 0's log ring (peer-mapped on other ranks)
  long long log_cap;
  unsigned long long target;       // free-running: stop when ticket reaches it
  int mode;                        // 0 free-running, 1 replay
  int model;                       // adpsgd_model_kind (NONE / QUADRATIC)
  int my_rank;
  const ReplayEv* rev;
  QuadParams q;
  float gamma;
  long long d;                     // real dimension
  long long n4;                    // d_pad / 4
  long long compute_ns;
  uint2 seed;
  unsigned long long watchdog_ns;
  int wait_free;                   // free-running loop: 0 Alg. 1, 1 App. A, 2 App. A + compensation
  long long link_ns;               // nominal model-transfer time of a 1x link (R21)
  int fuse;                        // fuse a due passive local step into the pair that holds its lock
  unsigned long long fuse_wait_ns; // a due passive stays absorbable this long before stepping alone
  int coop;                        // cooperative cross-GPU events (both GPUs process the tiles)
};

cudaError_t launch_engine(const EngineParams& p, int grid, int threads, bool cooperative, cudaStream_t s);
int engine_max_ctas_per_sm(int threads);

// ---------------------------------------------------- standalone kernels ----
// Pair/local update with external, inline-quadratic, snapshot-quadratic or no gradient.
cudaError_t launch_event(float* xi, float* xj, const float* g, const float* xhat, long long d,
                         long long n4, float gamma, const QuadParams& q, unsigned long long k,
                         int grad_mode, cudaStream_t s, const unsigned long long* guard = nullptr);
cudaError_t launch_quad_grad(const float* xhat, float* g, long long d, long long n4,
                             const QuadParams& q, unsigned long long k, cudaStream_t s);
// lsq (kind 3) / logreg (kind 4): g = sum_m grad F(xhat; (A[idx_m], b[idx_m]))
cudaError_t launch_linear_grad(int kind, const float* A, const float* b, int S, const int* idx,
                               int M, uint2 batch_key, unsigned long long k, const float* xhat,
                               float* g, long long d, cudaStream_t s);
// config 1's whole replay in ONE launch: per event t, the lsq / logreg gradients read at X_t,
// then event t (k_lin_replay, one CTA walking the schedule in order)
struct LinRead {
  const float* x;                  // row read (state X_t)
  float* g;                        // gradient slot written
  const int* idx;                  // explicit batch indices, or null (device Philox)
  unsigned long long k;            // random-draw key
};
struct LinEventOp {
  float *xi, *xj;                  // event t (xi null: reads only)
  const float* g;                  // its gradient slot, null for NO_GRAD
  int ff;                          // App. A flush-first order
  int r0, r1;                      // its reads: LinRead[r0, r1)
};
struct LinReplayParams {
  int kind, S, M, nops;
  const float *A, *b;
  uint2 key;
  const LinRead* reads;            // device arrays
  const LinEventOp* ops;
  float gamma;
  long long d, n4;
};
cudaError_t launch_lin_replay(const LinReplayParams& p, cudaStream_t s);
cudaError_t launch_copy(float* dst, const float* src, long long n4, cudaStream_t s);
cudaError_t launch_fill_hash(float* x, long long n, uint32_t seed, cudaStream_t s);   // diagnostics
// App. A local-update compensation of a pulled model: out = fl(x - fl(gamma gp))
cudaError_t launch_comp_row(const float* x, const float* gp, float gamma, float* out, long long n4, cudaStream_t s);
cudaError_t launch_consensus_sum(const float* X, int n_rows, long long d_pad, long long d,
                                 double* sum, cudaStream_t s);
cudaError_t launch_consensus_finalize(const double* sum, int n, long long d, float* out, unsigned int* err,
                                      cudaStream_t s);
cudaError_t launch_consensus_fused(const float* X, int n_rows, long long d_pad, long long d, int n, float* out,
                                   double* acc, unsigned int* err, cudaStream_t s);   // world 1
cudaError_t launch_consensus_mk(const float* X, int n_rows, long long d_pad, long long d,
                                const double* sum, int n, double* acc, cudaStream_t s);
cudaError_t launch_ar_grad_sum(const float* x, float* gsum, long long d, long long n4,
                               const QuadParams& q, unsigned long long k_base, int n_local,
                               const int* local_ids, cudaStream_t s);
// bookkeeping of a host-path event: ticket = max(ticket, k+1), updates/gossips++, log entry
cudaError_t launch_step_commit(GlobalCtl* gctl0, WorkerCtl* ctl_i, LogEntry* log, long long log_cap,
                               long long k, int i, int j, unsigned int flags, int grad,
                               cudaStream_t s);
cudaError_t launch_set_u64(unsigned long long* p, unsigned long long v, cudaStream_t s);
// super-learner group leader: lock + ticket, then log + unlock (reading R22)
cudaError_t launch_super_lock(unsigned int* lock, unsigned long long* ticket, unsigned long long* kout,
                              unsigned int* err, unsigned long long watchdog_ns, cudaStream_t s);
cudaError_t launch_super_commit(LogEntry* log, long long log_cap, const unsigned long long* kin, int i, int j,
                                unsigned int flags, WorkerCtl* ctl_i, unsigned long long* committed,
                                unsigned int* lock, cudaStream_t s);
cudaError_t launch_ar_update(float* x, const float* gsum, float gamma, int n, long long d,
                             long long n4, cudaStream_t s);
cudaError_t launch_delay(unsigned long long ns, cudaStream_t s);
constexpr int kDpMaxDeg = 16;
cudaError_t launch_dpsgd(const float* const* nbr, const int* deg, const float* w_self, float w_nb, const float* xin,
                         float* xout, int n_local, long long d_pad, long long d, const QuadParams& q, int model,
                         float gamma, unsigned long long k_base, const int* local_ids, cudaStream_t s);
cudaError_t launch_init_rows(float* X, int n_rows, long long d_pad, long long d, const float* x0,
                             cudaStream_t s);

// 3xTF32 tcgen05 GEMM (gemm.cu): C = A . B^T, A [M x K], B [N x K] row-major fp32,
// described by SWIZZLE_128B fp32 tensor maps (box 32 x 128 for A, 32 x bn for B);
// the hi / lo split happens in shared memory
struct GemmGather {                // gathered-operand / epilogue arguments (MLP GEMMs)
  const float* x;                  // gathered rows: x + row * ld
  long long ld;
  const int* idx;                  // row of each batch sample (GEMM1: NULL -> Philox draw below)
  int* idx_out;                    // GEMM1 publishes the batch indices here (may be NULL)
  uint2 key;
  unsigned long long k;
  int S;
  int cluster;                     // CTAs per cluster along z (split-K reduced in DSMEM), 1 = none
  const float* bias;               // GEMM1 epilogue: h = tanh(z + bias)
  // GEMM2's extra CTAs (the last red_ctas of grid.x): the MLP's batch reductions db1, dW2, db2
  // over h, dz1 [M x H] and dz2 [M x O] into g (offsets of b1 / W2 / b2)
  int red_ctas, r_M, r_H, r_O;
  const float *r_h, *r_dz1, *r_dz2;
  float* r_g;
  long long r_off_b1, r_off_W2, r_off_b2;
};
cudaError_t make_tmap_k_major(CUtensorMap* tm, const float* ptr, long long rows, long long cols, int box_rows);
cudaError_t make_tmap_mn_major(CUtensorMap* tm, const float* ptr, long long rows, long long cols);
cudaError_t launch_sum_planes(const float* src, float* dst, int planes, long long n, cudaStream_t s);
cudaError_t launch_gemm_tf32x3(const CUtensorMap& A, const CUtensorMap& B, float* C, int M, int N, int K, int splits,
                               int bn, cudaStream_t s, int cluster = 1);
cudaError_t launch_mlp_gemm1(const CUtensorMap& B, const GemmGather& gg, float* h, int M, int N, int K, int splits,
                             int bn, cudaStream_t s);
cudaError_t launch_mlp_gemm2(const CUtensorMap& A, const GemmGather& gg, float* C, int M, int N, int K, int bn,
                             cudaStream_t s);

// MLP (kind 5): tcgen05-backed gradient (mlp.cu), 3 launches:
//   GEMM1 (batch draw, X rows gathered, split-K reduced in DSMEM) -> per-sample mid
//   (tanh, output layer, softmax-CE backward, dz1) -> GEMM2 (+ the batch reductions in extra CTAs)
struct MlpShape { int n_in, n_hid, n_out; };
struct MlpWork {                   // scratch carve-up + the fixed tensor maps, built once per context
  MlpShape sh;
  int M, splits, planes, bn1, bn2; // planes: GEMM1's cluster-reduced z1 planes (0: GEMM1 writes h)
  float *z1p, *hbuf, *dz1, *dz2;
  int* idx;
  CUtensorMap dz1_m;               // GEMM2 A (MN-major boxes of dz1)
  mutable CUtensorMap w1_m;        // GEMM1 B: W1 of the model row last used (rows never move)
  mutable const float* w1_src = nullptr;
};
size_t mlp_scratch_floats(const MlpShape& sh, int M);
bool mlp_supported(const MlpShape& sh, int M);
cudaError_t mlp_plan(MlpWork& wk, const MlpShape& sh, int M, float* scratch);
cudaError_t launch_mlp_grad(const MlpWork& wk, const float* X, const int* y, int S, const int* idx,
                            uint2 batch_key, unsigned long long k, const float* w, float* g, cudaStream_t s);
constexpr int kMlpLaunches = 3;

// one kernel of each translation unit (CUDA module), see preload_modules()
const void* kernels_module_anchor();
const void* engine_module_anchor();
const void* gemm_module_anchor();
const void* mlp_module_anchor();
const void* comm_module_anchor();

}  // namespace adp
