// device.cuh -- device-side building blocks of the AD-PSGD hot path (sm_100a).
//
// Shared by the standalone kernels (kernels.cu) and the persistent engine
// (engine.cu).  Nothing here is shared with the CPU oracle (oracle/).
//
// Rounding (reading R6): every fp32 op of the update rule and of the
// synthetic quadratic is an explicit round-to-nearest intrinsic (__fadd_rn,
// __fmul_rn, __fsub_rn), which nvcc never contracts into FFMA; the library is
// built without --use_fast_math, so no FTZ/DAZ.
#pragma once
#include <cstdint>
#include <utility>
#include <cuda_runtime.h>

namespace adp {

constexpr int kMaxLocal = 128;        // workers per GPU engine (config 5 at 1 GPU: 128)
constexpr uint32_t kStateIdle = 0, kStateClaimed = 1, kStateRunning = 2, kStateFinished = 3;

// ------------------------------------------------------------ control words --
// One per worker in its HOME GPU's control arena (peer-visible via CUDA IPC).
struct alignas(128) WorkerCtl {
  unsigned int lock;               // 0 free, 1 held (try-lock, system scope)
  unsigned int epoch;              // committed events touching this worker (replay order)
  unsigned long long updates;      // committed gradient updates made by this worker (p_i)
  unsigned long long gossips;      // pair averages initiated by / applied to this worker
  // cooperative cross-GPU event posted in this worker's mailbox (guest_tag):
  // this GPU's share of its tiles is claimed from guest_next, and at most
  // guest_nwork CTAs of this GPU join it (both reset by the poster)
  unsigned long long guest_next;   // claim word of this GPU's half (claim_word)
  unsigned int guest_eseq;         // unused (kept for the 128-byte layout)
  // App. A wait-free runtime (home GPU only; persists across adpsgd_run calls):
  // the computation thread's state and the shared gradient buffer g
  unsigned int wf_state;           // 0 = pull next, 1 = computing (until wf_ready_ns)
  unsigned long long wf_tread_cur; // read point t of the gradient being computed
  unsigned long long wf_tread_pub; // read point of the gradient in the buffer
  unsigned long long wf_ready_ns;  // compute phase of the current gradient ends
  unsigned int wf_pub;             // buffer holds a gradient (g != 0)
  unsigned int wf_buf;             // which of the worker's two gradient rows is the buffer
  unsigned int wf_comp_cur;        // current gradient was compensated
  unsigned int wf_comp_pub;        // buffered gradient was compensated
  // cooperative cross-GPU event (engine): a peer that holds this worker's lock
  // posts its event here so this GPU's CTAs process half of its tiles
  unsigned int guest_tag;          // (event seq << 2) | state, written by the initiator (release.sys)
  int guest_i;                     // initiating worker (its slot holds the event)
  // algorithmic HBM bytes moved in this worker's row by cross-GPU events that a
  // peer committed (this GPU's share of them; engine stats)
  double peer_bytes;
  unsigned int guest_nwork;        // CTAs of this GPU that tried to join the posted guest event
  unsigned int pad[7];
};
static_assert(sizeof(WorkerCtl) == 128, "WorkerCtl must be 128 B");

constexpr int kMaxGrid = 1024;     // engine CTAs per GPU (upper bound)

// One per rank; rank 0's `ticket` is the system-wide virtual counter k.
struct alignas(128) GlobalCtl {
  unsigned long long ticket;       // next k to hand out
  unsigned int error;              // latched device error (adpsgd_status code)
  unsigned int error_info;
  unsigned long long st_events, st_pair, st_cross;   // this rank's engine counters
  unsigned long long st_busy_ns;
  double st_bytes, st_nvl_bytes;
  unsigned int abort_flag;
  unsigned int pad0;
  unsigned long long committed;    // rank 0: events committed system-wide (== ticket when quiescent)
  unsigned long long st_busy_cross_ns;   // part of st_busy_ns spent in cross-GPU events
  unsigned int pad[8];
};

struct LogEntry {                  // == adpsgd_log_entry
  long long k;
  int i, j, tau;
  unsigned int flags;
  unsigned long long t0, t1;
};

struct Slot;                       // engine slot (internal.h)

// Per-worker descriptor, one table per process: pointers valid in THIS process
// (local device memory or IPC-mapped peer memory reached over NVLink).
struct WorkerDesc {
  float* x;                        // model row, d_pad floats
  WorkerCtl* ctl;
  int rank;                        // home rank
  int role;                        // 0 active, 1 passive
  int nb_off, nb_cnt;              // CSR neighbour range
  float straggle;                  // slowdown factor s_w >= 1
  int local;                       // index among this rank's workers, -1 if remote
  float* gb;                       // App. A: two gradient rows (2 * d_pad), local workers only
  float* gr;                       // engine replay with stale reads: T + 1 read-time gradient rows
  float link;                      // link slowdown L_w >= 1 (emulated slow network, R21)
  Slot* slot;                      // the worker's engine slot (home GPU's control arena; peer-mapped)
};

// --------------------------------------------------------------- hashing ----
// lowbias32 integer finaliser: defines the synthetic quadratic.
__device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

// Philox4x32-10 (Salmon et al. SC'11), used for batch sampling and neighbour choice.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u; k.y += 0xBB67AE85u;
  }
  return c;
}

// ------------------------------------------------------- synthetic quadratic --
// f(x) = 1/2 sum_c h_c (x_c - x*_c)^2; batch-SUM stochastic gradient
//   g_c = fl(fl(M h_c) fl(xhat_c - x*_c)) + fl(s (2r-1))
// with h_c, x*_c from the landscape word w_c and the noise grid v_c from the
// noise word (definition v3),
// K_k = lowbias32(lowbias32(lo(k) ^ noise_key) ^ hi(k)).
struct QuadParams {
  uint32_t data_key, noise_key;
  float Mf, s;
};

__host__ __device__ __forceinline__ uint32_t quad_event_key_h(uint32_t noise_key, unsigned long long k) {
  auto lb = [](uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
  };
  return lb(lb((uint32_t)k ^ noise_key) ^ (uint32_t)(k >> 32));
}

// The three uniform grids are built from bits instead of I2F + scale (same
// exact values, no conversion-pipe instructions):
//   (w>>16) * 2^-16        = bits(0x3f800000 | (w>>16)<<7) - 1
//   (w&0xffff) * 2^-15 - 1 = bits(0x40000000 | (w&0xffff)<<7) - 3
//   (u>>9) * 2^-22 - 1     = bits(0x40000000 | u>>9) - 3
// (each subtraction is exact by Sterbenz).
// Landscape word: Weyl sequence (c * 0x9E3779B1) ^ data_key (1 IMAD + 1 LOP3);
// noise word: two multiplies around one xorshift of (c ^ K_k), top 23 bits used.
__device__ __forceinline__ float quad_grad(float xhat, uint32_t c, uint32_t data_key, uint32_t kk,
                                           float Mf, float s) {
  const uint32_t w = (c * 0x9E3779B1u) ^ data_key;
  const float uh = __fsub_rn(__uint_as_float(0x3f800000u | ((w >> 9) & 0x007fff80u)), 1.0f);
  const float h = __fadd_rn(0.01f, __fmul_rn(0.99f, uh));
  const float xs = __fsub_rn(__uint_as_float(0x40000000u | ((w << 7) & 0x007fff80u)), 3.0f);
  uint32_t u = (c ^ kk) * 0x7feb352du;
  u ^= u >> 15;
  u *= 0x846ca68bu;
  const float v = __fsub_rn(__uint_as_float(0x40000000u | (u >> 9)), 3.0f);
  const float noise = __fmul_rn(s, v);
  const float det = __fmul_rn(__fmul_rn(Mf, h), __fsub_rn(xhat, xs));
  return __fadd_rn(det, noise);
}

// ------------------------------------------- programmatic dependent launch ----
// A kernel launched with programmatic stream serialization (launch_pdl) may start
// while its predecessor in the stream is still running: it does its independent
// setup, then waits here for the predecessor to complete and its memory to be
// visible.  Without that launch attribute the wait is a no-op.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// let the stream's next (PDL-launched) kernel start its setup now
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

constexpr bool kUsePdl = true;
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = kUsePdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// --------------------------------------------------------- memory helpers ----
// Model data is read through L2 (.cg): within one persistent launch a row is
// rewritten by other SMs / other GPUs between events, so L1 must not serve it.
__device__ __forceinline__ float4 ld_cg4(const float4* p) { return __ldcg(p); }
__device__ __forceinline__ void st_cg4(float4* p, float4 v) { __stcg(p, v); }

__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned int ld_acquire_sys(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(unsigned int* p, unsigned int v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// -------------------------------------------------- the fused update tile ----
// One float4 of the AD-PSGD event (Alg. 1 steps 4-6):
//   m = fl(fl(x_i + x_j) * 0.5)   (pair only)
//   x_j <- m
//   x_i <- fl(m - fl(gamma * g))  (g from the quadratic at xhat, or external)
enum GradMode { kGradNone = 0, kGradExternal = 1, kGradQuadInline = 2, kGradQuadSnapshot = 3 };
constexpr int kModeFlushFirst = 0x10;   // launch_event: grad_mode | kModeFlushFirst (App. A order)

// Random-draw key of a gradient read at X_t by worker i in the App. A runtime
// (reading R20): the gradient exists before its flush event k is known.
__host__ __device__ __forceinline__ unsigned long long read_key(unsigned long long t, int i) {
  return (1ull << 62) | (t << 20) | (unsigned long long)(uint32_t)i;
}

// kFF = App. A order (Alg. 2): x_i <- fl(x_i - fl(gamma g)) first,
// then m = fl(fl(x_i + x_j) * 0.5) to both endpoints.
// kPreJ = fused passive step (engine): event k-1 is x_j's own local update
// x_j <- fl(x_j - fl(gamma g(x_j; kkj))), applied before event k's average.
template <bool kPair, int kGrad, bool kFF = false, bool kPreJ = false>
__device__ __forceinline__ void update4(float4& a, float4& b, const float4 gext, const float4 xh,
                                        uint32_t c0, long long d, float gamma,
                                        const QuadParams& q, uint32_t kk, uint32_t kkj = 0u) {
  float av[4] = {a.x, a.y, a.z, a.w};
  float bv[4] = {b.x, b.y, b.z, b.w};
  if (kPair && kPreJ) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float gj = (long long)(c0 + e) < d ? quad_grad(bv[e], c0 + e, q.data_key, kkj, q.Mf, q.s) : 0.0f;
      bv[e] = __fsub_rn(bv[e], __fmul_rn(gamma, gj));
    }
  }
  const float gv[4] = {gext.x, gext.y, gext.z, gext.w};
  const float hv[4] = {xh.x, xh.y, xh.z, xh.w};
  float out[4], mv[4];
  const bool tail = (long long)c0 + 4 > d;       // only the last float4s of a row hold padding
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float xhat = (kGrad == kGradQuadInline) ? av[e] : hv[e];   // tau = 0: pre-average x_i
    float g = 0.0f;
    if (kGrad != kGradNone) {
      if (kGrad == kGradExternal) g = gv[e];
      else g = quad_grad(xhat, c0 + e, q.data_key, kk, q.Mf, q.s);
      if (tail && (long long)(c0 + e) >= d) g = 0.0f;                  // padding stays 0
    }
    if (kFF && kGrad != kGradNone) {
      const float xi = __fsub_rn(av[e], __fmul_rn(gamma, g));
      const float m = kPair ? __fmul_rn(__fadd_rn(xi, bv[e]), 0.5f) : xi;
      mv[e] = m;
      out[e] = m;
    } else {
      float m = av[e];
      if (kPair) m = __fmul_rn(__fadd_rn(av[e], bv[e]), 0.5f);
      mv[e] = m;
      out[e] = kGrad != kGradNone ? __fsub_rn(m, __fmul_rn(gamma, g)) : m;
    }
  }
  a = make_float4(out[0], out[1], out[2], out[3]);
  if (kPair) b = make_float4(mv[0], mv[1], mv[2], mv[3]);
}

// App. A computation thread: gradient of the pulled model, with
// the local-update compensation xhat = fl(x - fl(gamma g_p)) when comp.
__device__ __forceinline__ float4 pull4(const float4 x, const float4 gp, bool comp, uint32_t c0, long long d,
                                        float gamma, const QuadParams& q, uint32_t kk) {
  const float xv[4] = {x.x, x.y, x.z, x.w};
  const float pv[4] = {gp.x, gp.y, gp.z, gp.w};
  float out[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float xh = comp ? __fsub_rn(xv[e], __fmul_rn(gamma, pv[e])) : xv[e];
    out[e] = (long long)(c0 + e) < d ? quad_grad(xh, c0 + e, q.data_key, kk, q.Mf, q.s) : 0.0f;
  }
  return make_float4(out[0], out[1], out[2], out[3]);
}

// ------------------------------------------------- bulk-copy (TMA) staging ---
// cp.async.bulk global->shared copies completing on an mbarrier (complete_tx),
// so a CTA keeps kStages tiles of x_i / x_j in flight (HBM or NVLink peer
// addresses alike) without holding them in registers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
// order this thread's (and, after a barrier + fence, the CTA's) generic-proxy
// accesses before subsequent async-proxy (bulk copy) accesses
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

// Dynamic tile claiming.  An event's float4 range is cut into tiles of kTile4
// float4; this GPU's share is the tile list t(c) = c * stride + off for c in
// [0, n) (stride 2 / off 0 or 1 for the halves of a cooperative cross-GPU
// event, else stride 1), dealt in nc = ceil(n / kChunk) chunks of consecutive
// c.  The claim word packs (event seq mod 2^16) << 48 | nc << 32 | chunks
// claimed; one atomicAdd claims a chunk and names the event it belongs to, so
// a CTA that owns a chunk pins its event (the event commits when all its tiles
// are credited) and a late claim on an exhausted counter is harmless (the
// next publish overwrites the word).  Every CTA that joined an event keeps
// claiming until no chunk is left: no CTA waits for a fixed share, and a CTA
// held up on NVLink never delays a local event's tiles.  The next chunk is
// claimed when the current one starts, so its latency hides behind its tiles.
__host__ __device__ __forceinline__ unsigned long long claim_word(unsigned int seq, unsigned int nc) {
  return ((unsigned long long)(seq & 0xFFFFu) << 48) | ((unsigned long long)(nc & 0xFFFFu) << 32);
}
__host__ __device__ __forceinline__ unsigned int claim_seq(unsigned long long w) { return (unsigned int)(w >> 48); }
__host__ __device__ __forceinline__ unsigned int claim_nc(unsigned long long w) {
  return (unsigned int)(w >> 32) & 0xFFFFu;
}
constexpr unsigned int kClaimSeqMask = 0xFFFFu;
__host__ __device__ __forceinline__ unsigned int claim_idx(unsigned long long w) { return (unsigned int)w; }

// chunk = ceil(n / nc) tiles (nc from the claim word, so every claimer agrees)
struct TileClaim {
  unsigned long long* ctr;
  unsigned int n, stride, off, chunk;
  unsigned int c, end, ahead;      // current chunk's next / end c; chunk claimed ahead
  bool out;
  // first = the chunk index the join's claim returned, nc = the word's chunk count
  __device__ __forceinline__ void init(unsigned long long* ctr_, unsigned int n_, unsigned int stride_,
                                       unsigned int off_, unsigned int first, unsigned int nc) {
    ctr = ctr_; n = n_; stride = stride_; off = off_; out = false;
    chunk = (n_ + nc - 1) / nc;
    c = first * chunk;
    end = c + chunk < n ? c + chunk : n;
    ahead = claim_idx(atomicAdd(ctr, 1ull));
  }
  __device__ __forceinline__ int next() {           // thread 0 only; -1 once exhausted
    if (c >= end) {
      if (out || ahead * chunk >= n) { out = true; return -1; }
      c = ahead * chunk;
      end = c + chunk < n ? c + chunk : n;
      ahead = claim_idx(atomicAdd(ctr, 1ull));      // used when this chunk is done
    }
    return (int)(c++ * stride + off);
  }
};

// Per-CTA staging pipeline: kStages tiles of x_i / x_j in flight, filled by
// cp.async.bulk (TMA bulk copies, local HBM or a peer GPU alike) completing on
// an mbarrier (complete_tx).  `consumed` (tile uses so far) advances
// identically in every thread and sets each stage's mbarrier parity.
template <int kTile4, int kStages>
struct Stager {
  // each of the engine's 512 threads applies kTile4 / 512 float4 of a staged tile: a tile size
  // that is not a multiple of 512 would silently leave part of every tile unwritten
  static_assert(kTile4 % 512 == 0, "kTile4 must be a multiple of the engine's 512 threads");
  float4* buf;      // [kStages][2][kTile4]
  uint64_t* bar;    // [kStages] full barriers
  int* stile;       // [kStages] tile held by each stage, -1 = none (shared memory)
  uint32_t consumed;

  __device__ __forceinline__ void issue(uint32_t g, const float4* xi4, const float4* xj4, long long base,
                                        long long hi) {
    const uint32_t s = g % kStages;
    const long long cnt = (hi - base) < kTile4 ? (hi - base) : kTile4;
    const uint32_t bytes = (uint32_t)cnt * 16u;
    mbar_arrive_tx(bar + s, xj4 ? 2u * bytes : bytes);
    bulk_g2s(buf + (size_t)s * 2 * kTile4, xi4 + base, bytes, bar + s);
    if (xj4) bulk_g2s(buf + (size_t)s * 2 * kTile4 + kTile4, xj4 + base, bytes, bar + s);
  }

  // Claim-driven loop shared by events and pulls: thread 0 claims a tile per
  // stage use and issues its copies kStages uses ahead; every thread reads the
  // stage's tile from stile[] (written before a CTA barrier the readers pass).
  // body(tile, a[], b[]) consumes one staged tile.  Returns the tiles done.
  template <class Body>
  __device__ __forceinline__ unsigned int drive(TileClaim& cl, const float4* s0, const float4* s1,
                                                long long hi, Body&& body) {
    if (threadIdx.x == 0) {
      fence_proxy_async();
      for (int t = 0; t < kStages; ++t) {
        const int tile = cl.next();
        stile[(consumed + t) % kStages] = tile;
        if (tile >= 0) issue(consumed + t, s0, s1, (long long)tile * kTile4, hi);
      }
    }
    __syncthreads();
    unsigned int done = 0;
    for (uint32_t g = consumed;; ++g) {
      const uint32_t s = g % kStages;
      const int tile = stile[s];
      if (tile < 0) break;
      body.prefetch((long long)tile * kTile4);
      mbar_wait(bar + s, (g / kStages) & 1u);
      constexpr int kPer = kTile4 / 512;
      const float4* sa = buf + (size_t)s * 2 * kTile4;
      const float4* sb = sa + kTile4;
      float4 a[kPer], b[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int off = u * 512 + (int)threadIdx.x;
        a[u] = sa[off];
        b[u] = s1 ? sb[off] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      __syncthreads();                                  // stage s drained, stile[s] free
      if (threadIdx.x == 0) {
        const int nt = cl.next();
        stile[s] = nt;
        if (nt >= 0) issue(g + kStages, s0, s1, (long long)nt * kTile4, hi);
      }
      body.template consume<kPer>((long long)tile * kTile4, a, b);
      ++done;
    }
    consumed += done;
    return done;
  }
};

// One event's update on staged tiles (Alg. 1 steps 4-6 / App. A order);
// kP float4 per thread per tile (kTile4 / 512).
template <int kP, bool kPair, int kGrad, bool kFF, bool kPreJ>
struct EventBody {
  float4* xi4;
  float4* xj4;
  const float4* g4;
  long long hi, d;
  float gamma;
  QuadParams q;
  uint32_t kk, kkj;
  float4 gx[kP];
  __device__ __forceinline__ void prefetch(long long base) {   // external gradient (L2), before the wait
    if (kGrad == kGradExternal) {
#pragma unroll
      for (int u = 0; u < kP; ++u) {
        const long long idx = base + u * 512 + (int)threadIdx.x;
        gx[u] = idx < hi ? ld_cg4(g4 + idx) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
  template <int kPer>
  __device__ __forceinline__ void consume(long long base, float4* a, float4* b) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const long long idx = base + u * 512 + (int)threadIdx.x;
      if (idx < hi) {
        update4<kPair, kGrad, kFF, kPreJ>(a[u], b[u], kGrad == kGradExternal ? gx[u] : make_float4(0.f, 0.f, 0.f, 0.f),
                                          make_float4(0.f, 0.f, 0.f, 0.f), (uint32_t)(idx * 4), d, gamma, q, kk, kkj);
        if (kPair) st_cg4(xj4 + idx, b[u]);
        st_cg4(xi4 + idx, a[u]);
      }
    }
  }
};

// A gradient read (App. A pull, or the read-time gradient of an
// engine-replayed stale read): gout = gradient at the staged x,
// compensated by the staged gp when comp.
struct ReadBody {
  float4* gout;
  long long hi, d;
  float gamma;
  QuadParams q;
  uint32_t kk;
  bool comp;
  __device__ __forceinline__ void prefetch(long long) {}
  template <int kPer>
  __device__ __forceinline__ void consume(long long base, float4* a, float4* b) {
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const long long idx = base + u * 512 + (int)threadIdx.x;
      if (idx < hi) st_cg4(gout + idx, pull4(a[u], b[u], comp, (uint32_t)(idx * 4), d, gamma, q, kk));
    }
  }
};

// Process float4 range [lo, hi) of one event with `nthreads` threads of a CTA.
// Loads of the (possibly remote) partner row are issued first, U-deep, so that
// NVLink latency overlaps the local HBM loads (SURVEY 8(a) sketch).
template <bool kPair, int kGrad, int U, bool kFF = false>
__device__ __forceinline__ void event_range(float4* __restrict__ xi4, float4* __restrict__ xj4,
                                            const float4* __restrict__ g4,
                                            const float4* __restrict__ xh4, long long lo,
                                            long long hi, int tid, int nthreads, long long d,
                                            float gamma, const QuadParams& q, uint32_t kk) {
  for (long long base = lo + tid; base < hi; base += (long long)nthreads * U) {
    float4 a[U], b[U], gg[U], hh[U];
#pragma unroll
    for (int u = 0; u < U; ++u) b[u] = gg[u] = hh[u] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long idx = base + (long long)u * nthreads;
      if (kPair && idx < hi) b[u] = ld_cg4(xj4 + idx);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long idx = base + (long long)u * nthreads;
      if (idx < hi) {
        a[u] = ld_cg4(xi4 + idx);
        if (kGrad == kGradExternal) gg[u] = ld_cg4(g4 + idx);
        if (kGrad == kGradQuadSnapshot) hh[u] = ld_cg4(xh4 + idx);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long idx = base + (long long)u * nthreads;
      if (idx < hi) {
        update4<kPair, kGrad, kFF>(a[u], b[u], gg[u], hh[u], (uint32_t)(idx * 4), d, gamma, q, kk);
        if (kPair) st_cg4(xj4 + idx, b[u]);
        st_cg4(xi4 + idx, a[u]);
      }
    }
  }
}

}  // namespace adp
