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
  // push request (cross-GPU pair events, two-sided NVLink protocol): the GPU
  // computing an event asks this worker's home GPU to push the row to it
  unsigned int req_tag;            // (request seq << 2) | state, written remotely (release.sys)
  int req_consumer;                // worker whose landing buffer receives the row
  unsigned int req_tag16;          // consumer's event seq (low 16 bits) for the counters
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
  unsigned int pad[8];
};
static_assert(sizeof(WorkerCtl) == 128, "WorkerCtl must be 128 B");

constexpr int kMaxGrid = 1024;     // per-CTA push counters per landing buffer

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
  float* land;                     // landing row (partner rows pushed here), null if world 1
  unsigned int* pcnt;              // kMaxGrid per-CTA push counters of the landing row
  int rank;                        // home rank
  int role;                        // 0 active, 1 passive
  int nb_off, nb_cnt;              // CSR neighbour range
  float straggle;                  // slowdown factor s_w >= 1
  int local;                       // index among this rank's workers, -1 if remote
  float* gb;                       // App. A: two gradient rows (2 * d_pad), local workers only
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

// Per-CTA staging pipeline state.  `consumed` advances identically in every
// thread.  full[s] completes once per use of stage s (TMA bytes landed);
// empty[s] completes once per use when every warp has copied the stage to
// registers (one arrival per warp), so no CTA-wide barrier sits in the loop.
template <int kTile4, int kStages, bool kWarpEmpty = true>
struct Stager {
  float4* buf;      // [kStages][2][kTile4]
  uint64_t* bar;    // [kStages] full
  uint64_t* empty;  // [kStages] empty
  uint32_t consumed;

  // tile use g goes into stage g % kStages once use g - kStages has been drained
  __device__ __forceinline__ void issue(uint32_t g, const float4* xi4, const float4* xj4, long long base,
                                        long long hi) {
    const uint32_t s = g % kStages;
    if (kWarpEmpty && g >= kStages) mbar_wait(empty + s, ((g / kStages) - 1u) & 1u);
    const long long cnt = (hi - base) < kTile4 ? (hi - base) : kTile4;
    const uint32_t bytes = (uint32_t)cnt * 16u;
    mbar_arrive_tx(bar + s, xj4 ? 2u * bytes : bytes);
    bulk_g2s(buf + (size_t)s * 2 * kTile4, xi4 + base, bytes, bar + s);
    if (xj4) bulk_g2s(buf + (size_t)s * 2 * kTile4 + kTile4, xj4 + base, bytes, bar + s);
  }

  // One event over the float4 range [0, hi): this CTA takes tiles first,
  // first + step, first + 2*step, ... (interleaved across the grid, so all
  // CTAs sweep the rows together -- measured ~5% more HBM throughput than
  // contiguous per-CTA slices, tools/membench.cu).
  static __device__ __forceinline__ long long tiles_of(long long first, long long step, long long hi) {
    const long long tot = (hi + kTile4 - 1) / kTile4;
    return tot > first ? (tot - first + step - 1) / step : 0;
  }

  template <bool kPair, int kGrad, bool kFF = false, bool kPreJ = false>
  __device__ __forceinline__ void run(float4* xi4, float4* xj4, long long first, long long step,
                                      long long hi, long long d, float gamma, const QuadParams& q,
                                      uint32_t kk, const float4* g4 = nullptr, uint32_t kkj = 0u) {
    run_range<kPair, kGrad, kFF, kPreJ>(xi4, xj4, xj4, first, step, hi, 0, tiles_of(first, step, hi), d, gamma,
                                        q, kk, g4, kkj);
  }

  // Tiles [t0, t1) of this CTA's list; the partner row is read from xj_src and
  // the average written to xj_dst (equal for an in-place pair; for a cross-GPU
  // event xj_src is the local landing row and xj_dst the peer's model row).
  // kGradExternal reads the gradient row g4 directly (L2), issued before the
  // stage wait so it overlaps the bulk copies.
  template <bool kPair, int kGrad, bool kFF = false, bool kPreJ = false>
  __device__ __forceinline__ void run_range(float4* xi4, const float4* xj_src, float4* xj_dst, long long first,
                                            long long step, long long hi, long long t0, long long t1,
                                            long long d, float gamma, const QuadParams& q, uint32_t kk,
                                            const float4* g4 = nullptr, uint32_t kkj = 0u) {
    const long long n_t = t1 - t0;
    if (n_t <= 0) return;
    if (threadIdx.x == 0) {
      fence_proxy_async();
      for (long long t = 0; t < n_t && t < kStages; ++t)
        issue(consumed + (uint32_t)t, xi4, kPair ? xj_src : nullptr, (first + (t0 + t) * step) * kTile4, hi);
    }
    for (long long t = 0; t < n_t; ++t) {
      const uint32_t g = consumed + (uint32_t)t;
      const uint32_t s = g % kStages;
      const long long base = (first + (t0 + t) * step) * kTile4;
      constexpr int kPer = kTile4 / 512;
      float4 gx[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        gx[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (kGrad == kGradExternal) {
          const long long idx = base + u * 512 + (int)threadIdx.x;
          if (idx < hi) gx[u] = ld_cg4(g4 + idx);
        }
      }
      mbar_wait(bar + s, (g / kStages) & 1u);
      const float4* sa = buf + (size_t)s * 2 * kTile4;
      const float4* sb = sa + kTile4;
      float4 a[kPer], b[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int off = u * 512 + (int)threadIdx.x;
        a[u] = sa[off];
        b[u] = kPair ? sb[off] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (kWarpEmpty) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(empty + s);   // this warp is done with stage s
      } else {
        __syncthreads();                                        // stage s read by every thread
      }
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const long long idx = base + u * 512 + (int)threadIdx.x;
        if (idx < hi) {
          update4<kPair, kGrad, kFF, kPreJ>(a[u], b[u], gx[u], make_float4(0.f, 0.f, 0.f, 0.f), (uint32_t)(idx * 4),
                                            d, gamma, q, kk, kkj);
          if (kPair) st_cg4(xj_dst + idx, b[u]);
          st_cg4(xi4 + idx, a[u]);
        }
      }
      if (threadIdx.x == 0 && t + kStages < n_t)
        issue(g + kStages, xi4, kPair ? xj_src : nullptr, (first + (t0 + t + kStages) * step) * kTile4, hi);
    }
    consumed += (uint32_t)n_t;
  }

  // App. A pull (computation thread): gout = gradient at the
  // pulled model x, compensated by the buffered gradient gp when gp != null.
  // x and gp are staged like x_i / x_j of a pair event; x is not written.
  __device__ __forceinline__ void pull(const float4* x4, const float4* gp4, float4* gout, long long first,
                                       long long step, long long hi, long long d, float gamma, const QuadParams& q,
                                       uint32_t kk) {
    const long long n_t = tiles_of(first, step, hi);
    if (n_t <= 0) return;
    const bool comp = gp4 != nullptr;
    if (threadIdx.x == 0) {
      fence_proxy_async();
      for (long long t = 0; t < n_t && t < kStages; ++t)
        issue(consumed + (uint32_t)t, x4, gp4, (first + t * step) * kTile4, hi);
    }
    for (long long t = 0; t < n_t; ++t) {
      const uint32_t g = consumed + (uint32_t)t;
      const uint32_t s = g % kStages;
      mbar_wait(bar + s, (g / kStages) & 1u);
      const float4* sa = buf + (size_t)s * 2 * kTile4;
      const float4* sb = sa + kTile4;
      const long long base = (first + t * step) * kTile4;
      constexpr int kPer = kTile4 / 512;
      float4 a[kPer], b[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int off = u * 512 + (int)threadIdx.x;
        a[u] = sa[off];
        b[u] = comp ? sb[off] : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (kWarpEmpty) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(empty + s);
      } else {
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const long long idx = base + u * 512 + (int)threadIdx.x;
        if (idx < hi) st_cg4(gout + idx, pull4(a[u], b[u], comp, (uint32_t)(idx * 4), d, gamma, q, kk));
      }
      if (threadIdx.x == 0 && t + kStages < n_t)
        issue(g + kStages, x4, gp4, (first + (t + kStages) * step) * kTile4, hi);
    }
    consumed += (uint32_t)n_t;
  }

  // Push side of a cross-GPU event: copy this CTA's tiles of the local row src
  // into the consumer's landing row dst (a peer address: NVLink writes only) and
  // publish progress as cnt = (tag16 << 16) | tiles_done, release at system scope
  // every kPublish tiles.  Never waits on another GPU.
  template <int kPublish = 8>
  __device__ __forceinline__ void push(const float4* src, float4* dst, unsigned int* cnt, unsigned int tag16,
                                       long long first, long long step, long long hi) {
    const long long n_t = tiles_of(first, step, hi);
    if (n_t <= 0) return;
    if (threadIdx.x == 0) {
      fence_proxy_async();
      for (long long t = 0; t < n_t && t < kStages; ++t)
        issue(consumed + (uint32_t)t, src, nullptr, (first + t * step) * kTile4, hi);
    }
    for (long long t = 0; t < n_t; ++t) {
      const uint32_t g = consumed + (uint32_t)t;
      const uint32_t s = g % kStages;
      mbar_wait(bar + s, (g / kStages) & 1u);
      const float4* sa = buf + (size_t)s * 2 * kTile4;
      const long long base = (first + t * step) * kTile4;
      constexpr int kPer = kTile4 / 512;
      float4 a[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) a[u] = sa[u * 512 + (int)threadIdx.x];
      if (kWarpEmpty) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(empty + s);
      } else {
        __syncthreads();
      }
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const long long idx = base + u * 512 + (int)threadIdx.x;
        if (idx < hi) st_cg4(dst + idx, a[u]);
      }
      if (threadIdx.x == 0 && t + kStages < n_t)
        issue(g + kStages, src, nullptr, (first + (t + kStages) * step) * kTile4, hi);
      if ((t + 1) % kPublish == 0 || t + 1 == n_t) {
        __threadfence_system();                   // every thread's peer stores are performed
        __syncthreads();
        if (threadIdx.x == 0) st_release_sys(cnt, (tag16 << 16) | (unsigned int)(t + 1));
      }
    }
    consumed += (uint32_t)n_t;
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
