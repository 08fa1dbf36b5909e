// kernels.cu -- standalone (stream-ordered) kernels of the AD-PSGD hot path.
//
// Used by the host executor (adpsgd_replay HOST, adpsgd_step, adpsgd_gossip),
// the consensus output and the AllReduce-SGD baseline.
// The persistent free-running/replay engine lives in engine.cu and reuses the
// same per-float4 update (device.cuh: event_range / update4).
#include <algorithm>

#include "internal.h"

namespace adp {

namespace {

constexpr int kThreads = 512;
constexpr int kUnroll = 4;

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// grid sized to whole waves of the 148 SMs (2 CTAs/SM of 512 threads)
int stream_grid(long long n4) {
  long long want = (n4 + (long long)kThreads * kUnroll - 1) / ((long long)kThreads * kUnroll);
  long long cap = 2LL * sm_count();
  if (want < 1) want = 1;
  return (int)(want < cap ? want : cap);
}

// ----------------------------------------------------------- event pass ----
// Each CTA takes a contiguous slice of the float4 range (DRAM-page friendly).
template <bool kPair, int kGrad, bool kFF = false>
__global__ void __launch_bounds__(kThreads, 2) k_event(float* xi, float* xj, const float* g,
                                                    const float* xhat, long long d, long long n4,
                                                    float gamma, QuadParams q, uint32_t kk,
                                                    const unsigned long long* guard) {
  pdl_wait();                               // launched with PDL: the predecessor's rows / gradient
  pdl_trigger();
  if (guard && *guard == ~0ull) return;     // the event's lock wait timed out (error latched): skip
  const long long per = (n4 + gridDim.x - 1) / gridDim.x;
  const long long lo = (long long)blockIdx.x * per;
  const long long hi = lo + per < n4 ? lo + per : n4;
  event_range<kPair, kGrad, kUnroll, kFF>(reinterpret_cast<float4*>(xi), reinterpret_cast<float4*>(xj),
                                     reinterpret_cast<const float4*>(g),
                                     reinterpret_cast<const float4*>(xhat), lo, hi,
                                     threadIdx.x, blockDim.x, d, gamma, q, kk);
}

__global__ void __launch_bounds__(kThreads) k_quad_grad(const float* __restrict__ xhat,
                                                        float* __restrict__ g, long long d,
                                                        long long n4, QuadParams q, uint32_t kk) {
  pdl_wait();                               // PDL launch: wait for the predecessor grid
  pdl_trigger();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 x = ld_cg4(reinterpret_cast<const float4*>(xhat) + i);
    const float xv[4] = {x.x, x.y, x.z, x.w};
    float gv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t c = (uint32_t)(i * 4 + e);
      gv[e] = (long long)c < d ? quad_grad(xv[e], c, q.data_key, kk, q.Mf, q.s) : 0.0f;
    }
    st_cg4(reinterpret_cast<float4*>(g) + i, make_float4(gv[0], gv[1], gv[2], gv[3]));
  }
}

// ----------------------------------------------- lsq / logreg gradient -----
// One CTA per event (d ~ 1024, M ~ 32).  Phase 1: each warp
// forms r_m = a_m . xhat (fp32, lane-strided partial sums + shuffle tree) and
// the per-sample coefficient (lsq: r - b; logreg: -y sigma(-y r)).  Phase 2:
// g_c = sum_m coef_m a_{m,c}, each thread owning columns.
constexpr int kLinThreads = 256;
constexpr int kMaxM = 1024;

__device__ __forceinline__ int32_t batch_index(uint2 key, unsigned long long k, uint32_t m, int S) {
  const uint4 o = philox4x32_10(make_uint4((uint32_t)k, m, 0x42415443u, (uint32_t)(k >> 32)), key);
  return (int32_t)(((unsigned long long)o.x * (unsigned long long)(uint32_t)S) >> 32);
}

__global__ void __launch_bounds__(kLinThreads) k_linear_grad(int kind, const float* __restrict__ A,
                                                             const float* __restrict__ b, int S,
                                                             const int* __restrict__ idx_in, int M,
                                                             uint2 key, unsigned long long k,
                                                             const float* __restrict__ xhat,
                                                             float* __restrict__ g, long long d) {
  pdl_wait();                               // PDL launch: wait for the predecessor grid
  pdl_trigger();
  __shared__ float coef[kMaxM];
  __shared__ int sidx[kMaxM];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int m = threadIdx.x; m < M; m += blockDim.x)
    sidx[m] = idx_in ? idx_in[m] : batch_index(key, k, (uint32_t)m, S);
  __syncthreads();
  for (int m = warp; m < M; m += nw) {
    const float* a = A + (long long)sidx[m] * d;
    float acc = 0.0f;
    for (long long c = lane; c < d; c += 32) acc = fmaf(a[c], __ldcg(xhat + c), acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const float bm = b[sidx[m]];
      if (kind == 3) {
        coef[m] = acc - bm;
      } else {
        const float z = -bm * acc;                       // -y a.x
        coef[m] = -bm / (1.0f + expf(-z));               // -y sigma(-y a.x)
      }
    }
  }
  __syncthreads();
  for (long long c = threadIdx.x; c < d; c += blockDim.x) {
    float acc = 0.0f;
    for (int m = 0; m < M; ++m) acc = fmaf(coef[m], A[(long long)sidx[m] * d + c], acc);
    g[c] = acc;
  }
}

// Same gradient, vectorised for d % 4 == 0 (config 1 is latency-bound, SURVEY
// 8(d)): 1024 threads; phase 1 gives each warp whole samples (8 independent
// float4 loads per lane at d = 1024 instead of 32 dependent scalar ones);
// phase 2 splits the M samples into 4 quarters per float4 column group and
// adds the quarters in a fixed order (deterministic).
constexpr int kLinThreadsV = 1024;
struct LinSmem {
  float coef[kMaxM];
  int sidx[kMaxM];
  float4 quarter[3][256];
};

__device__ __forceinline__ void linear_grad_v_body(LinSmem& sm, int kind, const float* __restrict__ A,
                                                   const float* __restrict__ b, int S,
                                                   const int* __restrict__ idx_in, int M, uint2 key,
                                                   unsigned long long k, const float* __restrict__ xhat,
                                                   float* __restrict__ g, long long d) {
  float* coef = sm.coef;
  int* sidx = sm.sidx;
  float4 (*quarter)[256] = sm.quarter;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const long long d4 = d >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(xhat);
  for (int m = threadIdx.x; m < M; m += blockDim.x)
    sidx[m] = idx_in ? idx_in[m] : batch_index(key, k, (uint32_t)m, S);
  __syncthreads();
  for (int m = warp; m < M; m += nw) {
    const float4* a4 = reinterpret_cast<const float4*>(A + (long long)sidx[m] * d);
    float acc = 0.0f;
#pragma unroll 8
    for (long long c = lane; c < d4; c += 32) {        // unrolled: the loads of a row are in flight together
      const float4 av = __ldg(a4 + c), xv = __ldcg(x4 + c);
      acc = fmaf(av.x, xv.x, acc);
      acc = fmaf(av.y, xv.y, acc);
      acc = fmaf(av.z, xv.z, acc);
      acc = fmaf(av.w, xv.w, acc);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const float bm = b[sidx[m]];
      if (kind == 3) {
        coef[m] = acc - bm;
      } else {
        const float z = -bm * acc;                       // -y a.x
        coef[m] = -bm / (1.0f + expf(-z));               // -y sigma(-y a.x)
      }
    }
  }
  __syncthreads();
  const int q = threadIdx.x >> 8, t = threadIdx.x & 255;           // sample quarter, column group
  for (long long c0 = 0; c0 < d4; c0 += 256) {
    const long long c = c0 + t;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c < d4)
#pragma unroll 8
      for (int m = q; m < M; m += 4) {
        const float4 av = __ldg(reinterpret_cast<const float4*>(A + (long long)sidx[m] * d) + c);
        const float cm = coef[m];
        acc.x = fmaf(cm, av.x, acc.x);
        acc.y = fmaf(cm, av.y, acc.y);
        acc.z = fmaf(cm, av.z, acc.z);
        acc.w = fmaf(cm, av.w, acc.w);
      }
    if (q > 0) quarter[q - 1][t] = acc;
    __syncthreads();
    if (q == 0 && c < d4) {
      for (int r = 0; r < 3; ++r) {
        const float4 o = quarter[r][t];
        acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
      }
      reinterpret_cast<float4*>(g)[c] = acc;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kLinThreadsV) k_linear_grad_v(int kind, const float* __restrict__ A,
                                                                const float* __restrict__ b, int S,
                                                                const int* __restrict__ idx_in, int M,
                                                                uint2 key, unsigned long long k,
                                                                const float* __restrict__ xhat,
                                                                float* __restrict__ g, long long d) {
  pdl_wait();                               // PDL launch: wait for the predecessor grid
  pdl_trigger();
  __shared__ LinSmem sm;
  linear_grad_v_body(sm, kind, A, b, S, idx_in, M, key, k, xhat, g, d);
}

// Config 1's replay in ONE launch (latency-bound): one CTA walks the schedule in
// order; at event t it first computes the lsq / logreg gradients whose stale read point is X_t
// (the reads due before event t) into their slots, then -- after a CTA barrier -- applies
// event t (the pair average and update, Alg. 1 steps 4-6); a barrier orders event t's writes
// before event t + 1's reads.  The same code as the standalone gradient and event kernels, so
// the results are identical to the per-event launches it replaces.
__global__ void __launch_bounds__(kLinThreadsV) k_lin_replay(LinReplayParams p) {
  __shared__ LinSmem sm;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int e = 0; e < p.nops; ++e) {
    const LinEventOp op = p.ops[e];
    for (int r = op.r0; r < op.r1; ++r) {
      const LinRead rd = p.reads[r];
      linear_grad_v_body(sm, p.kind, p.A, p.b, p.S, rd.idx, p.M, p.key, rd.k, rd.x, rd.g, p.d);
    }
    __syncthreads();
    if (op.xi) {
      float4* xi4 = reinterpret_cast<float4*>(op.xi);
      float4* xj4 = reinterpret_cast<float4*>(op.xj);
      const float4* g4 = reinterpret_cast<const float4*>(op.g);
      for (long long c = threadIdx.x; c < p.n4; c += blockDim.x) {
        float4 a = __ldcg(xi4 + c), bb = op.xj ? __ldcg(xj4 + c) : z;
        const float4 gg = op.g ? __ldcg(g4 + c) : z;
        const uint32_t c0 = (uint32_t)(c * 4);
        if (op.xj) {
          if (!op.g) update4<true, kGradNone>(a, bb, gg, z, c0, p.d, p.gamma, QuadParams{}, 0u);
          else if (op.ff) update4<true, kGradExternal, true>(a, bb, gg, z, c0, p.d, p.gamma, QuadParams{}, 0u);
          else update4<true, kGradExternal>(a, bb, gg, z, c0, p.d, p.gamma, QuadParams{}, 0u);
          __stcg(xj4 + c, bb);
        } else if (op.g) {
          update4<false, kGradExternal>(a, bb, gg, z, c0, p.d, p.gamma, QuadParams{}, 0u);
        }
        __stcg(xi4 + c, a);
      }
    }
    __syncthreads();
  }
}

__global__ void k_copy(float4* __restrict__ dst, const float4* __restrict__ src, long long n4) {
  pdl_wait();                               // PDL launch: wait for the predecessor grid
  pdl_trigger();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x)
    st_cg4(dst + i, ld_cg4(src + i));
}

// pseudo-random values in [-1, 1) (diagnostic operands: GEMM timing)
__global__ void k_fill_hash(float* __restrict__ x, long long n, uint32_t seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    x[i] = __uint_as_float(0x40000000u | (lowbias32((uint32_t)i ^ seed) >> 9)) - 3.0f;
}

// App. A compensation (footnote at P:1265-1268): out = fl(x - fl(gamma gp))
__global__ void k_comp_row(const float4* __restrict__ x, const float4* __restrict__ gp, float gamma,
                           float4* __restrict__ out, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 a = ld_cg4(x + i), g = ld_cg4(gp + i);
    st_cg4(out + i, make_float4(__fsub_rn(a.x, __fmul_rn(gamma, g.x)), __fsub_rn(a.y, __fmul_rn(gamma, g.y)),
                                __fsub_rn(a.z, __fmul_rn(gamma, g.z)), __fsub_rn(a.w, __fmul_rn(gamma, g.w))));
  }
}

// ------------------------------------------------------ consensus output ---
// sum[c] = sum over rows of X[r][c] in fp64 (reading: fp64 accumulation)
__global__ void k_consensus_sum(const float* __restrict__ X, int n_rows, long long d_pad,
                                long long d, double* __restrict__ sum) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < d;
       c += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < n_rows; ++r) s += (double)__ldcg(X + (long long)r * d_pad + c);
    sum[c] = s;
  }
}

// float4 form of k_consensus_sum for R <= 8 local rows (same fp64 row order)
template <int R>
__global__ void __launch_bounds__(256) k_consensus_sum4(const float4* __restrict__ X, long long d_pad4, long long d4,
                                                        double* __restrict__ sum) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < d4;
       c += (long long)gridDim.x * blockDim.x) {
    float4 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = __ldcg(X + (long long)r * d_pad4 + c);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      s0 += (double)v[r].x; s1 += (double)v[r].y; s2 += (double)v[r].z; s3 += (double)v[r].w;
    }
    double2* o = reinterpret_cast<double2*>(sum + 4 * c);
    o[0] = make_double2(s0, s1);
    o[1] = make_double2(s2, s3);
  }
}

// x_bar = fl32(sum / n); a non-finite sum means some worker's model diverged
// (S:289): latch ADPSGD_E_DIVERGED for the next adpsgd_sync
__global__ void k_consensus_finalize(const double* __restrict__ sum, int n, long long d,
                                     float* __restrict__ out, unsigned int* err) {
  bool bad = false;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < d;
       c += (long long)gridDim.x * blockDim.x) {
    const double v = sum[c];
    bad |= !isfinite(v);
    out[c] = __double2float_rn(__ddiv_rn(v, (double)n));
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicCAS(err, 0u, 6u);
}

// World 1: x_bar = fl32(fp64 sum / n) and, when acc != null, M_k's sum of
// (mean - x)^2 in ONE read of the rows (the second loop re-reads the same lines
// from L2).  x_bar is bitwise the sum + finalize result (same fp64 row order).
__global__ void k_consensus_fused(const float* __restrict__ X, int n_rows, long long d_pad, long long d, int n,
                                  float* __restrict__ out, double* acc, unsigned int* err) {
  double part = 0.0;
  bool bad = false;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < d;
       c += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < n_rows; ++r) s += (double)__ldcg(X + (long long)r * d_pad + c);
    bad |= !isfinite(s);
    const double mean = __ddiv_rn(s, (double)n);
    out[c] = __double2float_rn(mean);
    if (acc)
      for (int r = 0; r < n_rows; ++r) {
        const double e = mean - (double)__ldcg(X + (long long)r * d_pad + c);
        part += e * e;
      }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicCAS(err, 0u, 6u);
  if (!acc) return;
#pragma unroll
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) atomicAdd(acc, v);
  }
}

// float4 form for R <= 8 local rows (d % 4 == 0): the R rows' values stay in
// registers for the M_k pass, and each coordinate's fp64 sum is accumulated in the
// same row order as k_consensus_fused, so x-bar is bitwise the same.
template <int R>
__global__ void __launch_bounds__(256) k_consensus_fused4(const float4* __restrict__ X, long long d_pad4, long long d4,
                                                          int n, float4* __restrict__ out, double* acc,
                                                          unsigned int* err) {
  double part = 0.0;
  bool bad = false;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < d4;
       c += (long long)gridDim.x * blockDim.x) {
    float4 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = __ldcg(X + (long long)r * d_pad4 + c);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      s0 += (double)v[r].x; s1 += (double)v[r].y; s2 += (double)v[r].z; s3 += (double)v[r].w;
    }
    bad |= !isfinite(s0) || !isfinite(s1) || !isfinite(s2) || !isfinite(s3);
    const double m0 = __ddiv_rn(s0, (double)n), m1 = __ddiv_rn(s1, (double)n);
    const double m2 = __ddiv_rn(s2, (double)n), m3 = __ddiv_rn(s3, (double)n);
    out[c] = make_float4(__double2float_rn(m0), __double2float_rn(m1), __double2float_rn(m2), __double2float_rn(m3));
    if (acc)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double e0 = m0 - (double)v[r].x, e1 = m1 - (double)v[r].y;
        const double e2 = m2 - (double)v[r].z, e3 = m3 - (double)v[r].w;
        part += e0 * e0 + e1 * e1 + e2 * e2 + e3 * e3;
      }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicCAS(err, 0u, 6u);
  if (!acc) return;
#pragma unroll
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) atomicAdd(acc, v);
  }
}

// M_k partial: sum over local rows and coordinates of (mean - x)^2, fp64
__global__ void k_consensus_mk(const float* __restrict__ X, int n_rows, long long d_pad, long long d,
                               const double* __restrict__ sum, int n, double* acc) {
  double part = 0.0;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < d;
       c += (long long)gridDim.x * blockDim.x) {
    const double mean = sum[c] / (double)n;
    for (int r = 0; r < n_rows; ++r) {
      const double e = mean - (double)__ldcg(X + (long long)r * d_pad + c);
      part += e * e;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) atomicAdd(acc, v);
  }
}

// ---------------------------------------------------- AllReduce-SGD baseline
// gsum[c] = sum over this rank's workers w of g_c(x; event k_base + w_global)
__global__ void __launch_bounds__(kThreads) k_ar_grad_sum(const float* __restrict__ x,
                                                          float* __restrict__ gsum, long long d,
                                                          long long n4, QuadParams q,
                                                          unsigned long long k_base, int n_local,
                                                          const int* __restrict__ local_ids) {
  pdl_wait();                               // PDL launch: wait for the predecessor grid
  pdl_trigger();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 xv4 = ld_cg4(reinterpret_cast<const float4*>(x) + i);
    const float xv[4] = {xv4.x, xv4.y, xv4.z, xv4.w};
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int w = 0; w < n_local; ++w) {
      const uint32_t kk = quad_event_key_h(q.noise_key, k_base + (unsigned long long)local_ids[w]);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t c = (uint32_t)(i * 4 + e);
        if ((long long)c < d) acc[e] = __fadd_rn(acc[e], quad_grad(xv[e], c, q.data_key, kk, q.Mf, q.s));
      }
    }
    st_cg4(reinterpret_cast<float4*>(gsum) + i, make_float4(acc[0], acc[1], acc[2], acc[3]));
  }
}

// x <- fl(x - fl(gamma * fl(gsum / n)))   (reading R12: mean of the gradients)
__global__ void __launch_bounds__(kThreads) k_ar_update(float* __restrict__ x,
                                                        const float* __restrict__ gsum, float gamma,
                                                        int n, long long d, long long n4) {
  pdl_wait();                               // PDL launch: wait for the predecessor grid
  pdl_trigger();
  const float nf = (float)n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 xv = ld_cg4(reinterpret_cast<const float4*>(x) + i);
    const float4 gv = ld_cg4(reinterpret_cast<const float4*>(gsum) + i);
    float xa[4] = {xv.x, xv.y, xv.z, xv.w};
    const float ga[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if ((long long)(i * 4 + e) < d) xa[e] = __fsub_rn(xa[e], __fmul_rn(gamma, __fdiv_rn(ga[e], nf)));
    st_cg4(reinterpret_cast<float4*>(x) + i, make_float4(xa[0], xa[1], xa[2], xa[3]));
  }
}

// ------------------------------------------------------ D-PSGD baseline ----
// One synchronous round for this rank's rows (reading R19):
//   acc = fl(w_self x_i); acc = fl(acc + fl(w_nb x_j)) for j in N(i) ascending;
//   x_i' = fl(acc - fl(gamma g_i(x_i)))   (quadratic gradient, event k_base + i)
// in[l*kDpMaxDeg + t] points at neighbour t's pre-round row (local or halo).
__global__ void __launch_bounds__(kThreads) k_dpsgd(const float* const* __restrict__ nbr, const int* __restrict__ deg,
                                                    const float* __restrict__ w_self, float w_nb,
                                                    const float* __restrict__ xin, float* __restrict__ xout,
                                                    long long d_pad, long long d, QuadParams q, int model,
                                                    float gamma, unsigned long long k_base,
                                                    const int* __restrict__ local_ids) {
  pdl_wait();                               // PDL launch: wait for the predecessor grid
  pdl_trigger();
  __shared__ const float4* snb[kDpMaxDeg];
  const int l = blockIdx.y;
  const float4* xi = reinterpret_cast<const float4*>(xin + (long long)l * d_pad);
  float4* xo = reinterpret_cast<float4*>(xout + (long long)l * d_pad);
  const int nd = deg[l];
  const float ws = w_self[l];
  const uint32_t kk = quad_event_key_h(q.noise_key, k_base + (unsigned long long)local_ids[l]);
  if (threadIdx.x < nd) snb[threadIdx.x] = reinterpret_cast<const float4*>(nbr[l * kDpMaxDeg + threadIdx.x]);
  __syncthreads();
  const long long n4 = d_pad / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 x4 = ld_cg4(xi + i);
    const float xv[4] = {x4.x, x4.y, x4.z, x4.w};
    float acc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[e] = __fmul_rn(ws, xv[e]);
    for (int t = 0; t < nd; ++t) {
      const float4 y4 = ld_cg4(snb[t] + i);
      const float yv[4] = {y4.x, y4.y, y4.z, y4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] = __fadd_rn(acc[e], __fmul_rn(w_nb, yv[e]));
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const long long c = i * 4 + e;
      if (model != 0 && c < d)
        acc[e] = __fsub_rn(acc[e], __fmul_rn(gamma, quad_grad(xv[e], (uint32_t)c, q.data_key, kk, q.Mf, q.s)));
      if (c >= d) acc[e] = 0.0f;
    }
    st_cg4(xo + i, make_float4(acc[0], acc[1], acc[2], acc[3]));
  }
}

// straggler / emulated-compute delay: one thread spins on %globaltimer
__global__ void k_delay(unsigned long long ns) {
  const unsigned long long t0 = globaltimer();
  while (globaltimer() - t0 < ns) __nanosleep(1000);
}

__global__ void k_init_rows(float* X, int n_rows, long long d_pad, long long d, const float* x0) {
  const long long tot = (long long)n_rows * d_pad;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot;
       t += (long long)gridDim.x * blockDim.x) {
    const long long c = t % d_pad;
    X[t] = (c < d && x0) ? x0[c] : 0.0f;
  }
}

__global__ void k_step_commit(GlobalCtl* gctl0, WorkerCtl* ctl_i, LogEntry* log, long long log_cap,
                              long long k, int i, int j, unsigned int flags, int grad) {
  pdl_wait();                               // PDL launch: wait for the predecessor grid
  pdl_trigger();
  atomicMax(&gctl0->ticket, (unsigned long long)(k + 1));
  atomicMax(&gctl0->committed, (unsigned long long)(k + 1));
  if (grad) atomicAdd(&ctl_i->updates, 1ull);
  if (j >= 0) atomicAdd(&ctl_i->gossips, 1ull);
  if (log) {
    const unsigned long long t = globaltimer();
    LogEntry* e = log + (k % log_cap);
    e->k = k; e->i = i; e->j = j; e->tau = 0; e->flags = flags; e->t0 = t; e->t1 = t;
  }
}

__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }

// Super-learner (reading R22), run by the group leader: take the super-learner's
// lock (system-scope try-lock, possibly on a peer GPU), then the ticket k
// (rank 0's counter) while holding it; k goes to *kout for the group broadcast.
__global__ void k_super_lock(unsigned int* lock, unsigned long long* ticket, unsigned long long* kout,
                             unsigned int* err, unsigned long long watchdog_ns) {
  const unsigned long long t0 = globaltimer();
  while (atomicCAS_system(lock, 0u, 1u) != 0u) {
    if (globaltimer() - t0 > watchdog_ns) { atomicCAS(err, 0u, 7u); *kout = ~0ull; return; }
    __nanosleep(500);
  }
  __threadfence_system();
  *kout = atomicAdd_system(ticket, 1ull);
}

// ... and after every replica of the event is written (group barrier): log
// {k, i, j, 0, flags}, counters, release the lock.
__global__ void k_super_commit(LogEntry* log, long long log_cap, const unsigned long long* kin, int i, int j,
                               unsigned int flags, WorkerCtl* ctl_i, unsigned long long* committed,
                               unsigned int* lock) {
  const unsigned long long k = *kin;
  if (k == ~0ull) return;                        // lock timed out (error latched)
  const unsigned long long t = globaltimer();
  LogEntry* e = log + (long long)(k % (unsigned long long)log_cap);
  e->k = (long long)k; e->i = i; e->j = j; e->tau = 0; e->flags = flags; e->t0 = t; e->t1 = t;
  if (!(flags & 1u)) atomicAdd_system(&ctl_i->updates, 1ull);
  if (j >= 0) atomicAdd_system(&ctl_i->gossips, 1ull);
  atomicAdd_system(committed, 1ull);
  __threadfence_system();
  atomicExch_system(lock, 0u);
}

template <bool P, int G>
cudaError_t ev(float* xi, float* xj, const float* g, const float* xh, long long d, long long n4,
               float gamma, const QuadParams& q, uint32_t kk, cudaStream_t s, const unsigned long long* guard) {
  // programmatic dependent launch: the event's launch and prologue overlap its predecessor (in
  // the MLP chain, GEMM2) and it waits for that grid at griddepcontrol.wait
  return launch_pdl(k_event<P, G>, dim3(stream_grid(n4)), dim3(kThreads), 0, s, xi, xj, g, xh, d, n4, gamma, q, kk,
                    guard);
}

template <int G>
cudaError_t ev_ff(float* xi, float* xj, const float* g, const float* xh, long long d, long long n4,
                  float gamma, const QuadParams& q, uint32_t kk, cudaStream_t s, const unsigned long long* guard) {
  return launch_pdl(k_event<true, G, true>, dim3(stream_grid(n4)), dim3(kThreads), 0, s, xi, xj, g, xh, d, n4, gamma,
                    q, kk, guard);
}

}  // namespace

// k: random-draw key of the gradient (the event's k, or read_key for App. A events)
cudaError_t launch_event(float* xi, float* xj, const float* g, const float* xhat, long long d,
                         long long n4, float gamma, const QuadParams& q, unsigned long long k,
                         int grad_mode, cudaStream_t s, const unsigned long long* guard) {
  const uint32_t kk = quad_event_key_h(q.noise_key, k);
  const bool pair = xj != nullptr;
  if ((grad_mode & kModeFlushFirst) && pair) {     // App. A order; a local flush is Alg. 1's local step
    switch (grad_mode & 0xf) {
      case kGradNone: return ev<true, kGradNone>(xi, xj, g, xhat, d, n4, gamma, q, kk, s, guard);
      case kGradExternal: return ev_ff<kGradExternal>(xi, xj, g, xhat, d, n4, gamma, q, kk, s, guard);
      case kGradQuadInline: return ev_ff<kGradQuadInline>(xi, xj, g, xhat, d, n4, gamma, q, kk, s, guard);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (grad_mode & 0xf) {
    case kGradNone:
      return pair ? ev<true, kGradNone>(xi, xj, g, xhat, d, n4, gamma, q, kk, s, guard)
                  : cudaSuccess;
    case kGradExternal:
      return pair ? ev<true, kGradExternal>(xi, xj, g, xhat, d, n4, gamma, q, kk, s, guard)
                  : ev<false, kGradExternal>(xi, xj, g, xhat, d, n4, gamma, q, kk, s, guard);
    case kGradQuadInline:
      return pair ? ev<true, kGradQuadInline>(xi, xj, g, xhat, d, n4, gamma, q, kk, s, guard)
                  : ev<false, kGradQuadInline>(xi, xj, g, xhat, d, n4, gamma, q, kk, s, guard);
    case kGradQuadSnapshot:
      return pair ? ev<true, kGradQuadSnapshot>(xi, xj, g, xhat, d, n4, gamma, q, kk, s, guard)
                  : ev<false, kGradQuadSnapshot>(xi, xj, g, xhat, d, n4, gamma, q, kk, s, guard);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_quad_grad(const float* xhat, float* g, long long d, long long n4,
                             const QuadParams& q, unsigned long long k, cudaStream_t s) {
  return launch_pdl(k_quad_grad, dim3(stream_grid(n4)), dim3(kThreads), 0, s, xhat, g, d, n4, q,
                    quad_event_key_h(q.noise_key, k));
}

cudaError_t launch_linear_grad(int kind, const float* A, const float* b, int S, const int* idx,
                               int M, uint2 batch_key, unsigned long long k, const float* xhat,
                               float* g, long long d, cudaStream_t s) {
  if (M > kMaxM) return cudaErrorInvalidValue;
  if (d % 4 == 0)
    return launch_pdl(k_linear_grad_v, dim3(1), dim3(kLinThreadsV), 0, s, kind, A, b, S, idx, M, batch_key, k, xhat, g,
                      d);
  return launch_pdl(k_linear_grad, dim3(1), dim3(kLinThreads), 0, s, kind, A, b, S, idx, M, batch_key, k, xhat, g, d);
}

cudaError_t launch_lin_replay(const LinReplayParams& p, cudaStream_t s) {
  if (p.M > kMaxM || p.d % 4) return cudaErrorInvalidValue;
  if (p.nops == 0) return cudaSuccess;
  k_lin_replay<<<1, kLinThreadsV, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_copy(float* dst, const float* src, long long n4, cudaStream_t s) {
  return launch_pdl(k_copy, dim3(stream_grid(n4)), dim3(kThreads), 0, s, reinterpret_cast<float4*>(dst),
                    reinterpret_cast<const float4*>(src), n4);
}

cudaError_t launch_fill_hash(float* x, long long n, uint32_t seed, cudaStream_t s) {
  k_fill_hash<<<4 * sm_count(), 256, 0, s>>>(x, n, seed);
  return cudaGetLastError();
}

cudaError_t launch_comp_row(const float* x, const float* gp, float gamma, float* out, long long n4, cudaStream_t s) {
  k_comp_row<<<stream_grid(n4), kThreads, 0, s>>>(reinterpret_cast<const float4*>(x),
                                                  reinterpret_cast<const float4*>(gp), gamma,
                                                  reinterpret_cast<float4*>(out), n4);
  return cudaGetLastError();
}

cudaError_t launch_consensus_sum(const float* X, int n_rows, long long d_pad, long long d,
                                 double* sum, cudaStream_t s) {
  if (d % 4 == 0 && d_pad % 4 == 0 && n_rows >= 1 && n_rows <= 8) {
    const float4* X4 = reinterpret_cast<const float4*>(X);
    const int g = 4 * sm_count();
    switch (n_rows) {
#define ADPSGD_CS4(R) case R: k_consensus_sum4<R><<<g, 256, 0, s>>>(X4, d_pad / 4, d / 4, sum); break;
      ADPSGD_CS4(1) ADPSGD_CS4(2) ADPSGD_CS4(3) ADPSGD_CS4(4) ADPSGD_CS4(5) ADPSGD_CS4(6) ADPSGD_CS4(7) ADPSGD_CS4(8)
#undef ADPSGD_CS4
    }
    return cudaGetLastError();
  }
  k_consensus_sum<<<4 * sm_count(), 256, 0, s>>>(X, n_rows, d_pad, d, sum);
  return cudaGetLastError();
}

cudaError_t launch_consensus_finalize(const double* sum, int n, long long d, float* out, unsigned int* err,
                                      cudaStream_t s) {
  k_consensus_finalize<<<4 * sm_count(), 256, 0, s>>>(sum, n, d, out, err);
  return cudaGetLastError();
}

cudaError_t launch_consensus_fused(const float* X, int n_rows, long long d_pad, long long d, int n, float* out,
                                   double* acc, unsigned int* err, cudaStream_t s) {
  // float4 form: the caller's out (any d floats, ABI) must be 16-byte aligned for it
  if (d % 4 == 0 && d_pad % 4 == 0 && n_rows >= 1 && n_rows <= 8 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    const float4* X4 = reinterpret_cast<const float4*>(X);
    float4* o4 = reinterpret_cast<float4*>(out);
    const int g = 4 * sm_count();
    switch (n_rows) {
#define ADPSGD_CF4(R) case R: k_consensus_fused4<R><<<g, 256, 0, s>>>(X4, d_pad / 4, d / 4, n, o4, acc, err); break;
      ADPSGD_CF4(1) ADPSGD_CF4(2) ADPSGD_CF4(3) ADPSGD_CF4(4) ADPSGD_CF4(5) ADPSGD_CF4(6) ADPSGD_CF4(7) ADPSGD_CF4(8)
#undef ADPSGD_CF4
    }
    return cudaGetLastError();
  }
  k_consensus_fused<<<4 * sm_count(), 256, 0, s>>>(X, n_rows, d_pad, d, n, out, acc, err);
  return cudaGetLastError();
}

cudaError_t launch_consensus_mk(const float* X, int n_rows, long long d_pad, long long d,
                                const double* sum, int n, double* acc, cudaStream_t s) {
  k_consensus_mk<<<4 * sm_count(), 256, 0, s>>>(X, n_rows, d_pad, d, sum, n, acc);
  return cudaGetLastError();
}

cudaError_t launch_ar_grad_sum(const float* x, float* gsum, long long d, long long n4,
                               const QuadParams& q, unsigned long long k_base, int n_local,
                               const int* local_ids, cudaStream_t s) {
  return launch_pdl(k_ar_grad_sum, dim3(stream_grid(n4)), dim3(kThreads), 0, s, x, gsum, d, n4, q, k_base, n_local,
                    local_ids);
}

cudaError_t launch_ar_update(float* x, const float* gsum, float gamma, int n, long long d,
                             long long n4, cudaStream_t s) {
  return launch_pdl(k_ar_update, dim3(stream_grid(n4)), dim3(kThreads), 0, s, x, gsum, gamma, n, d, n4);
}

cudaError_t launch_step_commit(GlobalCtl* gctl0, WorkerCtl* ctl_i, LogEntry* log, long long log_cap,
                               long long k, int i, int j, unsigned int flags, int grad,
                               cudaStream_t s) {
  return launch_pdl(k_step_commit, dim3(1), dim3(1), 0, s, gctl0, ctl_i, log, log_cap, k, i, j, flags, grad);
}

cudaError_t launch_super_lock(unsigned int* lock, unsigned long long* ticket, unsigned long long* kout,
                              unsigned int* err, unsigned long long watchdog_ns, cudaStream_t s) {
  k_super_lock<<<1, 1, 0, s>>>(lock, ticket, kout, err, watchdog_ns);
  return cudaGetLastError();
}

cudaError_t launch_super_commit(LogEntry* log, long long log_cap, const unsigned long long* kin, int i, int j,
                                unsigned int flags, WorkerCtl* ctl_i, unsigned long long* committed,
                                unsigned int* lock, cudaStream_t s) {
  k_super_commit<<<1, 1, 0, s>>>(log, log_cap, kin, i, j, flags, ctl_i, committed, lock);
  return cudaGetLastError();
}

cudaError_t launch_set_u64(unsigned long long* p, unsigned long long v, cudaStream_t s) {
  k_set_u64<<<1, 1, 0, s>>>(p, v);
  return cudaGetLastError();
}

cudaError_t launch_dpsgd(const float* const* nbr, const int* deg, const float* w_self, float w_nb, const float* xin,
                         float* xout, int n_local, long long d_pad, long long d, const QuadParams& q, int model,
                         float gamma, unsigned long long k_base, const int* local_ids, cudaStream_t s) {
  // all rows of the round in one launch: ~2 waves of 512-thread CTAs over the GPU
  const int bx = (int)std::min<long long>((d_pad / 4 + kThreads - 1) / kThreads,
                                          std::max(1LL, 4LL * sm_count() / n_local));
  return launch_pdl(k_dpsgd, dim3(bx, n_local), dim3(kThreads), 0, s, nbr, deg, w_self, w_nb, xin, xout, d_pad, d, q,
                    model, gamma, k_base, local_ids);
}

cudaError_t launch_delay(unsigned long long ns, cudaStream_t s) {
  k_delay<<<1, 1, 0, s>>>(ns);
  return cudaGetLastError();
}

cudaError_t launch_init_rows(float* X, int n_rows, long long d_pad, long long d, const float* x0,
                             cudaStream_t s) {
  k_init_rows<<<4 * sm_count(), 256, 0, s>>>(X, n_rows, d_pad, d, x0);
  return cudaGetLastError();
}

// one kernel of this translation unit (module), for preload_modules()
const void* kernels_module_anchor() { return (const void*)k_set_u64; }

}  // namespace adp
