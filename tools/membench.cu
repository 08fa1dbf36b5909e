// membench.cu -- HBM streaming microbenchmarks that shape the fused gossip pass.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/membench tools/membench.cu
// Patterns on d = 25.6M fp32 rows: copy (1R1W), pair average (2R2W).
#include <cstdio>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int U, int MODE>   // MODE 0 ldcg/stcg, 1 default ld/st, 2 ld + st.cs (evict-first)
__global__ void avg_slice(float4* xi, float4* xj, long long n4, int pair) {
  const long long per = (n4 + gridDim.x - 1) / gridDim.x;
  const long long lo = blockIdx.x * per, hi = min(lo + per, n4);
  for (long long base = lo + threadIdx.x; base < hi; base += (long long)blockDim.x * U) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long i = base + (long long)u * blockDim.x;
      if (i < hi) {
        if (pair) b[u] = MODE == 0 ? __ldcg(xj + i) : xj[i];
        a[u] = MODE == 0 ? __ldcg(xi + i) : xi[i];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long i = base + (long long)u * blockDim.x;
      if (i < hi) {
        float4 m = a[u];
        if (pair) { m.x = (a[u].x + b[u].x) * 0.5f; m.y = (a[u].y + b[u].y) * 0.5f; m.z = (a[u].z + b[u].z) * 0.5f; m.w = (a[u].w + b[u].w) * 0.5f; }
        else { m.x += 1.f; }
        if (MODE == 2) { if (pair) __stcs(xj + i, m); __stcs(xi + i, m); }
        else if (MODE == 0) { if (pair) __stcg(xj + i, m); __stcg(xi + i, m); }
        else { if (pair) xj[i] = m; xi[i] = m; }
      }
    }
  }
}

template <int U>
__global__ void avg_stride(float4* xi, float4* xj, long long n4, int pair) {
  const long long T = (long long)gridDim.x * blockDim.x;
  for (long long base = blockIdx.x * (long long)blockDim.x + threadIdx.x; base < n4; base += T * U) {
    float4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long long i = base + u * T; if (i < n4) { if (pair) b[u] = __ldcg(xj + i); a[u] = __ldcg(xi + i); } }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      long long i = base + u * T;
      if (i < n4) {
        float4 m = a[u];
        if (pair) { m.x = (a[u].x + b[u].x) * 0.5f; m.y = (a[u].y + b[u].y) * 0.5f; m.z = (a[u].z + b[u].z) * 0.5f; m.w = (a[u].w + b[u].w) * 0.5f; } else m.x += 1.f;
        if (pair) __stcg(xj + i, m);
        __stcg(xi + i, m);
      }
    }
  }
}

// bulk-copy loads (+ STG or bulk-copy stores)
template <int TILE4, int S, bool BULKST, bool IL = false>
__global__ void avg_tma(float4* xi, float4* xj, long long n4, int pair) {
  extern __shared__ __align__(128) unsigned char sm[];
  float4* buf = (float4*)sm;
  uint64_t* bar = (uint64_t*)(sm + (size_t)S * 2 * TILE4 * 16);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long per = (n4 + gridDim.x - 1) / gridDim.x;
  const long long lo = IL ? 0 : blockIdx.x * per, hi = IL ? n4 : min(lo + per, n4);
  const long long tot_t = (n4 + TILE4 - 1) / TILE4;
  const long long nt = IL ? (tot_t > blockIdx.x ? (tot_t - blockIdx.x + gridDim.x - 1) / gridDim.x : 0)
                          : (hi - lo + TILE4 - 1) / TILE4;
  auto tbase = [&](long long t) { return IL ? (blockIdx.x + t * gridDim.x) * TILE4 : lo + t * TILE4; };
  auto issue = [&](long long t) {
    int s = t % S;
    long long base = tbase(t);
    uint32_t bytes = (uint32_t)min((long long)TILE4, hi - base) * 16;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(bar + s)), "r"(pair ? 2 * bytes : bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(smem_u32(buf + (size_t)s * 2 * TILE4)), "l"(xi + base), "r"(bytes), "r"(smem_u32(bar + s)) : "memory");
    if (pair) asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(smem_u32(buf + (size_t)s * 2 * TILE4 + TILE4)), "l"(xj + base), "r"(bytes), "r"(smem_u32(bar + s)) : "memory");
  };
  if (threadIdx.x == 0) for (long long t = 0; t < nt && t < S; ++t) issue(t);
  for (long long t = 0; t < nt; ++t) {
    int s = t % S;
    uint32_t ph = (t / S) & 1, ok;
    do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(smem_u32(bar + s)), "r"(ph) : "memory"); } while (!ok);
    float4* sa = buf + (size_t)s * 2 * TILE4;
    float4* sb = sa + TILE4;
    long long base = tbase(t);
    long long cnt = min((long long)TILE4, hi - base);
    for (int off = threadIdx.x; off < cnt; off += blockDim.x) {
      float4 a = sa[off], m = a;
      if (pair) { float4 b = sb[off]; m.x = (a.x + b.x) * 0.5f; m.y = (a.y + b.y) * 0.5f; m.z = (a.z + b.z) * 0.5f; m.w = (a.w + b.w) * 0.5f; } else m.x += 1.f;
      if (BULKST) { sa[off] = m; if (pair) sb[off] = m; }
      else { if (pair) __stcg(xj + base + off, m); __stcg(xi + base + off, m); }
    }
    if (BULKST) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t bytes = (uint32_t)cnt * 16;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(xi + base), "r"(smem_u32(sa)), "r"(bytes) : "memory");
        if (pair) asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(xj + base), "r"(smem_u32(sb)), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // smem reusable
      }
      __syncthreads();
    } else {
      __syncthreads();
    }
    if (threadIdx.x == 0 && t + S < nt) issue(t + S);
  }
  if (BULKST && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// warp-specialised variant: warp 15 only issues the bulk copies (waiting on
// per-stage "empty" barriers the 15 consumer warps arrive on); consumers wait
// on "full", copy the stage to registers, release it, compute and store.  No
// CTA-wide barrier in the loop.  Interleaved tiles across CTAs (engine layout).
template <int TILE4, int S>
__global__ void __launch_bounds__(512) avg_ws(float4* xi, float4* xj, long long n4, int pair) {
  constexpr int kCons = 480, kPer = TILE4 / kCons;
  static_assert(TILE4 % kCons == 0, "tile must be a multiple of the consumer count");
  extern __shared__ __align__(128) unsigned char sm[];
  float4* buf = (float4*)sm;
  uint64_t* full = (uint64_t*)(sm + (size_t)S * 2 * TILE4 * 16);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(empty + s)), "r"(kCons / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long tot_t = (n4 + TILE4 - 1) / TILE4;
  const long long nt = tot_t > blockIdx.x ? (tot_t - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto wait = [](uint64_t* b, uint32_t ph) {
    uint32_t ok;
    do { asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory"); } while (!ok);
  };
  if (threadIdx.x >= kCons) {                              // producer warp
    if (threadIdx.x == kCons) {
      for (long long t = 0; t < nt; ++t) {
        const int s = t % S;
        if (t >= S) wait(empty + s, ((t / S) - 1) & 1);
        const long long base = (blockIdx.x + t * gridDim.x) * TILE4;
        const uint32_t bytes = (uint32_t)min((long long)TILE4, n4 - base) * 16;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(full + s)), "r"(pair ? 2 * bytes : bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(smem_u32(buf + (size_t)s * 2 * TILE4)), "l"(xi + base), "r"(bytes), "r"(smem_u32(full + s)) : "memory");
        if (pair) asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(smem_u32(buf + (size_t)s * 2 * TILE4 + TILE4)), "l"(xj + base), "r"(bytes), "r"(smem_u32(full + s)) : "memory");
      }
    }
    return;
  }
  for (long long t = 0; t < nt; ++t) {
    const int s = t % S;
    wait(full + s, (t / S) & 1);
    const float4* sa = buf + (size_t)s * 2 * TILE4;
    const float4* sb = sa + TILE4;
    const long long base = (blockIdx.x + t * gridDim.x) * TILE4;
    float4 a[kPer], b[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) { a[u] = sa[u * kCons + threadIdx.x]; if (pair) b[u] = sb[u * kCons + threadIdx.x]; }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(smem_u32(empty + s)) : "memory");
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const long long i = base + u * kCons + threadIdx.x;
      if (i < n4) {
        float4 m = a[u];
        if (pair) { m.x = (a[u].x + b[u].x) * 0.5f; m.y = (a[u].y + b[u].y) * 0.5f; m.z = (a[u].z + b[u].z) * 0.5f; m.w = (a[u].w + b[u].w) * 0.5f; __stcg(xj + i, m); } else m.x += 1.f;
        __stcg(xi + i, m);
      }
    }
  }
}

int sms;
#define RUN2(name, launch, bytes) { float ms = timeit([&] { launch; }, it); CK(cudaGetLastError()); printf("%-48s %8.1f us %7.0f GB/s\n", name, ms * 1e3, (bytes) / (ms / 1e3) / 1e9); }

template <typename F>
float timeit(F f, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f(); f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / iters;
}

// remote-row microbenchmarks: x_j on GPU 1, kernel on GPU 0 (NVLink P2P)
template <int U>
__global__ void peer_read(const float4* src, float4* dst, long long n4) {   // remote -> local copy
  const long long T = (long long)gridDim.x * blockDim.x;
  for (long long base = blockIdx.x * (long long)blockDim.x + threadIdx.x; base < n4; base += T * U) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long long i = base + u * T; if (i < n4) v[u] = __ldcg(src + i); }
#pragma unroll
    for (int u = 0; u < U; ++u) { long long i = base + u * T; if (i < n4) __stcg(dst + i, v[u]); }
  }
}

int peer_main() {
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  if (ndev < 2) { printf("peer: need 2 GPUs\n"); return 0; }
  const long long d = 25600000, n4 = d / 4;
  float4 *xi, *xj, *buf;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&xj, d * 4)); CK(cudaMemset(xj, 0, d * 4));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&xi, d * 4)); CK(cudaMalloc(&buf, d * 4));
  CK(cudaMemset(xi, 0, d * 4));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int it = 20;
  printf("=== NVLink: x_j on GPU1, kernels on GPU0 (GB/s per direction over NVLink) ===\n");
  double bytes = 4.0 * d;
  RUN2("peer LDG remote->local copy U4 2/SM", (peer_read<4><<<sms * 2, 512>>>(xj, buf, n4)), bytes);
  RUN2("peer LDG remote->local copy U8 4/SM", (peer_read<8><<<sms * 4, 512>>>(xj, buf, n4)), bytes);
  RUN2("peer STG local->remote copy U4 2/SM", (peer_read<4><<<sms * 2, 512>>>(buf, xj, n4)), bytes);
  RUN2("cudaMemcpyPeer 1->0", (cudaMemcpyPeerAsync(buf, 0, xj, 1, d * 4)), bytes);
  RUN2("pair avg ldg/stg remote xj, stride U4 2/SM", (avg_stride<4><<<sms * 2, 512>>>(xi, xj, n4, 1)), bytes);
  RUN2("pair avg ldg/stg remote xj, stride U8 4/SM", (avg_stride<8><<<sms * 4, 512>>>(xi, xj, n4, 1)), bytes);
  {
    constexpr int T = 512, S = 4;
    size_t smem = (size_t)S * 2 * T * 16 + 64;
    cudaFuncSetAttribute(avg_tma<T, S, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(avg_tma<T, S, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    RUN2("pair avg IL tma T512 S4 + stg, 2/SM", (avg_tma<T, S, false, true><<<sms * 2, 512, smem>>>(xi, xj, n4, 1)), bytes);
    RUN2("pair avg IL tma T512 S4 + bulk st, 2/SM", (avg_tma<T, S, true, true><<<sms * 2, 512, smem>>>(xi, xj, n4, 1)), bytes);
  }
  // bidirectional: both GPUs push (or pull) 4d to/from each other at once
  float4 *yi, *ybuf;
  CK(cudaSetDevice(1));
  CK(cudaDeviceEnablePeerAccess(0, 0));
  CK(cudaMalloc(&yi, d * 4)); CK(cudaMalloc(&ybuf, d * 4));
  cudaStream_t s1; CK(cudaStreamCreate(&s1));
  CK(cudaSetDevice(0));
  cudaStream_t s0; CK(cudaStreamCreate(&s0));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) {
    auto both = [&] {
      if (mode == 0) {   // writes: GPU0 -> GPU1 buffer, GPU1 -> GPU0 buffer
        cudaSetDevice(0); peer_read<4><<<sms * 2, 512, 0, s0>>>(xi, ybuf, n4);
        cudaSetDevice(1); peer_read<4><<<sms * 2, 512, 0, s1>>>(yi, buf, n4);
      } else {           // reads: GPU0 pulls GPU1's row, GPU1 pulls GPU0's row
        cudaSetDevice(0); peer_read<4><<<sms * 2, 512, 0, s0>>>(yi, buf, n4);
        cudaSetDevice(1); peer_read<4><<<sms * 2, 512, 0, s1>>>(xi, ybuf, n4);
      }
      cudaSetDevice(0);
    };
    both(); cudaDeviceSynchronize(); cudaSetDevice(1); cudaDeviceSynchronize(); cudaSetDevice(0);
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < it; ++r) both();
    cudaDeviceSynchronize(); cudaSetDevice(1); cudaDeviceSynchronize(); cudaSetDevice(0);
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / it;
    printf("%-48s %8.1f us %7.0f GB/s per direction\n", mode == 0 ? "bidirectional push (both GPUs write peer)" :
           "bidirectional pull (both GPUs read peer)", s * 1e6, bytes / s / 1e9);
  }
  // symmetric cross-GPU pair events: GPU0 averages (xi, yi@GPU1) while GPU1 averages
  // (yi, xi@GPU0) -- the engine's all-cross pattern; per direction 8d per round
  // (4d of read responses + 4d of written averages)
  {
    constexpr int T = 1024, S = 3;
    size_t smem = (size_t)S * 2 * T * 16 + 64;
    for (int dev = 0; dev < 2; ++dev) {
      cudaSetDevice(dev);
      cudaFuncSetAttribute(avg_tma<T, S, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(avg_tma<T, S, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    cudaSetDevice(0);
    for (int kind = 0; kind < 3; ++kind) {
      auto both = [&] {
        for (int dev = 0; dev < 2; ++dev) {
          cudaSetDevice(dev);
          float4* a = dev == 0 ? xi : yi;      // local row
          float4* b = dev == 0 ? yi : xi;      // peer row
          cudaStream_t st = dev == 0 ? s0 : s1;
          if (kind == 0) avg_stride<4><<<sms * 2, 512, 0, st>>>(a, b, n4, 1);
          else if (kind == 1) avg_tma<T, S, false, true><<<sms * 2, 512, smem, st>>>(a, b, n4, 1);
          else avg_tma<T, S, true, true><<<sms * 2, 512, smem, st>>>(a, b, n4, 1);
        }
        cudaSetDevice(0);
      };
      both(); cudaDeviceSynchronize(); cudaSetDevice(1); cudaDeviceSynchronize(); cudaSetDevice(0);
      auto t0 = std::chrono::steady_clock::now();
      for (int r = 0; r < it; ++r) both();
      cudaDeviceSynchronize(); cudaSetDevice(1); cudaDeviceSynchronize(); cudaSetDevice(0);
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / it;
      const char* nm[3] = {"symmetric pair avg, ldg/stg stride U4 2/SM", "symmetric pair avg, tma T1024 S3 + stg",
                           "symmetric pair avg, tma T1024 S3 + bulk st"};
      printf("%-48s %8.1f us %7.0f GB/s per direction\n", nm[kind], s * 1e6, 2.0 * bytes / s / 1e9);
    }
  }
  return 0;
}

// G GPUs at once: GPU g pair-averages its row with GPU (g+1)'s row (reads it,
// writes the average back) -- every GPU both serves and drives NVLink traffic,
// per direction 8d per round per GPU (the engine's all-cross pattern at G GPUs)
int ring_main(int G) {
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  if (ndev < G) { printf("ring: need %d GPUs\n", G); return 0; }
  const long long d = 25600000, n4 = d / 4;
  constexpr int T = 1024, S = 3;
  size_t smem = (size_t)S * 2 * T * 16 + 64;
  std::vector<float4*> x(G);
  std::vector<cudaStream_t> st(G);
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < G; ++h) if (h != g) cudaDeviceEnablePeerAccess(h, 0);
    CK(cudaMalloc(&x[g], d * 4)); CK(cudaMemset(x[g], 0, d * 4));
    CK(cudaStreamCreate(&st[g]));
    cudaFuncSetAttribute(avg_tma<T, S, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int kind = 0; kind < 2; ++kind) {
    auto all = [&] {
      for (int g = 0; g < G; ++g) {
        cudaSetDevice(g);
        float4* b = x[(g + 1) % G];
        if (kind == 0) avg_stride<4><<<sms * 2, 512, 0, st[g]>>>(x[g], b, n4, 1);
        else avg_tma<T, S, false, true><<<sms * 2, 512, smem, st[g]>>>(x[g], b, n4, 1);
      }
    };
    auto sync = [&] { for (int g = 0; g < G; ++g) { cudaSetDevice(g); cudaDeviceSynchronize(); } };
    all(); sync();
    const int it = 20;
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < it; ++r) all();
    sync();
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / it;
    printf("ring of %d GPUs, pair avg with next GPU's row, %-22s %8.1f us %7.0f GB/s per GPU per direction\n", G,
           kind == 0 ? "ldg/stg stride U4" : "tma T1024 S3 + stg", s * 1e6, 8.0 * d / s / 1e9);
  }
  return 0;
}

// G GPUs at once, every GPU pair-averaging with ALL other GPUs concurrently
// (one stream and 1/(G-1) of the SMs per peer): the traffic pattern of the
// xor placement, where a GPU's cross events go to several peers
int mesh_main(int G) {
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  if (ndev < G || G < 3) { printf("mesh: need >= 3 GPUs\n"); return 0; }
  const long long d = 25600000, n4 = d / 4;
  constexpr int T = 1024, S = 3;
  size_t smem = (size_t)S * 2 * T * 16 + 64;
  std::vector<float4*> x(G), y(G);                      // x: row pulled by peers, y: this GPU's own rows
  std::vector<std::vector<cudaStream_t>> st(G, std::vector<cudaStream_t>(G));
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < G; ++h) if (h != g) cudaDeviceEnablePeerAccess(h, 0);
    CK(cudaMalloc(&x[g], d * 4)); CK(cudaMemset(x[g], 0, d * 4));
    CK(cudaMalloc(&y[g], d * 4 * (G - 1))); CK(cudaMemset(y[g], 0, d * 4 * (G - 1)));
    for (int h = 0; h < G; ++h) CK(cudaStreamCreate(&st[g][h]));
    cudaFuncSetAttribute(avg_tma<T, S, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long part = n4 / (G - 1);                  // each peer pair moves 1/(G-1) of a row
  auto all = [&] {
    for (int g = 0; g < G; ++g) {
      cudaSetDevice(g);
      int q = 0;
      for (int h = 0; h < G; ++h) {
        if (h == g) continue;
        avg_tma<T, S, false, true><<<2 * sms / (G - 1), 512, smem, st[g][h]>>>(y[g] + q * part, x[h] + q * part, part, 1);
        ++q;
      }
    }
  };
  auto sync = [&] { for (int g = 0; g < G; ++g) { cudaSetDevice(g); cudaDeviceSynchronize(); } };
  all(); sync();
  const int it = 20;
  auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < it; ++r) all();
  sync();
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / it;
  // per GPU per direction: its reads of peers' rows + its written averages, 8 bytes per pair element
  printf("mesh of %d GPUs, pair avg with every other GPU's row, tma T1024 S3 + stg %8.1f us %7.0f GB/s per GPU per direction\n",
         G, s * 1e6, 8.0 * (double)part * 4 * (G - 1) / s / 1e9);
  return 0;
}

// CTA-barrier TMA staging (the engine's variant 0) vs warp-specialised staging
int ws_main() {
  const long long d = 25600000, n4 = d / 4;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float4 *xi, *xj;
  CK(cudaMalloc(&xi, d * 4)); CK(cudaMalloc(&xj, d * 4));
  CK(cudaMemset(xi, 0, d * 4)); CK(cudaMemset(xj, 0, d * 4));
  const int it = 30;
  for (int pair = 0; pair <= 1; ++pair) {
    const double bytes = (pair ? 16.0 : 8.0) * d;
    printf("=== %s ===\n", pair ? "pair average 2R2W" : "local update 1R1W");
#define RUN3(name, launch) { float ms = timeit([&] { launch; }, it); CK(cudaGetLastError()); printf("%-48s %8.1f us %7.0f GB/s\n", name, ms * 1e3, bytes / (ms / 1e3) / 1e9); }
    {
      constexpr int T = 1536, S = 2;
      size_t smem = (size_t)S * 2 * T * 16 + 256;
      cudaFuncSetAttribute(avg_tma<T, S, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      RUN3("IL tma T1536 S2, CTA barrier (engine v0)", (avg_tma<T, S, false, true><<<sms * 2, 512, smem>>>(xi, xj, n4, pair)));
    }
    {
      constexpr int T = 1440, S = 2;
      size_t smem = (size_t)S * 2 * T * 16 + 256;
      cudaFuncSetAttribute(avg_ws<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      RUN3("IL warp-specialised T1440 S2", (avg_ws<T, S><<<sms * 2, 512, smem>>>(xi, xj, n4, pair)));
    }
    {
      constexpr int T = 960, S = 3;
      size_t smem = (size_t)S * 2 * T * 16 + 256;
      cudaFuncSetAttribute(avg_ws<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      RUN3("IL warp-specialised T960 S3", (avg_ws<T, S><<<sms * 2, 512, smem>>>(xi, xj, n4, pair)));
    }
    {
      constexpr int T = 480, S = 6;
      size_t smem = (size_t)S * 2 * T * 16 + 256;
      cudaFuncSetAttribute(avg_ws<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      RUN3("IL warp-specialised T480 S6", (avg_ws<T, S><<<sms * 2, 512, smem>>>(xi, xj, n4, pair)));
    }
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && !strcmp(argv[1], "ws")) return ws_main();
  if (argc > 2 && !strcmp(argv[1], "ring")) return ring_main(atoi(argv[2]));
  if (argc > 2 && !strcmp(argv[1], "mesh")) return mesh_main(atoi(argv[2]));
  if (argc > 1) return peer_main();
  const long long d = 25600000, n4 = d / 4;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float4 *xi, *xj;
  CK(cudaMalloc(&xi, d * 4)); CK(cudaMalloc(&xj, d * 4));
  CK(cudaMemset(xi, 0, d * 4)); CK(cudaMemset(xj, 0, d * 4));
  const int it = 30;
  for (int pair = 0; pair <= 1; ++pair) {
    double bytes = (pair ? 16.0 : 8.0) * d;
    printf("=== %s ===\n", pair ? "pair average 2R2W" : "local update 1R1W");
#define RUN(name, launch) { float ms = timeit([&] { launch; }, it); CK(cudaGetLastError()); printf("%-44s %8.1f us %7.0f GB/s\n", name, ms * 1e3, bytes / (ms / 1e3) / 1e9); }
    for (int cps = 1; cps <= 4; cps *= 2) {
      char nm[128];
      snprintf(nm, 128, "slice U4 ldcg 512thr x%d/SM", cps); RUN(nm, (avg_slice<4, 0><<<sms * cps, 512>>>(xi, xj, n4, pair)));
      snprintf(nm, 128, "slice U8 ldcg 256thr x%d/SM", cps * 2); RUN(nm, (avg_slice<8, 0><<<sms * cps * 2, 256>>>(xi, xj, n4, pair)));
      snprintf(nm, 128, "slice U4 default 512thr x%d/SM", cps); RUN(nm, (avg_slice<4, 1><<<sms * cps, 512>>>(xi, xj, n4, pair)));
      snprintf(nm, 128, "slice U4 st.cs 512thr x%d/SM", cps); RUN(nm, (avg_slice<4, 2><<<sms * cps, 512>>>(xi, xj, n4, pair)));
      snprintf(nm, 128, "stride U4 512thr x%d/SM", cps); RUN(nm, (avg_stride<4><<<sms * cps, 512>>>(xi, xj, n4, pair)));
    }
    {
      constexpr int T = 1024, S = 3;
      size_t smem = (size_t)S * 2 * T * 16 + 64;
      cudaFuncSetAttribute(avg_tma<T, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(avg_tma<T, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      RUN("tma ld T1024 S3 + stg, 2/SM", (avg_tma<T, S, false><<<sms * 2, 512, smem>>>(xi, xj, n4, pair)));
      RUN("tma ld T1024 S3 + bulk st, 2/SM", (avg_tma<T, S, true><<<sms * 2, 512, smem>>>(xi, xj, n4, pair)));
    }
    {
      constexpr int T = 512, S = 4;
      size_t smem = (size_t)S * 2 * T * 16 + 64;
      cudaFuncSetAttribute(avg_tma<T, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(avg_tma<T, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      RUN("tma ld T512 S4 + stg, 3/SM", (avg_tma<T, S, false><<<sms * 3, 256, smem>>>(xi, xj, n4, pair)));
      RUN("tma ld T512 S4 + bulk st, 3/SM", (avg_tma<T, S, true><<<sms * 3, 256, smem>>>(xi, xj, n4, pair)));
    }
    {
      constexpr int T = 2048, S = 3;
      size_t smem = (size_t)S * 2 * T * 16 + 64;
      cudaFuncSetAttribute(avg_tma<T, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(avg_tma<T, S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      RUN("tma ld T2048 S3 + stg, 1/SM", (avg_tma<T, S, false><<<sms, 1024, smem>>>(xi, xj, n4, pair)));
      RUN("tma ld T2048 S3 + bulk st, 1/SM", (avg_tma<T, S, true><<<sms, 1024, smem>>>(xi, xj, n4, pair)));
    }
    {
      constexpr int T = 512, S = 4;
      size_t smem = (size_t)S * 2 * T * 16 + 64;
      cudaFuncSetAttribute(avg_tma<T, S, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      RUN("IL tma ld T512 S4 + stg 512thr, 2/SM", (avg_tma<T, S, false, true><<<sms * 2, 512, smem>>>(xi, xj, n4, pair)));
      RUN("IL tma ld T512 S4 + stg 256thr, 3/SM", (avg_tma<T, S, false, true><<<sms * 3, 256, smem>>>(xi, xj, n4, pair)));
    }
    {
      constexpr int T = 1024, S = 3;
      size_t smem = (size_t)S * 2 * T * 16 + 64;
      cudaFuncSetAttribute(avg_tma<T, S, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      RUN("IL tma ld T1024 S3 + stg 512thr, 2/SM", (avg_tma<T, S, false, true><<<sms * 2, 512, smem>>>(xi, xj, n4, pair)));
    }
    {
      constexpr int T = 256, S = 6;
      size_t smem = (size_t)S * 2 * T * 16 + 64;
      cudaFuncSetAttribute(avg_tma<T, S, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      RUN("IL tma ld T256 S6 + stg 256thr, 4/SM", (avg_tma<T, S, false, true><<<sms * 4, 256, smem>>>(xi, xj, n4, pair)));
      RUN("IL tma ld T256 S6 + stg 256thr, 2/SM", (avg_tma<T, S, false, true><<<sms * 2, 256, smem>>>(xi, xj, n4, pair)));
    }
    for (int cps = 1; cps <= 2; ++cps) {
      char nm[128];
      snprintf(nm, 128, "stride U8 256thr x%d/SM", 2 * cps); RUN(nm, (avg_stride<8><<<sms * cps * 2, 256>>>(xi, xj, n4, pair)));
      snprintf(nm, 128, "stride U2 512thr x%d/SM", cps); RUN(nm, (avg_stride<2><<<sms * cps, 512>>>(xi, xj, n4, pair)));
      snprintf(nm, 128, "stride U4 1024thr x%d/SM", cps); RUN(nm, (avg_stride<4><<<sms * cps, 1024>>>(xi, xj, n4, pair)));
    }
    // reference: cudaMemcpy device-to-device (1R1W of 4d bytes)
    if (!pair) RUN("cudaMemcpy D2D (1R1W)", (cudaMemcpyAsync(xj, xi, d * 4, cudaMemcpyDeviceToDevice)));
  }
  return 0;
}
