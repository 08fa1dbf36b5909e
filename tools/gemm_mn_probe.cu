// Probe of the operand paths of gemm.cu in isolation (diagnostic): each combination against a
// host fp64 reference, then the config-3 GEMM1 / GEMM2 launches with per-CTA phase timestamps.
// Build: tools/gemm_probe_build.sh (compiles a copy of gemm.cu with kGemmTrace = true).
#include "gemm_traced.cu"
#include <cstdio>
#include <vector>
#include <cmath>
#include <algorithm>

using namespace adp;

// phase times over the CTAs of the last launch, relative to the earliest CTA start (us)
static void trace_report(int nb, int kbs) {
  std::vector<unsigned long long> t(1024 * 48);
  cudaMemcpyFromSymbol(t.data(), g_gemm_trace, sizeof(unsigned long long) * t.size());
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < nb; ++b) t0 = t[b * 48] < t0 ? t[b * 48] : t0;
  auto row = [&](const char* name, int i) {
    std::vector<double> v;
    for (int b = 0; b < nb; ++b) v.push_back((t[b * 48 + i] - t0) * 1e-3);
    std::sort(v.begin(), v.end());
    printf("   %-12s min %6.2f  med %6.2f  max %6.2f\n", name, v.front(), v[v.size() / 2], v.back());
  };
  row("start", 0);
  row("setup", 1);
  char nm[32];
  for (int kb = 0; kb < kbs && kb < 12; ++kb) {
    snprintf(nm, sizeof nm, "kb%d ready", kb); row(nm, 2 + kb);
    if (kb < 2) {
      snprintf(nm, sizeof nm, "kb%d A lds", kb); row(nm, 32 + 4 * kb);
      snprintf(nm, sizeof nm, "kb%d A lo", kb); row(nm, 33 + 4 * kb);
      snprintf(nm, sizeof nm, "kb%d A tst", kb); row(nm, 34 + 4 * kb);
      snprintf(nm, sizeof nm, "kb%d B lo", kb); row(nm, 35 + 4 * kb);
    }
    snprintf(nm, sizeof nm, "kb%d mma", kb); row(nm, 14 + kb);
  }
  row("accum", 26);
  row("tmem out", 27);
  row("pushed", 29);
  row("received", 30);
  row("end", 28);
}

int main() {
  const int M = 128, N = 128, K = 128, S = 512;
  // logical A(m, k), B(n, k)
  std::vector<float> Akm(K * M), Amk(M * K), Xs(S * N), Bnk(N * K);
  std::vector<int> idx(K);
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xFFFF) / 65536.0f - 0.5f; };
  for (int k = 0; k < K; ++k) for (int m = 0; m < M; ++m) { float v = rnd(); Akm[k * M + m] = v; Amk[m * K + k] = v; }
  for (int i = 0; i < S * N; ++i) Xs[i] = rnd();
  for (int k = 0; k < K; ++k) idx[k] = (k * 37 + 11) % S;
  for (int n = 0; n < N; ++n) for (int k = 0; k < K; ++k) Bnk[n * K + k] = Xs[idx[k] * N + n];
  std::vector<double> ref(M * N, 0.0);
  for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
    double a = 0; for (int k = 0; k < K; ++k) a += (double)Amk[m * K + k] * Bnk[n * K + k];
    ref[m * N + n] = a;
  }
  float *dAkm, *dAmk, *dX, *dB, *dC; int* dIdx;
  cudaMalloc(&dAkm, 4 * K * M); cudaMalloc(&dAmk, 4 * M * K); cudaMalloc(&dX, 4 * S * N); cudaMalloc(&dB, 4 * N * K);
  cudaMalloc(&dC, 4 * M * N); cudaMalloc(&dIdx, 4 * K);
  cudaMemcpy(dAkm, Akm.data(), 4 * K * M, cudaMemcpyHostToDevice);
  cudaMemcpy(dAmk, Amk.data(), 4 * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, Xs.data(), 4 * S * N, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bnk.data(), 4 * N * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dIdx, idx.data(), 4 * K, cudaMemcpyHostToDevice);
  CUtensorMap tA_k, tA_mn, tB_k;
  make_tmap_k_major(&tA_k, dAmk, M, K, 128);       // K-major A
  make_tmap_mn_major(&tA_mn, dAkm, K, M);       // MN-major A: [K x M] rows, 32 x 32 boxes
  make_tmap_k_major(&tB_k, dB, N, K, 64);          // K-major B
  GemmGather gg = {};
  gg.x = dX; gg.ld = N; gg.idx = dIdx; gg.cluster = 1;
  const dim3 grid(N / 64, M / 128, 1);
  auto check = [&](const char* name, cudaError_t e) {
    cudaError_t e2 = cudaDeviceSynchronize();
    std::vector<float> C(M * N);
    cudaMemcpy(C.data(), dC, 4 * M * N, cudaMemcpyDeviceToHost);
    double err = 0; int zeros = 0, bad = 0;
    for (int i = 0; i < M * N; ++i) {
      double d = std::fabs(C[i] - ref[i]); err = d > err ? d : err;
      zeros += C[i] == 0.0f; bad += d > 1e-3;
    }
    printf("%-28s launch %s sync %s max err %.3e zeros %d bad %d  C[0..3] %.4f %.4f %.4f %.4f ref %.4f %.4f\n", name,
           cudaGetErrorString(e), cudaGetErrorString(e2), err, zeros, bad, C[0], C[1], C[2], C[3], ref[0], ref[1]);
    if (bad) {   // where: first bad entries
      int shown = 0;
      for (int i = 0; i < M * N && shown < 6; ++i)
        if (std::fabs(C[i] - ref[i]) > 1e-3) { printf("   (%d,%d) %.4f ref %.4f\n", i / N, i % N, C[i], ref[i]); ++shown; }
    }
    cudaMemset(dC, 0, 4 * M * N);
  };
  cudaMemset(dC, 0, 4 * M * N);
  check("K/K tma", launch_one<64, kOpTma, kOpTma, kEpiStore>(tA_k, tB_k, dC, N, grid, K / 32, 0, gg, 0));
  check("MN tma / K tma", launch_one<64, kOpTmaMN, kOpTma, kEpiStore>(tA_mn, tB_k, dC, N, grid, K / 32, 0, gg, 0));
  check("K tma / MN gather", launch_one<64, kOpTma, kOpGatherMN, kEpiStore>(tA_k, tA_k, dC, N, grid, K / 32, 0, gg, 0));
  check("MN tma / MN gather", launch_one<64, kOpTmaMN, kOpGatherMN, kEpiStore>(tA_mn, tA_mn, dC, N, grid, K / 32, 0, gg, 0));
  // ---- how many clusters of the GEMM1 kernel can be resident at once
  for (int cs : {16, 8, 4}) {
    auto kern = k_gemm_tf32x3<64, kOpGatherK, kOpTma, kEpiClusterTanh>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gemm_smem(64, true, true));
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(8, 1, 16);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = gemm_smem(64, true, true);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = cs;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    printf("cluster %2d: max active clusters %d (%s), smem %zu\n", cs, n, cudaGetErrorString(e), gemm_smem(64, true, true));
  }
  // ---- config-3 shapes, traced: GEMM1 (gather K-major A, TMA B, cluster tanh) and GEMM2
  {
    const int I = 3072, H = 512, Mb = 128, Sx = 8192;
    float *X, *W, *h, *h4, *dz, *g; int* id;
    cudaMalloc(&h4, 4ll * 4 * Mb * H);
    cudaMalloc(&X, 4ll * Sx * I); cudaMalloc(&W, 4ll * H * I + 4 * H); cudaMalloc(&h, 4ll * Mb * H);
    cudaMalloc(&dz, 4ll * Mb * H); cudaMalloc(&g, 4ll * H * I); cudaMalloc(&id, 4 * Mb);
    cudaMemset(X, 0, 4ll * Sx * I); cudaMemset(W, 0, 4ll * H * I + 4 * H); cudaMemset(dz, 0, 4ll * Mb * H);
    for (int split : {16, 8}) for (int bn : {64, 32}) {
      if (bn == 32 && split == 16) continue;
      CUtensorMap tw, tdz;
      make_tmap_k_major(&tw, W, H, I, bn);
      GemmGather g1 = {};
      g1.x = X; g1.ld = I; g1.idx = nullptr; g1.idx_out = id; g1.key = make_uint2(1, 2); g1.k = 3; g1.S = Sx;
      g1.cluster = split == 16 ? 4 : split; g1.bias = W + (long long)H * I;
      const dim3 gr(H / bn, 1, split);
      for (int rep = 0; rep < 3; ++rep) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        cudaError_t e = launch_mlp_gemm1(tw, g1, h4, Mb, H, I, split, bn, 0);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep == 2) { printf("GEMM1 bn %d splits %d cluster %d: %s %.2f us\n", bn, split, g1.cluster, cudaGetErrorString(e), ms * 1e3); trace_report(gr.x * gr.y * gr.z, I / 32 / split); }
      }
      make_tmap_mn_major(&tdz, dz, Mb, H);
      (void)tdz;
    }
    CUtensorMap tdz;
    make_tmap_mn_major(&tdz, dz, Mb, H);
    GemmGather g2 = {};
    g2.x = X; g2.ld = I; g2.idx = id; g2.cluster = 1;
    const dim3 gr(I / 96, H / 128, 1);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaError_t e = launch_one<96, kOpTmaMN, kOpGatherMN, kEpiStore>(tdz, tdz, g, I, gr, Mb / 32, 0, g2, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) { printf("GEMM2 bn 96: %s %.2f us\n", cudaGetErrorString(e), ms * 1e3); trace_report(gr.x * gr.y * gr.z, Mb / 32); }
    }
  }
  return 0;
}
