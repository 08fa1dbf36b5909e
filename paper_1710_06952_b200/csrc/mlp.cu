// mlp.cu -- minibatch gradient of the 2-layer MLP (config 3, reading R18):
//   Z1 = X_b W1^T + b1, H = tanh(Z1), Z2 = H W2^T + b2, loss = sum_b CE(softmax(Z2_b), y_b)
//   g = sum over the batch of dloss/dw  (a SUM), flat layout [W1 | b1 | W2 | b2].
// Three launches per gradient:
//   1. GEMM1  h [M x H] = tanh(X_b W1^T + b1) on tcgen05 (3xTF32): draws the batch indices
//             (explicit or device Philox) and publishes them, gathers the X rows itself
//             (cp.async into the swizzled tiles: X_b is never written), W1 straight from the
//             model row through its own tensor map, split-K with the partials of each
//             thread-block cluster reduced in distributed shared memory (4 planes left at
//             config 3; a single cluster per tile finishes bias + tanh in the epilogue)
//   2. mid:   one CTA per sample -- h = tanh(sum of the planes + b1), the N = O output layer,
//             softmax-CE backward, dz1, dz2
//   3. GEMM2  dW1 [H x I] = dZ1^T X_b into g: dZ1 read MN-major by TMA (no transpose),
//             X rows gathered again (MN-major); extra CTAs of the same launch compute the
//             batch reductions (db1, dW2, db2)
// The tf32 hi / lo split of every operand happens in shared memory (gemm.cu).
#include "internal.h"

namespace adp {

namespace {

// GEMM1 tile, split-K and cluster sizes at config 3 (I = 3072, H = 512, M = 128): 512 / 64 = 8
// tiles x 16 splits = 128 CTAs (6 k-blocks each) in 32 clusters of 4 -> 4 partial planes.  (A
// cluster of 16 would finish tanh(z1 + b1) in the GEMM, but only 7 clusters of 16 -- 15 of 8 --
// fit on the GPU at once: two waves.)
constexpr int kG1BN = 64, kG1MaxSplits = 16, kG1Cluster = 4;

// one CTA per sample b, one thread per hidden unit u (blockDim = H): h (GEMM1's epilogue, or
// tanh(sum of GEMM1's partial planes + b1)),
// the N = O output layer (W2 column u kept in registers, per-warp shuffle sums then a
// fixed-order sum over warps), softmax-CE backward across the lanes of warp 0, dz1;
// writes dz1 (row b) and dz2
constexpr int kMaxOut = 32;

__global__ void __launch_bounds__(1024) k_mlp_mid(const float* __restrict__ z1p, int planes, int M,
                                                  float* __restrict__ hbuf, int H, int O,
                                                  const float* __restrict__ w, long long off_b1, long long off_W2,
                                                  long long off_b2, const int* __restrict__ y,
                                                  const int* __restrict__ idx, float* __restrict__ dz1buf,
                                                  float* __restrict__ dz2buf) {
  __shared__ float red[32][kMaxOut];
  __shared__ float dz2s[kMaxOut];
  __shared__ int s_lab;
  const int b = blockIdx.x, u = threadIdx.x;
  const int warp = u >> 5, lane = u & 31, nw = blockDim.x >> 5;
  const float* W2 = w + off_W2;
  float w2r[kMaxOut];
#pragma unroll
  for (int o = 0; o < kMaxOut; ++o) w2r[o] = o < O ? W2[(long long)o * H + u] : 0.0f;   // the model: before the wait
  const float b1u = w[off_b1 + u];
  const float b2l = (warp == 0 && lane < O) ? w[off_b2 + lane] : 0.0f;
  pdl_wait();                                   // GEMM1's h (or z1 planes) and batch indices
  pdl_trigger();
  if (u == 0) s_lab = y[idx[b]];                // the label's two dependent loads overlap the planes'

  float hv;
  if (planes == 0) hv = hbuf[(long long)b * H + u];             // GEMM1 finished tanh(z1 + b1)
  else {                                                         // the cluster-reduced planes, in order
    float s = 0.0f;
    for (int p = 0; p < planes; ++p) s += z1p[((long long)p * M + b) * H + u];
    hv = tanhf(s + b1u);
    hbuf[(long long)b * H + u] = hv;
  }
#pragma unroll
  for (int o = 0; o < kMaxOut; ++o) {
    if (o >= O) break;                          // O is uniform: no divergence, no dead shuffles
    float part = w2r[o] * hv;
#pragma unroll
    for (int q = 16; q; q >>= 1) part += __shfl_xor_sync(0xffffffffu, part, q);
    if (lane == 0) red[warp][o] = part;
  }
  __syncthreads();
  if (warp == 0) {
    float z = -INFINITY;
    if (lane < O) {
      z = b2l;
      for (int q = 0; q < nw; ++q) z += red[q][lane];
    }
    float mx = z;
#pragma unroll
    for (int q = 16; q; q >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, q));
    const float e = lane < O ? expf(z - mx) : 0.0f;
    float se = e;
#pragma unroll
    for (int q = 16; q; q >>= 1) se += __shfl_xor_sync(0xffffffffu, se, q);
    if (lane < O) {
      const float d = e / se - (lane == s_lab ? 1.0f : 0.0f);
      dz2s[lane] = d;
      dz2buf[(long long)b * O + lane] = d;
    }
  }
  __syncthreads();
  float dh = 0.0f;
#pragma unroll
  for (int o = 0; o < kMaxOut; ++o)
    if (o < O) dh = fmaf(w2r[o], dz2s[o], dh);
  const float dz = dh * (1.0f - hv * hv);
  dz1buf[(long long)b * H + u] = dz;
}

}  // namespace

// GEMM1 split-K: Z1 is only M x H (8 tiles of 128 x 64 at config 3), so K is split over a
// cluster of CTAs per tile: the largest power of two <= kG1MaxSplits dividing the k-blocks
// with <= 160 CTAs in all
int mlp_splits(const MlpShape& sh, int M) {
  const int kb = sh.n_in / 32, tiles = (M / 128) * (sh.n_hid / kG1BN);
  int best = 1;
  for (int s = 2; s <= kG1MaxSplits; s *= 2)
    if (kb % s == 0 && tiles * s <= 160) best = s;
  return best;
}

int mlp_planes(const MlpShape& sh, int M) {
  const int s = mlp_splits(sh, M);
  return s <= kG1Cluster ? 0 : s / kG1Cluster;     // 0: the GEMM writes h itself
}

size_t mlp_scratch_floats(const MlpShape& sh, int M) {
  const size_t H = sh.n_hid, O = sh.n_out;
  return (size_t)mlp_planes(sh, M) * M * H         // z1 partial planes
         + 2 * (size_t)M * H                       // h, dz1
         + (size_t)M * O                           // dz2
         + (size_t)M + 64;                         // idx
}

bool mlp_supported(const MlpShape& sh, int M) {
  return M % 128 == 0 && M <= 1024 && sh.n_hid % 128 == 0 && sh.n_hid <= 1024 && sh.n_in % 128 == 0 &&
         sh.n_out >= 1 && sh.n_out <= kMaxOut;
}

cudaError_t mlp_plan(MlpWork& wk, const MlpShape& sh, int M, float* scratch) {
  wk.sh = sh;
  wk.M = M;
  wk.splits = mlp_splits(sh, M);
  wk.planes = mlp_planes(sh, M);
  wk.bn1 = kG1BN;
  wk.bn2 = sh.n_in % 96 == 0 ? 96 : 64;
  const size_t H = sh.n_hid;
  float* p = scratch;
  wk.z1p = p; p += (size_t)wk.planes * M * H;
  wk.hbuf = p; p += (size_t)M * H;
  wk.dz1 = p; p += (size_t)M * H;
  wk.dz2 = p; p += (size_t)M * sh.n_out;
  wk.idx = reinterpret_cast<int*>(p);
  return make_tmap_mn_major(&wk.dz1_m, wk.dz1, M, H);          // GEMM2 A: 32 x 32 boxes of dz1 [M x H]
}

cudaError_t launch_mlp_grad(const MlpWork& wk, const float* X, const int* y, int S, const int* idx_in,
                            uint2 batch_key, unsigned long long k, const float* w, float* g, cudaStream_t s) {
  const int I = wk.sh.n_in, H = wk.sh.n_hid, O = wk.sh.n_out, M = wk.M;
  const long long off_b1 = (long long)H * I, off_W2 = off_b1 + H, off_b2 = off_W2 + (long long)O * H;
  cudaError_t e;
  if (wk.w1_src != w) {                                       // W1 [H x I], the first H*I floats of w
    if ((e = make_tmap_k_major(&wk.w1_m, w, H, I, wk.bn1)) != cudaSuccess) return e;
    wk.w1_src = w;
  }
  const CUtensorMap& w1 = wk.w1_m;
  // the chain GEMM1 -> mid -> GEMM2 uses programmatic dependent launch: each kernel's
  // setup (GEMM: barriers, TMEM, tensor-map prefetch) overlaps its predecessor's tail
  GemmGather g1 = {};
  g1.x = X; g1.ld = I; g1.idx = idx_in; g1.idx_out = wk.idx; g1.key = batch_key; g1.k = k; g1.S = S;
  g1.cluster = wk.planes ? kG1Cluster : wk.splits; g1.bias = w + off_b1;
  if ((e = launch_mlp_gemm1(w1, g1, wk.planes ? wk.z1p : wk.hbuf, M, H, I, wk.splits, wk.bn1, s)) != cudaSuccess)
    return e;
  if ((e = launch_pdl(k_mlp_mid, dim3(M), dim3(H), 0, s, (const float*)wk.z1p, wk.planes, M, wk.hbuf, H, O, w,
                      off_b1, off_W2, off_b2, y, (const int*)wk.idx, wk.dz1, wk.dz2)) != cudaSuccess)
    return e;
  // dW1 in 128 x 96 tiles (I = 3072: 4 x 32 = 128 CTAs) and, in extra CTAs of the same launch,
  // the batch reductions db1, dW2, db2
  GemmGather g2 = {};
  g2.x = X; g2.ld = I; g2.idx = wk.idx; g2.cluster = 1;
  const int units = (H + 31) / 32, rows = H / 128;
  g2.red_ctas = (units + rows - 1) / rows;
  g2.r_M = M; g2.r_H = H; g2.r_O = O; g2.r_h = wk.hbuf; g2.r_dz1 = wk.dz1; g2.r_dz2 = wk.dz2; g2.r_g = g;
  g2.r_off_b1 = off_b1; g2.r_off_W2 = off_W2; g2.r_off_b2 = off_b2;
  if ((e = launch_mlp_gemm2(wk.dz1_m, g2, g, H, I, M, wk.bn2, s)) != cudaSuccess) return e;
  return cudaGetLastError();
}

const void* mlp_module_anchor() { return (const void*)k_mlp_mid; }

}  // namespace adp
