// mlp.cu -- minibatch gradient of the 2-layer MLP (config 3, reading R18):
//   Z1 = X_b W1^T + b1, H = tanh(Z1), Z2 = H W2^T + b2, loss = sum_b CE(softmax(Z2_b), y_b)
//   g = sum over the batch of dloss/dw  (a SUM), flat layout [W1 | b1 | W2 | b2].
// The two large contractions run on the tensor cores (gemm.cu, tcgen05 3xTF32):
//   GEMM1  Z1      [M x H] = X_b  [M x I] . W1 [H x I]^T     (split-K partial planes)
//   GEMM2  dW1     [H x I] = dZ1^T [H x M] . X_b^T [I x M]^T  (written straight into g)
// The N = 10 layer, softmax-CE and the batch reductions run on CUDA cores (fp32).
#include "internal.h"

namespace adp {

namespace {

// batch indices: explicit, or Philox4x32-10(key = seed, ctr = (lo32(k), m, "BATC", hi32(k))) (as lsq/logreg)
__global__ void k_mlp_idx(const int* __restrict__ idx_in, int M, uint2 key, unsigned long long k, int S,
                          int* __restrict__ idx) {
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < M; m += gridDim.x * blockDim.x) {
    if (idx_in) { idx[m] = idx_in[m]; continue; }
    const uint4 o = philox4x32_10(make_uint4((uint32_t)k, (uint32_t)m, 0x42415443u, (uint32_t)(k >> 32)), key);
    idx[m] = (int)(((unsigned long long)o.x * (unsigned long long)(uint32_t)S) >> 32);
  }
}

__device__ __forceinline__ void split1(float v, float& h, float& l) {
  uint32_t a, b;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(a) : "f"(v));
  const float r = v - __uint_as_float(a);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(b) : "f"(r));
  h = __uint_as_float(a);
  l = __uint_as_float(b);
}

// X_b (M x I) and X_b^T (I x M), both as tf32 hi/lo planes; 32 x 32 tiles through smem
__global__ void k_mlp_gather(const float* __restrict__ X, int I, const int* __restrict__ idx, int M,
                             float* __restrict__ xh, float* __restrict__ xl, float* __restrict__ th,
                             float* __restrict__ tl) {
  __shared__ float t[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const float v = X[(long long)idx[r0 + r] * I + c0 + threadIdx.x];
    t[r][threadIdx.x] = v;
    float h, l;
    split1(v, h, l);
    xh[(long long)(r0 + r) * I + c0 + threadIdx.x] = h;
    xl[(long long)(r0 + r) * I + c0 + threadIdx.x] = l;
  }
  __syncthreads();
  for (int c = threadIdx.y; c < 32; c += blockDim.y) {
    float h, l;
    split1(t[threadIdx.x][c], h, l);
    th[(long long)(c0 + c) * M + r0 + threadIdx.x] = h;
    tl[(long long)(c0 + c) * M + r0 + threadIdx.x] = l;
  }
}

// one CTA per sample b: z1 = sum of split-K partials + b1, tanh, the N = O output
// layer, softmax-CE backward, dz1; writes h, dz1 (row b), dz2 and dZ1^T hi/lo (column b)
constexpr int kMidThreads = 256;
constexpr int kMaxOut = 32;

__global__ void __launch_bounds__(kMidThreads) k_mlp_mid(const float* __restrict__ z1p, int splits, int M, int H,
                                                         int O, const float* __restrict__ w,
                                                         long long off_b1, long long off_W2, long long off_b2,
                                                         const int* __restrict__ y, const int* __restrict__ idx,
                                                         float* __restrict__ hbuf, float* __restrict__ dz1buf,
                                                         float* __restrict__ dz2buf, float* __restrict__ dth,
                                                         float* __restrict__ dtl) {
  extern __shared__ float sh[];
  float* z1 = sh;            // H
  float* hh = sh + H;        // H
  __shared__ float z2[kMaxOut], dz2[kMaxOut];
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const float* b1 = w + off_b1;
  const float* W2 = w + off_W2;
  const float* b2 = w + off_b2;
  for (int u = threadIdx.x; u < H; u += blockDim.x) {
    float s = 0.0f;
    for (int p = 0; p < splits; ++p) s += z1p[((long long)p * M + b) * H + u];
    s += b1[u];
    const float hv = tanhf(s);
    z1[u] = hv;                                   // keep tanh(z1) for the derivative 1 - h^2
    hh[u] = hv;
    hbuf[(long long)b * H + u] = hv;
  }
  __syncthreads();
  for (int o = warp; o < O; o += nw) {
    float acc = 0.0f;
    for (int u = lane; u < H; u += 32) acc = fmaf(W2[(long long)o * H + u], hh[u], acc);
#pragma unroll
    for (int q = 16; q; q >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, q);
    if (lane == 0) z2[o] = acc + b2[o];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = -INFINITY;
    for (int o = 0; o < O; ++o) mx = fmaxf(mx, z2[o]);
    float se = 0.0f;
    for (int o = 0; o < O; ++o) se += expf(z2[o] - mx);
    const int yb = y[idx[b]];
    for (int o = 0; o < O; ++o) {
      const float pr = expf(z2[o] - mx) / se;
      dz2[o] = pr - (o == yb ? 1.0f : 0.0f);
      dz2buf[(long long)b * O + o] = dz2[o];
    }
  }
  __syncthreads();
  for (int u = threadIdx.x; u < H; u += blockDim.x) {
    float dh = 0.0f;
    for (int o = 0; o < O; ++o) dh = fmaf(W2[(long long)o * H + u], dz2[o], dh);
    const float dz = dh * (1.0f - z1[u] * z1[u]);
    dz1buf[(long long)b * H + u] = dz;
    float hi, lo;
    split1(dz, hi, lo);
    dth[(long long)u * M + b] = hi;
    dtl[(long long)u * M + b] = lo;
  }
}

// batch sums (fixed order): db1[u] = sum_b dz1, dW2[o][u] = sum_b dz2[b][o] h[b][u], db2[o] = sum_b dz2
__global__ void k_mlp_reduce(const float* __restrict__ hbuf, const float* __restrict__ dz1buf,
                             const float* __restrict__ dz2buf, int M, int H, int O, float* __restrict__ g,
                             long long off_b1, long long off_W2, long long off_b2) {
  const long long n = (long long)H + (long long)O * H + O;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x) {
    float acc = 0.0f;
    if (t < H) {
      for (int b = 0; b < M; ++b) acc += dz1buf[(long long)b * H + t];
      g[off_b1 + t] = acc;
    } else if (t < H + (long long)O * H) {
      const long long r = t - H;
      const int o = (int)(r / H), u = (int)(r % H);
      for (int b = 0; b < M; ++b) acc = fmaf(dz2buf[(long long)b * O + o], hbuf[(long long)b * H + u], acc);
      g[off_W2 + r] = acc;
    } else {
      const int o = (int)(t - H - (long long)O * H);
      for (int b = 0; b < M; ++b) acc += dz2buf[(long long)b * O + o];
      g[off_b2 + o] = acc;
    }
  }
}

}  // namespace

int mlp_splits(const MlpShape& sh) {
  const int kb = sh.n_in / 32;
  int best = 1;
  for (int s = 1; s <= 16; ++s)
    if (kb % s == 0) best = s;
  return best;
}

size_t mlp_scratch_floats(const MlpShape& sh, int M) {
  const size_t I = sh.n_in, H = sh.n_hid, O = sh.n_out;
  return 4 * (size_t)M * I           // X_b hi/lo, X_b^T hi/lo
         + 2 * H * I                 // W1 hi/lo
         + (size_t)mlp_splits(sh) * M * H  // Z1 partial planes
         + 2 * (size_t)M * H         // h, dz1
         + (size_t)M * O             // dz2
         + 2 * H * (size_t)M         // dZ1^T hi/lo
         + (size_t)M + 64;           // idx
}

bool mlp_supported(const MlpShape& sh, int M) {
  return M % 128 == 0 && sh.n_hid % 128 == 0 && sh.n_in % 128 == 0 && sh.n_out >= 1 && sh.n_out <= kMaxOut &&
         (size_t)2 * sh.n_hid * sizeof(float) <= 48 * 1024;
}

cudaError_t mlp_plan(MlpWork& wk, const MlpShape& sh, int M, float* scratch) {
  wk.sh = sh;
  wk.M = M;
  wk.splits = mlp_splits(sh);
  const size_t I = sh.n_in, H = sh.n_hid;
  float* p = scratch;
  wk.xh = p; p += (size_t)M * I;
  wk.xl = p; p += (size_t)M * I;
  wk.th = p; p += (size_t)M * I;
  wk.tl = p; p += (size_t)M * I;
  wk.w1h = p; p += H * I;
  wk.w1l = p; p += H * I;
  wk.z1p = p; p += (size_t)wk.splits * M * H;
  wk.hbuf = p; p += (size_t)M * H;
  wk.dz1 = p; p += (size_t)M * H;
  wk.dz2 = p; p += (size_t)M * sh.n_out;
  wk.dth = p; p += H * M;
  wk.dtl = p; p += H * M;
  wk.idx = reinterpret_cast<int*>(p);
  cudaError_t e;
  // GEMM1: A = X_b [M x I], B = W1 [H x I]
  if ((e = make_tmap_k_major(&wk.g1.Ah, wk.xh, M, I, 128)) != cudaSuccess) return e;
  if ((e = make_tmap_k_major(&wk.g1.Al, wk.xl, M, I, 128)) != cudaSuccess) return e;
  if ((e = make_tmap_k_major(&wk.g1.Bh, wk.w1h, H, I, 128)) != cudaSuccess) return e;
  if ((e = make_tmap_k_major(&wk.g1.Bl, wk.w1l, H, I, 128)) != cudaSuccess) return e;
  // GEMM2: A = dZ1^T [H x M], B = X_b^T [I x M]
  if ((e = make_tmap_k_major(&wk.g2.Ah, wk.dth, H, M, 128)) != cudaSuccess) return e;
  if ((e = make_tmap_k_major(&wk.g2.Al, wk.dtl, H, M, 128)) != cudaSuccess) return e;
  if ((e = make_tmap_k_major(&wk.g2.Bh, wk.th, I, M, 128)) != cudaSuccess) return e;
  return make_tmap_k_major(&wk.g2.Bl, wk.tl, I, M, 128);
}

cudaError_t launch_mlp_grad(const MlpWork& wk, const float* X, const int* y, int S, const int* idx_in,
                            uint2 batch_key, unsigned long long k, const float* w, float* g, cudaStream_t s) {
  const int I = wk.sh.n_in, H = wk.sh.n_hid, O = wk.sh.n_out, M = wk.M;
  const long long off_b1 = (long long)H * I, off_W2 = off_b1 + H, off_b2 = off_W2 + (long long)O * H;
  cudaError_t e;
  k_mlp_idx<<<1, 256, 0, s>>>(idx_in, M, batch_key, k, S, wk.idx);
  k_mlp_gather<<<dim3(I / 32, M / 32), dim3(32, 8), 0, s>>>(X, I, wk.idx, M, wk.xh, wk.xl, wk.th, wk.tl);
  if ((e = launch_split_tf32(w, wk.w1h, wk.w1l, (long long)H * I, s)) != cudaSuccess) return e;
  if ((e = launch_gemm_tf32x3(wk.g1, wk.z1p, M, H, I, wk.splits, 128, s)) != cudaSuccess) return e;
  k_mlp_mid<<<M, kMidThreads, 2 * H * sizeof(float), s>>>(wk.z1p, wk.splits, M, H, O, w, off_b1, off_W2, off_b2, y,
                                                          wk.idx, wk.hbuf, wk.dz1, wk.dz2, wk.dth, wk.dtl);
  k_mlp_reduce<<<64, 256, 0, s>>>(wk.hbuf, wk.dz1, wk.dz2, M, H, O, g, off_b1, off_W2, off_b2);
  if ((e = launch_gemm_tf32x3(wk.g2, g, H, I, M, 1, 128, s)) != cudaSuccess) return e;
  return cudaGetLastError();
}

const void* mlp_module_anchor() { return (const void*)k_mlp_idx; }

}  // namespace adp
