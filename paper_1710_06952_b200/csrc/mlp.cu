// mlp.cu -- minibatch gradient of the 2-layer MLP (config 3, reading R18):
//   Z1 = X_b W1^T + b1, H = tanh(Z1), Z2 = H W2^T + b2, loss = sum_b CE(softmax(Z2_b), y_b)
//   g = sum over the batch of dloss/dw  (a SUM), flat layout [W1 | b1 | W2 | b2].
// Four launches per gradient:
//   1. gather: batch indices (explicit or device Philox) and X_b [M x I], X_b^T [I x M] (fp32)
//   2. GEMM1  Z1 [M x H] = X_b . W1^T on tcgen05 (3xTF32, split-K partial planes; W1 read
//             straight from the model row through its own tensor map)
//   3. mid:   one CTA per sample -- sum the K-split planes + b1, tanh, the N = O output layer,
//             softmax-CE backward, dz1; writes h, dz1, dz2 and dZ1^T (fp32)
//   4. GEMM2  dW1 [H x I] = dZ1^T . (X_b^T)^T into g, with the batch reductions
//             (db1, dW2, db2) running beside it on a side stream (fork / join events)
// The tf32 hi / lo split of every operand happens in shared memory (gemm.cu).
#include "internal.h"

namespace adp {

namespace {

// batch indices (explicit, or Philox4x32-10(key = seed, ctr = (lo32(k), m, "BATC", hi32(k))), as
// lsq/logreg) and the gathered batch X_b [M x I] plus its transpose X_b^T [I x M]; 32 x 32 tiles
__global__ void k_mlp_gather(const float* __restrict__ X, int I, const int* __restrict__ idx_in, uint2 key,
                             unsigned long long k, int S, int M, int* __restrict__ idx, float* __restrict__ xb,
                             float* __restrict__ xbt) {
  __shared__ float t[32][33];
  __shared__ int rows[32];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  pdl_wait();                                   // the previous gradient's GEMM2 still reads xbt
  pdl_trigger();
  if (threadIdx.y == 0) {
    const int m = r0 + threadIdx.x;
    int v;
    if (idx_in) v = idx_in[m];
    else {
      const uint4 o = philox4x32_10(make_uint4((uint32_t)k, (uint32_t)m, 0x42415443u, (uint32_t)(k >> 32)), key);
      v = (int)(((unsigned long long)o.x * (unsigned long long)(uint32_t)S) >> 32);
    }
    rows[threadIdx.x] = v;
    if (blockIdx.x == 0) idx[m] = v;
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const float v = X[(long long)rows[r] * I + c0 + threadIdx.x];
    t[r][threadIdx.x] = v;
    xb[(long long)(r0 + r) * I + c0 + threadIdx.x] = v;
  }
  __syncthreads();
  for (int c = threadIdx.y; c < 32; c += blockDim.y) xbt[(long long)(c0 + c) * M + r0 + threadIdx.x] = t[threadIdx.x][c];
}

// one CTA per sample b, one thread per hidden unit u (blockDim = H): z1 = sum of the
// split-K partials + b1, tanh, the N = O output layer (W2 column u kept in registers,
// per-warp shuffle sums then a fixed-order sum over warps), softmax-CE backward across
// the lanes of warp 0, dz1; writes h, dz1 (row b), dz2 and dZ1^T (column b)
constexpr int kMaxOut = 32;

__global__ void __launch_bounds__(1024) k_mlp_mid(const float* __restrict__ z1p, int splits, int M, int H, int O,
                                                  const float* __restrict__ w, long long off_b1, long long off_W2,
                                                  long long off_b2, const int* __restrict__ y,
                                                  const int* __restrict__ idx, float* __restrict__ hbuf,
                                                  float* __restrict__ dz1buf, float* __restrict__ dz2buf,
                                                  float* __restrict__ dzt) {
  __shared__ float red[32][kMaxOut];
  __shared__ float dz2s[kMaxOut];
  const int b = blockIdx.x, u = threadIdx.x;
  const int warp = u >> 5, lane = u & 31, nw = blockDim.x >> 5;
  const float* W2 = w + off_W2;
  pdl_wait();                                   // GEMM1's split-K planes
  pdl_trigger();
  float s = 0.0f;
#pragma unroll 8
  for (int p = 0; p < splits; ++p) s += z1p[((long long)p * M + b) * H + u];
  s += w[off_b1 + u];
  const float hv = tanhf(s);
  hbuf[(long long)b * H + u] = hv;
  float w2r[kMaxOut];
#pragma unroll
  for (int o = 0; o < kMaxOut; ++o) {
    w2r[o] = o < O ? W2[(long long)o * H + u] : 0.0f;
    float part = w2r[o] * hv;
#pragma unroll
    for (int q = 16; q; q >>= 1) part += __shfl_xor_sync(0xffffffffu, part, q);
    if (lane == 0 && o < O) red[warp][o] = part;
  }
  __syncthreads();
  if (warp == 0) {
    float z = -INFINITY;
    if (lane < O) {
      z = w[off_b2 + lane];
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
      const float d = e / se - (lane == y[idx[b]] ? 1.0f : 0.0f);
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
  dzt[(long long)u * M + b] = dz;
}

// batch reductions (reading R18): db1[u] = sum_b dz1[b][u], dW2[o][u] = sum_b dz2[b][o] h[b][u],
// db2[o] = sum_b dz2[b][o] -- one warp per output, lane l sums samples l, l + 32, ..., then a
// shuffle tree in a fixed order (deterministic).  Runs on the side stream beside GEMM2.
__global__ void __launch_bounds__(256) k_mlp_reduce(const float* __restrict__ hbuf, const float* __restrict__ dz1,
                                                    const float* __restrict__ dz2, int M, int H, int O,
                                                    float* __restrict__ g, long long off_b1, long long off_W2,
                                                    long long off_b2) {
  const long long n = (long long)H + (long long)O * H + O;
  const int lane = threadIdx.x & 31;
  for (long long q = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < n;
       q += ((long long)gridDim.x * blockDim.x) >> 5) {
    float acc = 0.0f;
    if (q < H) {
      for (int b = lane; b < M; b += 32) acc += dz1[(long long)b * H + q];
    } else if (q < H + (long long)O * H) {
      const long long r = q - H;
      const int o = (int)(r / H), u = (int)(r % H);
      for (int b = lane; b < M; b += 32) acc = fmaf(dz2[(long long)b * O + o], hbuf[(long long)b * H + u], acc);
    } else {
      const int o = (int)(q - H - (long long)O * H);
      for (int b = lane; b < M; b += 32) acc += dz2[(long long)b * O + o];
    }
#pragma unroll
    for (int w = 16; w; w >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, w);
    if (lane == 0) {
      if (q < H) g[off_b1 + q] = acc;
      else if (q < H + (long long)O * H) g[off_W2 + (q - H)] = acc;
      else g[off_b2 + (q - H - (long long)O * H)] = acc;
    }
  }
}

}  // namespace

// GEMM1 split-K: Z1 is only M x H (4 tiles of 128 x 128 at config 3), so K is split to
// put ~128 CTAs of 128 x 64 tiles on the GPU (6 k-blocks each at I = 3072)
int mlp_splits(const MlpShape& sh, int M) {
  const int kb = sh.n_in / 32, tiles = (M / 128) * (sh.n_hid / 64);
  int best = 1;
  for (int s = 1; s <= 32; ++s)
    if (kb % s == 0 && tiles * s <= 160) best = s;
  return best;
}

size_t mlp_scratch_floats(const MlpShape& sh, int M) {
  const size_t I = sh.n_in, H = sh.n_hid, O = sh.n_out;
  return 2 * (size_t)M * I                         // X_b, X_b^T
         + (size_t)mlp_splits(sh, M) * M * H       // Z1 partial planes
         + 2 * (size_t)M * H                       // h, dz1
         + (size_t)M * O                           // dz2
         + H * (size_t)M                           // dZ1^T
         + (size_t)M + 64;                         // idx
}

bool mlp_supported(const MlpShape& sh, int M) {
  return M % 128 == 0 && sh.n_hid % 128 == 0 && sh.n_hid <= 1024 && sh.n_in % 128 == 0 && sh.n_out >= 1 &&
         sh.n_out <= kMaxOut;
}

cudaError_t mlp_plan(MlpWork& wk, const MlpShape& sh, int M, float* scratch) {
  wk.sh = sh;
  wk.M = M;
  wk.splits = mlp_splits(sh, M);
  const size_t I = sh.n_in, H = sh.n_hid;
  float* p = scratch;
  wk.xb = p; p += (size_t)M * I;
  wk.xbt = p; p += (size_t)M * I;
  wk.z1p = p; p += (size_t)wk.splits * M * H;
  wk.hbuf = p; p += (size_t)M * H;
  wk.dz1 = p; p += (size_t)M * H;
  wk.dz2 = p; p += (size_t)M * sh.n_out;
  wk.dzt = p; p += H * M;
  wk.idx = reinterpret_cast<int*>(p);
  cudaError_t e;
  if (!wk.side) {
    if ((e = cudaStreamCreateWithFlags(&wk.side, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&wk.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&wk.join, cudaEventDisableTiming)) != cudaSuccess) return e;
  }
  if ((e = make_tmap_k_major(&wk.x_b, wk.xb, M, I, 128)) != cudaSuccess) return e;      // GEMM1 A
  if ((e = make_tmap_k_major(&wk.dzt_m, wk.dzt, H, M, 128)) != cudaSuccess) return e;   // GEMM2 A
  return make_tmap_k_major(&wk.xbt_m, wk.xbt, I, M, I % 96 == 0 ? 96 : 64);             // GEMM2 B
}

cudaError_t launch_mlp_grad(const MlpWork& wk, const float* X, const int* y, int S, const int* idx_in,
                            uint2 batch_key, unsigned long long k, const float* w, float* g, cudaStream_t s) {
  const int I = wk.sh.n_in, H = wk.sh.n_hid, O = wk.sh.n_out, M = wk.M;
  const long long off_b1 = (long long)H * I, off_W2 = off_b1 + H, off_b2 = off_W2 + (long long)O * H;
  CUtensorMap w1;                                             // W1 [H x I], the first H*I floats of w
  cudaError_t e = make_tmap_k_major(&w1, w, H, I, 64);
  if (e != cudaSuccess) return e;
  // the chain gather -> GEMM1 -> mid -> GEMM2 uses programmatic dependent launch: each kernel's
  // setup (GEMM: barriers, TMEM, tensor-map prefetch) overlaps its predecessor's tail
  if ((e = launch_pdl(k_mlp_gather, dim3(I / 32, M / 32), dim3(32, 8), 0, s, X, I, idx_in, batch_key, k, S, M,
                      wk.idx, wk.xb, wk.xbt)) != cudaSuccess)
    return e;
  if ((e = launch_gemm_tf32x3(wk.x_b, w1, wk.z1p, M, H, I, wk.splits, 64, s)) != cudaSuccess) return e;
  if ((e = launch_pdl(k_mlp_mid, dim3(M), dim3(H), 0, s, (const float*)wk.z1p, wk.splits, M, H, O, w, off_b1,
                      off_W2, off_b2, y, (const int*)wk.idx, wk.hbuf, wk.dz1, wk.dz2, wk.dzt)) != cudaSuccess)
    return e;
  // the batch reductions on the side stream, beside GEMM2 (which leaves SMs free)
  if ((e = cudaEventRecord(wk.fork, s)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(wk.side, wk.fork, 0)) != cudaSuccess) return e;
  const long long nred = (long long)H + (long long)O * H + O;
  k_mlp_reduce<<<(unsigned)((nred * 32 + 255) / 256), 256, 0, wk.side>>>(wk.hbuf, wk.dz1, wk.dz2, M, H, O, g, off_b1,
                                                                          off_W2, off_b2);
  // dW1 in 128 x 96 tiles (I = 3072: 4 x 32 = 128 CTAs, one wave)
  if ((e = launch_gemm_tf32x3(wk.dzt_m, wk.xbt_m, g, H, I, M, 1, I % 96 == 0 ? 96 : 64, s)) != cudaSuccess)
    return e;
  if ((e = cudaEventRecord(wk.join, wk.side)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(s, wk.join, 0)) != cudaSuccess) return e;
  return cudaGetLastError();
}

const void* mlp_module_anchor() { return (const void*)k_mlp_gather; }

}  // namespace adp
