// gemm.cu -- 3xTF32 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   C[M x N] (fp32) = A[M x K] . B[N x K]^T,   A, B row-major (K-major), fp32
//
// Used by the MLP minibatch gradient (config 3): Z1 = X_b W1^T and
// dW1 = dZ1^T X_b.  Accuracy ~fp32 via the 3xTF32 split:
//   A = A_hi + A_lo, B = B_hi + B_lo (hi = rna_tf32(x), lo = rna_tf32(x - hi)),
//   C ~= A_hi B_hi + A_hi B_lo + A_lo B_hi   (three tcgen05.mma into one TMEM accumulator).
//
// CTA = 128 threads, tile 128 x BN, k-block 32 fp32 (= one 128-byte swizzle atom).
// warp 0 / lane 0: TMA producer (cp.async.bulk.tensor, SWIZZLE_128B, 4 tiles per stage)
// warp 1 / lane 0: MMA issuer (tcgen05.mma.cta_group::1.kind::tf32, M=128, N=BN, K=8)
// all 4 warps    : epilogue (tcgen05.ld 32x32b -> registers -> global)
// Split-K: blockIdx.z takes a K range and writes its own partial plane.
#include <cuda.h>
#include "internal.h"

namespace adp {

namespace {

constexpr int kBM = 128, kBK = 32, kGemmThreads = 128;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// shared-memory matrix descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);       // start address (16-B units)
  d |= (uint64_t)1u << 16;                        // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024u >> 4) << 32;              // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1u << 46;                        // descriptor version (sm_100)
  d |= (uint64_t)2u << 61;                        // layout: SWIZZLE_128B
  return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = BN
__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; "
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
      ::"r"(tmem_d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_tf32x3(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
                  const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl,
                  float* __restrict__ C, int ldc, int kb_per_split, long long split_stride) {
  constexpr uint32_t kATile = kBM * 128, kBTile = BN * 128;
  constexpr uint32_t kStage = 2 * kATile + 2 * kBTile;
  extern __shared__ unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], accum;
  __shared__ uint32_t tmem_base_s;
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;    // SW128 needs 1024-B alignment
  unsigned char* sbase = smem_raw + (base - smem_u32(smem_raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * kBM;
  const int kb0 = blockIdx.z * kb_per_split;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&accum, 1);
    mbar_fence_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmAh) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmBh) : "memory");
  }
  if (warp == 0) {                                           // TMEM: 128 lanes x BN fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)), "r"((uint32_t)BN) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  if (warp == 0 && lane == 0) {
    // ------------------------------------------------------------ producer
    for (int kb = 0; kb < kb_per_split; ++kb) {
      const int s = kb % STAGES;
      const uint32_t use = (uint32_t)(kb / STAGES);
      if (kb >= STAGES) mbar_wait(&empty[s], (use - 1u) & 1u);
      unsigned char* st = sbase + (size_t)s * kStage;
      mbar_arrive_tx(&full[s], kStage);
      const int kc = (kb0 + kb) * kBK;
      tma_load_2d(st, &tmAh, kc, m0, &full[s]);
      tma_load_2d(st + kATile, &tmAl, kc, m0, &full[s]);
      tma_load_2d(st + 2 * kATile, &tmBh, kc, n0, &full[s]);
      tma_load_2d(st + 2 * kATile + kBTile, &tmBl, kc, n0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------------------------------------------------- MMA issue
    constexpr uint32_t idesc = tf32_idesc(kBM, BN);
    for (int kb = 0; kb < kb_per_split; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (uint32_t)(kb / STAGES) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t st = base + (uint32_t)s * kStage;
      const uint64_t ah = sw128_desc(st), al = sw128_desc(st + kATile);
      const uint64_t bh = sw128_desc(st + 2 * kATile), bl = sw128_desc(st + 2 * kATile + kBTile);
#pragma unroll
      for (int kk = 0; kk < kBK / 8; ++kk) {                 // K = 8 tf32 = 32 B per MMA
        const uint64_t o = (uint64_t)(kk * 32 >> 4);
        mma_tf32(tmem, ah + o, bh + o, idesc, (kb | kk) ? 1u : 0u);
        mma_tf32(tmem, ah + o, bl + o, idesc, 1u);
        mma_tf32(tmem, al + o, bh + o, idesc, 1u);
      }
      mma_commit(&empty[s]);                                // smem stage free when these complete
    }
    mma_commit(&accum);                                     // accumulator ready
  }
  __syncwarp();

  // ------------------------------------------------------------------ epilogue
  mbar_wait(&accum, 0u);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float* crow = C + (long long)blockIdx.z * split_stride + (long long)(m0 + warp * 32 + lane) * ldc + n0;
#pragma unroll 1
  for (int c = 0; c < BN / 32; ++c) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(c * 32);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
        "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
          "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    float4* dst = reinterpret_cast<float4*>(crow + c * 32);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      dst[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                           __uint_as_float(v[4 * q + 3]));
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)BN) : "memory");
  }
}

// hi = rna_tf32(x), lo = rna_tf32(x - hi)
__global__ void k_split_tf32(const float* __restrict__ x, float* __restrict__ hi, float* __restrict__ lo,
                             long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float v = x[i];
    uint32_t h, l;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
    const float r = v - __uint_as_float(h);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
    hi[i] = __uint_as_float(h);
    lo[i] = __uint_as_float(l);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

// 2-D fp32 tensor map over a row-major [rows x cols] matrix, box {32 cols, box_rows}, SWIZZLE_128B
cudaError_t make_tmap_k_major(CUtensorMap* tm, const float* ptr, long long rows, long long cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)cols * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), gdim, gstride, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

__global__ void k_sum_planes(const float* __restrict__ src, float* __restrict__ dst, int planes, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float acc = 0.0f;
    for (int p = 0; p < planes; ++p) acc += src[(long long)p * n + i];
    dst[i] = acc;
  }
}

cudaError_t launch_sum_planes(const float* src, float* dst, int planes, long long n, cudaStream_t s) {
  k_sum_planes<<<592, 256, 0, s>>>(src, dst, planes, n);
  return cudaGetLastError();
}

cudaError_t launch_split_tf32(const float* x, float* hi, float* lo, long long n, cudaStream_t s) {
  k_split_tf32<<<592, 256, 0, s>>>(x, hi, lo, n);
  return cudaGetLastError();
}

// C (+ z * split_stride) = A . B^T over K range of split z; M % 128 == 0, N % BN == 0, K % (32 * splits) == 0
cudaError_t launch_gemm_tf32x3(const GemmOperands& op, float* C, int M, int N, int K, int splits, int bn,
                               cudaStream_t s) {
  if (M % kBM || K % (kBK * splits) || (bn != 128 && bn != 256) || N % bn) return cudaErrorInvalidValue;
  const int kbps = K / kBK / splits;
  const long long sstride = (long long)M * N;
  dim3 grid(N / bn, M / kBM, splits);
  if (bn == 128) {
    constexpr int S = 3;                                    // 3 x 64 KB stages
    const size_t smem = (size_t)S * (2 * kBM * 128 + 2 * 128 * 128) + 1024;
    cudaFuncSetAttribute(k_gemm_tf32x3<128, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_gemm_tf32x3<128, S><<<grid, kGemmThreads, smem, s>>>(op.Ah, op.Al, op.Bh, op.Bl, C, N, kbps, sstride);
  } else {
    constexpr int S = 2;                                    // 2 x 96 KB stages
    const size_t smem = (size_t)S * (2 * kBM * 128 + 2 * 256 * 128) + 1024;
    cudaFuncSetAttribute(k_gemm_tf32x3<256, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_gemm_tf32x3<256, S><<<grid, kGemmThreads, smem, s>>>(op.Ah, op.Al, op.Bh, op.Bl, C, N, kbps, sstride);
  }
  return cudaGetLastError();
}

const void* gemm_module_anchor() { return (const void*)k_sum_planes; }

}  // namespace adp
