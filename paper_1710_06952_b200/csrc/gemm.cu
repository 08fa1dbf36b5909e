// gemm.cu -- 3xTF32 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   C[M x N] (fp32) = A[M x K] . B[N x K]^T,   A, B row-major (K-major), fp32
//
// Used by the MLP minibatch gradient (config 3): Z1 = X_b W1^T and
// dW1 = dZ1^T X_b.  Accuracy ~fp32 via the 3xTF32 split:
//   A = A_hi + A_lo, B = B_hi + B_lo (hi = rna_tf32(x), lo = rna_tf32(x - hi)),
//   C ~= A_hi B_hi + A_hi B_lo + A_lo B_hi   (three tcgen05.mma into one TMEM accumulator).
// The operands are read ONCE, as fp32: TMA brings a 128-byte-swizzled fp32 tile
// into shared memory, which serves as hi as is (the tensor core drops the low 13
// mantissa bits: hi = trunc_tf32(x)), and the CTA writes lo = rna_tf32(x - hi)
// into a second tile of the same swizzled layout -- so no hi/lo planes are ever
// written to HBM (round 1 pre-split W1, X_b and dZ1^T in separate passes: 3 extra
// launches and ~19 MB per gradient).
//
// CTA = 256 threads, tile 128 x BN (BN = 64 / 96 / 128), k-block 32 fp32 (= one
// 128-byte swizzle atom), STAGES k-blocks in flight.  Per k-block:
//   thread 0     : TMA producer (refills the stage the previous k-block used once
//                  its MMAs have drained it: one k-block of slack)
//   all threads  : write lo of the staged tiles, fence.proxy.async, barrier
//   thread 32    : MMA issuer (tcgen05.mma.cta_group::1.kind::tf32, M=128, N=BN, K=8)
// then all 8 warps run the epilogue (tcgen05.ld 32x32b -> registers -> global).
// Split-K: blockIdx.z takes a K range and writes its own partial plane.
#include <cuda.h>
#include "internal.h"

namespace adp {

namespace {

constexpr int kBM = 128, kBK = 32, kGemmThreads = 256;   // 8 warps: all split, warps w and w+4 share TMEM lanes

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

// The tensor core reads an fp32 word as tf32 by dropping its low 13 mantissa
// bits, so the staged fp32 tile already IS hi = trunc_tf32(x); only the
// remainder lo = rna_tf32(x - hi) (x - hi is exact) needs a tile of its own.
// The dropped lo*lo term is below 2^-20 |a b| (tests/test_gemm_gpu.py: error
// relative to sum |a||b| < 2e-6, against ~1e-3 for one TF32 product).
__device__ __forceinline__ float tf32_lo(float v) {
  const float r = v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
  uint32_t l;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
  return __uint_as_float(l);
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_tf32x3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  float* __restrict__ C, int ldc, int kb_per_split, long long split_stride) {
  constexpr uint32_t kATile = kBM * 128, kBTile = BN * 128;  // fp32 tiles (the hi halves after the split)
  constexpr uint32_t kStage = 2 * kATile + 2 * kBTile;       // [A32|hi][A lo][B32|hi][B lo]
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
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  constexpr uint32_t kTmemCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;   // power of 2
  if (warp == 0) {                                           // TMEM: 128 lanes x BN fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)), "r"(kTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base_s;

  auto load = [&](int kb) {                                  // thread 0: TMA fp32 A and B tiles of k-block kb
    const int s = kb % STAGES;
    unsigned char* st = sbase + (size_t)s * kStage;
    mbar_arrive_tx(&full[s], kATile + kBTile);
    const int kc = (kb0 + kb) * kBK;
    tma_load_2d(st, &tmA, kc, m0, &full[s]);
    tma_load_2d(st + 2 * kATile, &tmB, kc, n0, &full[s]);
  };
  pdl_wait();                                                // operands written by the predecessor
  pdl_trigger();
  if (threadIdx.x == 0)
    for (int kb = 0; kb < STAGES && kb < kb_per_split; ++kb) load(kb);

  constexpr uint32_t idesc = tf32_idesc(kBM, BN);
  for (int kb = 0; kb < kb_per_split; ++kb) {
    const int s = kb % STAGES;
    mbar_wait(&full[s], (uint32_t)(kb / STAGES) & 1u);
    // split the staged fp32 tiles: hi in place, lo into the stage's lo tiles
    float4* a32 = reinterpret_cast<float4*>(sbase + (size_t)s * kStage);
    float4* alo = reinterpret_cast<float4*>(sbase + (size_t)s * kStage + kATile);
    float4* b32 = reinterpret_cast<float4*>(sbase + (size_t)s * kStage + 2 * kATile);
    float4* blo = reinterpret_cast<float4*>(sbase + (size_t)s * kStage + 2 * kATile + kBTile);
#pragma unroll
    for (int q = threadIdx.x; q < (int)(kATile / 16); q += kGemmThreads) {
      const float4 v = a32[q];
      alo[q] = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
    }
#pragma unroll
    for (int q = threadIdx.x; q < (int)(kBTile / 16); q += kGemmThreads) {
      const float4 v = b32[q];
      blo[q] = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor-core reads
    __syncthreads();
    if (threadIdx.x == 32) {
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
      mma_commit(&empty[s]);                                // stage s free when these complete
      if (kb == kb_per_split - 1) mma_commit(&accum);       // accumulator ready
    }
    // refill the stage the previous k-block used, once its MMAs drained it
    if (threadIdx.x == 0 && kb >= 1 && kb - 1 + STAGES < kb_per_split) {
      const int sp = (kb - 1) % STAGES;
      mbar_wait(&empty[sp], (uint32_t)((kb - 1) / STAGES) & 1u);
      load(kb - 1 + STAGES);
    }
  }

  // ------------------------------------------------------------------ epilogue
  mbar_wait(&accum, 0u);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp w reads TMEM lanes 32 (w % 4) .. + 31 (its quadrant); warps w and w + 4 take alternate
  // 32-column chunks
  const int quad = warp & 3;
  float* crow = C + (long long)blockIdx.z * split_stride + (long long)(m0 + quad * 32 + lane) * ldc + n0;
#pragma unroll 1
  for (int c = warp >> 2; c < BN / 32; c += 2) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(c * 32);
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
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

// C (+ z * split_stride) = A . B^T over K range of split z; M % 128 == 0, N % BN == 0, K % (32 * splits) == 0.
cudaError_t launch_gemm_tf32x3(const CUtensorMap& A, const CUtensorMap& B, float* C, int M, int N, int K, int splits,
                               int bn, cudaStream_t s) {
  if (M % kBM || K % (kBK * splits) || (bn != 64 && bn != 96 && bn != 128) || N % bn) return cudaErrorInvalidValue;
  const int kbps = K / kBK / splits;
  const long long sstride = (long long)M * N;
  dim3 grid(N / bn, M / kBM, splits);
  if (bn == 128) {
    constexpr int S = 3;                                    // 3 x 64 KB stages
    const size_t smem = (size_t)S * (2 * kBM * 128 + 2 * 128 * 128) + 1024;
    cudaFuncSetAttribute(k_gemm_tf32x3<128, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return launch_pdl(k_gemm_tf32x3<128, S>, grid, dim3(kGemmThreads), smem, s, A, B, C, N, kbps, sstride);
  } else if (bn == 96) {
    constexpr int S = 3;                                    // 3 x 56 KB stages: 128 x 96 tiles
    const size_t smem = (size_t)S * (2 * kBM * 128 + 2 * 96 * 128) + 1024;
    cudaFuncSetAttribute(k_gemm_tf32x3<96, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return launch_pdl(k_gemm_tf32x3<96, S>, grid, dim3(kGemmThreads), smem, s, A, B, C, N, kbps, sstride);
  } else {
    constexpr int S = 3;                                    // 3 x 48 KB stages (config-3 replay A/B: 2 / 3 / 4
                                                            // stages 30.3-31.3k / 31.1k / 29.1k updates/s)
    const size_t smem = (size_t)S * (2 * kBM * 128 + 2 * 64 * 128) + 1024;
    cudaFuncSetAttribute(k_gemm_tf32x3<64, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return launch_pdl(k_gemm_tf32x3<64, S>, grid, dim3(kGemmThreads), smem, s, A, B, C, N, kbps, sstride);
  }
  return cudaGetLastError();
}

const void* gemm_module_anchor() { return (const void*)k_sum_planes; }

}  // namespace adp
