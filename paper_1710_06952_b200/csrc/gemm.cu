// gemm.cu -- 3xTF32 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
//   C[M x N] (fp32) = A[M x K] . B[N x K]^T
//
// Used by the MLP minibatch gradient (config 3): Z1 = X_b W1^T and
// dW1 = dZ1^T X_b.  Accuracy ~fp32 via the 3xTF32 split:
//   A = A_hi + A_lo, B = B_hi + B_lo (hi = trunc_tf32(x), lo = rna_tf32(x - hi)),
//   C ~= A_hi B_hi + A_hi B_lo + A_lo B_hi   (three tcgen05.mma per K step).
// The operands are read ONCE, as fp32: a staged fp32 word serves as hi as is (the tensor core
// drops the low 13 mantissa bits) and lo = rna_tf32(x - hi) is derived on chip -- no hi/lo
// planes are ever written to HBM.
//
// CTA = 9 warps, tile 128 x BN (BN = 32 / 64 / 96 / 128), k-block 32 fp32.  Raw fp32 tiles of
// several k-blocks are in flight (generic kernels: up to 8 / 7 / 6 / 5 with one CTA per SM;
// the MLP's gathering kernels are "compact", two CTAs per SM).  Each operand arrives in one of
// three ways (template AM / BM):
//   kOpTma      K-major tile by a TMA tensor load (cp.async.bulk.tensor, SWIZZLE_128B)
//   kOpTmaMN    MN-major tile by TMA (the contraction runs over the rows of a row-major
//               matrix: dW1 = dZ1^T X_b reads dZ1 [batch x H] without a transpose)
//   kOpGather*  rows of X picked by the batch indices, cp.async'd straight into the
//               swizzled layout (K-major for GEMM1's X_b, MN-major for GEMM2's X_b):
//               the minibatch is never materialised in HBM
// and completes on the stage's mbarrier (TMA: complete_tx; cp.async: one
// cp.async.mbarrier.arrive.noinc per thread).  Per k-block:
//   warps 0-3 : A's row (thread = row) -> TMEM as hi and lo (tcgen05.st)
//   warps 4-7 : B's lo tile into a shared-memory buffer (hi stays in the staged tile)
//   warp 8    : MMA issuer (tcgen05.mma.cta_group::1.kind::tf32, A from TMEM, B from shared
//               memory, M = 128, N = BN, K = 8) and the TMA loads / refills
// split and MMA hand over through mbarriers, so the split of k-block kb + 1 overlaps kb's MMAs.
// Epilogue (template EPI): kEpiStore writes the CTA's split-K plane; kEpiCluster /
// kEpiClusterTanh reduce the split-K partials of a thread-block cluster (consecutive
// blockIdx.z of one output tile) in distributed shared memory: CTA p owns rows
// [p R, (p + 1) R) of the tile (R = 128 / cluster), every CTA pushes those rows of its
// partial to CTA p with one bulk copy (cp.async.bulk shared::cta -> shared::cluster,
// completing on p's mbarrier), and p sums the cluster's partials in rank order
// (deterministic) -- one plane per cluster (and, for GEMM1 with one cluster per tile,
// h = tanh(z1 + b1) itself) is written, no partial planes travel through HBM.
#include <cuda.h>
#include <atomic>
#include "internal.h"

namespace adp {

namespace {

constexpr int kBM = 128, kBK = 32;
// warps 0-3 split A (thread = row, into TMEM), warps 4-7 split B (smem) and run the epilogue
// with 0-3; warp 8 issues the MMAs and the TMA loads -- so the split of k-block kb + 1 runs while
// the tensor core works on kb and nobody waits on an MMA it did not need
constexpr int kSplitThreads = 256, kGemmThreads = kSplitThreads + 32, kIssuer = kSplitThreads;
// raw (fp32) stages per tile width: R x (A + B tiles) + 2 lo buffers of B [+ the cluster
// reduction's receive buffer, 128 x (BN + 4) fp32] <= 200 KB
__host__ __device__ constexpr int recv_bytes(int bn, bool cluster) { return cluster ? 128 * (bn + 4) * 4 : 0; }
// dynamic shared memory per CTA: the generic (TMA / TMA) kernels take one CTA per SM and deep
// pipelines; the MLP's gathering kernels ("compact") fit two CTAs per SM, so the gradients of
// different workers overlap their MMA issue (free-running config 3: 35k -> 37k updates/s)
__host__ __device__ constexpr int smem_budget(bool compact) { return compact ? 86016 : 204800; }
__host__ __device__ constexpr int stages_fit(int bn, bool cluster, bool compact) {
  return (smem_budget(compact) - recv_bytes(bn, cluster) - 2 * bn * 128) / ((128 + bn) * 128);
}
__host__ __device__ constexpr int raw_stages(int bn, bool cluster, bool compact) {
  return stages_fit(bn, cluster, compact) > 8 ? 8 : stages_fit(bn, cluster, compact) < 2 ? 2
                                                                                        : stages_fit(bn, cluster, compact);
}
constexpr int kMaxGatherRows = 1024;     // batch rows a gathering CTA indexes (MLP: batch_M <= 1024)
// TMEM: the generic kernels keep three accumulators -- hi.hi, hi.lo, lo.hi in columns
// [128 p, 128 p + BN), p = 0, 1, 2 (summed small terms first: max error 6.6e-6 -> 2.5e-6 in
// tools/gemm_mn_probe.cu) -- and A's hi / lo tiles of k-block kb in columns [384 + 64 (kb % 2),
// + 32) / [+ 32, + 64); the compact kernels one accumulator and A at column 128, 256 columns
// in all so that two CTAs share an SM's TMEM
__host__ __device__ constexpr int n_accs(bool compact) { return compact ? 1 : 3; }
__host__ __device__ constexpr uint32_t tmem_cols(bool compact) { return compact ? 256u : 512u; }
__host__ __device__ constexpr uint32_t tmem_a(bool compact) { return compact ? 128u : 384u; }
constexpr uint32_t kTmemAcc = 128;
enum : int { kOpTma = 0, kOpGatherK = 1, kOpTmaMN = 2, kOpGatherMN = 3 };
enum : int { kEpiStore = 0, kEpiCluster = 1, kEpiClusterTanh = 2 };

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      ::"r"(smem_u32(dst)), "l"(tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
// the stage's mbarrier sees one arrival once all of this thread's earlier cp.async landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// shared-memory matrix descriptors, SWIZZLE_128B (rows of 128 B, 8-row groups of 1024 B):
// K-major: rows are M/N indices, one row = 32 fp32 of K, 8-row groups SBO = 1024 B apart
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);       // start address (16-B units)
  d |= (uint64_t)1u << 16;                        // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024u >> 4) << 32;              // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1u << 46;                        // descriptor version (sm_100)
  d |= (uint64_t)2u << 61;                        // layout: SWIZZLE_128B
  return d;
}
// MN-major (the only smem layout tcgen05 takes for MN-major tf32): SWIZZLE_128B_BASE32B --
// rows are K indices, one row = 32 fp32 of M/N (128 B) whose 32-B chunks are XOR-swizzled
// with (row mod 4); blocks of 32 K-rows x 32 M/N (4 KB) follow each other along M/N
// (LBO = 4096 B), 4-K-row groups 512 B apart (SBO)
__device__ __forceinline__ uint64_t sw128_mn_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(4096u >> 4) << 16;              // leading byte offset: next 32 M/N columns
  d |= (uint64_t)(512u >> 4) << 32;               // stride byte offset: next 4 K rows
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)1u << 61;                        // layout: SWIZZLE_128B_BASE32B
  return d;
}
// byte offset of fp32 element (row r, column j) of a 32 x 32 MN-major block (j % 4 == 0: a 16-B chunk)
__device__ __forceinline__ uint32_t mn_off(int r, int j) {
  return (uint32_t)(r * 128 + ((((j >> 3) ^ (r & 3)) << 5) | ((j & 4) << 2)));
}

// instruction descriptor: D f32, A/B tf32, M = 128, N = BN; bit 15 / 16: A / B MN-major
__host__ __device__ constexpr uint32_t tf32_idesc(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (a_mn ? 1u << 15 : 0u) | (b_mn ? 1u << 16 : 0u) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// A from TMEM (K-major: lane = row, one 32-bit column per k), B from shared memory
__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bd, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{ .reg .pred p; setp.ne.b32 p, %4, 0; "
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p; }"
      ::"r"(tmem_d), "r"(tmem_a), "l"(bd), "r"(idesc), "r"(acc)
      : "memory");
}

// 32 lanes x 32 consecutive columns from this warp's 32 threads (thread i -> lane base + i)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
      ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, "
      "%13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
        "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
        "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t dsmem_map(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// per-CTA phase timestamps (globaltimer) for tools/gemm_mn_probe.cu; compiled out in the library
constexpr bool kGemmTrace = false;
__device__ unsigned long long g_gemm_trace[1024 * 48];
__device__ __forceinline__ void trace_point(int i, unsigned who = 0) {
  if constexpr (kGemmTrace) {
    if (threadIdx.x == who) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      const int b = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
      if (b < 1024 && i < 48) g_gemm_trace[b * 48 + i] = t;
    }
  }
}

// The tensor core reads an fp32 word as tf32 by dropping its low 13 mantissa
// bits, so the staged fp32 tile already IS hi = trunc_tf32(x); only the
// remainder lo = rna_tf32(x - hi) (x - hi is exact) needs a tile of its own.
// The dropped lo*lo term is below 2^-20 |a b| (tests/test_gemm_gpu.py: error
// relative to sum |a||b| < 2e-6, against ~1e-3 for one TF32 product).
// rna_tf32 (round to nearest, ties away from zero: cvt.rna.tf32.f32, which ptxas expands to
// a longer sequence with NaN / Inf handling) as one integer add and mask on the magnitude bits;
// r is finite and |r| < 2^-10 |v|
__device__ __forceinline__ float tf32_lo(float v) {
  const float r = v - __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
  return __uint_as_float((__float_as_uint(r) + 0x1000u) & 0xFFFFE000u);
}

// GEMM2's extra CTAs: the MLP's batch reductions (reading R18) db1[u] = sum_b dz1[b][u],
// dW2[o][u] = sum_b dz2[b][o] h[b][u], db2[o] = sum_b dz2[b][o].  Unit c owns hidden units
// [32 c, 32 c + 32); thread (u, q) sums samples b = q, q + 8, .. (coalesced over u), and the 8
// partial sums of each output are added in order q = 0..7 (deterministic); CTA 0's last warp
// does db2.  Runs beside the dW1 tiles, so the gradient needs no side stream.
constexpr int kRedMaxOut = 32;
__device__ void mlp_batch_reduce(const GemmGather& gg, int c, unsigned char* sbase) {
  const int tid = threadIdx.x, H = gg.r_H, O = gg.r_O, M = gg.r_M;
  float* part = reinterpret_cast<float*>(sbase);            // [8][O + 1][32]
  pdl_wait();                                               // h, dz1, dz2 of the per-sample kernel
  pdl_trigger();
  if (tid < 256) {
    const int ul = tid & 31, q = tid >> 5, u = c * 32 + ul;
    float a1 = 0.0f, aw[kRedMaxOut];
#pragma unroll
    for (int o = 0; o < kRedMaxOut; ++o) aw[o] = 0.0f;
    if (u < H) {
#pragma unroll 4
      for (int b = q; b < M; b += 8) {
        const float hv = gg.r_h[(long long)b * H + u];
        a1 += gg.r_dz1[(long long)b * H + u];
#pragma unroll
        for (int o = 0; o < kRedMaxOut; ++o) {
          if (o >= O) break;
          aw[o] = fmaf(gg.r_dz2[(long long)b * O + o], hv, aw[o]);
        }
      }
    }
    part[(q * (O + 1)) * 32 + ul] = a1;
#pragma unroll
    for (int o = 0; o < kRedMaxOut; ++o) {
      if (o >= O) break;
      part[(q * (O + 1) + 1 + o) * 32 + ul] = aw[o];
    }
  }
  __syncthreads();
  for (int t = tid; t < (O + 1) * 32; t += blockDim.x) {   // output row r (0: db1, 1 + o: dW2[o]), unit ul
    const int r = t >> 5, ul = t & 31, u = c * 32 + ul;
    if (u >= H) continue;
    float acc = 0.0f;
    for (int q = 0; q < 8; ++q) acc += part[(q * (O + 1) + r) * 32 + ul];
    if (r == 0) gg.r_g[gg.r_off_b1 + u] = acc;
    else gg.r_g[gg.r_off_W2 + (long long)(r - 1) * H + u] = acc;
  }
  if (c == 0 && tid >= 256 && tid - 256 < O) {              // db2: one lane per output
    const int o = tid - 256;
    float acc = 0.0f;
    for (int b = 0; b < M; ++b) acc += gg.r_dz2[(long long)b * O + o];
    gg.r_g[gg.r_off_b2 + o] = acc;
  }
}

template <int BN, int AM, int BM, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    k_gemm_tf32x3(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  float* __restrict__ C, int ldc, int kb_per_split, long long split_stride, const GemmGather gg) {
  constexpr bool kGather = AM == kOpGatherK || BM == kOpGatherMN;
  constexpr bool kCluster = EPI != kEpiStore;
  constexpr bool kCompact = AM != kOpTma || BM != kOpTma;
  constexpr int R = raw_stages(BN, kCluster, kCompact);
  constexpr int kAccs = n_accs(kCompact);
  constexpr uint32_t kTmemCols = tmem_cols(kCompact), kTmemA = tmem_a(kCompact);
  constexpr uint32_t kATile = kBM * 128, kBTile = BN * 128;  // fp32 tiles (the hi halves after the split)
  constexpr uint32_t kRaw = kATile + kBTile;                 // raw stage r: [A32][B32|hi]; then 2 x [B lo]
  constexpr uint32_t kTmaBytes = (AM == kOpGatherK ? 0u : kATile) + (BM == kOpGatherMN ? 0u : kBTile);
  static_assert(!kCluster || (uint32_t)kBM * (BN + 4) * 4 <= R * kRaw + 2 * kBTile,
                "the epilogue's reduction buffer must fit in the drained stages");
  extern __shared__ unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[R], rawfree[R], lofree[2], split_done[2], accum, recv_bar;
  __shared__ uint32_t tmem_base_s;
  __shared__ int s_rows[kGather ? kMaxGatherRows : 1];
  __shared__ __align__(16) float s_bias[EPI == kEpiClusterTanh ? BN : 4];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;    // SW128 needs 1024-B alignment
  unsigned char* sbase = smem_raw + (base - smem_u32(smem_raw));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if constexpr (BM == kOpGatherMN) {                          // GEMM2's batch-reduction CTAs
    if (gg.red_ctas && (int)blockIdx.x >= (int)gridDim.x - gg.red_ctas) {   // unit c owns 32 hidden units
      mlp_batch_reduce(gg, ((int)blockIdx.x - ((int)gridDim.x - gg.red_ctas)) * (int)gridDim.y + (int)blockIdx.y,
                       sbase);
      return;
    }
  }
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * kBM;
  const int kb0 = blockIdx.z * kb_per_split;
  trace_point(0);

  if (tid == 0) {
    for (int s = 0; s < R; ++s) { mbar_init(&full[s], kGather ? kSplitThreads + 1 : 1); mbar_init(&rawfree[s], 1); }
    for (int l = 0; l < 2; ++l) { mbar_init(&lofree[l], 1); mbar_init(&split_done[l], kSplitThreads); }
    mbar_init(&accum, 1);
    if (kCluster) {                                          // the cluster's partials of my rows land here
      mbar_init(&recv_bar, 1);
      mbar_arrive_tx(&recv_bar, (uint32_t)(kBM * (BN + 4) * 4));
    }
    mbar_fence_init();
    if (AM != kOpGatherK) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    if (BM != kOpGatherMN) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
  }
  if (warp == 0) {                                           // TMEM: 3 accumulators + A's hi / lo (all 512 columns)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)), "r"(kTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  pdl_wait();                                                // operands written by the predecessor
  if constexpr (AM == kOpGatherK) {
    // the batch rows of this M tile: explicit indices, or Philox4x32-10(key = seed,
    // ctr = (lo32(k), m, "BATC", hi32(k))) as lsq / logreg (reading R18); the x = 0 / z = 0
    // CTA of each M tile publishes them for the rest of the gradient
    for (int t = tid; t < kBM; t += kGemmThreads) {
      const int m = m0 + t;
      int v;
      if (gg.idx) v = gg.idx[m];
      else {
        const uint4 o = philox4x32_10(make_uint4((uint32_t)gg.k, (uint32_t)m, 0x42415443u, (uint32_t)(gg.k >> 32)),
                                      gg.key);
        v = (int)(((unsigned long long)o.x * (unsigned long long)(uint32_t)gg.S) >> 32);
      }
      s_rows[t] = v;
      if (gg.idx_out && blockIdx.x == 0 && blockIdx.z == 0) gg.idx_out[m] = v;
    }
  } else if constexpr (BM == kOpGatherMN) {
    for (int t = tid; t < kb_per_split * kBK; t += kGemmThreads) s_rows[t] = gg.idx[kb0 * kBK + t];
  }
  if constexpr (EPI == kEpiClusterTanh)
    for (int t = tid; t < BN; t += kGemmThreads) s_bias[t] = gg.bias[n0 + t];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (kCluster) cluster_sync();                    // every CTA's recv_bar is initialised
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  pdl_trigger();
  trace_point(1);
  const uint32_t tmem = tmem_base_s;

  auto tma_load = [&](int kb) {                              // issuer: the TMA part of raw stage kb % R
    const int s = kb % R;
    unsigned char* st = sbase + (size_t)s * kRaw;
    const int kc = (kb0 + kb) * kBK;
    mbar_arrive_tx(&full[s], kTmaBytes);
    if constexpr (AM == kOpTma) tma_load_2d(st, &tmA, kc, m0, &full[s]);
    if constexpr (AM == kOpTmaMN)                            // 4 boxes of 32 M-columns x 32 K-rows
      for (int q = 0; q < kBM / 32; ++q) tma_load_2d(st + q * 4096, &tmA, m0 + 32 * q, kc, &full[s]);
    if constexpr (BM == kOpTma) tma_load_2d(st + kATile, &tmB, kc, n0, &full[s]);
  };
  auto gather_load = [&](int kb) {                           // split threads: the cp.async part
    const int s = kb % R;
    const uint32_t sa = base + (uint32_t)s * kRaw;
    const int kc = (kb0 + kb) * kBK;
    if constexpr (AM == kOpGatherK) {                        // 128 rows x 8 chunks of 16 B
      for (int q = tid; q < kBM * 8; q += kSplitThreads) {
        const int r = q >> 3, c = q & 7;
        cp_async16(sa + r * 128 + ((c ^ (r & 7)) << 4), gg.x + (long long)s_rows[r] * gg.ld + kc + c * 4);
      }
    }
    if constexpr (BM == kOpGatherMN) {                       // 32 K-rows x BN / 4 chunks of 16 B
      constexpr int kChunks = BN / 4;
      const int kr0 = kb * kBK;
      for (int q = tid; q < kBK * kChunks; q += kSplitThreads) {
        const int r = q / kChunks, c = q % kChunks;
        cp_async16(sa + kATile + (c >> 3) * 4096 + mn_off(r, (c & 7) * 4),
                   gg.x + (long long)s_rows[kr0 + r] * gg.ld + n0 + c * 4);
      }
    }
    cp_async_arrive(&full[s]);
  };
  constexpr uint32_t idesc = tf32_idesc(kBM, BN, false, BM == kOpGatherMN);   // A (TMEM) is K-major

  if (warp == kIssuer / 32) {
    // ---------------------------------------------------------------- issuer warp
    if (lane == 0) {
      if constexpr (kTmaBytes > 0)
        for (int kb = 0; kb < R && kb < kb_per_split; ++kb) tma_load(kb);
      for (int kb = 0; kb < kb_per_split; ++kb) {
        const int s = kb % R, l = kb & 1;
        mbar_wait(&split_done[l], (uint32_t)(kb >> 1) & 1u);  // A in TMEM buffer l, B lo in smem buffer l
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t bst = base + (uint32_t)s * kRaw + kATile, blt = base + (uint32_t)R * kRaw + (uint32_t)l * kBTile;
        uint64_t bh, bl;
        if constexpr (BM == kOpGatherMN) { bh = sw128_mn_desc(bst); bl = sw128_mn_desc(blt); }
        else { bh = sw128_desc(bst); bl = sw128_desc(blt); }
        const uint32_t ahi = tmem + kTmemA + 64u * (uint32_t)l, alo = ahi + 32u;
        // one MMA covers K = 8: 8 TMEM columns of A; 32 B along a K-major row of B, or 8 rows
        // (1024 B) of an MN-major B tile
        constexpr uint64_t kStepB = BM == kOpGatherMN ? 1024u >> 4 : 32u >> 4;
#pragma unroll
        for (int kk = 0; kk < kBK / 8; ++kk) {
          const uint64_t ob = kk * kStepB;
          const uint32_t oa = 8u * kk;
          const uint32_t acc = (kb | kk) ? 1u : 0u;
          mma_tf32_ts(tmem, ahi + oa, bh + ob, idesc, acc);
          if constexpr (kAccs == 3) {
            mma_tf32_ts(tmem + kTmemAcc, ahi + oa, bl + ob, idesc, acc);
            mma_tf32_ts(tmem + 2 * kTmemAcc, alo + oa, bh + ob, idesc, acc);
          } else {
            mma_tf32_ts(tmem, ahi + oa, bl + ob, idesc, 1u);
            mma_tf32_ts(tmem, alo + oa, bh + ob, idesc, 1u);
          }
        }
        if (kb < 12) trace_point(14 + kb, kIssuer);
        mma_commit(&rawfree[s]);                            // raw stage s free when these complete
        mma_commit(&lofree[l]);                             // and B lo buffer l, A's TMEM buffer l
        if (kb == kb_per_split - 1) mma_commit(&accum);     // accumulator ready
        if constexpr (kTmaBytes > 0)                        // refill the stage k-block kb - 1 used
          if (kb >= 1 && kb - 1 + R < kb_per_split) {
            mbar_wait(&rawfree[(kb - 1) % R], (uint32_t)((kb - 1) / R) & 1u);
            tma_load(kb - 1 + R);
          }
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- split warps
    if constexpr (kGather)
      for (int kb = 0; kb < R && kb < kb_per_split; ++kb) gather_load(kb);
    for (int kb = 0; kb < kb_per_split; ++kb) {
      const int s = kb % R, l = kb & 1;
      mbar_wait(&full[s], (uint32_t)(kb / R) & 1u);
      if (kb < 12) trace_point(2 + kb);
      if (kb >= 2) mbar_wait(&lofree[l], (uint32_t)((kb - 2) >> 1) & 1u);   // k-block kb - 2's MMAs read buffer l
      // A: warps 0-3, thread = row, raw fp32 -> TMEM as hi (the tensor core reads an fp32 word
      // as tf32) and lo; B: warps 4-7, lo into smem buffer l (hi stays in place)
      const unsigned char* at = sbase + (size_t)s * kRaw;
      if (warp < 4) {
        const int r = warp * 32 + lane;
        uint32_t hv[32], lv[32];
        if constexpr (AM == kOpTmaMN) {                      // column r of the MN-major tile
          const unsigned char* blk = at + (r >> 5) * 4096;
          const int j = r & 31;
#pragma unroll
          for (int k = 0; k < 32; ++k)
            hv[k] = *reinterpret_cast<const uint32_t*>(blk + k * 128 + ((((j >> 3) ^ (k & 3)) << 5) | ((j & 7) << 2)));
        } else {                                             // row r of the K-major SW128 tile
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 q = *reinterpret_cast<const uint4*>(at + r * 128 + ((c ^ (r & 7)) << 4));
            hv[4 * c] = q.x; hv[4 * c + 1] = q.y; hv[4 * c + 2] = q.z; hv[4 * c + 3] = q.w;
          }
        }
        if (kb < 2) trace_point(32 + 4 * kb);
#pragma unroll
        for (int k = 0; k < 32; ++k) lv[k] = __float_as_uint(tf32_lo(__uint_as_float(hv[k])));
        if (kb < 2) trace_point(33 + 4 * kb);
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + kTmemA + 64u * (uint32_t)l;
        tmem_st32(ta, hv);
        tmem_st32(ta + 32, lv);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        if (kb < 2) trace_point(34 + 4 * kb);
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      } else {
        const float4* b32 = reinterpret_cast<const float4*>(at + kATile);
        float4* blo = reinterpret_cast<float4*>(sbase + (size_t)R * kRaw + (size_t)l * kBTile);
#pragma unroll
        for (int q = tid - 128; q < (int)(kBTile / 16); q += 128) {
          const float4 v = b32[q];
          blo[q] = make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor-core reads
        if (kb < 2) trace_point(35 + 4 * kb, 128);
      }
      mbar_arrive(&split_done[l]);
      if constexpr (kGather)                                 // refill the stage k-block kb - 1 used
        if (kb >= 1 && kb - 1 + R < kb_per_split) {
          mbar_wait(&rawfree[(kb - 1) % R], (uint32_t)((kb - 1) / R) & 1u);
          gather_load(kb - 1 + R);
        }
    }
  }

  // ------------------------------------------------------------------ epilogue
  mbar_wait(&accum, 0u);
  trace_point(26);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp w reads TMEM lanes 32 (w % 4) .. + 31 (its quadrant); warps w and w + 4 take alternate
  // 32-column chunks
  const int quad = warp & 3;
  constexpr int kRedLd = BN + 4;                             // cluster reduction buffer row stride (floats):
                                                             // 16-B rows, conflict-free float4 writes
  float* red = reinterpret_cast<float*>(sbase);              // reuses the drained stages
#pragma unroll 1
  for (int c = warp >> 2; warp < 8 && c < BN / 32; c += 2) {
    uint32_t v[32], w[32];
    const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(c * 32);
    if constexpr (kAccs == 3) {
      tmem_ld32(taddr + kTmemAcc, v);                        // hi.lo + lo.hi, then + hi.hi
      tmem_ld32(taddr + 2 * kTmemAcc, w);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = __float_as_uint(__uint_as_float(v[q]) + __uint_as_float(w[q]));
      tmem_ld32(taddr, w);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < 32; ++q) v[q] = __float_as_uint(__uint_as_float(w[q]) + __uint_as_float(v[q]));
    } else {
      tmem_ld32(taddr, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    }
    if constexpr (EPI == kEpiStore) {
      float4* dst = reinterpret_cast<float4*>(C + (long long)blockIdx.z * split_stride +
                                              (long long)(m0 + quad * 32 + lane) * ldc + n0 + c * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        dst[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                             __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
    } else {
      float4* row = reinterpret_cast<float4*>(red + (quad * 32 + lane) * kRedLd + c * 32);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        row[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                             __uint_as_float(v[4 * q + 3]));
    }
  }
  trace_point(27);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if constexpr (kCluster) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // red -> bulk copies
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols) : "memory");
  }
  if constexpr (kCluster) {
    const int csz = gg.cluster;                              // cluster size along z (divides gridDim.z)
    const int rows = kBM / csz;
    const uint32_t rank = cluster_rank();
    const uint32_t slab = (uint32_t)(rows * kRedLd * 4);     // one CTA's share of one partial
    const uint32_t recv = base + (uint32_t)R * kRaw + 2 * kBTile;   // [csz][rows][kRedLd]
    if (tid == 0) {
      for (int p = 0; p < csz; ++p) {                        // rows of CTA p -> slot `rank` of p's buffer
        const uint32_t dst = dsmem_map(recv + rank * slab, (uint32_t)p);
        const uint32_t bar = dsmem_map(smem_u32(&recv_bar), (uint32_t)p);
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
            "r"(smem_u32(red) + (uint32_t)p * slab), "r"(slab), "r"(bar)
            : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    trace_point(29);
    mbar_wait(&recv_bar, 0u);
    trace_point(30);
    const float* rb = reinterpret_cast<const float*>(sbase + (size_t)R * kRaw + 2 * kBTile);
    float* cp = C + (long long)(blockIdx.z / csz) * split_stride;
    for (int e = tid; e < rows * (BN / 4); e += kGemmThreads) {
      const int r = e / (BN / 4), c = (e % (BN / 4)) * 4;
      float4 a = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      for (int p = 0; p < csz; ++p) {                        // rank order: deterministic
        const float4 v = *reinterpret_cast<const float4*>(rb + (size_t)p * rows * kRedLd + r * kRedLd + c);
        a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
      }
      if constexpr (EPI == kEpiClusterTanh) {
        const float4 bb = *reinterpret_cast<const float4*>(s_bias + c);
        a = make_float4(tanhf(a.x + bb.x), tanhf(a.y + bb.y), tanhf(a.z + bb.z), tanhf(a.w + bb.w));
      }
      *reinterpret_cast<float4*>(cp + (long long)(m0 + (int)rank * rows + r) * ldc + n0 + c) = a;
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // red read out before exit
  }
  trace_point(28);
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

CUresult encode_2d(CUtensorMap* tm, const float* ptr, long long rows, long long cols, int box_rows,
                   CUtensorMapSwizzle sw) {
  auto fn = encode_fn();
  if (!fn) return CUDA_ERROR_NOT_SUPPORTED;
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)cols * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), gdim, gstride, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

constexpr size_t gemm_smem(int bn, bool cluster, bool compact) {
  return (size_t)raw_stages(bn, cluster, compact) * (kBM * 128 + bn * 128) + 2 * bn * 128 + recv_bytes(bn, cluster) +
         1024;
}

// one launch: PDL always, a (1, 1, cluster) thread-block cluster when cluster > 1
template <int BN, int AM, int BM, int EPI>
cudaError_t launch_one(const CUtensorMap& A, const CUtensorMap& B, float* C, int ldc, dim3 grid, int kbps,
                       long long sstride, const GemmGather& gg, cudaStream_t s) {
  auto kern = k_gemm_tf32x3<BN, AM, BM, EPI>;
  const size_t smem = gemm_smem(BN, EPI != kEpiStore, AM != kOpTma || BM != kOpTma);
  // function attributes once per instantiation and device (a process may drive several GPUs)
  static std::atomic<unsigned long long> configured{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit, std::memory_order_acq_rel);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (kUsePdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (EPI != kEpiStore) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 1;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = (unsigned)gg.cluster;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, A, B, C, ldc, kbps, sstride, gg);
}

}  // namespace

// 2-D fp32 tensor map over a row-major [rows x cols] matrix, box {32 cols, box_rows}, SWIZZLE_128B
cudaError_t make_tmap_k_major(CUtensorMap* tm, const float* ptr, long long rows, long long cols, int box_rows) {
  if (!encode_fn()) return cudaErrorNotSupported;
  return encode_2d(tm, ptr, rows, cols, box_rows, CU_TENSOR_MAP_SWIZZLE_128B) == CUDA_SUCCESS ? cudaSuccess
                                                                                             : cudaErrorInvalidValue;
}

// the same over a matrix read MN-major (rows = K): 32 x 32 boxes, SWIZZLE_128B_ATOM_32B
cudaError_t make_tmap_mn_major(CUtensorMap* tm, const float* ptr, long long rows, long long cols) {
  if (!encode_fn()) return cudaErrorNotSupported;
  return encode_2d(tm, ptr, rows, cols, 32, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) == CUDA_SUCCESS
             ? cudaSuccess : cudaErrorInvalidValue;
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
// cluster > 1: the split-K partials of `cluster` consecutive splits are summed in DSMEM, so
// C receives splits / cluster planes (cluster in {2, 4, 8, 16}, dividing splits).
cudaError_t launch_gemm_tf32x3(const CUtensorMap& A, const CUtensorMap& B, float* C, int M, int N, int K, int splits,
                               int bn, cudaStream_t s, int cluster) {
  if (M % kBM || K % (kBK * splits) || (bn != 64 && bn != 96 && bn != 128) || N % bn) return cudaErrorInvalidValue;
  if (cluster < 1 || cluster > 16 || kBM % cluster || splits % cluster) return cudaErrorInvalidValue;
  const int kbps = K / kBK / splits;
  const long long sstride = (long long)M * N;
  const dim3 grid(N / bn, M / kBM, splits);
  GemmGather gg = {};
  gg.cluster = cluster;
  if (cluster == 1) {
    if (bn == 128) return launch_one<128, kOpTma, kOpTma, kEpiStore>(A, B, C, N, grid, kbps, sstride, gg, s);
    if (bn == 96) return launch_one<96, kOpTma, kOpTma, kEpiStore>(A, B, C, N, grid, kbps, sstride, gg, s);
    return launch_one<64, kOpTma, kOpTma, kEpiStore>(A, B, C, N, grid, kbps, sstride, gg, s);
  }
  if (bn == 128) return launch_one<128, kOpTma, kOpTma, kEpiCluster>(A, B, C, N, grid, kbps, sstride, gg, s);
  if (bn == 96) return launch_one<96, kOpTma, kOpTma, kEpiCluster>(A, B, C, N, grid, kbps, sstride, gg, s);
  return launch_one<64, kOpTma, kOpTma, kEpiCluster>(A, B, C, N, grid, kbps, sstride, gg, s);
}

// MLP GEMM1: X[idx] . W^T over `splits` K ranges, X rows gathered by the kernel (and the batch
// indices drawn by it), W via `B` (box rows = bn); the partials of gg.cluster consecutive splits
// are reduced in DSMEM: cluster == splits writes h = tanh(. + bias) [M x N] itself, otherwise
// splits / cluster planes of z (M x N apart) for the caller to finish
cudaError_t launch_mlp_gemm1(const CUtensorMap& B, const GemmGather& gg, float* out, int M, int N, int K, int splits,
                             int bn, cudaStream_t s) {
  if (M % kBM || M > kMaxGatherRows || K % (kBK * splits) || (bn != 32 && bn != 64) || N % bn || gg.cluster < 2 ||
      gg.cluster > 16 || splits % gg.cluster || kBM % gg.cluster)
    return cudaErrorInvalidValue;
  const dim3 grid(N / bn, M / kBM, splits);
  const int kbps = K / kBK / splits;
  const long long ss = (long long)M * N;
  if (gg.cluster == splits) {
    if (bn == 32) return launch_one<32, kOpGatherK, kOpTma, kEpiClusterTanh>(B, B, out, N, grid, kbps, ss, gg, s);
    return launch_one<64, kOpGatherK, kOpTma, kEpiClusterTanh>(B, B, out, N, grid, kbps, ss, gg, s);
  }
  if (bn == 32) return launch_one<32, kOpGatherK, kOpTma, kEpiCluster>(B, B, out, N, grid, kbps, ss, gg, s);
  return launch_one<64, kOpGatherK, kOpTma, kEpiCluster>(B, B, out, N, grid, kbps, ss, gg, s);
}

// MLP GEMM2: C [M x N] = A^T . X[idx] with A [K x M] row-major (MN-major tiles, `A` a box-32x32
// map over it) and X rows gathered by the kernel (MN-major); K = the batch
cudaError_t launch_mlp_gemm2(const CUtensorMap& A, const GemmGather& gg, float* C, int M, int N, int K, int bn,
                             cudaStream_t s) {
  if (M % kBM || K % kBK || K > kMaxGatherRows || (bn != 64 && bn != 96) || N % bn || gg.cluster != 1)
    return cudaErrorInvalidValue;
  // red_ctas extra columns of CTAs x the M / 128 rows give the batch reduction's 32-unit slices
  if (gg.red_ctas && (gg.r_O > kRedMaxOut || gg.red_ctas * (M / kBM) * 32 < gg.r_H)) return cudaErrorInvalidValue;
  const dim3 grid(N / bn + gg.red_ctas, M / kBM, 1);
  if (bn == 96) return launch_one<96, kOpTmaMN, kOpGatherMN, kEpiStore>(A, A, C, N, grid, K / kBK, 0, gg, s);
  return launch_one<64, kOpTmaMN, kOpGatherMN, kEpiStore>(A, A, C, N, grid, K / kBK, 0, gg, s);
}

const void* gemm_module_anchor() { return (const void*)k_sum_planes; }

}  // namespace adp
