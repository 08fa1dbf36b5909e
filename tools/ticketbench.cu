// Capacity of the engine's single system-wide ticket (rank 0's counter, taken by a
// compare-and-swap over NVLink -- engine.cu take_tickets): G GPUs x C concurrent takers each
// (one thread per CTA, as the engine's CTAs take tickets) race until `target` tickets are
// gone; prints tickets/s and CAS retries per ticket.  Diagnostic for SURVEY 8(e) / DESIGN 13.
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/ticketbench.cu -o tools/ticketbench
#include <cstdio>
#include <vector>
#include <chrono>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ unsigned long long ld_relaxed_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void k_take(unsigned long long* ticket, unsigned long long target, unsigned long long* taken,
                       unsigned long long* retries) {
  if (threadIdx.x) return;
  unsigned long long mine = 0, rt = 0;
  unsigned long long t = ld_relaxed_sys64(ticket);
  while (t < target) {
    const unsigned long long old = atomicCAS_system(ticket, t, t + 1);
    if (old == t) { ++mine; t = t + 1; t = ld_relaxed_sys64(ticket); }
    else { ++rt; t = old; }
  }
  atomicAdd(taken, mine);
  atomicAdd(retries, rt);
}

int main() {
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  for (int a = 0; a < ng; ++a)
    for (int b = 0; b < ng; ++b)
      if (a != b) { cudaSetDevice(a); cudaDeviceEnablePeerAccess(b, 0); cudaGetLastError(); }
  unsigned long long* ticket;
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&ticket, 8));
  std::vector<unsigned long long*> taken(ng), retries(ng);
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaMalloc(&taken[g], 8));
    CK(cudaMalloc(&retries[g], 8));
  }
  printf("{\"gpus_available\": %d, \"rows\": [\n", ng);
  bool first = true;
  for (int G = 1; G <= ng; G *= 2)
    for (int C : {8, 37, 148}) {
      const unsigned long long target = 200000;
      CK(cudaSetDevice(0));
      CK(cudaMemset(ticket, 0, 8));
      for (int g = 0; g < G; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaMemset(taken[g], 0, 8));
        CK(cudaMemset(retries[g], 0, 8));
        CK(cudaDeviceSynchronize());
      }
      const auto t0 = std::chrono::steady_clock::now();
      for (int g = 0; g < G; ++g) {
        CK(cudaSetDevice(g));
        k_take<<<C, 32>>>(ticket, target, taken[g], retries[g]);
      }
      for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
      const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      unsigned long long tk = 0, rt = 0;
      for (int g = 0; g < G; ++g) {
        unsigned long long a, b;
        CK(cudaSetDevice(g));
        CK(cudaMemcpy(&a, taken[g], 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&b, retries[g], 8, cudaMemcpyDeviceToHost));
        tk += a; rt += b;
      }
      printf("%s {\"gpus\": %d, \"takers_per_gpu\": %d, \"tickets\": %llu, \"seconds\": %.6f, "
             "\"tickets_per_s\": %.0f, \"cas_retries_per_ticket\": %.2f}", first ? "" : ",\n", G, C, tk, s, tk / s,
             (double)rt / (double)tk);
      first = false;
    }
  printf("\n]}\n");
  return 0;
}
