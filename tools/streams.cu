// streams.cu -- HBM read-pattern microbenchmark for k_hash_scan's token stream: every
// warp reads 2-KB chunks (lane l: 64 B at l*64 via two 256-bit loads), either walking
// its own contiguous range (as k_hash_scan) or interleaved across warps (chunk c ->
// warp c mod W).  Prints GB/s per pattern.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void ld256(const uint32_t* p, uint32_t (&t)[8]) {
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]), "=r"(t[6]), "=r"(t[7])
               : "l"(p));
}

template <int MODE>
__global__ void k_read(const uint32_t* __restrict__ tok, uint64_t n_chunks, unsigned long long* sink, int work) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5, TW = (gridDim.x * (uint64_t)blockDim.x) >> 5;
  uint32_t acc = 0;
  const uint64_t c0 = gw * n_chunks / TW, c1 = (gw + 1) * n_chunks / TW;
  for (uint64_t k = 0;; ++k) {
    uint64_t c;
    if (MODE == 0) { c = c0 + k; if (c >= c1) break; }
    else { c = gw + k * TW; if (c >= n_chunks) break; }
    const uint32_t* p = tok + c * 512 + lane * 16;
    uint32_t a[8], b[8];
    ld256(p, a);
    ld256(p + 8, b);
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) x ^= a[i] + b[i];
    for (int i = 0; i < work; ++i) x = x * 1664525u + 1013904223u;  // dependent ALU "compute"
    acc += x;
  }
  if (acc == 0x12345) atomicAdd(sink, 1ull);
}

int main() {
  const uint64_t bytes = 512ull << 20, n_chunks = bytes / 2048;
  uint32_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int work : {0, 200, 400}) {
    for (int warps_per_sm : {16, 32, 48}) {
      for (int mode = 0; mode < 2; ++mode) {
        const int threads = 512, blocks = 148 * warps_per_sm / 16;
        float best = 1e9f;
        for (int r = 0; r < 5; ++r) {
          cudaEventRecord(e0);
          if (mode == 0) k_read<0><<<blocks, threads>>>(buf, n_chunks, sink, work);
          else k_read<1><<<blocks, threads>>>(buf, n_chunks, sink, work);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        printf("{\"mode\": \"%s\", \"work\": %d, \"warps_per_sm\": %d, \"us\": %.1f, \"GBps\": %.0f}\n",
               mode ? "interleaved" : "contiguous", work, warps_per_sm, best * 1e3, bytes / (best * 1e-3) / 1e9);
      }
    }
  }
  return 0;
}
