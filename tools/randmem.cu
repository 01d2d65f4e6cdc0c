// randmem.cu -- random-access microbenchmark for the index layout decisions:
// throughput of independent random 16-B loads and 128-bit CAS into 64-B slots as a
// function of the table footprint (TLB reach, DRAM random-access efficiency).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/randmem tools/randmem.cu
//   build/randmem            (prints one JSON line per footprint)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// each thread: `per` independent random 16-B loads from distinct 64-B slots, 4 in flight
__global__ void k_load(const ulonglong2* __restrict__ t, uint64_t mask, int per, uint64_t seed,
                       unsigned long long* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t acc = 0;
  for (int i = 0; i < per; i += 4) {
    ulonglong2 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = t[(mix(seed + tid * per + i + q) & mask) * 4];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc += v[q].x ^ v[q].y;
  }
  if (acc == 0x1234567) atomicAdd(sink, 1ull);
}

__global__ void k_cas(ulonglong2* t, uint64_t mask, int per, uint64_t seed, unsigned long long* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t acc = 0;
  for (int i = 0; i < per; i += 4) {
    unsigned long long o[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t s = mix(seed + tid * per + i + q) & mask;
      unsigned long long* a = reinterpret_cast<unsigned long long*>(&t[s * 4]);
      asm volatile(
          "{\n\t.reg .b128 c, n, d;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 n, {%4, %5};\n\t"
          "atom.global.cas.b128 d, [%6], c, n;\n\tmov.b128 {%0, %1}, d;\n\t}"
          : "=l"(o[q][0]), "=l"(o[q][1])
          : "l"(0ull), "l"(0ull), "l"(s + 1), "l"(tid), "l"(a)
          : "memory");
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) acc += o[q][0];
  }
  if (acc == 0x1234567) atomicAdd(sink, 1ull);
}

int main() {
  const uint64_t max_bytes = 32ull << 30;
  void* buf = nullptr;
  if (cudaMalloc(&buf, max_bytes) != cudaSuccess) {
    printf("{\"error\": \"alloc\"}\n");
    return 1;
  }
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = 148 * 8, per = 64;
  const uint64_t n_acc = (uint64_t)threads * blocks * per;
  for (uint64_t bytes = 64ull << 20; bytes <= max_bytes; bytes <<= 1) {
    const uint64_t slots = bytes / 64, mask = slots - 1;
    cudaMemset(buf, 0, bytes);
    for (int kind = 0; kind < 2; ++kind) {
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        if (kind == 1) cudaMemset(buf, 0, bytes);
        cudaEventRecord(e0);
        if (kind == 0)
          k_load<<<blocks, threads>>>((const ulonglong2*)buf, mask, per, 17 + rep, sink);
        else
          k_cas<<<blocks, threads>>>((ulonglong2*)buf, mask, per, 17 + rep, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("{\"op\": \"%s\", \"table_mb\": %llu, \"ms\": %.4f, \"Gops\": %.3f}\n", kind ? "cas128" : "load16",
             (unsigned long long)(bytes >> 20), best, n_acc / (best * 1e-3) / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
