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

// the commit pattern: CAS on sector 0 of a 64-B slot plus a second access in the same slot
// (mode 1: atomicMax on sector 1, mode 2: 16-B store into sector 0, mode 3: store into sector 1)
__global__ void k_cas2(ulonglong2* t, uint64_t mask, int per, uint64_t seed, unsigned long long* sink, int mode) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t acc = 0;
  for (int i = 0; i < per; i += 4) {
    unsigned long long o[4][2];
    uint64_t ss[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t s = mix(seed + tid * per + i + q) & mask;
      ss[q] = s;
      unsigned long long* a = reinterpret_cast<unsigned long long*>(&t[s * 4]);
      asm volatile(
          "{\n\t.reg .b128 c, n, d;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 n, {%4, %5};\n\t"
          "atom.global.cas.b128 d, [%6], c, n;\n\tmov.b128 {%0, %1}, d;\n\t}"
          : "=l"(o[q][0]), "=l"(o[q][1])
          : "l"(0ull), "l"(0ull), "l"(s + 1), "l"(tid), "l"(a)
          : "memory");
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      acc += o[q][0];
      if (mode == 1) atomicMax(reinterpret_cast<unsigned int*>(&t[ss[q] * 4 + 3]) + 3, (unsigned)tid);
      if (mode == 2) t[ss[q] * 4 + 1] = make_ulonglong2(tid, acc);
      if (mode == 3) t[ss[q] * 4 + 3] = make_ulonglong2(tid, acc);
    }
  }
  if (acc == 0x1234567) atomicAdd(sink, 1ull);
}

// locality: CAS into groups of G consecutive 128-B lines (one 128-B line = 2 slots), the
// group chosen at random: lane l of a warp takes line (l % G) of group hash(warp, l / G)
__global__ void k_cas_group(ulonglong2* t, uint64_t mask_groups, int G, int per, uint64_t seed,
                            unsigned long long* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  uint64_t acc = 0;
  for (int i = 0; i < per; ++i) {
    const uint64_t g = mix(seed + (tid / 32) * per * 32 + i * 32 + lane / G) & mask_groups;
    const uint64_t slot = (g * G + (lane % G)) * 2;  // 2 x 64-B slots per line
    unsigned long long* a = reinterpret_cast<unsigned long long*>(&t[slot * 4]);
    unsigned long long o0, o1;
    asm volatile(
        "{\n\t.reg .b128 c, n, d;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 n, {%4, %5};\n\t"
        "atom.global.cas.b128 d, [%6], c, n;\n\tmov.b128 {%0, %1}, d;\n\t}"
        : "=l"(o0), "=l"(o1)
        : "l"(0ull), "l"(0ull), "l"(slot + 1), "l"(tid), "l"(a)
        : "memory");
    acc += o0;
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
  for (int G : {1, 2, 4, 8, 16, 32}) {  // grouped-CAS locality on a 16 GB table
    const uint64_t bytes = 16ull << 30, lines = bytes / 128;
    const uint64_t groups = lines / G;
    uint64_t pow2 = 1;
    while (pow2 * 2 <= groups) pow2 *= 2;
    float best = 1e30f;
    const int blk = 148 * 8, pr = 64;
    const uint64_t n_ops = (uint64_t)threads * blk * pr;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(buf, 0, bytes);
      cudaEventRecord(e0);
      k_cas_group<<<blk, threads>>>((ulonglong2*)buf, pow2 - 1, G, pr, 41 + rep, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("{\"op\": \"cas128_group\", \"G_lines\": %d, \"ms\": %.4f, \"Gops\": %.3f}\n", G, best,
           n_ops / (best * 1e-3) / 1e9);
  }
  for (int bmul : {1, 2, 4, 8})
  for (int mode = 0; mode < 4; ++mode) {  // commit pattern on a 16 GB table, 148 x bmul CTAs
    const uint64_t bytes = 16ull << 30, slots = bytes / 64, mask = slots - 1;
    float best = 1e30f;
    const int blk = 148 * bmul, pr = per * 8 / bmul;
    const uint64_t n_ops = (uint64_t)threads * blk * pr;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(buf, 0, bytes);
      cudaEventRecord(e0);
      k_cas2<<<blk, threads>>>((ulonglong2*)buf, mask, pr, 29 + rep, sink, mode);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("{\"op\": \"cas128+mode%d\", \"ctas\": %d, \"table_mb\": %llu, \"ms\": %.4f, \"Gops\": %.3f}\n",
           mode, blk, (unsigned long long)(bytes >> 20), best, n_ops / (best * 1e-3) / 1e9);
  }
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
