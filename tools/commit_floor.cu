// commit_floor.cu -- the random read-modify-write floor of the commit (VERDICT r01
// "prove a random-RMW floor"): the SAME access pattern as k_commit on a config-2 batch, without any
// of its logic -- per new block one 128-bit CAS that claims an empty 64-B slot's key, the 16-B
// payload store into the same sector, the sequential per-block inputs (h, d 8 B each, label 1 B)
// and output (slot 4 B), and for the first new block of every prompt an atomic exchange of its
// parent's first-child link (a random other slot).  Warp = one prompt's 88 new blocks (config 2:
// 128 blocks, the first 40 matched), lanes = blocks, 2 rounds of 32 claims in flight, a grid of
// 8 CTAs x 256 threads per SM striding over the prompts (k_commit's launch shape).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/commit_floor tools/commit_floor.cu
//   build/commit_floor [table_log2_slots ...]   (prints one JSON line per table size)
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <cstdlib>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

constexpr uint32_t kNew = 88;  // new blocks per prompt (config 2)

__global__ void __launch_bounds__(256) k_floor(ulonglong2* tab, uint64_t mask, uint32_t n_prompts,
                                               const uint64_t* __restrict__ hk, const uint64_t* __restrict__ dk,
                                               const uint8_t* __restrict__ lab, uint32_t* __restrict__ slot_out,
                                               uint64_t seed) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t stride = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n_prompts; p += stride) {
    for (uint32_t base = 0; base < kNew; base += 64) {
      uint64_t s[2];
      unsigned long long o[2][2];
      bool act[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const uint32_t b = base + 32 * r + lane;
        act[r] = b < kNew;
        const uint64_t k = static_cast<uint64_t>(p) * kNew + (act[r] ? b : 0);
        const uint64_t h = hk[k], d = dk[k];  // the claimed key (sequential input)
        s[r] = mix(seed ^ h ^ (d << 1)) & mask;
        unsigned long long* a = reinterpret_cast<unsigned long long*>(&tab[s[r] * 4]);
        o[r][0] = o[r][1] = ~0ull;
        if (act[r])
          asm volatile(
              "{\n\t.reg .b128 c, n, x;\n\tmov.b128 c, {%2, %3};\n\tmov.b128 n, {%4, %5};\n\t"
              "atom.global.cas.b128 x, [%6], c, n;\n\tmov.b128 {%0, %1}, x;\n\t}"
              : "=l"(o[r][0]), "=l"(o[r][1])
              : "l"(0ull), "l"(0ull), "l"(h | 1), "l"(d), "l"(a)
              : "memory");
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const uint32_t b = base + 32 * r + lane;
        if (!act[r]) continue;
        const uint64_t k = static_cast<uint64_t>(p) * kNew + b;
        if (o[r][0] == 0 && o[r][1] == 0)  // claimed: payload (creator, meta | parent, child)
          tab[s[r] * 4 + 1] = make_ulonglong2((static_cast<uint64_t>(lab[k]) << 40) | p, s[r]);
        slot_out[k] = static_cast<uint32_t>(s[r]);
        if (b == 0)  // the prompt's first new block links under its (existing) parent
          atomicExch(reinterpret_cast<unsigned int*>(&tab[(mix(seed + p) & mask) * 4 + 1]) + 3,
                     static_cast<unsigned>(s[r]));
      }
    }
  }
}

__global__ void k_keys(uint64_t* hk, uint64_t* dk, uint8_t* lab, uint64_t n, uint64_t seed) {
  for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
    hk[k] = mix(seed + 2 * k);
    dk[k] = mix(seed + 2 * k + 1);
    lab[k] = static_cast<uint8_t>(k & 1);
  }
}

int main(int argc, char** argv) {
  const uint32_t n_prompts = 65536;
  const uint64_t n_blocks = static_cast<uint64_t>(n_prompts) * kNew;  // 5,767,168 claims
  uint64_t *hk, *dk;
  uint8_t* lab;
  uint32_t* so;
  cudaMalloc(&hk, n_blocks * 8);
  cudaMalloc(&dk, n_blocks * 8);
  cudaMalloc(&lab, n_blocks);
  cudaMalloc(&so, n_blocks * 4);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int logs[8] = {30, 28, 26}, nl = 3;
  if (argc > 1) {
    nl = 0;
    for (int i = 1; i < argc && nl < 8; ++i) logs[nl++] = atoi(argv[i]);
  }
  for (int li = 0; li < nl; ++li) {
    const uint64_t slots = 1ull << logs[li], bytes = slots * 64;
    void* tab = nullptr;
    if (cudaMalloc(&tab, bytes) != cudaSuccess) {
      printf("{\"error\": \"alloc %llu\"}\n", (unsigned long long)bytes);
      cudaGetLastError();
      continue;
    }
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemset(tab, 0, bytes);
      // distinct random keys per repetition (fresh claims, like a new batch)
      k_keys<<<4 * nsm, 256>>>(hk, dk, lab, n_blocks, 1234567ull * (rep + 1));
      cudaEventRecord(e0);
      k_floor<<<8 * nsm, 256>>>(static_cast<ulonglong2*>(tab), slots - 1, n_prompts, hk, dk, lab, so,
                                0x9e3779b97f4a7c15ull * (rep + 1));
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("{\"op\": \"commit_floor\", \"table_slots_log2\": %d, \"table_gib\": %.1f, \"claims\": %llu, "
           "\"ms\": %.4f, \"Gclaims_per_s\": %.3f}\n",
           logs[li], bytes / 1073741824.0, (unsigned long long)n_blocks, best, n_blocks / (best * 1e-3) / 1e9);
    cudaFree(tab);
  }
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("{\"error\": \"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
