// Headroom probe (not product code): CUB's onesweep radix sort on the same
// shape as C4's ingest sort -- 626M 36-bit u64 keys with a u64 payload --
// for comparison with the hand-written sort.cu passes.
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdint>

__global__ void fill(uint64_t *k, uint64_t *v, size_t n)
{
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull;
    x ^= x >> 29;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 32;
    k[i] = x & ((1ull << 36) - 1);
    v[i] = i;
  }
}

int main(int argc, char **argv)
{
  size_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 625774225ull;
  uint64_t *k0, *k1, *v0, *v1;
  cudaMalloc(&k0, n * 8); cudaMalloc(&k1, n * 8); cudaMalloc(&v0, n * 8); cudaMalloc(&v1, n * 8);
  size_t tb = 0;
  cub::DoubleBuffer<uint64_t> kb(k0, k1), vb(v0, v1);
  cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)n, 0, 36);
  void *tmp; cudaMalloc(&tmp, tb);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 4; rep++) {
    fill<<<1184, 256>>>(k0, v0, n);
    cub::DoubleBuffer<uint64_t> kb2(k0, k1), vb2(v0, v1);
    cudaEventRecord(a);
    cub::DeviceRadixSort::SortPairs(tmp, tb, kb2, vb2, (int)n, 0, 36);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cub SortPairs u64/u64 n=%zu 36 bits: %.2f ms\n", n, ms);
  }
  // keys only u32 payload variant
  uint32_t *w0, *w1; cudaMalloc(&w0, n * 4); cudaMalloc(&w1, n * 4);
  for (int rep = 0; rep < 3; rep++) {
    fill<<<1184, 256>>>(k0, v0, n);
    cub::DoubleBuffer<uint64_t> kb2(k0, k1);
    cub::DoubleBuffer<uint32_t> wb(w0, w1);
    size_t tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, kb2, wb, (int)n, 0, 36);
    if (tb2 > tb) { printf("tmp too small\n"); break; }
    cudaEventRecord(a);
    cub::DeviceRadixSort::SortPairs(tmp, tb2, kb2, wb, (int)n, 0, 36);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("cub SortPairs u64/u32 n=%zu 36 bits: %.2f ms\n", n, ms);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
