// gather_bench.cu -- practical HBM roofline of the walks' access pattern: every
// warp gathers rows of `row_bytes` bytes at random row indices (as the
// aggregate / backward read Z[pos[q]]) and reduces them.  Reports GB/s of row
// bytes for several rows-in-flight settings.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench tools/gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int UNR>
__global__ void gather(const uint4* __restrict__ tab, const int* __restrict__ idx, int64_t n, int lanes_per_row,
                       float* out) {
  const int lane = threadIdx.x & 31, g = lane / lanes_per_row, l = lane % lanes_per_row, G = 32 / lanes_per_row;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (int64_t base = warp * G * UNR; base < n; base += nw * G * UNR) {
    uint4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t e = base + u * G + g;
      v[u] = e < n ? __ldg(tab + (int64_t)idx[e] * lanes_per_row + l) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) acc += __uint_as_float(v[u].x) + __uint_as_float(v[u].y) + __uint_as_float(v[u].w);
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  const int64_t rows = 21000000, row_bytes = 256, n = 21000000;
  const int lpr = row_bytes / 16;
  uint4* tab; int* idx; float* out;
  cudaMalloc(&tab, rows * row_bytes); cudaMalloc(&idx, n * 4); cudaMalloc(&out, 4);
  cudaMemset(tab, 0, rows * row_bytes);
  std::vector<int> h(n);
  std::mt19937 rng(1);
  for (int64_t i = 0; i < n; ++i) h[i] = (int)(rng() % rows);
  cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, int blocks, const char* name) {
    for (int w = 0; w < 3; ++w) kern<<<blocks, 256>>>(tab, idx, n, lpr, out);
    cudaEventRecord(a);
    for (int w = 0; w < 10; ++w) kern<<<blocks, 256>>>(tab, idx, n, lpr, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("%s blocks=%d: %.3f ms, %.0f GB/s of rows\n", name, blocks, ms, n * row_bytes / (ms * 1e-3) / 1e9);
  };
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    run(gather<2>, blocks, "UNR=2");
    run(gather<4>, blocks, "UNR=4");
    run(gather<8>, blocks, "UNR=8");
    run(gather<16>, blocks, "UNR=16");
  }
  // sequential rows for comparison
  for (int64_t i = 0; i < n; ++i) h[i] = (int)i;
  cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
  run(gather<8>, 148 * 8, "sequential UNR=8");
  return 0;
}
