// bulk_gather_bench.cu -- can 1-D TMA bulk copies (cp.async.bulk, one instruction per 256-byte row) feed
// random-row gathers faster than the register-held loads of the walks?  Each warp keeps a ring of S
// stages x R rows in shared memory: lane i < R issues the bulk copy of row i of a stage (completion on the
// stage's mbarrier with expect_tx), the warp consumes a stage (reads it back from shared memory) and
// refills it.  Reports GB/s of row bytes.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_gather_bench tools/bulk_gather_bench.cu
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int R, int S>
__global__ void __launch_bounds__(128) bulk_gather(const uint4* __restrict__ tab, const int* __restrict__ idx, int64_t n,
                                                   float* out) {
  constexpr int ROW = 256;
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + warp * (S * R * ROW);
  __shared__ uint64_t bars[4][S];
  if (lane < S) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[warp][lane])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncwarp();
  const int64_t gw = ((int64_t)blockIdx.x * 4 + warp), nw = (int64_t)gridDim.x * 4;
  const int64_t per = R;  // rows per stage
  int64_t next = gw * per;  // first row index of the next stage to issue (strided over warps)
  auto issue = [&](int s) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[warp][s])),
                   "r"(R * ROW));
    __syncwarp();
    const int64_t e = next + lane;
    if (lane < R) {
      const int64_t ee = e < n ? e : n - 1;
      const void* src = tab + (int64_t)idx[ee] * (ROW / 16);
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(ring + (s * R + lane) * ROW)),
          "l"(src), "r"(ROW), "r"(smem_u32(&bars[warp][s]))
          : "memory");
    }
    next += nw * per;
  };
  float acc = 0.f;
  const int64_t nsteps = (n + nw * per - 1) / (nw * per);
  for (int s = 0; s < S && s < nsteps; ++s) issue(s);
  for (int64_t it = 0; it < nsteps; ++it) {
    const int s = (int)(it % S);
    const uint32_t ph = (uint32_t)((it / S) & 1);
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok)
                   : "r"(smem_u32(&bars[warp][s])), "r"(ph)
                   : "memory");
    const float4* st = reinterpret_cast<const float4*>(ring + s * R * ROW);
#pragma unroll
    for (int i = lane; i < R * ROW / 16; i += 32) acc += st[i].x + st[i].w;
    __syncwarp();
    if (it + S < nsteps) issue(s);
  }
  if (acc == 1.2345f) out[0] = acc;
}

int main() {
  const int64_t rows = 21000000, row_bytes = 256, n = 21000000;
  uint4* tab; int* idx; float* out;
  cudaMalloc(&tab, rows * row_bytes); cudaMalloc(&idx, n * 4); cudaMalloc(&out, 4);
  cudaMemset(tab, 0, rows * row_bytes);
  std::vector<int> h(n);
  std::mt19937 rng(1);
  for (int64_t i = 0; i < n; ++i) h[i] = (int)(rng() % rows);
  cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, int R, int S, int blocks) {
    const int sm = 4 * S * R * 256;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    for (int w = 0; w < 2; ++w) kern<<<blocks, 128, sm>>>(tab, idx, n, out);
    cudaEventRecord(a);
    for (int w = 0; w < 5; ++w) kern<<<blocks, 128, sm>>>(tab, idx, n, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    cudaError_t e = cudaGetLastError();
    printf("bulk R=%d S=%d smem/block=%d KB blocks=%d: %.3f ms, %.0f GB/s of rows %s\n", R, S, sm / 1024, blocks, ms,
           n * row_bytes / (ms * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  for (int bpsm : {2, 4, 6}) {
    run(bulk_gather<8, 4>, 8, 4, 148 * bpsm);
    run(bulk_gather<16, 2>, 16, 2, 148 * bpsm);
    run(bulk_gather<8, 6>, 8, 6, 148 * bpsm);
    run(bulk_gather<16, 4>, 16, 4, 148 * std::min(bpsm, 3));
  }
  return 0;
}
