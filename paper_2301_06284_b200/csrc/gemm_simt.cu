// gemm_simt.cu -- typed grouped GEMM (forward) and segmented dW GEMM on the
// SIMT FFMA pipe.  This is the fp32 path (RGNN_F32, reading O16: kind::tf32
// cannot meet the 1e-4 fp32 tolerance) and the fallback for shapes the
// tcgen05 kernel does not cover.  Segment MM = PAPER.md Sec. 2.2
// ("apply the corresponding weight ... to each segment"), one W_r per
// relation, never replicated.  Gather-on-load of X rows = the GEMM
// template's gather list.  No scatter: Z rows are the (etype,dst)
// positions, written in place.
#include "kernels.cuh"

namespace rgnn {

// -------------------------------------------------------------- forward
// One CTA walks a contiguous range of tiles (W_r reloaded only when r
// changes).  256 threads = 16 row-groups x 16 col-groups; a thread owns a
// 4-row x N/16-col block of a 64-row half-tile.
template <typename T, int K, int N>
__global__ void __launch_bounds__(256) k_gemm_fwd_simt(GemmFwdArgs a) {
  constexpr int CN = N / 16;
  extern __shared__ float smem[];
  float* Ws = smem;                // [K][N]
  float* Xs = smem + K * N;        // [64][K+1]
  const T* X = static_cast<const T*>(a.X);
  T* Z = static_cast<T*>(a.Z);
  const int tid = threadIdx.x, ry = tid >> 4, cx = tid & 15;
  const int64_t ntiles = a.tiles ? a.num_tiles : (a.rows + kTileRows - 1) / kTileRows;
  const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * per, t1 = min(ntiles, t0 + per);
  int cur_r = -1;
  for (int64_t t = t0; t < t1; ++t) {
    int r, row0, row1;
    if (a.tiles) { Tile tl = a.tiles[t]; r = tl.r; row0 = tl.row0; row1 = tl.row1; }
    else { r = 0; row0 = (int)(t * kTileRows); row1 = (int)min(a.rows, (int64_t)row0 + kTileRows); }
    if (r != cur_r) {
      __syncthreads();
      const float* Wr = a.W + (size_t)r * K * N;
      for (int i = tid; i < K * N; i += 256) {
        float w = Wr[i];
        if constexpr (sizeof(T) == 2) w = __bfloat162float(__float2bfloat16_rn(w));  // W rounded RNE (O16)
        Ws[i] = w;
      }
      cur_r = r;
    }
    for (int h0 = row0; h0 < row1; h0 += 64) {
      __syncthreads();
      for (int i = tid; i < 64 * K; i += 256) {
        int rr = i / K, k = i - rr * K;
        int p = h0 + rr;
        float x = 0.f;
        if (p < row1) {
          int64_t xr = a.gather ? (int64_t)a.gather[p] : a.gofs + p;
          x = to_f(X[xr * K + k]);
        }
        Xs[rr * (K + 1) + k] = x;
      }
      __syncthreads();
      float acc[4][CN];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < CN; ++j) acc[i][j] = 0.f;
#pragma unroll 4
      for (int k = 0; k < K; ++k) {
        float xa[4], wb[CN];
#pragma unroll
        for (int i = 0; i < 4; ++i) xa[i] = Xs[(ry * 4 + i) * (K + 1) + k];
#pragma unroll
        for (int j = 0; j < CN; ++j) wb[j] = Ws[k * N + cx * CN + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < CN; ++j) acc[i][j] = fmaf(xa[i], wb[j], acc[i][j]);
      }
      // epilogue: RGAT src score from the fp32 accumulator, RGCN per-row 1/c, store Z
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int p = h0 + ry * 4 + i;
        if (a.A) {
          const float* A0 = a.A + (size_t)r * 2 * N + cx * CN;
          float sc = 0.f;
#pragma unroll
          for (int j = 0; j < CN; ++j) sc = fmaf(acc[i][j], A0[j], sc);
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
          if (cx == 0 && p < row1) a.s_src[p] = sc;
        }
        if (p < row1) {
          float sc = a.row_scale ? a.row_scale[p] : 1.f;
          T* zp = Z + (size_t)p * N + cx * CN;
#pragma unroll
          for (int j = 0; j < CN; ++j) zp[j] = from_f<T>(acc[i][j] * sc);
        }
      }
    }
  }
}

// -------------------------------------------------------------- dW split-K
// part[c] (K x N) = sum over rows p of chunk c of X[g(p)]^T B[p]; 32-row
// sub-tiles staged in smem; a thread owns a K/16 x N/16 block.  For RGAT,
// threads [0,K) also accumulate bvec = sum dpre X_src (the dst term lives in
// dst_term.cu).  part row stride = K*N + K.
template <typename T, int K, int N, bool RGAT>
__global__ void __launch_bounds__(256) k_gemm_dw_simt(GemmDwArgs a) {
  constexpr int KB = K / 16, NB = N / 16, SR = (K + N >= 192) ? 16 : 32;
  __shared__ float Xs[SR][K + 1];
  __shared__ float Bs[SR][N + 1];
  __shared__ float Dp[SR];
  const T* X = static_cast<const T*>(a.X);
  const T* Bz = static_cast<const T*>(a.Bz);
  const int tid = threadIdx.x, ky = tid >> 4, cx = tid & 15;
  for (int64_t c = blockIdx.x; c < a.num_chunks; c += gridDim.x) {
    int row0, row1;
    if (a.chunks) { Tile t = a.chunks[c]; row0 = t.row0; row1 = t.row1; }
    else { row0 = (int)(c * a.chunk_rows); row1 = (int)min(a.rows, (int64_t)row0 + a.chunk_rows); }
    float acc[KB][NB];
#pragma unroll
    for (int i = 0; i < KB; ++i)
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[i][j] = 0.f;
    float vacc = 0.f;
    for (int s0 = row0; s0 < row1; s0 += SR) {
      __syncthreads();
      for (int i = tid; i < SR * K; i += 256) {
        int rr = i / K, k = i - rr * K, p = s0 + rr;
        float x = 0.f;
        if (p < row1) {
          int64_t xr = a.gather ? (int64_t)a.gather[p] : a.gofs + p;
          x = to_f(X[xr * K + k]);
        }
        Xs[rr][k] = x;
      }
      for (int i = tid; i < SR * N; i += 256) {
        int rr = i / N, n = i - rr * N, p = s0 + rr;
        float b = 0.f;
        if (p < row1) {
          if (Bz) {
            b = to_f(Bz[(size_t)p * N + n]);
          } else {
            int64_t br = a.bgather ? (int64_t)a.bgather[p] : p;
            b = a.Bg[br * N + n] * (a.bscale ? a.bscale[p] : 1.f);
          }
        }
        Bs[rr][n] = b;
      }
      if (RGAT && tid < SR) Dp[tid] = (s0 + tid < row1) ? a.dpre[s0 + tid] : 0.f;
      __syncthreads();
#pragma unroll 4
      for (int rr = 0; rr < SR; ++rr) {
        float xa[KB], bb[NB];
#pragma unroll
        for (int i = 0; i < KB; ++i) xa[i] = Xs[rr][ky * KB + i];
#pragma unroll
        for (int j = 0; j < NB; ++j) bb[j] = Bs[rr][cx * NB + j];
#pragma unroll
        for (int i = 0; i < KB; ++i)
#pragma unroll
          for (int j = 0; j < NB; ++j) acc[i][j] = fmaf(xa[i], bb[j], acc[i][j]);
      }
      if constexpr (RGAT) {
        if (tid < K)
          for (int rr = 0; rr < SR; ++rr) vacc = fmaf(Dp[rr], Xs[rr][tid], vacc);
      }
    }
    float* out = a.part + (size_t)c * (K * N + K);
#pragma unroll
    for (int i = 0; i < KB; ++i)
#pragma unroll
      for (int j = 0; j < NB; ++j) out[(ky * KB + i) * N + cx * NB + j] = acc[i][j];
    if (tid < K) out[K * N + tid] = RGAT ? vacc : 0.f;
  }
}

// dW[r] = sum_c part[c] (+ (sum_c cpart[c]) (x) A[r,1] for RGAT), chunks of r in order.
// Split-K reduction, stage 1: the chunks of each relation are cut into groups of kRedGroup consecutive
// chunks and each group's partials are summed in chunk order into its first chunk, in place (one
// thread per (group, element): ~num_chunks * (K*N + K) / 8 independent sums).  Stage 2 (below) then
// sums the group leaders of a relation in order.  Deterministic; measured r02 on ogbn-mag with 592
// chunks: the single-stage per-element loop over 148 chunks per relation took 0.08-0.17 ms.
constexpr int kRedGroup = 8;
// grid = (element blocks, chunks): blockIdx.y = chunk c; blocks of non-leader chunks exit at once, a
// leader's blocks sum its group's partials for a contiguous slice of elements (coalesced, in chunk order).
// (r01 / early r02: one thread per (chunk, element) over the whole partial space, 7 of 8 threads idle and
// a 64-bit division per element -- 67 us on ogbn-mag.)
__global__ void __launch_bounds__(256) k_dw_group(int K, int N, const Tile* __restrict__ chunks,
                                                  const int32_t* __restrict__ chunk_seg, float* __restrict__ part,
                                                  float* __restrict__ cpart) {
  const int c = blockIdx.y;
  const int r = chunks[c].r, c0 = chunk_seg[r], c1 = chunk_seg[r + 1];
  if ((c - c0) % kRedGroup != 0) return;  // not a group leader
  const int cend = min(c1, c + kRedGroup);
  const int stride = K * N + K;
  const int tot = stride + (cpart ? K : 0);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
    const bool is_c = e >= stride;  // the destination-term partials [num_chunks, K]
    float* base = is_c ? cpart : part;
    const int w = is_c ? K : stride, ee = is_c ? e - stride : e;
    float acc = base[(size_t)c * w + ee];
    for (int d = c + 1; d < cend; ++d) acc += base[(size_t)d * w + ee];
    base[(size_t)c * w + ee] = acc;
  }
}

// vsum (optional): the per-relation destination-term sums c_r (vsum[r][1], from k_da_vsum) -- read
// once per element instead of every (k, n) thread summing the chunks' c_r partials again.
__global__ void k_dw_reduce(int K, int N, int R, int64_t num_chunks, const int32_t* __restrict__ chunk_seg,
                            const float* __restrict__ part, const int32_t* __restrict__ cseg,
                            const float* __restrict__ cpart, const float* __restrict__ A, float* __restrict__ dW,
                            const float* __restrict__ vsum, int gstep, int src_term) {
  const int64_t total = (int64_t)R * K * N;
  const int stride = K * N + K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int r = (int)(i / (K * N));
    int kn = (int)(i - (int64_t)r * K * N);
    int k = kn / N, n = kn - k * N;
    int c0 = chunk_seg ? chunk_seg[r] : 0, c1 = chunk_seg ? chunk_seg[r + 1] : (int)num_chunks;
    // four independent partial sums (chunk c goes to (c - c0) % 4), combined in a fixed order: the
    // loads of four chunks are in flight at once and the result stays deterministic
    // (with gstep = kRedGroup the loop visits the group leaders written by k_dw_group)
    float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
    int c = c0;
    for (; c + 3 * gstep < c1; c += 4 * gstep) {
      s0 += part[(size_t)c * stride + kn];
      s1 += part[(size_t)(c + gstep) * stride + kn];
      s2 += part[(size_t)(c + 2 * gstep) * stride + kn];
      s3 += part[(size_t)(c + 3 * gstep) * stride + kn];
    }
    if (c < c1) s0 += part[(size_t)c * stride + kn];
    if (c + gstep < c1) s1 += part[(size_t)(c + gstep) * stride + kn];
    if (c + 2 * gstep < c1) s2 += part[(size_t)(c + 2 * gstep) * stride + kn];
    float s = (s0 + s1) + (s2 + s3);
    if (A) {
      float cv = 0.f;
      if (vsum) {
        cv = vsum[((size_t)r * 2 + 1) * K + k];
      } else {
        for (int c = cseg[r]; c < cseg[r + 1]; c += gstep) cv += cpart[(size_t)c * K + k];
      }
      s = fmaf(cv, A[(size_t)r * 2 * N + N + n], s);
      // the score's source term (sum_p dpre_p x_src(p)) (x) A[r,0], when the gradient rows dZ carried
      // only alpha G_v (bwd_tm.cu)
      if (src_term && vsum) s = fmaf(vsum[((size_t)r * 2) * K + k], A[(size_t)r * 2 * N + n], s);
    }
    dW[i] = s;
  }
}

// Per-relation sums of the dA vectors: vsum[r][0][k] = sum_c bvec_c[k], vsum[r][1][k] = sum_c cpart_c[k].
__global__ void k_da_vsum(int K, int N, int R, const int32_t* __restrict__ chunk_seg, const float* __restrict__ part,
                          const int32_t* __restrict__ cseg, const float* __restrict__ cpart, float* __restrict__ vsum,
                          int gstep) {
  const int stride = K * N + K;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)R * 2 * K;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / (2 * K)), h = (int)((i / K) % 2), k = (int)(i % K);
    // four independent partial sums over the chunks, fixed combination order (deterministic)
    const int c0 = h == 0 ? chunk_seg[r] : cseg[r], c1 = h == 0 ? chunk_seg[r + 1] : cseg[r + 1];
    const float* base = h == 0 ? part + (size_t)K * N + k : cpart + k;
    const size_t st = h == 0 ? (size_t)stride : (size_t)K;
    float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
    int c = c0;
    for (; c + 3 * gstep < c1; c += 4 * gstep) {
      v0 += base[(size_t)c * st]; v1 += base[(size_t)(c + gstep) * st];
      v2 += base[(size_t)(c + 2 * gstep) * st]; v3 += base[(size_t)(c + 3 * gstep) * st];
    }
    if (c < c1) v0 += base[(size_t)c * st];
    if (c + gstep < c1) v1 += base[(size_t)(c + gstep) * st];
    if (c + 2 * gstep < c1) v2 += base[(size_t)(c + 2 * gstep) * st];
    vsum[i] = (v0 + v1) + (v2 + v3);
  }
}

// dA[r,h,n] = vsum[r][h] . W_r[:,n]  (h = 0: sum dpre x_src, h = 1: sum dpre x_dst).  One block of 8
// warps per (r, h, 32 columns): warp w sums k in its eighth of [0, K), lane = column; the eight partials
// are added in warp order (deterministic).  (The r01 kernel ran one serial K-loop per output on 8 blocks:
// 33 us on ogbn-mag.)
__global__ void __launch_bounds__(256) k_da(int K, int N, int R, const float* __restrict__ vsum,
                                            const float* __restrict__ W, float* __restrict__ dA, int round_bf16) {
  __shared__ float s_p[8][32];
  const int ncb = (N + 31) / 32;
  const int rh = blockIdx.x / ncb, cb = blockIdx.x % ncb;
  const int r = rh / 2, h = rh % 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = cb * 32 + lane;
  const float* v = vsum + ((size_t)r * 2 + h) * K;
  const int kper = (K + 7) / 8, k0 = warp * kper, k1 = min(K, k0 + kper);
  float acc = 0.f;
  if (n < N) {
    for (int k = k0; k < k1; ++k) {
      float w = W[((size_t)r * K + k) * N + n];
      if (round_bf16) w = __bfloat162float(__float2bfloat16_rn(w));
      acc = fmaf(v[k], w, acc);
    }
  }
  s_p[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && n < N) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += s_p[i][lane];
    dA[((size_t)r * 2 + h) * N + n] = t;
  }
}

// U[r,k] = sum_n W[r,k,n] A[r,1,n]: linear-operator fusion (Sec. 3.4.1 P:706-708,
// "calculate w_{a,r}^T W_r first"), so that A[r,1].(x_dst W_r) = x_dst . U[r].
// On the bf16 path W is the RNE-rounded weight (the same values the typed GEMM
// multiplies), so the score x_dst . U[r] equals A[r,1].(x_dst W_r) of the GEMM's W.
// U[r, k] = sum_n W[r, k, n] A[r, half, n]: one warp per (r, k) row, lanes stride over n (coalesced
// row reads), fixed xor-tree reduction (deterministic).  r01's thread-per-row version read the rows
// with a 4*N-byte stride between lanes and took ~25 us per call on ogbn-mag.
__global__ void k_fold_u(int R, int K, int N, const float* __restrict__ W, const float* __restrict__ A,
                         float* __restrict__ U, int round_bf16, int half) {
  const int lane = threadIdx.x & 31;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < R * K; i += (gridDim.x * blockDim.x) >> 5) {
    const int r = i / K;
    const float* w = W + (size_t)i * N;
    const float* a1 = A + (size_t)r * 2 * N + half * N;
    float s = 0.f;
    for (int n = lane; n < N; n += 32) {
      const float wn = round_bf16 ? __bfloat162float(__float2bfloat16_rn(w[n])) : w[n];
      s = fmaf(wn, a1[n], s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) U[i] = s;
  }
}

template <typename T, int K, int N>
static rgnn_status gemm_fwd_simt(const GemmFwdArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(float) * (K * N + 64 * (K + 1));
  auto kern = k_gemm_fwd_simt<T, K, N>;
  RGNN_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t ntiles = a.tiles ? a.num_tiles : (a.rows + kTileRows - 1) / kTileRows;
  if (ntiles == 0) return RGNN_OK;
  int dev, sms;
  RGNN_CUDA_TRY(cudaGetDevice(&dev));
  RGNN_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int64_t grid = std::min<int64_t>(ntiles, (int64_t)sms * 2);
  RGNN_LAUNCH(kern, (unsigned)grid, 256, smem, s, a);
  return RGNN_OK;
}

rgnn_status launch_gemm_fwd(int prec, int K, int N, const GemmFwdArgs& a, cudaStream_t s) {
  return RGNN_DISPATCH_KN(K, N, [&] {
    return prec == RGNN_BF16 ? gemm_fwd_simt<__nv_bfloat16, kK, kN>(a, s) : gemm_fwd_simt<float, kK, kN>(a, s);
  });
}

template <typename T, int K, int N>
static rgnn_status gemm_dw_simt(const GemmDwArgs& a, cudaStream_t s) {
  if (a.num_chunks == 0) return RGNN_OK;
  unsigned grid = (unsigned)std::min<int64_t>(a.num_chunks, 148 * 8);
  if (a.dpre) RGNN_LAUNCH((k_gemm_dw_simt<T, K, N, true>), grid, 256, 0, s, a);
  else RGNN_LAUNCH((k_gemm_dw_simt<T, K, N, false>), grid, 256, 0, s, a);
  return RGNN_OK;
}

rgnn_status launch_gemm_dw(int prec, int K, int N, const GemmDwArgs& a, cudaStream_t s) {
  return RGNN_DISPATCH_KN(K, N, [&] {
    return prec == RGNN_BF16 ? gemm_dw_simt<__nv_bfloat16, kK, kN>(a, s) : gemm_dw_simt<float, kK, kN>(a, s);
  });
}

rgnn_status launch_dw_reduce(int prec, int K, int N, int R, int64_t num_chunks, const int32_t* chunk_seg,
                             const float* part, const int32_t* cseg, const float* cpart, const float* A,
                             const float* W, float* dW, float* dA, float* dA_scratch, cudaStream_t s,
                             const Tile* chunks, bool src_term) {
  int64_t total = (int64_t)R * K * N;
  unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16));
  // two stages when the chunk table is known (the partials are summed in groups of kRedGroup chunks
  // in place first); the dst-term partials cpart are grouped along (they use the same chunks)
  int gstep = 1;
  if (chunks && chunk_seg && num_chunks > kRedGroup) {
    const int tot = K * N + K + (cpart ? K : 0);
    const dim3 grid_g((unsigned)std::min(8, (tot + 255) / 256), (unsigned)num_chunks);
    RGNN_LAUNCH(k_dw_group, grid_g, 256, 0, s, K, N, chunks, chunk_seg, const_cast<float*>(part),
                const_cast<float*>(cpart));
    gstep = kRedGroup;
  }
  float* vsum = dA ? dA_scratch : nullptr;
  if (dA) {  // per-relation vectors first: dA needs them and dW's destination term reads c_r from them
    unsigned g1 = (unsigned)std::max<int64_t>(1, ((int64_t)R * 2 * K + 127) / 128);
    RGNN_LAUNCH(k_da_vsum, g1, 128, 0, s, K, N, R, chunk_seg, part, cseg, cpart, vsum, gstep);
  }
  RGNN_LAUNCH(k_dw_reduce, grid, 256, 0, s, K, N, R, num_chunks, chunk_seg, part, cseg, cpart, A, dW,
              (A && dA) ? vsum : nullptr, gstep, src_term ? 1 : 0);
  if (dA) {
    const unsigned g2 = (unsigned)(R * 2 * ((N + 31) / 32));
    RGNN_LAUNCH(k_da, g2, 256, 0, s, K, N, R, vsum, W, dA, prec == RGNN_BF16 ? 1 : 0);
  }
  return RGNN_OK;
}

rgnn_status launch_fold_u(int prec, int R, int K, int N, const float* W, const float* A, float* U, cudaStream_t s,
                          int half) {
  unsigned grid = (unsigned)std::max(1, std::min((R * K + 7) / 8, 148 * 8));  // 8 warps (rows) per block
  RGNN_LAUNCH(k_fold_u, grid, 256, 0, s, R, K, N, W, A, U, prec == RGNN_BF16 ? 1 : 0, half);
  return RGNN_OK;
}

}  // namespace rgnn
