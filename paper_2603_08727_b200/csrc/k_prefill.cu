// k_prefill.cu — prefill attention statistics (P1-P3 of DESIGN.md §2).
//
// For every unit (sequence, layer, KV head) the G*W window query rows (the last W
// prompt queries of the G query heads sharing the KV head, Eq. 2, R1, R20)
// are scored against all P prompt keys on the tensor cores (mma.sync m16n8k16,
// bf16 x bf16 -> fp32; the operands are the caller's bf16 values, so every product is
// exact).  Two passes over K (the column sums need the final row normalisers):
//   pass 1: per row online max / sum-exp over the causally visible keys;
//   pass 2: p = exp(s - m) / l on keys [0, P-W), reduced over the rows into the
//           per-KV-head heavy-hitter seed acc1 = Σ p, acc2 = Σ p² (Eq. 9 samples,
//           P:218-226) — the column sums of Eq. 3 are Σ over KV heads of acc1.
// A third tiny kernel reduces those columns into entropy / variance / kurtosis and
// the OQ score in float64 (Eqs. 3-6; R2-R7), in a fixed order
// (bitwise deterministic).
#include <cstdlib>

#include "kernels.h"

namespace arkv {

constexpr int kPfKeys = 64;     // keys per smem tile
constexpr int kPfChunk = 2048;  // keys per CTA

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// PASS2 == false: write per-(row, chunk) partial (m, l).  PASS2 == true: merge those
// partials and emit acc_pf[u][j] = (Σ_rows p, Σ_rows p²) for keys j < P - W.
template <int KD, int MPW, bool PASS2>
__global__ void __launch_bounds__(256) prefill_pass_kernel(Geom g, const uint16_t* __restrict__ q_win,
                                                           const uint16_t* __restrict__ kmat, int P,
                                                           float2* __restrict__ partials, int n_chunks1,
                                                           float2* __restrict__ acc_pf) {
  constexpr int D = KD * 16;
  constexpr int LDS = D + 8;  // padded smem row (bf16 elements): conflict-free fragment reads
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint16_t* ks = (uint16_t*)smem_raw;                        // [2][kPfKeys][LDS]
  float* red = (float*)(ks + 2 * kPfKeys * LDS);             // PASS2: [n_warps][kPfKeys][2]
  const int R = g.G * g.W;
  float* rowm = red + (PASS2 ? (blockDim.x / 32) * kPfKeys * 2 : 0);  // PASS2: [R]
  float* rowil = rowm + R;

  const int u = blockIdx.y;
  const int kvh = u % g.Hkv;
  const int bl = u / g.Hkv;  // b*L + l
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int nw = blockDim.x >> 5;

  const int key_end_all = PASS2 ? (P - g.W) : P;
  const int c0 = blockIdx.x * kPfChunk;
  const int c1 = min(c0 + kPfChunk, key_end_all);
  if (c0 >= c1) return;

  const uint16_t* qb = q_win + ((int64_t)bl * g.Hq + kvh * g.G) * g.W * D;  // rows r = h*W + i
  const uint16_t* kb = kmat + ((int64_t)bl * g.Hkv + kvh) * (int64_t)P * D;
  const float sl2 = g.sm_scale * 1.4426950408889634f;

  // A fragments (query rows) for this warp's MPW m-tiles.
  uint32_t af[MPW][KD][4];
#pragma unroll
  for (int mi = 0; mi < MPW; ++mi) {
    int r0 = (warp * MPW + mi) * 16 + gq;
    int r1 = r0 + 8;
#pragma unroll
    for (int kc = 0; kc < KD; ++kc) {
      int c = kc * 16 + 2 * tq;
      af[mi][kc][0] = r0 < R ? *(const uint32_t*)(qb + (int64_t)r0 * D + c) : 0u;
      af[mi][kc][1] = r1 < R ? *(const uint32_t*)(qb + (int64_t)r1 * D + c) : 0u;
      af[mi][kc][2] = r0 < R ? *(const uint32_t*)(qb + (int64_t)r0 * D + c + 8) : 0u;
      af[mi][kc][3] = r1 < R ? *(const uint32_t*)(qb + (int64_t)r1 * D + c + 8) : 0u;
    }
  }

  // Row statistics.
  float rm[MPW][2], rl[MPW][2];
#pragma unroll
  for (int mi = 0; mi < MPW; ++mi)
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      rm[mi][hh] = -INFINITY;
      rl[mi][hh] = 0.f;
    }
  if (PASS2) {
    for (int r = threadIdx.x; r < R; r += blockDim.x) {
      const float2* pr = partials + ((int64_t)u * n_chunks1) * R + r;
      float M = -INFINITY;
      for (int c = 0; c < n_chunks1; ++c) M = fmaxf(M, pr[(int64_t)c * R].x);
      float L = 0.f;
      for (int c = 0; c < n_chunks1; ++c) {
        float2 v = pr[(int64_t)c * R];
        if (v.y > 0.f) L += v.y * exp2f(v.x - M);
      }
      rowm[r] = M;
      rowil[r] = 1.0f / L;
    }
    __syncthreads();
#pragma unroll
    for (int mi = 0; mi < MPW; ++mi)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        int r = (warp * MPW + mi) * 16 + gq + 8 * hh;
        rm[mi][hh] = r < R ? rowm[r] : 0.f;
        rl[mi][hh] = r < R ? rowil[r] : 0.f;  // 0 => padded rows contribute nothing
      }
  }

  const int n_tiles = (c1 - c0 + kPfKeys - 1) / kPfKeys;
  auto load_tile = [&](int ti, int buf) {
    int base = c0 + ti * kPfKeys;
    constexpr int VPR = D / 8;  // 16-byte vectors per row
    for (int idx = threadIdx.x; idx < kPfKeys * VPR; idx += blockDim.x) {
      int row = idx / VPR, vc = idx % VPR;
      int key = base + row;
      bool ok = key < c1;
      const uint16_t* src = kb + (int64_t)(ok ? key : c0) * D + vc * 8;
      cp_async16(ks + (buf * kPfKeys + row) * LDS + vc * 8, src, ok);
    }
    cp_async_commit();
  };

  load_tile(0, 0);
  for (int ti = 0; ti < n_tiles; ++ti) {
    const int buf = ti & 1;
    if (ti + 1 < n_tiles) {
      load_tile(ti + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint16_t* kt = ks + buf * kPfKeys * LDS;
    const int kbase = c0 + ti * kPfKeys;

    float acc[MPW][8][4];
#pragma unroll
    for (int mi = 0; mi < MPW; ++mi)
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[mi][nt][e] = 0.f;

#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const uint16_t* krow = kt + (nt * 8 + gq) * LDS + 2 * tq;
#pragma unroll
      for (int kc = 0; kc < KD; ++kc) {
        uint32_t b0 = *(const uint32_t*)(krow + kc * 16);
        uint32_t b1 = *(const uint32_t*)(krow + kc * 16 + 8);
#pragma unroll
        for (int mi = 0; mi < MPW; ++mi)
          mma_bf16_16816(acc[mi][nt], af[mi][kc][0], af[mi][kc][1], af[mi][kc][2], af[mi][kc][3], b0, b1);
      }
    }

    if (!PASS2) {
#pragma unroll
      for (int mi = 0; mi < MPW; ++mi) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          int r = (warp * MPW + mi) * 16 + gq + 8 * hh;
          int qp = P - g.W + (r % g.W);  // query position of row r = h*W + i
          float mx = -INFINITY;
#pragma unroll
          for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              int key = kbase + nt * 8 + 2 * tq + e;
              float s = acc[mi][nt][hh * 2 + e] * sl2;
              bool vis = (r < R) && key < c1 && key <= qp;
              s = vis ? s : -INFINITY;
              acc[mi][nt][hh * 2 + e] = s;
              mx = fmaxf(mx, s);
            }
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
          float mn = fmaxf(rm[mi][hh], mx);
          float sum = 0.f;
          if (mn != -INFINITY) {
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
#pragma unroll
              for (int e = 0; e < 2; ++e) sum += exp2f(acc[mi][nt][hh * 2 + e] - mn);
            rl[mi][hh] = (rm[mi][hh] == -INFINITY ? 0.f : rl[mi][hh] * exp2f(rm[mi][hh] - mn)) + sum;
            rm[mi][hh] = mn;
          }
        }
      }
    } else {
      // column partial sums over this thread's rows
      float c1s[8][2], c2s[8][2];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          float a1 = 0.f, a2 = 0.f;
#pragma unroll
          for (int mi = 0; mi < MPW; ++mi)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              float p = exp2f(acc[mi][nt][hh * 2 + e] * sl2 - rm[mi][hh]) * rl[mi][hh];
              a1 += p;
              a2 += p * p;
            }
          c1s[nt][e] = a1;
          c2s[nt][e] = a2;
        }
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
#pragma unroll
          for (int off = 4; off < 32; off <<= 1) {
            c1s[nt][e] += __shfl_xor_sync(0xffffffffu, c1s[nt][e], off);
            c2s[nt][e] += __shfl_xor_sync(0xffffffffu, c2s[nt][e], off);
          }
        }
      if (gq == 0) {
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            int col = nt * 8 + 2 * tq + e;
            red[(warp * kPfKeys + col) * 2 + 0] = c1s[nt][e];
            red[(warp * kPfKeys + col) * 2 + 1] = c2s[nt][e];
          }
      }
      __syncthreads();
      for (int col = threadIdx.x; col < kPfKeys; col += blockDim.x) {
        int key = kbase + col;
        if (key < c1) {
          float a1 = 0.f, a2 = 0.f;
          for (int w = 0; w < nw; ++w) {  // fixed order: deterministic
            a1 += red[(w * kPfKeys + col) * 2 + 0];
            a2 += red[(w * kPfKeys + col) * 2 + 1];
          }
          acc_pf[(int64_t)u * g.max_pos + key] = make_float2(a1, a2);
        }
      }
    }
    __syncthreads();
  }

  if (!PASS2) {
#pragma unroll
    for (int mi = 0; mi < MPW; ++mi)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float l = rl[mi][hh];
        l += __shfl_xor_sync(0xffffffffu, l, 1);
        l += __shfl_xor_sync(0xffffffffu, l, 2);
        int r = (warp * MPW + mi) * 16 + gq + 8 * hh;
        if (tq == 0 && r < R)
          partials[((int64_t)u * n_chunks1 + blockIdx.x) * R + r] = make_float2(rm[mi][hh], l);
      }
  }
}

// Moments of the key-mass distribution (Eqs. 3-5) and the OQ score (Eq. 6), float64,
// fixed reduction order.  One CTA per (sequence, layer).
__device__ double block_sum_d(double v, double* sh) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
    sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

// Eq. 3 column sums of one (sequence, layer) over its local KV heads, in a fixed
// order: c_j = Σ_{h,q} Ã[h,q,j] = Σ_kvh acc1[kvh][j].  Written in float64 so a
// KV-head-sharded run can all-reduce them across ranks (collective C1).
__global__ void prefill_colsum_kernel(Geom g, const float2* __restrict__ acc_pf, int P, double* __restrict__ colsum) {
  const int bl = blockIdx.y;
  const int n = P - g.W;
  const float2* base = acc_pf + (int64_t)bl * g.Hkv * g.max_pos;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    double c = 0.0;
    for (int h = 0; h < g.Hkv; ++h) c += (double)base[(int64_t)h * g.max_pos + j].x;
    colsum[(int64_t)bl * g.max_pos + j] = c;
  }
}

__global__ void __launch_bounds__(1024) prefill_moments_kernel(Geom g, const double* __restrict__ colsum, int P,
                                                               double* __restrict__ stats, double* __restrict__ oq,
                                                               double t1, double t2, double t3, double eps,
                                                               int32_t* err) {
  __shared__ double sh[33];
  const int bl = blockIdx.x;
  const int n = P - g.W;
  const double* c = colsum + (int64_t)bl * g.max_pos;
  double z = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) z += c[j];
  const double Z = block_sum_d(z, sh);  // Eq. 3 normaliser
  const double inv_n = 1.0 / (double)n;
  double hs = 0.0, s2 = 0.0, s4 = 0.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double p = c[j] / Z;
    if (p > 0.0) hs -= p * log(p);  // Eq. 3 entropy, natural log (R2)
    double dv = p - inv_n;          // p̄ = 1/n (R4)
    double d2 = dv * dv;
    s2 += d2;
    s4 += d2 * d2;
  }
  const double H = block_sum_d(hs, sh);
  const double m2 = block_sum_d(s2, sh) / (double)n;  // Eq. 4
  const double m4 = block_sum_d(s4, sh) / (double)n;
  if (threadIdx.x == 0) {
    double K = m2 > eps ? m4 / (m2 * m2) : 1.0;  // Eq. 5, Pearson (R5); flat -> 1 (R6)
    double Hc = fmax(H, eps), Vc = fmax(m2, eps), Kc = fmax(K, eps);
    if (stats) {
      stats[bl * 3 + 0] = Hc;
      stats[bl * 3 + 1] = Vc;
      stats[bl * 3 + 2] = Kc;
    }
    const double q = pow(Hc, 1.0 / t1) * pow(Vc, 1.0 / t2) * pow(Kc, 1.0 / t3);  // Eq. 6
    oq[bl] = q;
    // a NaN / Inf in q_win or K reaches the column sums
    if (!isfinite(Z) || !isfinite(q)) atomicOr(err, kErrNonFinite);
  }
}

template <int KD, int MPW>
static int launch_passes(const Geom& g, const uint16_t* q_win, const uint16_t* k, int P, float2* partials,
                         int n_chunks1, float2* acc_pf, cudaStream_t s) {
  const int R = g.G * g.W;
  const int mtiles = (R + 15) / 16;
  const int warps = (mtiles + MPW - 1) / MPW;
  const int threads = warps * 32;
  constexpr int D = KD * 16;
  size_t sm1 = (size_t)2 * kPfKeys * (D + 8) * 2;
  size_t sm2 = sm1 + (size_t)warps * kPfKeys * 2 * 4 + (size_t)2 * R * 4;
  auto k1 = prefill_pass_kernel<KD, MPW, false>;
  auto k2 = prefill_pass_kernel<KD, MPW, true>;
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  dim3 gr1(n_chunks1, g.n_units);
  k1<<<gr1, threads, sm1, s>>>(g, q_win, k, P, partials, n_chunks1, acc_pf);
  int n_chunks2 = (P - g.W + kPfChunk - 1) / kPfChunk;
  dim3 gr2(n_chunks2, g.n_units);
  k2<<<gr2, threads, sm2, s>>>(g, q_win, k, P, partials, n_chunks1, acc_pf);
  return 2;
}

bool prefill_ws_available(const Geom& g);  // k_prefill_ws.cu
int launch_prefill_ws(const Geom& g, const uint16_t* q_win, const uint16_t* k, int P, float2* partials, int n_chunks1,
                      float2* acc_pf, int num_sms, cudaStream_t s);  // k_prefill_ws.cu

int launch_prefill_begin(const Geom& g, const uint16_t* q_win, const uint16_t* k, int P, float* partials,
                         int n_chunks1, float2* acc_pf, double* colsum, cudaStream_t s) {
  // the warp-specialised persistent tcgen05 kernel (k_prefill_ws.cu) for G*W = 128, d = 128;
  // the mma.sync passes below for every other shape (ARKV_PREFILL_MMA=1 in tuning builds)
  if (prefill_ws_available(g) && tuning_knob("ARKV_PREFILL_MMA", 0) == 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int n = launch_prefill_ws(g, q_win, k, P, (float2*)partials, n_chunks1, acc_pf, sms, s);
    if (n >= 0) {
      dim3 grid((P - g.W + 255) / 256, g.batch * g.L);
      prefill_colsum_kernel<<<grid, 256, 0, s>>>(g, acc_pf, P, colsum);
      return n + 1;
    }
  }
  const int R = g.G * g.W;
  const int mtiles = (R + 15) / 16;
  const bool two = (mtiles % 2 == 0) && mtiles >= 2;
  int n = 0;
  float2* pp = (float2*)partials;
#define PF_CASE(KDV)                                                            \
  case KDV:                                                                     \
    n += two ? launch_passes<KDV, 2>(g, q_win, k, P, pp, n_chunks1, acc_pf, s)  \
             : launch_passes<KDV, 1>(g, q_win, k, P, pp, n_chunks1, acc_pf, s); \
    break;
  switch (g.d / 16) {
    PF_CASE(1)
    PF_CASE(2)
    PF_CASE(4)
    PF_CASE(8)
    default:
      return -1;
  }
#undef PF_CASE
  dim3 grid((P - g.W + 255) / 256, g.batch * g.L);
  prefill_colsum_kernel<<<grid, 256, 0, s>>>(g, acc_pf, P, colsum);
  return n + 1;
}

int launch_prefill_finish(const Geom& g, const double* colsum, int P, double* stats, double* oq, const double* tau,
                          double stat_eps, int32_t* err, cudaStream_t s) {
  prefill_moments_kernel<<<g.batch * g.L, 1024, 0, s>>>(g, colsum, P, stats, oq, tau[0], tau[1], tau[2], stat_eps,
                                                         err);
  return 1;
}

}  // namespace arkv
