// k_prefill_tc.cu — prefill attention statistics (P1) on the 5th-generation tensor cores.
//
// Same two passes as k_prefill.cu (Eq. 2; R1), for the paper's shapes
// (G·W = 128 window-query rows per KV head, d = 128):
//   pass 1: S = Q·K^T   (UMMA M = 128 query rows, N = 128 keys)  -> TMEM lane = row:
//           running row max / sum-exp stay thread-local;
//   pass 2: S^T = K·Q^T (UMMA M = 128 keys, N = 128 query rows)  -> TMEM lane = key:
//           acc1 = Σ_rows p, acc2 = Σ_rows p² stay thread-local (HH seed, Eq. 9 samples).
// Operands are staged in shared memory in the canonical K-major SWIZZLE_128B layout
// (8-row x 128-byte atoms, 16-byte chunk index XOR row % 8), one tcgen05.mma per
// 16-element K step issued by a single thread, accumulators double-buffered in TMEM
// (2 x 128 fp32 columns) so the epilogue of tile i overlaps the MMA of tile i + 1,
// completion signalled by tcgen05.commit on an mbarrier.  K tiles stream through a
// 2-deep cp.async ring (the next tile loads while the epilogue of the previous one runs),
// so two CTAs fit an SM.  8 warps: warps w and w + 4 read the same 32 TMEM lanes, each
// half of the 128 columns.
#include "kernels.h"

namespace arkv {
namespace pftc {

constexpr int D = 128;
constexpr int R = 128;                 // G·W rows
constexpr int NK = 128;                // keys per tile
constexpr int kChunk = 2048;           // keys per CTA (same partial layout as k_prefill.cu)
constexpr int kSub = 128 * 128;        // one [128 rows x 64 bf16] SW128 sub-tile (16 KB)
constexpr int kTileB = 2 * kSub;       // [128 x 128] bf16 = 32 KB
constexpr int kBufs = 2;  // 2 CTAs per SM (smem ~101 KB each; TMEM 2 x 256 columns)
constexpr int kThreads = 256;

struct __align__(8) Ctl {
  uint64_t mbar[2];
  uint32_t tmem;
  float rowc[R];  // pass 2: row max + log2(row sum) of pass 1
  float red[2][R][2];  // combine of the two column halves
};
constexpr int kSmem = 1024 /*align slack*/ + kTileB * (1 + kBufs) + (int)sizeof(Ctl);

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// 2^x on the SFU without exp2f's denormal fix-up (values below 2^-126 flush to 0)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool pred) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(pred ? 16 : 0));
}
// Row r, 16-byte chunk c (0..15 across the 128 dims) of a [128 x 128] bf16 tile.
__device__ __forceinline__ uint32_t sw128_off(int r, int c) {
  return (uint32_t)((c >> 3) * kSub + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}
// K-major SWIZZLE_128B UMMA shared-memory descriptor (SBO = 1024 B between 8-row groups).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(1024u >> 4) << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}
// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both K-major, M = 128, N = 128.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void mma_ss(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// 32 lanes x 32 consecutive fp32 columns of TMEM -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

template <bool PASS2>
__global__ void __launch_bounds__(kThreads, 2) prefill_tc_kernel(Geom g, const uint16_t* __restrict__ q_win,
                                                                 const uint16_t* __restrict__ kmat, int P,
                                                                 float2* __restrict__ partials, int n_chunks1,
                                                                 float2* __restrict__ acc_pf) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // SW128 atoms must be 1024-byte aligned
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sQ = base, sK = base + kTileB;
  Ctl& ctl = *reinterpret_cast<Ctl*>(gbase + kTileB * (1 + kBufs));

  const int u = blockIdx.y, kvh = u % g.Hkv, bl = u / g.Hkv;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int quad = warp & 3, half = warp >> 2;  // TMEM lanes 32*quad.., columns 64*half..
  const int key_end = PASS2 ? (P - g.W) : P;
  const int c0 = blockIdx.x * kChunk, c1 = min(c0 + kChunk, key_end);
  if (c0 >= c1) return;
  const int n_tiles = (c1 - c0 + NK - 1) / NK;
  const uint16_t* qb = q_win + ((int64_t)bl * g.Hq + kvh * g.G) * g.W * D;
  const uint16_t* kb = kmat + ((int64_t)bl * g.Hkv + kvh) * (int64_t)P * D;
  const float sl2 = g.sm_scale * 1.4426950408889634f;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(su32(&ctl.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&ctl.mbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // Q tile (all 128 rows x 128 dims) and the first K tiles
  for (int i = threadIdx.x; i < R * 16; i += kThreads) {
    const int r = i >> 4, c = i & 15;
    cp16(sQ + sw128_off(r, c), qb + (int64_t)r * D + c * 8, true);
  }
  auto load_k = [&](int t) {
    const int buf = t % kBufs, kb0 = c0 + t * NK;
    for (int i = threadIdx.x; i < NK * 16; i += kThreads) {
      const int r = i >> 4, c = i & 15;
      const int key = kb0 + r;
      const bool ok = key < c1;
      cp16(sK + buf * kTileB + sw128_off(r, c), kb + (int64_t)(ok ? key : c0) * D + c * 8, ok);
    }
  };
  load_k(0);
  if (n_tiles > 1) load_k(1);
  asm volatile("cp.async.commit_group;\n");
  // row statistics of pass 1 (pass 2 only)
  if (PASS2) {
    for (int r = threadIdx.x; r < R; r += kThreads) {
      const float2* pr = partials + (int64_t)u * n_chunks1 * R + r;
      float M = -INFINITY;
      for (int c = 0; c < n_chunks1; ++c) M = fmaxf(M, pr[(int64_t)c * R].x);
      float L = 0.f;
      for (int c = 0; c < n_chunks1; ++c) {
        const float2 v = pr[(int64_t)c * R];
        if (v.y > 0.f) L += v.y * exp2f(v.x - M);
      }
      ctl.rowc[r] = M + log2f(L);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = ctl.tmem;

  // per-thread state: pass 1 -> row statistics of row r; pass 2 -> nothing carried
  const int my_lane = quad * 32 + lane;  // TMEM lane: query row (pass 1) or key (pass 2)
  float run_m = -INFINITY, run_l = 0.f;

  auto epilogue = [&](int t) {
    const int acc = t & 1;
    mbar_wait(&ctl.mbar[acc], (t >> 1) & 1);
    // MMA t is complete: its K buffer takes tile t + 2, loading behind this epilogue
    if (t + 2 < n_tiles) load_k(t + 2);
    asm volatile("cp.async.commit_group;\n");
    __syncwarp();  // tcgen05.ld is .aligned: reconverge after the spin-wait
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * 128 + half * 64);
    const int kbase = c0 + t * NK;
    if (!PASS2) {
      const int r = my_lane;
      const int qp = P - g.W + (r % g.W);  // query position of row r = h*W + i
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        float v[32];
        tmem_ld32(taddr + cc * 32, v);
        float mx = -INFINITY;
        const int key0 = kbase + half * 64 + cc * 32;
        if (key0 + 31 < c1 && key0 + 31 <= P - g.W) {  // no key masked (all but the last tiles)
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v[i] *= sl2;
            mx = fmaxf(mx, v[i]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int key = key0 + i;
            v[i] = (key < c1 && key <= qp) ? v[i] * sl2 : -INFINITY;
            mx = fmaxf(mx, v[i]);
          }
        }
        const float mn = fmaxf(run_m, mx);
        if (mn != -INFINITY) {
          float sum = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) sum += ex2(v[i] - mn);
          run_l = (run_m == -INFINITY ? 0.f : run_l * ex2(run_m - mn)) + sum;
          run_m = mn;
        }
      }
    } else {
      const int key = kbase + my_lane;
      float a1 = 0.f, a2 = 0.f;
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        float v[32];
        tmem_ld32(taddr + cc * 32, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          // p = 2^(s - m_r) / l_r = 2^(s - (m_r + log2 l_r)): one row constant per element
          const float p = ex2(fmaf(v[i], sl2, -ctl.rowc[half * 64 + cc * 32 + i]));
          a1 += p;
          a2 += p * p;
        }
      }
      ctl.red[half][my_lane][0] = a1;
      ctl.red[half][my_lane][1] = a2;
      asm volatile("bar.sync 1, %0;\n" ::"n"(kThreads) : "memory");
      if (half == 0 && key < c1) {
        const float s1 = ctl.red[0][my_lane][0] + ctl.red[1][my_lane][0];
        const float s2 = ctl.red[0][my_lane][1] + ctl.red[1][my_lane][1];
        acc_pf[(int64_t)u * g.max_pos + key] = make_float2(s1, s2);
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(kThreads) : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  };

  for (int t = 0; t < n_tiles; ++t) {
    // K tile t landed (and Q): make the generic-proxy cp.async writes visible to the
    // tensor core's async proxy, then one thread issues the 8 K-steps of the MMA
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t kt = sK + (t % kBufs) * kTileB;
      const uint32_t a_base = PASS2 ? kt : sQ, b_base = PASS2 ? sQ : kt;
      const uint32_t d = tmem + (uint32_t)((t & 1) * 128);
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        const uint32_t off = (ks >> 2) * kSub + (ks & 3) * 32;
        mma_ss(d, umma_desc(a_base + off), umma_desc(b_base + off), ks > 0 ? 1u : 0u);
      }
      mma_commit(&ctl.mbar[t & 1]);
    }
    if (t >= 1) epilogue(t - 1);  // overlaps MMA t; loads tile t + 1 into MMA t - 1's buffer
  }
  epilogue(n_tiles - 1);

  if (!PASS2) {
    // merge the two column halves of each row and write the chunk partial
    ctl.red[half][my_lane][0] = run_m;
    ctl.red[half][my_lane][1] = run_l;
    __syncthreads();
    if (half == 0) {
      const float m0 = ctl.red[0][my_lane][0], l0 = ctl.red[0][my_lane][1];
      const float m1 = ctl.red[1][my_lane][0], l1 = ctl.red[1][my_lane][1];
      const float M = fmaxf(m0, m1);
      float L = 0.f;
      if (m0 != -INFINITY) L += l0 * exp2f(m0 - M);
      if (m1 != -INFINITY) L += l1 * exp2f(m1 - M);
      partials[((int64_t)u * n_chunks1 + blockIdx.x) * R + my_lane] = make_float2(M, L);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
  }
}

}  // namespace pftc

bool prefill_tc_available(const Geom& g) { return g.d == pftc::D && g.G * g.W == pftc::R; }

int launch_prefill_tc(const Geom& g, const uint16_t* q_win, const uint16_t* k, int P, float2* partials, int n_chunks1,
                      float2* acc_pf, cudaStream_t s) {
  if (!prefill_tc_available(g)) return -1;
  auto k1 = pftc::prefill_tc_kernel<false>;
  auto k2 = pftc::prefill_tc_kernel<true>;
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, pftc::kSmem);
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, pftc::kSmem);
  dim3 gr1((P + pftc::kChunk - 1) / pftc::kChunk, g.n_units);
  k1<<<gr1, pftc::kThreads, pftc::kSmem, s>>>(g, q_win, k, P, partials, n_chunks1, acc_pf);
  dim3 gr2((P - g.W + pftc::kChunk - 1) / pftc::kChunk, g.n_units);
  k2<<<gr2, pftc::kThreads, pftc::kSmem, s>>>(g, q_win, k, P, partials, n_chunks1, acc_pf);
  return 2;
}

}  // namespace arkv
