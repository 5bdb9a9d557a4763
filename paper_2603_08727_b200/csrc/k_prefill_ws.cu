// k_prefill_ws.cu — prefill attention statistics (P1) on the 5th-generation tensor cores,
// warp-specialised and persistent.
//
// The same two passes as k_prefill_tc.cu (Eq. 2; R1) for the paper's shapes
// (G·W = 128 window-query rows per KV head, d = 128):
//   pass 1: S = Q·K^T   (UMMA M = 128 query rows, N = 128 keys)  -> TMEM lane = row:
//           running row max / sum-exp per (unit, 2048-key chunk);
//   pass 2: S^T = K·Q^T (UMMA M = 128 keys, N = 128 query rows)  -> TMEM lane = key:
//           acc1 = Σ_rows p, acc2 = Σ_rows p² (HH seed, Eq. 9 samples) and the column sums.
// What differs from k_prefill_tc.cu (one CTA per chunk, all threads loading with cp.async,
// two K buffers, one tile in flight): one CTA per SM walks a contiguous range of
// (unit, chunk) items with
//   warp 0  TMA producer: Q once per unit and 128-key K tiles, both as two [128 x 64]
//           SWIZZLE_128B boxes (the canonical K-major UMMA layout), into a 4-stage ring
//           completing on mbarriers (expect_tx);
//   warp 1  MMA issuer: 8 tcgen05.mma per tile into one of 4 TMEM accumulators
//           (4 x 128 fp32 columns = all 512), tcgen05.commit frees the K stage and
//           publishes the accumulator;
//   warps 2.. epilogue (16): tcgen05.ld of their lane quadrant (warp % 4) and column group,
//           exponentials, reductions; one arrive per warp frees the accumulator.
// So up to 3 K tiles are in flight while the epilogue works, and no thread waits on its own
// loads.
#include <cuda.h>

#include <mutex>

#include "kernels.h"

namespace arkv {
namespace pfws {

constexpr int D = 128;
constexpr int R = 128;               // G·W rows
constexpr int NK = 128;              // keys per tile
constexpr int kChunk = 2048;         // keys per item (same partial layout as k_prefill.cu)
constexpr int kSub = 128 * 128;      // one [128 rows x 64 bf16] SW128 box (16 KB)
constexpr int kTileB = 2 * kSub;     // [128 x 128] bf16 = 32 KB
constexpr int kStages = 4;           // K ring
constexpr int kAcc = 4;              // TMEM accumulators (128 columns each)
#ifndef ARKV_PF_EPI_WARPS
#define ARKV_PF_EPI_WARPS 16
#endif
constexpr int kEpiWarps = ARKV_PF_EPI_WARPS;  // 4 lane quadrants x kCG column groups
constexpr int kCG = kEpiWarps / 4;
constexpr int kCols = 128 / kCG;             // accumulator columns per epilogue warp
static_assert(kCols == 32 || kCols == 64, "column group of 32 or 64");
// Pass-2 epilogue split: kTG = 1 -> the kCG warp groups take alternate tiles (each warp all
// 128 columns of its lane quadrant, no per-tile reduction or barrier); 0 -> every tile is
// split into kCG column groups reduced through shared memory (pass 1 always: its per-row
// running max/sum merge only once per item).  Requires kCG == kAcc.  Measured at configs[1]:
// pass 2 409 -> 373 us (ncu), both passes 0.866 -> 0.823 ms.
#ifndef ARKV_PF_TILE_GROUPS
#define ARKV_PF_TILE_GROUPS 1
#endif
constexpr bool kTG = ARKV_PF_TILE_GROUPS != 0;
constexpr int kThreads = 32 * (2 + kEpiWarps);

struct __align__(8) Ctl {
  uint64_t full[kStages], empty[kStages];
  uint64_t acc_full[kAcc], acc_empty[kAcc];
  uint64_t q_full, q_empty;
  uint32_t tmem;
  alignas(16) float rowc[R];  // pass 2: row max + log2(row sum) of pass 1, current unit (float4 reads)
  float red[2][kCG][R][2];  // combine of the column groups (pass 2: double-buffered by tile)
};
constexpr int kSmem = 1024 /*align slack*/ + kTileB * (1 + kStages) + (int)sizeof(Ctl);

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}
// 2^x for x <= 0 on the FMA pipe (offloads every kPolyEvery-th exponential from the MUFU
// unit; measured at configs[1]: every 3rd 1.00 ms, every 4th 0.92, every 8th 0.83, off
// 0.83-0.87 ms — the epilogue is issue-bound as much as MUFU-bound, so it is off).  x = n + f with n = rint(x) (magic-number
// rounding), f in [-1/2, 1/2]; 2^f by a degree-5 least-squares polynomial (max relative
// error 2.3e-7 in fp32 Horner, the same order as ex2.approx); 2^n added to the exponent
// bits.  x is clamped at -126 (the MUFU path flushes such values to 0; here they give
// ~1e-38).
#ifndef ARKV_PF_POLY_EVERY
#define ARKV_PF_POLY_EVERY 0
#endif
constexpr int kPolyEvery = ARKV_PF_POLY_EVERY;
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: rint(x) in the low mantissa bits
  const float f = x - (t - 12582912.f);
  float p = 1.3266970636323094e-3f;
  p = fmaf(p, f, 9.675459936261177e-3f);
  p = fmaf(p, f, 5.550742521882057e-2f);
  p = fmaf(p, f, 2.4022121727466583e-1f);
  p = fmaf(p, f, 6.931469440460205e-1f);
  p = fmaf(p, f, 1.0000001192092896f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}
// j: the element's index in a fully unrolled loop (folds to one path per element)
__device__ __forceinline__ float ex2_mix(float x, int j) {
  return (kPolyEvery > 0 && (j % (kPolyEvery > 0 ? kPolyEvery : 1)) == kPolyEvery - 1) ? ex2_poly(x) : ex2(x);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes) : "memory");
}
// 2-D TMA box load (SWIZZLE_128B per the tensor map) completing on an mbarrier
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* tm, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
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

// The CTA's items [i0, i1) of the flattened (unit, chunk) list, walked identically by the
// three roles.
struct Walk {
  int n_chunks, key_end;
  __device__ void item(int i, int& u, int& c0, int& c1, int& nt) const {
    u = i / n_chunks;
    c0 = (i % n_chunks) * kChunk;
    c1 = min(c0 + kChunk, key_end);
    nt = (c1 - c0 + NK - 1) / NK;
  }
};

template <bool PASS2>
__global__ void __launch_bounds__(kThreads, 1)
    prefill_ws_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK, Geom g, int P,
                      float2* __restrict__ partials, int n_chunks1, float2* __restrict__ acc_pf, int n_items) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // SW128 atoms must be 1024-byte aligned
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sQ = base, sK = base + kTileB;
  Ctl& ctl = *reinterpret_cast<Ctl*>(gbase + kTileB * (1 + kStages));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  Walk w;
  w.key_end = PASS2 ? (P - g.W) : P;
  w.n_chunks = (w.key_end + kChunk - 1) / kChunk;
  const int i0 = (int)((int64_t)blockIdx.x * n_items / gridDim.x);
  const int i1 = (int)((int64_t)(blockIdx.x + 1) * n_items / gridDim.x);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(su32(&ctl.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 32) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&ctl.full[i], 1);
      mbar_init(&ctl.empty[i], 1);
    }
    for (int i = 0; i < kAcc; ++i) {
      mbar_init(&ctl.acc_full[i], 1);
      mbar_init(&ctl.acc_empty[i], (PASS2 && kTG) ? 4 : kEpiWarps);  // the warps that read accumulator i
    }
    mbar_init(&ctl.q_full, 1);
    mbar_init(&ctl.q_empty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = ctl.tmem;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmK)) : "memory");
      asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmQ)) : "memory");
      int T = 0, cur_u = -1, n_q = 0;
      for (int i = i0; i < i1; ++i) {
        int u, c0, c1, nt;
        w.item(i, u, c0, c1, nt);
        if (u != cur_u) {
          // a new unit's Q: after every MMA reading the previous one has completed
          if (n_q > 0) mbar_wait(&ctl.q_empty, (n_q - 1) & 1);
          const int kvh = u % g.Hkv, bl = u / g.Hkv;
          const int qrow = (bl * g.Hq + kvh * g.G) * g.W;
          mbar_expect_tx(&ctl.q_full, kTileB);
          tma_2d(sQ, &tmQ, 0, qrow, &ctl.q_full);
          tma_2d(sQ + kSub, &tmQ, 64, qrow, &ctl.q_full);
          cur_u = u;
          ++n_q;
        }
        for (int t = 0; t < nt; ++t, ++T) {
          const int st = T % kStages;
          if (T >= kStages) mbar_wait(&ctl.empty[st], ((T / kStages) - 1) & 1);
          const int row = u * P + c0 + t * NK;
          const uint32_t dst = sK + st * kTileB;
          mbar_expect_tx(&ctl.full[st], kTileB);
          tma_2d(dst, &tmK, 0, row, &ctl.full[st]);
          tma_2d(dst + kSub, &tmK, 64, row, &ctl.full[st]);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int T = 0, cur_u = -1, n_q = 0;
      for (int i = i0; i < i1; ++i) {
        int u, c0, c1, nt;
        w.item(i, u, c0, c1, nt);
        if (u != cur_u) {
          if (n_q > 0) mma_commit(&ctl.q_empty);  // the previous unit's MMAs are all issued
          mbar_wait(&ctl.q_full, n_q & 1);
          cur_u = u;
          ++n_q;
        }
        for (int t = 0; t < nt; ++t, ++T) {
          const int st = T % kStages, ac = T % kAcc;
          mbar_wait(&ctl.full[st], (T / kStages) & 1);
          if (T >= kAcc) mbar_wait(&ctl.acc_empty[ac], ((T / kAcc) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t kt = sK + st * kTileB;
          const uint32_t a_base = PASS2 ? kt : sQ, b_base = PASS2 ? sQ : kt;
          const uint32_t d = tmem + (uint32_t)(ac * 128);
#pragma unroll
          for (int ks = 0; ks < D / 16; ++ks) {
            const uint32_t off = (ks >> 2) * kSub + (ks & 3) * 32;
            mma_ss(d, umma_desc(a_base + off), umma_desc(b_base + off), ks > 0 ? 1u : 0u);
          }
          mma_commit(&ctl.empty[st]);
          mma_commit(&ctl.acc_full[ac]);
        }
      }
    }
  } else {
    // ===================== epilogue (kEpiWarps warps) =====================
    // named barriers: 1 = all epilogue warps, 2 + quad = the kCG warps of one lane quadrant
    const int quad = warp & 3, half = (warp - 2) >> 2;  // TMEM lanes 32*quad.., columns kCols*half..
    const int my_lane = quad * 32 + lane;               // query row (pass 1) or key (pass 2)
    const int etid = threadIdx.x - 64;                  // 0..32*kEpiWarps-1
    const float sl2 = g.sm_scale * 1.4426950408889634f;
    int T = 0, cur_u = -1;
    float rc[PASS2 && !kTG ? kCols : 1];  // pass 2, column groups: this warp's row constants
    for (int i = i0; i < i1; ++i) {
      int u, c0, c1, nt;
      w.item(i, u, c0, c1, nt);
      if (PASS2 && u != cur_u) {
        // row constants of this unit from the pass-1 chunk partials
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kEpiWarps) : "memory");
        if (etid < R) {
          const float2* pr = partials + (int64_t)u * n_chunks1 * R + etid;
          float M = -INFINITY;
          for (int c = 0; c < n_chunks1; ++c) M = fmaxf(M, pr[(int64_t)c * R].x);
          float L = 0.f;
          for (int c = 0; c < n_chunks1; ++c) {
            const float2 v = pr[(int64_t)c * R];
            if (v.y > 0.f) L += v.y * exp2f(v.x - M);
          }
          ctl.rowc[etid] = M + log2f(L);
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kEpiWarps) : "memory");
#pragma unroll
        for (int j = 0; j < (PASS2 && !kTG ? kCols : 1); ++j) rc[j] = ctl.rowc[half * kCols + j];
      }
      cur_u = u;
      float run_m = -INFINITY, run_l = 0.f;
      const int qp = P - g.W + (my_lane % g.W);  // pass 1: query position of row my_lane = h*W + i
      for (int t = 0; t < nt; ++t, ++T) {
        // tile groups (kTG): group `half` takes the tiles T = half (mod kCG), all 128 columns
        // of its lane quadrant — no cross-warp reduction, no per-tile barrier
        if (PASS2 && kTG && (T % kCG) != half) continue;
        const int ac = T % kAcc;
        mbar_wait(&ctl.acc_full[ac], (T / kAcc) & 1);
        __syncwarp();
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        constexpr int NC = (PASS2 && kTG) ? 128 : kCols;  // this warp's accumulator columns
        const int col0 = (PASS2 && kTG) ? 0 : half * kCols;
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(ac * 128 + col0);
        const int kbase = c0 + t * NK;
        if (!PASS2) {
          // one 32-column chunk in registers at a time; the accumulator is released once
          // its last chunk has been read
          float v[1][32];
#pragma unroll
          for (int cc0 = 0; cc0 < NC / 32; ++cc0) {
            tmem_ld32(taddr + cc0 * 32, v[0]);
            if (cc0 == NC / 32 - 1) {
              asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
              __syncwarp();
              if (lane == 0) mbar_arrive(&ctl.acc_empty[ac]);
            }
            const int cc = 0;
            float mx = -INFINITY;
            const int key0 = kbase + col0 + cc0 * 32;
            bool raw = false;
            if (key0 + 31 < c1 && key0 + 31 <= P - g.W) {  // no key masked (all but the last tiles)
              // max on the raw logits: x -> x * sl2 (sl2 > 0) is monotone, and so is rounding
#pragma unroll
              for (int j = 0; j < 32; ++j) mx = fmaxf(mx, v[cc][j]);
              mx *= sl2;
              raw = true;
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const int key = key0 + j;
                v[cc][j] = (key < c1 && key <= qp) ? v[cc][j] * sl2 : -INFINITY;
                mx = fmaxf(mx, v[cc][j]);
              }
            }
            const float mn = fmaxf(run_m, mx);
            if (mn != -INFINITY) {
              float sum = 0.f;
              if (raw) {
#pragma unroll
                for (int j = 0; j < 32; ++j) sum += ex2_mix(fmaf(v[cc][j], sl2, -mn), j);
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j) sum += ex2(v[cc][j] - mn);
              }
              run_l = (run_m == -INFINITY ? 0.f : run_l * ex2(run_m - mn)) + sum;
              run_m = mn;
            }
          }
        } else {
          const int key = kbase + my_lane;
          float a1 = 0.f, a2 = 0.f;
          if (kTG) {
            // 4 x 32 columns, each chunk processed as soon as it is in registers; the row
            // constants come from shared memory (broadcast float4 reads)
#pragma unroll
            for (int cc = 0; cc < NC / 32; ++cc) {
              float v[32];
              tmem_ld32(taddr + cc * 32, v);
              if (cc == NC / 32 - 1) {
                asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(&ctl.acc_empty[ac]);
              }
#pragma unroll
              for (int j4 = 0; j4 < 8; ++j4) {
                const float4 r4 = *(const float4*)&ctl.rowc[cc * 32 + 4 * j4];
                const float rr[4] = {r4.x, r4.y, r4.z, r4.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float p = ex2_mix(fmaf(v[4 * j4 + e], sl2, -rr[e]), 4 * j4 + e);
                  a1 += p;
                  a2 += p * p;
                }
              }
            }
            if (key < c1) acc_pf[(int64_t)u * g.max_pos + key] = make_float2(a1, a2);
          } else {
            float v[NC / 32][32];
#pragma unroll
            for (int cc = 0; cc < NC / 32; ++cc) tmem_ld32(taddr + cc * 32, v[cc]);
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&ctl.acc_empty[ac]);
#pragma unroll
            for (int cc = 0; cc < NC / 32; ++cc)
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                // p = 2^(s - m_r) / l_r = 2^(s - (m_r + log2 l_r)): one row constant per element
                const float p = ex2_mix(fmaf(v[cc][j], sl2, -rc[PASS2 && !kTG ? cc * 32 + j : 0]), j);
                a1 += p;
                a2 += p * p;
              }
            // the quadrant's kCG warps hold the same keys: one barrier per tile (the buffer
            // is reused two tiles later, behind the next tile's barrier)
            float(&rd)[kCG][R][2] = ctl.red[T & 1];
            rd[half][my_lane][0] = a1;
            rd[half][my_lane][1] = a2;
            asm volatile("bar.sync %0, %1;\n" ::"r"(2 + quad), "n"(32 * kCG) : "memory");
            if (half == 0 && key < c1) {
              float s1 = rd[0][my_lane][0], s2 = rd[0][my_lane][1];
#pragma unroll
              for (int cg = 1; cg < kCG; ++cg) {
                s1 += rd[cg][my_lane][0];
                s2 += rd[cg][my_lane][1];
              }
              acc_pf[(int64_t)u * g.max_pos + key] = make_float2(s1, s2);
            }
          }
        }
      }
      if (!PASS2) {
        // merge the two column halves of each row and write the chunk partial
        ctl.red[0][half][my_lane][0] = run_m;
        ctl.red[0][half][my_lane][1] = run_l;
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kEpiWarps) : "memory");
        if (half == 0) {
          float M = -INFINITY;
#pragma unroll
          for (int cg = 0; cg < kCG; ++cg) M = fmaxf(M, ctl.red[0][cg][my_lane][0]);
          float L = 0.f;
#pragma unroll
          for (int cg = 0; cg < kCG; ++cg) {
            const float mc = ctl.red[0][cg][my_lane][0];
            if (mc != -INFINITY) L += ctl.red[0][cg][my_lane][1] * exp2f(mc - M);
          }
          partials[((int64_t)u * n_chunks1 + (c0 / kChunk)) * R + my_lane] = make_float2(M, L);
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kEpiWarps) : "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiled)p;
  });
  return fn;
}
// rows x 128 bf16 (row-major), boxes of [128 rows x 64 dims] with the 128-byte swizzle
static bool make_map(CUtensorMap* m, const void* ptr, int64_t rows) {
  EncodeTiled fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace pfws

bool prefill_ws_available(const Geom& g) { return g.d == pfws::D && g.G * g.W == pfws::R; }

// Both passes; returns the launches issued, or -1 (shape not supported / no tensor-map
// encoder: the caller falls back to k_prefill_tc.cu).
int launch_prefill_ws(const Geom& g, const uint16_t* q_win, const uint16_t* k, int P, float2* partials, int n_chunks1,
                      float2* acc_pf, int num_sms, cudaStream_t s) {
  if (!prefill_ws_available(g)) return -1;
  CUtensorMap tmQ, tmK;
  if (!pfws::make_map(&tmQ, q_win, (int64_t)g.batch * g.L * g.Hq * g.W) ||
      !pfws::make_map(&tmK, k, (int64_t)g.n_units * P))
    return -1;
  auto k1 = pfws::prefill_ws_kernel<false>;
  auto k2 = pfws::prefill_ws_kernel<true>;
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, pfws::kSmem);
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, pfws::kSmem);
  const int items1 = g.n_units * ((P + pfws::kChunk - 1) / pfws::kChunk);
  const int items2 = g.n_units * ((P - g.W + pfws::kChunk - 1) / pfws::kChunk);
  k1<<<std::min(num_sms, items1), pfws::kThreads, pfws::kSmem, s>>>(tmQ, tmK, g, P, partials, n_chunks1, acc_pf,
                                                                     items1);
  k2<<<std::min(num_sms, items2), pfws::kThreads, pfws::kSmem, s>>>(tmQ, tmK, g, P, partials, n_chunks1, acc_pf,
                                                                     items2);
  return 2;
}

}  // namespace arkv
