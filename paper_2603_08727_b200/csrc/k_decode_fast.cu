// k_decode_fast.cu — tensor-core decode attention over O ∪ Q for FRAG-layout caches
// (d = 128, 4-bit codes, G in {1,2,4,8}).  D1, D3, D7 of DESIGN.md §2.
//
// One CTA = one split of one unit: 1 producer warp + 4 consumer warps.
//  * The producer streams whole 32-token tiles (16 KB Original, 4.5 KB Quantized)
//    from HBM into a shared-memory ring with cp.async.bulk (the 1-D TMA engine,
//    SASS UBLKCP) completing on mbarriers — no registers are spent on bytes in
//    flight, and one CTA keeps up to kStages tiles in flight.
//  * Consumer warp c takes tiles c, c+4, ...  The FRAG layout (common.cuh) stores
//    every tile as lane-linear 16-byte quads, so each LDS.128 returns exactly a
//    lane's mma.sync.m16n8k16 operand registers (no transposes, no bank conflicts).
//      QK^T:  S[32 tok x 8] = K[32 x 128] · q^T    (M = tokens, N = heads padded to 8)
//      PV:    O^T[128 x 8] += V^T[128 x 32] · P'^T (M = dims, N = heads x {hi, lo})
//    Original tiles run bf16 x bf16; Quantized tiles run f16 x f16 on codes unpacked
//    in registers with one LOP3 per two codes (fp16 "1024 + c" magic, minus 1024),
//    the per-token scale/zero factored out of the contraction (x̃ = c·s + z,
//    P:296-297): logit = s_k·(q·c) + z_k·Σq, and P' = p·s_v with Σ p·z_v added at
//    the end.  P' is split into hi + lo halves (two columns each) so the 16-bit
//    operand keeps ~22 bits, and is transposed from the QK accumulator layout into
//    the PV operand layout with movmatrix.  Online softmax in the log2 domain.
//  * HH accumulation (Eq. 9, R19): in the W steps before a tailor the logits are
//    written out for the combine kernel; the new token (D1) is appended by the CTA
//    owning the last Original tile and folded into its partial.
#include <cstdlib>

#include "combine.cuh"

namespace arkv {

namespace fast {

constexpr int D = 128;
// C consumer warps, each owning SPW ring stages: item i -> warp i % C -> stage
// (i % C) + C * ((i / C) % SPW).  Every stage's mbarriers are thus waited on strictly in
// phase order by a single warp.  (A stage shared round-robin by several warps lets a
// fast warp wait two phases ahead, where try_wait.parity reports the preceding phase as
// complete — a real bug hit with 6 stages / 4 warps.)
constexpr int kStageBytes = 32 * 4 * D;  // one Original tile (16 KB) — the largest
constexpr float kLog2e = 1.4426950408889634f;

// ---- PTX helpers ------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
// Waits for the phase with the given parity; the suspend-time hint lets the hardware
// park the thread until the phase completes instead of spinning.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// ... with an L2 eviction policy (cache tiles are read once per step: evict_first)
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// Bulk prefetch of [src, src + bytes) into L2 (no completion tracking).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}
__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_f16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t movtrans(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(d) : "r"(a));
  return d;
}
__device__ __forceinline__ uint32_t lop3_mask_or(uint32_t a, uint32_t mask, uint32_t orv) {
  uint32_t d;
  asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(d) : "r"(a), "r"(mask), "r"(orv));  // (a & b) | c
  return d;
}
__device__ __forceinline__ uint32_t hsub2_1024(uint32_t x) {
  uint32_t d;
  const uint32_t m = 0x64006400u;
  asm volatile("sub.f16x2 %0, %1, %2;\n" : "=r"(d) : "r"(x), "r"(m));
  return d;
}
// 8 nibbles -> four f16x2 code pairs (exact small integers): (n0,n4), 16(n1,n5), (n2,n6), 16(n3,n7)
__device__ __forceinline__ void unpack8(uint32_t w, uint32_t (&x)[4]) {
  const uint32_t w8 = w >> 8;
  x[0] = hsub2_1024(lop3_mask_or(w, 0x000F000Fu, 0x64006400u));
  x[1] = hsub2_1024(lop3_mask_or(w, 0x00F000F0u, 0x64006400u));
  x[2] = hsub2_1024(lop3_mask_or(w8, 0x000F000Fu, 0x64006400u));
  x[3] = hsub2_1024(lop3_mask_or(w8, 0x00F000F0u, 0x64006400u));
}
// The same four code pairs as fp16 SUBNORMALS: a nibble masked into the low mantissa bits
// (exponent field 0) is exactly c * 2^-24 (16c * 2^-24 for the odd nibbles), so one LOP3
// per two codes gives an exactly scaled A operand — no "- 1024".  The tensor core keeps
// fp16 subnormal inputs, and every product and fp32 partial sum of the contraction is the
// exact-unpack value times 2^-24, so the caller's 2^24 factor (folded into the k scale)
// restores bit-identical logits.
__device__ __forceinline__ void unpack8_sub(uint32_t w, uint32_t (&x)[4]) {
  const uint32_t w8 = w >> 8;
  x[0] = w & 0x000F000Fu;
  x[1] = w & 0x00F000F0u;
  x[2] = w8 & 0x000F000Fu;
  x[3] = w8 & 0x00F000F0u;
}
#ifndef ARKV_QK_SUB
#define ARKV_QK_SUB 1
#endif
constexpr bool kQkSub = ARKV_QK_SUB != 0;
constexpr float kSubScale = 16777216.0f;  // 2^24
// QK^T of a tile as two independent accumulator chains (halves the MMA dependency depth;
// the fp32 sum order of the logits changes by one final add)
#ifndef ARKV_QK_SPLIT
#define ARKV_QK_SPLIT 1
#endif
constexpr bool kQkSplit = ARKV_QK_SPLIT != 0;
// Two e4m3 codes (the low / high 16 bits of w) -> f16x2 (lower code -> lower half).
__device__ __forceinline__ uint32_t e4m3x2_to_f16x2(uint32_t v16) {
  const __half2_raw h = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(v16 & 0xFFFFu), __NV_E4M3);
  return (uint32_t)h.x | ((uint32_t)h.y << 16);
}
__device__ __forceinline__ uint32_t e4m3x2_lo(uint32_t w) { return e4m3x2_to_f16x2(w); }
__device__ __forceinline__ uint32_t e4m3x2_hi(uint32_t w) { return e4m3x2_to_f16x2(w >> 16); }
// The same without the exact "- 1024": codes stay as f16 (1024 + c) / (1024 + 16c), the
// offset removed later in the fp32 zero-point term.  OFF by default (ARKV_PV_RAW=0): the
// PV accumulator then carries ~1024x the output's magnitude, and the fp32 cancellation
// grew to 1.5e-3 absolute at 32K contexts with ~17K Quantized tokens (round 2, full-size
// parity: at the tolerance); the exact unpack costs +0.8 % decode-kernel time.
__device__ __forceinline__ void unpack8_raw(uint32_t w, uint32_t (&x)[4]) {
  const uint32_t w8 = w >> 8;
  x[0] = lop3_mask_or(w, 0x000F000Fu, 0x64006400u);
  x[1] = lop3_mask_or(w, 0x00F000F0u, 0x64006400u);
  x[2] = lop3_mask_or(w8, 0x000F000Fu, 0x64006400u);
  x[3] = lop3_mask_or(w8, 0x00F000F0u, 0x64006400u);
}
#ifndef ARKV_PV_RAW
#define ARKV_PV_RAW 0
#endif
constexpr bool kPvRaw = ARKV_PV_RAW != 0;
// PV on SUBNORMAL codes (round 2): the V codes enter the PV contraction as fp16 subnormals
// c * 2^-24 (one LOP3 per two codes, as the QK logits already do: no "- 1024", no offset to
// cancel), and the 2^-24 is absorbed by scaling EVERY probability of the fast kernels by
// 2^-24: p' = 2^(s - m - 24).  The scale is common to l, Σ p z_v and o of every partial, so
// it cancels in o / l; the Quantized tiles' P' = p' * (s_v 2^24) keep today's fp16 range, the
// Original tiles' bf16 P' is just 2^-24 smaller.  Consumers of the merged (M, L) outside the
// kernel subtract DecodeArgs::pscale (the HH samples, the new token's weight).
#ifndef ARKV_PV_SUB
#define ARKV_PV_SUB 1
#endif
constexpr bool kPvSub = ARKV_PV_SUB != 0;
// log2 of 1 / (the probability scale) of the int-code kernels; the fp8 kernels (e4m3 codes
// convert to NORMAL fp16) keep unscaled probabilities
template <bool F8>
constexpr float kPScale = (kPvSub && !F8) ? 24.f : 0.f;
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *(uint32_t*)&v;
}
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  __half2 v = __floats2half2_rn(lo, hi);
  return *(uint32_t*)&v;
}
// 2^x on the SFU without exp2f's denormal-range fix-up (results below 2^-126 flush to 0:
// such probabilities are negligible next to the running max's 1)
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float f16_round(float x) { return __half2float(__float2half_rn(x)); }
__device__ __forceinline__ uint32_t word(const uint4& q, int i) { return i == 0 ? q.x : i == 1 ? q.y : i == 2 ? q.z : q.w; }

template <int C, int SPW>
struct Smem {
  static constexpr int kStages = C * SPW;
  uint8_t ring[kStages][kStageBytes];
  uint64_t full[kStages];
  uint64_t empty[kStages];
  float wm[C][8];                     // per warp, per head: running max (log2 domain)
  float wl[C][8];                     // sum of p
  float wz[C][8][4];                  // Σ p·z_v per head, per group
  float newtok[3][8];                 // new token: logit per head (log2), valid flag
  float cM[8], cIL[8];                // fused combine: merged max and 1/sum per head
  int is_last;                        // this CTA is the last split of its unit to finish
};

// Converts the fp32 P' block (thread holds rows gq, gq+8 x cols 2t, 2t+1) into the PV
// B operand: columns [hi heads | lo heads] for 2G <= 8, transposed with movmatrix.
template <int G, bool BF16>
__device__ __forceinline__ void make_b(const float (&v)[4], int t, uint32_t& b01, uint32_t& b23, uint32_t& c01,
                                       uint32_t& c23) {
  // v: [0] (row g, col 2t) [1] (row g, col 2t+1) [2] (row g+8, col 2t) [3] (row g+8, col 2t+1)
  float hi[4], lo[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    hi[i] = BF16 ? bf16_round(v[i]) : f16_round(v[i]);
    lo[i] = v[i] - hi[i];
  }
  auto pk = [](float a, float b) { return BF16 ? pack_bf16(a, b) : pack_f16(a, b); };
  uint32_t h0 = pk(hi[0], hi[1]), h1 = pk(hi[2], hi[3]);
  uint32_t l0 = pk(lo[0], lo[1]), l1 = pk(lo[2], lo[3]);
  if (G == 8) {
    b01 = movtrans(h0);
    b23 = movtrans(h1);
    c01 = movtrans(l0);
    c23 = movtrans(l1);
    return;
  }
  uint32_t r0, r1;
  if (G == 4) {
    uint32_t s0 = __shfl_xor_sync(0xffffffffu, l0, 2), s1 = __shfl_xor_sync(0xffffffffu, l1, 2);
    r0 = t < 2 ? h0 : s0;
    r1 = t < 2 ? h1 : s1;
  } else if (G == 2) {
    uint32_t s0 = __shfl_sync(0xffffffffu, l0, (threadIdx.x & 28)), s1 = __shfl_sync(0xffffffffu, l1, (threadIdx.x & 28));
    r0 = t == 0 ? h0 : (t == 1 ? s0 : 0u);
    r1 = t == 0 ? h1 : (t == 1 ? s1 : 0u);
  } else {  // G == 1: columns (hi h0, lo h0)
    r0 = t == 0 ? pk(hi[0], lo[0]) : 0u;
    r1 = t == 0 ? pk(hi[2], lo[2]) : 0u;
  }
  b01 = movtrans(r0);
  b23 = movtrans(r1);
  c01 = c23 = 0u;
}

// ---- consumer building blocks (split kernel and persistent kernel) --------------------
// q fragments of one unit: bf16 for Original tiles; f16 (with the 1/16 odd-nibble factor)
// for Quantized tiles; Σq per group for the zero-point term (this thread's two heads
// 2t, 2t+1 — only lanes with tq < G/2 matter).
template <int NG>
struct QFrag {
  uint32_t qb[8][2], qh[8][2];
  float qsum[2][NG];
};
template <int G, int NG, bool F8>
__device__ __forceinline__ void load_qfrag(const uint16_t* qp, int lane, QFrag<NG>& f) {
  const int gq = lane >> 2, tq = lane & 3;
  const int hq = gq;  // B operand column n = head gq
  const bool hv = hq < G;
  if (F8) {
    // fp8 Quantized tiles (FRAG, 8-bit): the standard f16 B fragment — k-step ks holds
    // dims 16ks + 2t, +1 (b0) and 16ks + 2t + 8, +9 (b1); no zero point, no Σq
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int x0 = tq * 32 + 4 * c;
      f.qb[c][0] = hv ? *(const uint32_t*)(qp + hq * D + x0) : 0u;
      f.qb[c][1] = hv ? *(const uint32_t*)(qp + hq * D + x0 + 2) : 0u;
      const int xb = 16 * c + 2 * tq;
      f.qh[c][0] = hv ? pack_f16(bf16_to_f(qp[hq * D + xb]), bf16_to_f(qp[hq * D + xb + 1])) : 0u;
      f.qh[c][1] = hv ? pack_f16(bf16_to_f(qp[hq * D + xb + 8]), bf16_to_f(qp[hq * D + xb + 9])) : 0u;
    }
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int gr = 0; gr < NG; ++gr) f.qsum[e][gr] = 0.f;
    return;
  }
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int x0 = tq * 32 + 4 * c;  // Original tiles: dims t*(d/4)+4c+{0,1} / +{2,3}
    f.qb[c][0] = hv ? *(const uint32_t*)(qp + hq * D + x0) : 0u;
    f.qb[c][1] = hv ? *(const uint32_t*)(qp + hq * D + x0 + 2) : 0u;
    // Quantized tiles: chunk c = 2jp + cc; nibble pairs (e, e+4) with e = 2cc (+1 for b1)
    const int jp = c >> 1, cc = c & 1;
    const int xb = 32 * jp + 8 * tq + 2 * cc;
    float f0 = hv ? bf16_to_f(qp[hq * D + xb + 0]) : 0.f, f4 = hv ? bf16_to_f(qp[hq * D + xb + 4]) : 0.f;
    float f1 = hv ? bf16_to_f(qp[hq * D + xb + 1]) : 0.f, f5 = hv ? bf16_to_f(qp[hq * D + xb + 5]) : 0.f;
    f.qh[c][0] = pack_f16(f0, f4);
    f.qh[c][1] = pack_f16(f1 * 0.0625f, f5 * 0.0625f);
  }
  // Σ_x q[h][x] per group: lane sums its 4 dims, segmented butterfly over the 32/NG lanes
  // of each group, then the owner lanes pick their heads' sums
#pragma unroll
  for (int e = 0; e < 2; ++e)
#pragma unroll
    for (int gr = 0; gr < NG; ++gr) f.qsum[e][gr] = 0.f;
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float v = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) v += bf16_to_f(qp[h * D + lane * 4 + i]);
#pragma unroll
    for (int off = 1; off < 32 / NG; off <<= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
#pragma unroll
    for (int gr = 0; gr < NG; ++gr) {
      const float sgr = __shfl_sync(0xffffffffu, v, gr * (32 / NG));
      if (2 * tq == h) f.qsum[0][gr] = sgr;
      if (2 * tq + 1 == h) f.qsum[1][gr] = sgr;
    }
  }
}

// Running flash state of one consumer warp: O^T accumulators (m-tile over dims,
// (dim g|g+8) x (col 2t|2t+1)) and, per head 2t+e, the running max (log2 domain), Σp and
// Σ p·z_v per group.
template <int NG>
struct Acc {
  float o[8][4];
  float m_run[2], l_run[2];
  float z_run[2][NG];
};
template <int NG>
__device__ __forceinline__ void acc_reset(Acc<NG>& s) {
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) s.o[i][e] = 0.f;
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    s.m_run[e] = -INFINITY;
    s.l_run[e] = 0.f;
#pragma unroll
    for (int gr = 0; gr < NG; ++gr) s.z_run[e][gr] = 0.f;
  }
}

// Tile processing, in three parts so a pipeline may stage an Original tile's K block and
// V^T block separately: qk_softmax (S = K q^T, HH logits, online-softmax update -> p),
// then pv_orig (Original tiles: O^T += V^T P'^T on the V^T block) or pv_quant (Quantized
// tiles, same staged tile).  consume_tile = the three for a tile staged whole.
// tb: the tile (or its K block) in shared memory; n_valid: rows in use; lrow: HH logits of
// this tile's first row, [row][G] (a.logits + (u row_stride + (isq ? cap_o : 0) + 32 tile) G)
// or nullptr outside the HH window.
template <int G, int NG, bool F8>
__device__ __forceinline__ void qk_softmax(const uint8_t* tb, bool isq, int n_valid, float* lrow, uint64_t lpol,
                                           const QFrag<NG>& f, Acc<NG>& s, float c2, bool sym, int lane,
                                           int src_lane, float (&p)[2][4], float (&zv)[2][2][NG]) {
  const int gq = lane >> 2, tq = lane & 3;
  // ---- S = K q^T, logits in the log2 domain ----
  float lg[2][4];  // [m-tile][(row g|g+8) x (col 2t|2t+1)]; zv: Quantized z_v of rows (g, g+8)
  if (!isq) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      // two accumulators per m-tile (kQkSplit): the 8 MMAs form two dependent chains of 4
      float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int qd = 0; qd < 4; ++qd) {
        const uint4 r0 = lds128(tb + (((mt * 2 + 0) * 4 + qd) * 32 + lane) * 16);
        const uint4 r1 = lds128(tb + (((mt * 2 + 1) * 4 + qd) * 32 + lane) * 16);
        float(&ac)[4] = acc[kQkSplit ? (qd & 1) : 0];
        mma_bf16(ac, r0.x, r1.x, r0.y, r1.y, f.qb[2 * qd][0], f.qb[2 * qd][1]);
        mma_bf16(ac, r0.z, r1.z, r0.w, r1.w, f.qb[2 * qd + 1][0], f.qb[2 * qd + 1][1]);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) lg[mt][e] = (kQkSplit ? acc[0][e] + acc[1][e] : acc[0][e]) * c2;
    }
  } else if (F8) {
    // fp8 e4m3 codes: one cvt.rn.f16x2.e4m3x2 per byte pair gives the f16 A fragment;
    // logit = s_k · (q · e4m3(c)) (no zero point)
    const float* sc = (const float*)(tb + 64 * D);  // [row][grp][k_scale, 0, v_scale, 0]
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      float acc[NG][4];
#pragma unroll
      for (int gr = 0; gr < NG; ++gr)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[gr][e] = 0.f;
#pragma unroll
      for (int kp = 0; kp < 4; ++kp) {
        const uint4 r = lds128(tb + ((mt * 4 + kp) * 32 + lane) * 16);
        const int gr0 = (32 * kp) / (D / NG), gr1 = (32 * kp + 16) / (D / NG);
        mma_f16(acc[gr0], e4m3x2_lo(r.x), e4m3x2_hi(r.x), e4m3x2_lo(r.y), e4m3x2_hi(r.y), f.qh[2 * kp][0],
                f.qh[2 * kp][1]);
        mma_f16(acc[gr1], e4m3x2_lo(r.z), e4m3x2_hi(r.z), e4m3x2_lo(r.w), e4m3x2_hi(r.w), f.qh[2 * kp + 1][0],
                f.qh[2 * kp + 1][1]);
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int j = mt * 16 + gq + 8 * hh;
        float l0 = 0.f, l1 = 0.f;
#pragma unroll
        for (int gr = 0; gr < NG; ++gr) {
          const float ks = sc[(j * NG + gr) * 4];
          l0 += ks * acc[gr][hh * 2 + 0];
          l1 += ks * acc[gr][hh * 2 + 1];
          zv[mt][hh][gr] = 0.f;
        }
        lg[mt][hh * 2 + 0] = l0 * c2;
        lg[mt][hh * 2 + 1] = l1 * c2;
      }
    }
  } else {
    const float* sc = (const float*)(tb + 32 * D);  // [row][grp][k_scale, k_zero, v_scale, v_zero]
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      float acc[NG][4], acc2[NG][4];  // acc2: odd jp when two jp share a group (kQkSplit)
#pragma unroll
      for (int gr = 0; gr < NG; ++gr)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[gr][e] = acc2[gr][e] = 0.f;
      const uint4 r0 = lds128(tb + ((mt * 2 + 0) * 32 + lane) * 16);
      const uint4 r1 = lds128(tb + ((mt * 2 + 1) * 32 + lane) * 16);
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {
        uint32_t x[4], y[4];
        if (kQkSub) {
          unpack8_sub(word(r0, jp), x);
          unpack8_sub(word(r1, jp), y);
        } else {
          unpack8(word(r0, jp), x);
          unpack8(word(r1, jp), y);
        }
        const int gr = (jp * 32) / (D / NG);
        float(&ac)[4] = (kQkSplit && NG <= 2 && (jp & 1)) ? acc2[gr] : acc[gr];
        mma_f16(ac, x[0], y[0], x[1], y[1], f.qh[2 * jp][0], f.qh[2 * jp][1]);
        mma_f16(ac, x[2], y[2], x[3], y[3], f.qh[2 * jp + 1][0], f.qh[2 * jp + 1][1]);
      }
      if (kQkSplit && NG <= 2) {
#pragma unroll
        for (int gr = 0; gr < NG; ++gr)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[gr][e] += acc2[gr][e];
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int j = mt * 16 + gq + 8 * hh;
        float l0 = 0.f, l1 = 0.f;
#pragma unroll
        for (int gr = 0; gr < NG; ++gr) {
          const float4 s4 = *(const float4*)(sc + (j * NG + gr) * 4);  // one LDS.128 per row and group
          const float ks = s4.x, vs = s4.z;
          float kz = s4.y, vz = s4.w;
          if (sym) {
            kz = -8.f * ks;
            vz = -8.f * vs;
          }
          const float ksc = kQkSub ? ks * kSubScale : ks;  // exact: power-of-two factor
          l0 += ksc * acc[gr][hh * 2 + 0] + kz * f.qsum[0][gr];
          l1 += ksc * acc[gr][hh * 2 + 1] + kz * f.qsum[1][gr];
          // PV runs on the raw magic-number codes (1024 + c for rows g, 1024 + 16c for
          // rows g+8, whose P' carries 1/16): the offset is removed here, in the z term
          zv[mt][hh][gr] = (kPvRaw && !kPvSub) ? vz - (hh ? 64.f : 1024.f) * vs : vz;
        }
        lg[mt][hh * 2 + 0] = l0 * c2;
        lg[mt][hh * 2 + 1] = l1 * c2;
      }
    }
  }
  // mask rows beyond the segment (only the last tile of a segment is partial).  Padding
  // heads (h >= G, columns of lanes tq >= G/2) are not masked: their logits are 0 (zero q
  // fragments), and no padding column enters the PV operand (make_b), the HH logits or the
  // merged statistics.
  if (n_valid < kTile) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (mt * 16 + gq + 8 * (e >> 1) >= n_valid) lg[mt][e] = -INFINITY;
  }
  if (lrow) {
    // logits [row][G]: this lane's heads 2t, 2t+1 of a row are adjacent — one 8-byte store
    // per (m-tile, row half); the 8 rows x G heads of one store instruction are contiguous
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int j = mt * 16 + gq + 8 * hh;
        if (j < n_valid && 2 * tq < G) {
          float* p = lrow + j * G + 2 * tq;
          if (G >= 2)
            st_hint((float2*)p, make_float2(lg[mt][2 * hh], lg[mt][2 * hh + 1]), lpol);
          else
            st_hint(p, lg[mt][2 * hh], lpol);
        }
      }
  }
  // ---- online softmax (per head = per (tq, e)) ----
  float tmax[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    float mx = fmaxf(fmaxf(lg[0][e], lg[0][e + 2]), fmaxf(lg[1][e], lg[1][e + 2]));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
    tmax[e] = mx;
  }
  float corr[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const float mn = fmaxf(s.m_run[e], tmax[e]);
    corr[e] = (mn == -INFINITY) ? 1.f : ex2_ftz(s.m_run[e] - mn);
    s.m_run[e] = mn;
    s.l_run[e] *= corr[e];
#pragma unroll
    for (int gr = 0; gr < NG; ++gr) s.z_run[e][gr] *= corr[e];
  }
  // rescale O^T columns: col 2t+e belongs to head (2t+e) % G, whose max lives in lane src_lane
  // (skipped when no head's running max moved — most tiles once the max has settled)
  if (__any_sync(0xffffffffu, corr[0] != 1.f || corr[1] != 1.f)) {
    const float c0 = __shfl_sync(0xffffffffu, corr[0], src_lane);
    const float c1 = __shfl_sync(0xffffffffu, G >= 2 ? corr[1] : corr[0], src_lane);
#pragma unroll
    for (int mv = 0; mv < 8; ++mv) {
      s.o[mv][0] *= c0;
      s.o[mv][1] *= c1;
      s.o[mv][2] *= c0;
      s.o[mv][3] *= c1;
    }
  }
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float mm = s.m_run[e & 1];
      p[mt][e] = (mm == -INFINITY) ? 0.f : ex2_ftz(lg[mt][e] - (mm + kPScale<F8>));  // ex2(-inf) = 0 for masked rows
      s.l_run[e & 1] += p[mt][e];
    }
}

// PV of an Original tile; vb: its V^T block in shared memory
template <int G, int NG>
__device__ __forceinline__ void pv_orig(const uint8_t* vb, int n_valid, const float (&p)[2][4], Acc<NG>& s,
                                        int lane) {
  const int tq = lane & 3;
  {
    if (n_valid < kTile) {
      // rows past the segment may hold stale bytes (NaN patterns): P' = 0 there, but
      // 0 * NaN = NaN inside the MMA, so zero them in the staged copy
      uint8_t* tw = const_cast<uint8_t*>(vb);
      for (int idx = lane; idx < (kTile - n_valid) * D; idx += 32) {
        const int j = n_valid + idx / D, x = idx % D;
        // FRAG V offset (common.cuh o_v_off) for d = 128
        const int mtv = x >> 4, r = x & 15, gg = r & 7, sel = r >> 3;
        const int kc = j >> 4, jj = j & 15, hi = jj >> 3, tt = jj & 7, t = tt >> 1, uu = tt & 1;
        const int k = (mtv * 2 + kc) * 4 + sel + 2 * hi;
        *(uint16_t*)(tw + lane_word(k, 4 * gg + t) * 4 + uu * 2) = 0;
      }
      // order these generic-proxy writes before the stage's next TMA (async-proxy) fill
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
    }
    uint32_t b01[2], b23[2], c01[2], c23[2];
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) make_b<G, true>(p[kc], tq, b01[kc], b23[kc], c01[kc], c23[kc]);
#pragma unroll
    for (int mv = 0; mv < 8; ++mv) {
#pragma unroll
      for (int kc = 0; kc < 2; ++kc) {
        const uint4 r = lds128(vb + ((mv * 2 + kc) * 32 + lane) * 16);
        mma_bf16(s.o[mv], r.x, r.y, r.z, r.w, b01[kc], b23[kc]);
        if (G == 8) mma_bf16(s.o[mv], r.x, r.y, r.z, r.w, c01[kc], c23[kc]);
      }
    }
  }
}

// PV of a Quantized tile staged whole (tb)
template <int G, int NG, bool F8>
__device__ __forceinline__ void pv_quant(const uint8_t* tb, const float (&p)[2][4], const float (&zv)[2][2][NG],
                                         Acc<NG>& s, int lane) {
  const int gq = lane >> 2, tq = lane & 3;
  if (F8) {
    // ---- PV on fp8 Quantized tiles: A = e4m3 V^T (converted), B = P' = p·s_v ----
    const float* sc = (const float*)(tb + 64 * D);
    uint32_t b01[NG][2], b23[NG][2], c01[NG][2], c23[NG][2];
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) {
#pragma unroll
      for (int gr = 0; gr < NG; ++gr) {
        float pv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e)
          pv[e] = p[kc][e] * sc[((kc * 16 + gq + 8 * (e >> 1)) * NG + gr) * 4 + 2];
        make_b<G, false>(pv, tq, b01[gr][kc], b23[gr][kc], c01[gr][kc], c23[gr][kc]);
      }
    }
    const uint8_t* vb = tb + 32 * D;
#pragma unroll
    for (int mv = 0; mv < 8; ++mv) {
      const uint4 r = lds128(vb + (mv * 32 + lane) * 16);
      const int gr = (mv * 16) / (D / NG);
      mma_f16(s.o[mv], e4m3x2_lo(r.x), e4m3x2_hi(r.x), e4m3x2_lo(r.y), e4m3x2_hi(r.y), b01[gr][0], b23[gr][0]);
      if (G == 8)
        mma_f16(s.o[mv], e4m3x2_lo(r.x), e4m3x2_hi(r.x), e4m3x2_lo(r.y), e4m3x2_hi(r.y), c01[gr][0], c23[gr][0]);
      mma_f16(s.o[mv], e4m3x2_lo(r.z), e4m3x2_hi(r.z), e4m3x2_lo(r.w), e4m3x2_hi(r.w), b01[gr][1], b23[gr][1]);
      if (G == 8)
        mma_f16(s.o[mv], e4m3x2_lo(r.z), e4m3x2_hi(r.z), e4m3x2_lo(r.w), e4m3x2_hi(r.w), c01[gr][1], c23[gr][1]);
    }
  } else {
    // ---- PV on Quantized tiles (f16 codes, P' = p·s_v / f) ----
    const float* sc = (const float*)(tb + 32 * D);
    uint32_t b01[NG][2], b23[NG][2], c01[NG][2], c23[NG][2];
#pragma unroll
    for (int kc = 0; kc < 2; ++kc) {
#pragma unroll
      for (int gr = 0; gr < NG; ++gr) {
        float vsc[2];  // v_scale (x 2^24: subnormal codes) x 1/16 for the odd-nibble rows g+8
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
          vsc[hh] = sc[((kc * 16 + gq + 8 * hh) * NG + gr) * 4 + 2] *
                    ((kPvSub ? kSubScale : 1.f) * (hh ? 0.0625f : 1.f));
        float pv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) pv[e] = p[kc][e] * vsc[e >> 1];
        make_b<G, false>(pv, tq, b01[gr][kc], b23[gr][kc], c01[gr][kc], c23[gr][kc]);
        // zero-point term Σ p·z_v
#pragma unroll
        for (int e = 0; e < 4; ++e) s.z_run[e & 1][gr] += p[kc][e] * zv[kc][e >> 1][gr];
      }
    }
    const uint8_t* vb = tb + 16 * D;
#pragma unroll
    for (int qd = 0; qd < 4; ++qd) {
      const uint4 r = lds128(vb + (qd * 32 + lane) * 16);
#pragma unroll
      for (int hm = 0; hm < 2; ++hm) {
        const int mv = 2 * qd + hm;
        const int gr = (mv * 16) / (D / NG);
        uint32_t x[4], y[4];
        if (kPvSub) {
          unpack8_sub(word(r, 2 * hm + 0), x);  // dim row g: c * 2^-24 (odd tokens 16c * 2^-24)
          unpack8_sub(word(r, 2 * hm + 1), y);  // dim row g+8
        } else if (kPvRaw) {
          unpack8_raw(word(r, 2 * hm + 0), x);  // dim row g
          unpack8_raw(word(r, 2 * hm + 1), y);  // dim row g+8
        } else {
          unpack8(word(r, 2 * hm + 0), x);
          unpack8(word(r, 2 * hm + 1), y);
        }
#pragma unroll
        for (int kc = 0; kc < 2; ++kc) {
          mma_f16(s.o[mv], x[2 * kc], y[2 * kc], x[2 * kc + 1], y[2 * kc + 1], b01[gr][kc], b23[gr][kc]);
          if (G == 8)
            mma_f16(s.o[mv], x[2 * kc], y[2 * kc], x[2 * kc + 1], y[2 * kc + 1], c01[gr][kc], c23[gr][kc]);
        }
      }
    }
  }
}

template <int G, int NG, bool F8>
__device__ __forceinline__ void consume_tile(const uint8_t* tb, bool isq, int n_valid, float* lrow, int /*row_stride*/,
                                             uint64_t lpol, const QFrag<NG>& f, Acc<NG>& s, float c2, bool sym,
                                             int lane, int src_lane) {
  float p[2][4];
  float zv[2][2][NG];
  qk_softmax<G, NG, F8>(tb, isq, n_valid, lrow, lpol, f, s, c2, sym, lane, src_lane, p, zv);
  if (!isq)
    pv_orig<G, NG>(tb + 64 * D, n_valid, p, s, lane);
  else
    pv_quant<G, NG, F8>(tb, p, zv, s, lane);
}

// Reduces l and z over the 8 row lanes (every lane ends with its heads' sums).
template <int NG>
__device__ __forceinline__ void acc_reduce_rows(Acc<NG>& s) {
#pragma unroll
  for (int e = 0; e < 2; ++e) {
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      s.l_run[e] += __shfl_xor_sync(0xffffffffu, s.l_run[e], off);
#pragma unroll
      for (int gr = 0; gr < NG; ++gr) s.z_run[e][gr] += __shfl_xor_sync(0xffffffffu, s.z_run[e][gr], off);
    }
  }
}

#ifdef ARKV_TUNING_KNOBS
// Tuning builds only: per-CTA start/end (globaltimer), SM id and unit/split of the split-K
// decode kernel, read back by arkv_debug_cta_times (scripts/cta_timeline.py).
constexpr int kCtaTimesMax = 16384;
__device__ unsigned long long g_cta_t[kCtaTimesMax][8];
__device__ int g_cta_on;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;\n" : "=l"(t));
  return t;
}
#endif

template <int G, int NG, int C, int SPW, bool F8>
__global__ void __launch_bounds__((C + 1) * 32, (C * SPW * kStageBytes <= 6 * kStageBytes) ? 2 : 1)
    decode_fast_kernel(DecodeArgs a, const __grid_constant__ UnitOrder cl) {
#ifdef ARKV_TUNING_KNOBS
  const unsigned long long t_start = gtimer();
#endif
  constexpr int kConsumers = C;
  constexpr int kStages = C * SPW;
  auto stage_of = [](int i) { return (i % C) + C * ((i / C) % SPW); };
  auto phase_of = [](int i) { return (i / C) / SPW; };
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem<C, SPW>& sm = *reinterpret_cast<Smem<C, SPW>*>(smem_raw);
  const Geom& g = a.g;
  griddep_wait();  // PDL: the previous kernel (tailor / combine) has completed
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;

  // unit and split of this CTA: from the cost-balanced launch list, or the uniform grid
  int ul, s, S;
  if (cl.n_units > 0) {
    const int c = blockIdx.x;
    int lo = 0, hi = cl.n_units - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((int)cl.pfx[mid] <= c) lo = mid; else hi = mid - 1;
    }
    ul = cl.perm[lo];
    s = c - cl.pfx[lo];
    S = cl.pfx[lo + 1] - cl.pfx[lo];
  } else {
    ul = blockIdx.y;
    s = blockIdx.x;
    S = a.n_splits;
  }
  const int b = ul / (a.n_layers * g.Hkv);
  const int rem = ul % (a.n_layers * g.Hkv);
  const int li = rem / g.Hkv, kvh = rem % g.Hkv;
  const int u = (b * g.L + a.layer0 + li) * g.Hkv + kvh;
  const UnitDesc dsc = a.desc[u];
  uint8_t* slot = a.slots + (int64_t)dsc.slot * g.slot_bytes;
  const int n_o = dsc.n_o, n_q = dsc.n_q, t_pos = dsc.t_next;
  const bool accm = (t_pos >= dsc.acc0) && (t_pos < dsc.trig);
  const int tiles_o = (n_o + 1 + kTile - 1) / kTile;
  const int tiles_q = (n_q + kTile - 1) / kTile;
  if (a.nsplit && s == 0 && threadIdx.x == 0) a.nsplit[u] = S;  // for the combine
  const int o0 = (int)((int64_t)s * tiles_o / S), o1 = (int)((int64_t)(s + 1) * tiles_o / S);
  const int q0 = (int)((int64_t)s * tiles_q / S), q1 = (int)((int64_t)(s + 1) * tiles_q / S);
  // work items: single Original tiles and groups of up to q_per Quantized tiles (the
  // Q stack grows down, so a group is one contiguous bulk copy), interleaved evenly so
  // byte-heavy (O) and ALU-heavy (Q) items alternate across the consumer warps
  const int q_per = a.q_group > 0 ? min(a.q_group, kStageBytes / g.tile_q) : kStageBytes / g.tile_q;
  const int n_oi = o1 - o0, n_qi = (q1 - q0 + q_per - 1) / q_per;
  const int n_work = n_oi + n_qi;
  const bool rev = a.item_order == 2 || (a.item_order == 1 && ((s + ul) & 1));
  auto item_of = [&](int i, bool& isq, int& first, int& ntiles) {
    int qb;
    if (rev) i = i < n_qi ? n_oi + i : i - n_qi;  // Quantized groups first
    if (a.interleave) {
      qb = (int)(((int64_t)i * n_qi) / max(n_work, 1));
      isq = (int)(((int64_t)(i + 1) * n_qi) / max(n_work, 1)) > qb;
    } else {  // all Original tiles first, then the Quantized groups
      isq = i >= n_oi;
      qb = isq ? i - n_oi : 0;
      if (!isq) qb = 0;
    }
    if (!a.interleave && !isq) {
      first = o0 + i;
      ntiles = 1;
      return;
    }
    if (isq) {
      first = q0 + qb * q_per;
      ntiles = min(q_per, q1 - first);
    } else {
      first = o0 + (i - qb);
      ntiles = 1;
    }
  };
  const bool owns_new = (o0 <= n_o / kTile) && (n_o / kTile < o1);
  const int row_stride = g.cap_o + g.cap_q;
  const int64_t qkv = (int64_t)(b * a.n_layers + li);
  const uint16_t* qp = a.q + (qkv * g.Hq + kvh * G) * D;
  const uint16_t* kn = a.k + (qkv * g.Hkv + kvh) * D;
  const uint16_t* vn = a.v + (qkv * g.Hkv + kvh) * D;
  const float c2 = g.sm_scale * kLog2e;
  const bool sym = g.mode == ARKV_QUANT_SYM;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  auto item_src = [&](int i, const uint8_t*& src, uint32_t& bytes) {
    bool isq;
    int first, ntiles;
    item_of(i, isq, first, ntiles);
    src = isq ? q_tile_ptr(slot, g, first + ntiles - 1) : o_tile_ptr(slot, g, first);
    bytes = isq ? (uint32_t)(ntiles * g.tile_q) : (uint32_t)g.tile_o;
  };
  // Self-refill (default): each consumer warp's lane 0 loads its own items — the first SPW
  // at the start, then item i + kStages into the stage it has just consumed.  A slow
  // (Quantized) item then delays only its own warp's next load; with one in-order producer
  // every other warp's refill waited behind it (head-of-line blocking), which dominated
  // calls with few items per CTA (per-layer calls, 8-GPU shards).
  const bool self_refill = a.self_refill != 0;
  if (warp == kConsumers) {
    // ===================== producer =====================
    if (lane == 0 && !self_refill) {
      const uint64_t pol_stream = l2_evict_first();
      // items in order (measured: polling stages out of order and busy-waiting costs the
      // co-scheduled consumer warp issue slots; try_wait suspends in hardware)
      const int ahead = a.prefetch;  // items requested into L2 ahead of the ring (0: off)
      for (int i = 0; i < min(ahead, n_work); ++i) {
        const uint8_t* src;
        uint32_t bytes;
        item_src(kStages + i, src, bytes);
        if (kStages + i < n_work) bulk_prefetch_l2(src, bytes);
      }
      for (int i = 0; i < n_work; ++i) {
        const int st = stage_of(i);
        if (ahead > 0 && i + kStages + ahead < n_work) {
          const uint8_t* psrc;
          uint32_t pbytes;
          item_src(i + kStages + ahead, psrc, pbytes);
          bulk_prefetch_l2(psrc, pbytes);
        }
        if (i >= kStages) mbar_wait(&sm.empty[st], (phase_of(i) - 1) & 1);
        const uint8_t* src;
        uint32_t bytes;
        item_src(i, src, bytes);
        mbar_expect_tx(&sm.full[st], bytes);
        if (a.l2_hints)
          bulk_g2s_hint(sm.ring[st], src, bytes, &sm.full[st], pol_stream);
        else
          bulk_g2s(sm.ring[st], src, bytes, &sm.full[st]);
      }
      griddep_launch_dependents();  // PDL: the combine may start launching (it waits for us)
    }
    __syncwarp();  // reconverge before warp-collective code and the aligned CTA barrier
    // the producer warp also appends the step's token (D1) when this CTA owns its tile
    if (owns_new) {
      // non-finite q / k / v of the step
      if (warp_step_nonfinite(qp, G * D, kn, vn, D, lane) && lane == 0) atomicOr(a.err, kErrNonFinite);
      const int tt = n_o / kTile, j = n_o % kTile;
      const SlotMeta meta = slot_meta(a.meta, g, dsc.slot);
      const bool fits = (n_o + 1 <= g.cap_o) &&
                        ((int64_t)tiles_o * g.tile_o + (int64_t)tiles_q * g.tile_q <= g.slot_bytes);
      if (!fits) {
        if (lane == 0) atomicOr(a.err, kErrCapacity);
      } else {
        uint8_t* tb = o_tile_ptr(slot, g, tt);
        for (int x = lane; x < D; x += 32) {
          *(uint16_t*)(tb + o_k_off(g, j, x)) = kn[x];
          *(uint16_t*)(tb + o_v_off(g, j, x)) = vn[x];
        }
        if (lane == 0) {
          meta.pos_o[n_o] = t_pos;
          meta.acc_o[n_o] = make_float2(0.f, 0.f);
        }
      }
      // its logits (log2 domain) for the G heads
      float kx[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) kx[i] = bf16_to_f(kn[lane * 4 + i]);
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) acc = fmaf(bf16_to_f(qp[h * D + lane * 4 + i]), kx[i], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) sm.newtok[0][h] = acc * c2;
      }
      __syncwarp();
      if (accm && lane < G)
        st_hint(a.logits + ((int64_t)u * row_stride + n_o) * G + lane, sm.newtok[0][lane], l2_evict_last());
    }
  } else {
    // ===================== consumers =====================
    const uint64_t lpol = l2_evict_last();  // HH logits stay in L2 for the combine
    const uint64_t pol_stream = l2_evict_first();
    auto issue = [&](int i) {  // lane 0: item i into its stage (the stage is free)
      const int st = stage_of(i);
      const uint8_t* src;
      uint32_t bytes;
      item_src(i, src, bytes);
      mbar_expect_tx(&sm.full[st], bytes);
      if (a.l2_hints)
        bulk_g2s_hint(sm.ring[st], src, bytes, &sm.full[st], pol_stream);
      else
        bulk_g2s(sm.ring[st], src, bytes, &sm.full[st]);
    };
    if (self_refill && lane == 0)
      for (int k = 0; k < SPW; ++k)
        if (warp + k * kConsumers < n_work) issue(warp + k * kConsumers);
    QFrag<NG> qf;
    load_qfrag<G, NG, F8>(qp, lane, qf);
    Acc<NG> acc;
    acc_reset(acc);
    // lane holding the running max of the heads of this thread's O^T columns
    const int src_t = G >= 2 ? ((2 * tq) % G) / 2 : 0;
    const int src_lane = (lane & ~3) | src_t;

    // one work item (staged in stage st) folded into the warp's flash state
    auto consume_item = [&](int i, int st) {
      bool isq;
      int first, ntiles;
      item_of(i, isq, first, ntiles);
      for (int jt = 0; jt < ntiles; ++jt) {
        const uint8_t* tb = sm.ring[st] + (isq ? (ntiles - 1 - jt) * g.tile_q : 0);
        const int tile = first + jt;
        const int n_valid = isq ? min(kTile, n_q - tile * kTile) : min(kTile, n_o - tile * kTile);
        float* lrow = (accm && !a.hh_nostore)
                          ? a.logits + ((int64_t)u * row_stride + (isq ? g.cap_o : 0) + tile * kTile) * G
                          : nullptr;
        consume_tile<G, NG, F8>(tb, isq, n_valid, lrow, row_stride, lpol, qf, acc, c2, sym, lane, src_lane);
      }
      __syncwarp();
    };
#ifdef ARKV_TUNING_KNOBS
    auto stamp_first = [&](int i) {
      if (i == 0 && lane == 0 && g_cta_on) {
        const int ci = cl.n_units > 0 ? (int)blockIdx.x : (int)(blockIdx.y * gridDim.x + blockIdx.x);
        if (ci < kCtaTimesMax) g_cta_t[ci][4] = gtimer();
      }
    };
#else
    auto stamp_first = [](int) {};
#endif
    for (int i = warp; i < n_work; i += kConsumers) {
      const int st = stage_of(i);
      mbar_wait(&sm.full[st], phase_of(i) & 1);
      __syncwarp();  // lanes may leave the spin-wait in different iterations; mma/movmatrix are .aligned
      stamp_first(i);
      consume_item(i, st);
      if (self_refill) {
        if (lane == 0 && i + kStages < n_work) {
          // this warp's reads of the stage (generic proxy) before the refill (async proxy)
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          issue(i + kStages);
        }
      } else if (lane == 0) {
        mbar_arrive(&sm.empty[st]);
      }
    }
    if (self_refill && warp == 0 && lane == 0) griddep_launch_dependents();  // PDL (the combine waits for us)
#ifdef ARKV_TUNING_KNOBS
    if (lane == 0 && g_cta_on && warp < 3) {
      const int ci = cl.n_units > 0 ? (int)blockIdx.x : (int)(blockIdx.y * gridDim.x + blockIdx.x);
      if (ci < kCtaTimesMax) g_cta_t[ci][5 + warp] = gtimer();
    }
#endif
    // ---- per-warp finalisation: reduce l and z over the 8 row lanes ----
    acc_reduce_rows(acc);
    if (gq == 0) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int h = 2 * tq + e;
        if (h < G) {
          sm.wm[warp][h] = acc.m_run[e];
          sm.wl[warp][h] = acc.l_run[e];
#pragma unroll
          for (int gr = 0; gr < NG; ++gr) sm.wz[warp][h][gr] = acc.z_run[e][gr];
        }
      }
    }
    // every consumer is done with the ring: reuse it for the O^T accumulators
    asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumers * 32) : "memory");
    float* ob = (float*)sm.ring[0] + warp * 8 * D;  // [col][dim]
#pragma unroll
    for (int mv = 0; mv < 8; ++mv) {
      const int x0 = mv * 16 + gq;
      ob[(2 * tq + 0) * D + x0] = acc.o[mv][0];
      ob[(2 * tq + 1) * D + x0] = acc.o[mv][1];
      ob[(2 * tq + 0) * D + x0 + 8] = acc.o[mv][2];
      ob[(2 * tq + 1) * D + x0 + 8] = acc.o[mv][3];
    }
  }
  __syncthreads();
  // ---- CTA merge of the consumer warps (+ the appended token) -> split partial ----
  const float* ob = (const float*)sm.ring[0];
  float* part = a.partials + ((int64_t)u * a.max_splits + s) * G * (D + 2);
  for (int idx = threadIdx.x; idx < G * D; idx += blockDim.x) {
    const int h = idx / D, x = idx % D;
    const int gr = x / (D / NG);
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kConsumers; ++w) M = fmaxf(M, sm.wm[w][h]);
    float snew = -INFINITY;
    if (owns_new) {
      snew = sm.newtok[0][h];
      M = fmaxf(M, snew);
    }
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < kConsumers; ++w) {
      const float mw = sm.wm[w][h];
      if (mw == -INFINITY) continue;
      const float cw = exp2f(mw - M);
      float ow = ob[(w * 8 + h) * D + x];
      if (G < 8) ow += ob[(w * 8 + h + G) * D + x];
      ow += sm.wz[w][h][gr];
      L += sm.wl[w][h] * cw;
      O += ow * cw;
    }
    if (owns_new) {
      const float cn = exp2f(snew - M - kPScale<F8>);  // the partials' probability scale (kPvSub)
      L += cn;
      O += cn * bf16_to_f(vn[x]);
    }
    part[h * (D + 2) + 2 + x] = O;
    if (x == 0) {
      part[h * (D + 2) + 0] = M;
      part[h * (D + 2) + 1] = L;
    }
  }
#ifdef ARKV_TUNING_KNOBS
  if (threadIdx.x == 0 && g_cta_on) {
    const int ci = cl.n_units > 0 ? (int)blockIdx.x : (int)(blockIdx.y * gridDim.x + blockIdx.x);
    if (ci < kCtaTimesMax) {
      unsigned smid;
      asm volatile("mov.u32 %0, %smid;\n" : "=r"(smid));
      g_cta_t[ci][0] = t_start;
      g_cta_t[ci][1] = gtimer();
      g_cta_t[ci][2] = ((unsigned long long)smid << 32) | (unsigned)(u * 64 + s);
      g_cta_t[ci][3] = ((unsigned long long)(o1 - o0) << 32) | (unsigned)(q1 - q0);
    }
  }
#endif
  // ---- fused combine: the last split CTA of the unit to finish merges all partials ----
  if (!a.fuse_combine) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = atomicAdd(&a.counters[u], 1);
    sm.is_last = prev == S - 1;
  }
  __syncthreads();
  if (sm.is_last) {
    __threadfence();
    combine_unit<G>(a, u, b, li, kvh, dsc, sm.cM, sm.cIL);
    if (threadIdx.x == 0) a.counters[u] = 0;
  }
}

// ---------------------------------------------------------------------------------------
// "Chunked" split-K pipeline (default): 3 CTAs per SM of 3 consumer warps each
// and no producer warp — every warp streams its own chunks through 2 private 12 KB stages
// (self-refill).  An Original tile is two chunks (its 8 KB K block, then its 8 KB V^T block);
// Quantized tiles go two per chunk (9 KB).  9 consumer warps per SM instead of 6: the
// Quantized path is issue-bound (fixed-latency dependency stalls with 1.5 warps per
// scheduler), the Original path HBM-bound either way.  The step's token (D1) is appended
// by warp 0 before it waits for its first chunk.
// ---------------------------------------------------------------------------------------
// chunk (stage) bytes: an 8 KB half Original tile or two 4.5 KB Quantized tiles.  (Measured:
// 9 KB chunks, an idle 5th warp or no minimum-blocks bound leave the kernel time unchanged;
// with any of them ~10 % of the first wave's CTAs start only when a CTA of the first wave
// finishes — a dispatch effect we could not remove.)
template <int C>
constexpr int chunk_bytes() { return 12288; }
template <int C>
struct Smem3 {
  static constexpr int kStages = 2 * C;
  static constexpr int kChunkBytes = chunk_bytes<C>();
  uint8_t ring[kStages][kChunkBytes];
  uint64_t full[kStages];
  float wm[C][8];
  float wl[C][8];
  float wz[C][8][4];
  float newtok[8];
  int is_last;  // fused combine: this CTA is the last split of its unit to finish
};

template <int G, int NG, bool F8, int C>
__global__ void __launch_bounds__(C * 32, 2) decode_chunk_kernel(DecodeArgs a, const __grid_constant__ UnitOrder cl) {
#ifdef ARKV_TUNING_KNOBS
  const unsigned long long t_start = gtimer();
#endif
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem3<C>& sm = *reinterpret_cast<Smem3<C>*>(smem_raw);
  const Geom& g = a.g;
  griddep_wait();  // PDL: the previous kernel (tailor / combine) has completed
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  int ul, s, S;
  if (cl.n_units > 0) {
    const int c = blockIdx.x;
    int lo = 0, hi = cl.n_units - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((int)cl.pfx[mid] <= c) lo = mid; else hi = mid - 1;
    }
    ul = cl.perm[lo];
    s = c - cl.pfx[lo];
    S = cl.pfx[lo + 1] - cl.pfx[lo];
  } else {
    ul = blockIdx.y;
    s = blockIdx.x;
    S = a.n_splits;
  }
  const int b = ul / (a.n_layers * g.Hkv);
  const int rem = ul % (a.n_layers * g.Hkv);
  const int li = rem / g.Hkv, kvh = rem % g.Hkv;
  const int u = (b * g.L + a.layer0 + li) * g.Hkv + kvh;
  const UnitDesc dsc = a.desc[u];
  uint8_t* slot = a.slots + (int64_t)dsc.slot * g.slot_bytes;
  const int n_o = dsc.n_o, n_q = dsc.n_q, t_pos = dsc.t_next;
  const bool accm = (t_pos >= dsc.acc0) && (t_pos < dsc.trig);
  const int tiles_o = (n_o + 1 + kTile - 1) / kTile;
  const int tiles_q = (n_q + kTile - 1) / kTile;
  if (a.nsplit && s == 0 && threadIdx.x == 0) a.nsplit[u] = S;  // for the combine
  const int o0 = (int)((int64_t)s * tiles_o / S), o1 = (int)((int64_t)(s + 1) * tiles_o / S);
  const int q0 = (int)((int64_t)s * tiles_q / S), q1 = (int)((int64_t)(s + 1) * tiles_q / S);
  const int q_per = max(1, chunk_bytes<C>() / g.tile_q);  // Quantized tiles per chunk (int4: 2 x 4.5 KB; fp8: 1)
  const int n_oi = o1 - o0, n_qi = (q1 - q0 + q_per - 1) / q_per;
  const int n_work = n_oi + n_qi;
  const bool rev = a.item_order == 2 || (a.item_order == 1 && ((s + ul) & 1));
  // item i -> Original tile (1 item = 2 chunks) or a group of <= 2 Quantized tiles (1 chunk)
  auto item_of = [&](int i, bool& isq, int& first, int& ntiles) {
    if (rev) i = i < n_qi ? n_oi + i : i - n_qi;  // Quantized groups first
    isq = i >= n_oi;
    if (!isq) {
      first = o0 + i;
      ntiles = 1;
    } else {
      first = q0 + (i - n_oi) * q_per;
      ntiles = min(q_per, q1 - first);
    }
  };
  const bool owns_new = (o0 <= n_o / kTile) && (n_o / kTile < o1);
  const int row_stride = g.cap_o + g.cap_q;
  const int64_t qkv = (int64_t)(b * a.n_layers + li);
  const uint16_t* qp = a.q + (qkv * g.Hq + kvh * G) * D;
  const uint16_t* kn = a.k + (qkv * g.Hkv + kvh) * D;
  const uint16_t* vn = a.v + (qkv * g.Hkv + kvh) * D;
  const float c2 = g.sm_scale * kLog2e;
  const bool sym = g.mode == ARKV_QUANT_SYM;
  // stage barriers: each warp initialises its own two (nobody else touches them)
  if (lane == 0) {
    mbar_init(&sm.full[2 * warp], 1);
    mbar_init(&sm.full[2 * warp + 1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  const uint64_t lpol = l2_evict_last();  // HH logits stay in L2 for the combine
  const uint64_t pol_stream = l2_evict_first();
  // the warp's chunk cursor: (item, part; the item's kind and tiles); part 1 = the V^T block
  // of an Original tile.  The item is decoded once, when the cursor reaches it.
  struct Cur {
    int i, part;
    bool isq;
    int first, ntiles;
  };
  auto make_cur = [&](int i) {
    Cur c{i, 0, false, 0, 0};
    if (i < n_work) item_of(i, c.isq, c.first, c.ntiles);
    return c;
  };
  auto next = [&](const Cur& c) {
    if (!c.isq && c.part == 0) {
      Cur d = c;
      d.part = 1;
      return d;
    }
    return make_cur(c.i + C);
  };
  auto issue = [&](const Cur& c, int st) {  // lane 0
    const uint8_t* src = c.isq ? q_tile_ptr(slot, g, c.first + c.ntiles - 1)
                               : o_tile_ptr(slot, g, c.first) + (c.part ? 64 * D : 0);
    const uint32_t bytes = c.isq ? (uint32_t)(c.ntiles * g.tile_q) : (uint32_t)(32 * D * 2);
    mbar_expect_tx(&sm.full[st], bytes);
    if (a.l2_hints)
      bulk_g2s_hint(sm.ring[st], src, bytes, &sm.full[st], pol_stream);
    else
      bulk_g2s(sm.ring[st], src, bytes, &sm.full[st]);
  };
  Cur fetch = make_cur(warp);
  if (lane == 0) {
    for (int k = 0; k < 2 && fetch.i < n_work; ++k) {
      issue(fetch, 2 * warp + k);
      fetch = next(fetch);
    }
  }
  fetch = next(next(make_cur(warp)));  // every lane tracks the cursor (lane 0 issued the first two)
  if (warp == 0 && owns_new) {
    // the step's token (D1): appended while the first chunks are in flight
    if (warp_step_nonfinite(qp, G * D, kn, vn, D, lane) && lane == 0) atomicOr(a.err, kErrNonFinite);
    const int tt = n_o / kTile, j = n_o % kTile;
    const SlotMeta meta = slot_meta(a.meta, g, dsc.slot);
    const bool fits = (n_o + 1 <= g.cap_o) &&
                      ((int64_t)tiles_o * g.tile_o + (int64_t)tiles_q * g.tile_q <= g.slot_bytes);
    if (!fits) {
      if (lane == 0) atomicOr(a.err, kErrCapacity);
    } else {
      uint8_t* tb = o_tile_ptr(slot, g, tt);
      for (int x = lane; x < D; x += 32) {
        *(uint16_t*)(tb + o_k_off(g, j, x)) = kn[x];
        *(uint16_t*)(tb + o_v_off(g, j, x)) = vn[x];
      }
      if (lane == 0) {
        meta.pos_o[n_o] = t_pos;
        meta.acc_o[n_o] = make_float2(0.f, 0.f);
      }
    }
    float kx[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) kx[i] = bf16_to_f(kn[lane * 4 + i]);
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float acc = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) acc = fmaf(bf16_to_f(qp[h * D + lane * 4 + i]), kx[i], acc);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) sm.newtok[h] = acc * c2;
    }
    __syncwarp();
    if (accm && lane < G)
      st_hint(a.logits + ((int64_t)u * row_stride + n_o) * G + lane, sm.newtok[lane], l2_evict_last());
  }
  QFrag<NG> qf;
  load_qfrag<G, NG, F8>(qp, lane, qf);
  Acc<NG> acc;
  acc_reset(acc);
  const int src_t = G >= 2 ? ((2 * tq) % G) / 2 : 0;
  const int src_lane = (lane & ~3) | src_t;
  float p[2][4];        // an Original tile's probabilities, from its K chunk to its V chunk
  int o_valid = kTile;  // ... and its rows in use
  Cur cur = make_cur(warp);
  uint32_t ph = 0;
  int k = 0;
#ifdef ARKV_TUNING_KNOBS
  bool first_chunk = true;
#endif
  while (cur.i < n_work) {
    const int st = 2 * warp + k;
    mbar_wait(&sm.full[st], (ph >> k) & 1u);
    __syncwarp();
#ifdef ARKV_TUNING_KNOBS
    if (first_chunk && warp == 0 && lane == 0 && g_cta_on) {
      const int ci = cl.n_units > 0 ? (int)blockIdx.x : (int)(blockIdx.y * gridDim.x + blockIdx.x);
      if (ci < kCtaTimesMax) g_cta_t[ci][4] = gtimer();
    }
    first_chunk = false;
#endif
    const bool isq = cur.isq;
    const int first = cur.first, ntiles = cur.ntiles;
    const uint8_t* tb = sm.ring[st];
    if (isq) {
      for (int jt = 0; jt < ntiles; ++jt) {
        const int tile = first + jt;
        const int n_valid = min(kTile, n_q - tile * kTile);
        float* lrow = accm ? a.logits + ((int64_t)u * row_stride + g.cap_o + tile * kTile) * G : nullptr;
        float pq[2][4];
        float zv[2][2][NG];
        const uint8_t* tq_ = tb + (ntiles - 1 - jt) * g.tile_q;
        qk_softmax<G, NG, F8>(tq_, true, n_valid, lrow, lpol, qf, acc, c2, sym, lane, src_lane, pq, zv);
        pv_quant<G, NG, F8>(tq_, pq, zv, acc, lane);
      }
    } else if (cur.part == 0) {
      o_valid = min(kTile, n_o - first * kTile);
      float* lrow = accm ? a.logits + ((int64_t)u * row_stride + first * kTile) * G : nullptr;
      float zv[2][2][NG];
      qk_softmax<G, NG, F8>(tb, false, o_valid, lrow, lpol, qf, acc, c2, sym, lane, src_lane, p, zv);
    } else {
      pv_orig<G, NG>(tb, o_valid, p, acc, lane);
    }
    __syncwarp();
    if (lane == 0 && fetch.i < n_work) {
      // this warp's reads of the stage (generic proxy) before the refill (async proxy)
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(fetch, st);
    }
    if (fetch.i < n_work) fetch = next(fetch);
    cur = next(cur);
    ph ^= 1u << k;
    k ^= 1;
  }
  if (warp == 0 && lane == 0) griddep_launch_dependents();  // PDL (the combine waits for us)
#ifdef ARKV_TUNING_KNOBS
  if (lane == 0 && g_cta_on) {
    const int ci = cl.n_units > 0 ? (int)blockIdx.x : (int)(blockIdx.y * gridDim.x + blockIdx.x);
    if (ci < kCtaTimesMax) g_cta_t[ci][5 + warp] = gtimer();
  }
#endif
  acc_reduce_rows(acc);
  if (gq == 0) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int h = 2 * tq + e;
      if (h < G) {
        sm.wm[warp][h] = acc.m_run[e];
        sm.wl[warp][h] = acc.l_run[e];
#pragma unroll
        for (int gr = 0; gr < NG; ++gr) sm.wz[warp][h][gr] = acc.z_run[e][gr];
      }
    }
  }
  __syncthreads();  // every warp is done with the ring: reuse it for the O^T accumulators
  {
    float* ob = (float*)sm.ring[0] + warp * 8 * D;  // [col][dim]
#pragma unroll
    for (int mv = 0; mv < 8; ++mv) {
      const int x0 = mv * 16 + gq;
      ob[(2 * tq + 0) * D + x0] = acc.o[mv][0];
      ob[(2 * tq + 1) * D + x0] = acc.o[mv][1];
      ob[(2 * tq + 0) * D + x0 + 8] = acc.o[mv][2];
      ob[(2 * tq + 1) * D + x0 + 8] = acc.o[mv][3];
    }
  }
  __syncthreads();
  // ---- CTA merge of the warps (+ the appended token) -> split partial ----
  const float* ob = (const float*)sm.ring[0];
  float* part = a.partials + ((int64_t)u * a.max_splits + s) * G * (D + 2);
  for (int idx = threadIdx.x; idx < G * D; idx += C * 32) {
    const int h = idx / D, x = idx % D;
    const int gr = x / (D / NG);
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < C; ++w) M = fmaxf(M, sm.wm[w][h]);
    float snew = -INFINITY;
    if (owns_new) {
      snew = sm.newtok[h];
      M = fmaxf(M, snew);
    }
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < C; ++w) {
      const float mw = sm.wm[w][h];
      if (mw == -INFINITY) continue;
      const float cw = exp2f(mw - M);
      float ow = ob[(w * 8 + h) * D + x];
      if (G < 8) ow += ob[(w * 8 + h + G) * D + x];
      ow += sm.wz[w][h][gr];
      L += sm.wl[w][h] * cw;
      O += ow * cw;
    }
    if (owns_new) {
      const float cn = exp2f(snew - M - kPScale<F8>);  // the partials' probability scale (kPvSub)
      L += cn;
      O += cn * bf16_to_f(vn[x]);
    }
    part[h * (D + 2) + 2 + x] = O;
    if (x == 0) {
      part[h * (D + 2) + 0] = M;
      part[h * (D + 2) + 1] = L;
    }
  }
  // ---- fused combine (tuning builds, ARKV_FUSE_COMBINE): the last split CTA of the unit
  // to finish merges all partials ----
  if (a.fuse_combine) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) sm.is_last = atomicAdd(&a.counters[u], 1) == S - 1;
    __syncthreads();
    if (sm.is_last) {
      __threadfence();
      combine_unit<G>(a, u, b, li, kvh, dsc, nullptr, nullptr);
      if (threadIdx.x == 0) a.counters[u] = 0;
    }
  }
#ifdef ARKV_TUNING_KNOBS
  if (threadIdx.x == 0 && g_cta_on) {
    const int ci = cl.n_units > 0 ? (int)blockIdx.x : (int)(blockIdx.y * gridDim.x + blockIdx.x);
    if (ci < kCtaTimesMax) {
      unsigned smid;
      asm volatile("mov.u32 %0, %smid;\n" : "=r"(smid));
      g_cta_t[ci][0] = t_start;
      g_cta_t[ci][1] = gtimer();
      g_cta_t[ci][2] = ((unsigned long long)smid << 32) | (unsigned)(u * 64 + s);
      g_cta_t[ci][3] = ((unsigned long long)(o1 - o0) << 32) | (unsigned)(q1 - q0);
    }
  }
#endif
}

template <int G, int NG, bool F8, int C>
static void launch_chunk(const DecodeArgs& a, int n_units_call, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                         const UnitOrder* cl) {
  const int smem = (int)sizeof(Smem3<C>);
  static UnitOrder uniform = [] {
    UnitOrder u;
    u.n_units = 0;
    u.n_ctas = 0;
    return u;
  }();
  const dim3 grid = cl ? dim3(cl->n_ctas) : dim3(a.n_splits, n_units_call);
  auto kern = decode_chunk_kernel<G, NG, F8, C>;
  static const bool once = [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    carveout_max(kern);
    return true;
  }();
  (void)once;
  if (ev0) cudaEventRecord(ev0, s);
#ifdef ARKV_TUNING_KNOBS
  if (tuning_knob("ARKV_DECODE_NOPDL", 0)) {
    kern<<<grid, dim3(C * 32), (size_t)smem, s>>>(a, cl ? *cl : uniform);
    if (ev1) cudaEventRecord(ev1, s);
    return;
  }
#endif
  launch_pdl(kern, grid, dim3(C * 32), (size_t)smem, s, a, cl ? *cl : uniform);
  if (ev1) cudaEventRecord(ev1, s);
}

template <int G, int NG, int C, int SPW, bool F8 = false>
static void launch_cfg(const DecodeArgs& a, int n_units_call, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                       const UnitOrder* cl) {
  const int smem = (int)sizeof(Smem<C, SPW>);
  static UnitOrder uniform = [] {
    UnitOrder u;
    u.n_units = 0;
    u.n_ctas = 0;
    return u;
  }();
  const dim3 grid = cl ? dim3(cl->n_ctas) : dim3(a.n_splits, n_units_call);
  auto kern = decode_fast_kernel<G, NG, C, SPW, F8>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (ev0) cudaEventRecord(ev0, s);
  launch_pdl(kern, grid, dim3((C + 1) * 32), (size_t)smem, s, a, cl ? *cl : uniform);
  if (ev1) cudaEventRecord(ev1, s);
}

// Default pipeline shape: 3 consumer warps x 2 stages (96 KB ring, 2 CTAs/SM): every
// consumer warp has its next item in flight while it computes the current one (with one
// stage per warp, the warp waited a full HBM round trip per item: 21 % of the stall
// samples of the Base_quant profile).  Measured at configs[1]: kernel 0.1693 -> 0.1565 ms
// vs 4 x 1.  For the paper's shape (G = 4, one group) alternatives are selectable for
// measurement in tuning builds (-DARKV_TUNING_KNOBS) with ARKV_FAST_CFG=10*C+SPW (41 | 42 | 62 |
// 43 | 81 | 22 | 23); the shipped library instantiates only the default.
template <int G, int NG>
static void launch_gn(const DecodeArgs& a, int n_units_call, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                      const UnitOrder* cl) {
  // 4: chunked, 4 warps x 2 CTAs/SM (12 KB chunks); 2: the producer-ring kernel.  (3 warps x
  // 3 CTAs/SM measured 25 % slower, and 5 warps x 2 CTAs/SM with 9 KB chunks compiles to the
  // same 168 registers with spills: register files are allocated in multi-warp units; 8 warps
  // x 1 CTA/SM with 2, 3 or 4 CTAs per SM per step: 1-6 % slower.)
  static const int pipe = tuning_knob("ARKV_FAST_PIPE", 4);
  if (pipe == 4) {
    const bool f8 = a.g.mode == ARKV_QUANT_FP8;
    f8 ? launch_chunk<G, NG, true, 4>(a, n_units_call, s, ev0, ev1, cl)
       : launch_chunk<G, NG, false, 4>(a, n_units_call, s, ev0, ev1, cl);
    return;
  }
  if (a.g.mode == ARKV_QUANT_FP8) {
    launch_cfg<G, NG, 3, 2, true>(a, n_units_call, s, ev0, ev1, cl);
    return;
  }
#ifdef ARKV_TUNING_KNOBS
  if (G == 4 && NG == 1) {
    switch (tuning_knob("ARKV_FAST_CFG", 32)) {
      case 42: launch_cfg<G, NG, 4, 2>(a, n_units_call, s, ev0, ev1, cl); return;
      case 62: launch_cfg<G, NG, 6, 2>(a, n_units_call, s, ev0, ev1, cl); return;
      case 43: launch_cfg<G, NG, 4, 3>(a, n_units_call, s, ev0, ev1, cl); return;
      case 81: launch_cfg<G, NG, 8, 1>(a, n_units_call, s, ev0, ev1, cl); return;
      case 41: launch_cfg<G, NG, 4, 1>(a, n_units_call, s, ev0, ev1, cl); return;
      case 22: launch_cfg<G, NG, 2, 2>(a, n_units_call, s, ev0, ev1, cl); return;
      case 23: launch_cfg<G, NG, 2, 3>(a, n_units_call, s, ev0, ev1, cl); return;
      default: break;
    }
  }
#endif
  launch_cfg<G, NG, 3, 2>(a, n_units_call, s, ev0, ev1, cl);
}

template <int G>
static int launch_g(const DecodeArgs& a, int n_units_call, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                    const UnitOrder* cl) {
  switch (a.g.ng) {
    case 1: launch_gn<G, 1>(a, n_units_call, s, ev0, ev1, cl); return 0;
    case 2: launch_gn<G, 2>(a, n_units_call, s, ev0, ev1, cl); return 0;
    case 4: launch_gn<G, 4>(a, n_units_call, s, ev0, ev1, cl); return 0;
    default: return -1;
  }
}

// ---------------------------------------------------------------------------------------
// Persistent, range-partitioned variant (decode_kernel = 3).
// The step's items form two global streams — every unit's Original tiles, then every
// unit's Quantized tiles in groups of q_per — and the plan (PersistPlan, a kernel
// parameter) gives every CTA an equal contiguous range of each, so all CTAs stream the
// same bytes of each kind with one pipeline fill and drain.  The kernel is read-only on
// the cache: each consumer warp flushes a partial (m, l, o) per (unit, phase) it touched,
// and decode_persist_combine merges a unit's partials, appends the step's token and
// folds it in.
// ---------------------------------------------------------------------------------------
struct PUnit {
  int u;  // global unit index
  int slot, n_o, n_q, tiles_q, items;
  bool accm;
};
// query rows of unit ul (index in the call)
__device__ __forceinline__ const uint16_t* punit_q(const DecodeArgs& a, int ul) {
  const Geom& g = a.g;
  const int b = ul / (a.n_layers * g.Hkv);
  const int rem = ul % (a.n_layers * g.Hkv);
  const int li = rem / g.Hkv, kvh = rem % g.Hkv;
  return a.q + ((int64_t)(b * a.n_layers + li) * g.Hq + kvh * g.G) * D;
}
__device__ __forceinline__ int punit_global(const DecodeArgs& a, int ul) {
  const Geom& g = a.g;
  const int b = ul / (a.n_layers * g.Hkv);
  const int rem = ul % (a.n_layers * g.Hkv);
  return (b * g.L + a.layer0 + rem / g.Hkv) * g.Hkv + rem % g.Hkv;
}
__device__ __forceinline__ void punit_fill(const DecodeArgs& a, const UnitDesc& dsc, int u, int f, int q_per,
                                           PUnit& p) {
  const Geom& g = a.g;
  p.u = u;
  p.slot = dsc.slot;
  p.n_o = dsc.n_o;
  p.n_q = dsc.n_q;
  p.tiles_q = (p.n_q + kTile - 1) / kTile;
  p.items = f == 0 ? (p.n_o + kTile - 1) / kTile : (p.tiles_q + q_per - 1) / q_per;
  p.accm = (dsc.t_next >= dsc.acc0) && (dsc.t_next < dsc.trig);
}
// Position in one phase range of a CTA: item k of unit ul.  Walks forward only (units
// with no items of the phase are stepped over); the next unit's descriptor is prefetched
// so a unit change does not stall the producer on a dependent load.
struct Walker {
  int ul, k, rem, U;
  PUnit p;
  UnitDesc nxt;
  __device__ __forceinline__ void prefetch(const DecodeArgs& a) {
    if (ul + 1 < U) nxt = a.desc[punit_global(a, ul + 1)];
  }
  __device__ __forceinline__ void init(const DecodeArgs& a, const int4& r, int f, int q_per, int n_units) {
    ul = r.x;
    k = r.y;
    rem = r.z;
    U = n_units;
    if (rem > 0) {
      const int u = punit_global(a, ul);
      punit_fill(a, a.desc[u], u, f, q_per, p);
      prefetch(a);
    }
  }
  __device__ __forceinline__ void next(const DecodeArgs& a, int f, int q_per) {
    if (--rem <= 0) return;
    ++k;
    while (k >= p.items) {
      k -= p.items;
      ++ul;
      punit_fill(a, nxt, punit_global(a, ul), f, q_per, p);
      prefetch(a);
    }
  }
};
// Ring of C x kPersistSpw stages: item j -> stage j % (C SPW), consumer warp j % C, so each
// stage has a single owner warp that waits on its barriers strictly in phase order.
template <int C>
struct PSmem {
  static constexpr int kSt = C * kPersistSpw;
  uint8_t ring[kSt][kStageBytes];
  uint64_t full[kSt];
  uint64_t empty[kSt];
  int4 info[kSt][2];  // per stage, written by the producer: (ul, u, k, phase), (n_o, n_q, tiles_q, accm)
};

template <int G, int NG, bool F8>
__global__ void __launch_bounds__((kPersistConsumers + 1) * 32, 2)
    decode_persist_kernel(const __grid_constant__ DecodeArgs a, const __grid_constant__ PersistPlan plan) {
  constexpr int C = kPersistConsumers;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  PSmem<C>& sm = *reinterpret_cast<PSmem<C>*>(smem_raw);
  const Geom& g = a.g;
  griddep_wait();  // PDL: the previous kernel (tailor / combine) has completed
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int c = blockIdx.x;
  const int n_work = plan.cta[0][c].z + plan.cta[1][c].z;
  const int q_per = kStageBytes / g.tile_q;
  const int row_stride = g.cap_o + g.cap_q;
  const float c2 = g.sm_scale * kLog2e;
  const bool sym = g.mode == ARKV_QUANT_SYM;
  const int n_units_call = g.batch * a.n_layers * g.Hkv;
  if (threadIdx.x == 0) {
    for (int i = 0; i < PSmem<C>::kSt; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    // where this CTA's partials live (per phase; -1: empty range), for the combine
    for (int f = 0; f < 2; ++f) {
      const int4 r = plan.cta[f][c];
      a.pcta[f * kPlanMaxCtas + c] = make_int4(r.z > 0 ? r.x : -1, r.w, plan.ue[f][c], 0);
    }
  }
  __syncthreads();
  if (n_work <= 0) {
    if (threadIdx.x == 0) griddep_launch_dependents();
    return;
  }

  if (warp == C) {
    // ============ producer: merges the two ranges by unit (a unit's Original tiles, then
    // its Quantized groups) so each consumer warp accumulates a unit across both kinds ============
    if (lane == 0) {
      const uint64_t pol_stream = l2_evict_first();
      Walker w0, w1;
      w0.init(a, plan.cta[0][c], 0, q_per, n_units_call);
      w1.init(a, plan.cta[1][c], 1, q_per, n_units_call);
      auto issue = [&](Walker& w, int f, int j) {
        const PUnit& p = w.p;
        // the CTAs holding a unit's first and last item of the phase, for the combine
        if (w.k == 0) a.pcover[(f * 2 + 0) * n_units_call + w.ul] = c;
        if (w.k == p.items - 1) a.pcover[(f * 2 + 1) * n_units_call + w.ul] = c;
        constexpr int NS = PSmem<C>::kSt;
        const int st = j % NS;
        if (j >= NS) mbar_wait(&sm.empty[st], ((j / NS) - 1) & 1);
        sm.info[st][0] = make_int4(w.ul, p.u, w.k, f);
        sm.info[st][1] = make_int4(p.n_o, p.n_q, p.tiles_q, p.accm ? 1 : 0);
        uint8_t* slot = a.slots + (int64_t)p.slot * g.slot_bytes;
        const uint8_t* src;
        uint32_t bytes;
        if (f == 0) {
          src = o_tile_ptr(slot, g, w.k);
          bytes = (uint32_t)g.tile_o;
        } else {
          const int first = w.k * q_per, nt = min(q_per, p.tiles_q - first);
          src = q_tile_ptr(slot, g, first + nt - 1);
          bytes = (uint32_t)(nt * g.tile_q);
        }
        mbar_expect_tx(&sm.full[st], bytes);  // release: orders the info writes above
        if (a.l2_hints)
          bulk_g2s_hint(sm.ring[st], src, bytes, &sm.full[st], pol_stream);
        else
          bulk_g2s(sm.ring[st], src, bytes, &sm.full[st]);
      };
      // per unit: Original tiles first on even CTAs, Quantized groups first on odd ones, so
      // co-resident CTAs tend to overlap HBM-bound and ALU-heavy work
      const bool q_first = (c & 1) && a.item_order != 0;
      for (int j = 0; j < n_work; ++j) {
        const bool take0 = w0.rem > 0 && (w1.rem <= 0 || (q_first ? w0.ul < w1.ul : w0.ul <= w1.ul));
        if (take0) {
          issue(w0, 0, j);
          w0.next(a, 0, q_per);
        } else {
          issue(w1, 1, j);
          w1.next(a, 1, q_per);
        }
      }
      griddep_launch_dependents();  // PDL: the combine may start launching (it waits for us)
    }
    __syncwarp();
    return;  // no CTA-wide barrier follows
  }

  // ===================== consumers =====================
  const int src_t = G >= 2 ? ((2 * tq) % G) / 2 : 0;
  const int src_lane = (lane & ~3) | src_t;
  QFrag<NG> qf;
  Acc<NG> acc;
  int cur = -1;
  // partial of (unit cur, this CTA, this warp): m, l and o (z term folded in)
  auto flush = [&]() {
    acc_reduce_rows(acc);
    const int4 r0 = plan.cta[0][c];
    const bool in0 = r0.z > 0 && cur >= r0.x && cur <= plan.ue[0][c];
    const int4 r = in0 ? r0 : plan.cta[1][c];
    const int slot_idx = r.w + (cur - r.x) * C + warp;
    float* part = a.pparts + (int64_t)slot_idx * G * (D + 2);
#pragma unroll
    for (int mv = 0; mv < 8; ++mv) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        // column 2t+(e&1) of dim row mv*16+gq+8(e>>1); for G < 8 columns h and h+G hold
        // the hi and lo halves of head h's P'
        float v = acc.o[mv][e];
        if (G == 4) v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (G == 2) v += __shfl_xor_sync(0xffffffffu, v, 1);
        if (G == 1) v += acc.o[mv][e ^ 1];
        const int h = G == 1 ? 0 : 2 * tq + (e & 1);
        const bool writer = G == 8 ? true : (G == 1 ? (tq == 0 && (e & 1) == 0) : (2 * tq < G));
        if (writer && h < G) {
          const int x = mv * 16 + gq + 8 * (e >> 1);
          const int gr = x / (D / NG);
          part[h * (D + 2) + 2 + x] = v + acc.z_run[e & 1][gr];
        }
      }
    }
    if (gq == 0) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int h = 2 * tq + e;
        if (h < G) {
          part[h * (D + 2) + 0] = acc.m_run[e];
          part[h * (D + 2) + 1] = acc.l_run[e];
        }
      }
    }
  };
  const uint64_t lpol = l2_evict_last();  // HH logits stay in L2 for the combine
  for (int j = warp; j < n_work; j += C) {
    constexpr int NS = PSmem<C>::kSt;
    const int st = j % NS;
    mbar_wait(&sm.full[st], (j / NS) & 1);
    __syncwarp();  // mma/movmatrix are .aligned
    const int4 i0 = sm.info[st][0], i1 = sm.info[st][1];
    if (i0.x != cur) {
      if (cur >= 0) flush();
      load_qfrag<G, NG, F8>(punit_q(a, i0.x), lane, qf);
      cur = i0.x;
      acc_reset(acc);
    }
    const int u = i0.y, k = i0.z;
    float* lbase = i1.w ? a.logits + (int64_t)u * row_stride * G : nullptr;
    if (i0.w == 0) {
      consume_tile<G, NG, F8>(sm.ring[st], false, min(kTile, i1.x - k * kTile), lbase ? lbase + k * kTile * G : nullptr,
                          row_stride, lpol, qf, acc, c2, sym, lane, src_lane);
    } else {
      const int first = k * q_per, nt = min(q_per, i1.z - first);
      for (int jt = 0; jt < nt; ++jt) {
        const int tile = first + jt;
        consume_tile<G, NG, F8>(sm.ring[st] + (nt - 1 - jt) * g.tile_q, true, min(kTile, i1.y - tile * kTile),
                            lbase ? lbase + (g.cap_o + tile * kTile) * G : nullptr, row_stride, lpol, qf, acc,
                            c2, sym, lane, src_lane);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[st]);
  }
  if (cur >= 0) flush();
}

// One CTA (G x D threads: one per head and dim) per unit: append the step's token (D1),
// its logits (and HH logit row), merge the unit's warp partials with it, write the output
// and the merged row statistics, advance the descriptor.
template <int G>
__global__ void __launch_bounds__(G * D) decode_persist_combine(DecodeArgs a) {
  griddep_wait();
  griddep_launch_dependents();
  constexpr int C = kPersistConsumers;
  const Geom& g = a.g;
  const int ul = blockIdx.x, n_units_call = gridDim.x;
  const int b = ul / (a.n_layers * g.Hkv);
  const int rem = ul % (a.n_layers * g.Hkv);
  const int li = rem / g.Hkv, kvh = rem % g.Hkv;
  const int u = (b * g.L + a.layer0 + li) * g.Hkv + kvh;
  const UnitDesc dsc = a.desc[u];
  const int n_o = dsc.n_o, tid = threadIdx.x, h = tid / D, x = tid % D, lane = tid & 31;
  const bool lead = x < 32;  // the first warp of head h's group
  const int64_t qkv = (int64_t)(b * a.n_layers + li);
  const uint16_t* qp = a.q + (qkv * g.Hq + kvh * G) * D;
  const uint16_t* kn = a.k + (qkv * g.Hkv + kvh) * D;
  const uint16_t* vn = a.v + (qkv * g.Hkv + kvh) * D;
  const bool accm = (dsc.t_next >= dsc.acc0) && (dsc.t_next < dsc.trig);
  const int row_stride = g.cap_o + g.cap_q;
  __shared__ float s_new[G], sM[G], sIL[G];
  __shared__ float s_w[kMaxUnitParts][G];  // merge weight 2^(m - M) of each slot (0: unused)
  __shared__ int s_slot[kMaxUnitParts];
  __shared__ int s_cov[4];
  // ---- the CTAs covering the unit (first, last per phase); cleared for the next step ----
  if (tid < 4) s_cov[tid] = a.pcover[(tid >> 1) * 2 * n_units_call + (tid & 1) * n_units_call + ul];
  // ---- append the token to the Original stack (row n_o) ----
  const uint16_t vx = vn[x];
  // non-finite q / k / v of the step
  if (bf16_nonfinite(qp[tid]) || (h == 0 && (bf16_nonfinite(kn[x]) || bf16_nonfinite(vx)))) atomicOr(a.err, kErrNonFinite);
  if (h == 0) {
    const int tiles_o = (n_o + 1 + kTile - 1) / kTile, tiles_q = (dsc.n_q + kTile - 1) / kTile;
    const bool fits =
        (n_o + 1 <= g.cap_o) && ((int64_t)tiles_o * g.tile_o + (int64_t)tiles_q * g.tile_q <= g.slot_bytes);
    uint8_t* slot = a.slots + (int64_t)dsc.slot * g.slot_bytes;
    if (fits) {
      uint8_t* tb = o_tile_ptr(slot, g, n_o / kTile);
      *(uint16_t*)(tb + o_k_off(g, n_o % kTile, x)) = kn[x];
      *(uint16_t*)(tb + o_v_off(g, n_o % kTile, x)) = vx;
      if (x == 0) {
        const SlotMeta meta = slot_meta(a.meta, g, dsc.slot);
        meta.pos_o[n_o] = dsc.t_next;
        meta.acc_o[n_o] = make_float2(0.f, 0.f);
      }
    } else if (x == 0) {
      atomicOr(a.err, kErrCapacity);
    }
  }
  // ---- its logit for head h (log2 domain) ----
  const float c2 = g.sm_scale * kLog2e;
  if (lead) {
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc = fmaf(bf16_to_f(qp[h * D + lane * 4 + i]), bf16_to_f(kn[lane * 4 + i]), acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      s_new[h] = acc * c2;
      if (accm) st_hint(a.logits + ((int64_t)u * row_stride + n_o) * G + h, acc * c2, l2_evict_last());
    }
  }
  __syncthreads();
  if (tid < 4) a.pcover[(tid >> 1) * 2 * n_units_call + (tid & 1) * n_units_call + ul] = -1;
  // ---- candidate partial slots: C per covering CTA and phase.  A slot whose warp processed
  // none of the unit's items holds l = 0 (slots start zeroed and every combine clears the
  // l of the slots it merged) ----
  const int nc0 = s_cov[0] >= 0 ? (s_cov[1] - s_cov[0] + 1) * C : 0;
  const int nc1 = s_cov[2] >= 0 ? (s_cov[3] - s_cov[2] + 1) * C : 0;
  const int ncand = min(nc0 + nc1, kMaxUnitParts);
  for (int k = tid; k < ncand; k += G * D) {
    const int f = k < nc0 ? 0 : 1, kk = f == 0 ? k : k - nc0;
    const int cc = s_cov[2 * f] + kk / C;
    int4 pc = a.pcta[f * kPlanMaxCtas + cc];
    // a CTA between the first and last covering ones may have an empty range of the phase
    // (fewer items than CTAs): skipped.  A unit inside a CTA's phase-0 span uses its
    // phase-0 slots even for Quantized items: enumerated once.
    bool use = pc.x >= 0;
    if (use && f == 1) {
      const int4 p0 = a.pcta[cc];
      if (p0.x >= 0 && ul >= p0.x && ul <= p0.z) {
        pc = p0;
        if (s_cov[0] >= 0 && cc >= s_cov[0] && cc <= s_cov[1]) use = false;
      }
    }
    s_slot[k] = use ? pc.y + (ul - pc.x) * C + kk % C : -1;
  }
  __syncthreads();
  const float* pp = a.pparts;
  // merged max and sum of head h (its lead warp)
  if (lead) {
    float M = s_new[h];
    for (int k = lane; k < ncand; k += 32) {
      if (s_slot[k] < 0) continue;
      const float* ph = pp + ((int64_t)s_slot[k] * G + h) * (D + 2);
      if (__ldcg(ph + 1) > 0.f) M = fmaxf(M, __ldcg(ph));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    float L = lane == 0 ? exp2f(s_new[h] - M - a.pscale) : 0.f;
    for (int k = lane; k < ncand; k += 32) {
      const float* ph = pp + ((int64_t)max(s_slot[k], 0) * G + h) * (D + 2);
      const float l = s_slot[k] >= 0 ? __ldcg(ph + 1) : 0.f;
      const float w = l > 0.f ? exp2f(__ldcg(ph) - M) : 0.f;
      s_w[k][h] = w;
      L += l * w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o);
    if (lane == 0) {
      sM[h] = M;
      sIL[h] = 1.0f / L;
      a.mstat[((int64_t)u * G + h) * 2 + 0] = M;
      a.mstat[((int64_t)u * G + h) * 2 + 1] = 1.0f / L;
    }
  }
  __syncthreads();
  float O = exp2f(s_new[h] - sM[h] - a.pscale) * bf16_to_f(vx);
#pragma unroll 4
  for (int k = 0; k < ncand; ++k) {
    const float w = s_w[k][h];
    if (w != 0.f) O += __ldcg(pp + ((int64_t)s_slot[k] * G + h) * (D + 2) + 2 + x) * w;
  }
  O *= sIL[h];
  const int64_t obase = (qkv * g.Hq + kvh * G) * D;
  if (a.out_fp32)
    ((float*)a.out)[obase + h * D + x] = O;
  else
    ((uint16_t*)a.out)[obase + h * D + x] = f_to_bf16_rne(O);
  // clear the merged slots' l for the next step's plan
  for (int k = tid; k < ncand * G; k += G * D)
    if (s_slot[k / G] >= 0) a.pparts[((int64_t)s_slot[k / G] * G + k % G) * (D + 2) + 1] = 0.f;
  if (tid == 0) {
    UnitDesc nd = dsc;
    nd.n_o = n_o + 1;
    nd.t_next = dsc.t_next + 1;
    a.desc[u] = nd;
  }
}

template <int G, int NG, bool F8>
static void launch_persist(const DecodeArgs& a, const PersistPlan& plan, int n_units_call, cudaStream_t s,
                           cudaEvent_t ev0, cudaEvent_t ev1) {
  auto kern = decode_persist_kernel<G, NG, F8>;
  const int smem = (int)sizeof(PSmem<kPersistConsumers>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (ev0) cudaEventRecord(ev0, s);
  launch_pdl(kern, dim3(plan.P), dim3((kPersistConsumers + 1) * 32), (size_t)smem, s, a, plan);
  if (ev1) cudaEventRecord(ev1, s);
  launch_pdl(decode_persist_combine<G>, dim3(n_units_call), dim3(G * D), 0, s, a);
}
template <int G>
static int launch_persist_g(const DecodeArgs& a, const PersistPlan& plan, int n_units_call, cudaStream_t s,
                            cudaEvent_t ev0, cudaEvent_t ev1) {
  const bool f8 = a.g.mode == ARKV_QUANT_FP8;
  switch (a.g.ng) {
    case 1: f8 ? launch_persist<G, 1, true>(a, plan, n_units_call, s, ev0, ev1)
               : launch_persist<G, 1, false>(a, plan, n_units_call, s, ev0, ev1); return 2;
    case 2: f8 ? launch_persist<G, 2, true>(a, plan, n_units_call, s, ev0, ev1)
               : launch_persist<G, 2, false>(a, plan, n_units_call, s, ev0, ev1); return 2;
    case 4: f8 ? launch_persist<G, 4, true>(a, plan, n_units_call, s, ev0, ev1)
               : launch_persist<G, 4, false>(a, plan, n_units_call, s, ev0, ev1); return 2;
    default: return -1;
  }
}

}  // namespace fast

bool decode_fast_available(const Geom& g) {
  const bool fmt = g.bits == 4 || (g.bits == 8 && g.mode == ARKV_QUANT_FP8);
  return g.layout == ARKV_LAYOUT_FRAG && g.d == fast::D && fmt && (g.ng == 1 || g.ng == 2 || g.ng == 4) &&
         (g.G == 1 || g.G == 2 || g.G == 4 || g.G == 8);
}

void launch_decode_combine(const DecodeArgs& a, int n_units_call, cudaStream_t s);  // k_decode.cu

void launch_decode_combine_hh(const DecodeArgs& a, const HhPlan& hp, int max_rows, cudaStream_t s);  // k_decode.cu

// Returns the launches issued, + 100 when the step's HH accumulation ran inside the combine.
float decode_fast_pscale(const Geom& g) {
  return g.mode == ARKV_QUANT_FP8 ? fast::kPScale<true> : fast::kPScale<false>;
}

int launch_decode_fast(const DecodeArgs& a, int n_units_call, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                       const PersistPlan* plan, const HhPlan* hh, int acc_rows, const UnitOrder* chunks) {
  if (!decode_fast_available(a.g)) return -1;
  if (plan) {  // persistent range-partitioned kernel + its combine
    switch (a.g.G) {
      case 1: return fast::launch_persist_g<1>(a, *plan, n_units_call, s, ev0, ev1);
      case 2: return fast::launch_persist_g<2>(a, *plan, n_units_call, s, ev0, ev1);
      case 4: return fast::launch_persist_g<4>(a, *plan, n_units_call, s, ev0, ev1);
      case 8: return fast::launch_persist_g<8>(a, *plan, n_units_call, s, ev0, ev1);
      default: return -1;
    }
  }
  int r = -1;
  switch (a.g.G) {
    case 1: r = fast::launch_g<1>(a, n_units_call, s, ev0, ev1, chunks); break;
    case 2: r = fast::launch_g<2>(a, n_units_call, s, ev0, ev1, chunks); break;
    case 4: r = fast::launch_g<4>(a, n_units_call, s, ev0, ev1, chunks); break;
    case 8: r = fast::launch_g<8>(a, n_units_call, s, ev0, ev1, chunks); break;
    default: return -1;
  }
  if (r < 0) return -1;
  if (a.fuse_combine) {  // the last split CTA of each unit merged the partials
    if (!hh) return 1;
    HhPlan hp = *hh;  // the heavy-hitter rows only (no combine blocks)
    hp.n_units = 0;
    launch_decode_combine_hh(a, hp, acc_rows, s);
    return 102;
  }
  if (hh) {
    launch_decode_combine_hh(a, *hh, acc_rows, s);
    return 102;
  }
  launch_decode_combine(a, n_units_call, s);
  return 2;
}

}  // namespace arkv

#ifdef ARKV_TUNING_KNOBS
// on >= 0: enable/disable recording; out != nullptr: copy n records (8 x u64 each: start, end,
// smid << 32 | unit * 64 + split, O tiles << 32 | Q tiles, first item staged, warp 0..2 done).
extern "C" int arkv_debug_cta_clear() {
  static unsigned long long zeros[arkv::fast::kCtaTimesMax][8] = {};
  cudaMemcpyToSymbol(arkv::fast::g_cta_t, zeros, sizeof(zeros));
  return (int)cudaGetLastError();
}
extern "C" int arkv_debug_occupancy(int which) {
  int nb = -1;
  if (which == 0)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, arkv::fast::decode_chunk_kernel<4, 1, false, 4>, 128,
                                                  sizeof(arkv::fast::Smem3<4>));
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, arkv::fast::decode_fast_kernel<4, 1, 3, 2, false>, 128,
                                                  sizeof(arkv::fast::Smem<3, 2>));
  return nb;
}
extern "C" int arkv_debug_cta_times(int on, unsigned long long* out, int n) {
  if (on >= 0) cudaMemcpyToSymbol(arkv::fast::g_cta_on, &on, sizeof(int));
  if (out) {
    cudaDeviceSynchronize();
    n = n < arkv::fast::kCtaTimesMax ? n : arkv::fast::kCtaTimesMax;
    cudaMemcpyFromSymbol(out, arkv::fast::g_cta_t, (size_t)n * 8 * sizeof(unsigned long long));
  }
  return (int)cudaGetLastError();
}
#endif
