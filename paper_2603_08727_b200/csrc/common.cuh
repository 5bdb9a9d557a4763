// common.cuh — geometry, device descriptors and the HBM tile layouts of the ARKV cache.
//
// A "unit" is one (sequence, layer, KV head).  Its tokens live in one arena SLOT of
// slot_bytes, used as a two-stack: 32-token Original tiles grow up from
// offset 0, 32-token Quantized tiles grow down from the end.  Eq. 1's byte budget
// (R10) bounds n_o*C_o + n_q*C_q <= B_bytes + C_o, so the stacks never
// meet in a slot of B_bytes + C_o + one tile of each kind.
//
// Two tile layouts:
//   PLAIN — token rows: O row = K[d] bf16 | V[d] bf16; Q row = K codes | V codes |
//           k_scale[ng] | k_zero[ng] | v_scale[ng] | v_zero[ng] (fp32).
//   FRAG  — "fragment-native": every 16-byte vector a lane loads is exactly the
//           register fragment of an mma.sync.m16n8k16 operand (K rows as the A
//           operand of QK^T, V transposed as the A operand of PV), so the fast
//           decode kernel streams tiles with fully coalesced 128-bit loads and no
//           shared-memory transposes.  Q tiles store 4-bit codes nibble-interleaved
//           for the fp16 "magic number" unpack (one LOP3 per two codes); per-token
//           scale/zero quads after the codes.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <stdint.h>

#include "../../include/arkv.h"

namespace arkv {

constexpr int kTile = 32;  // tokens per tile

// Device error flag bits (arkv_check).
enum : int32_t { kErrNonFinite = 1, kErrCapacity = 2, kErrIntegrity = 4 };

struct Geom {
  int32_t d, G, Hq, Hkv, L, batch, W, bits, g, ng, mode, layout;
  int32_t B;                      // budget tokens
  int32_t cost_o, cost_q;         // bytes per token (Eq. 1 C_orig, C_quant; R10)
  int32_t tile_o, tile_q;         // bytes per 32-token tile
  int32_t cap_o, cap_q;           // row capacity of the per-slot metadata (multiples of 32)
  int32_t max_pos, n_units;
  int64_t slot_bytes;             // bytes per slot (two-stack)
  int64_t meta_bytes;             // per-slot metadata: pos_o, pos_q, acc_o, acc_q
  float sm_scale, gamma;
  int32_t share;                  // 1: layer-shared token states (NEXT-3)
  float smooth;                   // λ of the smoothed scores (R34, NEXT-4); 0 = off
};

struct __align__(32) UnitDesc {
  int32_t slot;    // arena slot of the unit's tiles
  int32_t n_o;     // Original rows (window included; excludes the token of the running step)
  int32_t n_q;     // Quantized rows
  int32_t t_next;  // position of the next appended token
  int32_t trig;    // position of the next tailor (R12, R15)
  int32_t acc0;    // first position whose query is an Eq. 9 sample of that tailor (R19):
                   // max(trig - W, first query on the current cache)
  int32_t pad1, pad2;
};

// ---------------------------------------------------------------------------------
// Slot addressing
// ---------------------------------------------------------------------------------
__host__ __device__ inline uint8_t* o_tile_ptr(uint8_t* slot, const Geom& g, int tile) {
  return slot + (int64_t)tile * g.tile_o;
}
__host__ __device__ inline uint8_t* q_tile_ptr(uint8_t* slot, const Geom& g, int tile) {
  return slot + g.slot_bytes - (int64_t)(tile + 1) * g.tile_q;
}
struct SlotMeta {
  int32_t* pos_o;
  int32_t* pos_q;
  float2* acc_o;
  float2* acc_q;
  float* sp_o;  // smoothed score of each row at the tailor that wrote it (smooth > 0 only)
  float* sp_q;
};
__host__ __device__ inline SlotMeta slot_meta(uint8_t* meta_base, const Geom& g, int slot) {
  uint8_t* m = meta_base + (int64_t)slot * g.meta_bytes;
  SlotMeta s;
  s.pos_o = (int32_t*)m;
  s.pos_q = s.pos_o + g.cap_o;
  s.acc_o = (float2*)(s.pos_q + g.cap_q);
  s.acc_q = s.acc_o + g.cap_o;
  s.sp_o = (float*)(s.acc_q + g.cap_q);
  s.sp_q = s.sp_o + g.cap_o;
  return s;
}

// ---------------------------------------------------------------------------------
// Tile layouts: byte offset of element (token j in [0,32), dim x in [0,d)) in a tile.
// ---------------------------------------------------------------------------------
// Offset of per-lane word k of lane `lane` in a "lane word stream" block: lanes'
// words are grouped in quads so one 128-bit load per lane reads four consecutive
// words of that lane and a warp-wide load is one contiguous 512-byte segment.
__host__ __device__ inline int lane_word(int k, int lane) { return (((k >> 2) * 32 + lane) << 2) + (k & 3); }

// O tile, K element (bf16).
__host__ __device__ inline int o_k_off(const Geom& g, int j, int x) {
  if (g.layout != ARKV_LAYOUT_FRAG) return (j * 2 * g.d + x) * 2;
  // A operand of S = K q^T (m16n8k16, M = tokens): thread (gg,t) holds rows gg, gg+8
  // of each 16-token m-tile and, per 16-dim chunk c, dims t*(d/4)+4c+{0,1} (R0/R1)
  // and t*(d/4)+4c+{2,3} (R2/R3).
  int mt = j >> 4, jj = j & 15, h = jj >> 3, gg = jj & 7;
  int q4 = g.d >> 2;
  int t = x / q4, rem = x % q4, c = rem >> 2, e = rem & 3;
  int lane = 4 * gg + t;
  int k = ((mt * 2 + h) * (g.d >> 4) + c) * 2 + (e >> 1);
  return lane_word(k, lane) * 4 + (e & 1) * 2;
}
// O tile, V element (bf16).
__host__ __device__ inline int o_v_off(const Geom& g, int j, int x) {
  if (g.layout != ARKV_LAYOUT_FRAG) return (j * 2 * g.d + g.d + x) * 2;
  // A operand of O^T = V^T P^T (M = dims, K = tokens): thread (gg,t) holds dim rows
  // gg (sel 0) / gg+8 (sel 1) of each 16-dim m-tile and tokens 2t,2t+1 (hi 0) /
  // 2t+8,2t+9 (hi 1) of each 16-token k-step kc; register R = sel + 2 hi.
  int mtv = x >> 4, r = x & 15, gg = r & 7, sel = r >> 3;
  int kc = j >> 4, jj = j & 15, hi = jj >> 3, tt = jj & 7, t = tt >> 1, u = tt & 1;
  int lane = 4 * gg + t;
  int k = (mtv * 2 + kc) * 4 + sel + 2 * hi;
  return 64 * g.d + lane_word(k, lane) * 4 + u * 2;
}

// FRAG, 8-bit codes (fp8 e4m3, NEXT-2): every code byte sits where the f16 mma.sync
// fragment it converts into (one cvt.rn.f16x2.e4m3x2 per byte pair) needs it.
//  K block (A operand of S = K q^T, M = tokens, K = dims): quad ((mt*d/32 + ks/2)*32 + lane),
//    byte (ks&1)*8 + 2r + e holds token mt*16 + 8(r&1) + gg, dim 16ks + 8(r>>1) + 2t + e.
//  V block (A operand of O^T = V^T P'^T, M = dims, K = tokens): quad (mtv*32 + lane),
//    byte kc*8 + 2r + e holds dim 16mtv + 8(r&1) + gg, token 16kc + 8(r>>1) + 2t + e.
//  (lane = 4gg + t; register r = row half + 2 * column half.)
__host__ __device__ inline int f8_k_off(const Geom& g, int j, int x) {
  const int mt = j >> 4, rh = (j >> 3) & 1, gg = j & 7;
  const int ks = x >> 4, ch = (x >> 3) & 1, t = (x & 7) >> 1, e = x & 1;
  return ((mt * (g.d >> 5) + (ks >> 1)) * 32 + 4 * gg + t) * 16 + (ks & 1) * 8 + (rh + 2 * ch) * 2 + e;
}
__host__ __device__ inline int f8_v_off(const Geom& g, int j, int x) {
  const int mtv = x >> 4, rh = (x >> 3) & 1, gg = x & 7;
  const int kc = j >> 4, ch = (j >> 3) & 1, t = (j & 7) >> 1, e = j & 1;
  return 32 * g.d + (mtv * 32 + 4 * gg + t) * 16 + kc * 8 + (rh + 2 * ch) * 2 + e;
}
__host__ __device__ inline bool frag8(const Geom& g) { return g.layout == ARKV_LAYOUT_FRAG && g.bits == 8; }

// Q tile codes: returns the byte offset of the byte holding the code and its bit shift.
__host__ __device__ inline void q_k_loc(const Geom& g, int j, int x, int* byte, int* shift) {
  if (frag8(g)) {
    *byte = f8_k_off(g, j, x);
    *shift = 0;
    return;
  }
  if (g.layout != ARKV_LAYOUT_FRAG) {
    int bit = x * g.bits;
    *byte = j * g.cost_q + (bit >> 3);
    *shift = bit & 7;
    return;
  }
  // 4-bit, d % 32 == 0.  Word (row, t, jp) nibble e holds dim 32 jp + 8 t + e.
  int mt = j >> 4, jj = j & 15, h = jj >> 3, gg = jj & 7;
  int jp = x >> 5, t = (x >> 3) & 3, e = x & 7;
  int lane = 4 * gg + t;
  int k = (mt * 2 + h) * (g.d >> 5) + jp;
  int w = lane_word(k, lane);
  *byte = w * 4 + (e >> 1);
  *shift = (e & 1) * 4;
}
__host__ __device__ inline void q_v_loc(const Geom& g, int j, int x, int* byte, int* shift) {
  if (frag8(g)) {
    *byte = f8_v_off(g, j, x);
    *shift = 0;
    return;
  }
  if (g.layout != ARKV_LAYOUT_FRAG) {
    int bit = x * g.bits;
    *byte = j * g.cost_q + (g.d * g.bits >> 3) + (bit >> 3);
    *shift = bit & 7;
    return;
  }
  // V transposed: word (dim row, t) nibble e holds token (kc*16 + hi*8 + 2t + u)
  // with e = 2 kc + hi + 4 u.
  int mtv = x >> 4, r = x & 15, gg = r & 7, sel = r >> 3;
  int kc = j >> 4, jj = j & 15, hi = jj >> 3, tt = jj & 7, t = tt >> 1, u = tt & 1;
  int e = 2 * kc + hi + 4 * u;
  int lane = 4 * gg + t;
  int k = mtv * 2 + sel;
  int w = (g.d >> 3) * 32 + lane_word(k, lane);  // after the K block (16 d bytes = 4 d words)
  *byte = w * 4 + (e >> 1);
  *shift = (e & 1) * 4;
}
// which: 0 k_scale, 1 k_zero, 2 v_scale, 3 v_zero.
__host__ __device__ inline int q_sc_off(const Geom& g, int j, int which, int grp) {
  if (g.layout != ARKV_LAYOUT_FRAG) return j * g.cost_q + 2 * (g.d * g.bits >> 3) + (which * g.ng + grp) * 4;
  if (frag8(g)) return 64 * g.d + ((j * g.ng + grp) * 4 + which) * 4;
  // per row and group the four floats k_scale, k_zero, v_scale, v_zero are adjacent: one
  // 16-byte shared-memory load each in the decode kernel (conflict-free: rows 16 B apart)
  return 32 * g.d + ((j * g.ng + grp) * 4 + which) * 4;
}

// Inverse of q_k_loc / q_v_loc: the code held by slot s (s < 8/bits, at bit s*bits) of
// byte B of a Quantized tile.  Returns false for scale/zero bytes.
__host__ __device__ inline bool q_code_slot(const Geom& g, int B, int s, int* j, int* x, int* isv) {
  if (g.layout != ARKV_LAYOUT_FRAG) {
    const int per = 8 / g.bits, cb = g.d * g.bits / 8;
    const int row = B / g.cost_q, off = B % g.cost_q;
    if (off >= 2 * cb) return false;
    *j = row;
    *isv = off >= cb;
    *x = (*isv ? off - cb : off) * per + s;
    return true;
  }
  if (frag8(g)) {
    if (B >= 64 * g.d) return false;
    const bool v = B >= 32 * g.d;
    const int bl = v ? B - 32 * g.d : B;
    const int qd = bl >> 4, w = bl & 15, lane = qd & 31, gg = lane >> 2, t = lane & 3;
    const int hk = w >> 3, r = (w & 7) >> 1, e = w & 1, rh = r & 1, ch = r >> 1;
    if (!v) {
      const int q = qd >> 5, nq = g.d >> 5, mt = q / nq, ks = (q % nq) * 2 + hk;
      *j = mt * 16 + rh * 8 + gg;
      *x = ks * 16 + ch * 8 + 2 * t + e;
    } else {
      const int mtv = qd >> 5;
      *x = mtv * 16 + rh * 8 + gg;
      *j = hk * 16 + ch * 8 + 2 * t + e;
    }
    *isv = v ? 1 : 0;
    return true;
  }
  if (B >= 32 * g.d) return false;
  const bool v = B >= 16 * g.d;
  const int bl = v ? B - 16 * g.d : B;
  const int w = bl >> 2, bw = bl & 3;
  const int lane = (w >> 2) & 31, k = ((w >> 7) << 2) | (w & 3);
  const int gg = lane >> 2, t = lane & 3;
  const int e = 2 * bw + s;
  if (!v) {
    const int nq = g.d >> 5;
    const int mth = k / nq, jp = k % nq;
    *j = (mth >> 1) * 16 + (mth & 1) * 8 + gg;
    *x = 32 * jp + 8 * t + e;
    *isv = 0;
  } else {
    const int mtv = k >> 1, sel = k & 1;
    *x = 16 * mtv + 8 * sel + gg;
    *j = 16 * ((e >> 1) & 1) + 8 * (e & 1) + 2 * t + (e >> 2);
    *isv = 1;
  }
  return true;
}

// Programmatic dependent launch: a kernel launched with programmatic stream
// serialization may start while its predecessor drains; it must wait before touching
// memory the predecessor writes.  Both are no-ops for ordinary launches.
// L2 residency hints (createpolicy + .L2::cache_hint).  The HH window's logits and
// accumulators (~70 MB at configs[1]) are kept resident with evict_last while the cache
// tiles stream through with evict_first, so the logit round trip between the decode kernel
// and the HH combine stays in the 126 MB L2 instead of HBM.
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_hint(float* p, float v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;\n" ::"l"(p), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_hint(float2* p, float2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;\n" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol)
               : "memory");
}
__device__ __forceinline__ float ld_hint(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;\n" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float4 ld_hint4(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float2 ld_hint(const float2* p, uint64_t pol) {
  float2 v;
  asm volatile("ld.global.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;\n" : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
  return v;
}
// 2^x on the SFU (ex2.approx.ftz: max relative error 2^-22; results below 2^-126 flush to 0)
__device__ __forceinline__ float ex2_approx_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

__device__ __forceinline__ float bf16_to_f(uint16_t b) { return __uint_as_float(((uint32_t)b) << 16); }
// Non-finite bf16 inputs (Inf, NaN: all-ones exponent) — SPEC S:329 "non-finite input ->
// numeric error", raised through kErrNonFinite and arkv_check (include/arkv.h).
__device__ __forceinline__ bool bf16_nonfinite(uint16_t b) { return (b & 0x7F80u) == 0x7F80u; }
__device__ __forceinline__ bool bf16x2_nonfinite(uint32_t w) {
  const uint32_t t = ~w & 0x7F807F80u;  // a half is non-finite iff its exponent bits are all set
  return (t & 0xFFFFu) == 0u || (t >> 16) == 0u;
}
__device__ __forceinline__ bool bf16x8_nonfinite(const uint4& v) {
  return bf16x2_nonfinite(v.x) | bf16x2_nonfinite(v.y) | bf16x2_nonfinite(v.z) | bf16x2_nonfinite(v.w);
}
// Non-zero iff one of the 8 bf16 values has an all-ones exponent: per word (two halves) the
// masked exponents + 0x0080 carry into bit 15 exactly for 0x7F80 (3 integer ops per word).
__device__ __forceinline__ uint32_t bf16x8_expmax_bits(const uint4& v) {
  const uint32_t m = 0x7F807F80u, c = 0x00800080u, top = 0x80008000u;
  return (((v.x & m) + c) | ((v.y & m) + c) | ((v.z & m) + c) | ((v.w & m) + c)) & top;
}
// One warp checks the step's q rows (n_q elements) and new k/v rows (n_kv elements each).
__device__ __forceinline__ bool warp_step_nonfinite(const uint16_t* q, int n_q, const uint16_t* k, const uint16_t* v,
                                                    int n_kv, int lane) {
  bool bad = false;
  for (int i = lane; i < n_q; i += 32) bad |= bf16_nonfinite(q[i]);
  for (int i = lane; i < n_kv; i += 32) bad |= bf16_nonfinite(k[i]) | bf16_nonfinite(v[i]);
  return __any_sync(0xffffffffu, bad);
}

// The number a stored Quantized code stands for (R23): the integer (minus the symmetric
// offset), or the e4m3 value of an fp8 code (NEXT-2).
__device__ __forceinline__ float code_value(const Geom& g, uint32_t raw) {
  if (g.mode == ARKV_QUANT_FP8) {
    const __half_raw h = __nv_cvt_fp8_to_halfraw((__nv_fp8_storage_t)raw, __NV_E4M3);
    return __half2float(__half(h));
  }
  return (float)((int)raw - (g.mode == ARKV_QUANT_SYM ? (1 << (g.bits - 1)) : 0));
}
__device__ __forceinline__ uint16_t f_to_bf16_rne(float f) {
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

}  // namespace arkv
