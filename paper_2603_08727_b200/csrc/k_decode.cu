// k_decode.cu — decode attention over O ∪ Q (D1, D3, D7 of DESIGN.md §2).
//
// Split-K (flash-decoding) over each unit's 32-token tiles: split s of S takes an
// equal share of the unit's Original tiles and of its Quantized tiles, so every
// split streams the same bytes.  Each CTA appends the step's token (D1) if it owns
// the last Original tile, runs an online softmax over its tiles (Quantized tokens
// are dequantized in registers: x̃ = code·s + z), and writes a partial
// (m, l, o).  The combine kernel merges the partials, writes the output, performs
// the heavy-hitter accumulation acc1 += Σ_h p, acc2 += Σ_h p² of the W steps before
// the next tailor (Eq. 9 / R19) from the logits the split kernel kept, and advances
// the unit descriptor.  This generic kernel handles every layout/shape; the fast
// tensor-core kernel (k_decode_fast.cu) takes FRAG-layout 4-bit d=128 caches.
#include <cstdlib>

#include "combine.cuh"

namespace arkv {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ void unit_of(const DecodeArgs& a, int ul, int& b, int& li, int& kvh, int& u) {
  const Geom& g = a.g;
  b = ul / (a.n_layers * g.Hkv);
  int rem = ul % (a.n_layers * g.Hkv);
  li = rem / g.Hkv;
  kvh = rem % g.Hkv;
  u = (b * g.L + a.layer0 + li) * g.Hkv + kvh;
}

__device__ __forceinline__ void bf16x8_to_f(uint4 w, float (&f)[8]) {
  uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(ww[i] << 16);
    f[2 * i + 1] = __uint_as_float(ww[i] & 0xFFFF0000u);
  }
}

// Generic split kernel.  LG lanes per token, each lane owns 8 consecutive dims.
template <int G, int LG>
__global__ void __launch_bounds__(128) decode_split_generic(DecodeArgs a) {
  constexpr int TPP = 32 / LG;  // tokens per warp pass
  griddep_wait();
  const Geom& g = a.g;
  const int d = g.d;
  int b, li, kvh, u;
  unit_of(a, blockIdx.y, b, li, kvh, u);
  const UnitDesc dsc = a.desc[u];
  uint8_t* slot = a.slots + (int64_t)dsc.slot * g.slot_bytes;
  const SlotMeta sm = slot_meta(a.meta, g, dsc.slot);
  const int n_o = dsc.n_o, n_q = dsc.n_q, t = dsc.t_next;
  const bool accm = (t >= dsc.acc0) && (t < dsc.trig);
  const int tiles_o = (n_o + 1 + kTile - 1) / kTile;
  const int tiles_q = (n_q + kTile - 1) / kTile;
  const int S = a.n_splits, s = blockIdx.x;
  const int o0 = (int)((int64_t)s * tiles_o / S), o1 = (int)((int64_t)(s + 1) * tiles_o / S);
  const int q0 = (int)((int64_t)s * tiles_q / S), q1 = (int)((int64_t)(s + 1) * tiles_q / S);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tp = lane / LG, ld = lane % LG;
  const int x0 = ld * 8;
  const int row_stride = g.cap_o + g.cap_q;

  const uint16_t* qp = a.q + ((int64_t)(b * a.n_layers + li) * g.Hq + kvh * G) * d;
  const uint16_t* kn = a.k + ((int64_t)(b * a.n_layers + li) * g.Hkv + kvh) * d;
  const uint16_t* vn = a.v + ((int64_t)(b * a.n_layers + li) * g.Hkv + kvh) * d;
  const float qs = g.sm_scale * kLog2e;

  float qf[G][8];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    float f[8];
    bf16x8_to_f(*(const uint4*)(qp + h * d + x0), f);
#pragma unroll
    for (int i = 0; i < 8; ++i) qf[h][i] = f[i] * qs;
  }
  float m[G], l[G], o[G][8];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    m[h] = -INFINITY;
    l[h] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) o[h][i] = 0.f;
  }

  // Append the step's token (D1) — by the CTA owning the last Original tile.
  if (o0 <= n_o / kTile && n_o / kTile < o1 && warp == 0) {
    // non-finite q / k / v of the step
    if (warp_step_nonfinite(qp, G * d, kn, vn, d, lane) && lane == 0) atomicOr(a.err, kErrNonFinite);
    const int tt = n_o / kTile, j = n_o % kTile;
    bool fits = (n_o + 1 <= g.cap_o) &&
                ((int64_t)tiles_o * g.tile_o + (int64_t)tiles_q * g.tile_q <= g.slot_bytes);
    if (!fits) {
      if (lane == 0) atomicOr(a.err, kErrCapacity);
    } else {
      uint8_t* tb = o_tile_ptr(slot, g, tt);
      for (int x = lane; x < d; x += 32) {
        *(uint16_t*)(tb + o_k_off(g, j, x)) = kn[x];
        *(uint16_t*)(tb + o_v_off(g, j, x)) = vn[x];
      }
      if (lane == 0) {
        sm.pos_o[n_o] = t;
        sm.acc_o[n_o] = make_float2(0.f, 0.f);
      }
    }
  }

  const int n_work = (o1 - o0) + (q1 - q0);
  for (int wi = warp; wi < n_work; wi += 4) {
    const bool isq = wi >= (o1 - o0);
    const int tile = isq ? q0 + (wi - (o1 - o0)) : o0 + wi;
    const uint8_t* tb = isq ? q_tile_ptr(slot, g, tile) : o_tile_ptr(slot, g, tile);
    for (int p0 = 0; p0 < kTile; p0 += TPP) {
      const int j = p0 + tp;
      const int row = tile * kTile + j;
      const bool valid = isq ? row < n_q : row <= n_o;
      float kf[8], vf[8];
      if (valid) {
        if (!isq) {
          if (row == n_o) {
            bf16x8_to_f(*(const uint4*)(kn + x0), kf);
            bf16x8_to_f(*(const uint4*)(vn + x0), vf);
          } else if (g.layout != ARKV_LAYOUT_FRAG) {
            bf16x8_to_f(*(const uint4*)(tb + o_k_off(g, j, x0)), kf);
            bf16x8_to_f(*(const uint4*)(tb + o_v_off(g, j, x0)), vf);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              kf[i] = bf16_to_f(*(const uint16_t*)(tb + o_k_off(g, j, x0 + i)));
              vf[i] = bf16_to_f(*(const uint16_t*)(tb + o_v_off(g, j, x0 + i)));
            }
          }
        } else {
          const int grp = x0 / g.g;
          const float ks = *(const float*)(tb + q_sc_off(g, j, 0, grp));
          const float kz = *(const float*)(tb + q_sc_off(g, j, 1, grp));
          const float vs = *(const float*)(tb + q_sc_off(g, j, 2, grp));
          const float vz = *(const float*)(tb + q_sc_off(g, j, 3, grp));
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            int byte, shift;
            q_k_loc(g, j, x0 + i, &byte, &shift);
            const float ck = code_value(g, (tb[byte] >> shift) & ((1u << g.bits) - 1u));
            q_v_loc(g, j, x0 + i, &byte, &shift);
            const float cv = code_value(g, (tb[byte] >> shift) & ((1u << g.bits) - 1u));
            kf[i] = ck * ks + kz;
            vf[i] = cv * vs + vz;
          }
        }
      }
      float sc[G];
#pragma unroll
      for (int h = 0; h < G; ++h) {
        float acc = 0.f;
        if (valid) {
#pragma unroll
          for (int i = 0; i < 8; ++i) acc = fmaf(qf[h][i], kf[i], acc);
        }
#pragma unroll
        for (int msk = 1; msk < LG; msk <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, msk);
        sc[h] = acc;
      }
      if (valid) {
        if (accm && ld == 0) {
          const int ridx = isq ? g.cap_o + row : row;
#pragma unroll
          for (int h = 0; h < G; ++h) a.logits[((int64_t)u * row_stride + ridx) * G + h] = sc[h];
        }
#pragma unroll
        for (int h = 0; h < G; ++h) {
          float mn = fmaxf(m[h], sc[h]);
          float cr = exp2f(m[h] - mn);
          float p = exp2f(sc[h] - mn);
          l[h] = l[h] * cr + p;
#pragma unroll
          for (int i = 0; i < 8; ++i) o[h][i] = fmaf(p, vf[i], o[h][i] * cr);
          m[h] = mn;
        }
      }
    }
  }

  // merge the TPP lane groups of the warp (same dims, different tokens)
#pragma unroll
  for (int msk = LG; msk < 32; msk <<= 1) {
#pragma unroll
    for (int h = 0; h < G; ++h) {
      float mo = __shfl_xor_sync(0xffffffffu, m[h], msk);
      float lo = __shfl_xor_sync(0xffffffffu, l[h], msk);
      float mn = fmaxf(m[h], mo);
      float ca = mn == -INFINITY ? 0.f : exp2f(m[h] - mn);
      float cb = mn == -INFINITY ? 0.f : exp2f(mo - mn);
      l[h] = l[h] * ca + lo * cb;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float oo = __shfl_xor_sync(0xffffffffu, o[h][i], msk);
        o[h][i] = o[h][i] * ca + oo * cb;
      }
      m[h] = mn;
    }
  }
  // merge the 4 warps through shared memory
  __shared__ float sm_m[4][G], sm_l[4][G];
  extern __shared__ float sm_o[];  // [4][G][d]
  if (lane < LG) {
#pragma unroll
    for (int h = 0; h < G; ++h) {
      if (lane == 0) {
        sm_m[warp][h] = m[h];
        sm_l[warp][h] = l[h];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) sm_o[(warp * G + h) * d + x0 + i] = o[h][i];
    }
  }
  __syncthreads();
  float* part = a.partials + ((int64_t)u * a.max_splits + s) * G * (d + 2);
  for (int idx = threadIdx.x; idx < G * d; idx += blockDim.x) {
    int h = idx / d, x = idx % d;
    float M = -INFINITY;
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w][h]);
    float L = 0.f, O = 0.f;
    for (int w = 0; w < 4; ++w) {
      float c = (M == -INFINITY) ? 0.f : exp2f(sm_m[w][h] - M);
      L += sm_l[w][h] * c;
      O += sm_o[(w * G + h) * d + x] * c;
    }
    part[h * (d + 2) + 2 + x] = O;
    if (x == 0) {
      part[h * (d + 2) + 0] = M;
      part[h * (d + 2) + 1] = L;
    }
  }
}

// Combine: merge split partials, write the output, HH accumulation, advance the unit.
template <int G>
__global__ void __launch_bounds__(1024) decode_combine(DecodeArgs a) {
  griddep_wait();
  griddep_launch_dependents();
  int b, li, kvh, u;
  unit_of(a, blockIdx.x, b, li, kvh, u);
  const UnitDesc dsc = a.desc[u];
  __shared__ float sM[G], sIL[G];
  combine_unit<G>(a, u, b, li, kvh, dsc, sM, sIL);
}

// Heavy-hitter accumulation (Eq. 9, D3; R19): in the W steps before a unit's next
// tailor, every cached row gets acc1 += Σ_h p, acc2 += Σ_h p² with p = 2^(s - M) / L
// from the step's logits and the merged row statistics.  Launched after the combine
// (the descriptor already counts the appended token); one thread per row.
template <int G>
__global__ void __launch_bounds__(256) decode_hh_acc(DecodeArgs a) {
  griddep_wait();
  const Geom& g = a.g;
  int b, li, kvh, u;
  unit_of(a, blockIdx.y, b, li, kvh, u);
  const UnitDesc dsc = a.desc[u];
  const int t = dsc.t_next - 1;  // the step just attended
  if (!((t >= dsc.acc0) && (t < dsc.trig))) return;
  const bool first = t == dsc.acc0;
  const int n_rows = dsc.n_o + dsc.n_q;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  float M[G], IL[G];
#pragma unroll
  for (int h = 0; h < G; ++h) {
    M[h] = a.mstat[((int64_t)u * G + h) * 2 + 0];
    IL[h] = a.mstat[((int64_t)u * G + h) * 2 + 1];
  }
  const SlotMeta sm = slot_meta(a.meta, g, dsc.slot);
  const int row_stride = g.cap_o + g.cap_q;
  const bool isq = i >= dsc.n_o;
  const int ridx = isq ? g.cap_o + (i - dsc.n_o) : i;
  float a1 = 0.f, a2 = 0.f;
#pragma unroll
  for (int h = 0; h < G; ++h) {
    const float p = exp2f(a.logits[((int64_t)u * row_stride + ridx) * G + h] - M[h] - a.pscale) * IL[h];
    a1 += p;
    a2 += p * p;
  }
  float2* ap = isq ? &sm.acc_q[i - dsc.n_o] : &sm.acc_o[i];
  if (first) {
    *ap = make_float2(a1, a2);
  } else {
    const float2 c = *ap;
    *ap = make_float2(c.x + a1, c.y + a2);
  }
}

#ifndef ARKV_HH_LANE_MERGE
#define ARKV_HH_LANE_MERGE 0
#endif
constexpr bool kHhLaneMerge = ARKV_HH_LANE_MERGE != 0;

// one combine thread per (head, dim) up to 1024 (measured: latency-bound otherwise)
static int combine_threads(const Geom& g) { return std::min(1024, std::max(128, (g.G * g.d + 31) / 32 * 32)); }

// Split combine with the step's HH accumulation in the same grid (saves the separate
// decode_hh_acc launch and its drain).  Combine blocks as decode_combine; an HH block
// recomputes its unit's merged (M, 1/L) with the combine's own code (bit-identical: the
// default lane-per-head merge_splits; ARKV_HH_LANE_MERGE=1 with ARKV_COMBINE_WARP_MERGE=1
// is the whole-warp merge_ml_warp in both, measured in DESIGN §16b and not the default) —
// then folds rows [chunk * R, chunk * R + R) exactly as decode_hh_acc does.
// (8 rows per thread run as 256-thread blocks: bounding them at 256 threads leaves the rows'
// logits and accumulators in registers — at 1024 the 64-register cap spilled them)
// (3 blocks/SM via launch bounds: spills, step +2 us; not kept)
template <int G, int kHhRowsPerThread>
__global__ void __launch_bounds__(kHhRowsPerThread == 8 ? 256 : 1024) decode_combine_hh(DecodeArgs a, const HhPlan hp) {
  griddep_wait();
  griddep_launch_dependents();
  const Geom& g = a.g;
  if ((int)blockIdx.x < hp.n_units) {
    int b, li, kvh, u;
    unit_of(a, blockIdx.x, b, li, kvh, u);
    const UnitDesc dsc = a.desc[u];
    combine_unit<G>(a, u, b, li, kvh, dsc, nullptr, nullptr);
    return;
  }
  // block -> (entry, chunk of its rows, KV head): binary search of the entry's first chunk
  const int idx = blockIdx.x - hp.n_units;
  const int cg = idx / g.Hkv, kvh = idx - cg * g.Hkv;
  int lo = 0, hi = hp.n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (hp.coff[mid] <= cg) lo = mid; else hi = mid - 1;
  }
  const int4 en = hp.e[lo];
  const int R = blockDim.x * kHhRowsPerThread;
  const int n_rows = en.y, r0 = (cg - hp.coff[lo]) * R;
  const int b = en.x / a.n_layers, li = en.x % a.n_layers;
  const int u = (b * g.L + a.layer0 + li) * g.Hkv + kvh;
  const bool first = (en.z & 1) != 0;
  const int S_hh = (en.z >> 1) > 0 ? (en.z >> 1) : a.n_splits;  // no dependent nsplit load
  const int n_o = n_rows - en.w;  // Original rows, the appended token included
  // the slot is not changed by the combine's descriptor advance
  // (the descriptor load before the accumulator addresses costs nothing measurable: with the
  // slot known up front — slot == unit in the first HH window — the step time was unchanged)
  const SlotMeta sm = slot_meta(a.meta, g, a.desc[u].slot);
  const int row_stride = g.cap_o + g.cap_q;
  // every row load of the thread is issued before the merged statistics are needed (the
  // logits do not depend on them): kHhRowsPerThread rows x (G logits + acc) in flight
  float lg[kHhRowsPerThread][G];
  float2 ac[kHhRowsPerThread];
  const uint64_t pol = l2_evict_last();  // logits and accumulators stay L2-resident over the window
#pragma unroll
  for (int k = 0; k < kHhRowsPerThread; ++k) {
    const int i = r0 + threadIdx.x + k * blockDim.x;
    const bool ok = i < n_rows;
    const bool isq = i >= n_o;
    const int ridx = isq ? g.cap_o + (i - n_o) : i;
    const float* lp = a.logits + ((int64_t)u * row_stride + ridx) * G;  // the row's G logits: one vector load
    if constexpr (G == 4) {
      const float4 v4 = ok ? ld_hint4(lp, pol) : make_float4(0.f, 0.f, 0.f, 0.f);
      lg[k][0] = v4.x;
      lg[k][1] = v4.y;
      lg[k][2] = v4.z;
      lg[k][3] = v4.w;
    } else {
#pragma unroll
      for (int h = 0; h < G; ++h) lg[k][h] = ok ? ld_hint(lp + h, pol) : 0.f;
    }
  }
  // the accumulators' addresses wait for the descriptor's slot: loaded after every logit load
  // has been issued
#pragma unroll
  for (int k = 0; k < kHhRowsPerThread; ++k) {
    const int i = r0 + threadIdx.x + k * blockDim.x;
    ac[k] = make_float2(0.f, 0.f);
    if (i < n_rows && !first) ac[k] = ld_hint(i >= n_o ? &sm.acc_q[i - n_o] : &sm.acc_o[i], pol);
  }
  // the unit's merged (M, 1/L) per head, merged by each warp itself (lane h merges head h
  // with the combine's code, bit for bit, and broadcasts it): no block barrier between the
  // rows' loads and their use (a __syncthreads here was the kernel's top stall)
  float sM[G], sIL[G];
  if constexpr (kHhLaneMerge) {
    // the whole warp merges (one memory round trip instead of ceil(S / 8) dependent ones);
    // lane h holds head h's result
    const int lane = threadIdx.x & 31;
    const float* part = a.partials + (int64_t)u * a.max_splits * G * (g.d + 2);
    float M, L;
    merge_ml_warp<G>(part, lane, S_hh, g.d, M, L);
    const float ilh = 1.0f / L;
#pragma unroll
    for (int h = 0; h < G; ++h) {
      sM[h] = __shfl_sync(0xffffffffu, M, h);
      sIL[h] = __shfl_sync(0xffffffffu, ilh, h);
    }
  } else {
    const int lane = threadIdx.x & 31;
    float mh = 0.f, ilh = 0.f;
    if (lane < G) {
      const float* part = a.partials + (int64_t)u * a.max_splits * G * (g.d + 2);
      float M, L, O;
      merge_splits<G, false>(part, lane, 0, S_hh, g.d, M, L, O);
      mh = M;
      ilh = 1.0f / L;
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < G; ++h) {
      sM[h] = __shfl_sync(0xffffffffu, mh, h);
      sIL[h] = __shfl_sync(0xffffffffu, ilh, h);
    }
  }
#pragma unroll
  for (int k = 0; k < kHhRowsPerThread; ++k) {
    const int i = r0 + threadIdx.x + k * blockDim.x;
    if (i >= n_rows) break;
    float a1 = 0.f, a2 = 0.f;
#pragma unroll
    for (int h = 0; h < G; ++h) {
      const float p = ex2_approx_ftz(lg[k][h] - sM[h] - a.pscale) * sIL[h];  // rel. error < 2^-22
      a1 += p;
      a2 += p * p;
    }
    float2* ap = i >= n_o ? &sm.acc_q[i - n_o] : &sm.acc_o[i];
    st_hint(ap, make_float2(ac[k].x + a1, ac[k].y + a2), pol);
  }
}

void launch_decode_combine_hh(const DecodeArgs& a, const HhPlan& hp, int max_rows, cudaStream_t s) {
  // 256 threads x 8 rows per HH block (measured against 512 x 4: more rows in flight per
  // thread, the same 2048 rows per block); the combine blocks loop over their G * d outputs
  static const int rpt = tuning_knob("ARKV_HH_RPT", 8);
  HhPlan p = hp;
  const int threads = rpt == 8 ? 256 : combine_threads(a.g);
  const int R = threads * rpt;
  (void)max_rows;
  p.coff[0] = 0;
  for (int i = 0; i < p.n; ++i) p.coff[i + 1] = p.coff[i] + std::max(1, (p.e[i].y + R - 1) / R);
  p.n_chunks = p.coff[p.n];
  const dim3 grid(p.n_units + p.n_chunks * a.g.Hkv);
#define HH_CASE(GV)                                                                                          \
  case GV:                                                                                                   \
    if (rpt == 8) {                                                                                          \
      static const bool once = (carveout_max(decode_combine_hh<GV, 8>), true);                               \
      (void)once;                                                                                            \
      launch_pdl(decode_combine_hh<GV, 8>, grid, dim3(threads), 0, s, a, p);                                 \
    } else                                                                                                   \
      launch_pdl(decode_combine_hh<GV, 4>, grid, dim3(threads), 0, s, a, p);                                 \
    break;
  switch (a.g.G) {
    HH_CASE(1)
    HH_CASE(2)
    HH_CASE(4)
    HH_CASE(8)
    default: break;
  }
#undef HH_CASE
}

void launch_decode_hh_acc(const DecodeArgs& a, int n_units_call, int max_rows, cudaStream_t s) {
  dim3 grid((max_rows + 255) / 256, n_units_call);
  switch (a.g.G) {
    case 1: launch_pdl(decode_hh_acc<1>, grid, dim3(256), 0, s, a); break;
    case 2: launch_pdl(decode_hh_acc<2>, grid, dim3(256), 0, s, a); break;
    case 4: launch_pdl(decode_hh_acc<4>, grid, dim3(256), 0, s, a); break;
    case 8: launch_pdl(decode_hh_acc<8>, grid, dim3(256), 0, s, a); break;
    default: break;
  }
}

// k_decode_fast.cu: returns -1 if the cache is not eligible.
int launch_decode_fast(const DecodeArgs& a, int n_units_call, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1,
                       const PersistPlan* plan, const HhPlan* hh, int acc_rows, const UnitOrder* chunks);
void launch_decode_combine(const DecodeArgs& a, int n_units_call, cudaStream_t s);


template <int G>
static void launch_g(const DecodeArgs& a, int n_units_call, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1) {
  dim3 grid(a.n_splits, n_units_call);
  size_t smem = (size_t)4 * G * a.g.d * sizeof(float);
  if (ev0) cudaEventRecord(ev0, s);
  switch (a.g.d / 8) {
#define LG_CASE(LGV) \
  case LGV:          \
    launch_pdl(decode_split_generic<G, LGV>, grid, dim3(128), smem, s, a); \
    break;
    LG_CASE(2)
    LG_CASE(4)
    LG_CASE(8)
    LG_CASE(16)
    LG_CASE(32)
#undef LG_CASE
    default:
      break;
  }
  if (ev1) cudaEventRecord(ev1, s);
  launch_pdl(decode_combine<G>, dim3(n_units_call), dim3(combine_threads(a.g)), 0, s, a);
}

void launch_decode_combine(const DecodeArgs& a, int n_units_call, cudaStream_t s) {
  static const bool once = (carveout_max(decode_combine<1>), carveout_max(decode_combine<2>),
                            carveout_max(decode_combine<4>), carveout_max(decode_combine<8>), true);
  (void)once;
  switch (a.g.G) {
    case 1: launch_pdl(decode_combine<1>, dim3(n_units_call), dim3(combine_threads(a.g)), 0, s, a); break;
    case 2: launch_pdl(decode_combine<2>, dim3(n_units_call), dim3(combine_threads(a.g)), 0, s, a); break;
    case 4: launch_pdl(decode_combine<4>, dim3(n_units_call), dim3(combine_threads(a.g)), 0, s, a); break;
    case 8: launch_pdl(decode_combine<8>, dim3(n_units_call), dim3(combine_threads(a.g)), 0, s, a); break;
    default: break;
  }
}

int launch_decode(const Geom& g, int layer0, int n_layers, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                  void* out, int out_fp32, uint8_t* slots, uint8_t* meta, UnitDesc* desc, float* partials,
                  float* logits, float* mstat, int32_t* counters, int acc_rows, int n_splits, int max_splits,
                  int fast, int32_t* err, cudaStream_t s, cudaEvent_t ev0, cudaEvent_t ev1, const PlanArgs& plan) {
  DecodeArgs a;
  a.persist = fast && plan.plan ? 1 : 0;
  a.pparts = plan.pparts;
  a.pcta = plan.pcta;
  a.pcover = plan.pcover;
  a.g = g;
  a.layer0 = layer0;
  a.n_layers = n_layers;
  a.n_splits = n_splits;
  a.max_splits = max_splits;
  a.q = q;
  a.k = k;
  a.v = v;
  a.slots = slots;
  a.meta = meta;
  a.desc = desc;
  a.partials = partials;
  a.logits = logits;
  a.mstat = mstat;
  a.counters = counters;
  a.nsplit = (fast && plan.chunks && !plan.plan) ? plan.nsplit : nullptr;
  {
    a.q_group = tuning_knob("ARKV_QGROUP", 0);          // default: as many Q tiles as fit a stage
    a.interleave = tuning_knob("ARKV_INTERLEAVE", 0);   // measured: interleaving O/Q items is slower
    a.fuse_combine = tuning_knob("ARKV_FUSE_COMBINE", 0);  // measured: the separate combine kernel is faster
    a.prefetch = tuning_knob("ARKV_PREFETCH", 0);
    a.item_order = tuning_knob("ARKV_ITEM_ORDER", 1);   // measured: alternating O-first / Q-first CTAs -1.2 %
    a.l2_hints = tuning_knob("ARKV_L2_HINTS", 1);
    a.self_refill = tuning_knob("ARKV_SELF_REFILL", 1);
#ifdef ARKV_TUNING_KNOBS
    a.hh_nostore = tuning_knob("ARKV_HH_NOSTORE", 0);  // measurement of the store cost only
#else
    a.hh_nostore = 0;
#endif
  }
  a.pscale = fast ? decode_fast_pscale(g) : 0.f;
  a.out = out;
  a.out_fp32 = out_fp32;
  a.err = err;
  const int n_units_call = g.batch * n_layers * g.Hkv;
  int n = -1;
  if (fast) {
    n = launch_decode_fast(a, n_units_call, s, ev0, ev1, plan.plan, acc_rows > 0 ? plan.hh : nullptr, acc_rows,
                           a.nsplit ? plan.chunks : nullptr);
    if (n < 0) return n;
    if (n >= 100) return n - 100;  // the combine folded the HH accumulation
  } else {
    switch (g.G) {
      case 1: launch_g<1>(a, n_units_call, s, ev0, ev1); break;
      case 2: launch_g<2>(a, n_units_call, s, ev0, ev1); break;
      case 4: launch_g<4>(a, n_units_call, s, ev0, ev1); break;
      case 8: launch_g<8>(a, n_units_call, s, ev0, ev1); break;
      default: return -1;
    }
    n = 2;
  }
  if (acc_rows > 0) {
    launch_decode_hh_acc(a, n_units_call, acc_rows, s);
    ++n;
  }
  return n;
}

}  // namespace arkv
