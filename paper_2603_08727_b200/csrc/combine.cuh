// combine.cuh — merge of a unit's split partials (flash-decoding reduction).
//
// partial[s][h] = (m, l, o[d]) with m in the log2 domain and o unnormalised relative
// to 2^m.  out[h][x] = Σ_s o_s 2^(m_s - M) / Σ_s l_s 2^(m_s - M).  Also records the
// merged (M, 1/L) per head for the heavy-hitter accumulation kernel and advances the
// unit descriptor (n_o += 1, t_next += 1).  Used by the stand-alone combine kernel and
// by the last-arriving CTA of the fused decode kernel.
#pragma once
#include "kernels.h"

namespace arkv {

// Merged max M (log2 domain), sum L and — WITH_O — output element o[x] of head h over the
// S split partials.  The (m, l, o) of up to kB splits are loaded as one batch of
// independent loads: one memory round trip per kB splits instead of three dependent ones
// (max, sum, output).  For S <= kB the order (global max, then the sums in split order) is
// the plain reduction's.  The HH rows of the fused combine call it without O and get the
// combine's M and L bit for bit.
template <int G, bool WITH_O>
__device__ __forceinline__ void merge_splits(const float* part, int h, int x, int S, int d, float& M, float& L,
                                             float& O) {
  constexpr int kB = 8;
  M = -INFINITY;
  L = 0.f;
  O = 0.f;
  for (int s0 = 0; s0 < S; s0 += kB) {
    float m[kB], l[kB], o[kB];
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      const int s = s0 + j;
      const float* p = part + (s * G + h) * (d + 2);
      m[j] = s < S ? __ldcg(p) : -INFINITY;
      l[j] = s < S ? __ldcg(p + 1) : 0.f;
      o[j] = (WITH_O && s < S) ? __ldcg(p + 2 + x) : 0.f;
    }
    float bm = M;
#pragma unroll
    for (int j = 0; j < kB; ++j) bm = fmaxf(bm, m[j]);
    if (bm == -INFINITY) continue;
    if (M != -INFINITY) {
      const float c = exp2f(M - bm);
      L *= c;
      if (WITH_O) O *= c;
    }
    M = bm;
#pragma unroll
    for (int j = 0; j < kB; ++j) {
      if (m[j] != -INFINITY) {
        const float w = exp2f(m[j] - M);
        L += l[j] * w;
        if (WITH_O) O += o[j] * w;
      }
    }
  }
}

// Merged (M, L) of every head over the S split partials, computed by one whole warp: lane
// h + G j takes head h's splits j, j + 32/G, j + 2 (32/G), ... (up to 32/G x kB splits per
// memory round trip — one round trip for the usual S <= 64 at G = 4, where merge_splits
// takes ceil(S / 8) dependent ones), then the 32/G lanes of a head fold their (m, l) with
// a butterfly.  Every lane returns its own head's (M, L).  The sum order differs from
// merge_splits' (rounding only: both are the flash-decoding reduction of the same terms).
template <int G>
__device__ __forceinline__ void merge_ml_warp(const float* part, int lane, int S, int d, float& M, float& L) {
  constexpr int J = 32 / G;  // lanes per head
  constexpr int kB = 4;
  const int h = lane % G, j = lane / G;
  M = -INFINITY;
  L = 0.f;
  for (int s0 = 0; s0 < S; s0 += J * kB) {
    float m[kB], l[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const int s = s0 + j + k * J;
      const float* p = part + (s * G + h) * (d + 2);
      m[k] = s < S ? __ldcg(p) : -INFINITY;
      l[k] = s < S ? __ldcg(p + 1) : 0.f;
    }
    float bm = M;
#pragma unroll
    for (int k = 0; k < kB; ++k) bm = fmaxf(bm, m[k]);
    if (bm == -INFINITY) continue;
    if (M != -INFINITY) L *= exp2f(M - bm);
    M = bm;
#pragma unroll
    for (int k = 0; k < kB; ++k)
      if (m[k] != -INFINITY) L += l[k] * exp2f(m[k] - M);
  }
#pragma unroll
  for (int off = G; off < 32; off <<= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, M, off), l2 = __shfl_xor_sync(0xffffffffu, L, off);
    const float mn = fmaxf(M, m2);
    if (mn != -INFINITY)
      L = (M != -INFINITY ? L * exp2f(M - mn) : 0.f) + (m2 != -INFINITY ? l2 * exp2f(m2 - mn) : 0.f);
    M = mn;
  }
}

template <int G>
__device__ __forceinline__ void combine_unit(const DecodeArgs& a, int u, int b, int li, int kvh, const UnitDesc& dsc,
                                             float* /*sM*/, float* /*sIL*/) {
  const Geom& g = a.g;
  const int d = g.d;
  const int S = a.nsplit ? a.nsplit[u] : a.n_splits;
  const float* part = a.partials + (int64_t)u * a.max_splits * G * (d + 2);
  const int64_t obase = ((int64_t)(b * a.n_layers + li) * g.Hq + kvh * G) * d;
#ifndef ARKV_COMBINE_WARP_MERGE
#define ARKV_COMBINE_WARP_MERGE 0
#endif
  if constexpr (ARKV_COMBINE_WARP_MERGE != 0) {
    // every warp merges all heads' (M, L) with all 32 lanes (merge_ml_warp: one round trip),
    // then each thread (head, dim) sums its S output partials at the known M: the loads of
    // a batch of kB splits are independent (no running rescale between batches)
    const int lane = threadIdx.x & 31;
    // the thread's first (head, dim): its first kB splits' (m, o) are loaded before the
    // warp merge (they do not depend on M), so a call with S <= kB takes one round trip
    constexpr int kB = 8;  // 16 spills under the 1024-thread bound (64 registers)
    float pm[kB], po[kB];
    {
      const int idx = threadIdx.x, h = idx / d, x = idx % d;
      const bool ok = idx < G * d;
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        const float* p = part + (j * G + h) * (d + 2);
        pm[j] = ok && j < S ? __ldcg(p) : -INFINITY;
        po[j] = ok && j < S ? __ldcg(p + 2 + x) : 0.f;
      }
    }
    float Mw, Lw;
    merge_ml_warp<G>(part, lane, S, d, Mw, Lw);
    float wM[G], wL[G];
#pragma unroll
    for (int h = 0; h < G; ++h) {
      wM[h] = __shfl_sync(0xffffffffu, Mw, h);
      wL[h] = __shfl_sync(0xffffffffu, Lw, h);
    }
    for (int idx = threadIdx.x; idx < G * d; idx += blockDim.x) {
      const int h = idx / d, x = idx % d;
      float M = wM[0], L = wL[0];
#pragma unroll
      for (int k = 1; k < G; ++k)
        if (h == k) {
          M = wM[k];
          L = wL[k];
        }
      float O = 0.f;
      int s0 = 0;
      if (idx == (int)threadIdx.x) {  // the prefetched first batch
#pragma unroll
        for (int j = 0; j < kB; ++j)
          if (pm[j] != -INFINITY) O += po[j] * exp2f(pm[j] - M);
        s0 = kB;
      }
      for (; s0 < S; s0 += kB) {
        float m[kB], o[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) {
          const float* p = part + ((s0 + j) * G + h) * (d + 2);
          m[j] = s0 + j < S ? __ldcg(p) : -INFINITY;
          o[j] = s0 + j < S ? __ldcg(p + 2 + x) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < kB; ++j)
          if (m[j] != -INFINITY) O += o[j] * exp2f(m[j] - M);
      }
      const float IL = 1.0f / L;
      O *= IL;
      if (a.out_fp32)
        ((float*)a.out)[obase + idx] = O;
      else
        ((uint16_t*)a.out)[obase + idx] = f_to_bf16_rne(O);
      if (x == 0) {
        a.mstat[((int64_t)u * G + h) * 2 + 0] = M;
        a.mstat[((int64_t)u * G + h) * 2 + 1] = IL;
      }
    }
  } else {
    // one thread per (head, dim); each merges its head's split statistics itself (redundant
    // across the head's d threads, but no shared-memory round and no __syncthreads)
    for (int idx = threadIdx.x; idx < G * d; idx += blockDim.x) {
      const int h = idx / d, x = idx % d;
      float M, L, O;
      merge_splits<G, true>(part, h, x, S, d, M, L, O);
      const float IL = 1.0f / L;
      O *= IL;
      if (a.out_fp32)
        ((float*)a.out)[obase + idx] = O;
      else
        ((uint16_t*)a.out)[obase + idx] = f_to_bf16_rne(O);
      if (x == 0) {
        a.mstat[((int64_t)u * G + h) * 2 + 0] = M;
        a.mstat[((int64_t)u * G + h) * 2 + 1] = IL;
      }
    }
  }
  if (threadIdx.x == 0) {
    UnitDesc nd = dsc;
    nd.n_o = dsc.n_o + 1;
    nd.t_next = dsc.t_next + 1;
    a.desc[u] = nd;
  }
}

}  // namespace arkv
