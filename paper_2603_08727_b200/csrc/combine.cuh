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

template <int G>
__device__ __forceinline__ void combine_unit(const DecodeArgs& a, int u, int b, int li, int kvh, const UnitDesc& dsc,
                                             float* sM, float* sIL) {
  const Geom& g = a.g;
  const int d = g.d;
  const int S = a.n_splits;
  const float* part = a.partials + (int64_t)u * a.max_splits * G * (d + 2);
  if (threadIdx.x < G) {
    const int h = threadIdx.x;
    float M = -INFINITY;
    for (int s = 0; s < S; ++s) M = fmaxf(M, __ldcg(part + (s * G + h) * (d + 2)));
    float L = 0.f;
    for (int s = 0; s < S; ++s) {
      const float ms = __ldcg(part + (s * G + h) * (d + 2));
      if (ms != -INFINITY) L += __ldcg(part + (s * G + h) * (d + 2) + 1) * exp2f(ms - M);
    }
    sM[h] = M;
    sIL[h] = 1.0f / L;
    a.mstat[((int64_t)u * G + h) * 2 + 0] = M;
    a.mstat[((int64_t)u * G + h) * 2 + 1] = 1.0f / L;
  }
  __syncthreads();
  const int64_t obase = ((int64_t)(b * a.n_layers + li) * g.Hq + kvh * G) * d;
  for (int idx = threadIdx.x; idx < G * d; idx += blockDim.x) {
    const int h = idx / d, x = idx % d;
    float O = 0.f;
    for (int s = 0; s < S; ++s) {
      const float ms = __ldcg(part + (s * G + h) * (d + 2));
      if (ms != -INFINITY) O += __ldcg(part + (s * G + h) * (d + 2) + 2 + x) * exp2f(ms - sM[h]);
    }
    O *= sIL[h];
    if (a.out_fp32)
      ((float*)a.out)[obase + idx] = O;
    else
      ((uint16_t*)a.out)[obase + idx] = f_to_bf16_rne(O);
  }
  if (threadIdx.x == 0) {
    UnitDesc nd = dsc;
    nd.n_o = dsc.n_o + 1;
    nd.t_next = dsc.t_next + 1;
    a.desc[u] = nd;
  }
}

}  // namespace arkv
