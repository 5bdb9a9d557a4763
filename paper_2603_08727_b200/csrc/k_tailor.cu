// k_tailor.cu — the tri-state tailor (D4-D6 / P4 of DESIGN.md §2).
//
//  select: heavy-hitter score S = μ + γ·max(0, acc2/N − μ²), μ = acc1/N, N = G·n_rows
//          (Eq. 9; R18, R20), then a block-wide 64-bit radix select of
//          the two rank thresholds of Eq. 10 over composite keys
//          (S desc, position asc; R22) -> new state per old row.
//  scan:   block-wide exclusive scans -> for every NEW row its source row (the
//          compaction map); writes the unit descriptor (counts, slot, next trigger).
//  move:   one CTA per destination tile: gathers its 32 tokens (Original copy,
//          Quantized -> Original promotion (R24), Original -> Quantized group
//          quantization with fp32 scale/zero in the oracle's operation order (R23),
//          Quantized -> Quantized code copy (R25)), assembles the tile in shared
//          memory and writes it out with coalesced 16-byte stores into a fresh slot.
#include <cstdlib>

#include "kernels.h"

namespace arkv {

enum : int32_t { kSrcInput = 1, kSrcOldO = 2, kSrcOldQ = 3 };

__device__ __forceinline__ uint64_t hh_key(float2 acc, int pos, float invN, float gamma) {
  float mu = __fmul_rn(acc.x, invN);
  float var = __fsub_rn(__fmul_rn(acc.y, invN), __fmul_rn(mu, mu));
  var = fmaxf(var, 0.f);
  float S = __fadd_rn(mu, __fmul_rn(gamma, var));
  uint32_t b = __float_as_uint(S);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // order-preserving map of fp32
  if (S == 0.f) b = 0x80000000u;                    // -0 == +0
  return ((uint64_t)b << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)pos);
}

struct RowView {
  const float2* acc_o;
  const float2* acc_q;
  const float* sp_o;  // smoothed scores of the previous tailor (R34; smooth > 0, decode only)
  const float* sp_q;
  const int32_t* pos_o;
  const int32_t* pos_q;
  int n_elig_o, n_q;
  bool prefill;
  __device__ float sp(int i) const { return i < n_elig_o ? sp_o[i] : sp_q[i - n_elig_o]; }
  __device__ void get(int i, float2& a, int& p) const {
    if (i < n_elig_o) {
      a = acc_o[i];
      p = prefill ? i : pos_o[i];
    } else {
      a = acc_q[i - n_elig_o];
      p = pos_q[i - n_elig_o];
    }
  }
};

// Score -> 64-bit composite key (S desc, position asc; R22).
__device__ __forceinline__ uint64_t score_key(float S, int pos) {
  uint32_t b = __float_as_uint(S);
  b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);  // order-preserving map of fp32
  if (S == 0.f) b = 0x80000000u;                    // -0 == +0
  return ((uint64_t)b << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)pos);
}
__device__ __forceinline__ float hh_score(float2 acc, float invN, float gamma) {
  float mu = __fmul_rn(acc.x, invN);
  float var = fmaxf(__fsub_rn(__fmul_rn(acc.y, invN), __fmul_rn(mu, mu)), 0.f);
  return __fadd_rn(mu, __fmul_rn(gamma, var));
}
__device__ __forceinline__ RowView make_rowview(const Geom& g, const TailorJob& jb, uint8_t* meta,
                                               const float2* acc_pf) {
  RowView rv;
  if (jb.old_slot < 0) {
    rv.acc_o = acc_pf + (int64_t)jb.unit * g.max_pos;
    rv.pos_o = nullptr;
    rv.acc_q = nullptr;
    rv.pos_q = nullptr;
    rv.sp_o = rv.sp_q = nullptr;
    rv.prefill = true;
  } else {
    SlotMeta sm = slot_meta(meta, g, jb.old_slot);
    rv.acc_o = sm.acc_o;
    rv.acc_q = sm.acc_q;
    rv.pos_o = sm.pos_o;
    rv.pos_q = sm.pos_q;
    rv.sp_o = sm.sp_o;
    rv.sp_q = sm.sp_q;
    rv.prefill = false;
  }
  rv.n_elig_o = jb.n_o_old - jb.n_win_old;
  rv.n_q = jb.n_q_old;
  return rv;
}

// Layer-shared states: per group of H_kv consecutive jobs (one (sequence, layer)), the sum
// over its KV heads of the Eq. 9 score of each eligible row; checks that the heads' rows
// hold the same positions.
__global__ void __launch_bounds__(256) tailor_scores_kernel(Geom g, TailorJobs jobs, uint8_t* meta,
                                                            const float2* __restrict__ acc_pf,
                                                            float* __restrict__ out, int64_t stride,
                                                            int32_t* err) {
  griddep_wait();
  const int k0 = blockIdx.y * g.Hkv;
  const TailorJob& j0 = jobs.j[k0];
  const int n_e = j0.n_o_old - j0.n_win_old + j0.n_q_old;
  const float invN = j0.n_rows > 0 ? 1.0f / (float)(g.G * j0.n_rows) : 0.f;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_e) return;
  float sum = 0.f;
  int p0 = 0;
  for (int h = 0; h < g.Hkv; ++h) {
    const RowView rv = make_rowview(g, jobs.j[k0 + h], meta, acc_pf);
    float2 a;
    int p;
    rv.get(i, a, p);
    if (h == 0) p0 = p;
    else if (p != p0) atomicOr(err, kErrIntegrity);
    sum = __fadd_rn(sum, hh_score(a, invN, g.gamma));
  }
  out[(int64_t)blockIdx.y * stride + i] = sum;
}

void launch_tailor_scores(const Geom& g, const TailorJobs& jobs, int n_jobs, int max_ne, uint8_t* meta,
                          const float2* acc_pf, float* out, int64_t stride, int32_t* err, cudaStream_t s) {
  dim3 grid((max(max_ne, 1) + 255) / 256, n_jobs / g.Hkv);
  launch_pdl(tailor_scores_kernel, grid, dim3(256), 0, s, g, jobs, meta, acc_pf, out, stride, err);
}

__global__ void __launch_bounds__(1024) tailor_select_kernel(Geom g, TailorJobs jobs, uint8_t* meta,
                                                             const float2* __restrict__ acc_pf,
                                                             int8_t* __restrict__ st_scratch, int st_stride,
                                                             const float* __restrict__ sscore,
                                                             const float* __restrict__ ext, int64_t ext_stride,
                                                             int ext_heads, float* __restrict__ ssm) {
  __shared__ uint32_t hist[2][256];
  __shared__ uint64_t sh_prefix[2];
  __shared__ uint32_t sh_rem[2];
  griddep_wait();
  const TailorJob jb = jobs.j[blockIdx.x];
  int8_t* st = st_scratch + (int64_t)blockIdx.x * st_stride;  // [old O rows | old Q rows]
  const int n_elig_o = jb.n_o_old - jb.n_win_old;
  const int n_e = n_elig_o + jb.n_q_old;
  const int q_off = st_stride - g.cap_q;

  // window rows are always Original (A13); identity jobs keep every row Original
  for (int i = threadIdx.x; i < jb.n_o_old; i += blockDim.x)
    if (i >= n_elig_o || jb.identity) st[i] = 1;
  if (jb.identity) return;

  const RowView rv = make_rowview(g, jb, meta, acc_pf);
  const float invN = jb.n_rows > 0 ? 1.0f / (float)(g.G * jb.n_rows) : 0.f;
  const float gamma = g.gamma;
  // layer-shared states (NEXT-3): the score is the mean over the layer's KV
  // heads — the sum per row comes from tailor_scores_kernel (this cache's heads; the
  // layer's jobs are consecutive and waves are aligned to layers) or from the sums
  // exchanged across KV-head shards
  const float* ssum = nullptr;
  float nheads = (float)g.Hkv;
  if (g.share) {
    if (jb.ext_row >= 0) {
      ssum = ext + (int64_t)jb.ext_row * ext_stride;
      nheads = (float)ext_heads;
    } else {
      ssum = sscore + (int64_t)(blockIdx.x / g.Hkv) * st_stride;
    }
  }
  // R34 (NEXT-4): tokens the previous tailor scored and kept (position <= prev_thr) rank by
  // S~ = λ S~_prev + (1 - λ) S; the others by S
  const float lam = g.smooth;
  auto score_of = [&](int i, int& p) -> float {
    float2 a;
    rv.get(i, a, p);
    float S = g.share ? __fdiv_rn(__ldcg(ssum + i), nheads) : hh_score(a, invN, gamma);
    if (lam > 0.f && p <= jb.prev_thr) S = __fadd_rn(__fmul_rn(lam, rv.sp(i)), __fmul_rn(__fsub_rn(1.f, lam), S));
    return S;
  };
  auto key_of = [&](int i) -> uint64_t {
    if (lam == 0.f && !g.share) {
      float2 a;
      int p;
      rv.get(i, a, p);
      return hh_key(a, p, invN, gamma);
    }
    int p;
    const float S = score_of(i, p);
    return score_key(S, p);
  };

  const uint32_t kk[2] = {(uint32_t)jb.n_oe, (uint32_t)(jb.n_oe + jb.n_q_new)};
  if (threadIdx.x < 2) {
    sh_prefix[threadIdx.x] = 0;
    sh_rem[threadIdx.x] = kk[threadIdx.x];
  }
  __shared__ uint64_t sh_mask[2];
  __shared__ int sh_done[2];
  __shared__ uint32_t wsum[2][8];
  if (threadIdx.x < 2) {
    sh_mask[threadIdx.x] = 0;
    sh_done[threadIdx.x] = kk[threadIdx.x] == 0;
  }
  __syncthreads();
  for (int pass = 7; pass >= 0 && !(sh_done[0] && sh_done[1]); --pass) {
    for (int i = threadIdx.x; i < 512; i += blockDim.x) (&hist[0][0])[i] = 0;
    const uint64_t p0 = sh_prefix[0], p1 = sh_prefix[1], m0 = sh_mask[0], m1 = sh_mask[1];
    const bool d0 = sh_done[0], d1 = sh_done[1];
    // read before the digit search below rewrites it (one writer per selection and pass)
    const uint32_t rem_in[2] = {sh_rem[0], sh_rem[1]};
    __syncthreads();
    const int sh = pass * 8;
#pragma unroll 4
    for (int i = threadIdx.x; i < n_e; i += blockDim.x) {
      const uint64_t key = key_of(i);
      const uint32_t dg = (uint32_t)(key >> sh) & 0xFFu;
      if (!d0 && (key & m0) == p0) atomicAdd(&hist[0][dg], 1u);
      if (!d1 && (key & m1) == p1) atomicAdd(&hist[1][dg], 1u);
    }
    __syncthreads();
    // parallel digit search: threads [256 s, 256 s + 256) scan selection s's bins from
    // the top digit down (inclusive prefix sums via warp shuffles)
    const int sel = threadIdx.x >> 8, bi = threadIdx.x & 255, lw = (threadIdx.x >> 5) & 7, ln = threadIdx.x & 31;
    uint32_t h = 0, incl = 0;
    if (sel < 2) {
      h = hist[sel][255 - bi];
      incl = h;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (ln >= o) incl += v;
      }
      if (ln == 31) wsum[sel][lw] = incl;
    }
    __syncthreads();
    if (sel < 2 && !(sel ? d1 : d0)) {
      for (int w = 0; w < lw; ++w) incl += wsum[sel][w];
      const uint32_t rem = rem_in[sel], excl = incl - h;
      if (h > 0 && excl < rem && rem <= incl) {
        const int dgt = 255 - bi;
        sh_prefix[sel] |= ((uint64_t)dgt) << sh;
        sh_mask[sel] |= 0xFFull << sh;
        if (rem - excl == h) sh_done[sel] = 1;  // the whole bucket is taken: threshold found
        else sh_rem[sel] = rem - excl;
      }
    }
    __syncthreads();
  }
  // thresholds: k-th largest key (k == 0 -> nothing selected)
  const uint64_t T1 = kk[0] == 0 ? ~0ull : sh_prefix[0];
  const uint64_t T2 = kk[1] == 0 ? ~0ull : sh_prefix[1];
  float* sso = ssm ? ssm + (int64_t)blockIdx.x * st_stride : nullptr;
  for (int i = threadIdx.x; i < n_e; i += blockDim.x) {
    uint64_t key;
    if (sso) {  // the move kernel stores every kept row's smoothed score in the new slot
      int p;
      const float S = score_of(i, p);
      key = score_key(S, p);
      sso[i < n_elig_o ? i : q_off + (i - n_elig_o)] = S;
    } else {
      key = key_of(i);
    }
    int8_t s = key >= T1 ? 1 : (key >= T2 ? 2 : 3);
    if (i < n_elig_o)
      st[i] = s;
    else
      st[q_off + (i - n_elig_o)] = s;
  }
}

// Block-wide exclusive scan of two counters.
__device__ int2 block_exscan2(int2 v, int2* sh, int2* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int2 x = v;
  for (int off = 1; off < 32; off <<= 1) {
    int a = __shfl_up_sync(0xffffffffu, x.x, off);
    int b = __shfl_up_sync(0xffffffffu, x.y, off);
    if (lane >= off) {
      x.x += a;
      x.y += b;
    }
  }
  __syncthreads();
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    int2 run = make_int2(0, 0);
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      int2 t = sh[i];
      sh[i] = run;
      run.x += t.x;
      run.y += t.y;
    }
    sh[32] = run;
  }
  __syncthreads();
  int2 base = sh[w];
  *total = sh[32];
  return make_int2(base.x + x.x - v.x, base.y + x.y - v.y);
}

__global__ void __launch_bounds__(1024) tailor_scan_kernel(Geom g, TailorJobs jobs, UnitDesc* desc,
                                                           const int8_t* __restrict__ st_scratch, int st_stride,
                                                           int32_t* __restrict__ src_scratch, int src_stride,
                                                           int32_t* err) {
  __shared__ int2 sh[33];
  griddep_wait();
  const TailorJob jb = jobs.j[blockIdx.x];
  const int8_t* st = st_scratch + (int64_t)blockIdx.x * st_stride;
  const int q_off = st_stride - g.cap_q;
  int32_t* src_o = src_scratch + (int64_t)blockIdx.x * src_stride;
  int32_t* src_q = src_o + g.cap_o;
  const int n_elig_o = jb.n_o_old - jb.n_win_old;
  const int kindO = jb.old_slot < 0 ? kSrcInput : kSrcOldO;

  // S1: old eligible O rows; S2: old Q rows.
  int2 tot1, tot2;
  {
    const int n = n_elig_o;
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int a = threadIdx.x * per, b = min(a + per, n);
    int2 c = make_int2(0, 0);
    for (int i = a; i < b; ++i) {
      c.x += st[i] == 1;
      c.y += st[i] == 2;
    }
    int2 ex = block_exscan2(c, sh, &tot1);
    // placed after the S2 counts are known: compute S2 totals first
    __syncthreads();
    const int n2 = jb.n_q_old;
    const int per2 = (n2 + blockDim.x - 1) / blockDim.x;
    const int a2 = threadIdx.x * per2, b2 = min(a2 + per2, n2);
    int2 c2 = make_int2(0, 0);
    for (int i = a2; i < b2; ++i) {
      c2.x += st[q_off + i] == 1;
      c2.y += st[q_off + i] == 2;
    }
    int2 ex2 = block_exscan2(c2, sh, &tot2);
    // S1 rows: O -> new O index ex.x + ...; Q -> new Q index tot2.y + ex.y + ...
    int o = ex.x, q = tot2.y + ex.y;
    for (int i = a; i < b; ++i) {
      int8_t s = st[i];
      if (s == 1) src_o[o++] = (kindO << 28) | i;
      else if (s == 2) src_q[q++] = (kindO << 28) | i;
    }
    // S2 rows: O -> tot1.x + ex2.x + ...; Q -> ex2.y + ...
    int o2 = tot1.x + ex2.x, q2 = ex2.y;
    for (int i = a2; i < b2; ++i) {
      int8_t s = st[q_off + i];
      if (s == 1) src_o[o2++] = (kSrcOldQ << 28) | i;
      else if (s == 2) src_q[q2++] = (kSrcOldQ << 28) | i;
    }
  }
  // window rows (old O rows [n_elig_o, n_o_old)) close the new O segment in order
  const int n_oe_got = tot1.x + tot2.x;
  for (int i = threadIdx.x; i < jb.n_win_old; i += blockDim.x)
    src_o[n_oe_got + i] = (kindO << 28) | (n_elig_o + i);
  if (threadIdx.x == 0) {
    const int n_q_got = tot1.y + tot2.y;
    if (n_oe_got != jb.n_oe || n_q_got != jb.n_q_new) atomicOr(err, kErrIntegrity);
    UnitDesc dd;
    dd.slot = jb.new_slot;
    dd.n_o = jb.n_oe + jb.n_win_old;
    dd.n_q = jb.n_q_new;
    dd.t_next = jb.t_next;
    dd.trig = jb.trig_new;
    dd.acc0 = jb.acc0_new;
    dd.pad1 = dd.pad2 = 0;
    desc[jb.unit] = dd;
  }
}

// ---------------------------------------------------------------------------------
// Move: build destination tiles.
// ---------------------------------------------------------------------------------
struct SrcRef {
  const uint8_t* old_slot;
  const uint16_t* pk;  // prefill rows of this unit [P][d]
  const uint16_t* pv;
};

__device__ __forceinline__ uint32_t read_code(const Geom& g, const uint8_t* tile, int j, int x, bool isv) {
  int byte, shift;
  if (isv) q_v_loc(g, j, x, &byte, &shift);
  else q_k_loc(g, j, x, &byte, &shift);
  uint32_t w = tile[byte];
  if (g.bits == 8) return w;
  return (w >> shift) & ((1u << g.bits) - 1u);
}

// Codes are first collected one per byte in cbuf[isv][token][dim] (shared memory), then
// packed into the tile layout by pack_codes (no read-modify-write on shared words).
__device__ __forceinline__ void write_code(const Geom& g, uint8_t* cbuf, int j, int x, bool isv, uint32_t c) {
  cbuf[((isv ? kTile : 0) + j) * g.d + x] = (uint8_t)c;
}

__device__ __forceinline__ void pack_codes(const Geom& g, uint8_t* tile, const uint8_t* cbuf, int tbytes) {
  const int per = 8 / g.bits;
  for (int B = threadIdx.x; B < tbytes; B += blockDim.x) {
    int j, x, isv;
    if (!q_code_slot(g, B, 0, &j, &x, &isv)) continue;  // scale / zero bytes
    uint32_t v = 0;
    for (int s = 0; s < per; ++s) {
      q_code_slot(g, B, s, &j, &x, &isv);
      v |= (uint32_t)cbuf[((isv ? kTile : 0) + j) * g.d + x] << (s * g.bits);
    }
    tile[B] = (uint8_t)v;
  }
}

__device__ __forceinline__ float read_o(const Geom& g, const uint8_t* tile, int j, int x, bool isv) {
  int off = isv ? o_v_off(g, j, x) : o_k_off(g, j, x);
  return bf16_to_f(*(const uint16_t*)(tile + off));
}

template <int VPL, int DC>  // values per lane = ceil(d / 32); DC = compile-time head dim (0: runtime)
__global__ void __launch_bounds__(256) tailor_move_kernel(Geom g_in, TailorJobs jobs, int n_jobs, uint8_t* slots,
                                                          uint8_t* meta, const uint16_t* __restrict__ pk,
                                                          const uint16_t* __restrict__ pv, int P,
                                                          const int32_t* __restrict__ src_scratch, int src_stride,
                                                          const float* __restrict__ ssm, int32_t* err) {
  extern __shared__ __align__(16) uint8_t tile[];
  griddep_wait();
  Geom g = g_in;
  if (DC) g.d = DC;  // lets the tile-layout index maps fold their divisions into shifts
  const int jix = job_of_tile(jobs, n_jobs, blockIdx.x);
  const TailorJob jb = jobs.j[jix];
  const int n_o_new = jb.n_oe + jb.n_win_old;
  const int tiles_o = (n_o_new + kTile - 1) / kTile;
  int tid = blockIdx.x - jobs.tile_off[jix];
  const bool dstQ = tid >= tiles_o;
  if (dstQ) tid -= tiles_o;
  const int tbytes = dstQ ? g.tile_q : g.tile_o;
  uint8_t* cbuf = tile + ((tbytes + 15) & ~15);  // [2][32][d] code bytes (Quantized tiles)
  const int zbytes = dstQ ? ((tbytes + 15) & ~15) + 2 * kTile * g.d : tbytes;
  for (int i = threadIdx.x * 4; i < zbytes; i += blockDim.x * 4) *(uint32_t*)(tile + i) = 0u;
  __syncthreads();

  const int32_t* src = src_scratch + (int64_t)jix * src_stride + (dstQ ? g.cap_o : 0);
  uint8_t* nslot = slots + (int64_t)jb.new_slot * g.slot_bytes;
  const uint8_t* oslot = jb.old_slot >= 0 ? slots + (int64_t)jb.old_slot * g.slot_bytes : nullptr;
  SlotMeta nm = slot_meta(meta, g, jb.new_slot);
  SlotMeta om;
  if (jb.old_slot >= 0) om = slot_meta(meta, g, jb.old_slot);
  const uint16_t* upk = pk ? pk + (int64_t)jb.unit * P * g.d : nullptr;
  const uint16_t* upv = pv ? pv + (int64_t)jb.unit * P * g.d : nullptr;
  const int n_new = dstQ ? jb.n_q_new : n_o_new;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qmaxv = (1 << (g.bits - 1)) - 1;
  const int off = g.mode == ARKV_QUANT_SYM ? (1 << (g.bits - 1)) : 0;

  int gidx[VPL];  // quantization group of each of this lane's dims
#pragma unroll
  for (int t = 0; t < VPL; ++t) gidx[t] = (lane + 32 * t) / g.g;
  for (int j = warp; j < kTile; j += blockDim.x >> 5) {
    const int row = tid * kTile + j;
    if (row >= n_new) continue;
    const int32_t sref = src[row];
    const int kind = sref >> 28, orow = sref & 0x0FFFFFFF;
    int pos;
    if (kind == kSrcInput) pos = orow;
    else if (kind == kSrcOldO) pos = om.pos_o[orow];
    else pos = om.pos_q[orow];
    if (lane == 0) {
      if (dstQ) {
        nm.pos_q[row] = pos;
        nm.acc_q[row] = make_float2(0.f, 0.f);
      } else {
        nm.pos_o[row] = pos;
        nm.acc_o[row] = make_float2(0.f, 0.f);
      }
      if (ssm) {  // R34: the row's smoothed score at this tailor (read only if it was eligible)
        const int st_stride = max(g.max_pos, g.cap_o) + g.cap_q;
        const float sc = ssm[(int64_t)jix * st_stride + (kind == kSrcOldQ ? st_stride - g.cap_q + orow : orow)];
        (dstQ ? nm.sp_q : nm.sp_o)[row] = sc;
      }
    }
    const uint8_t* qt = nullptr;
    const uint8_t* ot = nullptr;
    int oj = orow & 31;
    if (kind == kSrcOldQ) qt = q_tile_ptr((uint8_t*)oslot, g, orow >> 5);
    if (kind == kSrcOldO) ot = o_tile_ptr((uint8_t*)oslot, g, orow >> 5);

    if (kind == kSrcOldQ && dstQ) {
      // Q -> Q: copy codes and scales (R25)
      for (int x = lane; x < g.d; x += 32) {
        write_code(g, cbuf, j, x, false, read_code(g, qt, oj, x, false));
        write_code(g, cbuf, j, x, true, read_code(g, qt, oj, x, true));
      }
      for (int w = lane; w < 4 * g.ng; w += 32) {
        int which = w / g.ng, grp = w % g.ng;
        *(float*)(tile + q_sc_off(g, j, which, grp)) = *(const float*)(qt + q_sc_off(g, oj, which, grp));
      }
      continue;
    }
    // materialise bf16 values (K and V) for this token
    float kvv[2][VPL];
#pragma unroll
    for (int t = 0; t < VPL; ++t) {
      int x = lane + 32 * t;
      float kx = 0.f, vx = 0.f;
      if (x < g.d) {
        if (kind == kSrcInput) {
          kx = bf16_to_f(upk[(int64_t)orow * g.d + x]);
          vx = bf16_to_f(upv[(int64_t)orow * g.d + x]);
          if (!isfinite(kx) || !isfinite(vx)) atomicOr(err, kErrNonFinite);
        } else if (kind == kSrcOldO) {
          kx = read_o(g, ot, oj, x, false);
          vx = read_o(g, ot, oj, x, true);
        } else {
          // Q -> O promotion (R24): bf16_rne(f32(f32(code*s) + z))
          int grp = x / g.g;
          float ks = *(const float*)(qt + q_sc_off(g, oj, 0, grp));
          float kz = *(const float*)(qt + q_sc_off(g, oj, 1, grp));
          float vs = *(const float*)(qt + q_sc_off(g, oj, 2, grp));
          float vz = *(const float*)(qt + q_sc_off(g, oj, 3, grp));
          const float ck = code_value(g, read_code(g, qt, oj, x, false));
          const float cv = code_value(g, read_code(g, qt, oj, x, true));
          kx = bf16_to_f(f_to_bf16_rne(__fadd_rn(__fmul_rn(ck, ks), kz)));
          vx = bf16_to_f(f_to_bf16_rne(__fadd_rn(__fmul_rn(cv, vs), vz)));
        }
      }
      kvv[0][t] = kx;
      kvv[1][t] = vx;
    }
    if (!dstQ) {
#pragma unroll
      for (int t = 0; t < VPL; ++t) {
        int x = lane + 32 * t;
        if (x < g.d) {
          *(uint16_t*)(tile + o_k_off(g, j, x)) = (uint16_t)(__float_as_uint(kvv[0][t]) >> 16);
          *(uint16_t*)(tile + o_v_off(g, j, x)) = (uint16_t)(__float_as_uint(kvv[1][t]) >> 16);
        }
      }
      continue;
    }
    // O -> Q: group quantization (R23), fp32 op order identical to the oracle
    for (int kv = 0; kv < 2; ++kv) {
      for (int grp = 0; grp < g.ng; ++grp) {
        float mn = INFINITY, mx = -INFINITY, am = 0.f;
#pragma unroll
        for (int t = 0; t < VPL; ++t) {
          int x = lane + 32 * t;
          if (x < g.d && gidx[t] == grp) {
            float v = kvv[kv][t];
            mn = fminf(mn, v);
            mx = fmaxf(mx, v);
            am = fmaxf(am, fabsf(v));
          }
        }
        for (int o = 16; o > 0; o >>= 1) {
          mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
          am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
        }
        float s, z;
        bool flat;
        if (g.mode == ARKV_QUANT_FP8) {  // NEXT-2: s = f32(max|x| / 448), z = 0
          flat = am == 0.f;
          s = flat ? 1.f : __fdiv_rn(am, 448.f);
          z = 0.f;
        } else if (g.mode == ARKV_QUANT_SYM) {
          flat = am == 0.f;
          s = flat ? 1.f : __fdiv_rn(am, (float)qmaxv);
          z = 0.f;
        } else {
          flat = mx == mn;
          s = flat ? 1.f : __fdiv_rn(__fsub_rn(mx, mn), (float)((1 << g.bits) - 1));
          z = mn;
        }
#pragma unroll
        for (int t = 0; t < VPL; ++t) {
          int x = lane + 32 * t;
          if (x < g.d && gidx[t] == grp) {
            int c;
            if (flat) {
              c = 0;
            } else if (g.mode == ARKV_QUANT_FP8) {  // e4m3 byte: RNE, satfinite
              c = (int)__nv_cvt_float_to_fp8(__fdiv_rn(kvv[kv][t], s), __NV_SATFINITE, __NV_E4M3);
            } else if (g.mode == ARKV_QUANT_SYM) {
              c = __float2int_rn(__fdiv_rn(kvv[kv][t], s));
              c = max(-qmaxv, min(qmaxv, c));
            } else {
              c = __float2int_rn(__fdiv_rn(__fsub_rn(kvv[kv][t], mn), s));
              c = max(0, min((1 << g.bits) - 1, c));
            }
            write_code(g, cbuf, j, x, kv == 1, (uint32_t)(c + off));
          }
        }
        if (lane == 0) {
          *(float*)(tile + q_sc_off(g, j, kv * 2 + 0, grp)) = s;
          *(float*)(tile + q_sc_off(g, j, kv * 2 + 1, grp)) = z;
        }
      }
    }
  }
  __syncthreads();
  if (dstQ) {
    pack_codes(g, tile, cbuf, tbytes);
    __syncthreads();
  }
  uint8_t* dst = dstQ ? q_tile_ptr(nslot, g, tid) : o_tile_ptr(nslot, g, tid);
  for (int i = threadIdx.x * 16; i < tbytes; i += blockDim.x * 16) *(uint4*)(dst + i) = *(const uint4*)(tile + i);
}

// ---------------------------------------------------------------------------------
// Move, FRAG layout / d = 128 / 4-bit (the paper's shapes): the 32 rows of a destination
// tile are first materialised row-major in shared memory (16-byte loads for prompt rows
// and for the K block of old Original tiles, whose 16-byte quads are 8 consecutive dims
// of one token), quantised there when the tile is Quantized, and the tile is then
// written straight to HBM one 16-byte quad per thread — each quad's contents come from
// the FRAG maps of common.cuh specialised to d = 128 (no per-element layout arithmetic
// on the store side).
// ---------------------------------------------------------------------------------
constexpr int kMoveTilesPerCta = 4;  // tailor_move_frag_kernel: destination tiles per CTA
namespace mvf {
constexpr int D = 128;
constexpr int kRowH = D + 8;    // staged row stride in bf16 (pad: conflict-free transposed reads)
constexpr int kRowC = D + 8;    // code row stride in bytes (8-byte aligned rows)
struct Smem {
  uint16_t stage[2][kTile][kRowH];  // K, V rows (bf16 bits)
  uint8_t code[2][kTile][kRowC];    // K, V codes (Quantized tiles)
  float4 sc[kTile][D / 16];         // per row and group: k_scale, k_zero, v_scale, v_zero (ng <= 8)
};
}  // namespace mvf

template <int NG>
__global__ void __launch_bounds__(256, 6) tailor_move_frag_kernel(Geom g_in, TailorJobs jobs, uint8_t* slots,
                                                               uint8_t* meta, const uint16_t* __restrict__ pk,
                                                               const uint16_t* __restrict__ pv, int P,
                                                               const int32_t* __restrict__ src_scratch,
                                                               int src_stride, const float* __restrict__ ssm,
                                                               int32_t* err, int n_jobs) {
  using namespace mvf;
  __shared__ __align__(16) Smem sm;
  griddep_wait();
  Geom g = g_in;
  g.d = D;
  g.bits = 4;
  g.ng = NG;
  g.layout = ARKV_LAYOUT_FRAG;
  constexpr int GS = D / NG;  // group size
  // this CTA's destination tiles: kMoveTilesPerCta consecutive tiles of one job (the
  // per-CTA setup amortised over several tiles; ncu: it was ~25 % of the kernel's
  // instructions with one tile per CTA)
  const int jix = job_of_tile(jobs, n_jobs, blockIdx.x);
  const TailorJob jb = jobs.j[jix];
  const int n_o_new = jb.n_oe + jb.n_win_old;
  const int tiles_o = (n_o_new + kTile - 1) / kTile;
  const int tiles_all = tiles_o + (jb.n_q_new + kTile - 1) / kTile;
  const int t_first = (blockIdx.x - jobs.tile_off[jix]) * kMoveTilesPerCta;
  uint8_t* nslot = slots + (int64_t)jb.new_slot * g.slot_bytes;
  const uint8_t* oslot = jb.old_slot >= 0 ? slots + (int64_t)jb.old_slot * g.slot_bytes : nullptr;
  SlotMeta nm = slot_meta(meta, g, jb.new_slot);
  SlotMeta om;
  if (jb.old_slot >= 0) om = slot_meta(meta, g, jb.old_slot);
  const uint16_t* upk = pk ? pk + (int64_t)jb.unit * P * D : nullptr;
  const uint16_t* upv = pv ? pv + (int64_t)jb.unit * P * D : nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int off = g.mode == ARKV_QUANT_SYM ? 8 : 0;
  uint32_t nonfinite_bits = 0u;
  for (int rep = 0; rep < kMoveTilesPerCta; ++rep) {
  int tid = t_first + rep;
  if (tid >= tiles_all) break;
  if (rep > 0) __syncthreads();  // the previous tile's phase 2 is done with the staging buffers
  const bool dstQ = tid >= tiles_o;
  if (dstQ) tid -= tiles_o;
  const int32_t* src = src_scratch + (int64_t)jix * src_stride + (dstQ ? g.cap_o : 0);
  const int n_new = dstQ ? jb.n_q_new : n_o_new;

  // ---- phase 0: the source reference and position of the warp's kTile / 8 rows in two
  // batched rounds (lane r < kTile / 8 handles row warp + 8 r) instead of two dependent
  // loads per row inside the row loop ----
  constexpr int RPW = kTile / 8;
  int my_sref = 0;
  {
    const int row = tid * kTile + warp + 8 * lane;
    if (lane < RPW && row < n_new) {
      my_sref = src[row];
      const int kind = my_sref >> 28, orow = my_sref & 0x0FFFFFFF;
      const int pos = kind == kSrcInput ? orow : (kind == kSrcOldO ? om.pos_o[orow] : om.pos_q[orow]);
      if (dstQ) {
        nm.pos_q[row] = pos;
        nm.acc_q[row] = make_float2(0.f, 0.f);
      } else {
        nm.pos_o[row] = pos;
        nm.acc_o[row] = make_float2(0.f, 0.f);
      }
      if (ssm) {  // R34: the row's smoothed score at this tailor (read only if it was eligible)
        const int st_stride = max(g.max_pos, g.cap_o) + g.cap_q;
        const float sc = ssm[(int64_t)jix * st_stride + (kind == kSrcOldQ ? st_stride - g.cap_q + orow : orow)];
        (dstQ ? nm.sp_q : nm.sp_o)[row] = sc;
      }
    }
  }
  // ---- phase 1: one warp per row.  The warp's prompt rows (the prefill-end tailor's only
  // source) are first copied into the staging rows with cp.async, all kTile / 8 in flight
  // at once and no registers held (ncu: with one row load in flight per warp, 35 % of the
  // stall samples waited on it; loading them into registers instead measured slower, 57
  // instead of 40 registers) ----
  {
    bool any = false;
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
      const int32_t sref = __shfl_sync(0xffffffffu, my_sref, r);
      const int j = warp + 8 * r;
      if (tid * kTile + j < n_new && (sref >> 28) == kSrcInput) {
        const uint16_t* rowp = (lane < 16 ? upk : upv) + (int64_t)(sref & 0x0FFFFFFF) * D + (lane & 15) * 8;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&sm.stage[lane >> 4][j][(lane & 15) * 8])),
                     "l"(rowp)
                     : "memory");
        any = true;
      }
    }
    if (any) asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
  }
  for (int j = warp, r = 0; j < kTile; j += 8, ++r) {
    const int row = tid * kTile + j;
    const int32_t sref = __shfl_sync(0xffffffffu, my_sref, r);
    if (row >= n_new) {  // rows past the segment: zeros (defined bytes; masked by the readers)
      for (int i = lane; i < 2 * kRowH / 2; i += 32) ((uint32_t*)sm.stage[i / (kRowH / 2)][j])[i % (kRowH / 2)] = 0u;
      if (dstQ) {
        for (int i = lane; i < 2 * kRowC / 4; i += 32) ((uint32_t*)sm.code[i / (kRowC / 4)][j])[i % (kRowC / 4)] = 0u;
        if (lane < NG) sm.sc[j][lane] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      continue;
    }
    const int kind = sref >> 28, orow = sref & 0x0FFFFFFF;
    const int oj = orow & 31;
    if (kind == kSrcOldQ) {
      const uint8_t* qt = q_tile_ptr((uint8_t*)oslot, g, orow >> 5);
      if (dstQ) {  // Q -> Q: keep codes and scales (R25)
        for (int x = lane; x < D; x += 32) {
          sm.code[0][j][x] = (uint8_t)read_code(g, qt, oj, x, false);
          sm.code[1][j][x] = (uint8_t)read_code(g, qt, oj, x, true);
        }
        if (lane < NG) sm.sc[j][lane] = *(const float4*)(qt + q_sc_off(g, oj, 0, lane));
        continue;
      }
      // Q -> O promotion (R24): bf16_rne(f32(f32(code * s) + z))
      for (int x = lane; x < D; x += 32) {
        const float4 s4 = *(const float4*)(qt + q_sc_off(g, oj, 0, x / GS));
        const int ck = (int)read_code(g, qt, oj, x, false) - off;
        const int cv = (int)read_code(g, qt, oj, x, true) - off;
        sm.stage[0][j][x] = f_to_bf16_rne(__fadd_rn(__fmul_rn((float)ck, s4.x), s4.y));
        sm.stage[1][j][x] = f_to_bf16_rne(__fadd_rn(__fmul_rn((float)cv, s4.z), s4.w));
      }
    } else if (kind == kSrcInput) {
      // prompt row: 16 lanes x 16 B of K, 16 lanes x 16 B of V, staged above
      const uint4 pr = *(const uint4*)&sm.stage[lane >> 4][j][(lane & 15) * 8];
      nonfinite_bits |= bf16x8_expmax_bits(pr);  // prompt values entering the cache
    } else {
      // old Original row: K quad (t, q) holds dims 32t + 8q .. +7 of the token (FRAG K map)
      const uint8_t* ot = o_tile_ptr((uint8_t*)oslot, g, orow >> 5);
      const int mth = ((oj >> 4) << 1) | ((oj >> 3) & 1), gg = oj & 7;
      if (lane < 16) {
        const int t = lane >> 2, q = lane & 3;
        *(uint4*)&sm.stage[0][j][32 * t + 8 * q] = *(const uint4*)(ot + ((mth * 4 + q) * 32 + 4 * gg + t) * 16);
      }
      for (int x = lane; x < D; x += 32) sm.stage[1][j][x] = *(const uint16_t*)(ot + o_v_off(g, oj, x));
    }
    if (!dstQ) continue;
    // O -> Q: group quantisation (R23), fp32 op order identical to the oracle.  Lane owns
    // dims 4 lane .. 4 lane + 3 (one group: g >= 4); the lanes of a group reduce together.
    __syncwarp();
    constexpr int LPG = GS / 4;  // lanes per group
    float4 scv;                  // k_scale, k_zero, v_scale, v_zero of this lane's group
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint2 raw = *(const uint2*)&sm.stage[h][j][4 * lane];
      const float xv[4] = {__uint_as_float(raw.x << 16), __uint_as_float(raw.x & 0xFFFF0000u),
                           __uint_as_float(raw.y << 16), __uint_as_float(raw.y & 0xFFFF0000u)};
      const bool sym = g.mode == ARKV_QUANT_SYM;
      float mn = fminf(fminf(xv[0], xv[1]), fminf(xv[2], xv[3]));
      float mx = fmaxf(fmaxf(xv[0], xv[1]), fmaxf(xv[2], xv[3]));
      float am = 0.f;
      if (sym) {
        am = fmaxf(fmaxf(fabsf(xv[0]), fabsf(xv[1])), fmaxf(fabsf(xv[2]), fabsf(xv[3])));
#pragma unroll
        for (int o = 1; o < LPG; o <<= 1) am = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, o));
      } else if (LPG == 32) {
        // one group per warp (g = d, the paper's "per-token scale"): sm_100a's f32 warp
        // reduction instead of five shuffle + min/max rounds (exact: min/max of the values)
        asm("redux.sync.min.f32 %0, %0, 0xffffffff;\n" : "+f"(mn));
        asm("redux.sync.max.f32 %0, %0, 0xffffffff;\n" : "+f"(mx));
      } else {
#pragma unroll
        for (int o = 1; o < LPG; o <<= 1) {
          mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
      }
      const bool flat = sym ? am == 0.f : mx == mn;
      const float s = flat ? 1.f : (sym ? __fdiv_rn(am, 7.f) : __fdiv_rn(__fsub_rn(mx, mn), 15.f));
      const float z = sym ? 0.f : mn;
      // code = rint(f32(f32(x - z) / s)): the quotient through the reciprocal is within
      // 3e-6 of the correctly rounded one (|q| <= 15), so it rounds to the same integer
      // unless it lies within 1e-5 of a half-integer — then the exact division decides
      const float r = __frcp_rn(s);
      const bool tiny = s < 1e-30f;
      uint32_t word = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float num = sym ? xv[e] : __fsub_rn(xv[e], mn);
        const float q = __fmul_rn(num, r);
        const float qr = rintf(q);
        // within 1e-5 of a half-integer <=> more than 0.5 - 1e-5 from the nearest integer
        int c = (tiny || fabsf(q - qr) > 0.5f - 1e-5f) ? __float2int_rn(__fdiv_rn(num, s)) : (int)qr;
        // asymmetric codes need no clamp or flat test: 0 <= x - mn <= mx - mn, so the rounded
        // quotient lies in [0, 15 (1 + 2^-23)] and rounds into [0, 15]; a flat group has
        // x - mn = 0 -> code 0 (s = 1)
        if (sym) c = flat ? 0 : max(-7, min(7, c));
        word |= (uint32_t)((c + off) & 0xFF) << (8 * e);
      }
      *(uint32_t*)&sm.code[h][j][4 * lane] = word;
      if (h == 0) {
        scv.x = s;
        scv.y = z;
      } else {
        scv.z = s;
        scv.w = z;
      }
    }
    if (lane % LPG == 0) sm.sc[j][lane / LPG] = scv;
  }
  __syncthreads();

  // ---- phase 2: 16-byte output quads straight to HBM ----
  if (!dstQ) {
    uint8_t* dst = o_tile_ptr(nslot, g, tid);
    for (int i = threadIdx.x; i < 2 * 512; i += 256) {
      const int qd = i & 511, ql = qd & 31, kq = qd >> 5;  // quad index = (k >> 2) * 32 + lane
      const int gg = ql >> 2, t = ql & 3;
      uint4 v;
      if (i < 512) {
        // K block: kq = mth * 4 + q -> token mth*8 + gg (mth = 2mt + h), dims 32t + 8q .. +7
        const int j = (kq >> 2) * 8 + gg, q = kq & 3;
        v = *(const uint4*)&sm.stage[0][j][32 * t + 8 * q];
      } else {
        // V^T block: kq = mtv * 2 + kc; word (sel, hi) = dim 16mtv + 8sel + gg, tokens
        // 16kc + 8hi + 2t + {0, 1}
        const int mtv = kq >> 1, kc = kq & 1;
        uint32_t w[4];
#pragma unroll
        for (int hi = 0; hi < 2; ++hi)
#pragma unroll
          for (int sel = 0; sel < 2; ++sel) {
            const int x = 16 * mtv + 8 * sel + gg, j0 = 16 * kc + 8 * hi + 2 * t;
            w[sel + 2 * hi] = (uint32_t)sm.stage[1][j0][x] | ((uint32_t)sm.stage[1][j0 + 1][x] << 16);
          }
        v = make_uint4(w[0], w[1], w[2], w[3]);
      }
      *(uint4*)(dst + (i < 512 ? 0 : 64 * D) + (int64_t)qd * 16) = v;
    }
  } else {
    uint8_t* dst = q_tile_ptr(nslot, g, tid);
    // code blocks: 2 x 128 quads (K block 16 d bytes, V block 16 d bytes)
    for (int i = threadIdx.x; i < 256; i += 256) {
      const int isv = i >> 7, qd = i & 127, ql = qd & 31, kq = qd >> 5;
      const int gg = ql >> 2, t = ql & 3;
      uint32_t w[4];
      if (!isv) {
        // K codes: word k = mth * 4 + jp (kq = mth), nibble e = dim 32jp + 8t + e of token mth*8 + gg
        const int j = kq * 8 + gg;
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {
          const uint2 c8 = *(const uint2*)&sm.code[0][j][32 * jp + 8 * t];
          uint32_t a = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) a |= ((c8.x >> (8 * e)) & 0xFu) << (4 * e);
#pragma unroll
          for (int e = 0; e < 4; ++e) a |= ((c8.y >> (8 * e)) & 0xFu) << (4 * (e + 4));
          w[jp] = a;
        }
      } else {
        // V codes: word k = mtv * 2 + sel (kq = mtv), dim 16mtv + 8sel + gg; nibble e = 2kc +
        // hi + 4u holds token 16kc + 8hi + 2t + u
#pragma unroll
        for (int wi = 0; wi < 4; ++wi) {
          const int k = kq * 4 + wi, mtv = k >> 1, sel = k & 1;
          const int x = 16 * mtv + 8 * sel + gg;
          uint32_t a = 0;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int kc = (e >> 1) & 1, hi = e & 1, u = e >> 2;
            a |= ((uint32_t)sm.code[1][16 * kc + 8 * hi + 2 * t + u][x] & 0xFu) << (4 * e);
          }
          w[wi] = a;
        }
      }
      *(uint4*)(dst + isv * 16 * D + (int64_t)qd * 16) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    // scales: [row][group] quads after the codes
    for (int i = threadIdx.x; i < kTile * NG; i += 256)
      *(float4*)(dst + 32 * D + i * 16) = sm.sc[i / NG][i % NG];
  }
  }  // rep
  if (nonfinite_bits) atomicOr(err, kErrNonFinite);
}

int launch_tailor(const Geom& g, const TailorJobs& jobs, int n_jobs, int max_tiles, uint8_t* slots, uint8_t* meta,
                  UnitDesc* desc, const uint16_t* pk, const uint16_t* pv, int P, const float2* acc_pf,
                  int8_t* st_scratch, int32_t* src_scratch, const SharedScores& shs, int32_t* err, cudaStream_t s) {
  const int st_stride = max(g.max_pos, g.cap_o) + g.cap_q;
  const int src_stride = g.cap_o + g.cap_q;
  int extra = 0;
  if (g.share && jobs.j[0].ext_row < 0) {  // local heads: one score pass per (sequence, layer)
    int max_ne = 0;
    for (int k = 0; k < n_jobs; ++k)
      max_ne = max(max_ne, jobs.j[k].n_o_old - jobs.j[k].n_win_old + jobs.j[k].n_q_old);
    launch_tailor_scores(g, jobs, n_jobs, max_ne, meta, acc_pf, shs.sscore, st_stride, err, s);
    extra = 1;
  }
  launch_pdl(tailor_select_kernel, dim3(n_jobs), dim3(1024), 0, s, g, jobs, meta, acc_pf, st_scratch, st_stride,
             (const float*)shs.sscore, shs.ext, shs.ext_stride, shs.ext_heads, g.smooth > 0.f ? shs.ssm : nullptr);
  launch_pdl(tailor_scan_kernel, dim3(n_jobs), dim3(1024), 0, s, g, jobs, desc, (const int8_t*)st_scratch, st_stride,
             src_scratch, src_stride, err);
  // a 1-D grid of exactly the jobs' destination tiles (frag: kMoveTilesPerCta per CTA)
  const bool frag = g.layout == ARKV_LAYOUT_FRAG && g.d == mvf::D && g.bits == 4 &&
                    tuning_knob("ARKV_MOVE_GENERIC", 0) == 0;
  const int tpc = frag ? kMoveTilesPerCta : 1;
  TailorJobs mj = jobs;
  mj.tile_off[0] = 0;
  for (int k = 0; k < n_jobs; ++k) {
    const int tiles = (mj.j[k].n_oe + mj.j[k].n_win_old + kTile - 1) / kTile + (mj.j[k].n_q_new + kTile - 1) / kTile;
    mj.tile_off[k + 1] = mj.tile_off[k] + (tiles + tpc - 1) / tpc;
  }
  (void)max_tiles;
  const dim3 grid(std::max(1, mj.tile_off[n_jobs]));
  const float* ssm = g.smooth > 0.f ? shs.ssm : nullptr;
  if (frag) {
    switch (g.ng) {
      case 1: launch_pdl(tailor_move_frag_kernel<1>, grid, dim3(256), 0, s, g, mj, slots, meta, pk, pv, P,
                         (const int32_t*)src_scratch, src_stride, ssm, err, n_jobs); return 3 + extra;
      case 2: launch_pdl(tailor_move_frag_kernel<2>, grid, dim3(256), 0, s, g, mj, slots, meta, pk, pv, P,
                         (const int32_t*)src_scratch, src_stride, ssm, err, n_jobs); return 3 + extra;
      case 4: launch_pdl(tailor_move_frag_kernel<4>, grid, dim3(256), 0, s, g, mj, slots, meta, pk, pv, P,
                         (const int32_t*)src_scratch, src_stride, ssm, err, n_jobs); return 3 + extra;
      case 8: launch_pdl(tailor_move_frag_kernel<8>, grid, dim3(256), 0, s, g, mj, slots, meta, pk, pv, P,
                         (const int32_t*)src_scratch, src_stride, ssm, err, n_jobs); return 3 + extra;
      default: break;
    }
  }
  size_t smem = (size_t)max(g.tile_o, ((g.tile_q + 15) & ~15) + 2 * kTile * g.d);
  const int vpl = (g.d + 31) / 32;
#define MV_LAUNCH(V, DCV)                                                                                         \
  cudaFuncSetAttribute(tailor_move_kernel<V, DCV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
  launch_pdl(tailor_move_kernel<V, DCV>, grid, dim3(256), smem, s, g, mj, n_jobs, slots, meta, pk, pv, P,         \
             (const int32_t*)src_scratch, src_stride, ssm, err);
#define MV_CASE(V)       \
  case V:                \
    MV_LAUNCH(V, 0)      \
    break;
  if (g.d == 128) {
    MV_LAUNCH(4, 128)
    return 3 + extra;
  }
  switch (vpl) {
    MV_CASE(1)
    MV_CASE(2)
    MV_CASE(4)
    MV_CASE(8)
    default:
      return -1;
  }
#undef MV_CASE
#undef MV_LAUNCH
  return 3 + extra;
}

}  // namespace arkv
