// kernels.h — host-side launch wrappers of the ARKV device kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "common.cuh"

namespace arkv {

// Measurement knobs.  The shipped library reads no environment variable: every knob
// returns its measured default.  A/B builds (`ARKV_NVCC_FLAGS=-DARKV_TUNING_KNOBS`) read
// the named variable instead; none of them changes results, only launch shapes.
int tuning_knob(const char* name, int def);

#ifndef ARKV_MAX_JOBS
#define ARKV_MAX_JOBS 256
#endif
constexpr int kMaxJobs = ARKV_MAX_JOBS;  // tailor jobs per launch (kernel-parameter array: 15 KB of the 32 KB limit)

// One unit's tailor (Eq. 10) in a wave: sources -> a fresh slot.
struct TailorJob {
  int32_t unit;       // global unit index (b*L + l)*H_kv + kvh
  int32_t old_slot;   // -1 for the prefill tailor (sources are the prompt rows)
  int32_t new_slot;
  int32_t n_o_old;    // old Original rows (prefill: P)
  int32_t n_q_old;    // old Quantized rows (prefill: 0)
  int32_t n_win_old;  // window rows present in the old rows (prefill W, decode W-1)
  int32_t n_oe;       // eligible tokens kept Original
  int32_t n_q_new;    // tokens kept Quantized
  int32_t trig_new;   // next tailor position
  int32_t acc0_new;   // first HH accumulation position of the next tailor (R19; UnitDesc::acc0)
  int32_t n_rows;     // Eq. 9 window queries of this tailor (prefill W; decode min(W, queries
                      // since the previous tailor or the prompt)): N = G * n_rows samples
  int32_t t_next;     // position of the next appended token
  int32_t identity;   // 1: no selection, every old row stays Original (prefill ingest)
  int32_t ext_row;    // layer-shared states: row of the exchanged score sums (-1: local heads only)
  int32_t prev_thr;   // smoothed scores (R34): rows with position <= prev_thr were scored and kept
                      // by the previous tailor (their smoothed score is in the slot meta); -1: none
};
struct TailorJobs {
  TailorJob j[kMaxJobs];
  int32_t tile_off[kMaxJobs + 1];  // move kernels: first CTA of each job (a 1-D grid of exactly
                                   // the jobs' destination tiles; filled by launch_tailor)
};
// job of destination tile `t` of a move launch (binary search of tile_off)
__device__ __forceinline__ int job_of_tile(const TailorJobs& jobs, int n_jobs, int t) {
  int lo = 0, hi = n_jobs - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (jobs.tile_off[mid] <= t) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Prefill statistics: passes 1-2 + local Eq. 3 column sums; then the
// moments / OQ score from (possibly all-reduced) column sums.  Return launches.
int launch_prefill_begin(const Geom& g, const uint16_t* q_win, const uint16_t* k, int P, float* partials,
                         int n_chunks1, float2* acc_pf, double* colsum, cudaStream_t s);
int launch_prefill_finish(const Geom& g, const double* colsum, int P, double* stats, double* oq, const double* tau,
                          double stat_eps, int32_t* err, cudaStream_t s);

// Tailor of a wave of jobs (D4-D6).
// Layer-shared states (NEXT-3): the scores of a tailor come either from this cache's KV
// heads (sscore, written by launch_tailor_scores inside launch_tailor) or from exchanged sums
// over every shard's heads (ext, ext_stride floats per due (sequence, layer), ext_heads heads).
struct SharedScores {
  float* ssm = nullptr;  // smoothed scores (R34): [job][old O rows | old Q rows], select -> move
  float* sscore = nullptr;
  const float* ext = nullptr;
  int64_t ext_stride = 0;
  int ext_heads = 0;
};
int launch_tailor(const Geom& g, const TailorJobs& jobs, int n_jobs, int max_tiles, uint8_t* slots, uint8_t* meta,
                  UnitDesc* desc, const uint16_t* pk, const uint16_t* pv, int P, const float2* acc_pf,
                  int8_t* st_scratch, int32_t* src_scratch, const SharedScores& shs, int32_t* err, cudaStream_t s);
// Sums over the jobs' KV heads (consecutive groups of H_kv jobs) of the Eq. 9 scores of the
// eligible rows: out[group * stride + i].
void launch_tailor_scores(const Geom& g, const TailorJobs& jobs, int n_jobs, int max_ne, uint8_t* meta,
                          const float2* acc_pf, float* out, int64_t stride, int32_t* err, cudaStream_t s);

struct DecodeArgs {
  Geom g;
  int layer0, n_layers, n_splits, max_splits;
  const uint16_t* q;
  const uint16_t* k;
  const uint16_t* v;
  uint8_t* slots;
  uint8_t* meta;
  UnitDesc* desc;
  float* partials;
  float* logits;
  float* mstat;  // [unit][G][2]: merged max (log2) and 1/sum of the step, for the HH kernel
  int32_t* counters;  // [unit]: split CTAs finished this step (fused combine); reset by the last
  int32_t* nsplit;    // [unit]: this step's split count, written by split 0 of the chunk-list
                      // launch (UnitOrder) and read by the combines; nullptr: every unit n_splits
  int q_group;        // fast kernel: Quantized tiles per bulk copy (0 = as many as fit a stage)
  int interleave;     // fast kernel: interleave Original and Quantized work items
  int fuse_combine;   // fast kernel: the last split CTA of a unit merges the partials
  int prefetch;       // fast kernel: items prefetched into L2 ahead of the shared-memory ring
  int item_order;     // fast kernel: 0 Original tiles first; 1 Quantized groups first on odd
                      // (split + unit) CTAs; 2 Quantized groups first everywhere
  float pscale;       // log2 of the scale of the partials' probabilities (fast int-code kernels:
                      // 24, see k_decode_fast.cu kPvSub; fp8 and generic: 0): HH samples use
                      // 2^(s - M - pscale) / L
  int self_refill;    // split kernel: each consumer warp loads its own next item (no in-order producer)
  int hh_nostore;     // tuning builds only (results wrong): the split kernel skips the HH logit stores
  int l2_hints;       // fast kernels: cache tiles stream with L2 evict_first (HH logits and
                      // accumulators are kept with evict_last either way)
  void* out;
  int out_fp32;
  int32_t* err;
  // persistent decode kernel (decode_persist_kernel / decode_persist_combine)
  int persist;
  float* pparts;     // partial slots (m, l, o) per (CTA, phase, unit in its range, warp); l = 0: unused
  int4* pcta;        // [2][kPlanMaxCtas]: (first unit or -1 if empty, slot base, last unit) of each
                     // CTA's phase range, for the combine
  int32_t* pcover;   // [2][2][n_units]: first / last CTA covering each unit's phase items (-1: none)
};

// Work plan of the persistent decode kernel, passed by value as a kernel
// parameter (no host-to-device copy in the stream).  The step's items form two streams —
// phase 0: every unit's Original tiles (16 KB each); phase 1: every unit's Quantized tiles
// in groups of q_per — and each stream is cut into P equal contiguous ranges, one per CTA,
// so every CTA gets the same bytes of each kind (the kinds cost differently: HBM-bound vs.
// ALU-heavy).  A CTA streams its phase-0 range, then its phase-1 range; the kernel walks
// unit boundaries itself from the descriptors.
constexpr int kPersistConsumers = 3;
constexpr int kPersistSpw = 2;  // ring stages per consumer warp (next item in flight while computing)
constexpr int kPlanMaxCtas = 320;  // 2 CTAs/SM x <= 160 SMs
// partial slots one combine merges (C per covering CTA and phase)
constexpr int kMaxUnitParts = 512;
struct PersistPlan {
  int P;
  // per phase, per CTA: x = unit (index in the call) of its first item, y = that item's
  // index within the unit, z = items in the range, w = first partial slot of the range
  // (C slots per unit from x to ue; a unit in both of a CTA's ranges uses its phase-0 slots)
  int4 cta[2][kPlanMaxCtas];
  int ue[2][kPlanMaxCtas];  // unit of the range's last item
};
// Heavy-hitter accumulation fused into the split combine (D3; R19): the (sequence, layer)
// pairs of a call whose step lies in their HH window, from the host's count schedule (the
// same test as the device's, so no descriptor read races the combine's advance).  Passed
// by value as a kernel parameter.  Blocks [0, n_units) of decode_combine_hh merge the
// split partials; the others each take kRows rows of one (entry, KV head).
constexpr int kMaxHhEntries = 256;
struct HhPlan {
  int n;           // entries
  int n_units;     // units of the call (= combine blocks)
  int n_chunks;    // row chunks of all entries (HH blocks = n_chunks x H_kv)
  int pad_;
  int4 e[kMaxHhEntries];  // x = b * n_layers + li; y = rows (n_o after the append + n_q);
                          // z = bit 0: the window's first step (acc := sample), bits 1..:
                          // the entry's split count this step (0: n_splits); w = n_q
  int coff[kMaxHhEntries + 1];  // first chunk of each entry (its own row count: no empty blocks)
};
// Split-K launch order of the fast decode kernel ("cost-balanced splits").
// The host gives each unit a split count in proportion to its estimated time (Original tiles
// + Quantized tiles weighted by their measured relative cost; in all exactly `waves` CTAs per
// CTA slot) and orders the units by piece cost, longest first (LPT), so the last wave is
// filled by the shortest pieces.  CTA c of the 1-D grid runs split c - pfx[i] of unit perm[i]
// for the i with pfx[i] <= c < pfx[i + 1].  Passed by value as a kernel parameter (kept
// small: a 16 KB per-CTA list measured +7 us of launch latency per step).  n_units = 0: the
// uniform grid (n_splits x units).
constexpr int kMaxOrderUnits = 1024;
struct UnitOrder {
  int n_units;
  int n_ctas;
  uint16_t perm[kMaxOrderUnits];     // unit (index in the call) of each position
  uint16_t pfx[kMaxOrderUnits + 1];  // first CTA of each position
};
struct PlanArgs {
  const UnitOrder* chunks = nullptr;  // split-K fast kernel: cost-balanced launch order, or nullptr
  int32_t* nsplit = nullptr;          // [unit] split counts of a chunk-list launch (workspace)
  const HhPlan* hh = nullptr;         // fused HH plan (split-K fast kernel), or nullptr
  const PersistPlan* plan = nullptr;  // host plan, or nullptr: split-K kernels
  float* pparts = nullptr;
  int4* pcta = nullptr;
  int32_t* pcover = nullptr;
};

// Decode attention (D1, D3, D7) for units [layer0, layer0+n) of all sequences.
int launch_decode(const Geom& g, int layer0, int n_layers, const uint16_t* q, const uint16_t* k, const uint16_t* v,
                  void* out, int out_fp32, uint8_t* slots, uint8_t* meta, UnitDesc* desc, float* partials,
                  float* logits, float* mstat, int32_t* counters, int acc_rows, int n_splits, int max_splits,
                  int fast, int32_t* err, cudaStream_t s, cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr,
                  const PlanArgs& plan = PlanArgs());

}  // namespace arkv

namespace arkv {
// Launch with programmatic stream serialization (PDL): the kernel may begin while the
// previous kernel on the stream drains; it calls griddep_wait() before dependent reads.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Keeps an SM's shared-memory carveout at its maximum for this kernel.  Kernels that run
// between decode launches with a smaller carveout (the combines) left SMs configured so that
// only one 100 KB decode CTA fit until they drained (timeline at configs[1]: 33 of 148 SMs
// with one CTA for the first 40 % of the kernel).
template <typename K>
inline void carveout_max(K kern) {
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
}

// k_decode_fast.cu: true when the tensor-core decode kernel supports this cache.
bool decode_fast_available(const Geom& g);
// k_decode_fast.cu: DecodeArgs::pscale of the fast kernels.
float decode_fast_pscale(const Geom& g);
}  // namespace arkv
