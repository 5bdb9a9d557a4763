// kernels.h — host-side launch wrappers of the ARKV device kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "common.cuh"

namespace arkv {

constexpr int kMaxJobs = 96;  // tailor jobs per launch (kernel-parameter array)

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
  int32_t t_next;     // position of the next appended token
  int32_t identity;   // 1: no selection, every old row stays Original (prefill ingest)
  int32_t pad;
};
struct TailorJobs {
  TailorJob j[kMaxJobs];
};

// Prefill statistics: passes 1-2 + local Eq. 3 column sums; then the
// moments / OQ score from (possibly all-reduced) column sums.  Return launches.
int launch_prefill_begin(const Geom& g, const uint16_t* q_win, const uint16_t* k, int P, float* partials,
                         int n_chunks1, float2* acc_pf, double* colsum, cudaStream_t s);
int launch_prefill_finish(const Geom& g, const double* colsum, int P, double* stats, double* oq, const double* tau,
                          double stat_eps, cudaStream_t s);

// Tailor of a wave of jobs (D4-D6).
int launch_tailor(const Geom& g, const TailorJobs& jobs, int n_jobs, int max_tiles, uint8_t* slots, uint8_t* meta,
                  UnitDesc* desc, const uint16_t* pk, const uint16_t* pv, int P, const float2* acc_pf,
                  int8_t* st_scratch, int32_t* src_scratch, int32_t* err, cudaStream_t s);

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
  int q_group;        // fast kernel: Quantized tiles per bulk copy (0 = as many as fit a stage)
  int interleave;     // fast kernel: interleave Original and Quantized work items
  int fuse_combine;   // fast kernel: the last split CTA of a unit merges the partials
  int producer_mode;  // fast kernel: 0 refill stages in item order, 1 whichever frees first
  void* out;
  int out_fp32;
  int32_t* err;
  // persistent decode kernel (decode_persist_kernel): host-built work plan (PlanView) and
  // one partial per (unit, covering CTA, consumer warp)
  const int32_t* plan;
  int plan_U, plan_P;
  float* pparts;
};

// Work plan of the persistent decode kernel (int32, host-built each step).
// The step's items form two streams — phase 0: every unit's Original tiles (16 KB each);
// phase 1: every unit's Quantized tiles in groups of q_per — and each stream is split into
// P equal contiguous ranges, one per CTA, so every CTA gets the same bytes of each kind
// (the two kinds cost differently: HBM-bound vs. ALU-heavy).  A CTA streams its phase-0
// range, then its phase-1 range.
struct PlanView {
  // per phase f: cta_lo [P + 1] first item of each CTA's range (cta_lo(f)[P] = items);
  // cta_u0 [P] unit (index in the call) of item cta_lo(f)[c]; item_first [U + 1] first item
  // of each unit; cta_first / cta_last [U] CTAs covering the unit's phase-f items
  // (cta_last = cta_first - 1 when it has none).  Then part_base [U + 1]: first partial
  // slot of each unit (C slots per covering CTA, phase 0 first).
  const int32_t* base;
  int U, P, ps;  // ps: ints per phase
  __host__ __device__ PlanView(const int32_t* p, int U_, int P_) : base(p), U(U_), P(P_), ps(2 * P_ + 3 * U_ + 2) {}
  __host__ __device__ const int32_t* cta_lo(int f) const { return base + f * ps; }
  __host__ __device__ const int32_t* cta_u0(int f) const { return base + f * ps + P + 1; }
  __host__ __device__ const int32_t* item_first(int f) const { return base + f * ps + 2 * P + 1; }
  __host__ __device__ const int32_t* cta_first(int f) const { return base + f * ps + 2 * P + U + 2; }
  __host__ __device__ const int32_t* cta_last(int f) const { return base + f * ps + 2 * P + 2 * U + 2; }
  __host__ __device__ const int32_t* part_base() const { return base + 2 * ps; }
};
__host__ __device__ inline int plan_ints(int U, int P) { return 2 * (2 * P + 1 + 3 * U + 1) + U + 1; }
constexpr int kPersistConsumers = 4;
// a unit's partials are listed in shared memory by its combine: the host plan keeps every
// unit within kMaxUnitParts / kPersistConsumers CTAs
constexpr int kMaxUnitParts = 512;
struct PlanArgs {
  const int32_t* plan = nullptr;  // device PlanView ints, or nullptr: split-K kernels
  int U = 0, P = 0;
  float* pparts = nullptr;
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

// k_decode_fast.cu: true when the tensor-core decode kernel supports this cache.
bool decode_fast_available(const Geom& g);
}  // namespace arkv
