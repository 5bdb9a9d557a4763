/*
 * arkv.h — C ABI of the B200-native ARKV decode hot path (libarkv.so).
 *
 * ARKV (arXiv 2603.08727, "P:n" = PAPER.md line n) keeps every cached token of a
 * (sequence, layer, KV head) "unit" in one of three states — Original (bf16),
 * Quantized (low-bit integer codes with an fp32 scale and zero per group) or Evicted
 * (§IV-A).  This library implements the data-parallel hot path:
 *   - arkv_prefill_stats: windowed attention statistics (Eqs. 2-5),
 *     OQ score and ratio (Eqs. 6-8, Alg. 1), prompt ingest and
 *     the prefill-end tailor (Eq. 10);
 *   - arkv_decode_step: append, budgeted top-k O/Q/E re-partition with
 *     quantize-on-demote (Eq. 10, Alg. 1), and decode attention over
 *     O ∪ Q with heavy-hitter accumulation fused in (Eq. 9).
 * Readings of the paper where it is silent or garbled ("R<k>") are listed in
 * DESIGN.md §3.
 *
 * Conventions
 *   - Every call returns arkv_status; no C++ exception crosses the ABI.
 *   - Device pointers are plain CUDA device addresses; host pointers are host
 *     memory.  All device memory is owned by the CALLER (e.g. torch tensors):
 *     the library never allocates device memory.  Size it with arkv_cache_bytes.
 *   - Launches are asynchronous on the caller's stream; a call synchronizes only
 *     where documented ("syncs").  No CUDA call is made at library load, so the
 *     host-only entry points work on a machine without a GPU.
 *   - Argument errors are reported synchronously.  Errors detected on the device
 *     (non-finite inputs, capacity overflow) set a device flag read by arkv_check.
 *   - One writer per cache.  One cache per GPU shard.
 *   - Tensors are dense, row-major, bf16 = raw IEEE bfloat16 bits (uint16).
 *     RoPE, if any, is already applied by the caller.
 */
#ifndef ARKV_H_
#define ARKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ARKV_OK = 0,
  ARKV_ERR_INVALID_ARG = -1, /* null pointer, bad index, wrong size */
  ARKV_ERR_CONFIG = -2,      /* H_q % H_kv, d % g, bits not in {2,4,8}, B <= 2W (R14) */
  ARKV_ERR_SEQUENCE = -3,    /* decode before prefill, prefill twice, position >= max_positions */
  ARKV_ERR_WINDOW = -4,      /* prompt_len < W + 2 and no rho_override (R28) */
  ARKV_ERR_LAYOUT = -5,      /* budget / bit-width differ from the cache's */
  ARKV_ERR_CAPACITY = -6,    /* arena or workspace too small */
  ARKV_ERR_DEVICE = -7,      /* device flag: non-finite input or integrity failure */
  ARKV_ERR_CUDA = -8,        /* a CUDA runtime call failed */
  ARKV_ERR_NO_DEVICE = -9    /* no usable sm_100 device */
} arkv_status;

/* Layout of the tiles in HBM. */
enum { ARKV_LAYOUT_AUTO = 0, ARKV_LAYOUT_PLAIN = 1, ARKV_LAYOUT_FRAG = 2 };
/* Quantization mode (R23).  ARKV_QUANT_FP8 (NEXT-2; the paper's FP8 Q tokens, P:333,
   P:486): quant_bits = 8, each code is an OCP e4m3 byte, per-group fp32 scale
   s = max|x| / 448 (zero slot kept, always 0); code = e4m3_rne_satfinite(f32(x / s)). */
enum { ARKV_QUANT_ASYM = 0, ARKV_QUANT_SYM = 1, ARKV_QUANT_FP8 = 2 };

typedef struct arkv_config {
  int32_t n_layers;      /* L */
  int32_t n_q_heads;     /* H_q */
  int32_t n_kv_heads;    /* H_kv held by this process (G = H_q / H_kv, contiguous groups, R27) */
  int32_t head_dim;      /* d in {16, 32, 64, 128} (else ARKV_ERR_CONFIG) */
  int32_t batch;         /* sequences held by this process */
  int32_t window;        /* W, protected recency window (32 in P:368) */
  int32_t budget_tokens; /* B per (seq, layer, KV head) in bf16-token equivalents;
                            B_bytes = B * 4 * d (Eq. 1 in bytes, R10, R11) */
  int32_t quant_bits;    /* 2 | 4 | 8 (R23) */
  int32_t group_size;    /* g, divides d (0 -> d, "per-token scale") */
  int32_t quant_mode;    /* ARKV_QUANT_ASYM (scale, zero=min) | ARKV_QUANT_SYM | ARKV_QUANT_FP8 */
  int32_t max_positions; /* prompt + decode steps upper bound */
  int32_t max_prompt;    /* largest prompt_len passed to arkv_prefill_stats */
  int32_t layout;        /* ARKV_LAYOUT_* (AUTO: FRAG when d % 32 == 0 and bits == 4) */
  int32_t n_spare_slots; /* tailor staging slots (0 -> batch * n_kv_heads) */
  int32_t max_splits;    /* split-K fan-out cap of the decode kernel (0 -> 64) */
  int32_t decode_kernel; /* 0 auto (tensor-core kernel for FRAG 4-bit d=128), 1 generic, 2 fast split-K,
                           3 fast persistent (range-partitioned) */
  double alpha;          /* slack factor, 0.75 */
  double tau[3];         /* OQ temperatures 7.774, 5.407, 5.528 */
  double gamma;          /* HH variance weight 263.81 */
  double stat_eps;       /* clamp of H, V, K (R6), 1e-30 */
  float sm_scale;        /* softmax scale, 0 -> 1/sqrt(d) (R27) */
  int32_t state_sharing; /* 0: one token-state set per KV head (R20); 1: one per layer, from the
                            Eq. 9 score averaged across the layer's KV heads (NEXT-3;
                            all KV heads of a layer must live in this cache) */
  float smooth;          /* λ of the "smoothed" heavy-hitter scores (Alg. 1; reading R34,
                            NEXT-4): S~ = λ S~(previous tailor) + (1 - λ) S for tokens the previous
                            tailor scored and kept; 0 = off (R21, default); must lie in [0, 1) */
} arkv_config;

typedef struct arkv_cache arkv_cache; /* opaque, host-side; owned by the library */

/* Paper defaults for everything but the shapes (alpha, tau, gamma, W = 32, 4-bit,
   g = d, asymmetric).  Host only. */
arkv_status arkv_config_default(arkv_config* cfg);

/* Validates cfg and returns the device bytes the caller must allocate:
   arena (persistent cache: slots, per-slot metadata, unit descriptors, error flag)
   and workspace (split-K partials, HH logits, tailor and prefill scratch).
   Host only; no CUDA call. */
arkv_status arkv_cache_bytes(const arkv_config* cfg, size_t* arena_bytes, size_t* workspace_bytes);

/* Creates the host-side cache object over caller-owned device buffers (256-byte
   aligned) of at least the sizes above.  Selects the current CUDA device; fails
   with ARKV_ERR_NO_DEVICE unless it is sm_100. */
arkv_status arkv_cache_create(const arkv_config* cfg, void* d_arena, size_t arena_bytes,
                              void* d_workspace, size_t workspace_bytes, arkv_cache** out);
arkv_status arkv_cache_destroy(arkv_cache* cache);

/* Prefill (Alg. 1 prefill phase).
   q_win  [B][L][H_q][W][d] bf16 device: queries of prompt positions P-W .. P-1.
   k, v   [B][L][H_kv][P][d] bf16 device: the prompt's keys/values (P = prompt_len).
   rho_override [B][L] host double or NULL: replaces Eq. 7's ratio (required when
          prompt_len < W + 2, R28; used for cross-implementation parity).
   d_stats [B][L][3] device double or NULL: entropy, variance, kurtosis after clamps
          (Eqs. 3-5, R2-R6).
   d_oq   [B][L] device double or NULL: OQ score q_l (Eq. 6).
   h_rho  [B][L] host double or NULL: the ratio used (Eq. 7, or the override).
   Computes the statistics, ingests the prompt as Original tokens and runs the
   prefill-end tailor when prompt_len > B - W (R14).  Syncs once (rho to host). */
arkv_status arkv_prefill_stats(arkv_cache* cache, const void* q_win, const void* k, const void* v,
                               int32_t prompt_len, const double* rho_override, double* d_stats,
                               double* d_oq, double* h_rho, void* stream);

/* The same prefill in two halves, for runs whose sequences' KV heads are sharded over
   several processes.  arkv_prefill_begin runs the two attention passes and writes the
   local Eq. 3 column sums c[b][l][j] = Σ_{local q heads, window queries} Ã (j < P - W)
   into d_colsum [B][L][max_positions] device double (NULL: internal buffer).  The
   caller sums d_colsum over the ranks that share the sequences (e.g. NCCL all-reduce,
   collective C1) and passes it to arkv_prefill_finish, which computes Eqs. 3-7 from it,
   ingests the prompt and runs the prefill-end tailor (syncs once).  prompt_len must be
   >= W + 2 for begin. */
arkv_status arkv_prefill_begin(arkv_cache* cache, const void* q_win, const void* k, int32_t prompt_len,
                               double* d_colsum, void* stream);
arkv_status arkv_prefill_finish(arkv_cache* cache, const void* k, const void* v, int32_t prompt_len,
                                const double* d_colsum, const double* rho_override, double* d_stats, double* d_oq,
                                double* h_rho, void* stream);

/* One decode step for layers [layer0, layer0 + n_layers) of every sequence.
   q [B][n_layers][H_q][d], k, v [B][n_layers][H_kv][d] bf16 device (the new token of
   each sequence at the layer's next position).  out [B][n_layers][H_q][d] device,
   fp32 if out_fp32 else bf16.  budget_tokens and quant_bits must equal the cache's
   (else ARKV_ERR_LAYOUT).  Per unit: append as Original (D1) -> tailor if the unit
   exceeds B_bytes (R12, R13) -> attention over O ∪ Q (D7) with HH accumulation in
   the W steps before the next tailor (R19).  Updates states, codes, scales, zeros
   and accumulators in place.  Never syncs. */
arkv_status arkv_decode_step(arkv_cache* cache, int32_t layer0, int32_t n_layers, const void* q,
                             const void* k, const void* v, int32_t budget_tokens, int32_t quant_bits,
                             void* out, int32_t out_fp32, void* stream);

/* Host-side, no sync: current counts of a (sequence, layer) (all its KV heads share
   them, R20), its next token position and its next tailor position (R15). */
arkv_status arkv_unit_counts(const arkv_cache* cache, int32_t b, int32_t layer, int32_t* n_o,
                             int32_t* n_q, int32_t* next_pos, int32_t* next_tailor);

/* Export of one unit by position, into caller host buffers sized for n_pos = next_pos
   positions (syncs).  state[n_pos] int8: 0 absent, 1 Original, 2 Quantized, 3 Evicted.
   o_k, o_v [n_pos][d] bf16 bits (valid where state == 1); q_k, q_v [n_pos][d] int16
   unpacked codes (signed in symmetric mode; valid where state == 2); k_scale, k_zero,
   v_scale, v_zero [n_pos][d/g] fp32.  Any pointer may be NULL. */
typedef struct arkv_unit_export {
  int8_t* state;
  uint16_t* o_k;
  uint16_t* o_v;
  int16_t* q_k;
  int16_t* q_v;
  float* k_scale;
  float* k_zero;
  float* v_scale;
  float* v_zero;
  int32_t n_pos;
  int32_t n_o;
  int32_t n_q;
  int32_t pad_;
} arkv_unit_export;
arkv_status arkv_export_unit(arkv_cache* cache, int32_t b, int32_t layer, int32_t kvh,
                             arkv_unit_export* out, void* stream);

/* Syncs the stream and converts the device error flag into a status (and clears it):
   ARKV_ERR_DEVICE when, since the last check,
     - a decode step's q, k or v held a non-finite bf16 value (Inf / NaN);
     - a prompt K/V row entering the cache (kept by the prefill-end tailor, or ingested)
       held one, or a NaN / Inf in q_win or K reached the Eq. 3 column sums or q_l;
     - a slot would overflow (capacity) or a tailor's counts or positions disagreed with
       the host schedule (integrity).
   Evicted prompt V rows are never read and are not checked. */
arkv_status arkv_check(arkv_cache* cache, void* stream);

/* Host only.  Count schedule of one unit (R9, R12, R14, R15): prefill of prompt_len
   tokens then n_steps decode appends at ratio rho.  Writes up to max_events events
   of 4 int32 (step, n_o, n_q, n_evicted) — step -1 is the prefill tailor — and their
   number to *n_events.  Used to cross-check the host schedule against the oracle. */
arkv_status arkv_schedule(const arkv_config* cfg, int32_t prompt_len, double rho, int32_t n_steps,
                          int32_t* events, int32_t max_events, int32_t* n_events);

/* Host only.  Verifies the cache's tile layout: the Original-tile element
   offsets are a bijection onto the tile's 2-byte cells, the Quantized-tile code bits plus
   the fp32 scale/zero cells cover the tile exactly once, and the code-slot inverse used by
   the tailor's packing pass inverts the forward map.  ARKV_ERR_DEVICE on a violation. */
arkv_status arkv_layout_check(const arkv_config* cfg, int64_t* n_checked);

/* Layer-shared token states across KV-head shards (state_sharing = 1, NEXT-3; collective
   C3 of DESIGN.md §8).  The group-averaged tailor score needs every KV head of
   the layer; when a sequence's heads are split over processes:
   1. arkv_tailor_scores (async on stream): for each (sequence, layer) whose tailor the NEXT
      call runs — arkv_prefill_finish after arkv_prefill_begin (every (b, l) when the prompt
      needs the prefill-end tailor), else arkv_decode_step(layer0, n_layers) — writes row
      r = d_scores[r * stride + i], the fp32 sum over this cache's KV heads of the Eq. 9
      score of eligible row i, in (b, l) order; *n_rows = the rows written (0: no tailor).
      ARKV_ERR_CAPACITY when max_rows or stride (>= eligible rows) is too small.
   2. The caller sums the buffers across the shards (NCCL all-reduce, in place).
   3. arkv_set_tailor_scores(cache, d_sum, stride, total_kv_heads): the next
      arkv_decode_step / arkv_prefill_finish uses sum / total_kv_heads as the score of its
      tailors, then forgets the pointer (the buffer must stay valid until that call's work
      has run on its stream).
   Without step 3 the score averages this cache's KV heads only. */
arkv_status arkv_tailor_scores(arkv_cache* cache, int32_t layer0, int32_t n_layers, float* d_scores, int64_t stride,
                               int32_t max_rows, int32_t* n_rows, void* stream);
arkv_status arkv_set_tailor_scores(arkv_cache* cache, const float* d_scores, int64_t stride, int32_t total_kv_heads);

/* Host only.  Builds the persistent decode kernel's work plan (decode_kernel = 3;
   DESIGN.md §6) for n_units units with the given Original / Quantized row counts and at
   most max_ctas CTAs, then replays one step on the host — the producer's unit-merged item
   order, each consumer warp's partial slot, the coverage table and the combine's slot
   enumeration — checking that every item is streamed exactly once, no two partials share
   a slot, and each unit's combine merges exactly its own partials.  *ctas_used = the grid
   the plan chose.  ARKV_ERR_DEVICE on a violated invariant, ARKV_ERR_INVALID_ARG on
   counts outside the cache's capacity. */
arkv_status arkv_persist_plan_check(const arkv_config* cfg, const int32_t* n_o, const int32_t* n_q,
                                    int32_t n_units, int32_t max_ctas, int32_t* ctas_used);

/* Host only.  Builds the split-K decode kernel's cost-balanced launch order (DESIGN.md §6,
   "cost-balanced split-K launch order") for n_pairs (sequence, layer) pairs of a call with
   the given Original rows before the step's append (n_o) and Quantized rows (n_q), each
   pair with the cache's H_kv KV heads, on a GPU of num_sms SMs (2 CTAs per SM), then
   replays what the kernel derives from it: every unit of the call exactly once, each
   unit's split count in 1 .. max_splits and equal for the KV heads of a pair, the kernel's
   split ranges covering each unit's Original and Quantized tiles exactly once, at most
   2 x 2 num_sms CTAs plus one per unit whose cost share rounds to zero, and pieces in
   non-increasing estimated cost (LPT).  *n_ctas = the
   grid.  ARKV_ERR_DEVICE on a violated invariant, ARKV_ERR_CAPACITY when the call has more
   units than the order holds (the kernel then uses its uniform grid),
   ARKV_ERR_INVALID_ARG on counts outside the cache's capacity. */
arkv_status arkv_split_order_check(const arkv_config* cfg, const int32_t* n_o, const int32_t* n_q, int32_t n_pairs,
                                   int32_t num_sms, int32_t* n_ctas);

/* Host only.  Statistics -> OQ score (Eq. 6 with the R6 clamps applied to the raw
   moments). */
arkv_status arkv_oq_score(const arkv_config* cfg, double entropy, double m2, double m4, double* stats3,
                          double* score);

/* Live timing of the decode attention kernel with CUDA events recorded on the launching
   stream around every launch (bench roofline).  arkv_profile(1) enables and resets;
   arkv_profile_read (syncs) returns the summed kernel time in ms, the number of timed
   launches and their summed algorithmic bytes (cache segments read + the step's token
   read and appended + query read).  which = 0: decode attention kernel.
   which = 1 (host only, no sync, always on): the algorithmic bytes of every arkv_decode_step
   call since the cache was created (attention bytes as for which = 0 plus the
   output written; + 16 B per row of units in their HH window; per tailor, 8 B per eligible
   row + the unit's segments read once + the survivors written); launches = calls,
   total_ms = 0. */
arkv_status arkv_profile(arkv_cache* cache, int32_t enable);
arkv_status arkv_profile_read(arkv_cache* cache, int32_t which, double* total_ms, int64_t* launches,
                              double* alg_bytes);

/* Introspection: what = 0 -> tile layout in use (ARKV_LAYOUT_PLAIN / _FRAG);
   1 -> decode kernel in use (0 generic, 1 tensor-core split-K kernel, 2 tensor-core
   persistent kernel, 3 auto: split-K, or the persistent kernel for a call whose bytes are
   mostly Quantized tiles).  -1 on error. */
int32_t arkv_cache_info(const arkv_cache* cache, int32_t what);

/* Number of kernel launches issued by this cache so far (bench accounting). */
int64_t arkv_launch_count(const arkv_cache* cache);

/* Build/feature string, e.g. "arkv sm_100a layouts=plain,frag fast=mma.sync". */
const char* arkv_version(void);
const char* arkv_status_string(arkv_status s);

#ifdef __cplusplus
}
#endif
#endif /* ARKV_H_ */
