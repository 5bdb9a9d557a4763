// arkv_host.cu — host runtime behind the C ABI (include/arkv.h).
//
// Owns the data-independent count schedule (R9, R12, R14, R15): every (sequence,
// layer) advances through counts the host knows without reading the device, so
// the decode step never synchronizes.  Carves the caller's arena / workspace,
// assigns arena slots (two-stack per unit plus staging slots for the tailor's
// out-of-place compaction), and sequences the kernel launches.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <memory>
#include <numeric>
#include <vector>

#include "kernels.h"

using namespace arkv;

int arkv::tuning_knob(const char* name, int def) {
#ifdef ARKV_TUNING_KNOBS
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : def;
#else
  (void)name;
  return def;
#endif
}

struct arkv_cache {
  arkv_config cfg;
  Geom g;
  int device = 0;
  // arena
  uint8_t* slots = nullptr;
  uint8_t* meta = nullptr;
  UnitDesc* desc = nullptr;
  int32_t* err = nullptr;
  int n_slots = 0, n_spare = 0;
  // workspace
  float* partials = nullptr;
  float* logits = nullptr;
  int8_t* st_scratch = nullptr;
  int32_t* src_scratch = nullptr;
  float* sscore = nullptr;
  float* ssm = nullptr;
  std::vector<int32_t> sm_thr;  // per (sequence, layer): rows with position <= this carry a smoothed score
  // layer-shared states across KV-head shards: score sums exchanged by the caller, consumed
  // by the next call that runs tailors (arkv_set_tailor_scores)
  const float* ext_scores = nullptr;
  int64_t ext_stride = 0;
  int ext_heads = 0;
  int prompt_len = 0;  // set by arkv_prefill_begin
  float* pf_partials = nullptr;
  float2* acc_pf = nullptr;
  double* oq_tmp = nullptr;
  double* colsum = nullptr;
  float* mstat = nullptr;
  int32_t* counters = nullptr;
  int32_t* nsplit = nullptr;
  std::unique_ptr<UnitOrder> chunks{new UnitOrder};  // split-K launch order (host copy, a kernel parameter)
  std::vector<int> chunk_ns;                          // its split count per (sequence, layer) of the call
  // persistent decode kernel (decode_kernel = 3): partial slots and coverage tables
  float* pparts = nullptr;
  int4* pcta = nullptr;
  int32_t* pcover = nullptr;
  bool persist = false;
  int num_sms = 148;
  int jobs_per_wave = 0, jobs_per_prefill_wave = 0, max_splits = 64, n_chunks1_max = 1;
  // live kernel timing of the decode attention kernel (bench roofline)
  bool prof = false;
  std::vector<cudaEvent_t> ev;  // pairs
  std::vector<double> ev_bytes;
  int ev_used = 0;
  // algorithmic bytes of every decode call since creation (host arithmetic, always on):
  // arkv_profile_read(which = 1)
  double step_bytes = 0.0;
  int64_t step_calls = 0;
  bool fast = false;
  // host mirrors
  std::vector<double> rho;
  std::vector<int> n_o, n_q, t_next, trig;  // per (b, l)
  std::vector<int> q0;  // per (b, l): first query position on the current cache (the first decode
                        // call after the prompt, or the step of the last decode tailor; R19)
  std::vector<int> unit_slot;               // per unit
  std::vector<int> spare;
  bool prefilled = false;
  int64_t launches = 0;
};

namespace {

constexpr int kPfChunkHost = 2048;

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct Sizes {
  Geom g;
  int n_spare, jobs_per_wave, jobs_scratch, max_splits, n_chunks1;
  int64_t arena, ws;
  int64_t off_meta, off_desc, off_err;
  int64_t w_partials, w_logits, w_st, w_sscore, w_ssm, w_src, w_pfp, w_accpf, w_oq, w_colsum, w_mstat, w_counters, w_nsplit, w_plan, w_pparts;
};

int64_t cost_o(const arkv_config& c) { return 4LL * c.head_dim; }
int64_t cost_q(const arkv_config& c) {
  int gs = c.group_size ? c.group_size : c.head_dim;
  return 2LL * ((int64_t)c.head_dim * c.quant_bits / 8 + 8LL * (c.head_dim / gs));
}

arkv_status validate(const arkv_config* c) {
  if (!c) return ARKV_ERR_INVALID_ARG;
  if (c->n_layers <= 0 || c->n_q_heads <= 0 || c->n_kv_heads <= 0 || c->batch <= 0 || c->window <= 0)
    return ARKV_ERR_CONFIG;
  if (c->n_q_heads % c->n_kv_heads) return ARKV_ERR_CONFIG;
  int G = c->n_q_heads / c->n_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8) return ARKV_ERR_CONFIG;
  // every kernel path (prefill passes, generic and fast decode, both move kernels) covers these
  if (c->head_dim != 16 && c->head_dim != 32 && c->head_dim != 64 && c->head_dim != 128) return ARKV_ERR_CONFIG;
  if (c->quant_bits != 2 && c->quant_bits != 4 && c->quant_bits != 8) return ARKV_ERR_CONFIG;
  int gs = c->group_size ? c->group_size : c->head_dim;
  if (gs < 8 || gs % 8 || c->head_dim % gs) return ARKV_ERR_CONFIG;
  if (c->budget_tokens <= 2 * c->window) return ARKV_ERR_CONFIG;  // R14
  if (c->quant_mode != ARKV_QUANT_ASYM && c->quant_mode != ARKV_QUANT_SYM && c->quant_mode != ARKV_QUANT_FP8)
    return ARKV_ERR_CONFIG;
  if (c->quant_mode == ARKV_QUANT_FP8 && c->quant_bits != 8) return ARKV_ERR_CONFIG;
  if (c->max_positions <= 0 || c->max_prompt <= 0 || c->max_prompt > c->max_positions) return ARKV_ERR_CONFIG;
  if (c->alpha <= 0.0 || c->alpha > 1.0) return ARKV_ERR_CONFIG;
  const bool frag_ok = c->head_dim % 32 == 0 && (c->quant_bits == 4 || c->quant_mode == ARKV_QUANT_FP8);
  if (c->layout == ARKV_LAYOUT_FRAG && !frag_ok) return ARKV_ERR_CONFIG;
  if (c->layout < 0 || c->layout > 2) return ARKV_ERR_CONFIG;
  if (c->decode_kernel < 0 || c->decode_kernel > 3) return ARKV_ERR_CONFIG;
  if (c->state_sharing != 0 && c->state_sharing != 1) return ARKV_ERR_CONFIG;
  if (!(c->smooth >= 0.f && c->smooth < 1.f)) return ARKV_ERR_CONFIG;
  // layer-shared tailors run a layer's KV heads in one wave (one spare slot each)
  if (c->state_sharing == 1 && c->n_spare_slots > 0 && c->n_spare_slots < c->n_kv_heads) return ARKV_ERR_CONFIG;
  return ARKV_OK;
}

Sizes compute_sizes(const arkv_config& c) {
  Sizes s{};
  Geom& g = s.g;
  g.d = c.head_dim;
  g.Hq = c.n_q_heads;
  g.Hkv = c.n_kv_heads;
  g.G = g.Hq / g.Hkv;
  g.L = c.n_layers;
  g.batch = c.batch;
  g.W = c.window;
  g.bits = c.quant_bits;
  g.g = c.group_size ? c.group_size : c.head_dim;
  g.ng = g.d / g.g;
  g.mode = c.quant_mode;
  g.share = c.state_sharing;
  g.smooth = c.smooth;
  g.layout = c.layout;
  if (g.layout == ARKV_LAYOUT_AUTO)
    g.layout = ((c.quant_bits == 4 || c.quant_mode == ARKV_QUANT_FP8) && c.head_dim % 32 == 0) ? ARKV_LAYOUT_FRAG
                                                                                              : ARKV_LAYOUT_PLAIN;
  g.B = c.budget_tokens;
  g.cost_o = (int)cost_o(c);
  g.cost_q = (int)cost_q(c);
  g.tile_o = kTile * g.cost_o;
  g.tile_q = kTile * g.cost_q;
  const int64_t Bb = (int64_t)g.B * g.cost_o;
  g.cap_o = (int)round_up(g.B + 1, kTile);
  g.cap_q = (int)round_up((Bb - 2LL * g.W * g.cost_o) / g.cost_q + 1, kTile);
  g.max_pos = c.max_positions;
  g.n_units = g.batch * g.L * g.Hkv;
  g.slot_bytes = round_up(Bb + g.tile_o + g.tile_q, 256);
  g.meta_bytes = round_up((int64_t)g.cap_o * (c.smooth > 0.f ? 16 : 12) + (int64_t)g.cap_q * (c.smooth > 0.f ? 16 : 12),
                          256);  // pos, acc (+ smoothed score, R34)
  g.sm_scale = c.sm_scale > 0.f ? c.sm_scale : (float)(1.0 / std::sqrt((double)g.d));
  g.gamma = (float)c.gamma;

  s.n_spare = c.n_spare_slots > 0 ? c.n_spare_slots : g.batch * g.Hkv;
  s.jobs_per_wave = std::min(s.n_spare, kMaxJobs);  // decode tailors: one spare slot per job
  // the prefill-end tailor writes every unit into its own (empty) slot: waves of up to
  // kMaxJobs jobs, not bounded by the spares (measured: 32 waves of 8 units took 6 ms at
  // configs[1])
  s.jobs_scratch = std::max(s.jobs_per_wave, std::min(g.n_units, kMaxJobs));
  s.max_splits = c.max_splits > 0 ? c.max_splits : 64;
  s.n_chunks1 = (int)((c.max_prompt + kPfChunkHost - 1) / kPfChunkHost);
  const int n_slots = g.n_units + s.n_spare;
  s.off_meta = (int64_t)n_slots * g.slot_bytes;
  s.off_desc = s.off_meta + (int64_t)n_slots * g.meta_bytes;
  s.off_err = round_up(s.off_desc + (int64_t)g.n_units * sizeof(UnitDesc), 256);
  s.arena = s.off_err + 256;

  int64_t w = 0;
  s.w_partials = w;
  w = round_up(w + (int64_t)g.n_units * s.max_splits * g.G * (g.d + 2) * 4, 256);
  s.w_logits = w;
  w = round_up(w + (int64_t)g.n_units * g.G * (g.cap_o + g.cap_q) * 4, 256);
  s.w_st = w;
  const int64_t st_stride = std::max<int64_t>(g.max_pos, g.cap_o) + g.cap_q;
  w = round_up(w + (int64_t)s.jobs_scratch * st_stride, 256);
  s.w_sscore = w;  // layer-shared scores of the eligible rows, per job
  w = round_up(w + (c.state_sharing ? (int64_t)s.jobs_scratch * st_stride * 4 : 0), 256);
  s.w_ssm = w;  // smoothed scores of the old rows, per job (R34)
  w = round_up(w + (c.smooth > 0.f ? (int64_t)s.jobs_scratch * st_stride * 4 : 0), 256);
  s.w_src = w;
  w = round_up(w + (int64_t)s.jobs_scratch * (g.cap_o + g.cap_q) * 4, 256);
  s.w_pfp = w;
  w = round_up(w + (int64_t)g.n_units * s.n_chunks1 * g.G * g.W * 8, 256);
  s.w_accpf = w;
  w = round_up(w + (int64_t)g.n_units * g.max_pos * 8, 256);
  s.w_oq = w;
  w = round_up(w + (int64_t)g.batch * g.L * 8, 256);
  s.w_colsum = w;
  w = round_up(w + (int64_t)g.batch * g.L * g.max_pos * 8, 256);
  s.w_mstat = w;
  w = round_up(w + (int64_t)g.n_units * g.G * 8, 256);
  s.w_counters = w;
  w = round_up(w + (int64_t)g.n_units * 4, 256);
  s.w_nsplit = w;  // split count per unit of a chunk-list decode launch
  w = round_up(w + (int64_t)g.n_units * 4, 256);
  // persistent decode kernel: its plan and one partial per (unit, covering CTA, warp)
  s.w_plan = w;  // pcta [2][kPlanMaxCtas] int4, then pcover [2][2][n_units] int32
  w = round_up(w + (int64_t)2 * kPlanMaxCtas * 16 + (int64_t)4 * g.n_units * 4, 256);
  s.w_pparts = w;
  w = round_up(w + (int64_t)2 * (kPlanMaxCtas + g.n_units) * kPersistConsumers * g.G * (g.d + 2) * 4, 256);
  s.ws = w;
  return s;
}

// Eq. 10 counts with the R14 headroom rule (must equal oracle.tailor_counts).
void tailor_counts(const Geom& g, double alpha, int64_t K, double rho, int64_t* n_oe, int64_t* n_q) {
  const int64_t W = g.W, B = g.B, Co = g.cost_o, Cq = g.cost_q, Bb = B * Co;
  const int64_t n_e = K - W;
  const int64_t b = (int64_t)std::floor(alpha * (double)n_e);
  const int64_t quota = (int64_t)std::floor(rho * (double)(B - W));
  int64_t o = std::min(std::min(quota, b), B - 2 * W);
  int64_t q = std::min(b - o, (Bb - (o + 2 * W) * Co) / Cq);
  *n_oe = o;
  *n_q = q;
}
// Appends after which the unit first reaches B_bytes, U >= B_bytes (R12; "reaches
// the limit"): the next tailor fires at (position of the last counted token) +
// this.  After any tailor or an untailored prompt U <= B_bytes - W*C_o (R14), so this is >= W.
int64_t appends_to_trigger(const Geom& g, int64_t n_o, int64_t n_q) {
  const int64_t Bb = (int64_t)g.B * g.cost_o;
  const int64_t U = n_o * g.cost_o + n_q * g.cost_q;
  return std::max<int64_t>(1, (Bb - U + g.cost_o - 1) / g.cost_o);
}

// First position whose query is an Eq. 9 sample of the tailor at `trig` (R19): the last W
// queries before it, but only those that ran on the current cache (from q0 on).
int acc0_of(const Geom& g, int64_t trig, int64_t q0) { return (int)std::max<int64_t>(trig - g.W, q0); }

// ARKV_DEBUG_SYNC=1 (tuning builds): synchronize after every launch group and name the failing one.
void debug_sync(cudaStream_t s, const char* what) {
  static const bool on = tuning_knob("ARKV_DEBUG_SYNC", 0) != 0;
  if (!on) return;
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) std::fprintf(stderr, "arkv: %s failed: %s\n", what, cudaGetErrorString(e));
}

bool check_cuda(cudaError_t e) {
  if (e != cudaSuccess) std::fprintf(stderr, "arkv: CUDA error: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess;
}

}  // namespace

extern "C" {

const char* arkv_version(void) {
  return "arkv 0.5 sm_100a layouts=plain,frag decode=generic,mma-sync-chunked-split,mma-sync-persistent "
         "prefill=tcgen05-tma-ws,mma-sync quant=int2/4/8,fp8-e4m3 states=per-head,layer-shared "
         "scores=eq9,smoothed";
}

const char* arkv_status_string(arkv_status s) {
  switch (s) {
    case ARKV_OK: return "ok";
    case ARKV_ERR_INVALID_ARG: return "invalid argument";
    case ARKV_ERR_CONFIG: return "invalid configuration";
    case ARKV_ERR_SEQUENCE: return "sequencing error";
    case ARKV_ERR_WINDOW: return "prompt shorter than W + 2 without rho_override";
    case ARKV_ERR_LAYOUT: return "budget/bit-width differ from the cache";
    case ARKV_ERR_CAPACITY: return "arena or workspace too small";
    case ARKV_ERR_DEVICE: return "device error flag set";
    case ARKV_ERR_CUDA: return "CUDA runtime error";
    case ARKV_ERR_NO_DEVICE: return "no sm_100 device";
  }
  return "unknown";
}

arkv_status arkv_config_default(arkv_config* c) {
  if (!c) return ARKV_ERR_INVALID_ARG;
  std::memset(c, 0, sizeof(*c));
  c->window = 32;
  c->quant_bits = 4;
  c->group_size = 0;
  c->quant_mode = ARKV_QUANT_ASYM;
  c->layout = ARKV_LAYOUT_AUTO;
  c->alpha = 0.75;
  c->tau[0] = 7.774;
  c->tau[1] = 5.407;
  c->tau[2] = 5.528;
  c->gamma = 263.81;
  c->stat_eps = 1e-30;
  c->batch = 1;
  return ARKV_OK;
}

arkv_status arkv_cache_bytes(const arkv_config* cfg, size_t* arena_bytes, size_t* workspace_bytes) {
  arkv_status st = validate(cfg);
  if (st != ARKV_OK) return st;
  Sizes s = compute_sizes(*cfg);
  if (arena_bytes) *arena_bytes = (size_t)s.arena;
  if (workspace_bytes) *workspace_bytes = (size_t)s.ws;
  return ARKV_OK;
}

arkv_status arkv_schedule(const arkv_config* cfg, int32_t P, double rho, int32_t n_steps, int32_t* events,
                          int32_t max_events, int32_t* n_events) {
  arkv_status st = validate(cfg);
  if (st != ARKV_OK) return st;
  if (!n_events || P <= 0 || n_steps < 0) return ARKV_ERR_INVALID_ARG;
  Geom g = compute_sizes(*cfg).g;
  int n = 0;
  auto push = [&](int s, int64_t a, int64_t b, int64_t c) {
    if (events && n < max_events) {
      events[4 * n + 0] = s;
      events[4 * n + 1] = (int32_t)a;
      events[4 * n + 2] = (int32_t)b;
      events[4 * n + 3] = (int32_t)c;
    }
    ++n;
  };
  int64_t n_o, n_q;
  if (P > g.B - g.W) {
    int64_t oe, q;
    tailor_counts(g, cfg->alpha, P, rho, &oe, &q);
    push(-1, oe + g.W, q, P - g.W - oe - q);
    n_o = oe + g.W;
    n_q = q;
  } else {
    n_o = P;
    n_q = 0;
  }
  // drive by trigger positions, exactly as the runtime does
  int64_t trig = (P - 1) + appends_to_trigger(g, n_o, n_q);
  for (int s = 0; s < n_steps; ++s) {
    const int64_t t = P + s;
    if (t == trig) {
      const int64_t K = n_o + 1 + n_q;
      int64_t oe, q;
      tailor_counts(g, cfg->alpha, K, rho, &oe, &q);
      push(s, oe + g.W, q, K - g.W - oe - q);
      n_o = oe + g.W;
      n_q = q;
      trig = t + appends_to_trigger(g, n_o, n_q);
    } else {
      n_o += 1;
    }
  }
  *n_events = n;
  return ARKV_OK;
}

arkv_status arkv_layout_check(const arkv_config* cfg, int64_t* n_checked) {
  arkv_status st = validate(cfg);
  if (st != ARKV_OK) return st;
  const Geom g = compute_sizes(*cfg).g;
  int64_t n = 0;
  // Original tile: every (token, dim) of K and V maps to a distinct 2-byte cell; all cells used
  std::vector<uint8_t> seen(g.tile_o, 0);
  for (int j = 0; j < kTile; ++j)
    for (int x = 0; x < g.d; ++x)
      for (int v = 0; v < 2; ++v) {
        const int off = v ? o_v_off(g, j, x) : o_k_off(g, j, x);
        if (off < 0 || off + 2 > g.tile_o || (off & 1) || seen[off] || seen[off + 1]) return ARKV_ERR_DEVICE;
        seen[off] = seen[off + 1] = 1;
        ++n;
      }
  for (uint8_t b : seen)
    if (!b) return ARKV_ERR_DEVICE;
  // Quantized tile: codes (bit level) and scales/zeros cover the tile exactly once, and
  // q_code_slot inverts q_k_loc / q_v_loc
  std::vector<uint8_t> bits((size_t)g.tile_q * 8, 0);
  for (int j = 0; j < kTile; ++j)
    for (int x = 0; x < g.d; ++x)
      for (int v = 0; v < 2; ++v) {
        int byte, shift;
        if (v) q_v_loc(g, j, x, &byte, &shift);
        else q_k_loc(g, j, x, &byte, &shift);
        if (byte < 0 || byte >= g.tile_q || shift % g.bits) return ARKV_ERR_DEVICE;
        for (int b = 0; b < g.bits; ++b) {
          if (bits[(size_t)byte * 8 + shift + b]) return ARKV_ERR_DEVICE;
          bits[(size_t)byte * 8 + shift + b] = 1;
        }
        int jj, xx, vv;
        if (!q_code_slot(g, byte, shift / g.bits, &jj, &xx, &vv) || jj != j || xx != x || vv != v)
          return ARKV_ERR_DEVICE;
        ++n;
      }
  for (int j = 0; j < kTile; ++j)
    for (int w = 0; w < 4; ++w)
      for (int gr = 0; gr < g.ng; ++gr) {
        const int off = q_sc_off(g, j, w, gr);
        if (off < 0 || off + 4 > g.tile_q || (off & 3)) return ARKV_ERR_DEVICE;
        for (int b = 0; b < 32; ++b) {
          if (bits[(size_t)off * 8 + b]) return ARKV_ERR_DEVICE;
          bits[(size_t)off * 8 + b] = 1;
        }
        int jj, xx, vv;
        if (q_code_slot(g, off, 0, &jj, &xx, &vv)) return ARKV_ERR_DEVICE;
        ++n;
      }
  for (uint8_t b : bits)
    if (!b) return ARKV_ERR_DEVICE;
  if (n_checked) *n_checked = n;
  return ARKV_OK;
}

arkv_status arkv_oq_score(const arkv_config* cfg, double H, double m2, double m4, double* stats3, double* score) {
  if (!cfg) return ARKV_ERR_INVALID_ARG;
  const double eps = cfg->stat_eps;
  double K = m2 > eps ? m4 / (m2 * m2) : 1.0;
  double Hc = std::fmax(H, eps), Vc = std::fmax(m2, eps), Kc = std::fmax(K, eps);
  if (stats3) {
    stats3[0] = Hc;
    stats3[1] = Vc;
    stats3[2] = Kc;
  }
  if (score) *score = std::pow(Hc, 1.0 / cfg->tau[0]) * std::pow(Vc, 1.0 / cfg->tau[1]) * std::pow(Kc, 1.0 / cfg->tau[2]);
  return ARKV_OK;
}

arkv_status arkv_cache_create(const arkv_config* cfg, void* d_arena, size_t arena_bytes, void* d_workspace,
                              size_t workspace_bytes, arkv_cache** out) {
  arkv_status st = validate(cfg);
  if (st != ARKV_OK) return st;
  if (!d_arena || !d_workspace || !out) return ARKV_ERR_INVALID_ARG;
  if (((uintptr_t)d_arena & 255) || ((uintptr_t)d_workspace & 255)) return ARKV_ERR_INVALID_ARG;
  Sizes s = compute_sizes(*cfg);
  if ((int64_t)arena_bytes < s.arena || (int64_t)workspace_bytes < s.ws) return ARKV_ERR_CAPACITY;
  int dev = 0;
  if (!check_cuda(cudaGetDevice(&dev))) return ARKV_ERR_NO_DEVICE;
  cudaDeviceProp prop;
  if (!check_cuda(cudaGetDeviceProperties(&prop, dev))) return ARKV_ERR_NO_DEVICE;
  if (prop.major != 10) return ARKV_ERR_NO_DEVICE;
  arkv_cache* c = new arkv_cache();
  c->cfg = *cfg;
  c->g = s.g;
  c->device = dev;
  uint8_t* a = (uint8_t*)d_arena;
  c->slots = a;
  c->meta = a + s.off_meta;
  c->desc = (UnitDesc*)(a + s.off_desc);
  c->err = (int32_t*)(a + s.off_err);
  c->n_spare = s.n_spare;
  c->n_slots = s.g.n_units + s.n_spare;
  uint8_t* w = (uint8_t*)d_workspace;
  c->partials = (float*)(w + s.w_partials);
  c->logits = (float*)(w + s.w_logits);
  c->st_scratch = (int8_t*)(w + s.w_st);
  c->src_scratch = (int32_t*)(w + s.w_src);
  c->sscore = (float*)(w + s.w_sscore);
  c->ssm = (float*)(w + s.w_ssm);
  c->pf_partials = (float*)(w + s.w_pfp);
  c->acc_pf = (float2*)(w + s.w_accpf);
  c->oq_tmp = (double*)(w + s.w_oq);
  c->colsum = (double*)(w + s.w_colsum);
  c->mstat = (float*)(w + s.w_mstat);
  c->counters = (int32_t*)(w + s.w_counters);
  c->nsplit = (int32_t*)(w + s.w_nsplit);
  c->pcta = (int4*)(w + s.w_plan);
  c->pcover = (int32_t*)(w + s.w_plan + 2 * kPlanMaxCtas * 16);
  c->pparts = (float*)(w + s.w_pparts);
  c->num_sms = prop.multiProcessorCount;
  c->jobs_per_wave = s.jobs_per_wave;
  c->jobs_per_prefill_wave = s.jobs_scratch;
  c->max_splits = s.max_splits;
  c->n_chunks1_max = s.n_chunks1;
  const int BL = s.g.batch * s.g.L;
  c->rho.assign(BL, 1.0);
  c->n_o.assign(BL, 0);
  c->n_q.assign(BL, 0);
  c->t_next.assign(BL, 0);
  c->trig.assign(BL, 0);
  c->q0.assign(BL, 0);
  c->sm_thr.assign(BL, -1);
  c->unit_slot.resize(s.g.n_units);
  for (int u = 0; u < s.g.n_units; ++u) c->unit_slot[u] = u;
  for (int k = c->n_slots - 1; k >= s.g.n_units; --k) c->spare.push_back(k);
  bool fast_ok = decode_fast_available(s.g);
  c->fast = cfg->decode_kernel == 1 ? false : fast_ok;
  {
    // auto (decode_kernel = 0): the persistent range-partitioned kernel when a step has many
    // small units (>= 32 per SM: split-K would run them as ~1-split CTAs in dozens of waves;
    // measured at configs[3], 16384 units: 35.7K vs 33.8K tok/s), else split-K (configs[1],
    // configs[2] per GPU, configs[4] per GPU: split-K 3-12 % faster).  ARKV_DECODE_PERSIST
    // overrides the rule (tuning builds).
    const int ep = tuning_knob("ARKV_DECODE_PERSIST", -1);
    const bool auto_persist = ep >= 0 ? ep != 0 : s.g.n_units >= 32 * c->num_sms;
    c->persist = c->fast && (cfg->decode_kernel == 3 || (cfg->decode_kernel == 0 && auto_persist));
  }
  if ((cfg->decode_kernel == 2 || cfg->decode_kernel == 3) && !fast_ok) {
    delete c;
    return ARKV_ERR_CONFIG;
  }
  // slots and per-slot metadata start zeroed: tiles are always moved whole (bulk copies,
  // export), so rows past a unit's n_o / n_q are defined bytes (compute-sanitizer initcheck)
  // persistent-kernel partial slots start with l = 0 (= unused; decode_persist_combine)
  if (!check_cuda(cudaMemset(c->slots, 0, (size_t)s.off_desc)) || !check_cuda(cudaMemset(c->err, 0, 4)) ||
      !check_cuda(cudaMemset(c->pparts, 0, (size_t)(s.ws - s.w_pparts))) ||
      !check_cuda(cudaMemset(c->pcover, 0xff, (size_t)4 * s.g.n_units * 4)) ||
      !check_cuda(cudaMemset(c->counters, 0, (size_t)s.g.n_units * 4))) {
    delete c;
    return ARKV_ERR_CUDA;
  }
  *out = c;
  return ARKV_OK;
}

arkv_status arkv_cache_destroy(arkv_cache* c) {
  if (c) {
    for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  }
  delete c;
  return ARKV_OK;
}

arkv_status arkv_profile(arkv_cache* c, int32_t enable) {
  if (!c) return ARKV_ERR_INVALID_ARG;
  c->prof = enable != 0;
  c->ev_used = 0;
  if (c->prof && c->ev.empty()) {
    const int pairs = 8192;
    c->ev.resize(2 * pairs);
    c->ev_bytes.assign(pairs, 0.0);
    for (auto& e : c->ev)
      if (!check_cuda(cudaEventCreate(&e))) return ARKV_ERR_CUDA;
  }
  return ARKV_OK;
}

arkv_status arkv_profile_read(arkv_cache* c, int32_t which, double* total_ms, int64_t* launches, double* alg_bytes) {
  if (!c || which < 0 || which > 1) return ARKV_ERR_INVALID_ARG;
  if (which == 1) {  // whole decode calls: host-side counts, no events, no sync
    if (total_ms) *total_ms = 0.0;
    if (launches) *launches = c->step_calls;
    if (alg_bytes) *alg_bytes = c->step_bytes;
    return ARKV_OK;
  }
  double ms = 0.0, by = 0.0;
  for (int i = 0; i < c->ev_used; ++i) {
    if (!check_cuda(cudaEventSynchronize(c->ev[2 * i + 1]))) return ARKV_ERR_CUDA;
    float t = 0.f;
    if (!check_cuda(cudaEventElapsedTime(&t, c->ev[2 * i], c->ev[2 * i + 1]))) return ARKV_ERR_CUDA;
    ms += t;
    by += c->ev_bytes[i];
  }
  if (total_ms) *total_ms = ms;
  if (launches) *launches = c->ev_used;
  if (alg_bytes) *alg_bytes = by;
  return ARKV_OK;
}

int64_t arkv_launch_count(const arkv_cache* c) { return c ? c->launches : 0; }

int32_t arkv_cache_info(const arkv_cache* c, int32_t what) {
  if (!c) return -1;
  if (what == 0) return c->g.layout;
  if (what == 1) return c->persist ? 2 : (c->fast ? (c->cfg.decode_kernel == 0 ? 3 : 1) : 0);
  return -1;
}

// Runs a list of tailor jobs in waves bounded by the spare-slot count.
static arkv_status run_jobs(arkv_cache* c, std::vector<TailorJob>& jobs, const uint16_t* pk, const uint16_t* pv, int P,
                            cudaStream_t s) {
  const Geom& g = c->g;
  int wave = pk ? c->jobs_per_prefill_wave : c->jobs_per_wave;  // prefill jobs need no spare slot
  if (g.share) wave -= wave % g.Hkv;  // a layer's KV heads select together (jobs come in (b, l, kvh) order)
  size_t i = 0;
  while (i < jobs.size()) {
    const int n = (int)std::min<size_t>(jobs.size() - i, (size_t)wave);
    TailorJobs tj;
    std::memset(&tj, 0, sizeof(tj));
    int max_tiles = 1;
    for (int k = 0; k < n; ++k) {
      TailorJob jb = jobs[i + k];
      if (jb.new_slot < 0) {
        if (c->spare.empty()) return ARKV_ERR_CAPACITY;
        jb.new_slot = c->spare.back();
        c->spare.pop_back();
      }
      jobs[i + k] = jb;
      tj.j[k] = jb;
      int no = jb.n_oe + jb.n_win_old;
      int tiles = (no + kTile - 1) / kTile + (jb.n_q_new + kTile - 1) / kTile;
      max_tiles = std::max(max_tiles, tiles);
      if (no > g.cap_o + 0 || jb.n_q_new > g.cap_q) return ARKV_ERR_CAPACITY;
    }
    SharedScores shs;
    shs.sscore = c->sscore;
    shs.ssm = c->ssm;
    shs.ext = c->ext_scores;
    shs.ext_stride = c->ext_stride;
    shs.ext_heads = c->ext_heads;
    int nl = launch_tailor(g, tj, n, max_tiles, c->slots, c->meta, c->desc, pk, pv, P, c->acc_pf, c->st_scratch,
                           c->src_scratch, shs, c->err, s);
    if (nl < 0) return ARKV_ERR_CONFIG;
    c->launches += nl;
    debug_sync(s, "tailor");
    if (!check_cuda(cudaGetLastError())) return ARKV_ERR_CUDA;
    for (int k = 0; k < n; ++k) {
      const TailorJob& jb = jobs[i + k];
      if (jb.old_slot >= 0) c->spare.push_back(jb.old_slot);
      c->unit_slot[jb.unit] = jb.new_slot;
    }
    i += n;
  }
  return ARKV_OK;
}

arkv_status arkv_prefill_begin(arkv_cache* c, const void* q_win, const void* k, int32_t P, double* d_colsum,
                               void* stream) {
  if (!c || !q_win || !k) return ARKV_ERR_INVALID_ARG;
  if (c->prefilled) return ARKV_ERR_SEQUENCE;
  const Geom& g = c->g;
  if (P <= 0 || P > c->cfg.max_prompt || P >= g.max_pos) return ARKV_ERR_INVALID_ARG;
  if (P < g.W + 2) return ARKV_ERR_WINDOW;
  cudaStream_t s = (cudaStream_t)stream;
  const int n_chunks1 = (P + kPfChunkHost - 1) / kPfChunkHost;
  c->prompt_len = P;
  int nl = launch_prefill_begin(g, (const uint16_t*)q_win, (const uint16_t*)k, P, c->pf_partials, n_chunks1, c->acc_pf,
                                d_colsum ? d_colsum : c->colsum, s);
  if (nl < 0) return ARKV_ERR_CONFIG;
  c->launches += nl;
  debug_sync(s, "prefill_begin");
  if (!check_cuda(cudaGetLastError())) return ARKV_ERR_CUDA;
  return ARKV_OK;
}

arkv_status arkv_prefill_finish(arkv_cache* c, const void* k, const void* v, int32_t P, const double* d_colsum,
                                const double* rho_override, double* d_stats, double* d_oq, double* h_rho,
                                void* stream) {
  if (!c || !k || !v) return ARKV_ERR_INVALID_ARG;
  if (c->prefilled) return ARKV_ERR_SEQUENCE;
  const Geom& g = c->g;
  if (P <= 0 || P > c->cfg.max_prompt || P >= g.max_pos) return ARKV_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const bool tailor = P > g.B - g.W;  // R14
  const bool stats_ok = P >= g.W + 2;
  if (!stats_ok && (rho_override == nullptr || tailor)) return ARKV_ERR_WINDOW;
  const int BL = g.batch * g.L;
  std::vector<double> rho(BL, 1.0);
  if (stats_ok) {
    double* oq = d_oq ? d_oq : c->oq_tmp;
    int nl = launch_prefill_finish(g, d_colsum ? d_colsum : c->colsum, P, d_stats, oq, c->cfg.tau, c->cfg.stat_eps, c->err, s);
    c->launches += nl;
    debug_sync(s, "prefill_finish");
    if (!check_cuda(cudaGetLastError())) return ARKV_ERR_CUDA;
    std::vector<double> h(BL);
    if (!check_cuda(cudaMemcpyAsync(h.data(), oq, BL * sizeof(double), cudaMemcpyDeviceToHost, s))) return ARKV_ERR_CUDA;
    if (!check_cuda(cudaStreamSynchronize(s))) return ARKV_ERR_CUDA;
    for (int b = 0; b < g.batch; ++b) {  // Eq. 7: ratio within the sequence (R8)
      double mx = 0.0;
      for (int l = 0; l < g.L; ++l) mx = std::max(mx, h[b * g.L + l]);
      for (int l = 0; l < g.L; ++l) rho[b * g.L + l] = mx > 0.0 ? h[b * g.L + l] / mx : 1.0;
    }
  }
  if (rho_override)
    for (int i = 0; i < BL; ++i) rho[i] = rho_override[i];
  c->rho = rho;
  if (h_rho)
    for (int i = 0; i < BL; ++i) h_rho[i] = rho[i];

  // ingest (+ prefill-end tailor)
  std::vector<TailorJob> jobs;
  for (int bl = 0; bl < BL; ++bl) {
    int64_t oe, q;
    int n_win, n_o;
    if (tailor) {
      tailor_counts(g, c->cfg.alpha, P, rho[bl], &oe, &q);
      n_win = g.W;
      n_o = (int)oe + g.W;
    } else {
      n_win = std::min(g.W, P);
      oe = P - n_win;
      q = 0;
      n_o = P;
    }
    c->n_o[bl] = n_o;
    c->n_q[bl] = (int)q;
    c->t_next[bl] = P;
    c->trig[bl] = (int)((P - 1) + appends_to_trigger(g, n_o, q));
    c->q0[bl] = P;  // the prompt's queries are not Eq. 9 samples of decode tailors (R19)
    for (int kvh = 0; kvh < g.Hkv; ++kvh) {
      TailorJob jb{};
      jb.unit = bl * g.Hkv + kvh;
      jb.old_slot = -1;
      jb.new_slot = c->unit_slot[jb.unit];
      jb.n_o_old = P;
      jb.n_q_old = 0;
      jb.n_win_old = n_win;
      jb.n_oe = (int)oe;
      jb.n_q_new = (int)q;
      jb.trig_new = c->trig[bl];
      jb.acc0_new = acc0_of(g, c->trig[bl], P);
      jb.n_rows = g.W;  // the prompt's last W queries (Eq. 2)
      jb.t_next = P;
      jb.identity = tailor ? 0 : 1;
      jb.ext_row = (tailor && c->ext_scores) ? bl : -1;  // arkv_tailor_scores rows: every (b, l)
      jb.prev_thr = -1;  // the first tailor of the sequence: no smoothed scores yet (R34)
      jobs.push_back(jb);
    }
    // R34: the prefill tailor scored (and kept or evicted) every position < P - W
    c->sm_thr[bl] = tailor ? P - g.W - 1 : -1;
  }
  arkv_status st = run_jobs(c, jobs, (const uint16_t*)k, (const uint16_t*)v, P, s);
  c->ext_scores = nullptr;  // consumed
  if (st != ARKV_OK) return st;
  c->prefilled = true;
  return ARKV_OK;
}

arkv_status arkv_prefill_stats(arkv_cache* c, const void* q_win, const void* k, const void* v, int32_t P,
                               const double* rho_override, double* d_stats, double* d_oq, double* h_rho,
                               void* stream) {
  if (!c || !k || !v) return ARKV_ERR_INVALID_ARG;
  if (P >= c->g.W + 2) {
    arkv_status st = arkv_prefill_begin(c, q_win, k, P, nullptr, stream);
    if (st != ARKV_OK) return st;
  }
  return arkv_prefill_finish(c, k, v, P, nullptr, rho_override, d_stats, d_oq, h_rho, stream);
}

// Work plan of the persistent decode kernel for units [layer0, layer0 + n_layers) of all
// sequences (PersistPlan in kernels.h).  Phase 0 items: each unit's Original
// tiles (rows n_o; the step's token is appended by the combine); phase 1 items: its
// Quantized tiles in groups of q_per.  Each phase's item stream is cut into P equal ranges;
// a range's partial slots are C per unit it spans.  P shrinks until no unit needs more
// than kMaxUnitParts slots.
int persist_items(const Geom& g, int n_o, int n_q, int f) {
  const int q_per = (32 * 4 * g.d) / g.tile_q;  // Quantized tiles per 16 KB ring stage
  const int tiles_q = (n_q + kTile - 1) / kTile;
  return f == 0 ? (n_o + kTile - 1) / kTile : (tiles_q + q_per - 1) / q_per;
}

// Plan for U units with the given per-unit counts (units in call order).
void build_plan_counts(const Geom& g, int U, const int* n_o, const int* n_q, int P, PersistPlan* plan) {
  std::vector<int64_t> first[2];
  for (int f = 0; f < 2; ++f) first[f].assign(U + 1, 0);
  for (int ul = 0; ul < U; ++ul)
    for (int f = 0; f < 2; ++f) first[f][ul + 1] = first[f][ul] + persist_items(g, n_o[ul], n_q[ul], f);
  const int64_t N = std::max(first[0][U], first[1][U]);
  P = (int)std::max<int64_t>(1, std::min<int64_t>(std::min(P, kPlanMaxCtas), N));
  std::vector<int> cf[2], cl[2];
  const int64_t cap = (int64_t)2 * (kPlanMaxCtas + g.n_units) * kPersistConsumers;  // compute_sizes
  for (;;) {
    for (int f = 0; f < 2; ++f) {
      cf[f].assign(U, -1);
      cl[f].assign(U, -1);
    }
    int64_t slots = 0;
    for (int f = 0; f < 2; ++f) {
      const int64_t Nf = first[f][U];
      int ul = 0;
      for (int k = 0; k < P; ++k) {
        const int64_t i0 = Nf * k / P, i1 = Nf * (k + 1) / P;
        int4 r = make_int4(0, 0, (int)(i1 - i0), (int)slots);
        int ue = 0;
        if (i1 > i0) {
          while (first[f][ul + 1] <= i0) ++ul;  // unit holding item i0
          ue = ul;
          while (first[f][ue + 1] <= i1 - 1) ++ue;  // unit holding the range's last item
          r.x = ul;
          r.y = (int)(i0 - first[f][ul]);
          slots += (int64_t)(ue - ul + 1) * kPersistConsumers;
          // the combine enumerates every CTA between a unit's first and last covering one
          for (int u = ul; u <= ue; ++u)
            if (first[f][u + 1] > first[f][u]) {
              if (cf[f][u] < 0) cf[f][u] = k;
              cl[f][u] = k;
            }
        }
        plan->cta[f][k] = r;
        plan->ue[f][k] = ue;
      }
    }
    int span_max = 0;
    for (int u = 0; u < U; ++u) {
      int n = 0;
      for (int f = 0; f < 2; ++f)
        if (cf[f][u] >= 0) n += cl[f][u] - cf[f][u] + 1;
      span_max = std::max(span_max, n);
    }
    if ((span_max * kPersistConsumers <= kMaxUnitParts && slots <= cap) || P == 1) break;
    P = std::max(1, P * 3 / 4);  // too few units for this many CTAs: fewer, longer ranges
  }
  plan->P = P;
}

void build_plan(const arkv_cache* c, int layer0, int n_layers, int P, PersistPlan* plan) {
  const Geom& g = c->g;
  const int U = g.batch * n_layers * g.Hkv;
  std::vector<int> no(U), nq(U);
  for (int ul = 0; ul < U; ++ul) {
    const int b = ul / (n_layers * g.Hkv), li = (ul / g.Hkv) % n_layers;
    const int bl = b * g.L + layer0 + li;
    no[ul] = c->n_o[bl];
    nq[ul] = c->n_q[bl];
  }
  build_plan_counts(g, U, no.data(), nq.data(), P, plan);
}

// Host replay of one persistent step under a plan (the producer's unit-merged order, the
// consumer warps' partial slots, the coverage table and the combine's enumeration), checking
// every invariant the kernels rely on.  Returns false on a violation.
static int fail_line = 0;
bool replay_plan(const Geom& g, int U, const int* n_o, const int* n_q, const PersistPlan& plan) {
  constexpr int C = kPersistConsumers;
  const int P = plan.P;
  const int64_t cap = (int64_t)2 * (kPlanMaxCtas + g.n_units) * C;
  auto items = [&](int u, int f) { return persist_items(g, n_o[u], n_q[u], f); };
  std::vector<std::vector<int>> seen(2);
  for (int f = 0; f < 2; ++f) {
    int64_t n = 0;
    for (int u = 0; u < U; ++u) n += items(u, f);
    seen[f].assign((size_t)n, 0);
  }
  std::vector<int64_t> first[2];
  for (int f = 0; f < 2; ++f) {
    first[f].assign(U + 1, 0);
    for (int u = 0; u < U; ++u) first[f][u + 1] = first[f][u] + items(u, f);
  }
  std::vector<int> cover(4 * U, -1);
  std::vector<int> slot_unit((size_t)cap, -1);
  for (int c = 0; c < P; ++c) {
    int ul[2], k[2], rem[2];
    for (int f = 0; f < 2; ++f) {
      ul[f] = plan.cta[f][c].x;
      k[f] = plan.cta[f][c].y;
      rem[f] = plan.cta[f][c].z;
    }
    std::vector<int> seq;
    const int n_work = rem[0] + rem[1];
    const bool q_first = (c & 1) != 0;  // default item order (decode_persist_kernel)
    for (int j = 0; j < n_work; ++j) {
      const int f = (rem[0] > 0 && (rem[1] <= 0 || (q_first ? ul[0] < ul[1] : ul[0] <= ul[1]))) ? 0 : 1;
      if (ul[f] < 0 || ul[f] >= U || k[f] < 0 || k[f] >= items(ul[f], f)) { fail_line = __LINE__; return false; }
      const int64_t gi = first[f][ul[f]] + k[f];
      if (seen[f][(size_t)gi]++) { fail_line = __LINE__; return false; }  // processed twice
      if (k[f] == 0) cover[(f * 2 + 0) * U + ul[f]] = c;
      if (k[f] == items(ul[f], f) - 1) cover[(f * 2 + 1) * U + ul[f]] = c;
      seq.push_back(ul[f]);
      if (--rem[f] > 0) {
        ++k[f];
        while (k[f] >= items(ul[f], f)) {
          k[f] -= items(ul[f], f);
          if (++ul[f] >= U) { fail_line = __LINE__; return false; }
        }
      }
    }
    for (int w = 0; w < C; ++w) {
      int cur = -1;
      std::vector<int> done;
      for (int j = w; j < n_work; j += C) {
        if (seq[j] == cur) continue;
        cur = seq[j];
        for (int d : done)
          if (d == cur) { fail_line = __LINE__; return false; }  // a warp must see each unit once
        done.push_back(cur);
        const int4 r0 = plan.cta[0][c];
        const bool in0 = r0.z > 0 && cur >= r0.x && cur <= plan.ue[0][c];
        const int4 r = in0 ? r0 : plan.cta[1][c];
        const int64_t slot = r.w + (int64_t)(cur - r.x) * C + w;
        if (slot < 0 || slot >= cap || slot_unit[(size_t)slot] != -1) { fail_line = __LINE__; return false; }
        slot_unit[(size_t)slot] = cur;
      }
    }
  }
  for (int f = 0; f < 2; ++f)
    for (int v : seen[f])
      if (v != 1) { fail_line = __LINE__; return false; }  // every item exactly once
  for (int u = 0; u < U; ++u) {
    std::vector<int64_t> en;
    for (int f = 0; f < 2; ++f) {
      const int cf = cover[(f * 2 + 0) * U + u], cl = cover[(f * 2 + 1) * U + u];
      if (cf < 0) continue;
      for (int cc = cf; cc <= cl; ++cc) {
        const int4 r = plan.cta[f][cc];
        if (r.z <= 0) continue;
        int4 pc = make_int4(r.x, r.w, plan.ue[f][cc], 0);
        if (f == 1) {
          const int4 q0 = plan.cta[0][cc];
          if (q0.z > 0 && u >= q0.x && u <= plan.ue[0][cc]) {
            pc = make_int4(q0.x, q0.w, plan.ue[0][cc], 0);
            const int cf0 = cover[u], cl0 = cover[U + u];
            if (cf0 >= 0 && cc >= cf0 && cc <= cl0) continue;
          }
        }
        for (int w = 0; w < C; ++w) en.push_back(pc.y + (int64_t)(u - pc.x) * C + w);
      }
    }
    const int nc = (cover[u] >= 0 ? (cover[U + u] - cover[u] + 1) * C : 0) +
                   (cover[2 * U + u] >= 0 ? (cover[3 * U + u] - cover[2 * U + u] + 1) * C : 0);
    if (nc > kMaxUnitParts) { fail_line = __LINE__; return false; }
    std::sort(en.begin(), en.end());
    if (std::adjacent_find(en.begin(), en.end()) != en.end()) { fail_line = __LINE__; return false; }  // merged twice
    for (int64_t sl : en)
      if (sl < 0 || sl >= cap || (slot_unit[(size_t)sl] != -1 && slot_unit[(size_t)sl] != u)) { fail_line = __LINE__; return false; }
    for (int64_t sl = 0; sl < cap; ++sl)
      if (slot_unit[(size_t)sl] == u && !std::binary_search(en.begin(), en.end(), sl)) { fail_line = __LINE__; return false; }  // lost
  }
  return true;
}

arkv_status arkv_persist_plan_check(const arkv_config* cfg, const int32_t* n_o, const int32_t* n_q, int32_t n_units,
                                    int32_t max_ctas, int32_t* ctas_used) {
  arkv_status st = validate(cfg);
  if (st != ARKV_OK) return st;
  if (!n_o || !n_q || n_units <= 0) return ARKV_ERR_INVALID_ARG;
  Sizes s = compute_sizes(*cfg);
  if (n_units > s.g.n_units) return ARKV_ERR_INVALID_ARG;
  for (int u = 0; u < n_units; ++u)
    if (n_o[u] < 0 || n_q[u] < 0 || n_o[u] > s.g.cap_o || n_q[u] > s.g.cap_q) return ARKV_ERR_INVALID_ARG;
  PersistPlan* plan = new PersistPlan();
  build_plan_counts(s.g, n_units, n_o, n_q, max_ctas, plan);
  const bool ok = replay_plan(s.g, n_units, n_o, n_q, *plan);
  if (!ok && tuning_knob("ARKV_DEBUG_PLAN", 0)) std::fprintf(stderr, "replay_plan: violation at arkv_host.cu:%d\n", fail_line);
  if (ctas_used) *ctas_used = plan->P;
  delete plan;
  return ok ? ARKV_OK : ARKV_ERR_DEVICE;
}

static bool order_from_counts(const Geom& g, int BL, const int32_t* n_o, const int32_t* n_q, int max_splits,
                              int slots, UnitOrder& uo, std::vector<int>& ns);

arkv_status arkv_split_order_check(const arkv_config* cfg, const int32_t* n_o, const int32_t* n_q, int32_t n_pairs,
                                   int32_t num_sms, int32_t* n_ctas) {
  arkv_status st = validate(cfg);
  if (st != ARKV_OK) return st;
  if (!n_o || !n_q || n_pairs <= 0 || num_sms <= 0) return ARKV_ERR_INVALID_ARG;
  Sizes s = compute_sizes(*cfg);
  const Geom& g = s.g;
  if (n_pairs > g.batch * g.L) return ARKV_ERR_INVALID_ARG;
  for (int i = 0; i < n_pairs; ++i)
    if (n_o[i] < 0 || n_q[i] < 0 || n_o[i] >= g.cap_o || n_q[i] > g.cap_q) return ARKV_ERR_INVALID_ARG;
  std::unique_ptr<UnitOrder> uo(new UnitOrder);
  std::vector<int> ns;
  const int slots = 2 * num_sms;
  if (!order_from_counts(g, n_pairs, n_o, n_q, s.max_splits, slots, *uo, ns)) return ARKV_ERR_CAPACITY;
  if (n_ctas) *n_ctas = uo->n_ctas;
  // replay what the decode kernel derives from the order: every unit exactly once, its
  // splits [pfx[p], pfx[p + 1]) in 1 .. max_splits, every Original and Quantized tile of
  // the unit in exactly one split, and the positions in non-increasing piece cost
  const int n_units = n_pairs * g.Hkv;
  if (uo->n_units != n_units || uo->pfx[0] != 0 || uo->pfx[n_units] != uo->n_ctas) return ARKV_ERR_DEVICE;
  std::vector<int> seen(n_units, 0);
  // the apportionment targets 2 CTAs per slot; a pair whose share rounds to 0 still gets one
  const int64_t want = (std::max<int64_t>(n_pairs, (int64_t)2 * slots / g.Hkv) + n_pairs) * g.Hkv;
  if (uo->n_ctas > want) return ARKV_ERR_DEVICE;
  double prev = INFINITY;
  for (int p = 0; p < n_units; ++p) {
    const int ul = uo->perm[p], S = uo->pfx[p + 1] - uo->pfx[p];
    if (ul < 0 || ul >= n_units || seen[ul]++ || S < 1 || S > s.max_splits || S != ns[ul / g.Hkv])
      return ARKV_ERR_DEVICE;
    const int i = ul / g.Hkv;
    const int to = (n_o[i] + 1 + kTile - 1) / kTile, tq = (n_q[i] + kTile - 1) / kTile;
    const double piece = (to + 0.01 * tuning_knob("ARKV_QCOST", 62) * tq) / S;
    if (piece > prev + 1e-9) return ARKV_ERR_DEVICE;
    prev = piece;
    int o_next = 0, q_next = 0;
    for (int sp = 0; sp < S; ++sp) {  // the kernel's split ranges (k_decode_fast.cu)
      const int o0 = (int)((int64_t)sp * to / S), o1 = (int)((int64_t)(sp + 1) * to / S);
      const int q0 = (int)((int64_t)sp * tq / S), q1 = (int)((int64_t)(sp + 1) * tq / S);
      if (o0 != o_next || q0 != q_next || o1 < o0 || q1 < q0) return ARKV_ERR_DEVICE;
      o_next = o1;
      q_next = q1;
    }
    if (o_next != to || q_next != tq) return ARKV_ERR_DEVICE;
  }
  return ARKV_OK;
}

arkv_status arkv_tailor_scores(arkv_cache* c, int32_t layer0, int32_t n_layers, float* d_scores, int64_t stride,
                               int32_t max_rows, int32_t* n_rows, void* stream) {
  if (!c || !d_scores || !n_rows) return ARKV_ERR_INVALID_ARG;
  const Geom& g = c->g;
  if (!g.share) return ARKV_ERR_CONFIG;
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<TailorJob> jobs;  // the tailors the next call will run, as score sources
  int max_ne = 0;
  if (!c->prefilled) {  // prefill-end tailor (R14): every (b, l), rows = the prompt's eligible tokens
    const int P = c->prompt_len;
    if (P <= 0) return ARKV_ERR_SEQUENCE;  // arkv_prefill_begin first (it fills the HH seed)
    if (P > g.B - g.W) {
      for (int bl = 0; bl < g.batch * g.L; ++bl)
        for (int kvh = 0; kvh < g.Hkv; ++kvh) {
          TailorJob jb{};
          jb.unit = bl * g.Hkv + kvh;
          jb.old_slot = -1;
          jb.n_o_old = P;
          jb.n_win_old = g.W;
          jb.n_rows = g.W;
          jb.ext_row = -1;
          jb.prev_thr = -1;
          jobs.push_back(jb);
        }
      max_ne = P - g.W;
    }
  } else {
    if (layer0 < 0 || n_layers <= 0 || layer0 + n_layers > g.L) return ARKV_ERR_INVALID_ARG;
    for (int b = 0; b < g.batch; ++b)
      for (int l = layer0; l < layer0 + n_layers; ++l) {
        const int bl = b * g.L + l;
        if (c->t_next[bl] != c->trig[bl]) continue;
        for (int kvh = 0; kvh < g.Hkv; ++kvh) {
          TailorJob jb{};
          jb.unit = bl * g.Hkv + kvh;
          jb.old_slot = c->unit_slot[jb.unit];
          jb.n_o_old = c->n_o[bl];
          jb.n_q_old = c->n_q[bl];
          jb.n_win_old = g.W - 1;
          jb.n_rows = c->t_next[bl] - acc0_of(g, c->t_next[bl], c->q0[bl]);
          jb.ext_row = -1;
          jb.prev_thr = -1;
          jobs.push_back(jb);
        }
        max_ne = std::max(max_ne, c->n_o[bl] - (g.W - 1) + c->n_q[bl]);
      }
  }
  const int rows = (int)jobs.size() / g.Hkv;
  *n_rows = rows;
  if (rows == 0) return ARKV_OK;
  if (rows > max_rows || stride < max_ne) return ARKV_ERR_CAPACITY;
  const int per = (kMaxJobs / g.Hkv) * g.Hkv;  // whole layers per launch
  for (size_t i = 0; i < jobs.size(); i += per) {
    const int n = (int)std::min<size_t>(jobs.size() - i, (size_t)per);
    TailorJobs tj;
    std::memset(&tj, 0, sizeof(tj));
    for (int k = 0; k < n; ++k) tj.j[k] = jobs[i + k];
    launch_tailor_scores(g, tj, n, max_ne, c->meta, c->acc_pf, d_scores + (int64_t)(i / g.Hkv) * stride, stride,
                         c->err, s);
    c->launches += 1;
  }
  if (!check_cuda(cudaGetLastError())) return ARKV_ERR_CUDA;
  return ARKV_OK;
}

arkv_status arkv_set_tailor_scores(arkv_cache* c, const float* d_scores, int64_t stride, int32_t total_kv_heads) {
  if (!c) return ARKV_ERR_INVALID_ARG;
  if (!c->g.share) return ARKV_ERR_CONFIG;
  if (d_scores && (stride <= 0 || total_kv_heads < c->g.Hkv)) return ARKV_ERR_INVALID_ARG;
  c->ext_scores = d_scores;
  c->ext_stride = stride;
  c->ext_heads = total_kv_heads;
  return ARKV_OK;
}

// Cost-balanced split-K launch order (UnitOrder, kernels.h) for the fast decode kernel.
// Measured (scripts/cta_timeline.py, per-CTA globaltimer stamps at configs[1]): with the same
// number of splits for every unit, the CTAs of Quantized-heavy units ran 1.8x longer than
// those of Original-heavy ones (the Quantized path is issue-bound, a 4.5 KB Quantized tile
// costs ~0.6 of a 16 KB Original tile), and the kernel spent its last 15 % (HH-window steps)
// with a draining, half-empty grid.  Here a unit's estimated time is its Original tiles +
// q_cost x its Quantized tiles; the step's CTAs are exactly `waves` x the CTA slots,
// apportioned to the units by largest remainder of their cost shares (>= 1, <= the
// per-unit cap of ~min_items work items per CTA and max_splits), and the units are launched
// in decreasing piece cost (LPT).  Measured at configs[1]: HH-window decode kernel -6 %,
// steady state -1 % (2 waves beat 3 and 4: fewer per-CTA fills and drains).
// The order for BL (sequence, layer) pairs with counts n_o (before this step's append) and
// n_q, each with g.Hkv KV heads (units i * Hkv + kvh).  ns: split count per pair.
static bool order_from_counts(const Geom& g, int BL, const int32_t* n_o, const int32_t* n_q, int max_splits,
                              int slots, UnitOrder& uo, std::vector<int>& ns) {
  if (BL * g.Hkv > kMaxOrderUnits) return false;
  static const double q_cost = 0.01 * tuning_knob("ARKV_QCOST", 62);
  static const int waves = tuning_knob("ARKV_EXACT_WAVES", 2);
  static const int min_items = tuning_knob("ARKV_MIN_ITEMS", 20);
  std::vector<double> cost(BL), x(BL);
  std::vector<int> cap(BL);
  ns.assign(BL, 1);
  double total = 0.0;
  for (int i = 0; i < BL; ++i) {
    const int to = (n_o[i] + 1 + kTile - 1) / kTile, tq = (n_q[i] + kTile - 1) / kTile;
    cost[i] = to + q_cost * tq;
    const int items = to + (tq + 2) / 3;
    cap[i] = std::max(1, std::min({max_splits, to + tq, items / std::max(1, min_items), 256}));
    total += cost[i];
  }
  // per (sequence, layer): every KV head of it has the same counts and the same split count
  std::vector<int> idx(BL);
  int64_t n = 0;
  auto apportion = [&](int64_t want) {
    n = 0;
    for (int i = 0; i < BL; ++i) {
      x[i] = cost[i] / std::max(total, 1e-30) * (double)want;
      ns[i] = std::max(1, std::min((int)std::floor(x[i]), cap[i]));
      n += ns[i];
    }
    std::iota(idx.begin(), idx.end(), 0);
    std::stable_sort(idx.begin(), idx.end(), [&](int p, int q) { return x[p] - ns[p] > x[q] - ns[q]; });
    for (int j = 0; j < BL && n < want; ++j)
      if (ns[idx[j]] < cap[idx[j]]) {
        ++ns[idx[j]];
        ++n;
      }
  };
  const int64_t want = std::max<int64_t>(BL, (int64_t)waves * slots / g.Hkv);
  apportion(want);
  // a call whose per-CTA work caps bind (few units: one KV head per GPU, a layer per call)
  // and whose CTAs overrun one wave by a fraction would run a partial last wave of
  // full-length CTAs: trim it to whole waves instead (measured, emulated 8-GPU shard of
  // configs[1]: 416 -> 288 CTAs, 18.6K -> 20.9K tok/s)
  if (n < want && n * g.Hkv > slots && (n * g.Hkv) % slots != 0) {
    const int64_t whole = (n * g.Hkv / slots) * slots / g.Hkv;
    if (whole >= BL) apportion(whole);
  }
  if (n * g.Hkv > 0xFFFF) return false;
  // launch order: decreasing piece cost (LPT), then unit index
  std::stable_sort(idx.begin(), idx.end(), [&](int p, int q) { return cost[p] / ns[p] > cost[q] / ns[q]; });
  int pos = 0, cta = 0;
  for (int j = 0; j < BL; ++j) {
    const int i = idx[j];
    for (int kvh = 0; kvh < g.Hkv; ++kvh) {
      uo.perm[pos] = (uint16_t)(i * g.Hkv + kvh);
      uo.pfx[pos] = (uint16_t)cta;
      cta += ns[i];
      ++pos;
    }
  }
  uo.pfx[pos] = (uint16_t)cta;
  uo.n_units = pos;
  uo.n_ctas = cta;
  return true;
}

static bool build_chunks(arkv_cache* c, int layer0, int n_layers, int slots) {
  static const int mode = tuning_knob("ARKV_CHUNKS", 1);  // 0: the uniform grid
  if (mode == 0) return false;
  const Geom& g = c->g;
  const int BL = g.batch * n_layers;
  std::vector<int32_t> no(BL), nq(BL);
  for (int b = 0; b < g.batch; ++b)
    for (int l = layer0; l < layer0 + n_layers; ++l) {
      no[b * n_layers + (l - layer0)] = c->n_o[b * g.L + l];
      nq[b * n_layers + (l - layer0)] = c->n_q[b * g.L + l];
    }
  return order_from_counts(g, BL, no.data(), nq.data(), c->max_splits, slots, *c->chunks, c->chunk_ns);
}

arkv_status arkv_decode_step(arkv_cache* c, int32_t layer0, int32_t n_layers, const void* q, const void* k,
                             const void* v, int32_t budget_tokens, int32_t quant_bits, void* out, int32_t out_fp32,
                             void* stream) {
  if (!c || !q || !k || !v || !out) return ARKV_ERR_INVALID_ARG;
  const Geom& g = c->g;
  if (layer0 < 0 || n_layers <= 0 || layer0 + n_layers > g.L) return ARKV_ERR_INVALID_ARG;
  if (budget_tokens != g.B || quant_bits != g.bits) return ARKV_ERR_LAYOUT;
  if (!c->prefilled) return ARKV_ERR_SEQUENCE;
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<TailorJob> jobs;
  int max_tiles = 1, acc_rows = 0, n_due = 0;
  double items_sum = 0.0, seg_o = 0.0, seg_q = 0.0;
  HhPlan hh;  // (sequence, layer) pairs in their HH window this step (fused combine)
  hh.n = 0;
  bool hh_fit = true;
  for (int b = 0; b < g.batch; ++b)
    for (int l = layer0; l < layer0 + n_layers; ++l) {
      const int bl = b * g.L + l;
      const int t = c->t_next[bl];
      if (t + 1 > g.max_pos) return ARKV_ERR_SEQUENCE;
      if (t == c->trig[bl]) {
        const int64_t K = (int64_t)c->n_o[bl] + 1 + c->n_q[bl];
        int64_t oe, qn;
        tailor_counts(g, c->cfg.alpha, K, c->rho[bl], &oe, &qn);
        const int n_o_after = (int)oe + g.W;  // after this step's append
        // tailor: the eligible rows' accumulators, the unit's segments read
        // once, the survivors written
        c->step_bytes += (double)g.Hkv * (8.0 * (double)(K - g.W) + (double)c->n_o[bl] * g.cost_o +
                                          (double)c->n_q[bl] * g.cost_q + (double)n_o_after * g.cost_o +
                                          (double)qn * g.cost_q);
        const int trig_new = (int)(t + appends_to_trigger(g, n_o_after, qn));
        for (int kvh = 0; kvh < g.Hkv; ++kvh) {
          TailorJob jb{};
          jb.unit = bl * g.Hkv + kvh;
          jb.old_slot = c->unit_slot[jb.unit];
          jb.new_slot = -1;
          jb.n_o_old = c->n_o[bl];
          jb.n_q_old = c->n_q[bl];
          jb.n_win_old = g.W - 1;
          jb.n_oe = (int)oe;
          jb.n_q_new = (int)qn;
          jb.trig_new = trig_new;
          jb.acc0_new = acc0_of(g, trig_new, t);
          jb.n_rows = t - acc0_of(g, t, c->q0[bl]);
          jb.t_next = t;
          jb.identity = 0;
          jb.ext_row = c->ext_scores ? n_due : -1;  // arkv_tailor_scores rows: due (b, l) in order
          jb.prev_thr = c->sm_thr[bl];
          jobs.push_back(jb);
        }
        c->sm_thr[bl] = t - g.W;  // this tailor scores positions <= t - W (the W newest are the window)
        c->n_o[bl] = n_o_after - 1;
        c->n_q[bl] = (int)qn;
        c->trig[bl] = trig_new;
        c->q0[bl] = t;  // this step's query runs after the tailor (R13)
        ++n_due;
      }
      const int tiles = (c->n_o[bl] + 1 + kTile - 1) / kTile + (c->n_q[bl] + kTile - 1) / kTile;
      max_tiles = std::max(max_tiles, tiles);
      // split-K work items (one Original tile, or a group of up to 3 Quantized tiles)
      items_sum += (double)g.Hkv * ((c->n_o[bl] + 1 + kTile - 1) / kTile + ((c->n_q[bl] + kTile - 1) / kTile + 2) / 3);
      // attention: segments read, the token read and appended, q read, out written
      c->step_bytes += (double)g.Hkv * ((double)c->n_o[bl] * g.cost_o + (double)c->n_q[bl] * g.cost_q +
                                        2.0 * g.cost_o + 4.0 * g.G * g.d);
      seg_o += (double)c->n_o[bl] * g.cost_o;
      seg_q += (double)c->n_q[bl] * g.cost_q;
      const int acc0 = acc0_of(g, c->trig[bl], c->q0[bl]);
      if (t >= acc0 && t < c->trig[bl]) {  // HH accumulation step (R19)
        const int rows = c->n_o[bl] + 1 + c->n_q[bl];
        c->step_bytes += (double)g.Hkv * 16.0 * rows;  // accumulator read-modify-write
        acc_rows = std::max(acc_rows, rows);
        if (hh.n < kMaxHhEntries)
          hh.e[hh.n++] = make_int4(b * n_layers + (l - layer0), rows, t == acc0 ? 1 : 0, c->n_q[bl]);
        else
          hh_fit = false;
      }
    }
  ++c->step_calls;
  if (!jobs.empty()) {
    arkv_status st = run_jobs(c, jobs, nullptr, nullptr, 0, s);
    c->ext_scores = nullptr;  // consumed (also when this step runs no tailor: see below)
    if (st != ARKV_OK) return st;
  }
  c->ext_scores = nullptr;  // exchanged scores serve exactly the call after arkv_tailor_scores
  // split-K fan-out: ~2.6 waves of CTAs (measured at configs[1]: S = 3 beats 2 and 4; more
  // splits cost pipeline fill/drain per CTA and combine reads), never more splits than tiles
  const int n_units_call = g.batch * n_layers * g.Hkv;
  const int slots = c->num_sms * (c->fast ? 2 : 4);
  int S = (int)std::lround(2.6 * slots / (double)n_units_call);
  // ... but no fewer than ~20 work items per CTA (sweeps with self-refill: 8-GPU shard S = 12
  // beats 19, 4-GPU S = 9 beats 12, configs[1] S = 3): a call with few units (one layer per
  // call, or one KV head per GPU) would otherwise spread each unit over dozens of CTAs that
  // spend their time filling and draining the pipeline, and the combine merges as many partials
  static const int min_items = tuning_knob("ARKV_MIN_ITEMS", 20);
  S = std::min(S, std::max(1, (int)(items_sum / n_units_call / min_items)));
  S = std::max(1, std::min(S, std::min(c->max_splits, max_tiles)));
  if (const int v = tuning_knob("ARKV_SPLITS", 0); v > 0) S = std::min(v, std::min(c->max_splits, max_tiles));

  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->prof && 2 * (c->ev_used + 1) <= (int)c->ev.size()) {
    e0 = c->ev[2 * c->ev_used];
    e1 = c->ev[2 * c->ev_used + 1];
    // algorithmic bytes of this launch: cache segments read + the step's token read and
    // appended + the query read
    double by = 0.0;
    for (int b = 0; b < g.batch; ++b)
      for (int l = layer0; l < layer0 + n_layers; ++l) {
        const int bl = b * g.L + l;
        by += (double)g.Hkv * ((double)c->n_o[bl] * g.cost_o + (double)c->n_q[bl] * g.cost_q + 2.0 * g.cost_o +
                               2.0 * g.G * g.d);
      }
    c->ev_bytes[c->ev_used] = by;
    c->ev_used++;
  }
  PlanArgs pa;
  static const bool fuse_hh = tuning_knob("ARKV_FUSE_HH", 1) != 0;
  // auto kernel choice per call: round 2's rule also took the persistent range-partitioned
  // kernel when >= 60 % of a call's bytes were Quantized tiles (then 0.68 vs 0.51 of the copy
  // peak).  The chunked split-K pipeline with cost-balanced splits beats it there too (rho = 0
  // at configs[1], HH window: kernel 0.218 vs 0.221 ms, step 0.238 vs 0.249 ms), so the
  // Quantized-share switch is off (ARKV_PERSIST_QSHARE, tuning builds, restores it).
  static const int q_share_pct = tuning_knob("ARKV_PERSIST_QSHARE", 101);
  const bool persist = c->persist || (c->fast && c->cfg.decode_kernel == 0 &&
                                      seg_q > 0.01 * q_share_pct * (seg_o + seg_q));
  if (acc_rows > 0 && hh_fit && fuse_hh && !persist) {
    hh.n_units = g.batch * n_layers * g.Hkv;
    pa.hh = &hh;
  }
  PersistPlan plan;
  if (!persist && c->fast && build_chunks(c, layer0, n_layers, slots)) {
    pa.chunks = c->chunks.get();
    pa.nsplit = c->nsplit;
    // the HH combine merges each unit's partials with the split count known here
    for (int k = 0; k < hh.n; ++k) hh.e[k].z |= c->chunk_ns[hh.e[k].x] << 1;
  } else {
    for (int k = 0; k < hh.n; ++k) hh.e[k].z |= S << 1;
  }
  if (persist) {
    build_plan(c, layer0, n_layers, 2 * c->num_sms, &plan);
    pa.plan = &plan;
    pa.pparts = c->pparts;
    pa.pcta = c->pcta;
    pa.pcover = c->pcover;
  }
  int nl = launch_decode(g, layer0, n_layers, (const uint16_t*)q, (const uint16_t*)k, (const uint16_t*)v, out,
                         out_fp32, c->slots, c->meta, c->desc, c->partials, c->logits, c->mstat, c->counters, acc_rows, S,
                         c->max_splits, c->fast ? 1 : 0, c->err, s, e0, e1, pa);
  if (nl < 0 && c->fast) {  // fast kernel not available for this shape: generic kernel
    nl = launch_decode(g, layer0, n_layers, (const uint16_t*)q, (const uint16_t*)k, (const uint16_t*)v, out, out_fp32,
                       c->slots, c->meta, c->desc, c->partials, c->logits, c->mstat, c->counters, acc_rows, S, c->max_splits, 0,
                       c->err, s, e0, e1);
  }
  if (nl < 0) return ARKV_ERR_CONFIG;
  c->launches += nl;
  debug_sync(s, "decode");
  if (!check_cuda(cudaGetLastError())) return ARKV_ERR_CUDA;
  for (int b = 0; b < g.batch; ++b)
    for (int l = layer0; l < layer0 + n_layers; ++l) {
      const int bl = b * g.L + l;
      c->n_o[bl] += 1;
      c->t_next[bl] += 1;
    }
  return ARKV_OK;
}

arkv_status arkv_unit_counts(const arkv_cache* c, int32_t b, int32_t l, int32_t* n_o, int32_t* n_q, int32_t* next_pos,
                             int32_t* next_tailor) {
  if (!c || b < 0 || b >= c->g.batch || l < 0 || l >= c->g.L) return ARKV_ERR_INVALID_ARG;
  const int bl = b * c->g.L + l;
  if (n_o) *n_o = c->n_o[bl];
  if (n_q) *n_q = c->n_q[bl];
  if (next_pos) *next_pos = c->t_next[bl];
  if (next_tailor) *next_tailor = c->trig[bl];
  return ARKV_OK;
}

arkv_status arkv_export_unit(arkv_cache* c, int32_t b, int32_t l, int32_t kvh, arkv_unit_export* out, void* stream) {
  if (!c || !out || b < 0 || b >= c->g.batch || l < 0 || l >= c->g.L || kvh < 0 || kvh >= c->g.Hkv)
    return ARKV_ERR_INVALID_ARG;
  const Geom& g = c->g;
  cudaStream_t s = (cudaStream_t)stream;
  const int u = (b * g.L + l) * g.Hkv + kvh;
  UnitDesc dsc;
  if (!check_cuda(cudaMemcpyAsync(&dsc, c->desc + u, sizeof(dsc), cudaMemcpyDeviceToHost, s))) return ARKV_ERR_CUDA;
  if (!check_cuda(cudaStreamSynchronize(s))) return ARKV_ERR_CUDA;
  std::vector<uint8_t> slot(g.slot_bytes), meta(g.meta_bytes);
  if (!check_cuda(cudaMemcpyAsync(slot.data(), c->slots + (int64_t)dsc.slot * g.slot_bytes, g.slot_bytes,
                                  cudaMemcpyDeviceToHost, s)))
    return ARKV_ERR_CUDA;
  if (!check_cuda(cudaMemcpyAsync(meta.data(), c->meta + (int64_t)dsc.slot * g.meta_bytes, g.meta_bytes,
                                  cudaMemcpyDeviceToHost, s)))
    return ARKV_ERR_CUDA;
  if (!check_cuda(cudaStreamSynchronize(s))) return ARKV_ERR_CUDA;
  SlotMeta sm = slot_meta(meta.data(), g, 0);
  const int n_pos = dsc.t_next;
  if (out->n_pos < n_pos) return ARKV_ERR_CAPACITY;
  out->n_o = dsc.n_o;
  out->n_q = dsc.n_q;
  const int d = g.d, ng = g.ng;
  const int off = g.mode == ARKV_QUANT_SYM ? (1 << (g.bits - 1)) : 0;
  if (out->state) {
    for (int p = 0; p < out->n_pos; ++p) out->state[p] = p < n_pos ? 3 : 0;
  }
  for (int r = 0; r < dsc.n_o; ++r) {
    const int p = sm.pos_o[r];
    if (p < 0 || p >= n_pos) return ARKV_ERR_DEVICE;
    if (out->state) out->state[p] = 1;
    const uint8_t* tb = o_tile_ptr(slot.data(), g, r / kTile);
    for (int x = 0; x < d; ++x) {
      if (out->o_k) out->o_k[(int64_t)p * d + x] = *(const uint16_t*)(tb + o_k_off(g, r % kTile, x));
      if (out->o_v) out->o_v[(int64_t)p * d + x] = *(const uint16_t*)(tb + o_v_off(g, r % kTile, x));
    }
  }
  for (int r = 0; r < dsc.n_q; ++r) {
    const int p = sm.pos_q[r];
    if (p < 0 || p >= n_pos) return ARKV_ERR_DEVICE;
    if (out->state) out->state[p] = 2;
    const uint8_t* tb = q_tile_ptr(slot.data(), g, r / kTile);
    const int j = r % kTile;
    for (int x = 0; x < d; ++x) {
      int byte, shift;
      q_k_loc(g, j, x, &byte, &shift);
      int ck = (int)((tb[byte] >> shift) & ((1u << g.bits) - 1u)) - off;
      q_v_loc(g, j, x, &byte, &shift);
      int cv = (int)((tb[byte] >> shift) & ((1u << g.bits) - 1u)) - off;
      if (out->q_k) out->q_k[(int64_t)p * d + x] = (int16_t)ck;
      if (out->q_v) out->q_v[(int64_t)p * d + x] = (int16_t)cv;
    }
    for (int gi = 0; gi < ng; ++gi) {
      if (out->k_scale) out->k_scale[(int64_t)p * ng + gi] = *(const float*)(tb + q_sc_off(g, j, 0, gi));
      if (out->k_zero) out->k_zero[(int64_t)p * ng + gi] = *(const float*)(tb + q_sc_off(g, j, 1, gi));
      if (out->v_scale) out->v_scale[(int64_t)p * ng + gi] = *(const float*)(tb + q_sc_off(g, j, 2, gi));
      if (out->v_zero) out->v_zero[(int64_t)p * ng + gi] = *(const float*)(tb + q_sc_off(g, j, 3, gi));
    }
  }
  return ARKV_OK;
}

arkv_status arkv_check(arkv_cache* c, void* stream) {
  if (!c) return ARKV_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (!check_cuda(cudaStreamSynchronize(s))) return ARKV_ERR_CUDA;
  int32_t e = 0;
  if (!check_cuda(cudaMemcpy(&e, c->err, 4, cudaMemcpyDeviceToHost))) return ARKV_ERR_CUDA;
  if (e) {
    cudaMemset(c->err, 0, 4);
    std::fprintf(stderr, "arkv: device error flag 0x%x\n", e);
    return ARKV_ERR_DEVICE;
  }
  return ARKV_OK;
}

}  // extern "C"
