// gpuar_api.cu -- libgpuar's C ABI (include/gpuar.h): handle, argument checks, launch
// policy (which kernel, grid, shared-memory budget), stream ordering, sticky errors and
// the host-buffer pipeline of gpuar_select_host.  No torch types anywhere: plain
// pointers and sizes.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/gpuar.h"
#include "gpuar_internal.cuh"

using namespace gpuar;

namespace {

constexpr int kRowsMaxWarps = 32;      // compiled variants: <=16, <=20, <=24, <=32 warps per CTA
constexpr int kRowsDefaultWarps = 24;   // r01 sweep: 24 warps x 2 slots -> 5.92 TB/s (16x3: 5.13)
constexpr size_t kHostChunkBytes = 64ull << 20;  // gpuar_select_host row-chunk size

struct Chunked {
  float* stage[2] = {nullptr, nullptr};
  size_t stage_floats = 0;
  int32_t* idx = nullptr;
  float* tau = nullptr;
  uint32_t* trials = nullptr;
  size_t out_cap = 0;
  float* vec = nullptr;
  size_t vec_cap = 0;
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr};
};

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  if (!v || !*v) return dflt;
  return std::atoi(v);
}

}  // namespace

struct gpuar_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t M = 0, Kcap = 0;
  uint64_t seed = 0;
  uint32_t epoch = 0;
  uint64_t offset = 0;
  uint32_t max_trials = GPUAR_DEFAULT_MAX_TRIALS;
  // registration
  const float* alpha = nullptr;
  int64_t rows = 0, ld = 0;
  int path = kPathNone;
  // device scratch
  DevStats* d_stats = nullptr;
  DevCounters* d_ctr = nullptr;
  uint32_t ticket_phase = 0;  // DevCounters::next set of the next shared-vector launch
  uint32_t grab_override = 0; // tuning knobs, read from the environment once at create time
  uint32_t team_override = 0;
  bool pdl = true;            // programmatic dependent launch of the shared-vector kernels
  uint32_t no_prefetch = 0;
  uint32_t no_endgame = 0;
  double* d_part_sum = nullptr;
  uint32_t* d_part_max = nullptr;
  int stats_blocks = 1;
  uint16_t* d_pref = nullptr;
  uint32_t* d_thr = nullptr;  // classic-rule acceptance thresholds T_j of the shared vector
  uint32_t n_pref = 0, group_shift = 0;
  int shared_path = kPathSmemF32;  // which shared-vector path M implies
  uint32_t shared_smem = 0;
  // device properties
  int num_sms = 148;
  int smem_optin = 227 * 1024;
  // rows policy
  int rows_warps = 0, rows_stages = 0, rows_grid = 0, rows_lb = 3;
  uint32_t stage_bytes = 0;
  // shared policy
  int sh_block = 256, sh_grid = 0;
  // selection rule (gpuar_set_rule)
  int rule = kRuleClassic;
  float w = 1.0f;
  int am_grid = 0;
  bool am_smem = true;
  // SSA network (gpuar_set_network), borrowed device pointers
  const int32_t* net_reac = nullptr;
  const float* net_rate = nullptr;
  const int32_t* net_didx = nullptr;
  const int32_t* net_dval = nullptr;
  int64_t net_N = 0, net_D = 0;
  int ssa_warps = 0, ssa_grid = 0;
  int32_t* d_dep_ptr = nullptr;  // dependency lists of the registered network (handle-owned)
  int32_t* d_dep_idx = nullptr;
  uint32_t dep_total = 0;
  bool ssa_deps = false;
  // inverse transform (GPUAR_RULE_IT): sequential binary64 prefix sums of the shared vector
  double* d_prefix = nullptr;
  bool prefix_valid = false;
  uint32_t ssa_net_bytes = 0, ssa_warp_bytes = 0;
  Chunked host;
  cudaEvent_t order_ev = nullptr;  // orders a new stream after the old one (gpuar_set_stream)
};

namespace {

struct DeviceGuard {
  int dev;
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int d) : dev(d) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {  // restore only what was switched
    if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  }
};

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return GPUAR_OK;
  if (e == cudaErrorMemoryAllocation) return GPUAR_ENOMEM;
  return GPUAR_ECUDA;
}

// Which shared-vector path M implies, and its shared-memory footprint.
void plan_shared(gpuar_handle* h) {
  const uint64_t budget = (uint64_t)h->smem_optin - 1024u;
  const uint64_t M = (uint64_t)h->M;
  // staged by a bulk copy of the 16-byte hull: up to 16 bytes of slack
  if (4u * M + 16u <= budget) {
    h->shared_path = kPathSmemF32;
    h->n_pref = 0;
    h->group_shift = 0;
    h->shared_smem = (uint32_t)(((4u * M + 15u) & ~15ull) + 16u);
  } else if (2u * M + 16u <= budget) {
    h->shared_path = kPathSmemBf16;
    h->n_pref = (uint32_t)M;
    h->group_shift = 0;
    h->shared_smem = (uint32_t)(((2u * M + 15u) & ~15ull) + 16u);
  } else {
    uint32_t s = 1;
    while (2u * ((M + (1ull << s) - 1) >> s) + 16u > budget) ++s;
    h->shared_path = kPathSmemGroup;
    h->group_shift = s;
    h->n_pref = (uint32_t)((M + (1ull << s) - 1) >> s);
    h->shared_smem = (uint32_t)(((2u * h->n_pref + 15u) & ~15ull) + 16u);
  }
  // CTA size: the largest block whose resident threads per SM reach 3/4 of the best any size
  // gets.  Fewer, larger CTAs amortise the per-CTA set-up (staging, statistics, team choice,
  // barrier): 1 x 1024 threads beat 5 x 256 (the occupancy maximum at 48 registers) on every
  // smem-vector config, +4-7 % (session-2 sweep, GPUAR_SH_BLOCK).  GPUAR_SH_CTAS_PER_SM caps
  // the CTAs per SM, GPUAR_SH_BLOCK forces a size (tuning).
  const int cap = env_int("GPUAR_SH_CTAS_PER_SM", 0);
  const int force_block = env_int("GPUAR_SH_BLOCK", 0);
  int nb[3] = {0, 0, 0}, best_threads = 0;
  const int blocks[3] = {256, 512, 1024};
  for (int i = 0; i < 3; ++i) {
    if (force_block > 0 && blocks[i] != force_block) continue;
    int n = select_shared_blocks_per_sm(h->shared_path, blocks[i], h->shared_smem);
    if (cap > 0) n = std::min(n, cap);
    nb[i] = n;
    best_threads = std::max(best_threads, n * blocks[i]);
  }
  h->sh_grid = 0;
  for (int i = 2; i >= 0; --i) {
    if (nb[i] > 0 && 4 * nb[i] * blocks[i] >= 3 * best_threads) {
      h->sh_block = blocks[i];
      h->sh_grid = nb[i] * h->num_sms;
      break;
    }
  }
  if (h->sh_grid <= 0) {  // no size qualified (an unsupported GPUAR_SH_BLOCK, or the
    h->sh_block = 256;     // occupancy query failed): one 256-thread CTA per SM
    h->sh_grid = h->num_sms;
  }
}

// Rows ring: W warps x S slots of ceil16(4M) + 16 bytes (the 16-aligned cover of a row).
int plan_rows(gpuar_handle* h) {
  const uint64_t budget = (uint64_t)h->smem_optin - 1024u;
  const uint64_t sb = ((4ull * (uint64_t)h->M + 15ull) & ~15ull) + 16ull;
  int W = env_int("GPUAR_ROWS_WARPS", kRowsDefaultWarps);
  W = std::max(1, std::min(W, kRowsMaxWarps));
  int S = env_int("GPUAR_ROWS_STAGES", 0);    // 1, 2 or 4 (powers of two: slot by shift)
  auto fits = [&](int w, int s) { return (((uint64_t)w * s * 8u + 127u) & ~127ull) + (uint64_t)w * s * sb <= budget; };
  if (S != 1 && S != 2 && S != 4) {
    S = 4;
    while (S > 2 && !fits(W, S)) S >>= 1;
  }
  if (S > 1 && !fits(W, S) && W > 16) S = 1;   // many warps with no prefetch beat few with it
  while (W > 1 && !fits(W, S)) --W;
  if (!fits(W, S)) return GPUAR_EINVAL;  // M too large for the row pipeline
  h->rows_warps = W;
  h->rows_stages = S;
  h->rows_lb = std::max(0, std::min(5, env_int("GPUAR_ROWS_LOG2_BLOCK", 3)));  // B = 8 (r01 A/B)
  h->stage_bytes = (uint32_t)sb;
  const size_t sh = (((size_t)W * S * 8u + 127u) & ~(size_t)127u) + (size_t)W * S * sb;
  const int n = select_rows_blocks_per_sm(W, sh);
  if (n <= 0) return GPUAR_EINVAL;
  h->rows_grid = n * h->num_sms;
  return GPUAR_OK;
}

// n_epochs > 1 (gpuar_select_epochs; shared vector, classic rule only): one launch works the
// n_epochs * K items of n consecutive calls, outputs [n_epochs][K].
int launch_select(gpuar_handle* h, const float* alpha, int64_t rows, int64_t ld, int64_t K, uint64_t s0,
                  int32_t* idx, float* tau, uint32_t* trials, cudaStream_t st, uint32_t n_epochs = 1) {
  cudaError_t e;
  if (rows == 1) {
    SharedParams p{};
    p.alpha = alpha;
    p.thr = h->d_thr;
    p.prefilter = h->d_pref;
    p.stats = h->d_stats;
    p.ctr = h->d_ctr;
    p.idx = idx;
    p.tau = tau;
    p.trials = trials;
    p.M = (uint32_t)h->M;
    p.K = (uint32_t)(K * n_epochs);  // work items
    p.Ksel = (uint32_t)K;
    p.n_epochs = n_epochs;
    p.kinv = 1.0f / (float)K;
    p.s0 = (uint32_t)s0;
    p.epoch = h->epoch;
    p.seed_lo = (uint32_t)h->seed;
    p.seed_hi = (uint32_t)(h->seed >> 32);
    p.max_trials = h->max_trials;
    p.n_pref = h->n_pref;
    p.group_shift = h->group_shift;
    p.smem_bytes = h->shared_smem;
    p.w = h->w;
    p.grab_override = h->grab_override;
    p.team_override = h->team_override;
    p.no_prefetch = h->no_prefetch;
    p.no_endgame = h->no_endgame;
    if (h->rule == kRuleArgmin) {
      e = launch_argmin_shared(p, h->am_smem, h->am_grid, 256, st, h->pdl);
    } else if (h->rule == kRuleIT) {
      e = cudaSuccess;
      if (!h->d_prefix) e = cudaMalloc(&h->d_prefix, (sizeof(double) * (size_t)h->M + 15u) & ~(size_t)15);
      if (e == cudaSuccess && !h->prefix_valid) {
        e = launch_it_prefix(alpha, (uint32_t)h->M, h->d_prefix, st);
        h->prefix_valid = e == cudaSuccess;
      }
      const bool smem = (size_t)h->M * 8u + 1024u <= (size_t)h->smem_optin;
      if (e == cudaSuccess) e = launch_it_select(p, h->d_prefix, smem, h->num_sms * 8, st, h->pdl);
    } else {
      p.phase = h->ticket_phase;
      {
        const uint64_t nwarps = std::max<uint64_t>(1u, (uint64_t)h->sh_grid * (uint64_t)h->sh_block / 32u);
        const uint64_t Q = (uint64_t)K * n_epochs;
        const uint64_t fair = std::max<uint64_t>(1u, Q / nwarps);
        // static first chunk: 3/4 of the fair share (the device raises it to 15/16 at p > 1/4,
        // pool_setup).  A/B on one box against 1/2: c3 uniform +3 %, c3 exponential +0.7 %, the
        // rest +-0.6 %; with fewer items than threads select_shared_pre_kernel works it before
        // the PDL wait (c2 +1.6 %).  7/8 and 15/16 everywhere lost 3-8 % on the heavy tails.
        uint64_t first = fair * 3u / 4u;
        if (fair <= 4u) {
          const uint64_t stripe = (Q + kStripes - 1u) / kStripes;
          const uint64_t per = std::max<uint64_t>(1u, nwarps / kStripes);  // fewest warps any stripe has
          first = (stripe + per - 1u) / per;
        }
        p.fair = (uint32_t)fair;
        p.first_base = (uint32_t)first;
      }
      e = launch_select_shared(p, h->shared_path, h->sh_grid, h->sh_block, st, h->pdl);
      if (e == cudaSuccess) h->ticket_phase ^= 1u;
    }
  } else {
    RowsParams p{};
    p.alpha = alpha;
    p.ctr = h->d_ctr;
    p.idx = idx;
    p.tau = tau;
    p.trials = trials;
    p.ld = (uint64_t)ld;
    p.M = (uint32_t)h->M;
    p.K = (uint32_t)K;
    p.s0 = (uint32_t)s0;
    p.epoch = h->epoch;
    p.seed_lo = (uint32_t)h->seed;
    p.seed_hi = (uint32_t)(h->seed >> 32);
    p.max_trials = h->max_trials;
    p.log2_stages = h->rows_stages == 4 ? 2u : (h->rows_stages == 2 ? 1u : 0u);
    p.stage_bytes = h->stage_bytes;
    p.stats_only = 0;
    p.rule = h->rule;
    p.w = h->w;
    p.log2_block = (uint32_t)h->rows_lb;
    const int64_t per_cta = (int64_t)h->rows_warps << h->rows_lb;
    const int grid = (int)std::min<int64_t>(h->rows_grid, (K + per_cta - 1) / per_cta);
    e = launch_select_rows(p, std::max(grid, 1), h->rows_warps, st, h->pdl);
  }
  return cuda_status(e);
}

int check_err_flag(gpuar_handle* h) {
  unsigned int err = 0;
  cudaError_t e = cudaMemcpyAsync(&err, &h->d_ctr->err, sizeof(err), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_status(e);
  if (err) {
    e = cudaMemsetAsync(&h->d_ctr->err, 0, sizeof(unsigned int), h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    return e == cudaSuccess ? GPUAR_EPROPENSITY : cuda_status(e);
  }
  return GPUAR_OK;
}

int register_shared(gpuar_handle* h, const float* d_alpha) {
  if (!h->d_thr) {  // first shared vector of this handle: M acceptance thresholds
    const cudaError_t a = cudaMalloc(&h->d_thr, (sizeof(uint32_t) * (size_t)h->M + 15u) & ~(size_t)15);
    if (a != cudaSuccess) return cuda_status(a);
  }
  cudaError_t e = launch_stats(d_alpha, (uint32_t)h->M, h->d_part_sum, h->d_part_max, h->d_stats, h->d_ctr,
                               h->stats_blocks, h->stream, h->pdl);
  if (e == cudaSuccess)
    e = launch_thresholds(d_alpha, (uint32_t)h->M, h->d_stats, h->d_thr, h->d_pref, h->n_pref, h->group_shift,
                          h->shared_path, h->stream, h->pdl);
  if (e != cudaSuccess) return cuda_status(e);
  h->alpha = d_alpha;
  h->rows = 1;
  h->ld = h->M;
  h->path = h->shared_path;
  h->prefix_valid = false;
  return GPUAR_OK;
}

}  // namespace

extern "C" {

const char* gpuar_strerror(int status) {
  switch (status) {
    case GPUAR_OK: return "success";
    case GPUAR_EINVAL: return "invalid argument";
    case GPUAR_ENOMEM: return "out of memory";
    case GPUAR_ECUDA: return "CUDA error";
    case GPUAR_ENOTSET: return "propensities not set";
    case GPUAR_EPROPENSITY: return "invalid propensity (negative, -0.0, NaN or Inf)";
    default: return "unknown status";
  }
}

int gpuar_create(gpuar_t* out, int64_t M, int64_t K, uint64_t seed) {
  if (!out || M < 1 || M > 0x7fffffffll || K < 1 || K > 0xffffffffll) return GPUAR_EINVAL;
  gpuar_handle* h = new (std::nothrow) gpuar_handle();
  if (!h) return GPUAR_ENOMEM;
  if (cudaGetDevice(&h->device) != cudaSuccess) {
    delete h;
    return GPUAR_ECUDA;
  }
  h->M = M;
  h->Kcap = K;
  h->seed = seed;
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device);
  cudaDeviceGetAttribute(&h->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
  set_select_shared_limits(h->smem_optin);
  set_select_rows_limits(h->smem_optin);
  set_argmin_limits(h->smem_optin);
  set_ssa_limits(h->smem_optin);
  set_it_limits(h->smem_optin);
  {
    const size_t am_sh = (size_t)((M + 3) & ~3ll) * 8u;  // alpha and RN(1/alpha) in smem
    h->am_smem = am_sh + 1024u <= (size_t)h->smem_optin;
    // one resident wave of 256-thread CTAs (the selections are assigned statically per warp)
    h->am_grid = h->num_sms * std::max(1, argmin_blocks_per_sm(h->am_smem, h->am_smem ? am_sh : 0));
  }
  // stats launch shape depends on M only -> identical reduction tree on every rank
  h->stats_blocks = (int)std::min<int64_t>((M + 4095) / 4096, 512);
  plan_shared(h);
  h->grab_override = (uint32_t)std::max(0, env_int("GPUAR_GRAB", 0));
  {
    const int g = env_int("GPUAR_TEAM", 0);  // 1, 2, 4, ..., 32 (else the model decides)
    h->team_override = (g >= 1 && g <= 32 && (g & (g - 1)) == 0) ? (uint32_t)g : 0u;
  }
  h->no_prefetch = (uint32_t)std::max(0, env_int("GPUAR_NO_PREFETCH", 0));
  h->no_endgame = (uint32_t)std::max(0, env_int("GPUAR_NO_ENDGAME", 0));
  h->pdl = env_int("GPUAR_NO_PDL", 0) == 0;
  cudaError_t e = cudaMalloc(&h->d_stats, sizeof(DevStats));
  if (e == cudaSuccess) e = cudaMalloc(&h->d_ctr, sizeof(DevCounters));
  if (e == cudaSuccess) e = cudaMalloc(&h->d_part_sum, sizeof(double) * h->stats_blocks);
  if (e == cudaSuccess) e = cudaMalloc(&h->d_part_max, sizeof(uint32_t) * h->stats_blocks);
  if (e == cudaSuccess && h->n_pref) e = cudaMalloc(&h->d_pref, (sizeof(uint16_t) * h->n_pref + 15u) & ~(size_t)15);
  if (e == cudaSuccess) e = cudaMemset(h->d_ctr, 0, sizeof(DevCounters));
  if (e == cudaSuccess) e = cudaMemset(h->d_stats, 0, sizeof(DevStats));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    gpuar_destroy(h);
    return cuda_status(e);
  }
  *out = h;
  return GPUAR_OK;
}

int gpuar_destroy(gpuar_t h) {
  if (!h) return GPUAR_OK;
  DeviceGuard g(h->device);
  cudaError_t e = cudaStreamSynchronize(h->stream);
  Chunked& c = h->host;
  if (c.s_in) cudaStreamSynchronize(c.s_in);
  if (c.s_out) cudaStreamSynchronize(c.s_out);
  for (int i = 0; i < 2; ++i) {
    cudaFree(c.stage[i]);
    if (c.ev_in[i]) cudaEventDestroy(c.ev_in[i]);
    if (c.ev_comp[i]) cudaEventDestroy(c.ev_comp[i]);
  }
  cudaFree(c.idx);
  cudaFree(c.tau);
  cudaFree(c.trials);
  cudaFree(c.vec);
  if (c.s_in) cudaStreamDestroy(c.s_in);
  if (c.s_out) cudaStreamDestroy(c.s_out);
  cudaFree(h->d_stats);
  cudaFree(h->d_ctr);
  cudaFree(h->d_part_sum);
  cudaFree(h->d_part_max);
  cudaFree(h->d_pref);
  cudaFree(h->d_thr);
  cudaFree(h->d_prefix);
  if (h->order_ev) cudaEventDestroy(h->order_ev);
  cudaFree(h->d_dep_ptr);
  cudaFree(h->d_dep_idx);
  delete h;
  return e == cudaSuccess ? GPUAR_OK : GPUAR_ECUDA;
}

int gpuar_set_stream(gpuar_t h, void* stream) {
  if (!h) return GPUAR_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (s == h->stream) return GPUAR_OK;
  // The handle's device scratch (work-stealing tickets, statistics) is shared by all its
  // launches: order the new stream after everything already queued on the old one.
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  if (!h->order_ev) {
    cudaError_t e = cudaEventCreateWithFlags(&h->order_ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_status(e);
  }
  cudaError_t e = cudaEventRecord(h->order_ev, h->stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, h->order_ev, 0);
  if (e != cudaSuccess) return cuda_status(e);
  h->stream = s;
  return GPUAR_OK;
}

int gpuar_set_propensities(gpuar_t h, const float* d_alpha, int64_t rows, int64_t ld) {
  if (!h || !d_alpha) return GPUAR_EINVAL;
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  if (rows == 1) return register_shared(h, d_alpha);
  if (rows < 1 || rows > h->Kcap || ld < h->M) return GPUAR_EINVAL;
  if ((reinterpret_cast<uintptr_t>(d_alpha) & 15u) != 0) return GPUAR_EINVAL;
  if (h->rows_warps == 0) {
    const int st = plan_rows(h);
    if (st != GPUAR_OK) return st;
  }
  h->alpha = d_alpha;
  h->rows = rows;
  h->ld = ld;
  h->path = kPathRows;
  return GPUAR_OK;
}

int gpuar_select(gpuar_t h, int64_t K, int32_t* d_idx, float* d_tau, uint32_t* d_trials) {
  if (!h || !d_idx || K < 1 || K > h->Kcap) return GPUAR_EINVAL;
  if (h->path == kPathNone) return GPUAR_ENOTSET;
  if (h->rows != 1 && K != h->rows) return GPUAR_EINVAL;
  if (h->rows == 1 && h->rule == kRuleITScan) return GPUAR_EINVAL;  // IT linear scan: matrix only
  if (h->offset + (uint64_t)K > (1ull << 32)) return GPUAR_EINVAL;
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  const int st = launch_select(h, h->alpha, h->rows, h->ld, K, h->offset, d_idx, d_tau, d_trials, h->stream);
  if (st == GPUAR_OK) ++h->epoch;
  return st;
}

int gpuar_select_epochs(gpuar_t h, int64_t K, int64_t n_epochs, int32_t* d_idx, float* d_tau, uint32_t* d_trials) {
  if (!h || !d_idx || K < 1 || K > h->Kcap || n_epochs < 1 || n_epochs > 65536) return GPUAR_EINVAL;
  if ((uint64_t)K * (uint64_t)n_epochs > 0xffffffffull) return GPUAR_EINVAL;
  if (h->path == kPathNone) return GPUAR_ENOTSET;
  if (h->rows != 1 && K != h->rows) return GPUAR_EINVAL;
  if (h->rows == 1 && h->rule == kRuleITScan) return GPUAR_EINVAL;
  if (h->offset + (uint64_t)K > (1ull << 32)) return GPUAR_EINVAL;
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  if (h->rows == 1 && h->rule == kRuleClassic && n_epochs > 1) {
    // one launch for all epochs: the fixed cost of a launch (ramp, staging, drain) is paid once
    const int st = launch_select(h, h->alpha, 1, h->ld, K, h->offset, d_idx, d_tau, d_trials, h->stream,
                                 (uint32_t)n_epochs);
    if (st == GPUAR_OK) h->epoch += (uint32_t)n_epochs;
    return st;
  }
  for (int64_t e = 0; e < n_epochs; ++e) {  // other rules and the matrix: one launch per epoch
    const int st = launch_select(h, h->alpha, h->rows, h->ld, K, h->offset, d_idx + e * K,
                                 d_tau ? d_tau + e * K : nullptr, d_trials ? d_trials + e * K : nullptr, h->stream);
    if (st != GPUAR_OK) return st;
    ++h->epoch;
  }
  return GPUAR_OK;
}

int gpuar_select_host(gpuar_t h, const float* h_alpha, int64_t rows, int64_t ld, int64_t K, int32_t* h_idx,
                      float* h_tau, uint32_t* h_trials) {
  if (!h || !h_alpha || !h_idx || !h_tau || !h_trials || K < 1 || K > h->Kcap) return GPUAR_EINVAL;
  if (!(rows == 1 || rows == K)) return GPUAR_EINVAL;
  if (rows != 1 && ld < h->M) return GPUAR_EINVAL;
  if (rows == 1 && h->rule == kRuleITScan) return GPUAR_EINVAL;  // IT linear scan: matrix only
  if (h->offset + (uint64_t)K > (1ull << 32)) return GPUAR_EINVAL;
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  Chunked& c = h->host;
  cudaError_t e = cudaSuccess;
  if (!c.s_in) {
    e = cudaStreamCreateWithFlags(&c.s_in, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c.s_out, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&c.ev_in[i], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_comp[i], cudaEventDisableTiming);
    }
    if (e != cudaSuccess) return cuda_status(e);
  }
  if (c.out_cap < (size_t)K) {
    cudaFree(c.idx);
    cudaFree(c.tau);
    cudaFree(c.trials);
    c.idx = nullptr;
    c.tau = nullptr;
    c.trials = nullptr;
    c.out_cap = 0;
    e = cudaMalloc(&c.idx, 4 * K);
    if (e == cudaSuccess) e = cudaMalloc(&c.tau, 4 * K);
    if (e == cudaSuccess) e = cudaMalloc(&c.trials, 4 * K);
    if (e != cudaSuccess) return cuda_status(e);
    c.out_cap = (size_t)K;
  }
  int st = GPUAR_OK;
  if (rows == 1) {
    // shared vector: H2D of M floats, stats, select, D2H of the outputs
    if (c.vec_cap < (size_t)h->M) {
      cudaFree(c.vec);
      c.vec = nullptr;
      c.vec_cap = 0;
      e = cudaMalloc(&c.vec, 4 * h->M);
      if (e != cudaSuccess) return cuda_status(e);
      c.vec_cap = (size_t)h->M;
    }
    e = cudaMemcpyAsync(c.vec, h_alpha, 4 * h->M, cudaMemcpyHostToDevice, h->stream);
    if (e != cudaSuccess) return cuda_status(e);
    st = register_shared(h, c.vec);
    if (st == GPUAR_OK) st = launch_select(h, c.vec, 1, h->M, K, h->offset, c.idx, c.tau, c.trials, h->stream);
    if (st != GPUAR_OK) return st;
    e = cudaMemcpyAsync(h_idx, c.idx, 4 * K, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_tau, c.tau, 4 * K, cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_trials, c.trials, 4 * K, cudaMemcpyDeviceToHost, h->stream);
    if (e != cudaSuccess) return cuda_status(e);
  } else {
    if (h->rows_warps == 0) {
      st = plan_rows(h);
      if (st != GPUAR_OK) return st;
    }
    const int64_t R = std::max<int64_t>(1, std::min<int64_t>(K, (int64_t)(kHostChunkBytes / (4 * (size_t)ld))));
    if (c.stage_floats < (size_t)(R * ld)) {
      for (int i = 0; i < 2; ++i) {
        cudaFree(c.stage[i]);
        c.stage[i] = nullptr;
      }
      c.stage_floats = 0;
      for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaMalloc(&c.stage[i], 4 * (size_t)R * ld);
      if (e != cudaSuccess) return cuda_status(e);
      c.stage_floats = (size_t)(R * ld);
    }
    // make the side streams start after everything already queued on the handle's stream
    cudaEvent_t start = c.ev_comp[1];
    e = cudaEventRecord(start, h->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.s_in, start, 0);
    const int64_t nchunks = (K + R - 1) / R;
    for (int64_t i = 0; i < nchunks && e == cudaSuccess; ++i) {
      const int b = (int)(i & 1);
      const int64_t r0 = i * R;
      const int64_t nr = std::min<int64_t>(R, K - r0);
      if (i >= 2) e = cudaStreamWaitEvent(c.s_in, c.ev_comp[b], 0);  // slot free
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(c.stage[b], h_alpha + r0 * ld, 4 * (size_t)nr * ld, cudaMemcpyHostToDevice, c.s_in);
      if (e == cudaSuccess) e = cudaEventRecord(c.ev_in[b], c.s_in);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(h->stream, c.ev_in[b], 0);
      if (e != cudaSuccess) break;
      st = launch_select(h, c.stage[b], nr, ld, nr, h->offset + r0, c.idx + r0, c.tau + r0, c.trials + r0,
                         h->stream);
      if (st != GPUAR_OK) return st;
      e = cudaEventRecord(c.ev_comp[b], h->stream);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(c.s_out, c.ev_comp[b], 0);
      if (e == cudaSuccess) e = cudaMemcpyAsync(h_idx + r0, c.idx + r0, 4 * nr, cudaMemcpyDeviceToHost, c.s_out);
      if (e == cudaSuccess) e = cudaMemcpyAsync(h_tau + r0, c.tau + r0, 4 * nr, cudaMemcpyDeviceToHost, c.s_out);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(h_trials + r0, c.trials + r0, 4 * nr, cudaMemcpyDeviceToHost, c.s_out);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.s_out);
    if (e != cudaSuccess) return cuda_status(e);
    h->alpha = nullptr;
    h->path = kPathNone;
    h->rows = 0;
  }
  ++h->epoch;
  return check_err_flag(h);
}

int gpuar_set_rule(gpuar_t h, int rule, float w) {
  if (!h) return GPUAR_EINVAL;
  if (rule == GPUAR_RULE_CLASSIC || rule == GPUAR_RULE_IT || rule == GPUAR_RULE_IT_SCAN) {
    if (w != 1.0f) return GPUAR_EINVAL;
  } else if (rule == GPUAR_RULE_ARGMIN) {
    if (!(w >= 1.0f) || !std::isfinite(w)) return GPUAR_EINVAL;
  } else {
    return GPUAR_EINVAL;
  }
  h->rule = rule;
  h->w = w;
  return GPUAR_OK;
}

int gpuar_set_network(gpuar_t h, int64_t N, int64_t D, const int32_t* d_reac, const float* d_rate,
                      const int32_t* d_didx, const int32_t* d_dval) {
  if (!h || !d_reac || !d_rate || !d_didx || !d_dval || N < 1 || N > 0x7fffffffll || D < 1 || D > 32)
    return GPUAR_EINVAL;
  const uint64_t M = (uint64_t)h->M;
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  // Dependency lists (host, once per network): reaction j changes species S_j; the
  // propensities to refresh after j fires are the reactions with a reactant in S_j.
  std::vector<int32_t> reac(2 * M), didx(M * D), dval(M * D);
  cudaError_t e = cudaMemcpy(reac.data(), d_reac, 8 * M, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(didx.data(), d_didx, 4 * M * D, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(dval.data(), d_dval, 4 * M * D, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e);
  std::vector<std::vector<int32_t>> users((size_t)N);
  for (uint64_t j = 0; j < M; ++j) {
    const int32_t r0 = reac[2 * j], r1 = reac[2 * j + 1];
    if (r0 >= N || r1 >= N) return GPUAR_EINVAL;
    if (r0 >= 0) users[r0].push_back((int32_t)j);
    if (r1 >= 0 && r1 != r0) users[r1].push_back((int32_t)j);
  }
  std::vector<int32_t> ptr(M + 1, 0), idx;
  std::vector<char> mark(M, 0);
  for (uint64_t j = 0; j < M; ++j) {
    std::vector<int32_t> dep;
    for (int64_t d = 0; d < D; ++d) {
      const int32_t sp = didx[j * D + d];
      if (sp >= N) return GPUAR_EINVAL;
      if (sp < 0 || dval[j * D + d] == 0) continue;
      for (int32_t r : users[sp])
        if (!mark[r]) {
          mark[r] = 1;
          dep.push_back(r);
        }
    }
    std::sort(dep.begin(), dep.end());
    for (int32_t r : dep) mark[r] = 0;
    idx.insert(idx.end(), dep.begin(), dep.end());
    ptr[j + 1] = (int32_t)idx.size();
  }
  const uint64_t net0 = ((M * (16u + 8u * (uint64_t)D)) + 15u) & ~15ull;  // int4 descriptors + didx/dval
  const uint64_t dep_bytes = ((4u * (M + 1u + idx.size())) + 15u) & ~15ull;
  const uint64_t per_warp = ((4u * M + 15u) & ~15ull) + ((4u * ((uint64_t)N + 1u) + 15u) & ~15ull);
  const uint64_t budget = (uint64_t)h->smem_optin - 1024u;
  if (net0 + per_warp > budget) return GPUAR_EINVAL;  // network + one realization must fit on chip
  // keep the dependency lists on chip if at least 8 warps still fit, else recompute every step
  const bool deps = net0 + dep_bytes + 8u * per_warp <= budget;
  const uint64_t net = net0 + (deps ? dep_bytes : 0u);
  int W = (int)std::min<uint64_t>(24, (budget - net) / per_warp);
  const size_t sh = (size_t)net + (size_t)W * per_warp;
  cudaFree(h->d_dep_ptr);
  cudaFree(h->d_dep_idx);
  h->d_dep_ptr = h->d_dep_idx = nullptr;
  h->dep_total = 0;
  if (deps) {
    e = cudaMalloc(&h->d_dep_ptr, 4 * (M + 1));
    if (e == cudaSuccess) e = cudaMalloc(&h->d_dep_idx, 4 * std::max<size_t>(1, idx.size()));
    if (e == cudaSuccess) e = cudaMemcpy(h->d_dep_ptr, ptr.data(), 4 * (M + 1), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !idx.empty())
      e = cudaMemcpy(h->d_dep_idx, idx.data(), 4 * idx.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_status(e);
    h->dep_total = (uint32_t)idx.size();
  }
  h->ssa_deps = deps;
  const int n = ssa_blocks_per_sm(W, sh);
  if (n <= 0) return GPUAR_EINVAL;
  h->net_reac = d_reac;
  h->net_rate = d_rate;
  h->net_didx = d_didx;
  h->net_dval = d_dval;
  h->net_N = N;
  h->net_D = D;
  h->ssa_warps = W;
  h->ssa_grid = n * h->num_sms;
  h->ssa_net_bytes = (uint32_t)net;
  h->ssa_warp_bytes = (uint32_t)per_warp;
  return GPUAR_OK;
}

int gpuar_ssa_run(gpuar_t h, int32_t* d_X, double* d_t, uint32_t* d_steps, int64_t K, int32_t n_steps, double t_end) {
  if (!h || !d_X || !d_t || K < 1 || K > h->Kcap || n_steps < 0) return GPUAR_EINVAL;
  if (!h->net_reac) return GPUAR_ENOTSET;
  if (h->offset + (uint64_t)K > (1ull << 32)) return GPUAR_EINVAL;
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  SsaParams p{};
  p.reac = h->net_reac;
  p.rate = h->net_rate;
  p.didx = h->net_didx;
  p.dval = h->net_dval;
  p.X = d_X;
  p.t = d_t;
  p.steps = d_steps;
  p.ctr = h->d_ctr;
  p.t_end = t_end;
  p.N = (uint32_t)h->net_N;
  p.M = (uint32_t)h->M;
  p.D = (uint32_t)h->net_D;
  p.K = (uint32_t)K;
  p.s0 = (uint32_t)h->offset;
  p.epoch0 = h->epoch;
  p.seed_lo = (uint32_t)h->seed;
  p.seed_hi = (uint32_t)(h->seed >> 32);
  p.max_trials = h->max_trials;
  p.n_steps = n_steps;
  p.net_bytes = h->ssa_net_bytes;
  p.warp_bytes = h->ssa_warp_bytes;
  p.dep_ptr = h->ssa_deps ? h->d_dep_ptr : nullptr;
  p.dep_idx = h->ssa_deps ? h->d_dep_idx : nullptr;
  p.dep_total = h->dep_total;
  const int grid = (int)std::min<int64_t>(h->ssa_grid, (K + h->ssa_warps - 1) / h->ssa_warps);
  const int st = cuda_status(launch_ssa(p, std::max(grid, 1), h->ssa_warps, h->stream));
  if (st == GPUAR_OK) h->epoch += (uint32_t)n_steps;
  return st;
}

int gpuar_set_selection_offset(gpuar_t h, int64_t s0) {
  if (!h || s0 < 0 || s0 > 0xffffffffll) return GPUAR_EINVAL;
  h->offset = (uint64_t)s0;
  return GPUAR_OK;
}

int gpuar_set_epoch(gpuar_t h, uint32_t epoch) {
  if (!h) return GPUAR_EINVAL;
  h->epoch = epoch;
  return GPUAR_OK;
}

int gpuar_get_epoch(gpuar_t h, uint32_t* epoch) {
  if (!h || !epoch) return GPUAR_EINVAL;
  *epoch = h->epoch;
  return GPUAR_OK;
}

int gpuar_set_max_trials(gpuar_t h, uint32_t n) {
  if (!h || n == 0) return GPUAR_EINVAL;
  h->max_trials = n;
  return GPUAR_OK;
}

int gpuar_get_stats(gpuar_t h, float* amax, double* a0, float* p) {
  if (!h) return GPUAR_EINVAL;
  if (h->path == kPathNone || h->rows != 1) return GPUAR_ENOTSET;
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  DevStats s;
  cudaError_t e = cudaMemcpyAsync(&s, h->d_stats, sizeof(s), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_status(e);
  const int st = check_err_flag(h);
  if (st != GPUAR_OK) return st;
  if (!s.valid) return GPUAR_EPROPENSITY;
  float am;
  std::memcpy(&am, &s.amax_bits, 4);
  if (amax) *amax = am;
  if (a0) *a0 = s.a0d;
  if (p) *p = s.p;
  return GPUAR_OK;
}

int gpuar_row_stats(gpuar_t h, float* d_amax, double* d_a0) {
  if (!h || !d_amax || !d_a0) return GPUAR_EINVAL;
  if (h->path != kPathRows) return GPUAR_ENOTSET;
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  RowsParams p{};
  p.alpha = h->alpha;
  p.ctr = h->d_ctr;
  p.amax_out = d_amax;
  p.a0_out = d_a0;
  p.ld = (uint64_t)h->ld;
  p.M = (uint32_t)h->M;
  p.K = (uint32_t)h->rows;
  p.max_trials = h->max_trials;
  p.log2_stages = h->rows_stages == 4 ? 2u : (h->rows_stages == 2 ? 1u : 0u);
  p.stage_bytes = h->stage_bytes;
  p.stats_only = 1;
  p.log2_block = (uint32_t)h->rows_lb;
  const int64_t per_cta = (int64_t)h->rows_warps << h->rows_lb;
  const int grid = (int)std::min<int64_t>(h->rows_grid, (h->rows + per_cta - 1) / per_cta);
  return cuda_status(launch_select_rows(p, std::max(grid, 1), h->rows_warps, h->stream, h->pdl));
}

int gpuar_sync(gpuar_t h) {
  if (!h) return GPUAR_EINVAL;
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  cudaError_t e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_status(e);
  return check_err_flag(h);
}

int gpuar_histogram(gpuar_t h, const int32_t* d_idx, const uint32_t* d_trials, int64_t K, uint64_t* d_hist,
                    uint64_t* d_totals) {
  if (!h || !d_idx || !d_hist || !d_totals || K < 1 || K > 0xffffffffll) return GPUAR_EINVAL;
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  return cuda_status(launch_histogram(d_idx, d_trials, (uint32_t)K, (uint32_t)h->M,
                                      reinterpret_cast<unsigned long long*>(d_hist),
                                      reinterpret_cast<unsigned long long*>(d_totals), h->num_sms * 4, h->stream));
}

int gpuar_bench_philox(gpuar_t h, int64_t n_threads, int32_t calls, uint32_t* d_sink) {
  if (!h || !d_sink || n_threads < 1 || n_threads > 0x7fffffffll || calls < 1) return GPUAR_EINVAL;
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  return cuda_status(launch_bench_philox((uint32_t)n_threads, (uint32_t)calls, (uint32_t)h->seed,
                                         (uint32_t)(h->seed >> 32), d_sink, h->stream));
}

int gpuar_last_team(gpuar_t h, int32_t* team) {
  if (!h || !team) return GPUAR_EINVAL;
  DeviceGuard g(h->device);
  if (!g.ok) return GPUAR_ECUDA;
  unsigned int t = 0;
  cudaError_t e = cudaMemcpyAsync(&t, &h->d_ctr->team, sizeof(t), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_status(e);
  *team = (int32_t)t;
  return GPUAR_OK;
}

int gpuar_path(gpuar_t h, int32_t* path) {
  if (!h || !path) return GPUAR_EINVAL;
  *path = h->path;
  return GPUAR_OK;
}

}  // extern "C"
