// Checkpointing configuration (NEXT-4): the wasted-time model and its optimum, §4.3
// "Optimizing Checkpointing Configuration" and the optimal configuration
// module.  Host arithmetic only, in double.  All time quantities share one
// unit (R-27 reads the model in iterations: f = full checkpoints per iteration, so the
// full-checkpoint interval FCF = 1/f iterations; b = differentials per batched write).
#include <cmath>

#include "../../include/lowdiff.h"

namespace {
bool valid(const lowdiff_sys_params* p) {
  return p && p->N > 0 && p->M > 0 && p->W > 0 && p->S > 0 && p->T > 0 && p->R_F >= 0 && p->R_D > 0;
}
}  // namespace

extern "C" {

// Eq. 3:
//   T_wasted = (N T / M) (b/2 + R_F + R_D/2 (1/(f b) - 1)) + N T S f / W
// The model needs f b <= 1 (a batch never spans more than one full-checkpoint interval; otherwise
// the merge-count term R_D/2 (1/(f b) - 1) would be negative): f b > 1 is E_INVALID.
lowdiff_status lowdiff_wasted_time(const lowdiff_sys_params* p, double f, double b, double* out) {
  if (!valid(p) || !out || !(f > 0) || !(b > 0) || f * b > 1.0) return LOWDIFF_E_INVALID;
  const double failures = p->N * p->T / p->M;                      // N x (T / M)
  const double recovery = b / 2.0 + p->R_F + p->R_D / 2.0 * (1.0 / (f * b) - 1.0);
  const double steady = p->N * p->T * p->S * f / p->W;              // N x (S / W) x f T
  *out = failures * recovery + steady;
  return LOWDIFF_OK;
}

// Eq. 5, from the first-order conditions of Eq. 4:
//   f* = cbrt(R_D W^2 / (4 S^2 M^2)),   b* = cbrt(2 S R_D M / W)
lowdiff_status lowdiff_optimal_config(const lowdiff_sys_params* p, double* f_star, double* b_star) {
  if (!valid(p) || !f_star || !b_star) return LOWDIFF_E_INVALID;
  *f_star = std::cbrt(p->R_D * p->W * p->W / (4.0 * p->S * p->S * p->M * p->M));
  *b_star = std::cbrt(2.0 * p->S * p->R_D * p->M / p->W);
  return LOWDIFF_OK;
}

// Eq. 5 restricted to the model's domain f b <= 1.  When the stationary point lies outside it,
// Eq. 3 is minimised on the boundary f b = 1, where the merge term vanishes:
//   T(f, 1/f) = (N T / M)(1/(2 f) + R_F) + N T S f / W  ->  f_c = sqrt(W / (2 M S)), b_c = 1 / f_c.
lowdiff_status lowdiff_optimal_config_feasible(const lowdiff_sys_params* p, double* f_opt, double* b_opt,
                                               double* f_unc, double* b_unc, int32_t* clamped) {
  if (!valid(p) || !f_opt || !b_opt) return LOWDIFF_E_INVALID;
  double fs, bs;
  lowdiff_optimal_config(p, &fs, &bs);
  if (f_unc) *f_unc = fs;
  if (b_unc) *b_unc = bs;
  const bool out = fs * bs > 1.0;
  if (clamped) *clamped = out ? 1 : 0;
  if (!out) {
    *f_opt = fs;
    *b_opt = bs;
  } else {
    *f_opt = std::sqrt(p->W / (2.0 * p->M * p->S));
    *b_opt = 1.0 / *f_opt;
  }
  return LOWDIFF_OK;
}

// Stepwise runtime adaptation: move the integer configuration (full-checkpoint
// interval in iterations, batch size) one step toward the rounded Eq. 5 optimum for the current
// parameter estimates -- one iteration of FCF change per 10% of distance (at least 1), one batch
// step -- but only while the step lowers Eq. 3.
lowdiff_status lowdiff_config_step(const lowdiff_sys_params* p, int64_t* fcf, int32_t* batch) {
  if (!valid(p) || !fcf || !batch || *fcf < 1 || *batch < 1) return LOWDIFF_E_INVALID;
  if (*batch > *fcf) return LOWDIFF_E_INVALID;   // f b <= 1: the batch fits the full interval
  double fs, bs;
  lowdiff_optimal_config_feasible(p, &fs, &bs, nullptr, nullptr, nullptr);
  const int64_t fcf_t = std::llround(std::fmax(1.0, 1.0 / fs));
  const int32_t b_t = (int32_t)std::lround(std::fmax(1.0, bs));
  int64_t nf = *fcf;
  if (nf != fcf_t) {
    const int64_t d = fcf_t - nf, mag = d > 0 ? d : -d;
    const int64_t stp = mag / 10 > 0 ? mag / 10 : 1;
    nf += d > 0 ? stp : -stp;
  }
  int32_t nb = *batch + (b_t > *batch ? 1 : (b_t < *batch ? -1 : 0));
  if (nb > nf) nb = (int32_t)nf;   // stay inside f b <= 1
  double cur, nxt;
  lowdiff_wasted_time(p, 1.0 / (double)*fcf, (double)*batch, &cur);
  lowdiff_wasted_time(p, 1.0 / (double)nf, (double)nb, &nxt);
  if (nxt <= cur) { *fcf = nf; *batch = nb; }
  return LOWDIFF_OK;
}

// Failure-injection simulator: one pass over a Poisson failure process of rate N / M
// (the N GPUs, each with mean time between failures M) over the productive time [0, T), charging
// every failure with the wasted time Alg. 1's recovery implies for the configuration (f, b):
// hardware -> lost work since the last persisted batch + R_F + R_D per persisted batch since the
// last full checkpoint; software (LowDiff+) -> R_S for restoring the CPU replica.
// Random numbers: splitmix64 over a counter, inter-arrival then kind per event.
namespace {
struct SplitMix {
  uint64_t seed, i = 0;
  double next() {
    uint64_t z = seed + (++i) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * 0x1p-53;
  }
};
}  // namespace

lowdiff_status lowdiff_simulate_failures(const lowdiff_sys_params* p, double f, double b, double sw_fraction,
                                         double R_S, uint64_t seed, lowdiff_sim_report* out) {
  if (!valid(p) || !out || !(f > 0) || !(b > 0) || f * b > 1.0 || !(sw_fraction >= 0 && sw_fraction <= 1) ||
      !(R_S >= 0))
    return LOWDIFF_E_INVALID;
  SplitMix rng{seed};
  const double mean_gap = p->M / p->N, interval = 1.0 / f;
  lowdiff_sim_report r{};
  double now = 0.0;
  for (;;) {
    now += -std::log1p(-rng.next()) * mean_gap;
    const bool sw = rng.next() < sw_fraction;
    if (now >= p->T) break;
    r.failures += 1;
    if (sw) {
      r.recovery += R_S;
    } else {
      r.hw_failures += 1;
      const double since_full = std::fmod(now, interval);
      r.lost_work += std::fmod(since_full, b);
      r.recovery += p->R_F + p->R_D * std::floor(since_full / b);
    }
  }
  r.steady = p->N * (p->S / p->W) * std::floor(f * p->T);
  r.wasted = r.lost_work + r.recovery + r.steady;
  r.effective_ratio = p->T / (p->T + r.wasted);
  *out = r;
  return LOWDIFF_OK;
}

}  // extern "C"
