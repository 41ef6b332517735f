/*
 * gpuar.h -- C ABI of libgpuar: GPU acceptance-rejection (GPU-AR) selection of the K
 * next reactions of K independent Gillespie SSA realizations on NVIDIA B200 (sm_100a).
 *
 * Method: arXiv 1404.0027 (Neri & Mestivier 2014).  Citations are to
 * /root/reference/PAPER.md line numbers (section in parentheses); DESIGN.md Rn are the
 * readings of the paper this library implements.
 *
 * Selection s (global index s_g = offset + s) draws trials i = 0, 1, 2, ...: a candidate
 * reaction j uniform on [0, M) and a uniform u in [0, 1), and accepts the first trial
 * with fl32(u * alpha_max) < alpha_j (§Methods "A GPU
 * acceptance-rejection algorithm", with the threshold T = alpha_max of PAPER.md:361-365).
 * The time step is tau = ln(1/u1) / alpha_0 (§Methods "The SSA").
 * Random bits come from Philox4x32-10 with counter {i>>1, s_g, epoch, 0} and key
 * {seed lo32, seed hi32}; trial i uses words (x0,x1) for even i and (x2,x3) for odd i;
 * j = (x_a * M) >> 32, u = (x_b >> 8) * 2^-24.  tau uses counter {0, s_g, epoch, 1}:
 * u1 = (2*(x0 >> 9) + 1) * 2^-24, tau = -logf(u1) / fl32(alpha_0).  Outputs are a pure
 * function of (alpha, seed, epoch, s_g, max_trials): independent of launch geometry,
 * GPU count and sharding.
 *
 * Conventions (all entry points):
 *  - Every call returns an int status: GPUAR_OK (0) or a negative GPUAR_E* code.  No C++
 *    exception crosses the ABI.  gpuar_strerror() maps a code to static text.
 *  - Device pointers are BORROWED: the caller (normally a torch tensor) owns them and
 *    keeps them alive and unmodified until the work enqueued on the handle's stream
 *    completes.  Host pointers (gpuar_select_host only) are borrowed for the call's
 *    duration; the call is synchronous.
 *  - All device work is asynchronous on the handle's stream (default: the legacy default
 *    stream of the device current at create time).  No entry point except gpuar_sync,
 *    gpuar_get_stats, gpuar_select_host and gpuar_destroy synchronizes the host.
 *  - A handle is not thread-safe; distinct handles are independent.  A handle binds to the
 *    CUDA device current at gpuar_create; later calls switch to it and restore the
 *    caller's current device.
 *  - Device-detected input errors (a negative, -0.0, NaN or Inf propensity) are STICKY:
 *    they cannot be reported by the asynchronous call that enqueued the work, so the next
 *    gpuar_sync / gpuar_get_stats (or gpuar_select_host) returns GPUAR_EPROPENSITY once
 *    and clears the flag.  Affected selections output idx = -1, trials = 0, tau = NaN.
 *  - An all-zero propensity vector/row is NOT an error: every selection of it outputs
 *    idx = -1, trials = 0, tau = +inf (alpha_0 = 0: no reaction can ever fire; R9).
 *  - idx = -1 with trials = max_trials means "rejected": no acceptance within max_trials
 *    (the paper's sentinel M+1; R8).
 */
#ifndef GPUAR_H
#define GPUAR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GPUAR_OK            0
#define GPUAR_EINVAL       (-1)   /* bad argument (size, pointer, alignment, state)      */
#define GPUAR_ENOMEM       (-2)   /* device or pinned-host allocation failed               */
#define GPUAR_ECUDA        (-3)   /* a CUDA runtime call or kernel launch failed           */
#define GPUAR_ENOTSET      (-4)   /* gpuar_select/get_stats before gpuar_set_propensities  */
#define GPUAR_EPROPENSITY  (-5)   /* sticky: a propensity was negative, -0.0, NaN or Inf   */

/* Opaque handle. */
typedef struct gpuar_handle *gpuar_t;

/* Default per-selection trial cap (R7): P(reject) = (1-p)^(2^20). */
#define GPUAR_DEFAULT_MAX_TRIALS (1u << 20)

/* Create a selector for M reactions and up to K selections per gpuar_select call.
 * Allocates the handle's device scratch (statistics, counters, large-M prefilter) on the
 * current device (the shared-vector thresholds are allocated by gpuar_set_propensities).  epoch = 0, selection offset = 0, max_trials = 2^20, stream = 0.
 * M in [1, 2^31-1], K in [1, 2^32-1].  Errors: EINVAL, ENOMEM, ECUDA.  *out is set only on
 * success. */
int gpuar_create(gpuar_t *out, int64_t M, int64_t K, uint64_t seed);

/* Drain the handle's stream and free its scratch.  NULL is a no-op.  Always GPUAR_OK
 * unless the stream reported an asynchronous CUDA error (ECUDA; the handle is still freed). */
int gpuar_destroy(gpuar_t h);

/* Enqueue all later work on `stream` (a cudaStream_t of the handle's device, passed as
 * void* so this header does not need the CUDA headers).  The new stream is ordered after
 * the work already queued on the previous one (event wait): a handle's launches share its
 * device scratch and must never overlap.  Use one handle per concurrent stream.
 * Kernels are launched with programmatic dependent launch (an early-scheduled grid waits in
 * its first instruction until every earlier grid of the stream has completed), so stream
 * order is exactly that of plain launches; GPUAR_NO_PDL=1 in the environment at
 * gpuar_create turns the attribute off. */
int gpuar_set_stream(gpuar_t h, void *stream);

/* Register the propensities (device pointer, binary32, BORROWED).
 *   rows == 1 : one shared M-vector for every selection (configs c1/c2/c3/c5); enqueues
 *               the statistics pass (alpha_max exact, alpha_0 summed in binary64 with a
 *               fixed tree, validity), then the classic rule's acceptance thresholds
 *               T_j (R22; M words of handle scratch, allocated on the first
 *               shared vector: ENOMEM) and, for M beyond the shared-memory capacity, their
 *               exact 16-bit shared-memory prefilter.  The pointer is kept: call again
 *               after mutating the buffer.  ld is ignored (pass M).
 *   rows == K : per-realization matrix, row r (pitch ld >= M floats, row-major
 *               D[r*ld + j]) belongs to local selection r; its
 *               alpha_max / alpha_0 are reduced inside gpuar_select.  d_alpha must be
 *               16-byte aligned (rows are streamed with 1-D bulk async copies).
 * Errors: EINVAL (NULL pointer, rows not in {1, K}, ld < M, misaligned matrix base, or
 * a matrix whose row cannot fit one shared-memory ring slot: M > 57 000 on B200),
 * ENOMEM, ECUDA.  Invalid values are reported later as sticky EPROPENSITY. */
int gpuar_set_propensities(gpuar_t h, const float *d_alpha, int64_t rows, int64_t ld);

/* Select for local s in [0, K): global index s_g = offset + s, current epoch.  Writes
 * d_idx[s] (int32, -1 = rejected/degenerate), d_tau[s] (binary32), d_trials[s]
 * (uint32: the 1-based index of the accepted trial; max_trials if rejected; 0 if
 * degenerate/invalid).  Then epoch += 1.  Outputs must not alias.  d_tau or d_trials may
 * be NULL (not written).
 * Errors: EINVAL (K < 1, K > capacity, K != rows for a matrix, offset + K > 2^32, NULL
 * d_idx), ENOTSET, ECUDA. */
int gpuar_select(gpuar_t h, int64_t K, int32_t *d_idx, float *d_tau, uint32_t *d_trials);

/* n_epochs consecutive selects in one call: outputs [n_epochs][K] (epoch e at d_idx + e*K,
 * and likewise d_tau / d_trials, which may be NULL), bit-identical to n_epochs gpuar_select
 * calls on the same registration (selection s_g = offset + s at epochs epoch .. epoch +
 * n_epochs - 1); then epoch += n_epochs.  For a shared vector under the classic rule the
 * n_epochs * K selections are ONE launch (one work-stealing pool over all of them), so the
 * per-launch ramp, staging and drain are paid once -- how an SSA driver that keeps the
 * vector for several steps calls select (§Methods: the selection repeats
 * every time step); other rules and the matrix run one launch per epoch.
 * Errors: as gpuar_select, and EINVAL for n_epochs < 1, n_epochs > 65536 or
 * K * n_epochs >= 2^32 (nothing enqueued, epoch unchanged).  When one of the per-epoch
 * launches of the looped case fails, the epoch has advanced by the launches enqueued before
 * it. */
int gpuar_select_epochs(gpuar_t h, int64_t K, int64_t n_epochs, int32_t *d_idx, float *d_tau, uint32_t *d_trials);

/* End-to-end variant for HOST buffers: copies h_alpha (rows x ld floats, or M floats
 * when rows == 1) to the device, selects, and copies the K outputs back, pipelining
 * host->device copies, selection and device->host copies in row chunks on the handle's
 * stream plus two internal streams.  Pinned (page-locked) host buffers give overlap;
 * pageable ones work but serialise.  Synchronous: returns after the outputs are in host
 * memory.  Device staging is owned by the handle (allocated on first use, freed by
 * gpuar_destroy).  Replaces any previously registered propensities.  epoch += 1.
 * Errors: as set_propensities + select, ENOMEM, and EPROPENSITY (reported directly). */
int gpuar_select_host(gpuar_t h, const float *h_alpha, int64_t rows, int64_t ld, int64_t K,
                      int32_t *h_idx, float *h_tau, uint32_t *h_trials);

/* Selection rule (R1, R16-R19).
 *   GPUAR_RULE_CLASSIC (default, w must be 1): classic AR with first accept, the hot path
 *     described at the top of this header; samples alpha_j / alpha_0.
 *   GPUAR_RULE_ARGMIN (w >= 1): the paper's printed GPU algorithm (PAPER.md:304-380,
 *     pseudo-code PAPER.md:498-560): T = fl32(w * alpha_max); every reaction j draws v_j
 *     (Philox counter {j >> 2, s_g, epoch, 3}, word j & 3, v = (x >> 8) 2^-24),
 *     u_j = fl32(v_j T), eligible iff u_j < alpha_j with rating R_j = fl32(u_j / alpha_j),
 *     else R_j = 1; idx = argmin_j R_j (ties to the lowest j), -1 if min R >= 1; trials = M.
 *     Its law is NOT alpha_j / alpha_0 (R1).
 *   GPUAR_RULE_IT (w must be 1): the classic inverse transform, the direct method the paper
 *     replaces (§Methods "The SSA"): u2 = (x >> 8) 2^-24 from Philox
 *     counter {0, s_g, epoch, 2}; idx = the smallest j with C_j > u2 * alpha_0, C_j the
 *     SEQUENTIAL binary64 prefix sum fl64(C_{j-1} + alpha_j) and alpha_0 = C_{M-1} (the last
 *     positive j if rounding ever leaves no crossing); trials = 1 (0 for a degenerate or
 *     invalid vector/row); tau as for the classic rule with fl32(C_{M-1}).  Shared vector:
 *     C computed once per registered vector, then one binary search per selection.  Matrix:
 *     per row, block prefix sums + a search of the crossing block (R24: bit-identical
 *     to the sequential sums, which a row whose partial sums round recomputes sequentially).
 *   GPUAR_RULE_IT_SCAN (w must be 1; matrix only): the same selection by a linear scan of the
 *     row from j = 0 ("iterate in the cumulative distribution"), whose step
 *     count is random -- the cost the paper holds against IT.  Identical outputs to IT.
 * Applies to later gpuar_select / gpuar_select_host calls (IT_SCAN with a shared vector:
 * EINVAL from gpuar_select / gpuar_select_host).
 * Errors: EINVAL (unknown rule, w out of range). */
#define GPUAR_RULE_CLASSIC 0
#define GPUAR_RULE_ARGMIN  1
#define GPUAR_RULE_IT      2
#define GPUAR_RULE_IT_SCAN 3
int gpuar_set_rule(gpuar_t h, int rule, float w);

/* NEXT-2: the full SSA loop around the selector.
 * gpuar_set_network registers a mass-action network of N species and the handle's M
 * reactions (device pointers, BORROWED): d_reac[M][2] reactant species (-1 = none; equal
 * entries = dimerisation), d_rate[M] rate constants, d_didx[M][D] / d_dval[M][D] the sparse
 * change vector v_j (species -1 = unused slot; species distinct within a reaction).
 * Propensity a_j = c_j, c_j X_a, c_j X_a X_b, or c_j X_a (X_a - 1) / 2 (+0 if X_a < 2), in
 * binary32 left to right (R20).  The network plus one realization's state and
 * row (4M + 4N bytes) must fit in shared memory (EINVAL otherwise).  gpuar_set_network is
 * SYNCHRONOUS: it reads the network once to build, per reaction j, the list of reactions
 * whose propensity reads a species j changes (only those are recomputed after j fires;
 * the row stays identical to a full recomputation); EINVAL for species indices >= N.
 * gpuar_ssa_run advances K realizations (d_X[K][N] int32 and d_t[K] binary64, in place)
 * by up to n_steps steps each: step i of realization k (selection s_g = offset + k) uses
 * epoch + i: propensities, classic-AR selection and tau exactly as gpuar_select on that
 * row; alpha_0 = 0 -> halted; t + tau > t_end -> halted (state kept); a rejected
 * selection fires nothing (R21); else X += v_j, t += tau.  d_steps[k] (may be
 * NULL) receives the number of events fired.  Then epoch += n_steps.  Asynchronous.
 * Errors: EINVAL, ENOTSET (no network), ECUDA; invalid propensities -> sticky EPROPENSITY. */
int gpuar_set_network(gpuar_t h, int64_t N, int64_t D, const int32_t *d_reac, const float *d_rate,
                      const int32_t *d_didx, const int32_t *d_dval);
int gpuar_ssa_run(gpuar_t h, int32_t *d_X, double *d_t, uint32_t *d_steps, int64_t K, int32_t n_steps,
                  double t_end);

/* Global index of local selection 0 (sharding: rank r of G -> r*K/G).  s0 in [0, 2^32). */
int gpuar_set_selection_offset(gpuar_t h, int64_t s0);

/* Epoch = Philox counter word 2.  set_epoch replays any earlier call bit-exactly. */
int gpuar_set_epoch(gpuar_t h, uint32_t epoch);
int gpuar_get_epoch(gpuar_t h, uint32_t *epoch);

/* Per-selection trial cap n >= 1 (default 2^20).  EINVAL for n == 0. */
int gpuar_set_max_trials(gpuar_t h, uint32_t n);

/* Synchronous read of the shared-vector statistics: alpha_max, alpha_0 (binary64) and the
 * per-trial acceptance probability p = alpha_0 / (M alpha_max) (0 for an all-zero vector).
 * Any pointer may be NULL.  Errors: ENOTSET (no shared vector registered), EPROPENSITY
 * (sticky), ECUDA. */
int gpuar_get_stats(gpuar_t h, float *amax, double *a0, float *p);

/* Per-row statistics of the registered matrix (validation aid, asynchronous): for r in
 * [0, rows) writes d_amax[r] and d_a0[r] (binary64) with the same reduction the select
 * kernel uses.  Errors: ENOTSET (no matrix registered), EINVAL (NULL pointer). */
int gpuar_row_stats(gpuar_t h, float *d_amax, double *d_a0);

/* Drain the handle's stream; report asynchronous errors.  Errors: EPROPENSITY (sticky,
 * then cleared), ECUDA. */
int gpuar_sync(gpuar_t h);

/* Validation histogram (asynchronous, additive): d_hist[M+1] += counts of d_idx over
 * [0, K) with bin M for idx = -1; d_totals[0] += sum of d_trials; d_totals[1] += number
 * of idx = -1.  d_hist / d_totals are uint64 device arrays the caller zeroes. */
int gpuar_histogram(gpuar_t h, const int32_t *d_idx, const uint32_t *d_trials, int64_t K,
                    uint64_t *d_hist, uint64_t *d_totals);

/* Roofline aid: the Philox4x32-10 generate-and-fold microkernel (no memory traffic but
 * one word per thread).  n_threads threads each make `calls` Philox calls on the
 * handle's stream, folding the outputs into d_sink[thread].  Asynchronous. */
int gpuar_bench_philox(gpuar_t h, int64_t n_threads, int32_t calls, uint32_t *d_sink);

/* Which selection kernel the current registration uses (0 none, 1 shared vector: its
 * acceptance thresholds all in shared memory, 2 shared vector: per-element 16-bit threshold
 * brackets in shared memory, 3 shared vector: per-group 16-bit threshold bounds in shared
 * memory, 4 per-realization rows).  Pure host query. */
int gpuar_path(gpuar_t h, int32_t *path);

/* Team size (lanes per selection, a power of two in [1, 32]) the last classic-rule
 * gpuar_select on a shared vector used, as chosen on the device from p and K (DESIGN.md
 * §5.2); a round of a team covers 2*team consecutive canonical trials, so the trials a
 * selection computed are 2*team*ceil(trials/(2*team)).  0 before any such select.  The
 * matrix path always uses whole warps (32).  Synchronous (drains the handle's stream).
 * Errors: EINVAL, ECUDA. */
int gpuar_last_team(gpuar_t h, int32_t *team);

/* Static text for a status code. */
const char *gpuar_strerror(int status);

#ifdef __cplusplus
}
#endif

#endif /* GPUAR_H */
