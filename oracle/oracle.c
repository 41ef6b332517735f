/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for GPU acceptance-rejection
 * next-reaction selection (arXiv 1404.0027, Neri & Mestivier 2014).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this file's library.  The product
 * path (paper_1404_0027_b200/, libgpuar) never imports, links or executes it, and
 * this file shares no code, header, table or constant generator with the CUDA path.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 *        (x86-64 SSE: every `float` operation below is one IEEE-754 binary32
 *        round-to-nearest-even operation; FLT_EVAL_METHOD must be 0).
 *
 * What is computed, step by step, with the passage each step follows
 * (PAPER.md = /root/reference/PAPER.md line numbers, section in parentheses):
 *
 *   1. Propensity statistics: alpha_0 = sum_j alpha_j (§Methods
 *      "The Stochastic Simulation Algorithm"); threshold T = max_j alpha_j
 *      (PAPER.md:361-365 / 566-568, §Methods "Election step" / §Results, w = 1;
 *      DESIGN.md reading R2).  alpha_0 is summed sequentially in double.
 *   2. Classic acceptance-rejection (§Methods "A GPU
 *      acceptance-rejection algorithm"): "choose randomly a reaction index j and
 *      generate a random number u_{0,T} until u_{0,T} < alpha_j".  Trial i draws
 *      64 random bits from a Philox4x32-10 stream; candidate j = floor(x_a*M/2^32);
 *      u = (x_b >> 8) * 2^-24 in [0,1); u_{0,T} = fl32(u * T); accept iff
 *      u_{0,T} < alpha_j (strict).  The first accepted trial (smallest i) is the
 *      selection; trials = i + 1.  No acceptance within max_trials -> rejected
 *      (idx = -1; the paper's sentinel M+1; R8).
 *   3. Time step tau = (1/a0) ln(1/u1), u1 uniform.
 *      u1 = (2*(x>>9)+1) * 2^-24 in (0,1) from its own Philox stream (tag 1).
 *   4. Inverse-transform linear search, the classic direct method the paper
 *      replaces: smallest j with sum_{j'<=j} alpha_j' > u2*alpha_0.
 *   5. (NEXT-1) the paper's printed election + argmin rule.
 *   6. (NEXT-2) the full SSA loop around the selector: mass-action
 *      propensities, selection, X += v_j, t += tau.
 *
 * Philox4x32-10 is the counter-based generator of Salmon et al. (SC'11, "Parallel
 * random numbers: as easy as 1, 2, 3"), written out from its definition; the
 * north_star of BASELINE.json fixes it as the selection RNG.  Pinned by the
 * Random123 known-answer vectors in tests/golden/philox_kat.txt.
 *
 * Counter layout (R5/R12/R13): ctr = {call, s, epoch, tag}, key = {seed lo, seed hi}
 *   tag 0: AR trials, call = i >> 1, trial i uses words (x0,x1) if i even, (x2,x3) if odd
 *   tag 1: tau uniform u1 (call 0, word x0)
 *   tag 2: IT uniform u2  (call 0, word x0)
 *   tag 3: election draws of the paper's argmin rule (call j >> 2, word j & 3)
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>

#if !defined(FLT_EVAL_METHOD) || FLT_EVAL_METHOD != 0
#error "oracle needs FLT_EVAL_METHOD == 0 (binary32 evaluated in binary32)"
#endif

#define ORACLE_OK 0
#define ORACLE_EPROPENSITY (-5)

/* ------------------------------------------------------------------ Philox4x32-10 */

static void mulhilo32(uint32_t a, uint32_t b, uint32_t *hi, uint32_t *lo)
{
    uint64_t prod = (uint64_t)a * (uint64_t)b;
    *hi = (uint32_t)(prod >> 32);
    *lo = (uint32_t)prod;
}

/* One Philox4x32 round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
 * c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0). */
static void philox_round(uint32_t c[4], const uint32_t k[2])
{
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(0xD2511F53u, c[0], &hi0, &lo0);
    mulhilo32(0xCD9E8D57u, c[2], &hi1, &lo1);
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

/* Ten rounds; the key is bumped by the Weyl constants between rounds. */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            k[0] += 0x9E3779B9u;
            k[1] += 0xBB67AE85u;
        }
        philox_round(c, k);
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

static void draw(uint64_t seed, uint32_t call, uint32_t s, uint32_t epoch, uint32_t tag,
                 uint32_t out[4])
{
    uint32_t ctr[4] = {call, s, epoch, tag};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    oracle_philox4x32_10(ctr, key, out);
}

/* ------------------------------------------------------------------ mappings */

/* candidate index j = floor(x * M / 2^32) in [0, M)  (R5) */
uint32_t oracle_index(uint32_t x, uint32_t M)
{
    return (uint32_t)(((uint64_t)x * (uint64_t)M) >> 32);
}

/* u = (x >> 8) * 2^-24 in [0,1): 24 random bits, exact in binary32 (R3) */
float oracle_unit(uint32_t x)
{
    return (float)(x >> 8) * 0x1p-24f;
}

/* u1 = (2*(x >> 9) + 1) * 2^-24 in (0,1): never 0, so ln(1/u1) is finite (R10) */
float oracle_unit_open(uint32_t x)
{
    return (float)(2u * (x >> 9) + 1u) * 0x1p-24f;
}

/* The acceptance test of PAPER.md:296: u_{0,T} < alpha_j, with u_{0,T} = fl32(u * T). */
int oracle_accept(float u, float amax, float alpha_j)
{
    float u0T = u * amax;
    return u0T < alpha_j;
}

/* ------------------------------------------------------------------ statistics */

/* alpha_max (binary32 max), alpha_0 (sequential double sum).  A propensity must be
 * +0.0 or a positive finite binary32 (R9): returns ORACLE_EPROPENSITY on a
 * set sign bit (negative, -0.0, -NaN) or a non-finite value. */
int oracle_stats(const float *alpha, int64_t M, float *amax_out, double *a0_out)
{
    float amax = 0.0f;
    double a0 = 0.0;
    int ok = 1;
    for (int64_t j = 0; j < M; ++j) {
        float a = alpha[j];
        if (signbit(a) || !isfinite(a)) ok = 0;
        if (a > amax) amax = a;
        a0 += (double)a;
    }
    *amax_out = ok ? amax : NAN;
    *a0_out = ok ? a0 : NAN;
    return ok ? ORACLE_OK : ORACLE_EPROPENSITY;
}

/* ------------------------------------------------------------------ one selection */

/* Classic AR with T = alpha_max, for global selection index s.
 * Outputs idx (-1 = rejected or degenerate), trials, tau (binary32) and tau_ref
 * (double, for the relative-tolerance check). */
void oracle_ar_one(const float *alpha, int64_t M, float amax, double a0,
                   uint64_t seed, uint32_t s, uint32_t epoch, uint32_t max_trials,
                   int32_t *idx, uint32_t *trials, float *tau, double *tau_ref)
{
    if (amax == 0.0f) {                       /* all-zero: no reaction can fire (R9) */
        *idx = -1;
        *trials = 0;
        *tau = INFINITY;
        *tau_ref = INFINITY;
        return;
    }
    *idx = -1;
    *trials = max_trials;
    for (uint32_t i = 0; i < max_trials; ++i) {
        uint32_t x[4];
        draw(seed, i >> 1, s, epoch, 0u, x);
        uint32_t xa = (i & 1u) ? x[2] : x[0];
        uint32_t xb = (i & 1u) ? x[3] : x[1];
        uint32_t j = oracle_index(xa, (uint32_t)M);
        float u = oracle_unit(xb);
        if (oracle_accept(u, amax, alpha[j])) {
            *idx = (int32_t)j;
            *trials = i + 1u;
            break;
        }
    }
    /* tau = (1/a0) ln(1/u1), in binary32 as -logf(u1)/a0f */
    uint32_t t[4];
    draw(seed, 0u, s, epoch, 1u, t);
    float u1 = oracle_unit_open(t[0]);
    float a0f = (float)a0;
    *tau = -logf(u1) / a0f;
    *tau_ref = -log((double)u1) / a0;
}

/* Inverse transform, linear search (SPEC.md select_it): the smallest
 * j with C_j = sum_{j'<=j} alpha_j' > u2 * a0 (strict).  C_j accumulates in double in
 * index order.  If rounding exhausts the scan, the last positive j is returned. */
int32_t oracle_it_one(const float *alpha, int64_t M, double a0, float u2)
{
    double target = (double)u2 * a0;
    double C = 0.0;
    int32_t last_pos = -1;
    for (int64_t j = 0; j < M; ++j) {
        C += (double)alpha[j];
        if (alpha[j] > 0.0f) last_pos = (int32_t)j;
        if (C > target) return (int32_t)j;
    }
    return last_pos;
}

/* ------------------------------------------------------------------ batches */

/* K selections, global indices s0 .. s0+K-1.  rows == 1: one shared M-vector for all
 * selections; rows == K: row r (pitch ld floats) belongs to local selection r.
 * Per-row statistics are recomputed for every row (amax_out/a0_out receive them,
 * may be NULL).  Returns ORACLE_EPROPENSITY if any row used is invalid (that row's
 * outputs are idx=-1, trials=0, tau=NaN). */
int oracle_ar_batch(const float *alpha, int64_t M, int64_t rows, int64_t ld, int64_t K,
                    uint64_t seed, uint32_t s0, uint32_t epoch, uint32_t max_trials,
                    int32_t *idx, float *tau, uint32_t *trials,
                    float *amax_out, double *a0_out, double *tau_ref, int nthreads)
{
    int status = ORACLE_OK;
    float shared_amax = 0.0f;
    double shared_a0 = 0.0;
    if (rows == 1) {
        if (oracle_stats(alpha, M, &shared_amax, &shared_a0) != ORACLE_OK)
            status = ORACLE_EPROPENSITY;
    }
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t r = 0; r < K; ++r) {
        const float *row = (rows == 1) ? alpha : alpha + r * ld;
        float amax;
        double a0;
        int ok;
        if (rows == 1) {
            amax = shared_amax;
            a0 = shared_a0;
            ok = (status == ORACLE_OK);
        } else {
            ok = (oracle_stats(row, M, &amax, &a0) == ORACLE_OK);
        }
        double tr = 0.0;
        if (ok) {
            oracle_ar_one(row, M, amax, a0, seed, s0 + (uint32_t)r, epoch, max_trials,
                          &idx[r], &trials[r], &tau[r], &tr);
        } else {
            idx[r] = -1;
            trials[r] = 0;
            tau[r] = NAN;
            tr = NAN;
            if (rows != 1) {
#pragma omp atomic write
                status = ORACLE_EPROPENSITY;
            }
        }
        if (amax_out) amax_out[r] = amax;
        if (a0_out) a0_out[r] = a0;
        if (tau_ref) tau_ref[r] = tr;
    }
    return status;
}

/* IT selections for the same (seed, s, epoch) on uniform stream tag 2. */
int oracle_it_batch(const float *alpha, int64_t M, int64_t rows, int64_t ld, int64_t K,
                    uint64_t seed, uint32_t s0, uint32_t epoch, int32_t *idx, int nthreads)
{
    int status = ORACLE_OK;
    float shared_amax = 0.0f;
    double shared_a0 = 0.0;
    if (rows == 1 && oracle_stats(alpha, M, &shared_amax, &shared_a0) != ORACLE_OK)
        status = ORACLE_EPROPENSITY;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t r = 0; r < K; ++r) {
        const float *row = (rows == 1) ? alpha : alpha + r * ld;
        float amax = shared_amax;
        double a0 = shared_a0;
        int ok = (rows == 1) ? (status == ORACLE_OK)
                             : (oracle_stats(row, M, &amax, &a0) == ORACLE_OK);
        if (!ok || amax == 0.0f) {
            idx[r] = -1;
            continue;
        }
        uint32_t x[4];
        draw(seed, 0u, s0 + (uint32_t)r, epoch, 2u, x);
        idx[r] = oracle_it_one(row, M, a0, oracle_unit(x[0]));
    }
    return status;
}

/* ------------------------------------------------------------------ the paper's printed rule (NEXT-1) */

/* Election + selection of PAPER.md:304-380 / pseudo-code PAPER.md:498-560 ("argmin rule"),
 * with the readings of DESIGN.md R16-R19:
 *   threshold T = fl32(w * alpha_max)  (T_w of PAPER.md:566-568);
 *   election: for every reaction j draw v_j = (x>>8) 2^-24 in [0,1)
 *     from Philox ctr {j >> 2, s, epoch, 3}, word j & 3; u_j = fl32(v_j * T);
 *     eligible iff u_j < D_j (then D_j > 0), rated R_j = fl32(u_j / D_j);
 *     not eligible: R_j = 1.0 (sentinel; the pseudo-code's T*10 is a bug);
 *   selection: j* = argmin_j R_j, ties to the lowest j;
 *     if R_j* >= 1 the election failed: rejected (idx -1; the paper's M+1).
 * trials = M (draws consumed). tau as for the classic rule. */
/* Election step: rating of reaction j for unit draw v_j. */
float oracle_election(float alpha_j, float v, float T)
{
    float u = v * T;                               /* u_{0,T} in [0, T) */
    return (u < alpha_j) ? u / alpha_j : 1.0f;     /* R >= 1 means "not eligible" */
}

/* Selection step: argmin of the ratings, ties to the lowest
 * index; -1 when the minimum is >= 1 (the election failed: rejection). */
int32_t oracle_selection(const float *R, int64_t M)
{
    float best = 1.0f;
    int32_t best_j = -1;
    for (int64_t j = 0; j < M; ++j) {
        if (R[j] < best) {
            best = R[j];
            best_j = (int32_t)j;
        }
    }
    return best_j;
}

void oracle_argmin_one(const float *alpha, int64_t M, float amax, double a0, float w,
                       uint64_t seed, uint32_t s, uint32_t epoch,
                       int32_t *idx, float *tau, double *tau_ref)
{
    if (amax == 0.0f) {
        *idx = -1;
        *tau = INFINITY;
        *tau_ref = INFINITY;
        return;
    }
    float T = w * amax;
    float best = 1.0f;
    int32_t best_j = -1;
    uint32_t x[4];
    for (int64_t j = 0; j < M; ++j) {
        if ((j & 3) == 0) draw(seed, (uint32_t)(j >> 2), s, epoch, 3u, x);
        float R = oracle_election(alpha[j], oracle_unit(x[j & 3]), T);
        if (R < best) {           /* oracle_selection, streamed: strict, ties keep the lowest j */
            best = R;
            best_j = (int32_t)j;
        }
    }
    *idx = best_j;                /* -1 when every rating is >= 1 */
    uint32_t t[4];
    draw(seed, 0u, s, epoch, 1u, t);
    float u1 = oracle_unit_open(t[0]);
    *tau = -logf(u1) / (float)a0;
    *tau_ref = -log((double)u1) / a0;
}

int oracle_argmin_batch(const float *alpha, int64_t M, int64_t rows, int64_t ld, int64_t K, float w,
                        uint64_t seed, uint32_t s0, uint32_t epoch,
                        int32_t *idx, float *tau, double *tau_ref, int nthreads)
{
    int status = ORACLE_OK;
    float shared_amax = 0.0f;
    double shared_a0 = 0.0;
    if (rows == 1 && oracle_stats(alpha, M, &shared_amax, &shared_a0) != ORACLE_OK)
        status = ORACLE_EPROPENSITY;
#pragma omp parallel for schedule(dynamic, 64) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t r = 0; r < K; ++r) {
        const float *row = (rows == 1) ? alpha : alpha + r * ld;
        float amax = shared_amax;
        double a0 = shared_a0;
        int ok = (rows == 1) ? (status == ORACLE_OK)
                             : (oracle_stats(row, M, &amax, &a0) == ORACLE_OK);
        if (!ok) {
            idx[r] = -1;
            tau[r] = NAN;
            tau_ref[r] = NAN;
            if (rows != 1) {
#pragma omp atomic write
                status = ORACLE_EPROPENSITY;
            }
            continue;
        }
        oracle_argmin_one(row, M, amax, a0, w, seed, s0 + (uint32_t)r, epoch, &idx[r], &tau[r], &tau_ref[r]);
    }
    return status;
}

/* ------------------------------------------------------------------ full SSA (NEXT-2) */

/* Mass-action propensity of a reaction with reactants r0, r1 (species index, -1 = none)
 * and rate constant c (Gillespie's direct method; "propensity function
 * a_j", updated at each step):  order 0: c;  order 1: c X_r0;  two different species:
 * c X_r0 X_r1;  dimerisation (r0 == r1): c X (X-1) / 2, and +0 when X < 2.  binary32,
 * evaluated left to right (R20). */
float oracle_propensity(const int32_t *X, int32_t r0, int32_t r1, float c)
{
    float a = c;
    if (r0 >= 0) {
        if (r1 == r0) {
            int32_t x = X[r0];
            if (x < 2) return 0.0f;
            a = a * (float)x;
            a = a * (float)(x - 1);
            return a * 0.5f;
        }
        a = a * (float)X[r0];
    }
    if (r1 >= 0) a = a * (float)X[r1];
    return a;
}

/* K independent SSA realizations (propensities, next reaction and tau,
 * "the system is updated using v_j, t <- t + tau", until t_end).  Realization k (global
 * selection index s0 + k) makes up to n_steps steps; step i uses epoch epoch0 + i:
 *   a_j = propensity(X_k) for every j; (idx, tau) = classic AR selection on that row;
 *   a0 = 0            -> halted (nothing can fire), state kept;
 *   t + tau > t_end   -> halted (the next event is past t_end), state kept;
 *   idx = -1 (rejected after max_trials) -> no event this step (R21);
 *   else X += v_idx (D sparse (species, delta) pairs, species -1 = unused), t += tau.
 * X is K x N int32 (in/out), t is K doubles (in/out), steps[k] = events fired.
 * Returns ORACLE_EPROPENSITY if a propensity was invalid (negative/non-finite). */
int oracle_ssa_run(int64_t N, int64_t M, int64_t D, const int32_t *reac, const float *rate,
                   const int32_t *didx, const int32_t *dval, int64_t K, int32_t *X, double *t,
                   uint32_t *steps, int32_t n_steps, double t_end, uint64_t seed, uint32_t s0,
                   uint32_t epoch0, uint32_t max_trials, int nthreads)
{
    int status = ORACLE_OK;
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1)
    {
        float *row = (float *)malloc(sizeof(float) * (size_t)M);
#pragma omp for schedule(dynamic, 16)
        for (int64_t k = 0; k < K; ++k) {
            int32_t *x = X + k * N;
            uint32_t fired = 0;
            for (int32_t i = 0; i < n_steps; ++i) {
                for (int64_t j = 0; j < M; ++j)
                    row[j] = oracle_propensity(x, reac[2 * j], reac[2 * j + 1], rate[j]);
                float amax;
                double a0;
                if (oracle_stats(row, M, &amax, &a0) != ORACLE_OK) {
#pragma omp atomic write
                    status = ORACLE_EPROPENSITY;
                    break;
                }
                if (amax == 0.0f) break;                      /* halted: nothing can fire */
                int32_t idx;
                uint32_t tr;
                float tau;
                double tau_ref;
                oracle_ar_one(row, M, amax, a0, seed, s0 + (uint32_t)k, epoch0 + (uint32_t)i, max_trials,
                              &idx, &tr, &tau, &tau_ref);
                if (t[k] + (double)tau > t_end) break;       /* next event past t_end */
                if (idx < 0) continue;                        /* rejected: no event this step */
                for (int64_t d = 0; d < D; ++d) {
                    int32_t sp = didx[idx * D + d];
                    if (sp >= 0) x[sp] += dval[idx * D + d];
                }
                t[k] += (double)tau;
                ++fired;
            }
            steps[k] = fired;
        }
        free(row);
    }
    return status;
}

/* Validation histogram: hist[M+1] (bin M = rejected/degenerate), plus the sum of trials. */
void oracle_histogram(const int32_t *idx, const uint32_t *trials, int64_t K, int64_t M,
                      uint64_t *hist, uint64_t *trials_sum)
{
    uint64_t tsum = 0;
    for (int64_t r = 0; r < K; ++r) {
        int32_t j = idx[r];
        hist[(j >= 0 && j < M) ? j : M] += 1u;
        tsum += trials[r];
    }
    *trials_sum = tsum;
}
