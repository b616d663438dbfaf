/*
 * oracle/oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation, in double precision, of
 * what the InPlace-ABN hot path computes.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, constant or helper with the CUDA product path
 * (paper_1712_02616_b200/csrc, include/iabn.h), and the product never calls it.
 *
 * Every function follows a passage of PAPER.md (arXiv 1712.02616, LaTeX
 * source); line numbers are PAPER.md lines.  Readings of passages the paper
 * leaves open are listed in DESIGN.md section "Readings" and referenced here
 * as R<k>.
 *
 * Layout (R11): x[n][c][s] (NCHW, layout 0) or x[n][s][c] (NHWC, layout 1),
 * s in [0, HW).  The "unit" of the paper (a fixed unit x whose
 * minibatch values are x_1..x_m) is one channel c; m = N*HW.
 *
 * Pins: tests/test_oracle_pins.py (worked examples, closed forms, finite
 * differences, PyTorch float64, three-way equivalence, mutation tests).
 * Parity unpinned (pinned only to our reading): running-var estimator and
 * momentum convention (R3; the biased branch is pinned to SPEC.md's reading), the
 * |gamma|+eps reparametrisation (R4), the subgradient at 0 (R5), local dgamma/dbeta
 * under sync (R7; pinned by their sum, the whole-batch gradient).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

#include "oracle.h"

/* Mutation hook for the test-of-tests (tests/test_oracle_mutants.py): each
 * value of ORACLE_MUTANT introduces one plausible mistake; 0 = correct. */
#ifndef ORACLE_MUTANT
#define ORACLE_MUTANT 0
#endif

static size_t at(int layout, int64_t C, int64_t HW, int64_t n, int64_t c, int64_t s)
{
#if ORACLE_MUTANT == 9
    (void)layout; /* mutant: layout ignored (NHWC read as NCHW) */
#else
    if (layout == ORACLE_NHWC)
        return (size_t)((n * HW + s) * C + c);
#endif
    return (size_t)((n * C + c) * HW + s);
}

/* Effective scale gamma~ (R4; "preventing gamma from getting less
 * than a given tolerance" / "fixing it to 1"). */
static double gamma_eff(int mode, double g, double eps)
{
    if (mode == ORACLE_GAMMA_PLAIN)
        return g;
    if (mode == ORACLE_GAMMA_FIXED_ONE)
        return 1.0;
    return fabs(g) + eps; /* ORACLE_GAMMA_ABS_EPS */
}

/* d gamma~ / d gamma, with sgn(0) = +1 (R4). */
static double gamma_eff_deriv(int mode, double g)
{
    if (mode == ORACLE_GAMMA_ABS_EPS)
        return g < 0.0 ? -1.0 : 1.0;
    return 1.0; /* PLAIN: identity; FIXED_ONE: grad w.r.t. gamma~ is returned (R4) */
}

/* Leaky ReLU: f(y) = y if y >= 0, a*y if y < 0. */
static double leaky(double y, double a)
{
    return y >= 0.0 ? y : a * y;
}

/* Inverse: f^-1(z) = z if z >= 0, z/a if z < 0. */
static double leaky_inv(double z, double a)
{
#if ORACLE_MUTANT == 2
    return z >= 0.0 ? z : z * a; /* mutant: multiplies instead of divides */
#else
    return z >= 0.0 ? z : z / a;
#endif
}

/* Derivative of f at a point whose sign is that of v (v = y, or v = z since
 * sign(z) = sign(y) for a > 0); f'(0) = 1 (R5). */
static double leaky_deriv(double v, double a)
{
#if ORACLE_MUTANT == 3
    return v >= 0.0 ? a : 1.0; /* mutant: branches swapped */
#else
    return v >= 0.0 ? 1.0 : a;
#endif
}

/* Minibatch statistics of one channel, PAPER.md:74-77:
 *   mu = (1/m) sum_j x_j,   sigma^2 = (1/m) sum_j (x_j - mu)^2   (two-pass). */
static void channel_stats(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                          int64_t c, double *mu_out, double *var_out)
{
    const double m = (double)(N * HW);
    double sum = 0.0;
    for (int64_t n = 0; n < N; ++n)
        for (int64_t s = 0; s < HW; ++s)
            sum += x[at(layout, C, HW, n, c, s)];
    const double mu = sum / m;
    double ss = 0.0;
    for (int64_t n = 0; n < N; ++n)
        for (int64_t s = 0; s < HW; ++s) {
            const double d = x[at(layout, C, HW, n, c, s)] - mu;
            ss += d * d;
        }
#if ORACLE_MUTANT == 4
    *var_out = ss / (m - 1.0); /* mutant: unbiased batch variance */
#else
    *var_out = ss / m;
#endif
    *mu_out = mu;
}

void oracle_channel_stats(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                          double *mean, double *var)
{
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c)
        channel_stats(N, C, HW, layout, x, c, &mean[c], &var[c]);
}

/*
 * Forward of "standard BN followed by leaky ReLU" (Fig. 2a),
 * which InPlace-ABN reproduces exactly (Alg. 1):
 *   x^ = (x - mu)/sqrt(sigma^2 + eps)   Eq.(1)
 *   y  = gamma~ x^ + beta
 *   z  = f(y)
 * Running statistics ("running mean"; formula R3):
 *   r_mu <- (1-alpha) r_mu + alpha mu;  r_var <- (1-alpha) r_var + alpha var*m/(m-1)
 * (var*m/(m-1) replaced by var when running_var_biased != 0).
 * running_mean/running_var may be NULL (skipped).  mean_out/var_out receive the
 * batch mean and biased batch variance.
 */
void oracle_forward(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                    const double *gamma, const double *beta, int gamma_mode, double eps,
                    double slope, double momentum, int running_var_biased,
                    double *running_mean, double *running_var, double *z,
                    double *mean_out, double *var_out)
{
    const double m = (double)(N * HW);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        double mu, var;
        channel_stats(N, C, HW, layout, x, c, &mu, &var);
#if ORACLE_MUTANT == 1
        const double rstd = 1.0 / sqrt(var); /* mutant: epsilon dropped from Eq.(1) */
#else
        const double rstd = 1.0 / sqrt(var + eps);
#endif
        const double g = gamma_eff(gamma_mode, gamma[c], eps);
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                const double xhat = (x[i] - mu) * rstd;
#if ORACLE_MUTANT == 5
                const double y = g * xhat - beta[c]; /* mutant: wrong sign of beta */
#else
                const double y = g * xhat + beta[c];
#endif
                z[i] = leaky(y, slope);
            }
        if (mean_out)
            mean_out[c] = mu;
        if (var_out)
            var_out[c] = var;
        if (running_mean)
            running_mean[c] = (1.0 - momentum) * running_mean[c] + momentum * mu;
        if (running_var) {
#if ORACLE_MUTANT == 10
            const double v = var; /* mutant: Bessel correction dropped */
            (void)running_var_biased;
#elif ORACLE_MUTANT == 13
            const double v = var * m / (m - 1.0); /* mutant: running_var_biased ignored */
            (void)running_var_biased;
#else
            const double v = running_var_biased ? var : var * m / (m - 1.0);
#endif
            running_var[c] = (1.0 - momentum) * running_var[c] + momentum * v;
        }
    }
}

/*
 * Eval-mode forward (at test time the statistics are fixed to
 * mu_T, sigma_T): z = f(gamma~ (x - r_mu)/sqrt(r_var + eps) + beta).
 */
void oracle_forward_eval(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                         const double *gamma, const double *beta, int gamma_mode, double eps,
                         double slope, const double *running_mean, const double *running_var,
                         double *z)
{
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        const double rstd = 1.0 / sqrt(running_var[c] + eps);
        const double g = gamma_eff(gamma_mode, gamma[c], eps);
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                z[i] = leaky(g * (x[i] - running_mean[c]) * rstd + beta[c], slope);
            }
    }
}

/*
 * Backward of the standard block from STORED x (Fig. 2a),
 * written as the original chain rule of the Appendix, an
 * independent derivation from the refactored BN* of PAPER.md:168:
 *   x^_j, y_j recomputed from x (Eq.(1));  dy_j = f'(y_j) dz_j
 *   dbeta = sum dy_j                          (:431)
 *   dgamma~ = sum dy_j x^_j                   (:430)
 *   dL/dx^_j = gamma~ dy_j                    (:432)
 *   dL/dvar = sum_j dL/dx^_j (x_j - mu) (-1/2)(var + eps)^(-3/2)   (:435, :439)
 *   dL/dmu  = sum_j dL/dx^_j (-rstd) + dL/dvar (-2/m) sum_j (x_j - mu)
 *             (:436, :440; the paper drops the second term, which is 0 in
 *             exact arithmetic -- kept here)
 *   dx_i = dL/dx^_i rstd + dL/dvar 2 (x_i - mu)/m + dL/dmu / m   (:444-449)
 * dgamma = dgamma~ * d gamma~/d gamma (R4).
 */
void oracle_backward_standard(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                              const double *dz, const double *gamma, const double *beta,
                              int gamma_mode, double eps, double slope, double *dx,
                              double *dgamma, double *dbeta)
{
    const double m = (double)(N * HW);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        double mu, var;
        channel_stats(N, C, HW, layout, x, c, &mu, &var);
        const double rstd = 1.0 / sqrt(var + eps);
        const double g = gamma_eff(gamma_mode, gamma[c], eps);
        double sdy = 0.0, sdyxh = 0.0, sdvar = 0.0, sdxh = 0.0, sxm = 0.0;
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                const double xm = x[i] - mu;
                const double xhat = xm * rstd;
                const double y = g * xhat + beta[c];
                const double dy = leaky_deriv(y, slope) * dz[i];
                const double dxhat = dy * g;
                sdy += dy;
                sdyxh += dy * xhat;
                sdvar += dxhat * xm;
                sdxh += dxhat;
                sxm += xm;
            }
        const double dvar = sdvar * (-0.5) * pow(var + eps, -1.5);
#if ORACLE_MUTANT == 6
        const double dmu = sdxh * rstd + dvar * (-2.0 / m) * sxm; /* mutant: sign of d x^/d mu */
#else
        const double dmu = sdxh * (-rstd) + dvar * (-2.0 / m) * sxm;
#endif
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                const double xm = x[i] - mu;
                const double y = g * xm * rstd + beta[c];
                const double dxhat = leaky_deriv(y, slope) * dz[i] * g;
#if ORACLE_MUTANT == 7
                dx[i] = dxhat * rstd + dvar * 2.0 * xm / m; /* mutant: dropped dL/dmu term */
#else
                dx[i] = dxhat * rstd + dvar * 2.0 * xm / m + dmu / m;
#endif
            }
        dbeta[c] = sdy;
#if ORACLE_MUTANT == 8
        dgamma[c] = sdyxh; /* mutant: forgets sgn(gamma) of the |gamma|+eps reparametrisation */
#else
        dgamma[c] = sdyxh * gamma_eff_deriv(gamma_mode, gamma[c]);
#endif
    }
}

/*
 * InPlace-ABN I backward from the stored z and sigma (Alg. 2):
 *   dy = phi_backward(z, dz)            (l.2)
 *   y  = phi^-1(z)                      (l.3)
 *   x^ = pi^-1(y) = (y - beta)/gamma~   (l.5)
 *   BN*(x^, dy, sigma) (l.6):
 *     dgamma~ = sum dy x^,  dbeta = sum dy,
 *     dx_i = (dy_i - dgamma~ x^_i / m - dbeta / m) gamma~ / sqrt(var + eps)
 * var is the biased batch variance saved by the forward (Alg. 1 l.3).
 */
void oracle_backward_inplace_I(int64_t N, int64_t C, int64_t HW, int layout, const double *z,
                               const double *dz, const double *var, const double *gamma,
                               const double *beta, int gamma_mode, double eps, double slope,
                               double *dx, double *dgamma, double *dbeta)
{
    const double m = (double)(N * HW);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        const double rstd = 1.0 / sqrt(var[c] + eps);
        const double g = gamma_eff(gamma_mode, gamma[c], eps);
        double sdy = 0.0, sdyxh = 0.0;
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                const double dy = leaky_deriv(z[i], slope) * dz[i];
                const double xhat = (leaky_inv(z[i], slope) - beta[c]) / g;
                sdy += dy;
                sdyxh += dy * xhat;
            }
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                const double dy = leaky_deriv(z[i], slope) * dz[i];
                const double xhat = (leaky_inv(z[i], slope) - beta[c]) / g;
                dx[i] = (dy - sdyxh * xhat / m - sdy / m) * g * rstd;
            }
        dbeta[c] = sdy;
        dgamma[c] = sdyxh * gamma_eff_deriv(gamma_mode, gamma[c]);
    }
}

/*
 * InPlace-ABN II backward, BN-dagger as a function of y (Alg. 2 l.7-8;
 * PAPER.md:181-190, Appendix :452-460):
 *   dbeta = sum dy;  dgamma~ = (1/gamma~)[sum dy_j y_j - beta dbeta]
 *   dx_i = [dy_i - dgamma~ y_i/(gamma~ m) - (dbeta - beta dgamma~/gamma~)/m] gamma~ rstd
 */
void oracle_backward_inplace_II(int64_t N, int64_t C, int64_t HW, int layout, const double *z,
                                const double *dz, const double *var, const double *gamma,
                                const double *beta, int gamma_mode, double eps, double slope,
                                double *dx, double *dgamma, double *dbeta)
{
    const double m = (double)(N * HW);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        const double rstd = 1.0 / sqrt(var[c] + eps);
        const double g = gamma_eff(gamma_mode, gamma[c], eps);
        const double b = beta[c];
        double sdy = 0.0, sdyy = 0.0;
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                const double dy = leaky_deriv(z[i], slope) * dz[i];
                sdy += dy;
                sdyy += dy * leaky_inv(z[i], slope);
            }
        const double dg = (sdyy - b * sdy) / g;
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                const double dy = leaky_deriv(z[i], slope) * dz[i];
                const double y = leaky_inv(z[i], slope);
                dx[i] = (dy - dg * y / (g * m) - (sdy - b * dg / g) / m) * g * rstd;
            }
        dbeta[c] = sdy;
        dgamma[c] = dg * gamma_eff_deriv(gamma_mode, gamma[c]);
    }
}

/*
 * Statistics of a minibatch split into shards (InPlace-ABN^sync, PAPER.md:315:
 * "a 'virtual' increase of batch size applied to the computation of BN
 * statistics").  Shard k holds counts[k], means[k][c], biased vars[k][c]; the
 * merged statistics are those of the concatenated batch:
 *   m = sum m_k;  mu = sum m_k mu_k / m;  var = sum m_k (var_k + (mu_k - mu)^2) / m
 */
void oracle_merge_stats(int64_t K, int64_t C, const double *counts, const double *means,
                        const double *vars, double *count_out, double *mean_out,
                        double *var_out)
{
    double m = 0.0;
    for (int64_t k = 0; k < K; ++k)
        m += counts[k];
    *count_out = m;
    for (int64_t c = 0; c < C; ++c) {
        double mu = 0.0;
        for (int64_t k = 0; k < K; ++k)
            mu += counts[k] * means[k * C + c];
        mu /= m;
        double v = 0.0;
        for (int64_t k = 0; k < K; ++k) {
            const double d = means[k * C + c] - mu;
            v += counts[k] * (vars[k * C + c] + d * d);
        }
        mean_out[c] = mu;
        var_out[c] = v / m;
    }
}

/*
 * Test-time folding: "the computation of networks trained with
 * batch normalization can be sped up by absorbing BN parameters into the
 * preceding Conv layer, by performing a simple update of the convolution
 * weights and biases.  This is possible because at test-time BN becomes a
 * linear operation."  With fixed statistics mu_T, sigma_T^2 the BN of output
 * channel k is y = g_k (v - mu_k)/sqrt(sigma_k^2 + eps) + beta_k, v = w_k . x + b_k, so
 *   w'_k = s_k w_k,  b'_k = s_k (b_k - mu_k) + beta_k,  s_k = g_k / sqrt(sigma_k^2 + eps)
 * (SPEC.md:239-247).  w is [cout][kper] row-major; bias NULL means 0.
 */
void oracle_fold_conv(int64_t cout, int64_t kper, const double *w, const double *bias,
                      const double *running_mean, const double *running_var,
                      const double *gamma, const double *beta, int gamma_mode, double eps,
                      double *w_out, double *bias_out)
{
    for (int64_t k = 0; k < cout; ++k) {
        const double s = gamma_eff(gamma_mode, gamma[k], eps) / sqrt(running_var[k] + eps);
        for (int64_t j = 0; j < kper; ++j)
            w_out[k * kper + j] = s * w[k * kper + j];
        const double b = bias ? bias[k] : 0.0;
#if ORACLE_MUTANT == 11
        bias_out[k] = s * b + beta[k]; /* forgot the running mean */
#else
        bias_out[k] = s * (b - running_mean[k]) + beta[k];
#endif
    }
}

/*
 * Parameter gradients of each shard under InPlace-ABN^sync (PAPER.md:315 statistics
 * of the whole, "virtual" batch; :356 "gradient-synchronized"), reading R7: every rank
 * returns its own contribution to dL/dbeta and dL/dgamma, so that the caller's
 * data-parallel gradient sum yields the gradient of the whole batch.  With x the
 * concatenation of the shards along N (shard k = samples [o_k, o_k + shard_n[k])),
 * mu and sigma^2 are those of the whole batch and, per shard k,
 *   dbeta_k   = sum_{i in k} dy_i
 *   dgamma~_k = sum_{i in k} dy_i x^_i
 * with x^_i, y_i from stored x (Eq.(1)) and dy_i = f'(y_i) dz_i; dgamma_k =
 * dgamma~_k d gamma~/d gamma (R4).  Outputs are [nshards][C].
 */
void oracle_param_grads_sharded(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                                const double *dz, const double *gamma, const double *beta,
                                int gamma_mode, double eps, double slope, int64_t nshards,
                                const int64_t *shard_n, double *dgamma, double *dbeta)
{
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        double mu, var;
        channel_stats(N, C, HW, layout, x, c, &mu, &var);
        const double rstd = 1.0 / sqrt(var + eps);
        const double g = gamma_eff(gamma_mode, gamma[c], eps);
        int64_t n0 = 0;
        for (int64_t k = 0; k < nshards; ++k) {
#if ORACLE_MUTANT == 12
            /* mutant: the shard's own statistics instead of the whole batch's */
            channel_stats(shard_n[k], C, HW, layout, x + (size_t)n0 * C * HW, c, &mu, &var);
            const double rstd_k = 1.0 / sqrt(var + eps);
#else
            const double rstd_k = rstd;
#endif
            double sdy = 0.0, sdyxh = 0.0;
            for (int64_t n = n0; n < n0 + shard_n[k]; ++n)
                for (int64_t s = 0; s < HW; ++s) {
                    const size_t i = at(layout, C, HW, n, c, s);
                    const double xhat = (x[i] - mu) * rstd_k;
                    const double y = g * xhat + beta[c];
                    const double dy = leaky_deriv(y, slope) * dz[i];
                    sdy += dy;
                    sdyxh += dy * xhat;
                }
            dbeta[k * C + c] = sdy;
            dgamma[k * C + c] = sdyxh * gamma_eff_deriv(gamma_mode, gamma[c]);
            n0 += shard_n[k];
        }
    }
}

/*
 * Other invertible activations ("Many activation functions are actually
 * invertible and can be computed in-place (e.g. sigmoid, hyperbolic tangent, Leaky ReLU,
 * and others)").  act: ORACLE_ACT_LEAKY (slope a), ORACLE_ACT_SIGMOID, ORACLE_ACT_TANH.
 *   sigmoid: f(y) = 1/(1 + e^-y), f'(y) = f(y)(1 - f(y)), f^-1(z) = log(z/(1 - z))
 *   tanh:    f(y) = tanh(y),      f'(y) = 1 - f(y)^2,    f^-1(z) = atanh(z)
 */
static double act_f(int act, double y, double a)
{
    if (act == ORACLE_ACT_SIGMOID)
        return 1.0 / (1.0 + exp(-y));
    if (act == ORACLE_ACT_TANH)
        return tanh(y);
    return leaky(y, a);
}
/* f'(y) computed from z = f(y) (Alg. 2 l.2: the backward sees only z) */
static double act_deriv_z(int act, double z, double a)
{
#if ORACLE_MUTANT == 14
    if (act == ORACLE_ACT_SIGMOID)
        return z * (1.0 + z); /* mutant: sign slip in the sigmoid derivative */
#else
    if (act == ORACLE_ACT_SIGMOID)
        return z * (1.0 - z);
#endif
    if (act == ORACLE_ACT_TANH)
        return 1.0 - z * z;
    return leaky_deriv(z, a);
}
static double act_inv(int act, double z, double a)
{
    if (act == ORACLE_ACT_SIGMOID)
        return log(z / (1.0 - z));
    if (act == ORACLE_ACT_TANH)
        return atanh(z);
    return leaky_inv(z, a);
}

/* Forward of BN followed by activation `act` from stored x (as oracle_forward, without
 * running statistics): z = act(gamma~ (x - mu) rstd + beta). */
void oracle_forward_act(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                        const double *gamma, const double *beta, int gamma_mode, double eps,
                        int act, double slope, double *z, double *mean_out, double *var_out)
{
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        double mu, var;
        channel_stats(N, C, HW, layout, x, c, &mu, &var);
        const double rstd = 1.0 / sqrt(var + eps);
        const double g = gamma_eff(gamma_mode, gamma[c], eps);
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                z[i] = act_f(act, g * (x[i] - mu) * rstd + beta[c], slope);
            }
        if (mean_out)
            mean_out[c] = mu;
        if (var_out)
            var_out[c] = var;
    }
}

/* Backward from STORED x for activation `act` (the chain rule of oracle_backward_standard,
 * PAPER.md:428-449, with dy = f'(y) dz, f'(y) from f(y) as written above). */
void oracle_backward_standard_act(int64_t N, int64_t C, int64_t HW, int layout,
                                  const double *x, const double *dz, const double *gamma,
                                  const double *beta, int gamma_mode, double eps, int act,
                                  double slope, double *dx, double *dgamma, double *dbeta)
{
    const double m = (double)(N * HW);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        double mu, var;
        channel_stats(N, C, HW, layout, x, c, &mu, &var);
        const double rstd = 1.0 / sqrt(var + eps);
        const double g = gamma_eff(gamma_mode, gamma[c], eps);
        double sdy = 0.0, sdyxh = 0.0, sdvar = 0.0, sdxh = 0.0, sxm = 0.0;
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                const double xm = x[i] - mu;
                const double xhat = xm * rstd;
                const double fy = act_f(act, g * xhat + beta[c], slope);
                const double dy = (act == ORACLE_ACT_SIGMOID ? fy * (1.0 - fy)
                                   : act == ORACLE_ACT_TANH ? 1.0 - fy * fy
                                   : leaky_deriv(g * xhat + beta[c], slope)) * dz[i];
                const double dxhat = dy * g;
                sdy += dy;
                sdyxh += dy * xhat;
                sdvar += dxhat * xm;
                sdxh += dxhat;
                sxm += xm;
            }
        const double dvar = sdvar * (-0.5) * pow(var + eps, -1.5);
        const double dmu = sdxh * (-rstd) + dvar * (-2.0 / m) * sxm;
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                const double xm = x[i] - mu;
                const double y = g * xm * rstd + beta[c];
                const double fy = act_f(act, y, slope);
                const double dy = (act == ORACLE_ACT_SIGMOID ? fy * (1.0 - fy)
                                   : act == ORACLE_ACT_TANH ? 1.0 - fy * fy
                                   : leaky_deriv(y, slope)) * dz[i];
                dx[i] = dy * g * rstd + dvar * 2.0 * xm / m + dmu / m;
            }
        dbeta[c] = sdy;
        dgamma[c] = sdyxh * gamma_eff_deriv(gamma_mode, gamma[c]);
    }
}

/* InPlace-ABN I backward from the stored z for activation `act` (Alg. 2 l.2-6,
 * PAPER.md:215-223): dy = f'(z) dz, x^ = (f^-1(z) - beta)/gamma~, BN* (PAPER.md:168). */
void oracle_backward_inplace_act(int64_t N, int64_t C, int64_t HW, int layout, const double *z,
                                 const double *dz, const double *var, const double *gamma,
                                 const double *beta, int gamma_mode, double eps, int act,
                                 double slope, double *dx, double *dgamma, double *dbeta)
{
    const double m = (double)(N * HW);
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < C; ++c) {
        const double rstd = 1.0 / sqrt(var[c] + eps);
        const double g = gamma_eff(gamma_mode, gamma[c], eps);
        double sdy = 0.0, sdyxh = 0.0;
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                const double dy = act_deriv_z(act, z[i], slope) * dz[i];
                const double xhat = (act_inv(act, z[i], slope) - beta[c]) / g;
                sdy += dy;
                sdyxh += dy * xhat;
            }
        for (int64_t n = 0; n < N; ++n)
            for (int64_t s = 0; s < HW; ++s) {
                const size_t i = at(layout, C, HW, n, c, s);
                const double dy = act_deriv_z(act, z[i], slope) * dz[i];
                const double xhat = (act_inv(act, z[i], slope) - beta[c]) / g;
                dx[i] = (dy - sdyxh * xhat / m - sdy / m) * g * rstd;
            }
        dbeta[c] = sdy;
        dgamma[c] = sdyxh * gamma_eff_deriv(gamma_mode, gamma[c]);
    }
}

int oracle_mutant_id(void) { return ORACLE_MUTANT; }
