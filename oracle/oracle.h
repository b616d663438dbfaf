/*
 * oracle/oracle.h -- TEST INFRASTRUCTURE ONLY (see oracle.c).  This header is
 * private to oracle/ and shares nothing with include/iabn.h.
 */
#ifndef IABN_ORACLE_H
#define IABN_ORACLE_H
#include <stdint.h>

#define ORACLE_NCHW 0
#define ORACLE_NHWC 1

#define ORACLE_GAMMA_ABS_EPS 0   /* gamma~ = |gamma| + eps (default, R4) */
#define ORACLE_GAMMA_PLAIN 1     /* gamma~ = gamma */
#define ORACLE_GAMMA_FIXED_ONE 2 /* gamma~ = 1 */

#define ORACLE_ACT_LEAKY 0   /* leaky ReLU with slope a (the paper's choice) */
#define ORACLE_ACT_SIGMOID 1
#define ORACLE_ACT_TANH 2

void oracle_channel_stats(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                          double *mean, double *var);
void oracle_forward(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                    const double *gamma, const double *beta, int gamma_mode, double eps,
                    double slope, double momentum, int running_var_biased,
                    double *running_mean, double *running_var, double *z,
                    double *mean_out, double *var_out);
void oracle_forward_eval(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                         const double *gamma, const double *beta, int gamma_mode, double eps,
                         double slope, const double *running_mean, const double *running_var,
                         double *z);
void oracle_backward_standard(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                              const double *dz, const double *gamma, const double *beta,
                              int gamma_mode, double eps, double slope, double *dx,
                              double *dgamma, double *dbeta);
void oracle_backward_inplace_I(int64_t N, int64_t C, int64_t HW, int layout, const double *z,
                               const double *dz, const double *var, const double *gamma,
                               const double *beta, int gamma_mode, double eps, double slope,
                               double *dx, double *dgamma, double *dbeta);
void oracle_backward_inplace_II(int64_t N, int64_t C, int64_t HW, int layout, const double *z,
                                const double *dz, const double *var, const double *gamma,
                                const double *beta, int gamma_mode, double eps, double slope,
                                double *dx, double *dgamma, double *dbeta);
void oracle_merge_stats(int64_t K, int64_t C, const double *counts, const double *means,
                        const double *vars, double *count_out, double *mean_out,
                        double *var_out);
void oracle_fold_conv(int64_t cout, int64_t kper, const double *w, const double *bias,
                      const double *running_mean, const double *running_var,
                      const double *gamma, const double *beta, int gamma_mode, double eps,
                      double *w_out, double *bias_out);
void oracle_param_grads_sharded(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                                const double *dz, const double *gamma, const double *beta,
                                int gamma_mode, double eps, double slope, int64_t nshards,
                                const int64_t *shard_n, double *dgamma, double *dbeta);
void oracle_forward_act(int64_t N, int64_t C, int64_t HW, int layout, const double *x,
                        const double *gamma, const double *beta, int gamma_mode, double eps,
                        int act, double slope, double *z, double *mean_out, double *var_out);
void oracle_backward_standard_act(int64_t N, int64_t C, int64_t HW, int layout,
                                  const double *x, const double *dz, const double *gamma,
                                  const double *beta, int gamma_mode, double eps, int act,
                                  double slope, double *dx, double *dgamma, double *dbeta);
void oracle_backward_inplace_act(int64_t N, int64_t C, int64_t HW, int layout, const double *z,
                                 const double *dz, const double *var, const double *gamma,
                                 const double *beta, int gamma_mode, double eps, int act,
                                 double slope, double *dx, double *dgamma, double *dbeta);
int oracle_mutant_id(void);
#endif
