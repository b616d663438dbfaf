/*
 * include/iabn.h -- C ABI of the B200 (sm_100a) InPlace-ABN hot path.
 *
 * In-Place Activated BatchNorm, arXiv 1712.02616.
 * The calls follow the paper's statement of the problem:
 *   forward  (x, gamma, beta) -> z, saving z and sigma_B     Alg. 1
 *   backward (dL/dz, gamma, beta; saved z, sigma_B)
 *            -> (dL/dx, dL/dgamma, dL/dbeta)                  Alg. 2 (variant I)
 *   in-place sharing: z may be x, dL/dx may be dL/dz
 *   synchronized statistics across GPUs (InPlace-ABN^sync)
 *
 * Per channel c (the paper's "unit"), with m = N*H*W values:
 *   mu = (1/m) sum x,  var = (1/m) sum (x - mu)^2
 *   x^ = (x - mu)/sqrt(var + eps)                                     Eq.(1)
 *   y  = g x^ + beta,  g = |gamma| + eps (default; see flags)
 *   z  = f(y) = y (y >= 0), slope*y (y < 0)
 * backward (never reads x):
 *   dy = f'(z) dz (z >= 0 -> 1, else slope);  y = f^-1(z);  x^ = (y - beta)/g
 *   dbeta = sum dy;  dg = sum dy x^;  dgamma = sgn(gamma) dg
 *   dx = (dy - x^ dg/m - dbeta/m) g / sqrt(var + eps)
 *
 * Conventions for every entry point:
 *  - Activations x, z, dz, dx are DEVICE pointers to contiguous tensors of
 *    desc->n * desc->c * desc->hw elements, layout NCHW ([n][c][hw]) or NHWC
 *    ([n][hw][c]), storage dtype f32 or bf16 (arithmetic is always fp32, with
 *    fp64 cross-block / cross-GPU combines).  Base pointers must be 16-byte
 *    aligned.
 *  - Per-channel vectors (gamma, beta, running_*, save_*, dgamma, dbeta) are
 *    DEVICE pointers to fp32 [C].  Statistics buffers of the split-phase API are
 *    DEVICE fp64 arrays.
 *  - All pointers are caller-owned; the library allocates no device memory per
 *    call.  Scratch space is the caller's `ws` of at least
 *    iabn_workspace_bytes(desc) bytes (16-byte aligned, contents undefined on
 *    entry and exit).
 *  - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *    default stream).  Outputs are valid once the stream reaches them.
 *  - Argument validation is synchronous and happens before any launch; on an
 *    error nothing is launched and nothing is written.  Asynchronous device
 *    faults surface at the caller's next synchronisation.  Non-finite data is
 *    propagated, not checked.
 *  - Calls on distinct streams are thread-safe.  Global state: one-time kernel
 *    attribute setup and a thread-local error string (iabn_last_error).
 *  - Results are bitwise reproducible for a fixed (desc, flags, device,
 *    number of ranks): fixed reduction trees, no floating-point atomics.
 */
#ifndef IABN_H
#define IABN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IABN_VERSION 1

#if defined(IABN_BUILD) && defined(__GNUC__)
#define IABN_API __attribute__((visibility("default")))
#else
#define IABN_API
#endif

typedef enum iabn_status {
    IABN_OK = 0,
    IABN_ERR_INVALID_ARG = 1, /* null pointer, n/c/hw <= 0, eps <= 0 or non-finite,
                                 slope outside (0, 1], momentum outside [0, 1] */
    IABN_ERR_UNSUPPORTED = 2, /* misaligned base pointer, unknown dtype/layout, shape too large */
    IABN_ERR_ALIAS = 3,       /* partial overlap of buffers that must be equal or disjoint */
    IABN_ERR_DEGENERATE = 4,  /* training with fewer than 2 values per channel (global count) */
    IABN_ERR_WORKSPACE = 5,   /* ws == NULL or ws_bytes < iabn_workspace_bytes(desc) */
    IABN_ERR_CUDA = 6,        /* a launch failed (cudaGetLastError), or no usable device */
    IABN_ERR_NCCL = 7         /* NCCL unavailable or an NCCL call failed */
} iabn_status;

typedef enum iabn_dtype { IABN_F32 = 0, IABN_BF16 = 1 } iabn_dtype;
typedef enum iabn_layout { IABN_NCHW = 0, IABN_NHWC = 1 } iabn_layout;

/* flags (bitwise or) */
enum {
    /* gamma used as given (caller keeps |gamma| >= 1e-8; PAPER.md:133 needs gamma != 0)
       instead of the default effective scale g = |gamma| + eps. */
    IABN_GAMMA_PLAIN = 1u << 0,
    /* g = 1 ("fixing it to 1"); dgamma still returns dL/dg. */
    IABN_GAMMA_FIXED_ONE = 1u << 1,
    /* running_var tracks the biased batch variance (default: unbiased, var*m/(m-1)). */
    IABN_RUNNING_VAR_BIASED = 1u << 2,
    /* sync backward: return the all-rank sums as dgamma/dbeta (default: this rank's
       contribution, to be summed by the caller's data-parallel gradient reduction). */
    IABN_SYNC_GLOBAL_PARAM_GRADS = 1u << 3,
    /* backward: accumulate per-element products dy*x^ (InPlace-ABN I, Alg. 2 l.5-6).
       Default for the channel-resident schedule is the BN-dagger reduction of
       InPlace-ABN II (Alg. 2 l.7-8): sum dy and sum dy*y, then
       sum dy*x^ = (sum dy*y - beta sum dy)/g per channel -- the same gradient with
       fewer operations per element. */
    IABN_VARIANT_I = 1u << 5,
    /* forward with fixed running statistics (test time): no batch
       statistics, running stats read-only, save_* untouched. */
    IABN_EVAL = 1u << 4,
    /* schedule overrides (testing / benchmarking); default = automatic */
    IABN_FORCE_STREAMING = 1u << 8, /* multi-kernel streaming schedule */
    IABN_FORCE_FUSED = 1u << 9,     /* channel-resident cluster schedule (NCHW; for NHWC the
                                       channel-group schedule); IABN_ERR_UNSUPPORTED when the
                                       shape does not fit on chip */
    /* 1u << 10: reserved (was a one-launch cooperative variant of the streaming schedule,
       measured slower than three launches on every shape and removed) */
    IABN_FORCE_RESIDENT = 1u << 11,   /* NHWC: the whole tensor resident in the grid's shared
                                         memory, one cooperative launch (falls back to
                                         streaming when it does not fit) */
    /* iabn_{forward,backward}_sync: the channel-resident kernels with the cross-rank
       exchange inside the kernel (see "fused-collective sync" below) instead of reduce
       kernels + ncclAllReduce + apply kernels.  Also enabled by env IABN_SYNC_FUSED=1. */
    IABN_SYNC_FUSED = 1u << 12,
    /* Activation f after BN ("sigmoid, hyperbolic tangent, Leaky ReLU, and
       others" are invertible): default leaky ReLU with `slope`; these two select
       f = sigmoid or f = tanh (slope ignored), exclusive.  iabn_forward / iabn_backward
       only (the split-phase and synchronized entries return IABN_ERR_UNSUPPORTED), fp32
       storage only (IABN_ERR_UNSUPPORTED for bf16: the inverse of an 8-bit-mantissa
       sigmoid / tanh output is ill-conditioned); the small-layer and channel-resident
       schedules for NCHW, the channel-group schedule for NHWC (IABN_FORCE_FUSED /
       IABN_FORCE_STREAMING select), streaming otherwise.  The backward
       inverts z: x^ = (f^-1(z) - beta)/g, dy = f'(z) dz (Alg. 2), with z clamped into
       the open range of f first (saturated outputs, R17); variant II sums
       dy y and forms (Q - beta S1)/g per channel, IABN_VARIANT_I sums dy x^. */
    IABN_ACT_SIGMOID = 1u << 13,
    IABN_ACT_TANH = 1u << 14
};

typedef struct iabn_desc {
    int64_t n;      /* batch */
    int64_t c;      /* channels */
    int64_t hw;     /* height * width */
    int32_t dtype;  /* iabn_dtype: storage of x, z, dz, dx */
    int32_t layout; /* iabn_layout; contiguous only */
} iabn_desc;

/* Opaque communicator for the synchronized variant (owns one ncclComm_t). */
typedef struct iabn_comm_s *iabn_comm;

/* ------------------------------------------------------------------ queries */
IABN_API int iabn_version(void);
IABN_API const char *iabn_status_string(iabn_status s);
/* Thread-local detail text of the last non-OK status returned on this thread. */
IABN_API const char *iabn_last_error(void);
/* Number of kernels this process has launched through the library (all threads). */
IABN_API uint64_t iabn_launch_count(void);
/* Workspace bytes needed by every call on `desc` (0 if desc is invalid). */
IABN_API size_t iabn_workspace_bytes(const iabn_desc *desc);
/* Schedule the library would use: pass 0 = forward, 1 = backward.  On return
   *schedule is 0 (streaming), 1 (channel-resident fused), 3 (grid-resident NHWC:
   the whole tensor in the grid's shared memory), 4 (NHWC channel groups: a cluster holds
   a column group of all rows, 2-D TMA) or 5 (small NCHW layers held in registers); 2 is
   no longer returned,
   *cluster the CTAs per channel of the fused schedule (0 otherwise). */
IABN_API iabn_status iabn_query_schedule(const iabn_desc *desc, int pass, uint32_t flags, int *schedule,
                                int *cluster);

/* ------------------------------------------------------------------ forward
 * Alg. 1.  x: input [E]; z: output [E], z == x (in place) or
 * disjoint from x.  gamma, beta: [C].  running_mean/running_var: [C] in/out
 * (updated r <- (1-momentum) r + momentum*batch; pass both NULL to skip).
 * save_mean/save_var: [C] out, batch mean and BIASED batch variance (the sigma_B
 * of Alg. 1 l.3; the backward needs only save_var).  With IABN_EVAL: running
 * stats are inputs, save_* may be NULL.  eps > 0 and finite, slope in (0, 1],
 * momentum in [0, 1]. */
IABN_API iabn_status iabn_forward(const iabn_desc *desc, const void *x, void *z, const float *gamma,
                         const float *beta, float *running_mean, float *running_var,
                         float *save_mean, float *save_var, float momentum, float eps,
                         float slope, uint32_t flags, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ backward
 * Alg. 2 variant I: reads z and dz only, never x.
 * z: forward output [E] (read-only; must not overlap dx).  dz: dL/dz [E].
 * dx: dL/dx [E] out, dx == dz (in place) or disjoint.  save_var: [C] from the
 * forward; save_mean is accepted for symmetry and unused, may be
 * NULL.  dgamma, dbeta: [C] out (overwritten, not accumulated). */
IABN_API iabn_status iabn_backward(const iabn_desc *desc, const void *z, const void *dz, void *dx,
                          const float *gamma, const float *beta, const float *save_mean,
                          const float *save_var, float *dgamma, float *dbeta, float eps,
                          float slope, uint32_t flags, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ synchronized variant
 * Batch statistics span all ranks of `comm` (InPlace-ABN^sync):
 * per-channel (count, sum, sum of squares) are summed over ranks in fp64 with
 * ncclAllReduce on `stream` between the reduction and the apply kernels; the
 * backward sums (sum dy, sum dy x^) likewise.  Shards may have different n.
 * nranks == 1 takes the non-synchronized path (no collective).
 * NCCL is loaded at run time (libnccl.so.2); without it these return
 * IABN_ERR_NCCL.  id: 128 opaque bytes from rank 0, distributed by the caller. */
IABN_API iabn_status iabn_comm_get_unique_id(unsigned char id[128]);
/* Must be called with the CUDA device of this rank current (cudaSetDevice). */
IABN_API iabn_status iabn_comm_init(iabn_comm *out, int nranks, int rank, const unsigned char id[128]);
IABN_API iabn_status iabn_comm_destroy(iabn_comm comm);
IABN_API iabn_status iabn_forward_sync(const iabn_desc *desc, const void *x, void *z, const float *gamma,
                              const float *beta, float *running_mean, float *running_var,
                              float *save_mean, float *save_var, float momentum, float eps,
                              float slope, uint32_t flags, void *ws, size_t ws_bytes,
                              void *stream, iabn_comm comm);
IABN_API iabn_status iabn_backward_sync(const iabn_desc *desc, const void *z, const void *dz, void *dx,
                               const float *gamma, const float *beta, const float *save_mean,
                               const float *save_var, float *dgamma, float *dbeta, float eps,
                               float slope, uint32_t flags, void *ws, size_t ws_bytes,
                               void *stream, iabn_comm comm);

/* Per-phase device time of the synchronized calls (measurement; SURVEY.md section 8(d)
 * item 3).  With timing on, iabn_forward_sync / iabn_backward_sync record CUDA events
 * on their stream around [local reduction | all-reduce | apply] (the all-reduce is the
 * library's own ncclAllReduce call); iabn_comm_phase_ms waits for the last recorded
 * events and writes ms[6] = forward {reduce, all-reduce, apply}, backward {reduce,
 * all-reduce, apply} of the most recent calls (-1 where a pass has not run since timing
 * was switched on).  The fused-collective kernels exchange inside the kernel: their
 * whole pass is reported as "reduce", all-reduce and apply as 0.  Off by default (the
 * events cost ~1 us per phase and break the PDL overlap between the phases).
 * Errors: IABN_ERR_INVALID_ARG (NULL comm / ms), IABN_ERR_CUDA. */
IABN_API iabn_status iabn_comm_set_timing(iabn_comm comm, int on);
IABN_API iabn_status iabn_comm_phase_ms(iabn_comm comm, float ms[6]);

/* ------------------------------------------------------------------ fused-collective sync
 * With IABN_SYNC_FUSED (NCHW shapes the channel-resident schedule takes, at most 8
 * ranks on one node) iabn_{forward,backward}_sync run ONE kernel per pass: each rank
 * keeps its shard's channel slab in shared memory while the cluster owning channel c
 * stores its record -- (count, sum x, sum x^2) forward, (sum dy, sum dy y) backward,
 * fp64 -- into every rank's record buffer over NVLink (CUDA IPC mappings, exchanged
 * with ncclAllGather at the first call and whenever C grows: collective), waits for the
 * nranks records of c, folds them in rank order (bit-identical on every rank) and
 * writes its outputs from the still-resident slab: 2*E*b forward and 3*E*b backward
 * HBM bytes instead of 3*E*b / 5*E*b, no separate collective launch.  Requirements
 * (the caller's, as for NCCL counts): every rank calls with the same desc (equal
 * shards) and flags, in the same order.  A rank that never makes the call makes the
 * others trap after ~20 s instead of hanging.  Shapes the fused schedule cannot take
 * use the reduce / all-reduce / apply path.
 *
 * One-GPU emulation (tests and single-GPU measurement of the same kernels and record
 * protocol): the nranks shards of one tensor -- x, z, dz, dx hold nranks * desc->n
 * samples, shard r = samples [r n, (r+1) n) -- processed by one cooperative launch whose
 * clusters are split among virtual ranks that exchange records through local memory.
 * desc describes ONE shard.  Outputs: z / dx over the whole tensor; save_mean/save_var
 * and the running statistics once ([C], global); dgamma/dbeta [nranks][C] (row r = shard
 * r's contribution, or the global sums in every row with IABN_SYNC_GLOBAL_PARAM_GRADS).
 * Exchange buffers are library-owned, per (device, stream); the first call of a
 * (stream, nranks, larger C) allocates them synchronously (not inside a graph capture).
 * Errors: as iabn_forward / iabn_backward (workspace sized for the whole tensor), plus
 * IABN_ERR_INVALID_ARG (nranks outside [1, 8], IABN_EVAL) and IABN_ERR_UNSUPPORTED
 * (NHWC, or a shard the channel-resident schedule cannot take). */
IABN_API iabn_status iabn_forward_sync_emulated(const iabn_desc *desc, int nranks, const void *x,
                                                void *z, const float *gamma, const float *beta,
                                                float *running_mean, float *running_var,
                                                float *save_mean, float *save_var, float momentum,
                                                float eps, float slope, uint32_t flags, void *ws,
                                                size_t ws_bytes, void *stream);
IABN_API iabn_status iabn_backward_sync_emulated(const iabn_desc *desc, int nranks, const void *z,
                                                 const void *dz, void *dx, const float *gamma,
                                                 const float *beta, const float *save_mean,
                                                 const float *save_var, float *dgamma,
                                                 float *dbeta, float eps, float slope,
                                                 uint32_t flags, void *ws, size_t ws_bytes,
                                                 void *stream);

/* ------------------------------------------------------------------ split phase
 * The sync path in pieces, for callers with their own collective (e.g. a
 * torch.distributed process group) and for one-process multi-shard tests.
 * stats: fp64 [C][3] = (count, sum x, sum x^2) of this rank; sum them over
 * ranks, then pass the global array to iabn_forward_apply.
 * sums: fp64 [2C + 1] = ([C][2] = (sum dy, sum dy x^), then count m of this
 * rank); sum over ranks, then pass global and local arrays to
 * iabn_backward_apply (dgamma/dbeta come from sums_local unless
 * IABN_SYNC_GLOBAL_PARAM_GRADS). */
IABN_API iabn_status iabn_forward_reduce(const iabn_desc *desc, const void *x, double *stats, void *ws,
                                size_t ws_bytes, void *stream);
IABN_API iabn_status iabn_forward_apply(const iabn_desc *desc, const void *x, void *z,
                               const double *stats_global, const float *gamma,
                               const float *beta, float *running_mean, float *running_var,
                               float *save_mean, float *save_var, float momentum, float eps,
                               float slope, uint32_t flags, void *ws, size_t ws_bytes,
                               void *stream);
IABN_API iabn_status iabn_backward_reduce(const iabn_desc *desc, const void *z, const void *dz,
                                 const float *gamma, const float *beta, double *sums,
                                 float eps, float slope, uint32_t flags, void *ws,
                                 size_t ws_bytes, void *stream);
IABN_API iabn_status iabn_backward_apply(const iabn_desc *desc, const void *z, const void *dz, void *dx,
                                const double *sums_global, const double *sums_local,
                                const float *gamma, const float *beta, const float *save_var,
                                float *dgamma, float *dbeta, float eps, float slope,
                                uint32_t flags, void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ test time
 * Absorb the test-time BN of a Conv layer's output channels into the Conv's
 * weights and bias ("absorbing BN parameters into the preceding
 * Conv layer ... at test-time BN becomes a linear operation").
 * Per output channel k, with s_k = g_k / sqrt(running_var_k + eps) and g the
 * effective scale of the flags (|gamma|+eps default, gamma with GAMMA_PLAIN, 1
 * with GAMMA_FIXED_ONE):
 *   w_out[k][j] = s_k * w[k][j]                 (j < k_per_out, row-major [cout][k])
 *   bias_out[k] = s_k * (bias[k] - running_mean[k]) + beta[k]     (bias NULL = 0)
 * so that conv(x; w_out, bias_out) = BN_eval(conv(x; w, bias)).  The activation
 * is not folded (it is not linear).  All pointers are fp32 DEVICE arrays; w_out
 * may be w and bias_out may be bias (in place), any other overlap is
 * IABN_ERR_ALIAS.  Errors: IABN_ERR_INVALID_ARG (NULL required pointer, cout or
 * k_per_out <= 0, eps <= 0 or non-finite), IABN_ERR_UNSUPPORTED (misaligned w
 * / w_out: 16 bytes), IABN_ERR_CUDA.  s_k is formed in fp64, then rounded. */
IABN_API iabn_status iabn_fold_conv(int64_t cout, int64_t k_per_out, const float *w,
                                    const float *bias, const float *running_mean,
                                    const float *running_var, const float *gamma,
                                    const float *beta, float eps, uint32_t flags, float *w_out,
                                    float *bias_out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* IABN_H */
