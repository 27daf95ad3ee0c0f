/*
 * libsimopt_b200 -- C ABI of the B200-native (sm_100a) hot path of the
 * arXiv 2404.11631 simulation-optimization benchmark ("sobench").
 *
 * Every entry point takes plain device pointers and sizes plus a cudaStream_t
 * (passed as void*), enqueues its kernels on that stream and returns a status
 * code; results are valid once the stream reaches that point.  No entry point
 * synchronises the device unless documented.  Pointers are caller-owned device
 * memory (e.g. torch CUDA tensors); arrays are C-contiguous float64 unless noted.
 *
 * Reference interfaces replaced (paths relative to reference pkg/src/sobench):
 *   sampling.py  RngStream/uniform01/standard_normal/sample_returns/
 *                sample_demands/sample_indices/synth_classification
 *   backend.py   Backend.dot/vec_sum/matvec/matvec_t/axpy/map_kernel
 *   _kernels.py  fold_pairwise .. ecdf_count_block (the 14 numba kernels)
 *   tasks.py     build_sample_set, mv_objective/mv_gradient, nv_gradient_hat,
 *                nv_objective_exact, logistic_loss/gradient/hvp
 *   lmo.py       lmo_simplex_slack, lmo_single_budget
 *   frank_wolfe.py fw_step_size/fw_update
 *   sqn.py       hessian_update (bfgs_rank2_block)
 * Status codes map one-to-one onto sobench/errors.py exception classes.
 */
#ifndef SIMOPT_B200_H
#define SIMOPT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum simopt_status {
  SIMOPT_OK = 0,
  SIMOPT_E_DIMENSION = 1,          /* errors.DimensionMismatch      (errors.py:8)  */
  SIMOPT_E_CONFIG = 2,             /* errors.ConfigurationError     (errors.py:12) */
  SIMOPT_E_EMPTY = 3,              /* errors.EmptyRequest           (errors.py:16) */
  SIMOPT_E_INSUFFICIENT = 4,       /* errors.InsufficientSamples    (errors.py:20) */
  SIMOPT_E_INVALID_GRADIENT = 5,   /* errors.InvalidGradient        (errors.py:24) */
  SIMOPT_E_INVALID_CONSTRAINT = 6, /* errors.InvalidConstraint      (errors.py:28) */
  SIMOPT_E_SOLVER_STALL = 7,       /* errors.SolverStall            (errors.py:32) */
  SIMOPT_E_DEGENERATE_PAIR = 8,    /* errors.DegeneratePair         (errors.py:40) */
  SIMOPT_E_CUDA = 9                /* CUDA runtime failure (no reference analogue) */
};

/* Map-kernel ids for simopt_map_kernel (backend.py:34, MAP_KERNELS). */
enum simopt_map { SIMOPT_MAP_SIGMOID = 0, SIMOPT_MAP_NEGATE = 1, SIMOPT_MAP_EXP = 2 };

const char* simopt_last_error(void);
int simopt_abi_version(void);
/* Write the device %globaltimer (ns) to *out when the stream reaches this point. */
int simopt_timestamp(void* stream, int64_t* out);

/* Measurement (bench.py roofline.compute_roof): Philox4x64-10 blocks clo+1 .. clo+nblocks
 * of key (seed, sid), counter word 1 = 0, through the newsvendor resample's Philox core
 * with the words XOR-folded per thread into out[0 .. 8*SMs*256) -- the arithmetic floor of
 * a resample of nblocks blocks (nothing stored per block). */
int simopt_philox_floor(void* stream, uint64_t seed, uint64_t sid, uint64_t clo, int64_t nblocks,
                        uint64_t* out, int64_t out_len);

/* ------------------------------------------------------------ sampling.py */
/* uniform01 (sampling.py:87-102): n doubles of stream (seed, stream_id) at the
 * 128-bit block counter (ctr_hi:ctr_lo).  The caller advances the counter by
 * ceil(n/4).  Bit-identical to numpy Philox4x64-10 + Generator.random. */
int simopt_uniform01(void* stream, uint64_t seed, uint64_t stream_id, uint64_t ctr_lo,
                     uint64_t ctr_hi, int64_t n, double* out);

/* standard_normal (sampling.py:105-120): n normals from 2*ceil(n/2) uniforms via
 * Box-Muller with glibc-2.39-exact log1p/sin/cos (_kernels.py:178-190).  The
 * caller advances the counter by ceil(2*ceil(n/2)/4). */
int simopt_standard_normal(void* stream, uint64_t seed, uint64_t stream_id, uint64_t ctr_lo,
                           uint64_t ctr_hi, int64_t n, double* out);

/* sample_returns diag path (sampling.py:156-166): out[i*d+j] = mu[j] + sigma[j]*z[i*d+j]. */
int simopt_sample_returns_diag(void* stream, uint64_t seed, uint64_t stream_id, uint64_t ctr_lo,
                               uint64_t ctr_hi, int64_t n_samples, int64_t d, const double* mu,
                               const double* sigma, double* out);

/* Rows [row_lo, row_hi) of the diag sample_returns draw at the stream position (the
 * values the full n_samples x d draw has there): sample sharding, no RNG
 * communication.  out is (row_hi - row_lo) x d. */
int simopt_sample_returns_diag_rows(void* stream, uint64_t seed, uint64_t stream_id, uint64_t ctr_lo,
                                    uint64_t ctr_hi, int64_t row_lo, int64_t row_hi, int64_t d,
                                    const double* mu, const double* sigma, double* out);
/* Elements [e_lo, e_hi) of simopt_bernoulli_half's draw (row shards of the features). */
int simopt_bernoulli_half_range(void* stream, uint64_t seed, uint64_t stream_id, uint64_t ctr_lo,
                                uint64_t ctr_hi, int64_t e_lo, int64_t e_hi, double* out);

/* synth_classification features (sampling.py:246-255): out[i] = (u_i >= 0.5) as 0.0/1.0
 * for the n uniforms of the stream at the counter.  Caller advances by ceil(n/4). */
int simopt_bernoulli_half(void* stream, uint64_t seed, uint64_t stream_id, uint64_t ctr_lo,
                          uint64_t ctr_hi, int64_t n, double* out);
/* out[i] = (x[i] > thr) as 0.0/1.0 (sampling.py:261). */
int simopt_threshold(void* stream, const double* x, double thr, int64_t n, double* out);

/* ------------------------------------------------------------ backend.py */
/* Fixed-tree reductions (backend.py:80-141, _kernels.py:30-156): chunk-local
 * strictly sequential sums, chunk partials folded pairwise in index order.
 * Bit-identical to SequentialBackend/ParallelBackend for every chunk >= 1.
 * Scalar results are written to device memory (*out). */
int simopt_dot(void* stream, const double* x, const double* y, int64_t n, int64_t chunk,
               double* out);
int simopt_vec_sum(void* stream, const double* x, int64_t n, int64_t chunk, double* out);
/* Deterministic dot in one CTA (fixed strided assignment, fixed xor trees; no FMA) -- not the
 * reference's tree: the fused Newton-CG's scalars (d-vectors), where the tree's sequential
 * chunk chain is the cost.  Meant for n up to ~10^5. */
int simopt_dot_fast(void* stream, const double* x, const double* y, int64_t n, double* out);
/* Column sums out[c] = sum_r x[r][c] of a row-major rows x cols matrix in a fixed order
 * (256 row groups summed sequentially, then folded in group order): deterministic, not the
 * reference's tree -- the fused mean-variance path's sample mean at small N (C1), where the
 * tree's 4096-long chains are latency-bound. */
int simopt_col_sums_fast(void* stream, const double* x, int64_t rows, int64_t cols, double* out);
/* Two independent fixed-tree reductions in one launch: out_k = dot(x_k, y_k) (y_k != NULL)
 * or vec_sum(x_k) (y_k == NULL). */
int simopt_tree_sums2(void* stream, const double* x0, const double* y0, int64_t n0, double* out0,
                      const double* x1, const double* y1, int64_t n1, double* out1, int64_t chunk);
/* out[r] = fixed-tree dot of (a[row(r),:] - center) with x, row(r) = rows_idx ? rows_idx[r] : r.
 * center (length cols) and rows_idx (length rows, int64) may be NULL. */
int simopt_matvec(void* stream, const double* a, int64_t lda_rows, int64_t cols,
                  const int64_t* rows_idx, int64_t rows, const double* center, const double* x,
                  int64_t chunk, double* out);
/* out[j] = fixed-tree sum over r of x[r] * (a[row(r),j] - center[j]). */
int simopt_matvec_t(void* stream, const double* a, int64_t lda_rows, int64_t cols,
                    const int64_t* rows_idx, int64_t rows, const double* center,
                    const double* x, int64_t chunk, double* out);
int simopt_axpy(void* stream, double alpha, const double* x, const double* y, int64_t n,
                double* out);
int simopt_map_kernel(void* stream, int kernel, const double* x, int64_t n, double* out);
/* axpy with alpha read from device memory when the kernel runs (CUDA-graph replay of
 * Frank-Wolfe epochs whose step sizes change per epoch). */
int simopt_axpy_ptr(void* stream, const double* alpha, const double* x, const double* y, int64_t n,
                    double* out);
/* out = x*alpha - y elementwise (y may be NULL), e.g. tasks.py:62 and :85 epilogues. */
int simopt_scale_sub(void* stream, const double* x, double alpha, const double* y, int64_t n,
                     double* out);

/* ------------------------------------------------------------ lmo.py */
/* lmo_simplex_slack (lmo.py:56-65) and lmo_single_budget (lmo.py:68-89):
 * s_out = vertex (one-hot or zero).  A NaN in g ORs SIMOPT_E_INVALID_GRADIENT
 * into *status (device int, caller-zeroed) instead of failing synchronously.
 * Positivity of c is the caller's precondition (checked once per instance). */
int simopt_lmo_simplex_slack(void* stream, const double* g, int64_t n, double* s_out, int* status);
int simopt_lmo_single_budget(void* stream, const double* g, const double* c, double budget,
                             int64_t n, double* s_out, int* status);

/* *out = min(x) (NaN-propagating): feasibility all(w >= -tol) (tasks.py:289-290, :327-328). */
int simopt_min_value(void* stream, const double* x, int64_t n, double* out);

/* ------------------------------------------------------------ newsvendor */
/* Segment length and buckets per segment of the keyed demand layout. */
int simopt_nv_geometry(int64_t* seg, int64_t* buckets);
/* Epoch layout sizes: keys d*S u32,
 * bucket starts d*nseg*buckets u16, nseg = ceil(S/seg). */
int simopt_nv_layout(int64_t d, int64_t S, int64_t* nseg, int64_t* key_elems, int64_t* off_elems);

/* sample_demands (sampling.py:173-193) in the keyed ECDF layout: one u32 key per
 * draw D[j,s] = mu_j + sigma_j*z[j*S+s] (z = standard_normal(d*S) of the stream at
 * the given counter), counting-sorted by bucket per segment.  Every ECDF count
 * computed from it equals the count on the reference's sorted rows.  Caller
 * advances the counter by ceil(2*ceil(d*S/2)/4) and passes the same
 * (seed, stream_id, ctr) to every query of this epoch. */
int simopt_nv_resample(void* stream, uint64_t seed, uint64_t stream_id, uint64_t ctr_lo,
                       uint64_t ctr_hi, int64_t d, int64_t S, uint32_t* keys, uint16_t* off);

/* ECDF counts #{D[j,:] <= x_j} (ecdf_count_block, _kernels.py:245-259). */
int simopt_nv_counts(void* stream, const uint32_t* keys, const uint16_t* off, const double* mu,
                     const double* sigma, int64_t d, int64_t S, uint64_t seed, uint64_t stream_id,
                     uint64_t ctr_lo, uint64_t ctr_hi, const double* x, int64_t* counts);

/* Largest |z~ - z| between the key's fp32 approximation and the exact normal over the
 * first n normals of the draw (*out_max device double); *eps (host) = the bound the
 * ECDF queries rely on. */
int simopt_nv_approx_error(void* stream, uint64_t seed, uint64_t stream_id, uint64_t ctr_lo,
                           uint64_t ctr_hi, int64_t n, double* out_max, double* eps);

/* Exact demand value of every stored key, in storage order (diagnostics / tests). */
int simopt_nv_decode(void* stream, const uint32_t* keys, const double* mu, const double* sigma,
                     int64_t d, int64_t S, uint64_t seed, uint64_t stream_id, uint64_t ctr_lo,
                     uint64_t ctr_hi, double* out);

/* ecdf_count_block on reference-format rows (each row sorted ascending). */
int simopt_ecdf_count_sorted(void* stream, const double* samples, int64_t rows, int64_t s,
                             const double* x, int64_t* counts);
/* nv_gradient_hat epilogue (tasks.py:158-160): g = (k - v) + ((h + v) * (counts / S)). */
int simopt_nv_grad_from_counts(void* stream, const int64_t* counts, int64_t S, const double* k,
                               const double* h, const double* v, int64_t d, double* g);
/* nv_gradient_exact (tasks.py:163-171): (k - v) + ((h + v) * Phi((x - mu) / sigma)), the
 * CDF as normal_cdf_block (_kernels.py:204-207) with glibc's erf. */
int simopt_nv_grad_exact(void* stream, const double* x, const double* mu, const double* sigma,
                         const double* k, const double* h, const double* v, int64_t d, double* g);

/* Device-resident FW state for one newsvendor run. */
typedef struct NvState {
  int64_t jstar;          /* LMO vertex index of the last gradient            */
  double sval;            /* vertex value C/c_j* if g_j* < 0 else 0            */
  unsigned blocks_done;   /* last-block-done counter (kept 0 between launches) */
  unsigned pad;           /* product counter of gradient steps (kept 0 between launches) */
  double best_val;        /* LMO value g_j* (C/c_j*) of the vertex (shard exchange) */
  int64_t exchange_failed; /* sticky: a peer exchange timed out; later ones do not wait */
} NvState;

#define NV_FLAG_NAN_GRADIENT 1 /* InvalidGradient at this step's LMO (lmo.py:78-79) */
#define NV_FLAG_NEGATIVE 2     /* iterate < -FEAS_TOL after this step (tasks.py:328) */
#define NV_FLAG_EXCHANGE_TIMEOUT 4 /* peer-memory LMO exchange gave up (a peer never arrived) */

/* One fused FW kernel (frank_wolfe.py:106-117 for NewsvendorProblem):
 *  do_update: x <- (gamma*((-1*x) + s)) + x with the vertex in *state, objective
 *             terms (newsvendor_cost_block) into terms[] unless terms == NULL,
 *             flags[step] |= NEGATIVE;
 *  do_grad:   g = nv_gradient_hat(x) (tasks.py:141-160), LMO argmin of
 *             g*(budget/c) (lmo.py:68-89) into *state, flags[grad_step] |= NAN. */
typedef struct NvIterArgs {
  int64_t d, S, nseg;
  const uint32_t* keys;       /* epoch layout (simopt_nv_resample)          */
  const uint16_t* off;
  uint64_t seed, sid, ctr_lo, ctr_hi;  /* the epoch's draw (exact fallback) */
  const double *mu, *sigma, *k, *h, *v, *c;
  double budget;
  const double* x_in; /* iterate before this step                               */
  double* x;          /* iterate after this step (== x_in when do_update == 0)  */
  double* g;
  double* terms;
  double gamma;
  int do_update, do_grad;
  int64_t step, grad_step;
  int* flags;
  NvState* state;
  double* part_v;
  int64_t* part_i;
  int64_t part_capacity;
  /* Product-sharded LMO fused into the step over NVLink peer memory (NULL: off).
   * peer_mb[q] = rank q's mailbox (simopt_peer_*), mailbox layout
   * [2 parities][world][4]: {value, global index, vertex value, sequence}.  The last
   * block publishes this rank's argmin to every peer, waits for all `world` entries
   * of sequence `seq`, and applies the global first-argmin (as simopt_nv_lmo_apply). */
  double* const* peer_mb;
  int64_t world, rank, j0;
  uint64_t seq;
  /* Device-resident step parameters (CUDA-graph replay of whole epochs; NULL: use the
   * by-value fields above): epoch_draw = {seed, sid, ctr_lo, ctr_hi} of the epoch's draw;
   * epoch_ctr -> epoch k, gamma = 2 / (k * inner_iters + m + 2) (frank_wolfe.py:62-66);
   * seq_ptr -> the peer exchange sequence, incremented by the step's last block. */
  const uint64_t* epoch_draw;
  const int64_t* epoch_ctr;
  int64_t inner_iters, m;
  uint64_t* seq_ptr;
  /* When non-NULL, the step's last block writes %globaltimer here once the step is
   * complete (the per-step elapsed time of the FW record, frank_wolfe.py:116). */
  int64_t* stamp;
} NvIterArgs;
int simopt_nv_iter(void* stream, const NvIterArgs* args);

/* The recorded quantities of M consecutive newsvendor FW steps in one launch
 * (frank_wolfe.py:110-117 for NewsvendorProblem): iterate m is row (r0 + m) % H of xs
 * (H rows of d doubles); spent[m] = fixed-tree dot(c, x_m) (check_feasible, tasks.py:326)
 * and objs[m] = fixed-tree sum of newsvendor_cost_block(x_m) (tasks.py:171-173,
 * _kernels.py:210-223) -- bit for bit what simopt_nv_cost_terms followed by
 * simopt_tree_sums2 give, with chunk_size `chunk`. */
int simopt_nv_epoch_records(void* stream, const double* xs, int64_t H, int64_t r0, int64_t M,
                            const double* c, const double* mu, const double* sigma,
                            const double* unit, const double* hold, const double* sell, int64_t d,
                            int64_t chunk, double* spent, double* objs);

/* Peer mailboxes (CUDA IPC over NVLink/NVSwitch): alloc returns a zeroed device buffer and
 * its 64-byte IPC handle; open maps a peer's handle (cudaIpcMemLazyEnablePeerAccess);
 * close/free release them. */
int simopt_peer_alloc(int64_t bytes, void** ptr, void* handle64);
int simopt_peer_open(const void* handle64, void** ptr);
int simopt_peer_close(void* ptr);
int simopt_peer_free(void* ptr);

/* Product-sharded LMO: every rank owns products [j0, j0 + d_local).
 * pack: send[0..2] = {best_val, j* + j0, sval} of this rank's k_nv_iter argmin.
 * apply: recv = the world ranks' packs in rank order; the global first-argmin
 * (lexicographic (value, global index), i.e. np.argmin over the full vector, lmo.py:84)
 * is written back: state->jstar = global j* - j0 if this rank owns it else -1,
 * state->sval = its vertex value. */
int simopt_nv_lmo_pack(void* stream, const NvState* state, int64_t j0, double* send);
int simopt_nv_lmo_apply(void* stream, const double* recv, int64_t world, int64_t j0,
                        int64_t d_local, NvState* state);

/* newsvendor_cost_block (_kernels.py:210-223): out[j] = expected cost of product j. */
int simopt_nv_cost_terms(void* stream, const double* x, const double* mu, const double* sigma,
                         const double* unit, const double* hold, const double* sell, int64_t d,
                         double* out);

/* ------------------------------------------------------------ logistic / SQN */
/* c - z[idx] with c = sigmoid(t) (tasks.py:235-236); idx may be NULL. */
int simopt_logistic_resid(void* stream, const double* t, const double* z, const int64_t* idx,
                          int64_t n, double* out);
/* (c * (1 - c)) * tv with c = sigmoid(t) (tasks.py:250-252). */
int simopt_logistic_hvp_weights(void* stream, const double* t, const double* tv, int64_t n,
                                double* out);
/* logistic_loss_block (_kernels.py:193-201) with z[idx]; idx may be NULL. */
int simopt_logistic_loss_terms(void* stream, const double* t, const double* z, const int64_t* idx,
                               int64_t n, double* out);
/* bfgs_rank2_block over all rows (_kernels.py:226-242), h is n x n row-major. */
int simopt_bfgs_rank2(void* stream, double* h, const double* s, const double* u, double coef_su,
                      double coef_ss, int64_t n);
/* The same update with coef_su = -rho and coef_ss = (rho*rho)*(*kappa) + rho formed on the
 * device from kappa = y.(H y) (sqn.py:100-109): no host read between pairs. */
int simopt_bfgs_rank2_dev(void* stream, double* h, const double* s, const double* u, double rho,
                          const double* kappa, int64_t n);
/* h = diag(v) (sqn.py:96-97). */
int simopt_diag_fill(void* stream, double* h, int64_t n, double v);
enum simopt_vec { SIMOPT_VEC_SUB_SCALED = 0, SIMOPT_VEC_ADD = 1, SIMOPT_VEC_SUB = 2,
                  SIMOPT_VEC_SCALE = 3, SIMOPT_VEC_MUL = 4 };
/* out = x - alpha*y | x + y | x - y | x*alpha | x*y (numpy order, no FMA). */
int simopt_vec_op(void* stream, int op, double alpha, const double* x, const double* y, int64_t n,
                  double* out);
/* sample_indices (sampling.py:196-209) on the device for b <= 4096: out[0..b) of the
 * partial Fisher-Yates driven by uniform01(stream at counter, b).  Caller advances
 * the counter by ceil(b/4). */
int simopt_sample_indices(void* stream, uint64_t seed, uint64_t stream_id, uint64_t ctr_lo,
                          uint64_t ctr_hi, int64_t n, int64_t b, int64_t* out);
/* Device-resident SQN iteration (CUDA-graph replay of sqn.py:132-169).
 * sample_indices_dev: as simopt_sample_indices with (seed, stream_id, ctr_lo, ctr_hi) read
 * from device words[4], the counter advanced there by ceil(b/4) (RngStream.advance).
 * SqnCtl: k = the iteration being taken (1-based), rec = next trace row, beta.
 * sqn_step: out = x - (beta / k) * y (sqn.py:160-165).  sqn_record: sums[rec] = *val,
 * stamps[rec] = %globaltimer, then rec += 1, k += 1. */
typedef struct SqnCtl {
  int64_t k, rec;
  double beta;
  int64_t pad;
} SqnCtl;
int simopt_sample_indices_dev(void* stream, uint64_t* words, int64_t n, int64_t b, int64_t* out);
int simopt_sqn_step(void* stream, const SqnCtl* ctl, const double* x, const double* y, int64_t n,
                    double* out);
int simopt_sqn_record(void* stream, SqnCtl* ctl, const double* val, double* sums, int64_t* stamps);
/* lmo_general (lmo.py:92-160): argmin of s.g over {A s <= C, s >= 0} (A m x n row-major,
 * C > 0) by the reference's dense Bland simplex, one CTA, same pivots and arithmetic.
 * *status (device) = 0, SIMOPT_E_INVALID_GRADIENT (NaN in g), SIMOPT_E_SOLVER_STALL
 * (unbounded) or -SIMOPT_E_SOLVER_STALL (max_iters pivots without optimality). */
int simopt_lmo_general(void* stream, const double* A, const double* C, int64_t m, int64_t n,
                       const double* g, int64_t max_iters, double* s_out, int* status);
/* CG step halves on device scalars (Newton-CG, BASELINE configs[2]):
 * step1: alpha = *rr / *dhd; p += alpha*d; r -= alpha*hd.  step2: d = r + (*rr_new / *rr)*d.
 * Both are no-ops when *rr == 0 (the CG loop's early exit). */
int simopt_cg_step1(void* stream, double* p, double* r, const double* d, const double* hd,
                    const double* rr, const double* dhd, int64_t n);
int simopt_cg_step2(void* stream, double* d, const double* r, const double* rr_new, const double* rr,
                    int64_t n);
/* Explicit Hessian h = (1/n) X^T diag(dw) X (d x d, symmetric, written fully) on the FP64
 * tensor pipe; X is n x d row-major.  Oracle: tests/test_tasks.py:292-304, rtol 1e-10. */
int simopt_logistic_xtdx(void* stream, const double* x, const double* dw, int64_t n, int64_t d,
                         double* h);
/* Same swap sequence on host memory for large b (u = the b uniforms). */
int simopt_fisher_yates_host(int64_t n, int64_t b, const double* u, int64_t* out);

/* One mean-variance FW step after its gradient g, in one launch: lmo_simplex_slack (NaN ->
 * *status |= INVALID_GRADIENT), w_out = (gamma * ((-1 * w_in) + s)) + w_in with *gamma
 * read on the device, *wmin_out = min(w_out), and the fixed-tree *wsum_out = sum(w_out),
 * *lin_out = dot(w_out, mean) (frank_wolfe.py:106-117, lmo.py:56-65, backend.py:80-111);
 * bitwise equal to the separate lmo / axpy / axpy_ptr / min / dot / vec_sum calls.
 * exact == 0 (fused mode): the two sums are block-parallel in a fixed order instead
 * (deterministic, not the reference tree; the update and min stay bitwise). */
int simopt_mv_fw_tail(void* stream, const double* g, const double* w_in, const double* gamma,
                      const double* mean, int64_t d, int64_t chunk, double* w_out, int* status,
                      double* wmin_out, double* wsum_out, double* lin_out, int exact);

/* One mean-variance FW epoch in fused mode as ONE cooperative launch (frank_wolfe.py:106-117
 * for MeanVarProblem, tasks.py:67-85): ring row 0 holds the epoch's first iterate; for
 * m < M: g = inv * Xc^T Xc w_m - mean, lmo_simplex_slack, ring[m+1] = w_{m+1}, status[m]
 * (NaN -> INVALID_GRADIENT), wmin/wsum/lin of w_{m+1}, quad[m] = |Xc w_{m+1}|^2, stamps[m]
 * (%globaltimer).  Sums in fixed block-parallel orders, like simopt_fused_rows + the fused
 * simopt_mv_fw_tail.  X row-major rows x cols, cols <= 2048; SIMOPT_E_CONFIG otherwise. */
int simopt_mv_fw_epoch(void* stream, const double* X, int64_t rows, int64_t cols,
                       const double* mean, double inv, double* ring, int64_t M,
                       const double* gamma, int* status, double* wmin, double* wsum, double* lin,
                       double* quad, int64_t* stamps);

/* ------------------------------------------------------------ projections (projected SGD) */
/* Euclidean projection of y onto {x >= 0, c . x <= budget} (c == NULL: all ones, i.e.
 * the simplex-with-slack of lmo.py:20-24 for budget 1).  One CTA: bisection on the
 * multiplier, exact recompute on the active set.  A NaN in y sets *status = 1
 * (InvalidGradient) when status != NULL. */
int simopt_project_budget(void* stream, const double* y, const double* c, double budget, int64_t d,
                          double* out, int* status);
/* Clamp onto the box [lo, hi]^d. */
int simopt_project_box(void* stream, const double* y, double lo, double hi, int64_t d, double* out);

/* ------------------------------------------------------------ multi-PRNG streams */
/* Philox4x32-10 (Random123): out[4b..4b+3] = Philox4x32_10(ctr + b, {key0, key1}) for
 * b < nblocks, ctr a 128-bit counter of four little-endian u32 words (host array);
 * out 16-byte aligned. */
int simopt_philox4x32(void* stream, uint32_t key0, uint32_t key1, const uint32_t* ctr,
                      int64_t nblocks, uint32_t* out);
/* Per-stream SFC64 / xoshiro256++: state = device u64[n_streams][4] (SFC64: a, b, c,
 * counter as numpy.random.SFC64; xoshiro: s[0..3]), advanced in place by n outputs;
 * out is stream-major [n_streams][n]: u64 words (out_kind 0) or doubles
 * (w >> 11) * 2^-53 (out_kind 1). */
int simopt_sfc64(void* stream, uint64_t* state, int64_t n_streams, int64_t n, int out_kind,
                 void* out);
int simopt_xoshiro256pp(void* stream, uint64_t* state, int64_t n_streams, int64_t n, int out_kind,
                        void* out);
/* Host: n_streams xoshiro256++ states, states[k] = jump^k(seed_state) (2^128 apart). */
int simopt_xoshiro256pp_streams(const uint64_t* seed_state, int64_t n_streams, uint64_t* states);

/* Deterministic sharded reductions: matvec_t chunk partials before the
 * fold, out[c*cols + j] (c < ceil(rows/chunk)); and the fold of nch gathered partial
 * rows, out[j] = fold_pairwise(p[0*count+j], ..., p[(nch-1)*count+j]) (p clobbered).
 * A dot's partials are matvec_t_partials of the n x 1 matrix x against y. */
int simopt_matvec_t_partials(void* stream, const double* a, int64_t rows, int64_t cols,
                             const double* center, const double* x, int64_t chunk, double* out);
int simopt_fold_partials(void* stream, double* p, int64_t nch, int64_t count, double* out);

/* Cross-rank sum fused into the finish of a fused pass over NVLink peer memory (sample
 * sharding).  peers[q] = device pointer to rank q's receive buffer (CUDA IPC mapping of a
 * simopt_peer_alloc of simopt_peer_reduce_bytes(world, cols) bytes); every rank pushes its
 * per-column partial sums (and the side scalar) into slot `rank` of every peer buffer,
 * releases per-block flags, acquires all ranks' flags and sums the slots in rank order --
 * so every rank computes the same bits.  seq must increase by one per pass (double-buffered
 * by parity); *status = 1 if a peer never arrives (10 s) -- sticky: while *status != 0
 * later passes do not wait (they return local sums), so a broken peer fails fast. */
typedef struct SimoptPeerReduce {
  void* const* peers;
  int64_t world, rank;
  uint64_t seq;
  int* status;
} SimoptPeerReduce;
int64_t simopt_peer_reduce_bytes(int64_t world, int64_t cols);

/* ------------------------------------------------------------ bit-packed binary features */
/* Layout: row-major, W = ceil(d/64) u64 words per row, feature j = bit (j&63) of word j>>6.
 * bernoulli_bits: rows [row_lo, row_hi) of synth_classification's features
 * (sampling.py:246-255, MSB of each Philox word) straight into bits.
 * matvec_bits: the fixed-tree row dots (_kernels.py:71-121) over bits -- bit-identical to
 * simopt_matvec on the 0.0/1.0 matrix.  unpack_bits: 0.0/1.0 fp64 rows. */
int simopt_bernoulli_bits(void* stream, uint64_t seed, uint64_t stream_id, uint64_t ctr_lo,
                          uint64_t ctr_hi, int64_t row_lo, int64_t row_hi, int64_t d, uint64_t* out);
int simopt_matvec_bits(void* stream, const uint64_t* bits, int64_t rows, int64_t d, const double* v,
                       int64_t chunk, double* out);
/* matvec_bits over the gathered rows idx[0..rows) (nullable: rows 0..rows) of a bit matrix
 * with total_rows rows -- simopt_matvec's rows_idx form (tasks.py:205-213 batches).
 * matvec_t_bits: the fixed-tree column sums (_kernels.py:124-156) x^T X over bits, same
 * gather; bit-identical to simopt_matvec_t on the 0.0/1.0 matrix. */
int simopt_matvec_bits_idx(void* stream, const uint64_t* bits, int64_t total_rows, int64_t d,
                           const int64_t* idx, int64_t rows, const double* v, int64_t chunk,
                           double* out);
int simopt_matvec_t_bits(void* stream, const uint64_t* bits, int64_t total_rows, int64_t d,
                         const int64_t* idx, int64_t rows, const double* x, int64_t chunk,
                         double* out);
int simopt_unpack_bits(void* stream, const uint64_t* bits, int64_t rows, int64_t d, double* out);
/* simopt_fused_rows (LR_GRAD / LR_HVP modes) on bit-packed features, d <= 16384. */
int simopt_fused_rows_bits(void* stream, int mode, const uint64_t* bits, int64_t rows, int64_t cols,
                           const double* v, const double* rowaux, double col_scale, int accumulate,
                           int raw, double* t_out, double* dw_out, double* col_out,
                           double* scalar_out, const SimoptPeerReduce* peer);
/* Binary X on the integer tensor cores (csrc/hessian_i8.cu): bits_to_u8t builds X^T as u8 in
 * sample blocks [np/ch][d][ch + 32] (ch, np from u8t_geometry; padded rows are zero); xtdx_i8 computes
 * H = (1/n) X^T diag(dw) X exactly for dw rounded to 2^-e (5 x 8-bit limbs, u8 IMMA with
 * int32 accumulation; e from max(dw), read back once per call: not capturable), plus two
 * exact-residual refinement passes when 2^-40 max(dw)/mean(dw) > 1e-11; limbs = u8 scratch [5][np]. */
int simopt_u8t_geometry(int64_t n, int64_t* ch, int64_t* np);
int simopt_bits_to_u8t(void* stream, const uint64_t* bits, int64_t rows, int64_t d, int64_t np,
                       uint8_t* out);
int simopt_logistic_xtdx_i8(void* stream, const uint8_t* xt, int64_t np, int64_t n, int64_t d,
                            const double* dw, uint8_t* limbs, double* h);
/* The tcgen05 limb Hessian with its operands loaded by TMA (3-D tensor maps over the
 * sample-blocked X^T and the limb rows); same operands and result as xtdx_tc. */
int simopt_logistic_xtdx_tma(void* stream, const uint8_t* xt, int64_t np, int64_t n, int64_t d,
                             const double* dw, uint8_t* limbs, double* h);
/* The same on CTA pairs (cta_group::2, 256 x 96 tiles; slower on this B200, see DESIGN). */
int simopt_logistic_xtdx_pair(void* stream, const uint8_t* xt, int64_t np, int64_t n, int64_t d,
                              const double* dw, uint8_t* limbs, double* h);
/* Same result on the 5th-generation tensor cores: tcgen05.mma.kind::i8 with the five limb
 * accumulators resident in TMEM (128 x 96 tiles, one CTA per SM). */
int simopt_logistic_xtdx_tc(void* stream, const uint8_t* xt, int64_t np, int64_t n, int64_t d,
                            const double* dw, uint8_t* limbs, double* h);
/* Limb passes the calling thread's last xtdx_{i8,tc,tma,pair} call ran: 1, or 3 when the
 * precision guard added the two residual refinement passes (2^-40 max(dw)/mean(dw) > 1e-11). */
int simopt_xtdx_last_passes(void);
/* simopt_logistic_xtdx on bit-packed features (DMMA fragments expanded in registers). */
int simopt_logistic_xtdx_bits(void* stream, const uint64_t* xbits, const double* dw, int64_t n,
                              int64_t d, double* h);

/* Fused single pass over X (N x d row-major): t_r = x_r . v, wt_r = f(t_r), and
 * col_out[j] = (sum_r x_rj wt_r) * col_scale [- center[j] for MV], in ONE read of X.
 * Replaces each matvec + matvec_t pair of the reference (fast summation order, not
 * the fixed tree; ~1e-15 relative):
 *   SIMOPT_FUSED_MV       tasks.py:67-85  x = X - center; wt = t; *scalar_out = sum t^2
 *   SIMOPT_FUSED_LR_GRAD  tasks.py:216-236 wt = sigmoid(t) - rowaux[r] (labels);
 *                         dw_out[r] = c(1-c); *scalar_out = sum of loss terms
 *   SIMOPT_FUSED_LR_HVP   tasks.py:239-253 wt = rowaux[r] (= c(1-c)) * t
 * t_out / dw_out / col_out / scalar_out may be NULL; accumulate = 0 skips the column
 * sums (row pass only); raw = 1 writes the plain column sums (no scale, no centering:
 * the per-shard partial that a sample-sharded caller allreduces).  peer != NULL: the
 * column sums and the scalar are summed over ranks inside the finish kernel (see
 * SimoptPeerReduce) before the epilogue.  d <= 32768. */
#define SIMOPT_FUSED_MV 0
#define SIMOPT_FUSED_LR_GRAD 1
#define SIMOPT_FUSED_LR_HVP 2
int simopt_fused_rows(void* stream, int mode, const double* x, int64_t rows, int64_t cols,
                      const double* v, const double* center, const double* rowaux,
                      double col_scale, int accumulate, int raw, double* t_out, double* dw_out,
                      double* col_out, double* scalar_out, const SimoptPeerReduce* peer);
/* Launch geometry simopt_fused_rows uses for `cols` columns on the current device
 * (diagnostic, no launch): CTAs per cluster (column bands), resident clusters (from
 * cudaOccupancyMaxActiveClusters: how many C-CTA clusters the chip's GPCs hold at once)
 * and the grid.  vec: 16-byte aligned even rows. */
int simopt_fused_geometry(int mode, int64_t cols, int vec, int* cluster, int* clusters, int* grid);

/* ---- NCCL communicator (csrc/comm.cu; SURVEY 8(b) "NCCL communicator handle init/teardown").
 * Replaces the reference's in-process data-parallel split (sobench/backend.py:178-204) for
 * one process per GPU.  libnccl.so.2 is resolved at run time (the copy torch loaded, else the
 * loader path); without it every call returns SIMOPT_E_CUDA.  Rank 0 creates the 128-byte
 * unique id, the host broadcasts it (any channel), every rank calls comm_init.  Collectives
 * are enqueued on `stream` and are asynchronous like every other entry point. */
int simopt_comm_version(int* version);
int simopt_comm_unique_id(uint8_t* id128);
int simopt_comm_init(const uint8_t* id128, int world, int rank, void** comm);
int simopt_comm_destroy(void* comm);
int simopt_comm_allreduce_f64(void* comm, void* stream, const double* send, double* recv, int64_t n);
int simopt_comm_allreduce_min_f64(void* comm, void* stream, const double* send, double* recv,
                                  int64_t n);
int simopt_comm_allgather(void* comm, void* stream, const void* send, void* recv, int64_t bytes);
int simopt_comm_broadcast(void* comm, void* stream, const void* send, void* recv, int64_t bytes,
                          int root);

#ifdef __cplusplus
}
#endif
#endif /* SIMOPT_B200_H */
