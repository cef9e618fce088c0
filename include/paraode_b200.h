/*
 * paraode_b200 — C ABI of the B200-native ParaIEKS hot path.
 *
 * This is the drop-in boundary: a flat C interface (plain pointers and
 * sizes, no C++/torch types) whose entry points are what a binding of the
 * reference's C++ solver API (proj/include/paraode/) for this path needs.
 * Three layers sit on top of it: the source-compatible
 * C++ drop-in with the reference's own names and signatures
 * (include/paraode/paraode.hpp), a templated C++ shim over any dense matrix
 * type (include/paraode/paraode_b200.hpp), and the Python package
 * (paraode_b200/).
 *
 * Conventions
 *   - All arithmetic is IEEE fp64.  All matrices are ROW-MAJOR and
 *     contiguous; arrays of N matrices are N consecutive D x D blocks.
 *     (The reference's Eigen matrices are column-major; the layout is stated
 *     here, not inherited.)
 *   - State dimension D = dim * (nu + 1), states laid out dimension-major
 *     [y1, y1', .., y1^(nu), y2, ..] (proj/include/paraode/statespace.hpp:56-58).
 *   - Every pointer argument is HOST memory unless the call's `location`
 *     field says PODE_DEVICE (then all its pointers are device pointers on
 *     the context's GPU).
 *   - Every call returns a pode_code; on failure `status` (if non-NULL)
 *     carries the code, the first failing index and a message.  The codes
 *     map 1:1 to the reference's exception types
 *     (proj/include/paraode/errors.hpp:10-60).
 *   - There is no CPU fallback: without a usable B200 every compute entry
 *     point fails with PODE_ERR_CUDA.
 */
#ifndef PARAODE_B200_H_
#define PARAODE_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PODE_OK = 0,
  PODE_ERR_INVALID_INPUT = 1,   /* InvalidInputError */
  PODE_ERR_DIMENSION = 2,       /* DimensionError */
  PODE_ERR_SINGULAR_FACTOR = 3, /* SingularFactorError */
  PODE_ERR_LINEARIZATION = 4,   /* LinearizationError (time, index) */
  PODE_ERR_SCAN = 5,            /* ScanError ("elements [lo, hi]") */
  PODE_ERR_CUDA = 6,            /* no device / CUDA failure (no CPU fallback) */
  PODE_ERR_UNSUPPORTED = 7      /* state dimension outside the compiled range */
} pode_code;

enum { PODE_HOST = 0, PODE_DEVICE = 1 };

typedef struct {
  int32_t code;
  int32_t iteration; /* IEKS iteration at failure (1-based), 0 if n/a */
  int64_t index;     /* first failing element / step index, -1 if n/a */
  int64_t lo, hi;    /* element range for PODE_ERR_SCAN */
  double time;       /* grid time for PODE_ERR_LINEARIZATION */
  char msg[256];
} pode_status;

typedef struct pode_context pode_context;

/* One context = one GPU + one CUDA stream + cached device workspace.
 * Not reentrant; distinct contexts may be used concurrently. */
int pode_context_create(int32_t device, pode_context** out, pode_status* status);
void pode_context_destroy(pode_context* ctx);
/* Largest state dimension D compiled into this library: 112 for pode_ieks
 * (the large-state engine serves d = 28, nu = 1..3: D = 56, 84, 112); the
 * element operators, pode_rts, pode_eks and the sharded solve take D <= 16. */
int32_t pode_max_state_dim(void);
/* Number of kernels this library has launched on ctx (instrumentation). */
int64_t pode_kernel_launches(const pode_context* ctx);
/* The CUDA stream (cudaStream_t) the context launches on. */
void* pode_context_stream(pode_context* ctx);
/* Per-context engine options (replace process-wide environment knobs, so
 * concurrent contexts do not see each other's settings):
 *   PODE_OPT_CHUNK_LEN  time steps per chunk of the fused IEKS engines
 *                       (0 = automatic: ~256 chunks per SM; clamped to [2, N];
 *                       N = one chunk = the sequential Kalman recursion, seq_ieks)
 *   PODE_OPT_ENGINE     0 = automatic, 1 = fused engines only (PODE_ERR_UNSUPPORTED
 *                       when none serves the state), 2 = the element engine
 * Returns PODE_OK or PODE_ERR_INVALID_INPUT. */
typedef enum { PODE_OPT_CHUNK_LEN = 1, PODE_OPT_ENGINE = 2 } pode_option;
int pode_context_set_option(pode_context* ctx, int32_t option, int64_t value);
/* Per-kernel CUDA-event timing on the context stream (instrumentation):
 * pode_profile(ctx, 1) clears and starts recording, pode_profile(ctx, 0)
 * stops; pode_profile_read writes "kernel launches total_ms" lines into buf
 * and returns the full text length (-1 on error). */
int pode_profile(pode_context* ctx, int32_t enable);
int64_t pode_profile_read(pode_context* ctx, char* buf, int64_t size);

/* ------------------------------------------------------------- elements */
/* FilteringElement arrays (proj/include/paraode/parallel.hpp:20-26):
 * a, c_sqrt, j_sqrt: count*D*D; b, eta: count*D. */
typedef struct {
  double* a;
  double* b;
  double* c_sqrt;
  double* eta;
  double* j_sqrt;
} pode_filtering_elements;

/* SmoothingElement arrays (parallel.hpp:32-36): e, l_sqrt: count*D*D; g: count*D. */
typedef struct {
  double* e;
  double* g;
  double* l_sqrt;
} pode_smoothing_elements;

typedef struct {
  int64_t combine_invocations; /* ScanStats (sequential.hpp:42-50) */
  int64_t sequential_depth;
} pode_scan_stats;

/* Linear-Gaussian chain: init, N transitions (phi, q_sqrt) and N affine
 * observations z = H y - offset with noise R = r_sqrt r_sqrt^T
 * (statespace.hpp:36-48).  Observation n has obs_rows[n] <= obs_rows_max
 * real rows stored in the first rows of its obs_rows_max-row slot
 * (0 rows = vacuous, parallel.cpp:26-36); r_sqrt is the leading
 * obs_rows[n] x obs_rows[n] block of its M x M slot. */
typedef struct {
  int32_t state_dim;    /* D */
  int32_t obs_rows_max; /* M <= D */
  int64_t steps;        /* N >= 1 */
  const double* init_mean;     /* D */
  const double* init_cov_sqrt; /* D*D */
  const double* phi;           /* N*D*D, or D*D when phi_shared */
  const double* q_sqrt;        /* N*D*D, or D*D when q_shared */
  int32_t phi_shared;
  int32_t q_shared;
  const int32_t* obs_rows; /* N */
  const double* h;         /* N*M*D */
  const double* offset;    /* N*M */
  const double* r_sqrt;    /* N*M*M */
  int32_t location;        /* PODE_HOST / PODE_DEVICE for every pointer above */
} pode_chain;

/* make_filtering_element for every step (parallel.cpp:5-65); element 0
 * absorbs init when absorb_init != 0. `out` has chain->steps elements. */
int pode_make_filtering_elements(pode_context* ctx, const pode_chain* chain, int32_t absorb_init,
                                 pode_filtering_elements out, pode_status* status);

/* out[i] = lhs[i] ⊗_f rhs[i] (combine_filtering, parallel.cpp:67-100). */
int pode_combine_filtering(pode_context* ctx, int64_t count, int32_t state_dim,
                           pode_filtering_elements lhs, pode_filtering_elements rhs,
                           pode_filtering_elements out, int32_t location, pode_status* status);

/* Smoothing elements for nodes 0..N from the filtered marginals
 * (f_mean (N+1)*D, f_cov_sqrt (N+1)*D*D); node N is terminal
 * (parallel.cpp:112-144). `out` has chain->steps + 1 elements. */
int pode_make_smoothing_elements(pode_context* ctx, const pode_chain* chain, const double* f_mean,
                                 const double* f_cov_sqrt, pode_smoothing_elements out,
                                 pode_status* status);

/* out[i] = lhs[i] ⊗_s rhs[i] (combine_smoothing, parallel.cpp:146-156). */
int pode_combine_smoothing(pode_context* ctx, int64_t count, int32_t state_dim,
                           pode_smoothing_elements lhs, pode_smoothing_elements rhs,
                           pode_smoothing_elements out, int32_t location, pode_status* status);

/* Inclusive associative scans (associative_scan, parallel.hpp:136-149):
 * forward = prefixes e_0 ⊗ .. ⊗ e_i; reverse = suffixes e_i ⊗ .. ⊗ e_{n-1}
 * (operands kept in time order).  in and out may alias. */
int pode_scan_filtering(pode_context* ctx, int64_t count, int32_t state_dim,
                        pode_filtering_elements in, pode_filtering_elements out, int32_t reverse,
                        int32_t location, pode_scan_stats* stats, pode_status* status);
int pode_scan_smoothing(pode_context* ctx, int64_t count, int32_t state_dim,
                        pode_smoothing_elements in, pode_smoothing_elements out, int32_t reverse,
                        int32_t location, pode_scan_stats* stats, pode_status* status);

/* ------------------------------------------------------------- smoother */
/* Filtering and smoothing marginals at nodes 0..N (RtsResult,
 * sequential.hpp:52-56): means (N+1)*D, lower-triangular factors (N+1)*D*D.
 * Any output pointer may be NULL.  Pointers follow chain->location. */
typedef struct {
  double* filtered_mean;
  double* filtered_cov_sqrt;
  double* smoothed_mean;
  double* smoothed_cov_sqrt;
} pode_rts_out;

/* Replaces para_rts (proj/include/paraode/parallel.hpp:155-156). */
int pode_rts(pode_context* ctx, const pode_chain* chain, pode_rts_out out, pode_scan_stats* stats,
             pode_status* status);

/* ----------------------------------------------------------------- ieks */
/* Device vector-field registry (replaces InitialValueProblem's host
 * std::function callbacks, statespace.hpp:24-31). */
typedef enum {
  PODE_LOGISTIC = 1,   /* y' = y (1 - y)                       (problems.cpp:116-135) */
  PODE_RIGID_BODY = 2, /* Euler rigid body                     (problems.cpp:137-157) */
  PODE_VAN_DER_POL = 3,/* params[0] = mu                       (problems.cpp:159-179) */
  PODE_FITZHUGH_NAGUMO = 4, /* params = (a, b, c)              (new) */
  PODE_PLEIADES = 5,   /* 7-body, first order, d = 28          (new) */
  PODE_AFFINE = 6,     /* y' = L y + c; params = L (d*d row-major), c (d) */
  PODE_POLE = 7        /* y' = 1 / (t - a), d = 1, params = {a}: the reference's non-finite
                          field test (test_statespace.cpp:123-139) with the pole at time a */
} pode_problem_kind;

typedef struct {
  int32_t kind;
  int32_t dim;       /* d */
  double t_end;
  const double* y0;  /* d (host) */
  const double* params;
  int32_t n_params;  /* 0 = the shipped defaults for kind */
} pode_problem;

typedef struct {
  int32_t nu;    /* IWP order q >= 1 (IwpPrior, prior.hpp:12-18) */
  int32_t dim;   /* d */
  double sigma;  /* diffusion >= 0 */
} pode_prior;

typedef struct {
  int32_t max_iterations; /* IeksConfig (ieks.hpp:32-38) */
  double traj_rtol;
  double obj_atol;
  double obj_rtol;
  int32_t linearization;  /* 0 = EK1, 1 = EK0 */
} pode_ieks_config;

/* SolverReport (ieks.hpp:77-87).  Output arrays (N+1 nodes, original
 * coordinates) may be NULL; they follow `location`. */
typedef struct {
  double* means;           /* (N+1)*D          marginals[n].mean */
  double* cov_sqrt;        /* (N+1)*D*D        marginals[n].cov_sqrt (calibrated) */
  double* solution_means;  /* (N+1)*d */
  double* solution_covs;   /* (N+1)*d*d */
  double* objective_trace; /* trace_capacity (host) */
  int32_t trace_capacity;
  int32_t location;        /* PODE_HOST / PODE_DEVICE for the four arrays above */
  int32_t iterations;
  int32_t converged;
  double sigma_hat;
  pode_scan_stats scan_stats;
} pode_ieks_report;

/* Replaces para_ieks (proj/include/paraode/ieks.hpp:95-96): the full
 * Gauss-Newton loop on the device.  `grid` (n_nodes = N+1 host doubles)
 * must start at 0 and increase strictly. */
int pode_ieks(pode_context* ctx, const pode_problem* problem, const pode_prior* prior,
              const double* grid, int64_t n_nodes, const pode_ieks_config* config,
              pode_ieks_report* report, pode_status* status);

/* Batched para_ieks (the reference solves one
 * problem per call, ieks.cpp:114-217): `count` independent IVPs of one field
 * kind and dimension (parameters and initial values free, e.g. a parameter
 * sweep) sharing one prior, grid and config, fused into one pass sequence
 * per Gauss-Newton iteration on the lane engine (d <= 3, D <= 9; else
 * PODE_ERR_UNSUPPORTED).  Each IVP stops on its own by the reference's rule
 * and reports[i] receives what pode_ieks would report for problems[i]. */
int pode_ieks_batch(pode_context* ctx, const pode_problem* problems, int32_t count, const pode_prior* prior,
                    const double* grid, int64_t n_nodes, const pode_ieks_config* config,
                    pode_ieks_report* reports, pode_status* status);

/* Replaces eks_solve (proj/include/paraode/ieks.hpp:103-105, ieks.cpp:224-291):
 * one forward pass linearised at each step's own predicted mean (sequential
 * in time: one warp on the device), the smoother of those filtered
 * marginals (reverse scan), calibration and outputs.  The report has
 * iterations = 1, converged = 1 and a one-entry objective trace.
 * linearization: 0 = EK1, 1 = EK0. */
int pode_eks(pode_context* ctx, const pode_problem* problem, const pode_prior* prior,
             const double* grid, int64_t n_nodes, int32_t linearization,
             pode_ieks_report* report, pode_status* status);

/* Accuracy reference of the benchmark harness (problems.cpp:11-27): `steps`
 * classical RK4 steps of the registered field on [0, t_end]; table holds
 * (steps+1) * dim host doubles.  PODE_ERR_INVALID_INPUT if it diverges. */
int pode_rk4_table(pode_context* ctx, const pode_problem* problem, int64_t steps, double* table,
                   pode_status* status);

/* ---- time-axis sharding (one process per GPU) ----------
 * The reference has no multi-device path; this is the SURVEY.md §8(e)
 * partition of the same solve.  Shard r of R owns steps [s_r, e_r),
 * s_r = floor(N r / R), and reports nodes s_r .. e_r - 1 (the last shard
 * also node N).  Per iteration the shards exchange, through the caller's
 * all-gather: the forward aggregate of their steps (3D^2+2D doubles), the
 * backward mean aggregate (D^2+D) and the three stopping scalars; the
 * finalize exchanges the innovation sum and the smoothing aggregate
 * (2D^2+D).  Every fold of exchanged values runs in rank order on the
 * device, so all shards take identical stopping decisions. */

/* All-gather of `count` doubles from every rank into recv[rank * count + i]
 * (host memory).  Returns 0 on success. */
typedef int (*pode_allgather_fn)(void* user, const double* send, int64_t count, double* recv);

typedef struct {
  int32_t rank;
  int32_t ranks;
  pode_allgather_fn allgather;
  void* user;
} pode_shard_comm;

/* Device-side exchange (no host staging): bind an NCCL communicator to the
 * context; pode_ieks_sharded then all-gathers the chunk aggregates and
 * stopping scalars with ncclAllGather on device buffers on the context
 * stream, and comm->allgather may be NULL.  NCCL is loaded at run time
 * (dlopen of `nccl_path`, e.g. the libnccl.so.2 torch bundles; NULL: the
 * loader's search path).  pode_nccl_unique_id makes the 128-byte
 * ncclUniqueId on one rank; the caller broadcasts it to every rank (any
 * transport) before each rank calls pode_context_nccl_init.  One process
 * per GPU (NCCL rejects two ranks on one device). */
int pode_nccl_unique_id(const char* nccl_path, uint8_t id[128], pode_status* status);
int pode_context_nccl_init(pode_context* ctx, const char* nccl_path, const uint8_t id[128], int32_t rank,
                           int32_t ranks, pode_status* status);

/* Shard node range of `rank` (first node, number of reported nodes). */
void pode_shard_range(int64_t n_nodes, int32_t rank, int32_t ranks, int64_t* first_node, int64_t* count);

/* para_ieks over a time-axis shard: `grid` is the GLOBAL grid (n_nodes);
 * the report arrays hold this shard's nodes (pode_shard_range), the scalars
 * (iterations, converged, sigma_hat, objective trace) are global.  Requires
 * an ODE information operator the fused engine serves (d <= 3, D <= 9). */
int pode_ieks_sharded(pode_context* ctx, const pode_problem* problem, const pode_prior* prior,
                      const double* grid, int64_t n_nodes, const pode_ieks_config* config,
                      const pode_shard_comm* comm, pode_ieks_report* report, pode_status* status);

#ifdef __cplusplus
}
#endif

#endif /* PARAODE_B200_H_ */
