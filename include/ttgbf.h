/* ttgbf.h -- C-ABI of the B200-native TT grid-based filter (TT-GBF) hot path.
 *
 * Drop-in boundary for the reference's Python filter API
 * (ttpmf.filters / ttpmf.tensor_train / ttpmf.tt_algorithms).  Every entry
 * point takes plain pointers and sizes (device pointers unless stated) plus
 * a cudaStream_t passed as void*, launches hand-written sm_100a kernels and
 * returns a status code (0 = ok, see TTGBF_E_*).  No torch types appear here.
 *
 * Reference interface each entry point replaces (file:line in the reference
 * package pkg/src/ttpmf):
 *   ttgbf_filter_prior        filters.initial_pmd_tt            filters.py:497-513
 *   ttgbf_filter_measure      filters.measurement_update (TT)   filters.py:521-563
 *                             + filters.moments_from_pmd (TT)   filters.py:287-333
 *   ttgbf_filter_time_update  filters.tt_fft_pmf_step, lines after the moments:
 *                             grid_redesign (interp+finalize)   filters.py:799-824
 *                             kernel cross + tt_fft_convolve    filters.py:959-964
 *                             realign cross + finalize          filters.py:965-985
 *   ttgbf_tt_round            tensor_train.tt_round             tensor_train.py:327-360
 *   ttgbf_tt_hadamard         tensor_train.tt_hadamard          tensor_train.py:252-266
 *   ttgbf_tt_fft_convolve     tt_algorithms.tt_fft_convolve     tt_algorithms.py:642-666
 *   ttgbf_tt_interpolate      tt_algorithms.tt_interpolate      tt_algorithms.py:701-718
 *   ttgbf_tt_eval_many        tensor_train.tt_eval_many         tensor_train.py:129-158
 *   ttgbf_tt_eval_at_points   tt_algorithms.tt_eval_at_points   tt_algorithms.py:721-745
 *   ttgbf_tt_sum_moments      tensor_train.tt_sum / tt_dot with rank-one coordinate
 *                             TTs as used by moments_from_pmd   tensor_train.py:269-288
 *   ttgbf_greedy_cross        tt_algorithms.greedy_cross        tt_algorithms.py:463-596
 *                             (on the prior / likelihood / kernel black boxes)
 *   ttgbf_negative_mass       filters._negative_mass_tt         filters.py:427-436
 *   ttgbf_eval_blackbox       the cross black boxes: prior pdf, likelihood,
 *                             FFT kernel, realign evaluator     filters.py:504,697-729,969-979;
 *                                                               models.py:150-153
 *   ttgbf_rng_draws           numpy Generator.integers / choice as the cross
 *                             draws them                        tt_algorithms.py:341-433
 *   ttgbf_filter_time_update_std  filters.tt_pmf_step time update (Algorithm 2) filters.py:855-885
 *   ttgbf_dense_*             filters.dense_fft_pmf_step pieces  filters.py:888-934
 *                             (the dense FFT PMF on the GPU)
 */
#ifndef TTGBF_H
#define TTGBF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TTGBF_MAXD 16
#define TTGBF_MAXB 16

/* status codes */
#define TTGBF_OK 0
#define TTGBF_E_ARG 1          /* ValueError: shapes / configuration            */
#define TTGBF_E_NONFINITE 2    /* ValueError: evaluator returned a non-finite   */
#define TTGBF_E_DEGENERATE 3   /* DegenerateDensityError (filters.py:120)       */
#define TTGBF_E_WORKSPACE 4    /* per-filter workspace too small                */
#define TTGBF_E_CACHE 5        /* evaluator cache capacity exhausted            */
#define TTGBF_E_CUDA 6         /* CUDA launch / runtime error                   */
#define TTGBF_E_LINALG 7       /* numpy.linalg.LinAlgError (singular F)         */
#define TTGBF_E_DENSE_GUARD 8  /* DenseGuardError                                */
#define TTGBF_E_STATE_CAP 9    /* output TT larger than the per-filter state slab */

/* Equidistant axis: coordinate i = base + step * (i - off), evaluated with a
 * separate multiply and add (no FMA) so it equals numpy's construction in
 * grids.design_grid (off = (n-1)//2) and Grid.from_bounds (off = 0). */
typedef struct {
  double base;
  double step;
  int32_t off;
  int32_t n;
} ttgbf_axis;

/* Packed tensor train: core k (r[k] x n[k] x r[k+1], C order) starts at
 * data + off[k] (doubles). */
typedef struct {
  int32_t d;
  int32_t n[TTGBF_MAXD];
  int32_t r[TTGBF_MAXD + 1];
  int32_t pad;
  int64_t off[TTGBF_MAXD];
} ttgbf_tt;

/* CrossConfig (tt_algorithms.py:93-115).  rng_state = numpy PCG64 state of
 * default_rng(rng_seed): {state_lo, state_hi, inc_lo, inc_hi, has_uint32,
 * uinteger}.  cache_cap bounds the evaluator cache (entries). */
typedef struct {
  double tol;
  int32_t max_rank;
  int32_t max_sweeps;
  int32_t validation_count;
  int32_t pad;
  uint64_t rng_state[6];
  int64_t cache_cap;
} ttgbf_cross_cfg;

/* GridConfig rounding/normalisation policy (filters.py:129-161); a
 * round_max_rank <= 0 means None. */
typedef struct {
  double round_tol;
  int32_t round_max_rank;
  int32_t normalize_before_round;
  int64_t densify_guard;
} ttgbf_grid_cfg;

typedef struct {
  double achieved;
  int64_t calls;
  int32_t sweeps;
  int32_t converged;
} ttgbf_cross_info;

#define TTGBF_NRANKLOG 10
#define TTGBF_NMOM (1 + TTGBF_MAXD + TTGBF_MAXD * (TTGBF_MAXD + 1) / 2)

/* per-filter diagnostics (StepDiagnostics, filters.py:164-188) */
typedef struct {
  int32_t status;
  int32_t outlier;
  double mass_before_norm;
  double clipped_mass;
  ttgbf_cross_info cross[3];     /* prior|likelihood, kernel, realign */
  double raw_moments[TTGBF_NMOM];/* sum, first (d), second (i<=j), un-normalised */
  int64_t ws_peak;               /* bytes of workspace used */
  /* shape log: ranks of 0 input TT, 1 likelihood cross TT, 2 filtering TT,
   * 3 shifted TT, 4 kernel cross TT, 5 rounded convolution, 6 realign cross
   * TT, 7 output TT (used for the algorithmic FLOP count), 8 likelihood TT
   * and 9 kernel TT after the exact-rank squeeze (what the products use) */
  int32_t ranks[TTGBF_NRANKLOG][TTGBF_MAXD + 1];
  /* SM clock cycles of the stage sections (CTA leader): 0 likelihood cross,
   * 1 Hadamard+finalize, 2 moments, 3 interp+finalize, 4 kernel cross,
   * 5 FFT conv+round, 6 realign cross, 7 final finalize */
  int64_t cycles[8];
  /* engine profile (SM cycles, CTA leader, overlapping categories):
   * 0 miss sort, 1 evaluator, 2 cache lookup/insert, 3 core lstsq, 4 hunt,
   * 5 accept, 6 cache check, 7 tt_round, 8 svd, 9 qr, 10 rng choice,
   * 11 snapshot, 12 chain eval, 13 inject, 14 fft conv (incl. round),
   * 15 negative mass, 16 qr panel, 17 qr trailing update, 18 round R-multiply,
   * 19 round apply_q, 20 fft spectra+product, 21 svd rrqr, 22 rrqr rank sum (count, not cycles), 23 svd_rrqr calls,
   * 24 max rrqr rank (count), 25 svd jacobi, 26 svd U from reflectors, 27 svd Bt QR + V,
   * 28 svd calls with rank > 64 (count), 29 their cycles, 30 exact-rank squeeze of cross outputs, 31 core-solve factorisation (within 3) */
  int64_t prof[32];
  int64_t big_used;       /* steps that borrowed an overflow workspace */
  int64_t big_peak;       /* peak bytes used in an overflow workspace */
  int64_t big_wait;       /* SM cycles spent waiting for a free overflow workspace */
} ttgbf_diag;

/* Model constants (StateSpaceModel, models.py:85-153).  Matrices row-major
 * with leading dimension TTGBF_MAXD (F, Finv, LUq, H) or TTGBF_MAXB (LUr).
 * LUq / LUr: LAPACK dgetrf factors of numpy's lower Cholesky factors of
 * Q / R (what numpy.linalg.solve(chol, .) factors inside
 * GaussianDensity.logpdf, models.py:60-63): row-major LU, 0-based sequential
 * row swaps piv*, reciprocal pivots inv* = 1 / U_ii; logn_* the
 * GaussianDensity log normalisers (models.py:47-49). */
typedef struct {
  int32_t d;
  int32_t b;
  int32_t hkind;      /* 0 linear, 1 range_bearing, 2 range_bearing_deg,
                         3 norm_bearing_deg, 4 abs_first, 5 range_az_el,
                         6 chain_quadratic */
  int32_t nang;
  int32_t ang[TTGBF_MAXB];
  double F[TTGBF_MAXD * TTGBF_MAXD];
  double Finv[TTGBF_MAXD * TTGBF_MAXD];
  double LUq[TTGBF_MAXD * TTGBF_MAXD];
  int32_t pivq[TTGBF_MAXD];
  double invq[TTGBF_MAXD];
  double logn_q;
  double LUr[TTGBF_MAXB * TTGBF_MAXB];
  int32_t pivr[TTGBF_MAXB];
  double invr[TTGBF_MAXB];
  double logn_r;
  double H[TTGBF_MAXB * TTGBF_MAXD];
  double Q[TTGBF_MAXD * TTGBF_MAXD];
} ttgbf_model;

/* Gaussian prior (initial_pmd_tt): mean, dgetrf factors of the covariance's
 * lower Cholesky factor (as in ttgbf_model), log normaliser */
typedef struct {
  double mean[TTGBF_MAXD];
  double LU[TTGBF_MAXD * TTGBF_MAXD];
  int32_t piv[TTGBF_MAXD];
  double inv[TTGBF_MAXD];
  double logn;
} ttgbf_gauss;

/* per-filter step inputs: current grid, pre-convolution (filtering) grid,
 * predictive grid (from the host-side redesign), measurement */
typedef struct {
  ttgbf_axis cur[TTGBF_MAXD];
  ttgbf_axis filt[TTGBF_MAXD];
  ttgbf_axis pred[TTGBF_MAXD];
  double z[TTGBF_MAXB];
  int32_t has_z;
  int32_t active;
} ttgbf_filter_io;

/* Persistent multi-step run (device geometry): per-filter loop of
 * tt_fft_pmf_step over `steps` steps, re-initialising from the prior on
 * DegenerateDensityError and after kf steps (end of the trajectory). */
typedef struct {
  int32_t n_per_axis;
  int32_t kf;             /* trajectory length (measurements per filter) */
  int32_t steps;          /* filter steps attempted per filter in this launch */
  int32_t pad;
  double sigma_mult;
  ttgbf_axis prior_grid[TTGBF_MAXD];
  /* overflow workspaces: a step whose FFT product (kernel rank x filter rank
   * per bond) does not fit in its slot borrows one of nbig buffers of
   * big_bytes for the convolution + rounding (spin-acquired, big_locks
   * zero-initialised), then copies the rounded TT back.  nbig = 0: none. */
  int32_t nbig;
  int32_t pad2;
  int64_t big_bytes;
  void* big_ws;
  int32_t* big_locks;
  /* second, larger overflow class (nbig2 buffers of big2_bytes): a product
   * that fits big_bytes tries the first class, then this one; a larger one
   * waits for this class only.  nbig2 = 0: none. */
  int32_t nbig2;
  int32_t pad3;
  int64_t big2_bytes;
  void* big2_ws;
  int32_t* big2_locks;
} ttgbf_run_cfg;

#define TTGBF_NCOV (TTGBF_MAXD * (TTGBF_MAXD + 1) / 2)

/* one record per filter per attempted step; cov = filtered covariance, upper
 * triangle packed row-major (i <= j), d*(d+1)/2 entries used */
typedef struct {
  int32_t status;         /* 0 = step completed, else TTGBF_E_*; -1 = prior init failed */
  int32_t k;              /* trajectory index of the measurement used */
  int32_t spd_fixed;
  int32_t outlier;
  double mean[TTGBF_MAXD];
  double cov[TTGBF_NCOV];
  double mass_before_norm;
  double clipped_mass;
  int64_t calls[3];
  int32_t ranks[TTGBF_NRANKLOG][TTGBF_MAXD + 1];
  int64_t cycles;         /* SM clock cycles the step took on its CTA (0 in host emulation) */
} ttgbf_step_rec;

/* io[f].active is the filter's alive flag and io[f].cur its grid (in/out);
 * kstep[f] its trajectory position (in/out); Z: nfilt x kf x b measurements;
 * rec: nfilt x steps records.  Scheduling is per STEP: `nslots` persistent
 * CTAs (one per workspace slot of ws_bytes) repeatedly claim any filter that
 * still has steps to run (per-filter lock), run one step and release it, so
 * filters whose steps cost 10x more than others do not leave SMs idle.
 * sched: 2 + 2*nfilt int32, zero-initialised (cursor, done, locks, counts). */
int ttgbf_filter_run(const ttgbf_model* model, const ttgbf_gauss* prior, ttgbf_grid_cfg gcfg, ttgbf_cross_cfg xcfg,
                     ttgbf_run_cfg rcfg, ttgbf_filter_io* io, int32_t* kstep, const double* Z, int nfilt,
                     const int32_t* probes, int nprobes, const int32_t* seeds, int nseeds, ttgbf_tt* state_hdr,
                     double* state, int64_t state_cap, void* ws, int64_t ws_bytes, int32_t* sched,
                     int nslots, ttgbf_diag* diag, ttgbf_step_rec* rec, void* stream);

/* ---- filter stages: one CTA per filter, nfilt filters per launch ---------
 * state_hdr[f] / state + f*state_cap: the filter's TT weights (in/out).
 * ws + f*ws_bytes: per-filter workspace.  probes: negative-mass probe cells
 * (nprobes x d, int32) of default_rng(0); seeds: _seed_lattice cells
 * (nseeds x d) -- both depend only on the grid shape. */
int ttgbf_filter_prior(const ttgbf_model* model, const ttgbf_gauss* prior, ttgbf_grid_cfg gcfg,
                       ttgbf_cross_cfg xcfg, const ttgbf_filter_io* io, int nfilt,
                       const int32_t* probes, int nprobes, ttgbf_tt* state_hdr, double* state,
                       int64_t state_cap, void* ws, int64_t ws_bytes, ttgbf_diag* diag, void* stream);

int ttgbf_filter_measure(const ttgbf_model* model, ttgbf_grid_cfg gcfg, ttgbf_cross_cfg xcfg,
                         const ttgbf_filter_io* io, int nfilt, const int32_t* probes, int nprobes,
                         const int32_t* seeds, int nseeds, ttgbf_tt* state_hdr, double* state,
                         int64_t state_cap, void* ws, int64_t ws_bytes, ttgbf_diag* diag, void* stream);

int ttgbf_filter_time_update(const ttgbf_model* model, ttgbf_grid_cfg gcfg, ttgbf_cross_cfg xcfg,
                             const ttgbf_filter_io* io, int nfilt, const int32_t* probes, int nprobes,
                             const int32_t* seeds, int nseeds, ttgbf_tt* state_hdr, double* state,
                             int64_t state_cap, void* ws, int64_t ws_bytes, ttgbf_diag* diag,
                             void* stream);

/* Algorithm 2 time update of tt_pmf_step (filters.py:876-885): transition
 * cross over the 2d modes (io.pred = new grid, io.cur = old grid), backward
 * contraction with the filtering TT in the state (tt_einsum_tpm,
 * tt_algorithms.py:603-635), scale by the old cell volume, finalize.
 * diag.cross[1] receives the transition cross info; d <= 8. */
int ttgbf_filter_time_update_std(const ttgbf_model* model, ttgbf_grid_cfg gcfg, ttgbf_cross_cfg xcfg,
                                 const ttgbf_filter_io* io, int nfilt, const int32_t* probes, int nprobes,
                                 ttgbf_tt* state_hdr, double* state, int64_t state_cap, void* ws, int64_t ws_bytes,
                                 ttgbf_diag* diag, void* stream);

/* ---- TT primitives (batched over `count` independent items, one CTA each).
 * Inputs/outputs are arrays of packed TTs: hdr[i] with data + i*cap. ---- */
int ttgbf_tt_round(const ttgbf_tt* in_hdr, const double* in, int64_t in_cap, int count, double tol,
                   int max_rank, ttgbf_tt* out_hdr, double* out, int64_t out_cap, void* ws,
                   int64_t ws_bytes, int32_t* status, void* stream);

int ttgbf_tt_hadamard(const ttgbf_tt* a_hdr, const double* a, int64_t a_cap, const ttgbf_tt* b_hdr,
                      const double* b, int64_t b_cap, int count, ttgbf_tt* out_hdr, double* out,
                      int64_t out_cap, void* ws, int64_t ws_bytes, int32_t* status, void* stream);

int ttgbf_tt_fft_convolve(const ttgbf_tt* k_hdr, const double* k, int64_t k_cap, const ttgbf_tt* w_hdr,
                          const double* w, int64_t w_cap, int count, double tol, int max_rank,
                          ttgbf_tt* out_hdr, double* out, int64_t out_cap, void* ws, int64_t ws_bytes,
                          int32_t* status, void* stream);

/* old/new axes: arrays of d ttgbf_axis per item (device) */
int ttgbf_tt_interpolate(const ttgbf_tt* in_hdr, const double* in, int64_t in_cap, int count,
                         const ttgbf_axis* old_axes, const ttgbf_axis* new_axes, ttgbf_tt* out_hdr,
                         double* out, int64_t out_cap, void* ws, int64_t ws_bytes, int32_t* status,
                         void* stream);

/* idx: K x d int32 per item (item stride K*d); out: K per item */
int ttgbf_tt_eval_many(const ttgbf_tt* hdr, const double* data, int64_t cap, int count, const int32_t* idx,
                       int64_t K, double* out, void* ws, int64_t ws_bytes, int32_t* status, void* stream);

/* pts: K x d doubles per item; axes: d ttgbf_axis per item */
int ttgbf_tt_eval_at_points(const ttgbf_tt* hdr, const double* data, int64_t cap, int count,
                            const ttgbf_axis* axes, const double* pts, int64_t K, double* out, void* ws,
                            int64_t ws_bytes, int32_t* status, void* stream);

/* out per item: TTGBF_NMOM doubles (sum, first, second raw moments against
 * the axis coordinates; axes: d ttgbf_axis per item) */
int ttgbf_tt_sum_moments(const ttgbf_tt* hdr, const double* data, int64_t cap, int count,
                         const ttgbf_axis* axes, double* out, void* ws, int64_t ws_bytes, int32_t* status,
                         void* stream);

/* black-box kinds for ttgbf_greedy_cross */
#define TTGBF_BB_GAUSS 0       /* prior pdf on the grid (uses prior)           */
#define TTGBF_BB_LIKELIHOOD 1  /* p(z|x) on the grid (uses model, io.z)        */
#define TTGBF_BB_KERNEL 2      /* FFT kernel on the grid (uses model)          */
#define TTGBF_BB_REALIGN 3     /* conv TT (grid io.filt) at F^-1 y, y on io.pred */

int ttgbf_greedy_cross(int kind, const ttgbf_model* model, const ttgbf_gauss* prior, ttgbf_cross_cfg xcfg,
                       const ttgbf_filter_io* io, int count, const int32_t* seeds, int nseeds,
                       ttgbf_tt* out_hdr, double* out, int64_t out_cap, void* ws, int64_t ws_bytes,
                       ttgbf_diag* diag, void* stream);

/* The black boxes themselves at integer grid indices, without cross or cache
 * (the values greedy_cross samples).  Replaces, per kind:
 *   TTGBF_BB_GAUSS       initial_pmd_tt's eval_many           filters.py:504-505
 *                        (GaussianDensity.pdf, models.py:60-66)
 *   TTGBF_BB_LIKELIHOOD  StateSpaceModel.likelihood           models.py:150-153
 *                        (measure :146-148, angle_wrap_residual :72-82)
 *   TTGBF_BB_KERNEL      _kernel_values / fft_kernel_blackbox filters.py:697-729
 *   TTGBF_BB_REALIGN     the realign evaluator                filters.py:969-979
 *                        (tt_eval_at_points, tt_algorithms.py:721-745)
 * Item i uses io[i] (cur grid and z; filt/pred grids for REALIGN), the TT
 * tt_hdr[i] / tt + i*tt_cap (REALIGN only, may be NULL otherwise), idx + i*K*d
 * (int32, K x d) and writes out + i*K; status[i] receives the item status. */
int ttgbf_eval_blackbox(int kind, const ttgbf_model* model, const ttgbf_gauss* prior, const ttgbf_filter_io* io,
                        const ttgbf_tt* tt_hdr, const double* tt, int64_t tt_cap, int count, const int32_t* idx,
                        int64_t K, double* out, void* ws, int64_t ws_bytes, int32_t* status, void* stream);

/* negative mass of a normalised TT on grid `axes` (returned already
 * multiplied by the cell volume) */
int ttgbf_negative_mass(const ttgbf_tt* hdr, const double* data, int64_t cap, int count,
                        const ttgbf_axis* axes, int64_t guard, const int32_t* probes, int nprobes,
                        double* out, void* ws, int64_t ws_bytes, int32_t* status, void* stream);

/* The cross's random streams on the device (tt_algorithms.py:341-433 draw
 * through numpy.random.Generator): kind 0 = rng.integers(0, shape, size=(K, d))
 * -> out[K*d]; kind 1 = rng.choice(pop, size, replace=False) -> out[size].
 * state6 (device, in/out): PCG64 state lo/hi, increment lo/hi, has_uint32,
 * uinteger -- numpy's bit_generator.state after the call equals it.  One CTA;
 * ws >= 16 * (pop + size) + 2^20 bytes. */
int ttgbf_rng_draws(int kind, uint64_t* state6, const int32_t* shape, int d, int64_t K, int64_t pop, int64_t size,
                    int64_t* out, void* ws, int64_t ws_bytes, int32_t* status, void* stream);

/* library info */
int ttgbf_version(void);
int ttgbf_block_threads(void);
int64_t ttgbf_smem_bytes(void);
int ttgbf_ctas_per_sm(void);   /* resident CTAs per SM the kernels are built for */
const char* ttgbf_status_string(int status);
/* sizeof of the ABI structs, for binding checks: 0 axis, 1 tt, 2 cross_cfg,
 * 3 grid_cfg, 4 diag, 5 model, 6 gauss, 7 filter_io, 8 run_cfg, 9 step_rec */
int64_t ttgbf_sizeof(int which);

/* ---- dense grid filter: dense_fft_pmf_step (filters.py:888-934) --------
 * Weights are C-order float64 arrays over the grid `axes` (d <= 8 axes);
 * complex buffers are interleaved (re, im) float64.  `axes` and `shape` are
 * HOST arrays (read on the host, the geometry goes to the kernels by value);
 * every other pointer is device memory.  Each call launches on `stream` and
 * returns a status. */

/* initial_pmd_dense values N(x - mean; cov) (filters.py:487-494) */
int ttgbf_dense_prior(const ttgbf_gauss* prior, const ttgbf_axis* axes, int d, double* w, void* stream);
/* w *= p(z | x) (measurement_update, dense branch, filters.py:564-566) */
int ttgbf_dense_likelihood(const ttgbf_model* model, const double* z, const ttgbf_axis* axes, int d, double* w,
                           void* stream);
/* deterministic sums over the grid into out[]:
 *   mode 0: {sum max(w,0), sum min(w,0)}           (_finalize_dense, filters.py:439-451)
 *   mode 1: {sum w*cv, sum_k x_k w*cv}             (moments_from_pmd, filters.py:323-329)
 *   mode 2: {sum (x_i-m_i)(x_j-m_j) w*cv, i <= j}  (filters.py:330-332)
 * partials: ttgbf_dense_reduce_blocks() doubles of scratch. */
int ttgbf_dense_reduce(const double* w, const ttgbf_axis* axes, int d, int mode, double cell_volume,
                       const double* mean, double* partials, double* out, void* stream);
int ttgbf_dense_reduce_blocks(void);
/* w = max(w, 0) / mass (_finalize_dense) */
int ttgbf_dense_finalize(double* w, int64_t n, double mass, void* stream);
/* RegularGridInterpolator(old axes, w_old, "linear", fill 0) at the new grid's
 * nodes mapped by F^-1 (Finv row-major, leading dimension TTGBF_MAXD), written
 * as complex (filters.py:911-916) */
int ttgbf_dense_interp(const double* w_old, const ttgbf_axis* old_axes, const ttgbf_axis* new_axes, int d,
                       const double* Finv, double* out_complex, void* stream);
/* FFT kernel N(disp; 0, Q) * cell_volume / |det F| on ifftshift
 * displacements idx * steps, written as complex (filters.py:920-927) */
int ttgbf_dense_kernel(const ttgbf_model* model, const ttgbf_axis* axes, int d, const double* steps,
                       double cell_volume, double abs_det_f, double* out_complex, void* stream);
/* in-place DFT along `axis` (numpy.fft.fftn / ifftn per axis; inverse scales
 * by 1/n); roots_complex = exp(-2 pi i q / n), q < n (filters.py:732-736) */
int ttgbf_dense_dft(double* data_complex, const int32_t* shape, int d, int axis, int inverse,
                    const double* roots_complex, void* stream);
/* a *= b (complex, n elements); w = Re(a) */
int ttgbf_dense_cmul(double* a_complex, const double* b_complex, int64_t n, void* stream);
int ttgbf_dense_real(const double* a_complex, double* w, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* TTGBF_H */
