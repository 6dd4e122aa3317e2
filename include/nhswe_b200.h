/*
 * nhswe_b200.h -- C ABI of the B200-native adaptive non-hydrostatic SWE step.
 *
 * Drop-in boundary for the time-step hot path of the reference package
 * `nhswe` (arXiv 2505.17025; /root/reference/pkg/src/nhswe).  Every entry
 * point is a plain C function over device pointers and sizes (no torch
 * types); all work is enqueued asynchronously on the caller's CUDA stream
 * (`stream` is a cudaStream_t passed as void*, NULL = legacy stream).
 * Functions return 0 on success or a negative NH_E* launch/argument code.
 * Numerical failures (positivity, elliptic breakdown) are reported per
 * member through nh_status records in device memory, which the caller reads
 * after synchronising and maps to the reference exception types.
 *
 * State layout (reference grid.py:137-147 per field, plus a member axis):
 *   h, hu, hw : float64 [B][N][2], C-contiguous, node j of element e at
 *               index (b*N + e)*2 + j.
 */
#ifndef NHSWE_B200_H
#define NHSWE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NH_ABI_VERSION 5   /* 5: nh_pm_ldg_solve takes outer_left and residual_tol (general LDG flux); 2: nh_outputs gauge fields; 3: nh_pm_* (orders p > 1), w / w_x on nh_stream_advance;
                               4: residual gate (nh_scheme.residual_tol, nh_status resid_*) */

/* bottom model kinds (reference bathymetry.py:66-184 + harness models) */
#define NH_BOTTOM_FLAT 0          /* FlatBottom(h0)                         bathymetry.py:66-79   */
#define NH_BOTTOM_PLATE 1         /* HammackPlate(h0, zeta0, b, alpha)      bathymetry.py:82-116  */
#define NH_BOTTOM_QUARTIC_SLIDE 2 /* WhittakerSlide + SlideMotion           bathymetry.py:119-184 */
#define NH_BOTTOM_SMOOTH_BOX 3    /* harness: tanh-edged box uplift (configs 2, 4)                */
#define NH_BOTTOM_SLOPE_SLIDE 4   /* harness: Gaussian mound on a plane slope (configs 3, 5)      */

/* boundary kinds (hydrostatic.py:29-52) */
#define NH_BC_ABSORBING 0
#define NH_BC_WALL 1

/* step modes (adaptivity.py:127-163) */
#define NH_MODE_HYDROSTATIC 0     /* predictor only                                   */
#define NH_MODE_GLOBAL 1          /* predictor + correction on [0, N-1]                */
#define NH_MODE_ADAPTIVE 2        /* predictor + criterion mask + correction on ranges */
#define NH_MODE_CORRECT_GIVEN 3   /* no predictor: correct the input state on given flags
                                     (corrector.apply_correction, corrector.py:485-498) */

/* criterion kinds (adaptivity.py:21, 75-96) */
#define NH_CRIT_ETA_OVER_D 0
#define NH_CRIT_ETA_X 1
#define NH_CRIT_U 2
#define NH_CRIT_U_X 3
#define NH_CRIT_W 4
#define NH_CRIT_W_X 5

/* status codes */
#define NH_OK 0
#define NH_ERR_POSITIVITY_ENTRY 1   /* rhs entry check: PositivityError(element, t) hydrostatic.py:101-103 */
#define NH_ERR_POSITIVITY_STAGE1 2  /* _advance after stage 1: PositivityError(-1, t+dt) :216-217       */
#define NH_ERR_POSITIVITY_STAGE2 3  /* _advance after stage 2: PositivityError(-1, t+dt)                */
#define NH_ERR_SOLVE_NONFINITE 4    /* EllipticSolveError, corrector.py:356-357                        */
#define NH_ERR_SOLVE_PIVOT 5        /* zero pivot in the condensed elimination (singular system)         */
#define NH_ERR_SOLVE_RESIDUAL 6     /* EllipticSolveError: ||Ax-b|| / max(||b||, max|A| ||x||) of a
                                       step's batched system above residual_tol, corrector.py:359-366  */
#define NH_ERR_STRUCTURE 7          /* AssertionError: s12 > 0 violated at a flagged node,
                                       corrector.py:70-74 (s11 + s21 = 0 holds by construction)     */

/* launch / argument errors (return values) */
#define NH_E_ARG (-1)
#define NH_E_CUDA (-2)
#define NH_E_UNSUPPORTED (-3)

/* Per-member grid, bottom and boundary description (312 bytes).
 * Grid operator values must be the reference GridSpec's (grid.py:71-114):
 * they are 1-4 ulp off closed forms and are copied, not recomputed. */
typedef struct nh_member {
    double x_left;          /* GridSpec.x_left                              */
    double dx;              /* GridSpec.dx                                  */
    double dt;              /* fixed step (driver.py:84)                    */
    double eps;             /* sample-node inset 1e-9*dx (grid.py:87)       */
    double two_over_dx;     /* 2.0/dx (grid.py:215)                         */
    double weak_div[4];     /* M^-1 K, row-major                            */
    double lift_left[2];
    double lift_right[2];
    double mass[4];
    double stiffness[4];
    double deriv_ref[4];
    double bottom[12];      /* model parameters, layout in csrc/bathy.cuh   */
    int32_t bc_left;        /* NH_BC_*                                      */
    int32_t bc_right;
    int32_t bottom_kind;    /* NH_BOTTOM_*                                  */
    int32_t reserved;
} nh_member;

/* Scheme constants shared by all members of one call. */
typedef struct nh_scheme {
    double g;               /* GRAVITY                                      */
    double rho;             /* RHO_WATER                                    */
    double k_nh;            /* Criterion.k_nh                               */
    double c11, c12, c22;   /* FluxCoefficients (corrector.py:40-47)        */
    int32_t mode;           /* NH_MODE_*                                    */
    int32_t criterion;      /* NH_CRIT_*                                    */
    int32_t enlarge;        /* Criterion.enlarge                            */
    int32_t record_cfl;     /* track max advisory CFL (hydrostatic.py:199)  */
    double residual_tol;    /* residual gate of every elliptic solve (corrector.py:297,
                               359-366; the reference default is 1e-10); <= 0 disables the gate
                               (the norms are still accumulated)                                */
} nh_scheme;

/* Per-member result record, written by the device. */
typedef struct nh_status {
    uint64_t error_key;     /* all-ones = ok (caller initialises); else the smallest
                               (step<<34)|(code<<30)|(element+1) seen        */
    double cfl_max;         /* max advisory CFL seen (if record_cfl)        */
    int64_t flagged;        /* flagged elements summed over the steps       */
    int32_t steps_done;
    int32_t any_hw;         /* any(hw != 0) of the output state (w/w_x fallback) */
    double resid_max;       /* largest relative residual of the steps' elliptic solves
                               (the reference's `rel`, corrector.py:359-362)          */
    double resid_acc[4];    /* running sums of the current solve: ||Ax-b||^2, ||b||^2,
                               ||x||^2 and max|A| (device scratch; zero between solves) */
} nh_status;

/* Optional outputs of nh_advance. */
typedef struct nh_outputs {
    uint32_t* flag_bits;    /* [n_steps][B][ceil(N/32)] per-step mask bits, or NULL */
    double* p_nh;           /* [B][N][2] pressure of the last step (0 off ranges), or NULL */
    const uint32_t* given_flags; /* NH_MODE_CORRECT_GIVEN: [B][ceil(N/32)] */
    /* Gauges (driver.py:58-69, 88-94): h at n_gauges sample nodes after every
     * step, recorded on the device so the loop never syncs.  gauge_nodes[g] =
     * flat index e*2 + j of the node in a member's (N, 2) field; gauge_h is
     * [n_steps][B][n_gauges].  The host subtracts the depth at the gauge's
     * sample node and time, as the reference's record_gauges does. */
    const int32_t* gauge_nodes;
    double* gauge_h;
    int32_t n_gauges;
} nh_outputs;

int nh_abi_version(void);

/* Advance B independent channels by n_steps fused time steps, in place.
 * Replaces adaptivity.adaptive_step (adaptivity.py:127-163) called in the
 * loop of driver.simulate (driver.py:81-87); with n_steps == 1 and mode
 * NH_MODE_HYDROSTATIC it is hydrostatic.heun_step (hydrostatic.py:192-209),
 * with NH_MODE_CORRECT_GIVEN it is corrector.apply_correction
 * (corrector.py:485-498).  `time` [B] holds each member's t and is advanced
 * by t += dt per step (hydrostatic.py:206-209).  `status` [B] is
 * zero-initialised by the caller except error_key = ~0.
 * Limits (NH_E_UNSUPPORTED beyond them; nh_pm_advance with m = 2 has none):
 * n_elements <= 16 CTAs x (3 x 384 - 8) = 18304 per member (one cluster owns a
 * member); the alternating LDG flux family c12 = -1/2, c22 = 0 (any c11). */
int nh_advance(const nh_member* members, int n_members, int n_elements,
               double* h, double* hu, double* hw, double* time, int n_steps,
               const nh_scheme* scheme, const nh_outputs* outputs,
               nh_status* status, void* stream);

/* Streaming variant of nh_advance for large ensembles (same contract and
 * in-place semantics; modes HYDROSTATIC / GLOBAL / ADAPTIVE, every criterion --
 * the w / w_x all-zero-input fallback is one more kernel).  Every step is four kernels over
 * independent 120-element tiles of 128 threads (K_P predictor+criterion, K_S condensation,
 * K_X per-member tile chain, K_C reconstruction) with the vertical-momentum
 * update fused into the next step's load; state goes through HBM once per
 * step; after the loop K_fin applies the last pending update on the flagged
 * tiles.  `workspace` is device memory of at least
 * nh_stream_workspace_bytes(B, N) bytes.
 * Limits (NH_E_UNSUPPORTED beyond them; nh_pm_advance with m = 2 has none):
 * n_elements <= 32 x 8 x 120 = 30720 per member (K_X chains a member's
 * tiles with one warp); n_members x tiles < 2^31; the alternating LDG flux
 * family. */
int nh_stream_advance(const nh_member* members, int n_members, int n_elements,
                      double* h, double* hu, double* hw, double* time, int n_steps,
                      const nh_scheme* scheme, const nh_outputs* outputs,
                      nh_status* status, void* workspace, size_t workspace_bytes,
                      void* stream);
size_t nh_stream_workspace_bytes(int n_members, int n_elements);

/* Time loop of nh_stream_advance as a CUDA graph (default on; the
 * NH_STREAM_GRAPH=0 environment variable turns it off at load).  With
 * graphs on and per-kernel timing off, runs of >= 5 steps launch step 0,
 * then replay one captured graph of an (odd, even) step pair -- the ping-pong
 * buffers repeat with period 2 -- and launch a trailing odd step directly.
 * enable: 1 on, 0 off, -1 query.  Returns the previous setting. */
int nh_stream_graphs(int enable);

/* Per-kernel CUDA-event timing of nh_stream_advance (diagnostics for the
 * roofline report).  nh_stream_timing(1) clears and arms the recorder; every
 * later nh_stream_advance brackets each launch with events on its stream.
 * nh_stream_kernel_times waits for the last event and returns, per kernel
 * [K_P, K_S, K_X, K_C, K_fin, prep], the summed milliseconds and launch
 * counts since arming, then clears (timing stays armed until
 * nh_stream_timing(0)). */
#define NH_STREAM_NKERNELS 6
int nh_stream_timing(int enable);
int nh_stream_kernel_times(double* ms, long long* launches);

/* Number of kernels this library has enqueued since load (all entry points). */
long long nh_launch_count(void);

/* Self-test of the inline correctly rounded division / square root used in
 * the strict predictor against CUDA's __ddiv_rn / __dsqrt_rn on n random
 * operand pairs (all exponent ranges, zeros, denormals, inf, nan).
 * mismatches: device uint64[3] (division, sqrt, positive-divisor division),
 * accumulated. */
int nh_selftest_arith(long long n, unsigned long long seed, unsigned long long* mismatches,
                      void* stream);

/* ---------------------------------------------------------------------------
 * Polynomial orders p = 1..3 (m = p + 1 <= 4 GLL nodes per element; SURVEY.md
 * §8(f)4).  The reference grid and LDG templates are generic in m
 * (grid.py:19-114, corrector.py:173-370); these entry points run the same
 * step for any m with element-parallel kernels (csrc/pm_kernels.cu).  State
 * fields are [B][N][m].  Per-member m-node operators come in nh_pm_member
 * (the reference GridSpec's values, copied not recomputed); the nh_member
 * record supplies x_left, dx, dt, eps, 2/dx, bottom and boundaries (its P1
 * operator arrays are unused here).
 * ------------------------------------------------------------------------- */
#define NH_PM_MAX_NODES 4
typedef struct nh_pm_member {
    double weak_div[16];    /* M^-1 K, row-major m x m (leading dimension m) */
    double lift_left[4];    /* M^-1 e_first                                  */
    double lift_right[4];   /* M^-1 e_last                                   */
    double mass[16];        /* dx/2 * reference mass, row-major m x m       */
    double stiffness[16];   /* K[i][j] = int phi_i' phi_j (reference)       */
    double deriv_ref[16];   /* GLL differentiation matrix                   */
    double node_off[4];     /* 0.5*dx*(ref_j + 1): node j = x_left + dx*e + node_off[j] */
} nh_pm_member;

/* Workspace of nh_pm_advance in bytes. */
size_t nh_pm_workspace_bytes(int m, int n_members, int n_elements);

/* nh_advance for m nodes per element (modes HYDROSTATIC / GLOBAL / ADAPTIVE,
 * every criterion, any LDG flux; outputs flag_bits, p_nh [B][N][m], gauges
 * with flat node index e*m + j).  Per step: two Heun-stage kernels, then
 * flags, per-element LDG condensation, one chain thread per member,
 * reconstruction and the hw correction; with a flux outside the alternating
 * family the condensation / chain / reconstruction are replaced by one band
 * solve per range (see nh_pm_ldg_solve).  This is also the P1 (m = 2) path
 * for such a flux. */
int nh_pm_advance(const nh_member* members, const nh_pm_member* pm, int m,
                  int n_members, int n_elements, double* h, double* hu, double* hw,
                  double* time, int n_steps, const nh_scheme* scheme,
                  const nh_outputs* outputs, nh_status* status, void* workspace,
                  size_t workspace_bytes, void* stream);

/* rhs_operator (hydrostatic.py:88-184) and criterion_values
 * (adaptivity.py:75-96) for m nodes per element; fields [B][N][m]. */
int nh_pm_rhs(const nh_member* members, const nh_pm_member* pm, int m, int n_members,
              int n_elements, const double* h, const double* hu, const double* hw,
              const double* time, double g, double* t_h, double* t_hu, double* t_hw,
              nh_status* status, void* stream);
int nh_pm_criterion(const nh_member* members, const nh_pm_member* pm, int m, int n_members,
                    int n_elements, const double* h, const double* hu, const double* hw,
                    const double* time, int kind, double* values, void* stream);

/* Coefficient-level corrector functions for m nodes per element (fields
 * [B][N][m]; coef = [7][B][N][m] planes s11, s12, s22, f1, f2, phi, d_x):
 *  nh_pm_coefficients     phi_term + assemble_coefficients (corrector.py:100-170)
 *                         at the state's time, dt from the member record;
 *  nh_pm_ldg_solve        ldg_solve / solve_on_ranges (corrector.py:292-424) on
 *                         the flagged ranges (flags [B][ceil(N/32)]),
 *                         outer_right [B][N] = hu right of each element;
 *                         writes p (0 off the ranges) and hu on the ranges.
 *                         Any FluxCoefficients (corrector.py:40-47): the
 *                         alternating family (c12 = -1/2, c22 = 0) runs the
 *                         condensed chain; any other flux assembles each
 *                         range's band system as the reference does and
 *                         solves it by band elimination with partial
 *                         pivoting (what dgbsv does, corrector.py:352), with
 *                         the residual gate (residual_tol > 0).  That path
 *                         also needs outer_left [B][N] = hu left of each
 *                         element (NULL otherwise: its weight is 0);
 *  nh_pm_correct_momentum correct_momentum (corrector.py:427-482): hw_out =
 *                         hw + dt/rho * bottom pressure on the flagged elements. */
int nh_pm_coefficients(const nh_member* members, const nh_pm_member* pm, int m, int n_members,
                       int n_elements, const double* h, const double* hu, const double* hw,
                       const double* time, double g, double rho, double* coef, void* stream);
int nh_pm_ldg_solve(const nh_member* members, const nh_pm_member* pm, int m, int n_members,
                    int n_elements, const double* coef, const uint32_t* flags,
                    const double* outer_left, const double* outer_right, double rho, double c11,
                    double c12, double c22, double residual_tol, double* p, double* hu,
                    nh_status* status, void* workspace, size_t workspace_bytes, void* stream);
int nh_pm_correct_momentum(const nh_member* members, const nh_pm_member* pm, int m,
                           int n_members, int n_elements, const double* h, const double* p,
                           const double* coef, const uint32_t* flags, double rho,
                           const double* hw, double* hw_out, void* stream);

/* Semi-discrete tendency, hydrostatic.rhs_operator (hydrostatic.py:88-184).
 * Outputs t_h, t_hu, t_hw [B][N][2]. */
int nh_rhs(const nh_member* members, int n_members, int n_elements,
           const double* h, const double* hu, const double* hw, const double* time,
           double g, double* t_h, double* t_hu, double* t_hw,
           nh_status* status, void* stream);

/* Nodal indicator values, adaptivity.criterion_values (adaptivity.py:75-96). */
int nh_criterion(const nh_member* members, int n_members, int n_elements,
                 const double* h, const double* hu, const double* hw, const double* time,
                 int kind, double* values, void* stream);

/* evaluate_criterion's mask (adaptivity.py:99-113) from nodal indicator
 * values [B][N][nodes] (nh_criterion / nh_pm_criterion): flags[b][e] = max
 * over the element's nodes > k_nh, with the optional +-1 enlargement clipped
 * to the member. */
int nh_mask(const double* values, int n_members, int n_elements, int nodes, double k_nh,
            int enlarge, uint8_t* flags, void* stream);

/* max_wavespeed (hydrostatic.py:187-189): out[b] = max over the member's
 * nodes of |hu / h| + sqrt(g h), IEEE division and square root. */
int nh_max_wavespeed(const double* h, const double* hu, int n_members,
                     long long nodes_per_member, double g, double* out, void* stream);

/* Elliptic coefficients on all elements, corrector.phi_term +
 * assemble_coefficients (corrector.py:100-170).  coef [7][B][N][2] =
 * s11, s12, s22, f1, f2, phi, d_x (s21 = -s11). */
int nh_coefficients(const nh_member* members, int n_members, int n_elements,
                    const double* h, const double* hu, const double* hw, const double* time,
                    double g, double rho, double* coef, void* stream);

/* LDG solve from given coefficients on flagged ranges, corrector._solve_batched
 * / ldg_solve / solve_on_ranges (corrector.py:292-424).  coef as above
 * (only s11, s12, s22, f1, f2 read), flags [B][ceil(N/32)] (ranges = maximal
 * runs, split further where range_starts [B][ceil(N/32)] has a bit set, or
 * NULL: adjacent ranges are separate systems, as in the reference's
 * block-diagonal batch), outer_right [B][N] = outer hu trace used when
 * element e ends a range (corrector.py:388-403).  Outputs p, hu [B][N][2] on
 * flagged elements (untouched elsewhere).  The member's batched system is
 * checked like corrector.py:355-366: status.resid_max = ||Ax-b|| /
 * max(||b||, max|A| ||x||), NH_ERR_SOLVE_RESIDUAL above residual_tol (> 0). */
int nh_ldg_solve(const nh_member* members, int n_members, int n_elements,
                 const double* coef, const uint32_t* flags, const uint32_t* range_starts,
                 const double* outer_right, double rho, double c11, double c12, double c22,
                 double residual_tol, double* p, double* hu, nh_status* status, void* stream);

/* Vertical-momentum update from a solved pressure, corrector.correct_momentum
 * (corrector.py:441-482): hw_out = hw_in + dt/rho * bottom pressure on flagged
 * elements, hw_in elsewhere.  h = predictor depth, p [B][N][2] (0 off ranges),
 * coef as produced by nh_coefficients (phi, d_x planes read). */
int nh_correct_momentum(const nh_member* members, int n_members, int n_elements,
                        const double* h, const double* p, const double* coef,
                        const uint32_t* flags, double rho, const double* hw_in,
                        double* hw_out, void* stream);

/* Bottom channels at arbitrary points, BathymetryModel.sample
 * (bathymetry.py:43-57): out [6][B][n_points] = d, d_x, d_t, d_tt, d_xt, d_xx. */
int nh_bottom_sample(const nh_member* members, int n_members, const double* x, int n_points,
                     const double* time, double* out, void* stream);

/* Last CUDA runtime error string (diagnostics). */
const char* nh_last_cuda_error(void);

/* Launch geometry chosen for a member length (cluster size, tile, threads). */
int nh_plan(int n_elements, int n_members, int* cluster, int* tile, int* threads,
            int* smem_bytes);

#ifdef __cplusplus
}
#endif
#endif /* NHSWE_B200_H */
