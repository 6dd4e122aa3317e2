// The NH-SWE step for polynomial order p = m - 1 with m <= 4 GLL nodes per
// element.  The reference is generic in m: GridSpec builds
// the m-node operators (grid.py:71-114), rhs_operator uses them through
// matrix products (hydrostatic.py:88-184) and the LDG templates place 2m
// unknowns per element (corrector.py:173-370).  These kernels are the
// m-generic restatement of the P1 step (physics.cuh, stream_kp.cuh):
//
//   pm_stage<M,1>  Heun stage 1 at t: tendency (faces from the neighbours'
//                  end nodes, volume term, lifts, slope source), Q* = Q + dt k1
//   pm_stage<M,2>  stage 2 at t + dt, Heun combination, criterion value
//   pm_flags       mask: criterion, +-1 enlargement, global / w-fallback
//   pm_condense    LDG coefficients at t + dt and the element's 2m x 2m block
//                  eliminated to the same two-scalar super-element as P1:
//                    a_e = P(last node), z_e = Q(node 0) - c11 P(node 0)
//                  (with the alternating flux an element couples to its
//                  neighbours only through a_{e-1} and z_{e+1}, for any m)
//   pm_chain       one thread per member: Riccati sweep over the elements,
//                  then back-substitution -> (a_{e-1}, z_{e+1}) per element
//   pm_reconstruct the element unknowns -> hu, p
//   pm_correct     hw += dt/rho (6/quad p + d_x/quad (h p)_x + phi)
//
// Element-parallel, one thread per element, state [B][N][M] per field.  Not
// the throughput path (every config is P1, served by stream_kp.cu); written
// for parity with the reference at p = 2, 3, and checked at p = 1 against
// the P1 kernels.
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstring>
#include <algorithm>
#include "../../include/nhswe_b200.h"
#include "bathy.cuh"
#include "physics.cuh"

void nh_count_launch();   // capi.cu: the library's launch counter

namespace {

constexpr int PTB = 128;

struct PmArgs {
  const nh_member* members;
  const nh_pm_member* pm;
  const double* h_in;
  const double* hu_in;
  const double* hw_in;
  double* h_out;
  double* hu_out;
  double* hw_out;
  double* k1;       // [3][B*N*M] stage-1 tendency
  double* qs;       // [3][B*N*M] stage-1 state
  uint8_t* raw;     // [B*N] criterion flag before enlargement
  uint8_t* flags;   // [B*N]
  double* sup;      // [6][B*N] super-elements
  double* rec;      // [6M][B*N] element solution columns (g, alpha, beta)
  double* pdx;      // [2M][B*N] phi_j, d_x_j of flagged elements
  double* chain;    // [4][B*N] Riccati s_in, t_in, m, n
  double* io;       // [2][B*N] a_{e-1}, z_{e+1}
  double* p;        // [B*N*M] pressure of the step (0 off the ranges)
  double* time;
  nh_status* status;
  int* hw_any;      // [B]
  uint32_t* flag_bits;
  const int32_t* gauge_nodes;
  double* gauge_h;
  int n_gauges;
  const uint32_t* given;   // NH_MODE_CORRECT_GIVEN: [B][ceil(N/32)] ranges to correct
  const double* coef;      // coefficient-level calls: [7][B*N*M] s11 s12 s22 f1 f2 phi d_x
  const double* outer_right;   // coefficient-level solve: [B][N] hu right of each element
  const double* outer_left;    // ... and left of each element (general flux only)
  double* gen;      // general-flux band solve scratch, gen_doubles(M, N) per member
  int step;
  int corr;         // the step has a correction (mode != hydrostatic)
  int general;      // LDG flux outside the alternating family: pm_general_solve
  nh_scheme sch;
  int B, N;
};

template <int M>
struct Elem {
  double h[M], q[M], w[M];
};

// sample coordinate of node j of element e, bit-identical to GridSpec:
// edges = x_left + dx*e; nodes = edges + 0.5*dx*(ref + 1); inset +- 1e-9*dx
template <int M>
__device__ __forceinline__ double node_x(const nh_member& m, const nh_pm_member& c, int e, int j) {
  double x = __dadd_rn(__dadd_rn(m.x_left, __dmul_rn(m.dx, (double)e)), c.node_off[j]);
  if (j == 0) return __dadd_rn(x, m.eps);
  if (j == M - 1) return __dsub_rn(x, m.eps);
  return x;
}

template <int M>
__device__ __forceinline__ Elem<M> load_elem(const double* h, const double* hu, const double* hw,
                                             size_t o) {
  Elem<M> q;
#pragma unroll
  for (int j = 0; j < M; ++j) { q.h[j] = h[o + j]; q.q[j] = hu[o + j]; q.w[j] = hw[o + j]; }
  return q;
}

// (v @ A^T)[i] for a row-major m x m A: numpy's dgemm order (products summed
// from k = 0 with fused multiply-adds, as the P1 kernels' fma(v1, A1, v0*A0))
template <int M>
__device__ __forceinline__ double rowdot(const double (&v)[M], const double* A, int i) {
  double acc = RMUL(v[0], A[i * M]);
#pragma unroll
  for (int k = 1; k < M; ++k) acc = fma(v[k], A[i * M + k], acc);
  return acc;
}

// element derivative D(v) = (v @ deriv_ref^T) * (2/dx) (grid.py:214-215)
template <int M>
__device__ __forceinline__ void ederiv_m(const nh_member& m, const nh_pm_member& c,
                                         const double (&v)[M], double (&out)[M]) {
#pragma unroll
  for (int i = 0; i < M; ++i) out[i] = RMUL(rowdot<M>(v, c.deriv_ref, i), m.two_over_dx);
}

// Tendency of element e at time t (hydrostatic.py:99-183), q = its state,
// L = the left face's outer side, R = the right face's outer side.
template <int M>
__device__ __forceinline__ void tendency(const nh_member& m, const nh_pm_member& c, double g,
                                         const Elem<M>& q, const double (&d)[M],
                                         const double (&dxb)[M], const Side& L, const Side& R,
                                         bool slope, double (&t)[3][M]) {
  const double hg = 0.5 * g;
  double u[M], f2[M], f3[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    u[j] = RDIVP(q.q[j], q.h[j]);
    f2[j] = RADD(RMUL(q.q[j], u[j]), RMUL(RMUL(hg, q.h[j]), q.h[j]));
    f3[j] = RMUL(u[j], q.w[j]);
  }
  Side n0, nl;
  n0.h = q.h[0]; n0.hu = q.q[0]; n0.hw = q.w[0]; n0.d = d[0]; n0.u = u[0]; n0.rh = 0.0;
  nl.h = q.h[M - 1]; nl.hu = q.q[M - 1]; nl.hw = q.w[M - 1]; nl.d = d[M - 1]; nl.u = u[M - 1];
  nl.rh = 0.0;
#if !NH_STRICT
  n0.rh = nh_rcp(n0.h); nl.rh = nh_rcp(nl.h);
#endif
  double sp;
  const Face fl = face_flux<false>(L, n0, g, sp);
  const Face fr = face_flux<false>(nl, R, g, sp);
  const double* W = c.weak_div;
#pragma unroll
  for (int i = 0; i < M; ++i) {
    t[0][i] = RADD(RSUB(rowdot<M>(q.q, W, i), RMUL(fr.F1, c.lift_right[i])),
                   RMUL(fl.F1, c.lift_left[i]));
    double v2 = RADD(RSUB(rowdot<M>(f2, W, i), RMUL(fr.F2L, c.lift_right[i])),
                     RMUL(fl.F2R, c.lift_left[i]));
    t[1][i] = slope ? RADD(v2, RMUL(RMUL(g, q.h[i]), dxb[i])) : v2;
    t[2][i] = RADD(RSUB(rowdot<M>(f3, W, i), RMUL(fr.F3, c.lift_right[i])),
                   RMUL(fl.F3, c.lift_left[i]));
  }
}

// the outer sides of element e's two faces from the neighbours' end nodes
// (or the boundary ghosts, hydrostatic.py:127-140), at time t
template <int M>
__device__ __forceinline__ void face_sides(const nh_member& m, const nh_pm_member& c,
                                           const BottomTime& bt, const double* h,
                                           const double* hu, const double* hw, int b, int e,
                                           int N, const Elem<M>& q, const double (&d)[M],
                                           Side& L, Side& R) {
  if (e > 0) {
    const size_t o = ((size_t)b * N + e - 1) * M + (M - 1);
    L = make_side(h[o], hu[o], hw[o], bottom_depth(m, bt, node_x<M>(m, c, e - 1, M - 1)));
  } else {
    L = ghost_side(make_side(q.h[0], q.q[0], q.w[0], d[0]), m.bc_left);
  }
  if (e < N - 1) {
    const size_t o = ((size_t)b * N + e + 1) * M;
    R = make_side(h[o], hu[o], hw[o], bottom_depth(m, bt, node_x<M>(m, c, e + 1, 0)));
  } else {
    R = ghost_side(make_side(q.h[M - 1], q.q[M - 1], q.w[M - 1], d[M - 1]), m.bc_right);
  }
}

__device__ __forceinline__ bool has_slope(const nh_member& m) {
  // FlatBottom / HammackPlate sample an identically zero d_x: the reference
  // skips the g h d_x source (hydrostatic.py:176-178)
  return m.bottom_kind != NH_BOTTOM_FLAT && m.bottom_kind != NH_BOTTOM_PLATE;
}

// criterion_values (adaptivity.py:75-96) of one element; d = depth at the
// state's time
template <int M>
__device__ __forceinline__ void criterion_m(const nh_member& m, const nh_pm_member& c, int kind,
                                            const Elem<M>& q, const double (&d)[M],
                                            double (&v)[M]) {
  double a[M], r[M];
  switch (kind) {
    case NH_CRIT_ETA_OVER_D:
#pragma unroll
      for (int j = 0; j < M; ++j) v[j] = fabs(RDIVP(RSUB(q.h[j], d[j]), d[j]));
      return;
    case NH_CRIT_ETA_X:
#pragma unroll
      for (int j = 0; j < M; ++j) a[j] = RSUB(q.h[j], d[j]);
      break;
    case NH_CRIT_U:
    case NH_CRIT_U_X:
#pragma unroll
      for (int j = 0; j < M; ++j) a[j] = RDIVP(q.q[j], q.h[j]);
      break;
    default:
#pragma unroll
      for (int j = 0; j < M; ++j) a[j] = RDIVP(q.w[j], q.h[j]);
      break;
  }
  if (kind == NH_CRIT_U || kind == NH_CRIT_W) {
#pragma unroll
    for (int j = 0; j < M; ++j) v[j] = fabs(a[j]);
    return;
  }
  ederiv_m<M>(m, c, a, r);
#pragma unroll
  for (int j = 0; j < M; ++j) v[j] = fabs(r[j]);
}

__device__ __forceinline__ void atomic_max_pos(double* addr, double v) {
  atomicMax((unsigned long long*)addr, (unsigned long long)__double_as_longlong(v));
}

// ------------------------------------------------------------- Heun stages
template <int M, int STAGE>
__global__ void __launch_bounds__(PTB) pm_stage(PmArgs a) {
  const int idx = blockIdx.x * PTB + threadIdx.x;
  if (idx >= a.B * a.N) return;
  const int N = a.N, b = idx / N, e = idx - b * N;
  const nh_member& m = a.members[b];
  const nh_pm_member& c = a.pm[b];
  const double g = a.sch.g, dt = m.dt, t0 = a.time[b];
  const size_t BNM = (size_t)a.B * N * M, o = (size_t)idx * M;
  nh_status* st = a.status + b;
  const double* sh = STAGE == 1 ? a.h_in : a.qs;
  const double* sq = STAGE == 1 ? a.hu_in : a.qs + BNM;
  const double* sw = STAGE == 1 ? a.hw_in : a.qs + 2 * BNM;
  const Elem<M> q = load_elem<M>(sh, sq, sw, o);
  const BottomTime bt = bottom_time(m, STAGE == 1 ? t0 : t0 + dt);
  double d[M], dxb[M];
#pragma unroll
  for (int j = 0; j < M; ++j) bottom_d_dx(m, bt, node_x<M>(m, c, e, j), d[j], dxb[j]);
  if (STAGE == 1) {
    bool bad = false, hwnz = false;
    double speed = 0.0;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      bad |= !(q.h[j] > 0.0);
      hwnz |= q.w[j] != 0.0;
    }
    if (bad) { nh_report(st, a.step, NH_ERR_POSITIVITY_ENTRY, e); return; }
    if (a.sch.record_cfl) {   // max_wavespeed of the input (hydrostatic.py:187-189, 198-201)
#pragma unroll
      for (int j = 0; j < M; ++j)
        speed = fmax(speed, fabs(q.q[j] / q.h[j]) + sqrt(g * q.h[j]));
      atomic_max_pos(&st->cfl_max, speed * dt / m.dx);
    }
    if (hwnz && a.hw_any) a.hw_any[b] = 1;
  }
  Side L, R;
  face_sides<M>(m, c, bt, sh, sq, sw, b, e, N, q, d, L, R);
  double t[3][M];
  tendency<M>(m, c, g, q, d, dxb, L, R, has_slope(m), t);
  if (STAGE == 1) {
    bool bad = false;
#pragma unroll
    for (int f = 0; f < 3; ++f)
#pragma unroll
      for (int j = 0; j < M; ++j) a.k1[f * BNM + o + j] = t[f][j];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const double hs = RADD(q.h[j], RMUL(dt, t[0][j]));
      bad |= !(hs > 0.0);
      a.qs[o + j] = hs;
      a.qs[BNM + o + j] = RADD(q.q[j], RMUL(dt, t[1][j]));
      a.qs[2 * BNM + o + j] = RADD(q.w[j], RMUL(dt, t[2][j]));
    }
    if (bad) nh_report(st, a.step, NH_ERR_POSITIVITY_STAGE1, -1);
    return;
  }
  // stage 2: Heun combination Q~ = Q + dt (k1 + k2) / 2 (hydrostatic.py:205-209)
  const Elem<M> q0 = load_elem<M>(a.h_in, a.hu_in, a.hw_in, o);
  Elem<M> qp;
  bool bad = false;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    qp.h[j] = RADD(q0.h[j], RMUL(dt, RMUL(0.5, RADD(a.k1[o + j], t[0][j]))));
    qp.q[j] = RADD(q0.q[j], RMUL(dt, RMUL(0.5, RADD(a.k1[BNM + o + j], t[1][j]))));
    qp.w[j] = RADD(q0.w[j], RMUL(dt, RMUL(0.5, RADD(a.k1[2 * BNM + o + j], t[2][j]))));
    bad |= !(qp.h[j] > 0.0);
    a.h_out[o + j] = qp.h[j];
    a.hu_out[o + j] = qp.q[j];
    a.hw_out[o + j] = qp.w[j];
  }
  if (bad) nh_report(st, a.step, NH_ERR_POSITIVITY_STAGE2, -1);
  if (a.sch.mode == NH_MODE_ADAPTIVE) {   // criterion on the predictor, depth at t + dt
    double v[M];
    criterion_m<M>(m, c, a.sch.criterion, qp, d, v);
    double mx = v[0];
#pragma unroll
    for (int j = 1; j < M; ++j) mx = fmax(mx, v[j]);
    a.raw[idx] = mx > a.sch.k_nh ? 1 : 0;
  }
}

// ------------------------------------------------------------------- mask
__global__ void __launch_bounds__(PTB) pm_flags(PmArgs a) {
  const int idx = blockIdx.x * PTB + threadIdx.x;
  if (idx >= a.B * a.N) return;
  const int N = a.N, b = idx / N, e = idx - b * N;
  bool f = true;   // global mode, and the w / w_x fallback (adaptivity.py:153-154)
  const bool wcrit = a.sch.criterion == NH_CRIT_W || a.sch.criterion == NH_CRIT_W_X;
  if (a.given) {   // apply_correction on given ranges (corrector.py:485-498)
    f = (a.given[(size_t)b * ((N + 31) / 32) + (e >> 5)] >> (e & 31)) & 1u;
  } else if (a.sch.mode == NH_MODE_ADAPTIVE && !(wcrit && !a.hw_any[b])) {
    f = a.raw[idx] != 0;
    if (a.sch.enlarge) {   // enlarge_flags (adaptivity.py:99-104)
      if (e > 0) f = f || a.raw[idx - 1];
      if (e < N - 1) f = f || a.raw[idx + 1];
    }
  }
  a.flags[idx] = f ? 1 : 0;
  if (f) {
    atomicAdd((unsigned long long*)&a.status[b].flagged, 1ull);
    if (a.flag_bits) {
      const int nw = (N + 31) / 32;
      atomicOr(a.flag_bits + ((size_t)a.step * a.B + b) * nw + (e >> 5), 1u << (e & 31));
    }
  }
}

// ------------------------------------------------------------ condensation
// Gauss-Jordan with partial pivoting on the 2M x (2M + 3) augmented block
// [A | b | l | v]; returns false on a zero / non-finite pivot.
template <int M>
__device__ __forceinline__ bool gauss_jordan(double (&A)[2 * M][2 * M + 3]) {
  constexpr int R = 2 * M, C = 2 * M + 3;
  bool ok = true;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    int piv = k;
    double best = fabs(A[k][k]);
#pragma unroll
    for (int i = k + 1; i < R; ++i)
      if (fabs(A[i][k]) > best) { best = fabs(A[i][k]); piv = i; }
    if (piv != k) {
#pragma unroll
      for (int cc = 0; cc < C; ++cc) {
        double tmp = A[k][cc]; A[k][cc] = A[piv][cc]; A[piv][cc] = tmp;
      }
    }
    const double pv = A[k][k];
    ok = ok && pv != 0.0 && isfinite(pv);
    const double r = 1.0 / pv;
#pragma unroll
    for (int cc = k + 1; cc < C; ++cc) A[k][cc] *= r;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      if (i == k) continue;
      const double f = A[i][k];
#pragma unroll
      for (int cc = k + 1; cc < C; ++cc) A[i][cc] = fma(-f, A[k][cc], A[i][cc]);
    }
  }
  return ok;
}

__device__ __forceinline__ bool given_flag(const PmArgs& a, int b, int e) {
  return (a.given[(size_t)b * ((a.N + 31) / 32) + (e >> 5)] >> (e & 31)) & 1u;
}

__device__ __forceinline__ void store_super_pm(const PmArgs& a, int idx, const Super& S) {
  const size_t BN = (size_t)a.B * a.N;
  a.sup[idx] = S.ga; a.sup[BN + idx] = S.aa; a.sup[2 * BN + idx] = S.ba;
  a.sup[3 * BN + idx] = S.gz; a.sup[4 * BN + idx] = S.az; a.sup[5 * BN + idx] = S.bz;
}

// One flagged element's 2M x 2M LDG block (unknowns interleaved P0, Q0, P1,
// Q1, ... as the reference's template, corrector.py:187-203, values
// :329-336) eliminated to its super-element; the solution columns go to rec
// for the reconstruction, phi / d_x to pdx for the hw update.
template <int M>
__device__ __forceinline__ void condense_block(const PmArgs& a, const nh_pm_member& c,
                                               const NodeCoef (&nc)[M], const double (&dxb)[M],
                                               int b, int e, int idx, bool range_end) {
  const size_t BN = (size_t)a.B * a.N;
  constexpr int R = 2 * M;
  double A[R][R + 3];
  const double* Mm = c.mass;
  const double* K = c.stiffness;
  const double rho = a.sch.rho, inv_rho = 1.0 / rho, c11 = a.sch.c11;
#pragma unroll
  for (int i = 0; i < M; ++i) {
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const double Mij = Mm[i * M + j], Kij = K[i * M + j];
      A[2 * i][2 * j] = -Kij + Mij * nc[j].s11;
      A[2 * i][2 * j + 1] = Mij * (nc[j].s12 * inv_rho);
      A[2 * i + 1][2 * j + 1] = -Kij + Mij * (-nc[j].s11);
      A[2 * i + 1][2 * j] = Mij * (rho * nc[j].s22);
    }
    double f1[M], f2[M];
#pragma unroll
    for (int j = 0; j < M; ++j) { f1[j] = nc[j].f1 * inv_rho; f2[j] = nc[j].f2; }
    A[2 * i][R] = rowdot<M>(f1, Mm, i);
    A[2 * i + 1][R] = rowdot<M>(f2, Mm, i);
#pragma unroll
    for (int cc = R + 1; cc < R + 3; ++cc) { A[2 * i][cc] = 0.0; A[2 * i + 1][cc] = 0.0; }
  }
  // faces, alternating flux (c12 = -1/2, c22 = 0), corrector.py:205-224:
  //   left : P row -a_{e-1};  Q row -(Q0 + c11 (a_{e-1} - P0))
  //   right: P row +P_last (inside a range; p* = 0 at a range end);
  //          Q row +(z_{e+1} + c11 P_last)
  A[1][1] -= 1.0;
  A[1][0] += c11;
  if (!range_end) A[R - 2][R - 2] += 1.0;
  A[R - 1][R - 2] += c11;
  A[0][R + 1] = 1.0;
  A[1][R + 1] = c11;
  A[R - 1][R + 2] = -1.0;
  if (!gauss_jordan<M>(A)) nh_report(a.status + b, a.step, NH_ERR_SOLVE_PIVOT, e);
  Super S;
  S.ga = A[R - 2][R]; S.aa = A[R - 2][R + 1]; S.ba = A[R - 2][R + 2];
  S.gz = fma(-c11, A[0][R], A[1][R]);
  S.az = fma(-c11, A[0][R + 1], A[1][R + 1]);
  S.bz = fma(-c11, A[0][R + 2], A[1][R + 2]);
  store_super_pm(a, idx, S);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    a.rec[(size_t)(3 * r) * BN + idx] = A[r][R];
    a.rec[(size_t)(3 * r + 1) * BN + idx] = A[r][R + 1];
    a.rec[(size_t)(3 * r + 2) * BN + idx] = A[r][R + 2];
  }
#pragma unroll
  for (int j = 0; j < M; ++j) {
    a.pdx[(size_t)j * BN + idx] = nc[j].phi;
    a.pdx[(size_t)(M + j) * BN + idx] = dxb[j];
  }
}

// LDG coefficients of one element from its state at bottom time bt
// (corrector.py:100-170 per node: the P1 ldg_coefficients)
template <int M>
__device__ __forceinline__ void element_coefficients(const nh_member& m, const nh_pm_member& c,
                                                     const BottomTime& bt, const LdgConst& lk,
                                                     const Elem<M>& q, int e, NodeCoef (&nc)[M],
                                                     double (&dxb)[M]) {
  Chan ch[M];
  double eta[M], hx[M], ex[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const Bottom6 bb = bottom_all(m, bt, node_x<M>(m, c, e, j));
    ch[j] = Chan{bb.d, bb.d_x, bb.d_t, bb.d_tt, bb.d_xt, bb.d_xx};
    eta[j] = q.h[j] - bb.d;
    dxb[j] = bb.d_x;
  }
  ederiv_m<M>(m, c, q.h, hx);
  ederiv_m<M>(m, c, eta, ex);
#pragma unroll
  for (int j = 0; j < M; ++j) nc[j] = ldg_coefficients(q.h[j], q.q[j], q.w[j], hx[j], ex[j], ch[j], lk);
}

template <int M>
__global__ void __launch_bounds__(PTB) pm_condense(PmArgs a) {
  const int idx = blockIdx.x * PTB + threadIdx.x;
  if (idx >= a.B * a.N) return;
  const int N = a.N, b = idx / N, e = idx - b * N;
  const size_t o = (size_t)idx * M;
  if (!a.flags[idx]) {   // outside every range: a_e = 0, z_e = uncorrected hu at node 0
    store_super_pm(a, idx, super_gap(a.hu_out[o]));
    return;
  }
  const nh_member& m = a.members[b];
  const nh_pm_member& c = a.pm[b];
  const Elem<M> q = load_elem<M>(a.h_out, a.hu_out, a.hw_out, o);
  // coefficients at the predictor's time: t + dt in a step, the given state's
  // own time for apply_correction
  const BottomTime bt1 = bottom_time(m, a.given ? a.time[b] : a.time[b] + m.dt);
  NodeCoef nc[M];
  double dxb[M];
  element_coefficients<M>(m, c, bt1, make_ldg_const(m.dt, a.sch.g, a.sch.rho), q, e, nc, dxb);
  condense_block<M>(a, c, nc, dxb, b, e, idx, (e == N - 1) || !a.flags[idx + 1]);
}

// coefficient-level solve (ldg_solve / solve_on_ranges): the element blocks
// from given coefficient planes and flags; a gap element's z is the outer
// trace right of its left neighbour
template <int M>
__global__ void __launch_bounds__(PTB) pm_condense_coef(PmArgs a) {
  const int idx = blockIdx.x * PTB + threadIdx.x;
  if (idx >= a.B * a.N) return;
  const int N = a.N, b = idx / N, e = idx - b * N;
  const size_t BNM = (size_t)a.B * N * M, o = (size_t)idx * M;
  const bool f = given_flag(a, b, e);
  a.flags[idx] = f ? 1 : 0;
  if (!f) {
    store_super_pm(a, idx, super_gap(e > 0 ? a.outer_right[idx - 1] : 0.0));
    return;
  }
  NodeCoef nc[M];
  double dxb[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    nc[j].s11 = a.coef[o + j];
    nc[j].s12 = a.coef[BNM + o + j];
    nc[j].s22 = a.coef[2 * BNM + o + j];
    nc[j].f1 = a.coef[3 * BNM + o + j];
    nc[j].f2 = a.coef[4 * BNM + o + j];
    nc[j].phi = a.coef[5 * BNM + o + j];
    dxb[j] = a.coef[6 * BNM + o + j];
  }
  condense_block<M>(a, a.pm[b], nc, dxb, b, e, idx, (e == N - 1) || !given_flag(a, b, e + 1));
}

// coefficient planes of assemble_coefficients / phi_term at the state's time
template <int M>
__global__ void __launch_bounds__(PTB) pm_coef_kernel(PmArgs a, double* coef) {
  const int idx = blockIdx.x * PTB + threadIdx.x;
  if (idx >= a.B * a.N) return;
  const int N = a.N, b = idx / N, e = idx - b * N;
  const nh_member& m = a.members[b];
  const size_t BNM = (size_t)a.B * N * M, o = (size_t)idx * M;
  const Elem<M> q = load_elem<M>(a.h_in, a.hu_in, a.hw_in, o);
  NodeCoef nc[M];
  double dxb[M];
  element_coefficients<M>(m, a.pm[b], bottom_time(m, a.time[b]),
                          make_ldg_const(m.dt, a.sch.g, a.sch.rho), q, e, nc, dxb);
#pragma unroll
  for (int j = 0; j < M; ++j) {
    coef[o + j] = nc[j].s11; coef[BNM + o + j] = nc[j].s12; coef[2 * BNM + o + j] = nc[j].s22;
    coef[3 * BNM + o + j] = nc[j].f1; coef[4 * BNM + o + j] = nc[j].f2;
    coef[5 * BNM + o + j] = nc[j].phi; coef[6 * BNM + o + j] = dxb[j];
  }
}

// ------------------------------------------------- per-member chain, time
template <int M>
__global__ void __launch_bounds__(PTB) pm_chain(PmArgs a) {
  const int b = blockIdx.x * PTB + threadIdx.x;
  if (b >= a.B) return;
  const int N = a.N;
  const size_t BN = (size_t)a.B * N, base = (size_t)b * N;
  const nh_member& m = a.members[b];
  if (a.corr && !a.general) {
    double s = 0.0, t = 0.0;   // a_{-1} = 0: the left outer trace has zero weight
    for (int e = 0; e < N; ++e) {
      const size_t k = base + e;
      const Super S{a.sup[k], a.sup[BN + k], a.sup[2 * BN + k],
                    a.sup[3 * BN + k], a.sup[4 * BN + k], a.sup[5 * BN + k]};
      a.chain[k] = s; a.chain[BN + k] = t;
      double mm, nn;
      riccati_step(S, s, t, mm, nn);
      a.chain[2 * BN + k] = mm; a.chain[3 * BN + k] = nn;
    }
    // outer trace right of the member: the right ghost of hu (corrector.py:400-402)
    double z;
    if (a.outer_right) {
      z = a.outer_right[base + N - 1];
    } else {
      const double qn = a.hu_out[(base + N - 1) * M + M - 1];
      z = m.bc_right == NH_BC_WALL ? -qn : qn;
    }
    for (int e = N - 1; e >= 0; --e) {
      const size_t k = base + e;
      a.io[BN + k] = z;
      z = fma(a.chain[3 * BN + k], z, a.chain[2 * BN + k]);
      a.io[k] = fma(a.chain[BN + k], z, a.chain[k]);
    }
  }
  if (a.given) return;             // apply_correction: the time stays
  a.time[b] = a.time[b] + m.dt;   // t + dt per step (hydrostatic.py:206-209)
  a.status[b].steps_done += 1;
  if (a.hw_any) a.hw_any[b] = 0;
}

// ------------------------------------------------------ general LDG flux
// Any FluxCoefficients (corrector.py:40-47).  Outside the alternating family
// (c12 = -1/2, c22 = 0) an element couples to both neighbours through P and Q
// at both faces, so the two-scalar chain above does not apply.  This coverage
// path does what the reference does (corrector.py:173-234 pattern, :329-349
// values, :352 dgbsv): every range's node-interleaved band system is
// assembled in LAPACK general-band storage and solved by Gaussian
// elimination with partial pivoting (kl = ku = 2m - 1), one thread per
// member, its ranges in turn; the residual gate (corrector.py:359-366) is
// evaluated on the saved matrix.  Scratch per member (gen_doubles):
//   ab [3 band + 1][2 m N]  factorisation, column-major like dgbsv's work array
//   am [2 band + 1][2 m N]  the matrix as assembled (residual)
//   bx [2 m N]              right-hand side -> solution;  b0 [2 m N]  its copy
template <int M>
__host__ __device__ constexpr size_t gen_doubles(size_t N) {
  return (size_t)(3 * (2 * M - 1) + 1 + 2 * (2 * M - 1) + 1 + 2) * 2 * M * N;
}

template <int M>
__global__ void __launch_bounds__(PTB) pm_general_solve(PmArgs a) {
  const int b = blockIdx.x * PTB + threadIdx.x;
  if (b >= a.B) return;
  constexpr int BAND = 2 * M - 1, LDAB = 3 * BAND + 1, LDAM = 2 * BAND + 1;
  const int N = a.N;
  const size_t BN = (size_t)a.B * N, BNM = BN * M, base = (size_t)b * N;
  const nh_member& m = a.members[b];
  const nh_pm_member& c = a.pm[b];
  const double rho = a.sch.rho, inv_rho = 1.0 / rho;
  const double c11 = a.sch.c11, c12 = a.sch.c12, c22 = a.sch.c22;
  double* ab = a.gen + (size_t)b * gen_doubles<M>(N);
  double* am = ab + (size_t)LDAB * 2 * M * N;
  double* bx = am + (size_t)LDAM * 2 * M * N;
  double* b0 = bx + (size_t)2 * M * N;
  const LdgConst lk = make_ldg_const(m.dt, a.sch.g, rho);
  BottomTime bt1{0.0, 0.0, 0.0};
  if (!a.coef) bt1 = bottom_time(m, a.given ? a.time[b] : a.time[b] + m.dt);
  auto flagged = [&](int e) -> bool {
    return a.coef ? given_flag(a, b, e) : a.flags[base + e] != 0;
  };
  double r2 = 0.0, b2 = 0.0, x2 = 0.0, amax = 0.0;
  bool solved = false;
  int e = 0;
  while (e < N) {
    if (!flagged(e)) {
      if (a.p)
        for (int j = 0; j < M; ++j) a.p[(base + e) * M + j] = 0.0;
      ++e;
      continue;
    }
    const int e0 = e;
    while (e < N && flagged(e)) ++e;
    const int e1 = e - 1, n = e1 - e0 + 1, size = 2 * M * n;
    // outer hu traces of the range (corrector.py:388-403), read before the
    // range's own hu is replaced
    double outer_l, outer_r;
    if (a.coef) {
      outer_l = a.outer_left ? a.outer_left[base + e0] : 0.0;
      outer_r = a.outer_right[base + e1];
    } else {
      if (e0 > 0) {
        outer_l = a.hu_out[(base + e0 - 1) * M + M - 1];
      } else {
        const double q0 = a.hu_out[base * M];
        outer_l = m.bc_left == NH_BC_WALL ? -q0 : q0;
      }
      if (e1 < N - 1) {
        outer_r = a.hu_out[(base + e1 + 1) * M];
      } else {
        const double qn = a.hu_out[(base + N - 1) * M + M - 1];
        outer_r = m.bc_right == NH_BC_WALL ? -qn : qn;
      }
    }
    for (size_t k = 0; k < (size_t)LDAB * size; ++k) ab[k] = 0.0;
    for (size_t k = 0; k < (size_t)LDAM * size; ++k) am[k] = 0.0;
    auto add = [&](int r, int cc, double v) {
      ab[(size_t)cc * LDAB + (2 * BAND + r - cc)] += v;
      am[(size_t)cc * LDAM + (BAND + r - cc)] += v;
    };
    for (int k = 0; k < n; ++k) {
      const size_t idx = base + e0 + k, o = idx * M;
      NodeCoef nc[M];
      double dxb[M];
      if (a.coef) {
#pragma unroll
        for (int j = 0; j < M; ++j) {
          nc[j].s11 = a.coef[o + j];
          nc[j].s12 = a.coef[BNM + o + j];
          nc[j].s22 = a.coef[2 * BNM + o + j];
          nc[j].f1 = a.coef[3 * BNM + o + j];
          nc[j].f2 = a.coef[4 * BNM + o + j];
        }
      } else {
        const Elem<M> q = load_elem<M>(a.h_out, a.hu_out, a.hw_out, o);
        element_coefficients<M>(m, c, bt1, lk, q, e0 + k, nc, dxb);
#pragma unroll
        for (int j = 0; j < M; ++j) {
          a.pdx[(size_t)j * BN + idx] = nc[j].phi;
          a.pdx[(size_t)(M + j) * BN + idx] = dxb[j];
        }
        bool ok = true;
#pragma unroll
        for (int j = 0; j < M; ++j) ok = ok && !(nc[j].s12 <= 0.0);
        if (!ok) nh_report(a.status + b, a.step, NH_ERR_STRUCTURE, e0 + k);
      }
      const int r0 = 2 * M * k;
      double f1[M], f2[M];
#pragma unroll
      for (int j = 0; j < M; ++j) { f1[j] = nc[j].f1 * inv_rho; f2[j] = nc[j].f2; }
#pragma unroll
      for (int i = 0; i < M; ++i) {
#pragma unroll
        for (int j = 0; j < M; ++j) {
          const double Mij = c.mass[i * M + j], Kij = c.stiffness[i * M + j];
          add(r0 + 2 * i, r0 + 2 * j, -Kij + Mij * nc[j].s11);
          add(r0 + 2 * i, r0 + 2 * j + 1, Mij * (nc[j].s12 * inv_rho));
          add(r0 + 2 * i + 1, r0 + 2 * j + 1, -Kij + Mij * (-nc[j].s11));
          add(r0 + 2 * i + 1, r0 + 2 * j, Mij * (rho * nc[j].s22));
        }
        bx[r0 + 2 * i] = rowdot<M>(f1, c.mass, i);
        bx[r0 + 2 * i + 1] = rowdot<M>(f2, c.mass, i);
      }
      if (k + 1 < n) {   // interior face k | k + 1 (corrector.py:205-224)
        const int pL = r0 + 2 * (M - 1), qL = pL + 1, pR = r0 + 2 * M, qR = pR + 1;
        const int cols[4] = {pL, pR, qL, qR};
        const double sp[4] = {0.5 - c12, 0.5 + c12, c22, -c22};   // p* weights
        const double sq[4] = {c11, -c11, 0.5 + c12, 0.5 - c12};   // hu* weights
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (sp[t] != 0.0) { add(pL, cols[t], sp[t]); add(pR, cols[t], -sp[t]); }
          if (sq[t] != 0.0) { add(qL, cols[t], sq[t]); add(qR, cols[t], -sq[t]); }
        }
      }
    }
    // range ends: p* = 0; hu* keeps its interior-trace terms, the outer
    // traces go to the right-hand side (corrector.py:226-231, :346-347)
    add(1, 1, -(0.5 - c12));
    add(1, 0, c11);
    add(size - 1, size - 1, 0.5 + c12);
    add(size - 1, size - 2, c11);
    bx[1] += (0.5 + c12) * outer_l;
    bx[size - 1] -= (0.5 - c12) * outer_r;
    for (int k = 0; k < size; ++k) b0[k] = bx[k];
    // band LU with partial pivoting, the right-hand side carried along
    bool ok = true;
    int ju = 0;
    for (int j = 0; j < size; ++j) {
      double* col = ab + (size_t)j * LDAB + 2 * BAND;   // A(j + i, j) = col[i]
      const int km = min(BAND, size - 1 - j);
      int jp = 0;
      double best = fabs(col[0]);
      for (int i = 1; i <= km; ++i)
        if (fabs(col[i]) > best) { best = fabs(col[i]); jp = i; }
      if (!(best > 0.0) || !isfinite(best)) { ok = false; break; }
      ju = max(ju, min(j + BAND + jp, size - 1));
      if (jp) {
        for (int cc = j; cc <= ju; ++cc) {
          double* p0 = ab + (size_t)cc * LDAB + (2 * BAND + j - cc);
          const double tmp = p0[0]; p0[0] = p0[jp]; p0[jp] = tmp;
        }
        const double tb = bx[j]; bx[j] = bx[j + jp]; bx[j + jp] = tb;
      }
      const double rp = 1.0 / col[0];
      for (int i = 1; i <= km; ++i) {
        const double l = col[i] * rp;
        if (l == 0.0) continue;
        for (int cc = j + 1; cc <= ju; ++cc) {
          double* pc = ab + (size_t)cc * LDAB + (2 * BAND + j - cc);
          pc[i] = fma(-l, pc[0], pc[i]);
        }
        bx[j + i] = fma(-l, bx[j], bx[j + i]);
      }
    }
    if (ok) {
      for (int j = size - 1; j >= 0; --j) {
        double v = bx[j];
        const int cmax = min(size - 1, j + 2 * BAND);
        for (int cc = j + 1; cc <= cmax; ++cc)
          v = fma(-ab[(size_t)cc * LDAB + (2 * BAND + j - cc)], bx[cc], v);
        bx[j] = v / ab[(size_t)j * LDAB + 2 * BAND];
      }
    } else {
      nh_report(a.status + b, a.step, NH_ERR_SOLVE_PIVOT, e0);
    }
    // residual shares of this range (the reference's norms run over the
    // whole batched system of the step)
    bool fin = true;
    for (int r = 0; r < size; ++r) {
      double v = -b0[r];
      const int clo = max(0, r - BAND), chi = min(size - 1, r + BAND);
      for (int cc = clo; cc <= chi; ++cc) {
        const double av = am[(size_t)cc * LDAM + (BAND + r - cc)];
        v = fma(av, bx[cc], v);
        amax = fmax(amax, fabs(av));
      }
      r2 += v * v;
      b2 += b0[r] * b0[r];
      x2 += bx[r] * bx[r];
      fin = fin && isfinite(bx[r]);
    }
    solved = true;
    if (ok && !fin) nh_report(a.status + b, a.step, NH_ERR_SOLVE_NONFINITE, e0);
    for (int k = 0; k < n; ++k) {
      const size_t o = (base + e0 + k) * M;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        a.p[o + j] = rho * bx[2 * (M * k + j)];   // p = rho P (corrector.py:368)
        a.hu_out[o + j] = bx[2 * (M * k + j) + 1];
      }
    }
  }
  if (solved) {
    nh_status* st = a.status + b;
    const double scale = fmax(fmax(sqrt(b2), amax * sqrt(x2)), 1e-300);
    const double rel = sqrt(r2) / scale;
    if (rel > st->resid_max) st->resid_max = rel;
    if (a.sch.residual_tol > 0.0 && rel > a.sch.residual_tol)
      nh_report(st, a.step, NH_ERR_SOLVE_RESIDUAL, -1);
  }
}

// ----------------------------------------------------------- reconstruction
template <int M>
__global__ void __launch_bounds__(PTB) pm_reconstruct(PmArgs a) {
  const int idx = blockIdx.x * PTB + threadIdx.x;
  if (idx >= a.B * a.N) return;
  const size_t BN = (size_t)a.B * a.N, o = (size_t)idx * M;
  if (!a.flags[idx]) {
#pragma unroll
    for (int j = 0; j < M; ++j) a.p[o + j] = 0.0;
    return;
  }
  const double ai = a.io[idx], zi = a.io[BN + idx];
  bool fin = true;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    double x[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int r = 2 * j + u;
      x[u] = a.rec[(size_t)(3 * r) * BN + idx] + ai * a.rec[(size_t)(3 * r + 1) * BN + idx] +
             zi * a.rec[(size_t)(3 * r + 2) * BN + idx];
      fin = fin && isfinite(x[u]);
    }
    a.p[o + j] = a.sch.rho * x[0];   // p = rho P (corrector.py:368)
    a.hu_out[o + j] = x[1];
  }
  if (!fin) {
    const int b = idx / a.N;
    nh_report(a.status + b, a.step, NH_ERR_SOLVE_NONFINITE, idx - b * a.N);
  }
}

// --------------------------------------------------- vertical momentum update
template <int M>
__global__ void __launch_bounds__(PTB) pm_correct(PmArgs a) {
  const int idx = blockIdx.x * PTB + threadIdx.x;
  if (idx >= a.B * a.N) return;
  const int N = a.N, b = idx / N, e = idx - b * N;
  if (a.flags ? !a.flags[idx] : !given_flag(a, b, e)) return;
  const nh_member& m = a.members[b];
  const nh_pm_member& c = a.pm[b];
  const size_t BN = (size_t)a.B * N, BNM = BN * M, o = (size_t)idx * M;
  double hp[M], hx[M];
#pragma unroll
  for (int j = 0; j < M; ++j) hp[j] = a.h_out[o + j] * a.p[o + j];
  ederiv_m<M>(m, c, hp, hx);
  // central interface average of (h p), no lift at the domain ends
  // (corrector.py:427-438; p = 0 outside the ranges)
  if (e < N - 1) {
    const double hr = a.h_out[o + M] * a.p[o + M];
    const double avg = 0.5 * (hp[M - 1] + hr);
#pragma unroll
    for (int j = 0; j < M; ++j) hx[j] += (avg - hp[M - 1]) * c.lift_right[j];
  }
  if (e > 0) {
    const double hl = a.h_out[o - 1] * a.p[o - 1];
    const double avg = 0.5 * (hl + hp[0]);
#pragma unroll
    for (int j = 0; j < M; ++j) hx[j] -= (avg - hp[0]) * c.lift_left[j];
  }
  const double cdt = m.dt / a.sch.rho;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const double phi = a.coef ? a.coef[5 * BNM + o + j] : a.pdx[(size_t)j * BN + idx];
    const double dx = a.coef ? a.coef[6 * BNM + o + j] : a.pdx[(size_t)(M + j) * BN + idx];
    const double quad = 4.0 + dx * dx;
    const double bp = nh_div(6.0, quad) * a.p[o + j] + nh_div(dx, quad) * hx[j] + phi;
    a.hw_out[o + j] += cdt * bp;
  }
}

// h at the gauge nodes after the step (the correction leaves h unchanged)
template <int M>
__global__ void __launch_bounds__(PTB) pm_gauges(PmArgs a) {
  const size_t k = blockIdx.x * (size_t)PTB + threadIdx.x;
  if (k >= (size_t)a.B * a.n_gauges) return;
  const int b = (int)(k / a.n_gauges), gi = (int)(k % a.n_gauges);
  a.gauge_h[((size_t)a.step * a.B + b) * a.n_gauges + gi] =
      a.h_out[(size_t)b * a.N * M + a.gauge_nodes[gi]];
}

// ---------------------------------------------- single-function kernels
template <int M>
__global__ void __launch_bounds__(PTB) pm_rhs_kernel(PmArgs a, double* th, double* tq,
                                                     double* tw) {
  const int idx = blockIdx.x * PTB + threadIdx.x;
  if (idx >= a.B * a.N) return;
  const int N = a.N, b = idx / N, e = idx - b * N;
  const nh_member& m = a.members[b];
  const nh_pm_member& c = a.pm[b];
  const size_t o = (size_t)idx * M;
  const Elem<M> q = load_elem<M>(a.h_in, a.hu_in, a.hw_in, o);
  bool bad = false;
#pragma unroll
  for (int j = 0; j < M; ++j) bad |= !(q.h[j] > 0.0);
  if (bad) { nh_report(a.status + b, 0, NH_ERR_POSITIVITY_ENTRY, e); return; }
  const BottomTime bt = bottom_time(m, a.time[b]);
  double d[M], dxb[M];
#pragma unroll
  for (int j = 0; j < M; ++j) bottom_d_dx(m, bt, node_x<M>(m, c, e, j), d[j], dxb[j]);
  Side L, R;
  face_sides<M>(m, c, bt, a.h_in, a.hu_in, a.hw_in, b, e, N, q, d, L, R);
  double t[3][M];
  tendency<M>(m, c, a.sch.g, q, d, dxb, L, R, has_slope(m), t);
#pragma unroll
  for (int j = 0; j < M; ++j) { th[o + j] = t[0][j]; tq[o + j] = t[1][j]; tw[o + j] = t[2][j]; }
}

template <int M>
__global__ void __launch_bounds__(PTB) pm_crit_kernel(PmArgs a, int kind, double* out) {
  const int idx = blockIdx.x * PTB + threadIdx.x;
  if (idx >= a.B * a.N) return;
  const int N = a.N, b = idx / N, e = idx - b * N;
  const nh_member& m = a.members[b];
  const nh_pm_member& c = a.pm[b];
  const size_t o = (size_t)idx * M;
  const Elem<M> q = load_elem<M>(a.h_in, a.hu_in, a.hw_in, o);
  const BottomTime bt = bottom_time(m, a.time[b]);
  double d[M], v[M];
#pragma unroll
  for (int j = 0; j < M; ++j) d[j] = bottom_depth(m, bt, node_x<M>(m, c, e, j));
  criterion_m<M>(m, c, kind, q, d, v);
#pragma unroll
  for (int j = 0; j < M; ++j) out[o + j] = v[j];
}

int launch(void* k, int n, void** args, cudaStream_t s) {
  if (n <= 0) return 0;
  if (cudaLaunchKernel(k, dim3((unsigned)((n + PTB - 1) / PTB)), dim3(PTB), args, 0, s) !=
      cudaSuccess)
    return NH_E_CUDA;
  nh_count_launch();
  return 0;
}

template <int M>
int pm_advance_m(PmArgs a, int n_steps, double** A, double** Bb, const nh_outputs* out,
                 cudaStream_t s) {
  const int BN = a.B * a.N;
  void* args[1] = {&a};
  if (a.given) {   // the correction alone, in place on the given predictor state
    a.h_in = a.h_out = A[0]; a.hu_in = a.hu_out = A[1]; a.hw_in = a.hw_out = A[2];
    a.step = 0;
    int rc = launch((void*)pm_flags, BN, args, s);
    if (a.general) {
      if (!rc) rc = launch((void*)pm_general_solve<M>, a.B, args, s);
    } else {
      if (!rc) rc = launch((void*)pm_condense<M>, BN, args, s);
      if (!rc) rc = launch((void*)pm_chain<M>, a.B, args, s);
      if (!rc) rc = launch((void*)pm_reconstruct<M>, BN, args, s);
    }
    if (!rc) rc = launch((void*)pm_correct<M>, BN, args, s);
    if (!rc && out && out->p_nh &&
        cudaMemcpyAsync(out->p_nh, a.p, (size_t)BN * M * 8, cudaMemcpyDeviceToDevice, s) !=
            cudaSuccess)
      rc = NH_E_CUDA;
    return rc;
  }
  for (int k = 0; k < n_steps; ++k) {
    double** in = (k & 1) ? Bb : A;
    double** ou = (k & 1) ? A : Bb;
    a.h_in = in[0]; a.hu_in = in[1]; a.hw_in = in[2];
    a.h_out = ou[0]; a.hu_out = ou[1]; a.hw_out = ou[2];
    a.step = k;
    int rc = launch((void*)pm_stage<M, 1>, BN, args, s);
    if (!rc) rc = launch((void*)pm_stage<M, 2>, BN, args, s);
    if (!rc && a.corr) rc = launch((void*)pm_flags, BN, args, s);
    if (!rc && a.corr && a.general) rc = launch((void*)pm_general_solve<M>, a.B, args, s);
    if (!rc && a.corr && !a.general) rc = launch((void*)pm_condense<M>, BN, args, s);
    if (!rc) rc = launch((void*)pm_chain<M>, a.B, args, s);   // (general: time advance only)
    if (!rc && a.corr && !a.general) rc = launch((void*)pm_reconstruct<M>, BN, args, s);
    if (!rc && a.corr) rc = launch((void*)pm_correct<M>, BN, args, s);
    if (!rc && a.n_gauges > 0) rc = launch((void*)pm_gauges<M>, a.B * a.n_gauges, args, s);
    if (rc) return rc;
  }
  const size_t bytes = (size_t)BN * M * 8;
  if (n_steps & 1)
    for (int f = 0; f < 3; ++f)
      if (cudaMemcpyAsync(A[f], Bb[f], bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return NH_E_CUDA;
  if (out && out->p_nh && a.corr && n_steps > 0)
    if (cudaMemcpyAsync(out->p_nh, a.p, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return NH_E_CUDA;
  return 0;
}

size_t pm_doubles(int m, size_t BN) { return BN * (size_t)(18 * m + 12); }

// workspace partition (nh_pm_workspace_bytes); returns the ping-pong state
double* carve(PmArgs& a, void* workspace, int m, int B, int N, int*& hw_any) {
  const size_t BN = (size_t)B * N, BNM = BN * m;
  double* w = (double*)workspace;
  double* alt = w;            w += 3 * BNM;
  a.k1 = w;                   w += 3 * BNM;
  a.qs = w;                   w += 3 * BNM;
  a.sup = w;                  w += 6 * BN;
  a.rec = w;                  w += 6 * (size_t)m * BN;
  a.pdx = w;                  w += 2 * (size_t)m * BN;
  a.chain = w;                w += 4 * BN;
  a.io = w;                   w += 2 * BN;
  a.p = w;                    w += BNM;
  uint8_t* u8 = (uint8_t*)w;
  a.raw = u8;
  a.flags = u8 + BN;
  hw_any = (int*)(((uintptr_t)(u8 + 2 * BN) + 15) & ~(uintptr_t)15);
  return alt;
}

template <class F>
void* by_m(int m, F f2, F f3, F f4) { return m == 2 ? f2 : m == 3 ? f3 : f4; }

size_t gen_doubles_m(int m, size_t N) {
  return m == 2 ? gen_doubles<2>(N) : m == 3 ? gen_doubles<3>(N) : gen_doubles<4>(N);
}

bool alternating(double c12, double c22) { return c12 == -0.5 && c22 == 0.0; }

}  // namespace

extern "C" {

size_t nh_pm_workspace_bytes(int m, int n_members, int n_elements) {
  const size_t BN = (size_t)n_members * n_elements;
  return pm_doubles(m, BN) * 8 + 2 * BN + 4 * (size_t)n_members + 256;
}

int nh_pm_advance(const nh_member* members, const nh_pm_member* pm, int m, int B, int N,
                  double* h, double* hu, double* hw, double* time, int n_steps,
                  const nh_scheme* scheme, const nh_outputs* outputs, nh_status* status,
                  void* workspace, size_t workspace_bytes, void* stream) {
  if (!members || !pm || !h || !hu || !hw || !time || !scheme || !status || !workspace)
    return NH_E_ARG;
  if (m < 2 || m > NH_PM_MAX_NODES || B < 1 || N < 2 || n_steps < 0) return NH_E_ARG;
  if ((long long)B * N >= (1ll << 31)) return NH_E_UNSUPPORTED;
  if (workspace_bytes < nh_pm_workspace_bytes(m, B, N)) return NH_E_ARG;
  const nh_scheme& sc = *scheme;
  if (sc.mode < NH_MODE_HYDROSTATIC || sc.mode > NH_MODE_CORRECT_GIVEN) return NH_E_UNSUPPORTED;
  if (sc.mode == NH_MODE_CORRECT_GIVEN && (!outputs || !outputs->given_flags || n_steps != 1))
    return NH_E_ARG;
  if (n_steps == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t BN = (size_t)B * N, BNM = BN * m;
  PmArgs a;
  std::memset(&a, 0, sizeof a);
  int* hw_any = nullptr;
  double* alt = carve(a, workspace, m, B, N, hw_any);
  // a flux outside the alternating family: band solve per range (pm_general_solve)
  a.general = sc.mode != NH_MODE_HYDROSTATIC && !alternating(sc.c12, sc.c22);
  void* gen = nullptr;
  if (a.general) {
    if (cudaMallocAsync(&gen, gen_doubles_m(m, N) * (size_t)B * 8, s) != cudaSuccess) {
      cudaGetLastError();
      return NH_E_CUDA;
    }
    a.gen = (double*)gen;
  }
  const bool wcrit = sc.mode == NH_MODE_ADAPTIVE &&
                     (sc.criterion == NH_CRIT_W || sc.criterion == NH_CRIT_W_X);
  if (cudaMemsetAsync(a.raw, 0, BN, s) != cudaSuccess) return NH_E_CUDA;
  if (wcrit && cudaMemsetAsync(hw_any, 0, 4 * (size_t)B, s) != cudaSuccess) return NH_E_CUDA;
  a.members = members; a.pm = pm; a.time = time; a.status = status;
  a.hw_any = wcrit ? hw_any : nullptr;
  a.flag_bits = outputs ? outputs->flag_bits : nullptr;
  if (outputs && outputs->n_gauges > 0) {
    if (!outputs->gauge_nodes || !outputs->gauge_h) return NH_E_ARG;
    a.gauge_nodes = outputs->gauge_nodes; a.gauge_h = outputs->gauge_h;
    a.n_gauges = outputs->n_gauges;
  }
  a.corr = sc.mode != NH_MODE_HYDROSTATIC;
  a.given = sc.mode == NH_MODE_CORRECT_GIVEN ? outputs->given_flags : nullptr;
  a.sch = sc; a.B = B; a.N = N;
  double* A[3] = {h, hu, hw};
  double* Bb[3] = {alt, alt + BNM, alt + 2 * BNM};
  int rc;
  switch (m) {
    case 2: rc = pm_advance_m<2>(a, n_steps, A, Bb, outputs, s); break;
    case 3: rc = pm_advance_m<3>(a, n_steps, A, Bb, outputs, s); break;
    default: rc = pm_advance_m<4>(a, n_steps, A, Bb, outputs, s); break;
  }
  if (gen) cudaFreeAsync(gen, s);
  return rc;
}

int nh_pm_rhs(const nh_member* members, const nh_pm_member* pm, int m, int B, int N,
              const double* h, const double* hu, const double* hw, const double* time,
              double g, double* t_h, double* t_hu, double* t_hw, nh_status* status,
              void* stream) {
  if (!members || !pm || !h || !hu || !hw || !time || !t_h || !t_hu || !t_hw || !status)
    return NH_E_ARG;
  if (m < 2 || m > NH_PM_MAX_NODES || B < 1 || N < 2) return NH_E_ARG;
  PmArgs a;
  std::memset(&a, 0, sizeof a);
  a.members = members; a.pm = pm; a.h_in = h; a.hu_in = hu; a.hw_in = hw;
  a.time = const_cast<double*>(time); a.status = status; a.B = B; a.N = N; a.sch.g = g;
  void* args[4] = {&a, &t_h, &t_hu, &t_hw};
  void* k = m == 2 ? (void*)pm_rhs_kernel<2> : m == 3 ? (void*)pm_rhs_kernel<3>
                                                       : (void*)pm_rhs_kernel<4>;
  return launch(k, B * N, args, (cudaStream_t)stream);
}

int nh_pm_criterion(const nh_member* members, const nh_pm_member* pm, int m, int B, int N,
                    const double* h, const double* hu, const double* hw, const double* time,
                    int kind, double* values, void* stream) {
  if (!members || !pm || !h || !hu || !hw || !time || !values) return NH_E_ARG;
  if (m < 2 || m > NH_PM_MAX_NODES || B < 1 || N < 2 || kind < 0 || kind > NH_CRIT_W_X)
    return NH_E_ARG;
  PmArgs a;
  std::memset(&a, 0, sizeof a);
  a.members = members; a.pm = pm; a.h_in = h; a.hu_in = hu; a.hw_in = hw;
  a.time = const_cast<double*>(time); a.B = B; a.N = N;
  void* args[3] = {&a, &kind, &values};
  void* k = m == 2 ? (void*)pm_crit_kernel<2> : m == 3 ? (void*)pm_crit_kernel<3>
                                                        : (void*)pm_crit_kernel<4>;
  return launch(k, B * N, args, (cudaStream_t)stream);
}

int nh_pm_coefficients(const nh_member* members, const nh_pm_member* pm, int m, int B, int N,
                       const double* h, const double* hu, const double* hw, const double* time,
                       double g, double rho, double* coef, void* stream) {
  if (!members || !pm || !h || !hu || !hw || !time || !coef) return NH_E_ARG;
  if (m < 2 || m > NH_PM_MAX_NODES || B < 1 || N < 2) return NH_E_ARG;
  PmArgs a;
  std::memset(&a, 0, sizeof a);
  a.members = members; a.pm = pm; a.h_in = h; a.hu_in = hu; a.hw_in = hw;
  a.time = const_cast<double*>(time); a.B = B; a.N = N; a.sch.g = g; a.sch.rho = rho;
  void* args[2] = {&a, &coef};
  return launch(by_m(m, (void*)pm_coef_kernel<2>, (void*)pm_coef_kernel<3>,
                     (void*)pm_coef_kernel<4>), B * N, args, (cudaStream_t)stream);
}

int nh_pm_ldg_solve(const nh_member* members, const nh_pm_member* pm, int m, int B, int N,
                    const double* coef, const uint32_t* flags, const double* outer_left,
                    const double* outer_right, double rho, double c11, double c12, double c22,
                    double residual_tol, double* p, double* hu, nh_status* status,
                    void* workspace, size_t workspace_bytes, void* stream) {
  if (!members || !pm || !coef || !flags || !outer_right || !p || !hu || !status || !workspace)
    return NH_E_ARG;
  if (m < 2 || m > NH_PM_MAX_NODES || B < 1 || N < 2) return NH_E_ARG;
  if (workspace_bytes < nh_pm_workspace_bytes(m, B, N)) return NH_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  if (!alternating(c12, c22)) {   // general flux: one band solve per range
    if (!outer_left) return NH_E_ARG;
    PmArgs g;
    std::memset(&g, 0, sizeof g);
    g.members = members; g.pm = pm; g.status = status; g.B = B; g.N = N;
    g.coef = coef; g.given = flags; g.outer_left = outer_left; g.outer_right = outer_right;
    g.corr = 1; g.general = 1;
    g.sch.rho = rho; g.sch.c11 = c11; g.sch.c12 = c12; g.sch.c22 = c22;
    g.sch.residual_tol = residual_tol;
    g.hu_out = hu; g.p = p;
    void* gen = nullptr;
    if (cudaMallocAsync(&gen, gen_doubles_m(m, N) * (size_t)B * 8, s) != cudaSuccess) {
      cudaGetLastError();
      return NH_E_CUDA;
    }
    g.gen = (double*)gen;
    void* gargs[1] = {&g};
    const int rc = launch(by_m(m, (void*)pm_general_solve<2>, (void*)pm_general_solve<3>,
                               (void*)pm_general_solve<4>), B, gargs, s);
    cudaFreeAsync(gen, s);
    return rc;
  }
  PmArgs a;
  std::memset(&a, 0, sizeof a);
  int* hw_any = nullptr;
  carve(a, workspace, m, B, N, hw_any);
  a.members = members; a.pm = pm; a.status = status; a.B = B; a.N = N;
  a.coef = coef; a.given = flags; a.outer_right = outer_right; a.corr = 1;
  a.sch.rho = rho; a.sch.c11 = c11; a.sch.c12 = c12; a.sch.c22 = c22;
  a.hu_out = hu;
  a.p = p;
  a.time = nullptr;
  void* args[1] = {&a};
  int rc = launch(by_m(m, (void*)pm_condense_coef<2>, (void*)pm_condense_coef<3>,
                       (void*)pm_condense_coef<4>), B * N, args, s);
  if (!rc) rc = launch(by_m(m, (void*)pm_chain<2>, (void*)pm_chain<3>, (void*)pm_chain<4>), B,
                       args, s);
  if (!rc) rc = launch(by_m(m, (void*)pm_reconstruct<2>, (void*)pm_reconstruct<3>,
                            (void*)pm_reconstruct<4>), B * N, args, s);
  return rc;
}

int nh_pm_correct_momentum(const nh_member* members, const nh_pm_member* pm, int m, int B, int N,
                           const double* h, const double* p, const double* coef,
                           const uint32_t* flags, double rho, const double* hw, double* hw_out,
                           void* stream) {
  if (!members || !pm || !h || !p || !coef || !flags || !hw || !hw_out) return NH_E_ARG;
  if (m < 2 || m > NH_PM_MAX_NODES || B < 1 || N < 2) return NH_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = (size_t)B * N * m * 8;
  if (hw_out != hw && cudaMemcpyAsync(hw_out, hw, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return NH_E_CUDA;
  PmArgs a;
  std::memset(&a, 0, sizeof a);
  a.members = members; a.pm = pm; a.B = B; a.N = N;
  a.h_out = const_cast<double*>(h); a.p = const_cast<double*>(p); a.hw_out = hw_out;
  a.coef = coef; a.given = flags; a.flags = nullptr; a.sch.rho = rho;
  void* args[1] = {&a};
  return launch(by_m(m, (void*)pm_correct<2>, (void*)pm_correct<3>, (void*)pm_correct<4>), B * N,
                args, s);
}

}  // extern "C"
