// Element-level physics of one NH-SWE time step, in registers.
//
//  * face_flux / element_tendency : hydrostatic.py:88-184 (rhs_operator),
//    hydrostatic-reconstruction Rusanov flux, volume + lift + g h d_x terms.
//  * ldg_coefficients             : corrector.py:100-170 (phi_term,
//    assemble_coefficients), general (sloped) formulas -- the reference's
//    flat-bottom branches are bit-identical to them.
//  * local_condense               : one element's 4x4 LDG block
//    (corrector.py:173-234 sparsity, :329-349 values) eliminated to the
//    "super-element" form
//        a_e = ga + aa * a_{e-1} + ba * z_{e+1}
//        z_e = gz + az * a_{e-1} + bz * z_{e+1}
//    with a_e = P(node 1), z_e = Q(node 0) - c11 * P(node 0), P = p / rho,
//    Q = hu.  With the reference's alternating flux (c12 = -1/2, c22 = 0)
//    an element talks to its left neighbour only through a_{e-1} and to its
//    right neighbour only through z_{e+1}, so the node-interleaved banded
//    system that LAPACK dgbsv factorises (corrector.py:352) is solved exactly
//    by a chain of these 2-scalar couplings.
//  * merge                        : eliminating the shared unknowns of two
//    adjacent super-elements gives a super-element of the same form; the
//    parallel solve is a tree of merges (thread chunk -> warp -> CTA ->
//    cluster) followed by the matching back-substitution.
#pragma once
#include "nh_common.cuh"

struct Face {
  double F1, F2L, F2R, F3;   // F2L = F2 + corr_left (used by the element left of the face)
};

// Interface state on one side: conserved values, u = hu/h, 1/h, depth.
struct Side {
  double h, hu, hw, u, rh, d;
};

NH_DEV Side make_side(double h, double hu, double hw, double d) {
  Side s;
  s.h = h; s.hu = hu; s.hw = hw; s.d = d;
#if NH_STRICT
  s.rh = 0.0;
#else
  s.rh = nh_rcp(h);
#endif
  s.u = RDIVP(hu, h);
  return s;
}

// Both nodes of an element with the whole warp converged: the two divisions
// take their fast path and one warp vote decides whether to redo them with
// the complete IEEE sequence (bit-identical to make_side either way).
NH_DEV void make_sides_warp(double h0, double hu0, double hw0, double d0, double h1, double hu1,
                            double hw1, double d1, Side& n0, Side& n1) {
#if NH_STRICT
  n0.h = h0; n0.hu = hu0; n0.hw = hw0; n0.d = d0; n0.rh = 0.0;
  n1.h = h1; n1.hu = hu1; n1.hw = hw1; n1.d = d1; n1.rh = 0.0;
  bool bad = false;
  n0.u = nh_div_pos_fp(hu0, h0, bad);
  n1.u = nh_div_pos_fp(hu1, h1, bad);
  NH_WARP_FIX(bad, (n0.u = RDIVP(hu0, h0), n1.u = RDIVP(hu1, h1)));
#else
  n0 = make_side(h0, hu0, hw0, d0);
  n1 = make_side(h1, hu1, hw1, d1);
#endif
}

NH_DEV Side ghost_side(const Side& in, int bc) {
  Side s = in;
  if (bc == NH_BC_WALL) { s.hu = -in.hu; s.u = -in.u; }
  return s;
}

// hydrostatic.py:131-160 with the general (reconstructed) formulas.  They are
// bit-identical to the plain branch when dL == dR: hLs == hL,
// corr == 0, (hLs/hL) == 1.  LEVEL = true is that plain branch, used for
// flat-bottom members where dL == dR at every face: the reconstruction terms
// are exact zeros there (up to the sign of a zero flux, which no later
// operation can observe), so they are skipped.
// WARP = true: every lane of the warp calls this together (one vote per
// group of divisions / square roots instead of a branch per operation).
template <bool LEVEL = false, bool WARP = false>
NH_DEV Face face_flux(const Side& L, const Side& R, double g, double& speed) {
  const double hg = 0.5 * g;
  double hLs, hRs, cL = 0.0, cR = 0.0;
  if (LEVEL) {
    hLs = L.h; hRs = R.h;
  } else {
    double dm = nh_min(L.d, R.d);
    hLs = nh_max(RSUB(L.h, RSUB(L.d, dm)), 0.0);
    hRs = nh_max(RSUB(R.h, RSUB(R.d, dm)), 0.0);
    cL = RMUL(hg, RSUB(RMUL(L.h, L.h), RMUL(hLs, hLs)));
    cR = RMUL(hg, RSUB(RMUL(R.h, R.h), RMUL(hRs, hRs)));
  }
  double sL, sR;
#if NH_STRICT
  if (WARP) {
    bool bad = false;
    sL = nh_dsqrt_rn_fp(RMUL(g, hLs), bad);
    sR = nh_dsqrt_rn_fp(RMUL(g, hRs), bad);
    NH_WARP_FIX(bad, (sL = RSQRT(RMUL(g, hLs)), sR = RSQRT(RMUL(g, hRs))));
  } else
#endif
  {
    sL = RSQRT(RMUL(g, hLs));
    sR = RSQRT(RMUL(g, hRs));
  }
  double aL = RADD(fabs(L.u), sL);
  double aR = RADD(fabs(R.u), sR);
  speed = nh_max(aL, aR);
  double lam = RMUL(0.5, speed);
  double qL = RMUL(hLs, L.u), qR = RMUL(hRs, R.u);
  Face f;
  f.F1 = RSUB(RMUL(0.5, RADD(qL, qR)), RMUL(lam, RSUB(hRs, hLs)));
  double s2 = RADD(RADD(RMUL(qL, L.u), RMUL(qR, R.u)), RMUL(hg, RADD(RMUL(hLs, hLs), RMUL(hRs, hRs))));
  double F2 = RSUB(RMUL(0.5, s2), RMUL(lam, RSUB(qR, qL)));
  double wL, wR;
  if (LEVEL) {
    wL = L.hw; wR = R.hw;
  } else {
#if NH_STRICT
    // (hLs / hL) hwL is exactly hwL when hLs == hL (IEEE x / x == 1), and
    // when hwL is a zero (the quotient is >= 0, so the product is that zero:
    // hw stays identically 0 where no correction has ever acted)
    if (WARP) {
      wL = L.hw; wR = R.hw;
      const bool nL = hLs != L.h && L.hw != 0.0, nR = hRs != R.h && R.hw != 0.0;
      if (__any_sync(0xffffffffu, nL || nR)) {
        bool bad = false;
        double rL = nh_div_pos_fp(hLs, L.h, bad), rR = nh_div_pos_fp(hRs, R.h, bad);
        NH_WARP_FIX(bad, (rL = RDIVP(hLs, L.h), rR = RDIVP(hRs, R.h)));
        if (nL) wL = RMUL(rL, L.hw);
        if (nR) wR = RMUL(rR, R.hw);
      }
    } else {
      wL = (hLs == L.h) ? L.hw : RMUL(RDIVP(hLs, L.h), L.hw);
      wR = (hRs == R.h) ? R.hw : RMUL(RDIVP(hRs, R.h), R.hw);
    }
#else
    wL = (hLs == L.h) ? L.hw : (hLs * L.rh) * L.hw;
    wR = (hRs == R.h) ? R.hw : (hRs * R.rh) * R.hw;
#endif
  }
  f.F3 = RSUB(RMUL(0.5, RADD(RMUL(wL, L.u), RMUL(wR, R.u))), RMUL(lam, RSUB(wR, wL)));
  f.F2L = LEVEL ? F2 : RADD(F2, cL);
  f.F2R = LEVEL ? F2 : RADD(F2, cR);
  return f;
}

// Tendency of one element (hydrostatic.py:162-183).  n0/n1 = own nodes,
// fl = face at its left, fr = face at its right, dx0/dx1 = bottom slope
// (LEVEL: identically zero, the g h d_x source is skipped).
// The volume products keep numpy's dgemm rounding: fma(v1, W1, v0*W0).
template <bool LEVEL = false>
NH_DEV void element_tendency(const nh_member& m, double g, const Side& n0, const Side& n1,
                             const Face& fl, const Face& fr, double dx0, double dx1,
                             double t[6]) {
  const double hg = 0.5 * g;
  double f20 = RADD(RMUL(n0.hu, n0.u), RMUL(RMUL(hg, n0.h), n0.h));
  double f21 = RADD(RMUL(n1.hu, n1.u), RMUL(RMUL(hg, n1.h), n1.h));
  double f30 = RMUL(n0.u, n0.hw), f31 = RMUL(n1.u, n1.hw);
  const double* W = m.weak_div;
  const double* lr = m.lift_right;
  const double* ll = m.lift_left;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    double v1 = fma(n1.hu, W[2 * i + 1], RMUL(n0.hu, W[2 * i]));
    v1 = RSUB(v1, RMUL(fr.F1, lr[i]));
    t[0 + i] = RADD(v1, RMUL(fl.F1, ll[i]));
    double v2 = fma(f21, W[2 * i + 1], RMUL(f20, W[2 * i]));
    v2 = RSUB(v2, RMUL(fr.F2L, lr[i]));
    v2 = RADD(v2, RMUL(fl.F2R, ll[i]));
    t[2 + i] = LEVEL ? v2 : RADD(v2, RMUL(RMUL(g, i ? n1.h : n0.h), i ? dx1 : dx0));
    double v3 = fma(f31, W[2 * i + 1], RMUL(f30, W[2 * i]));
    v3 = RSUB(v3, RMUL(fr.F3, lr[i]));
    t[4 + i] = RADD(v3, RMUL(fl.F3, ll[i]));
  }
}

// ---------------------------------------------------------------- LDG part

struct Chan {     // bottom channels at one node
  double d, d_x, d_t, d_tt, d_xt, d_xx;
};

struct NodeCoef {
  double s11, s12, s22, f1, f2, phi;
};

// Scheme constants of the LDG system, computed once per member.
struct LdgConst {
  double rho, inv_rho, rho_dt, s12c, s22c, f2c, g, cdt;
};

NH_DEV LdgConst make_ldg_const(double dt, double g, double rho) {
  LdgConst k;
  k.rho = rho;
  k.inv_rho = 1.0 / rho;
  k.rho_dt = rho / dt;
  k.s12c = 0.25 * rho / dt;
  k.s22c = 3.0 * dt / rho;
  k.f2c = 0.5 * dt / rho;
  k.g = g;
  k.cdt = dt / rho;
  return k;
}

// corrector.py:100-170 at one node; h_x / eta_x are the element derivatives.
NH_DEV NodeCoef ldg_coefficients(double h, double hu, double hw, double h_x, double eta_x,
                                 const Chan& b, const LdgConst& k) {
  NodeCoef c;
  double ih = nh_rcp(h);
  double u = hu * ih;
  double acc = -b.d_tt;
  acc = acc + (-2.0 * u * b.d_xt - u * u * b.d_xx);
  acc = acc + (k.g * b.d_x) * eta_x;
  double quad = 4.0 + b.d_x * b.d_x;
  c.phi = nh_div(k.rho * h, quad) * acc;
  c.s22 = k.s22c * ih;
  c.s11 = (h_x - 1.5 * b.d_x) * ih;
  c.s12 = k.s12c * quad * ih;
  c.f1 = (0.25 * quad * ih) * (c.phi * b.d_x + k.rho_dt * hu);
  double f2 = (-2.0 * hw - (0.5 * b.d_x) * hu) * ih;
  f2 = f2 - k.f2c * quad * c.phi * ih;
  c.f2 = f2 - 2.0 * b.d_t;
  return c;
}

// Super-element coefficients (ga, aa, ba, gz, az, bz).
struct Super {
  double ga, aa, ba, gz, az, bz;
};

NH_DEV Super super_identity() { return Super{0.0, 1.0, 0.0, 0.0, 0.0, 1.0}; }
NH_DEV bool is_identity(const Super& s) {
  return s.ga == 0.0 && s.aa == 1.0 && s.ba == 0.0 && s.gz == 0.0 && s.az == 0.0 && s.bz == 1.0;
}

// An element outside every range: a_e = 0 (next element starts a range with
// P* = 0) and z_e = its uncorrected hu at node 0 (the outer trace seen by a
// range ending just before it, corrector.py:398-399).
NH_DEV Super super_gap(double hu0) { return Super{0.0, 0.0, 0.0, hu0, 0.0, 0.0}; }

// Gauss-Jordan (no pivoting) on the 4x4 element block with three right-hand
// sides [r | l | v]; l = (1, c11, 0, 0) carries a_{e-1}, v = (0, 0, 0, -1)
// carries z_{e+1}.  Unknown order (P0, Q0, P1, Q1).  Returns false on a zero
// or non-finite pivot.  rec = (u0, w0, v0, u3, w3, v3) for reconstruction.
NH_DEV bool local_condense(const nh_member& m, const NodeCoef& c0, const NodeCoef& c1,
                           double rho, double inv_rho, double c11, bool range_end, Super& S,
                           double rec[6]) {
  const double* M = m.mass;
  const double* K = m.stiffness;
  double A[4][7];
  const NodeCoef* cj[2] = {&c0, &c1};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const NodeCoef& q = *cj[j];
      double Mij = M[2 * i + j], Kij = K[2 * i + j];
      A[2 * i][2 * j] = -Kij + Mij * q.s11;
      A[2 * i][2 * j + 1] = Mij * (q.s12 * inv_rho);
      A[2 * i + 1][2 * j + 1] = -Kij + Mij * (-q.s11);
      A[2 * i + 1][2 * j] = Mij * (rho * q.s22);
    }
    A[2 * i][4] = fma(M[2 * i + 1], c1.f1 * inv_rho, M[2 * i] * (c0.f1 * inv_rho));
    A[2 * i + 1][4] = fma(M[2 * i + 1], c1.f2, M[2 * i] * c0.f2);
  }
  // faces (c12 = -1/2, c22 = 0): left  -Q* = -(Q0 + c11 (a - P0)),  -P* = -a
  //                              right +P* = P1 (interior only), +Q* = z + c11 P1
  A[1][1] -= 1.0;
  A[1][0] += c11;
  if (!range_end) A[2][2] += 1.0;
  A[3][2] += c11;
  A[0][5] = 1.0; A[1][5] = c11; A[2][5] = 0.0; A[3][5] = 0.0;
  A[0][6] = 0.0; A[1][6] = 0.0; A[2][6] = 0.0; A[3][6] = -1.0;
  bool ok = true;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double piv = A[k][k];
    ok = ok && (piv != 0.0) && isfinite(piv);
    double r = nh_rcp(piv);
#pragma unroll
    for (int c = k + 1; c < 7; ++c) A[k][c] *= r;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i == k) continue;
      double f = A[i][k];
#pragma unroll
      for (int c = k + 1; c < 7; ++c) A[i][c] = fma(-f, A[k][c], A[i][c]);
    }
  }
  S.ga = A[2][4]; S.aa = A[2][5]; S.ba = A[2][6];
  S.gz = fma(-c11, A[0][4], A[1][4]);
  S.az = fma(-c11, A[0][5], A[1][5]);
  S.bz = fma(-c11, A[0][6], A[1][6]);
  rec[0] = A[0][4]; rec[1] = A[0][5]; rec[2] = A[0][6];
  rec[3] = A[3][4]; rec[4] = A[3][5]; rec[5] = A[3][6];
  return ok;
}

// Residual gate of the elliptic solve (corrector.py:355-366).  The reference
// evaluates rel = ||A x - b|| / max(||b||, max|A| ||x||, 1e-300) over the
// step's whole batched band system and raises EllipticSolveError above
// residual_tol.  Every row of that system belongs to one flagged element, so
// the norms are sums (max) over elements: this is one element's share, at
// the solved unknowns x = (P0, Q0, P1, Q1) (P = p / rho) with the coupling
// values a_prev = P(e-1, node 1) (0 at a range start) and z_next = Q(e+1,
// node 0) - c11 P(e+1, node 0) (the outer hu trace at a range end).  The
// element block is built exactly as local_condense builds it -- the same
// entries as the reference's assembly (_block_template / _solve_batched).
struct ResidAcc {
  double r2, b2, x2, amax;
};

NH_DEV void ldg_residual(const nh_member& m, const NodeCoef& c0, const NodeCoef& c1, double rho,
                         double inv_rho, double c11, bool range_start, bool range_end,
                         double a_prev, double z_next, double P0, double Q0, double P1,
                         double Q1, ResidAcc& acc) {
  const double* M = m.mass;
  const double* K = m.stiffness;
  double A[4][4], r[4];
  const NodeCoef* cj[2] = {&c0, &c1};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const NodeCoef& q = *cj[j];
      double Mij = M[2 * i + j], Kij = K[2 * i + j];
      A[2 * i][2 * j] = -Kij + Mij * q.s11;
      A[2 * i][2 * j + 1] = Mij * (q.s12 * inv_rho);
      A[2 * i + 1][2 * j + 1] = -Kij + Mij * (-q.s11);
      A[2 * i + 1][2 * j] = Mij * (rho * q.s22);
    }
    r[2 * i] = fma(M[2 * i + 1], c1.f1 * inv_rho, M[2 * i] * (c0.f1 * inv_rho));
    r[2 * i + 1] = fma(M[2 * i + 1], c1.f2, M[2 * i] * c0.f2);
  }
  A[1][1] -= 1.0;
  A[1][0] += c11;
  if (!range_end) A[2][2] += 1.0;
  A[3][2] += c11;
  const double x[4] = {P0, Q0, P1, Q1};
  double res[4], amax = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double v = -r[i];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      v = fma(A[i][j], x[j], v);
      amax = nh_max(amax, fabs(A[i][j]));
    }
    res[i] = v;
  }
  // couplings: rows P0 / Q0 to P(e-1, 1) (-1, -c11), row Q1 to the right
  // neighbour (+1 on Q(e+1, 0), -c11 on P(e+1, 0)); a range end's z_next is
  // the outer trace, which the reference carries in b
  res[0] -= a_prev;
  res[1] -= c11 * a_prev;
  res[3] += z_next;
  double b3 = range_end ? r[3] - z_next : r[3];
  if (!range_start || !range_end) amax = nh_max(amax, nh_max(1.0, fabs(c11)));
  acc.r2 += res[0] * res[0] + res[1] * res[1] + res[2] * res[2] + res[3] * res[3];
  acc.b2 += r[0] * r[0] + r[1] * r[1] + r[2] * r[2] + b3 * b3;
  acc.x2 += P0 * P0 + Q0 * Q0 + P1 * P1 + Q1 * Q1;
  acc.amax = nh_max(acc.amax, amax);
}

// A warp's residual shares into the member's running sums (all 32 lanes
// converged; lanes without a flagged element pass zeros).
NH_DEV void resid_flush_warp(nh_status* st, ResidAcc a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a.r2 += __shfl_xor_sync(0xffffffffu, a.r2, o);
    a.b2 += __shfl_xor_sync(0xffffffffu, a.b2, o);
    a.x2 += __shfl_xor_sync(0xffffffffu, a.x2, o);
    a.amax = nh_max(a.amax, __shfl_xor_sync(0xffffffffu, a.amax, o));
  }
  if ((threadIdx.x & 31) == 0 && (a.amax > 0.0 || a.x2 > 0.0 || a.b2 > 0.0 || a.r2 != 0.0)) {
    atomicAdd(&st->resid_acc[0], a.r2);
    atomicAdd(&st->resid_acc[1], a.b2);
    atomicAdd(&st->resid_acc[2], a.x2);
    atomicMax(reinterpret_cast<unsigned long long*>(&st->resid_acc[3]),
              (unsigned long long)__double_as_longlong(a.amax));
  }
}

// The gate of one solve (after every element's share is in): rel as the
// reference computes it, the running max in resid_max, an error above tol
// (tol <= 0: record only), and the sums cleared for the next solve.  One
// thread per member.
NH_DEV void resid_check(nh_status* st, int step, double tol) {
  double* acc = st->resid_acc;
  // L2 reads: the sums were built by atomics of other CTAs
  const double r2 = __ldcg(acc), b2 = __ldcg(acc + 1), x2 = __ldcg(acc + 2), am = __ldcg(acc + 3);
  if (r2 == 0.0 && b2 == 0.0 && x2 == 0.0 && am == 0.0) return;   // no solve
  const double scale = fmax(fmax(sqrt(b2), am * sqrt(x2)), 1e-300);
  const double rel = sqrt(r2) / scale;
  if (rel > st->resid_max) st->resid_max = rel;
  if (tol > 0.0 && rel > tol) nh_report(st, step, NH_ERR_SOLVE_RESIDUAL, -1);
  acc[0] = acc[1] = acc[2] = acc[3] = 0.0;
}

// s12 > 0 at a flagged node (the reference asserts it when the coefficients
// are built, corrector.py:70-74; NaN passes, as with numpy's `s12 <= 0`).
NH_DEV bool ldg_structure_ok(const NodeCoef& c0, const NodeCoef& c1) {
  return !(c0.s12 <= 0.0) && !(c1.s12 <= 0.0);
}

// Merge two adjacent super-elements L (left) and R (right).  Also returns the
// back-substitution rows: A_L = AL . (1, a_in, z_in), Z_R = ZR . (1, a_in, z_in).
NH_DEV Super merge(const Super& L, const Super& R, double AL[3], double ZR[3]) {
  double iD = nh_rcp(1.0 - L.ba * R.az);
  AL[0] = fma(L.ba, R.gz, L.ga) * iD;
  AL[1] = L.aa * iD;
  AL[2] = L.ba * R.bz * iD;
  ZR[0] = fma(R.az, AL[0], R.gz);
  ZR[1] = R.az * AL[1];
  ZR[2] = fma(R.az, AL[2], R.bz);
  Super o;
  o.ga = fma(R.aa, AL[0], R.ga);
  o.aa = R.aa * AL[1];
  o.ba = fma(R.aa, AL[2], R.ba);
  o.gz = fma(L.bz, ZR[0], L.gz);
  o.az = fma(L.bz, ZR[1], L.az);
  o.bz = L.bz * ZR[2];
  return o;
}

NH_DEV Super merge2(const Super& L, const Super& R) {
  double AL[3], ZR[3];
  return merge(L, R, AL, ZR);
}

// Forward Riccati sweep state: the incoming a_{e-1} = s + t * z_e.
// For one super-element with incoming (s, t): z_e = m + n z_{e+1}, and the
// outgoing (s', t') for the next one.  Returns the elimination factors.
NH_DEV void riccati_step(const Super& S, double& s, double& t, double& mm, double& nn) {
  double rden = nh_rcp(1.0 - S.az * t);
  mm = fma(S.az, s, S.gz) * rden;
  nn = S.bz * rden;
  double at = S.aa * t;
  double s2 = fma(at, mm, fma(S.aa, s, S.ga));
  double t2 = fma(at, nn, S.ba);
  s = s2; t = t2;
}
