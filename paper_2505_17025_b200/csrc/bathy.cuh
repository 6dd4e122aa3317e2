// Device bottom models: d(x, t) and the five derivative channels.
//
// Restates reference bathymetry.py:66-184 (FlatBottom, HammackPlate,
// SlideMotion/WhittakerSlide) and the two harness models of SURVEY.md
// Appendix C (smoothed box uplift, Gaussian mound on a slope) whose numpy
// twins live in oracle/nhswe_oracle.py.  Nothing is stored in HBM: channels
// are evaluated in registers at the inset sample nodes (grid.py:84-90).
//
// Every function is templated on the model kind so the step kernel runs a
// straight-line path per member (KIND = -1 dispatches at run time).  Time
// factors are hoisted into BottomTime once per instant.  The two harness
// models are defined (here and in the oracle) with a cut-off -- S = 0 for
// |y| >= 23 (tanh box), G = 0 for |r| >= 10 (Gaussian) -- and with the
// deterministic exp / log1p below, so device and host evaluate them to the
// same bits.
#pragma once
#include "nh_common.cuh"

struct Bottom6 {
  double d, d_x, d_t, d_tt, d_xt, d_xx;
};

struct BottomTime {
  double a, b, c;   // model-specific time factors
};

// host-packed parameter layout (paper_2505_17025_b200/bathymetry.py pack()):
//  FLAT           h0
//  PLATE          h0, zeta0, b, alpha
//  QUARTIC_SLIDE  h0, Hs, Ls, x_start, a0, u_t, t1, t2, t3, 2/Ls
//  SMOOTH_BOX     h0, zeta0, b, alpha, w, 1/w, 1/w^2
//  SLOPE_SLIDE    d_top, tan, d_max, A, sigma, x0, u_t, t0, d_stop, x_stop, t_stop, 1/sigma
//                 (r = (x - xc) * (1/sigma): the harness model's definition, oracle SlopeSlide)

#define NH_BOX_YCUT 23.0
#define NH_SLIDE_RCUT 10.0

// Deterministic exp / log1p of the harness bottom models (oracle det_exp /
// det_log1p): IEEE +,-,* only -- Cody-Waite reduction and Horner polynomials,
// explicit round-to-nearest intrinsics (never contracted), same constants and
// order as the numpy definition, so host and device round identically.
// the Horner coefficients as constant-bank operands of the DADDs (as
// immediates every coefficient costs two uniform-register moves)
static __constant__ double NH_EXP_COEF[14] = {
    1.6059043836821613e-10, 2.08767569878681e-09, 2.505210838544172e-08,
    2.755731922398589e-07,  2.7557319223985893e-06, 2.48015873015873e-05,
    0.0001984126984126984,  0.001388888888888889, 0.008333333333333333,
    0.041666666666666664,   0.16666666666666666, 0.5, 1.0, 1.0};

__device__ __forceinline__ double nh_det_exp(double x) {
  const double k = rint(__dmul_rn(x, 1.4426950408889634));
  const double r = __dsub_rn(__dsub_rn(x, __dmul_rn(k, 0.6931471803691238)),
                             __dmul_rn(k, 1.9082149292705877e-10));
  const double* c = NH_EXP_COEF;
  double p = c[0];
#pragma unroll
  for (int n = 1; n < 14; ++n) p = __dadd_rn(__dmul_rn(p, r), c[n]);
  // p * 2^k: one multiplication by an exact power of two whenever 2^k is a
  // normal number -- the correctly rounded p 2^k, i.e. scalbn(p, k) bit for
  // bit (the library call is a dozen integer instructions)
  const int ki = (int)k;
  if (NH_LIKELY(ki >= -1022 && ki <= 1023))
    return __dmul_rn(p, __longlong_as_double((long long)(ki + 1023) << 52));
  return scalbn(p, ki);
}

// Two arguments at once: the same operations per argument as nh_det_exp (so
// the same bits), the two Horner chains interleaved in one basic block -- a
// single chain is 26 dependent fp64 operations.
__device__ __forceinline__ void nh_det_exp2(double xa, double xb, double& ya, double& yb) {
  const double ka = rint(__dmul_rn(xa, 1.4426950408889634));
  const double kb = rint(__dmul_rn(xb, 1.4426950408889634));
  const double ra = __dsub_rn(__dsub_rn(xa, __dmul_rn(ka, 0.6931471803691238)),
                              __dmul_rn(ka, 1.9082149292705877e-10));
  const double rb = __dsub_rn(__dsub_rn(xb, __dmul_rn(kb, 0.6931471803691238)),
                              __dmul_rn(kb, 1.9082149292705877e-10));
  const double* c = NH_EXP_COEF;
  double pa = c[0], pb = c[0];
#pragma unroll
  for (int n = 1; n < 14; ++n) {
    pa = __dadd_rn(__dmul_rn(pa, ra), c[n]);
    pb = __dadd_rn(__dmul_rn(pb, rb), c[n]);
  }
  const int ia = (int)ka, ib = (int)kb;
  if (NH_LIKELY(ia >= -1022 && ia <= 1023 && ib >= -1022 && ib <= 1023)) {
    ya = __dmul_rn(pa, __longlong_as_double((long long)(ia + 1023) << 52));
    yb = __dmul_rn(pb, __longlong_as_double((long long)(ib + 1023) << 52));
  } else {
    ya = scalbn(pa, ia);
    yb = scalbn(pb, ib);
  }
}

__device__ __forceinline__ double nh_det_log1p(double e) {
  const double z = __ddiv_rn(e, __dadd_rn(2.0, e));
  const double w = __dmul_rn(z, z);
  double s = 1.0 / 35.0;
#pragma unroll
  for (int k = 16; k >= 0; --k) s = __dadd_rn(__dmul_rn(s, w), 1.0 / (2 * k + 1));
  return __dmul_rn(2.0, __dmul_rn(z, s));
}

// sample coordinate of node j of an element whose index (as a double) is ed,
// bit-identical to GridSpec: edges = x_left + dx*e ; node1 = edges + dx ;
// inset +- 1e-9*dx
__device__ __forceinline__ double sample_xd(const nh_member& m, double ed, int j) {
  double edge = __dadd_rn(m.x_left, __dmul_rn(m.dx, ed));
  if (j == 0) return __dadd_rn(edge, m.eps);
  return __dsub_rn(__dadd_rn(edge, m.dx), m.eps);
}
__device__ __forceinline__ double sample_x(const nh_member& m, int e, int j) {
  return sample_xd(m, (double)e, j);
}

// SlideMotion.position (bathymetry.py:133-144): displacement, velocity, accel
__device__ __forceinline__ void motion_at(const double* p, double t, double& s, double& sp,
                                          double& spp) {
  double a0 = p[4], ut = p[5], t1 = p[6], t2 = p[7], t3 = p[8];
  double s1 = 0.5 * a0 * t1 * t1;
  if (t <= t1) {
    s = 0.5 * a0 * t * t; sp = a0 * t; spp = a0;
  } else if (t <= t2) {
    s = s1 + ut * (t - t1); sp = ut; spp = 0.0;
  } else if (t <= t3) {
    double q = t - t2;
    s = s1 + ut * (t - t1) - 0.5 * a0 * (q * q); sp = ut - a0 * q; spp = -a0;
  } else {
    double q = t3 - t2;
    s = s1 + ut * (t3 - t1) - 0.5 * a0 * (q * q); sp = 0.0; spp = 0.0;
  }
}

template <int KIND>
__device__ __forceinline__ BottomTime bottom_time_k(const nh_member& m, double t) {
  BottomTime bt{0.0, 0.0, 0.0};
  const double* p = m.bottom;
  if (KIND == NH_BOTTOM_PLATE) {
    bt.a = exp(-p[3] * fmax(t, 0.0));
  } else if (KIND == NH_BOTTOM_SMOOTH_BOX) {
    bt.a = nh_det_exp(__dmul_rn(-p[3], fmax(t, 0.0)));
  } else if (KIND == NH_BOTTOM_QUARTIC_SLIDE) {
    double s, sp, spp;
    motion_at(p, t, s, sp, spp);
    bt.a = p[3] + s; bt.b = sp; bt.c = spp;
  } else if (KIND == NH_BOTTOM_SLOPE_SLIDE) {
    double tt = fmax(t, 0.0), ts = p[10];
    if (tt >= ts) {
      bt.a = ts > 0.0 ? p[9] : p[5];
    } else {
      const double s = __ddiv_rn(tt, p[7]);
      const double E = nh_det_exp(__dmul_rn(-2.0, s));
      const double lc = __dsub_rn(__dadd_rn(s, nh_det_log1p(E)), 0.6931471805599453);  // ln cosh
      const double th = __ddiv_rn(__dsub_rn(1.0, E), __dadd_rn(1.0, E));               // tanh
      bt.a = __dadd_rn(p[5], __dmul_rn(__dmul_rn(p[6], p[7]), lc));
      bt.b = __dmul_rn(p[6], th);
      bt.c = __dmul_rn(__ddiv_rn(p[6], p[7]), __dsub_rn(1.0, __dmul_rn(th, th)));
    }
  }
  return bt;
}

__device__ __forceinline__ BottomTime bottom_time(const nh_member& m, double t) {
  switch (m.bottom_kind) {
    case NH_BOTTOM_PLATE: return bottom_time_k<NH_BOTTOM_PLATE>(m, t);
    case NH_BOTTOM_QUARTIC_SLIDE: return bottom_time_k<NH_BOTTOM_QUARTIC_SLIDE>(m, t);
    case NH_BOTTOM_SMOOTH_BOX: return bottom_time_k<NH_BOTTOM_SMOOTH_BOX>(m, t);
    case NH_BOTTOM_SLOPE_SLIDE: return bottom_time_k<NH_BOTTOM_SLOPE_SLIDE>(m, t);
    default: return bottom_time_k<NH_BOTTOM_FLAT>(m, t);
  }
}

// All six channels.  NEED_ALL = false evaluates only d and d_x (the others are
// returned as 0) for the predictor stages.
template <int KIND, bool NEED_ALL = true>
__device__ __forceinline__ Bottom6 bottom_eval(const nh_member& m, const BottomTime& bt,
                                               double x) {
  const double* p = m.bottom;
  Bottom6 b{p[0], 0.0, 0.0, 0.0, 0.0, 0.0};
  if (KIND == NH_BOTTOM_PLATE) {
    if (fabs(x) < p[2]) {
      double a = p[3], decay = bt.a;
      b.d = RSUB(p[0], RMUL(p[1], RSUB(1.0, decay)));
      if (NEED_ALL) {
        b.d_t = -p[1] * a * decay;
        b.d_tt = p[1] * a * a * decay;
      }
    }
  } else if (KIND == NH_BOTTOM_QUARTIC_SLIDE) {
    double c = p[9];
    double xi = RDIV(RMUL(2.0, RSUB(x, bt.a)), p[2]);
    if (fabs(xi) < 1.0) {
      double Hs = p[1], sp = bt.b, spp = bt.c;
#if NH_STRICT
      double x2 = RMUL(xi, xi), x3 = pow(xi, 3.0), x4 = pow(xi, 4.0);
#else
      double x2 = xi * xi, x3 = x2 * xi, x4 = x2 * x2;
#endif
      b.d = RSUB(p[0], RMUL(Hs, RSUB(1.0, x4)));
      b.d_x = RMUL(RMUL(RMUL(Hs, 4.0), x3), c);
      if (NEED_ALL) {
        b.d_xx = Hs * 12.0 * x2 * c * c;
        b.d_t = Hs * 4.0 * x3 * (-c * sp);
        b.d_xt = Hs * 12.0 * x2 * c * (-c * sp);
        double csp = c * sp;
        b.d_tt = Hs * (12.0 * x2 * (csp * csp) - 4.0 * x3 * c * spp);
      }
    }
  } else if (KIND == NH_BOTTOM_SMOOTH_BOX) {
    double y = RDIV(RSUB(fabs(x), p[2]), p[4]);
    if (y < NH_BOX_YCUT) {
      double decay = bt.a, z0 = p[1], al = p[3];
      double zeta = RMUL(z0, RSUB(1.0, decay));
      double E = nh_det_exp(RMUL(-2.0, fabs(y)));
      double inv1 = RDIV(1.0, RADD(1.0, E));
      double S = y >= 0.0 ? RMUL(E, inv1) : inv1;
      double sg = x >= 0.0 ? 1.0 : -1.0;
      double sech2 = RMUL(RMUL(RMUL(4.0, E), inv1), inv1);
      double Sx = RDIV(RMUL(RMUL(-0.5, sech2), sg), p[4]);
      b.d = RSUB(p[0], RMUL(zeta, S));
      b.d_x = RMUL(-zeta, Sx);
      if (NEED_ALL) {
        double zt = z0 * al * decay;
        double ztt = -z0 * al * al * decay;
        double th = (y >= 0.0 ? 1.0 : -1.0) * (1.0 - E) * inv1;
        double Sxx = RDIV(RMUL(sech2, th), RMUL(p[4], p[4]));
        b.d_t = -zt * S;
        b.d_tt = -ztt * S;
        b.d_xt = -zt * Sx;
        b.d_xx = -zeta * Sxx;
      }
    }
  } else if (KIND == NH_BOTTOM_SLOPE_SLIDE) {
    double ramp = RADD(p[0], RMUL(x, p[1]));
    bool on = ramp < p[2];
    b.d = on ? ramp : p[2];
    b.d_x = on ? p[1] : 0.0;
    // the model is defined with the packed reciprocal 1/sigma (p[11]): two
    // multiplications instead of two correctly rounded divisions per node
    double r = RMUL(RSUB(x, bt.a), p[11]);
    if (fabs(r) < NH_SLIDE_RCUT) {
      double G = RMUL(p[3], nh_det_exp(RMUL(RMUL(-0.5, r), r)));
      double Gx = RMUL(RMUL(-G, r), p[11]);
      b.d = RSUB(b.d, G);
      b.d_x = RSUB(b.d_x, Gx);
      if (NEED_ALL) {
        double Gxx = (G * (r * r - 1.0)) * (p[11] * p[11]);
        double v = bt.b, acc = bt.c;
        b.d_t = Gx * v;
        b.d_tt = -Gxx * v * v + Gx * acc;
        b.d_xt = Gxx * v;
        b.d_xx = -Gxx;
      }
    }
  }
  return b;
}

// Time-independent part of a node's depth for the predictor: the smoothed
// box's profile S(x) and S'(x) (everything but zeta(t)), so the two Heun
// stages of a step evaluate the profile once.  Other kinds carry nothing.
struct BottomSpace {
  double S, Sx;
  bool on;
};

template <int KIND>
__device__ __forceinline__ BottomSpace bottom_space(const nh_member& m, double x) {
  BottomSpace sp{0.0, 0.0, false};
  if (KIND == NH_BOTTOM_SMOOTH_BOX) {
    const double* p = m.bottom;
    double y = RDIV(RSUB(fabs(x), p[2]), p[4]);
    if (y < NH_BOX_YCUT) {
      double E = nh_det_exp(RMUL(-2.0, fabs(y)));
      double inv1 = RDIV(1.0, RADD(1.0, E));
      sp.S = y >= 0.0 ? RMUL(E, inv1) : inv1;
      double sg = x >= 0.0 ? 1.0 : -1.0;
      double sech2 = RMUL(RMUL(RMUL(4.0, E), inv1), inv1);
      sp.Sx = RDIV(RMUL(RMUL(-0.5, sech2), sg), p[4]);
      sp.on = true;
    }
  }
  return sp;
}

// d and d_x at time factor bt from a precomputed BottomSpace; bit-identical
// to bottom_eval<KIND, false>(m, bt, x).
template <int KIND>
__device__ __forceinline__ Bottom6 bottom_eval_sp(const nh_member& m, const BottomTime& bt,
                                                  double x, const BottomSpace& sp) {
  if (KIND == NH_BOTTOM_SMOOTH_BOX) {
    const double* p = m.bottom;
    Bottom6 b{p[0], 0.0, 0.0, 0.0, 0.0, 0.0};
    if (sp.on) {
      double zeta = RMUL(p[1], RSUB(1.0, bt.a));
      b.d = RSUB(p[0], RMUL(zeta, sp.S));
      b.d_x = RMUL(-zeta, sp.Sx);
    }
    return b;
  }
  return bottom_eval<KIND, false>(m, bt, x);
}

// d and d_x at both nodes of an element (predictor stages): bit-identical to
// two bottom_eval_sp calls; the slope slide's two Gaussians share one
// branch so their exp chains interleave (nh_det_exp2).
template <int KIND>
__device__ __forceinline__ void bottom_eval_sp2(const nh_member& m, const BottomTime& bt,
                                                double x0, double x1, const BottomSpace& s0,
                                                const BottomSpace& s1, Bottom6& b0, Bottom6& b1) {
  if (KIND == NH_BOTTOM_SLOPE_SLIDE) {
    const double* p = m.bottom;
    const double ramp0 = RADD(p[0], RMUL(x0, p[1])), ramp1 = RADD(p[0], RMUL(x1, p[1]));
    const bool on0 = ramp0 < p[2], on1 = ramp1 < p[2];
    b0 = Bottom6{on0 ? ramp0 : p[2], on0 ? p[1] : 0.0, 0.0, 0.0, 0.0, 0.0};
    b1 = Bottom6{on1 ? ramp1 : p[2], on1 ? p[1] : 0.0, 0.0, 0.0, 0.0, 0.0};
    const double r0 = RMUL(RSUB(x0, bt.a), p[11]), r1 = RMUL(RSUB(x1, bt.a), p[11]);
    const bool g0 = fabs(r0) < NH_SLIDE_RCUT, g1 = fabs(r1) < NH_SLIDE_RCUT;
    if (g0 || g1) {
      // a node outside the cut-off evaluates exp(0) and discards it
      double E0, E1;
      nh_det_exp2(g0 ? RMUL(RMUL(-0.5, r0), r0) : 0.0, g1 ? RMUL(RMUL(-0.5, r1), r1) : 0.0, E0, E1);
      if (g0) {
        const double G = RMUL(p[3], E0), Gx = RMUL(RMUL(-G, r0), p[11]);
        b0.d = RSUB(b0.d, G);
        b0.d_x = RSUB(b0.d_x, Gx);
      }
      if (g1) {
        const double G = RMUL(p[3], E1), Gx = RMUL(RMUL(-G, r1), p[11]);
        b1.d = RSUB(b1.d, G);
        b1.d_x = RSUB(b1.d_x, Gx);
      }
    }
    return;
  }
  b0 = bottom_eval_sp<KIND>(m, bt, x0, s0);
  b1 = bottom_eval_sp<KIND>(m, bt, x1, s1);
}

// KIND = -1: run-time dispatch on m.bottom_kind (CTA-uniform in the
// streaming kernels), one copy of the calling code instead of five
template <int KIND>
__device__ __forceinline__ BottomSpace bottom_space_k(const nh_member& m, double x) {
  if (KIND >= 0) return bottom_space<KIND>(m, x);
  if (m.bottom_kind == NH_BOTTOM_SMOOTH_BOX) return bottom_space<NH_BOTTOM_SMOOTH_BOX>(m, x);
  return BottomSpace{0.0, 0.0, false};
}

template <int KIND>
__device__ __forceinline__ Bottom6 bottom_eval_sp_k(const nh_member& m, const BottomTime& bt,
                                                    double x, const BottomSpace& sp) {
  if (KIND >= 0) return bottom_eval_sp<KIND>(m, bt, x, sp);
  switch (m.bottom_kind) {
    case NH_BOTTOM_PLATE: return bottom_eval_sp<NH_BOTTOM_PLATE>(m, bt, x, sp);
    case NH_BOTTOM_QUARTIC_SLIDE: return bottom_eval_sp<NH_BOTTOM_QUARTIC_SLIDE>(m, bt, x, sp);
    case NH_BOTTOM_SMOOTH_BOX: return bottom_eval_sp<NH_BOTTOM_SMOOTH_BOX>(m, bt, x, sp);
    case NH_BOTTOM_SLOPE_SLIDE: return bottom_eval_sp<NH_BOTTOM_SLOPE_SLIDE>(m, bt, x, sp);
    default: return bottom_eval_sp<NH_BOTTOM_FLAT>(m, bt, x, sp);
  }
}

template <bool NEED_ALL = true>
__device__ __forceinline__ Bottom6 bottom_eval_rt(const nh_member& m, const BottomTime& bt,
                                                  double x) {
  switch (m.bottom_kind) {
    case NH_BOTTOM_PLATE: return bottom_eval<NH_BOTTOM_PLATE, NEED_ALL>(m, bt, x);
    case NH_BOTTOM_QUARTIC_SLIDE: return bottom_eval<NH_BOTTOM_QUARTIC_SLIDE, NEED_ALL>(m, bt, x);
    case NH_BOTTOM_SMOOTH_BOX: return bottom_eval<NH_BOTTOM_SMOOTH_BOX, NEED_ALL>(m, bt, x);
    case NH_BOTTOM_SLOPE_SLIDE: return bottom_eval<NH_BOTTOM_SLOPE_SLIDE, NEED_ALL>(m, bt, x);
    default: return bottom_eval<NH_BOTTOM_FLAT, NEED_ALL>(m, bt, x);
  }
}

// run-time dispatch helpers for the non-hot kernels
__device__ __forceinline__ Bottom6 bottom_all(const nh_member& m, const BottomTime& bt, double x) {
  return bottom_eval_rt<true>(m, bt, x);
}
__device__ __forceinline__ double bottom_depth(const nh_member& m, const BottomTime& bt,
                                               double x) {
  return bottom_eval_rt<false>(m, bt, x).d;
}
__device__ __forceinline__ void bottom_d_dx(const nh_member& m, const BottomTime& bt, double x,
                                            double& d, double& d_x) {
  Bottom6 b = bottom_eval_rt<false>(m, bt, x);
  d = b.d; d_x = b.d_x;
}
