// Device bottom models: d(x, t) and the five derivative channels.
//
// Restates reference bathymetry.py:66-184 (FlatBottom, HammackPlate,
// SlideMotion/WhittakerSlide) and the two harness models of SURVEY.md
// Appendix C (smoothed box uplift, Gaussian mound on a slope) whose numpy
// twins live in oracle/nhswe_oracle.py.  Nothing is stored in HBM: each
// channel is evaluated in registers at the inset sample nodes
// (grid.py:84-90).  Time-only factors are hoisted into BottomTime once per
// (thread, instant).
#pragma once
#include "nh_common.cuh"

struct Bottom6 {
  double d, d_x, d_t, d_tt, d_xt, d_xx;
};

struct BottomTime {
  double a, b, c;   // model-specific time factors
};

// sample coordinate of node j of element e, bit-identical to GridSpec:
// edges = x_left + dx*e ; node1 = edges + 0.5*dx*2 ; inset +- 1e-9*dx
__device__ __forceinline__ double sample_x(const nh_member& m, int e, int j) {
  double edge = __dadd_rn(m.x_left, __dmul_rn(m.dx, (double)e));
  if (j == 0) return __dadd_rn(edge, m.eps);
  double node = __dadd_rn(edge, m.dx);
  return __dsub_rn(node, m.eps);
}

// SlideMotion.position (bathymetry.py:133-144): displacement, velocity, accel
__device__ __forceinline__ void motion_at(const double* p, double t, double& s, double& sp,
                                          double& spp) {
  // p: h0, Hs, Ls, x_start, a0, u_t, t1, t2, t3
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

__device__ __forceinline__ BottomTime bottom_time(const nh_member& m, double t) {
  BottomTime bt{0.0, 0.0, 0.0};
  const double* p = m.bottom;
  switch (m.bottom_kind) {
    case NH_BOTTOM_PLATE: {            // p: h0, zeta0, b, alpha
      bt.a = exp(-p[3] * fmax(t, 0.0));
      break;
    }
    case NH_BOTTOM_QUARTIC_SLIDE: {    // centre, sp, spp
      double s, sp, spp;
      motion_at(p, t, s, sp, spp);
      bt.a = p[3] + s; bt.b = sp; bt.c = spp;
      break;
    }
    case NH_BOTTOM_SMOOTH_BOX: {       // p: h0, zeta0, b, alpha, w
      bt.a = exp(-p[3] * fmax(t, 0.0));
      break;
    }
    case NH_BOTTOM_SLOPE_SLIDE: {
      // p: d_top, tan, d_max, A, sigma, x0, u_t, t0, d_stop, x_stop, t_stop
      double tt = fmax(t, 0.0), ts = p[10];
      if (tt >= ts) {
        bt.a = ts > 0.0 ? p[9] : p[5]; bt.b = 0.0; bt.c = 0.0;
      } else {
        double s = tt / p[7];
        double lc = s + log1p(exp(-2.0 * s)) - 0.6931471805599453;  // ln cosh(s)
        double th = tanh(s);
        bt.a = p[5] + p[6] * p[7] * lc;
        bt.b = p[6] * th;
        bt.c = (p[6] / p[7]) * (1.0 - th * th);
      }
      break;
    }
    default: break;
  }
  return bt;
}

// Depth only (criterion, interface reconstruction).
__device__ __forceinline__ double bottom_depth(const nh_member& m, const BottomTime& bt,
                                               double x) {
  const double* p = m.bottom;
  switch (m.bottom_kind) {
    case NH_BOTTOM_FLAT: return p[0];
    case NH_BOTTOM_PLATE:
      return fabs(x) < p[2] ? p[0] - p[1] * (1.0 - bt.a) : p[0];
    case NH_BOTTOM_QUARTIC_SLIDE: {
      double xi = 2.0 * (x - bt.a) / p[2];
      if (!(fabs(xi) < 1.0)) return p[0];
      double x2 = xi * xi;
      return p[0] - p[1] * (1.0 - x2 * x2);
    }
    case NH_BOTTOM_SMOOTH_BOX: {
      double zeta = p[1] * (1.0 - bt.a);
      double y = (fabs(x) - p[2]) / p[4];
      double E = exp(-2.0 * fabs(y));
      double inv1 = 1.0 / (1.0 + E);
      double S = y >= 0.0 ? E * inv1 : inv1;
      return p[0] - zeta * S;
    }
    case NH_BOTTOM_SLOPE_SLIDE: {
      double ramp = p[0] + x * p[1];
      double d0 = ramp < p[2] ? ramp : p[2];
      double r = (x - bt.a) / p[4];
      return d0 - p[3] * exp(-0.5 * r * r);
    }
    default: return p[0];
  }
}

// All six channels.
__device__ __forceinline__ Bottom6 bottom_all(const nh_member& m, const BottomTime& bt,
                                              double x) {
  const double* p = m.bottom;
  Bottom6 b{p[0], 0.0, 0.0, 0.0, 0.0, 0.0};
  switch (m.bottom_kind) {
    case NH_BOTTOM_FLAT: break;
    case NH_BOTTOM_PLATE: {
      if (fabs(x) < p[2]) {
        double a = p[3], decay = bt.a;
        b.d = p[0] - p[1] * (1.0 - decay);
        b.d_t = -p[1] * a * decay;
        b.d_tt = p[1] * a * a * decay;
      }
      break;
    }
    case NH_BOTTOM_QUARTIC_SLIDE: {
      double c = 2.0 / p[2];
      double xi = 2.0 * (x - bt.a) / p[2];
      if (fabs(xi) < 1.0) {
        double Hs = p[1], sp = bt.b, spp = bt.c;
        double x2 = xi * xi, x3 = x2 * xi;
        b.d = p[0] - Hs * (1.0 - x2 * x2);
        b.d_x = Hs * 4.0 * x3 * c;
        b.d_xx = Hs * 12.0 * x2 * c * c;
        b.d_t = Hs * 4.0 * x3 * (-c * sp);
        b.d_xt = Hs * 12.0 * x2 * c * (-c * sp);
        double csp = c * sp;
        b.d_tt = Hs * (12.0 * x2 * (csp * csp) - 4.0 * x3 * c * spp);
      }
      break;
    }
    case NH_BOTTOM_SMOOTH_BOX: {
      double decay = bt.a, z0 = p[1], al = p[3], w = p[4];
      double zeta = z0 * (1.0 - decay);
      double zt = z0 * al * decay;
      double ztt = -z0 * al * al * decay;
      double y = (fabs(x) - p[2]) / w;
      double E = exp(-2.0 * fabs(y));
      double inv1 = 1.0 / (1.0 + E);
      double S = y >= 0.0 ? E * inv1 : inv1;
      double sg = x >= 0.0 ? 1.0 : -1.0;
      double sech2 = 4.0 * E * inv1 * inv1;
      double Sx = -0.5 * sech2 * sg / w;
      double th = (y >= 0.0 ? 1.0 : -1.0) * (1.0 - E) * inv1;
      double Sxx = sech2 * th / (w * w);
      b.d = p[0] - zeta * S;
      b.d_x = -zeta * Sx;
      b.d_t = -zt * S;
      b.d_tt = -ztt * S;
      b.d_xt = -zt * Sx;
      b.d_xx = -zeta * Sxx;
      break;
    }
    case NH_BOTTOM_SLOPE_SLIDE: {
      double ramp = p[0] + x * p[1];
      bool on = ramp < p[2];
      double d0 = on ? ramp : p[2];
      double d0x = on ? p[1] : 0.0;
      double sig = p[4];
      double r = (x - bt.a) / sig;
      double G = p[3] * exp(-0.5 * r * r);
      double Gx = -G * r / sig;
      double Gxx = G * (r * r - 1.0) / (sig * sig);
      double v = bt.b, acc = bt.c;
      b.d = d0 - G;
      b.d_x = d0x - Gx;
      b.d_t = Gx * v;
      b.d_tt = -Gxx * v * v + Gx * acc;
      b.d_xt = Gxx * v;
      b.d_xx = -Gxx;
      break;
    }
    default: break;
  }
  return b;
}

// depth + slope (stage tendencies need d for reconstruction, d_x for the source)
__device__ __forceinline__ void bottom_d_dx(const nh_member& m, const BottomTime& bt, double x,
                                            double& d, double& d_x) {
  if (m.bottom_kind == NH_BOTTOM_FLAT) { d = m.bottom[0]; d_x = 0.0; return; }
  if (m.bottom_kind == NH_BOTTOM_PLATE) { d = bottom_depth(m, bt, x); d_x = 0.0; return; }
  Bottom6 b = bottom_all(m, bt, x);
  d = b.d; d_x = b.d_x;
}
