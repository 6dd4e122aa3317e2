// K_P of the streaming step (kernel in stream_kp.cu): load + pending hw
// correction, both Heun stages, criterion and flags of one tile.
#pragma once
#include <cooperative_groups.h>
#include "bathy.cuh"
#include "physics.cuh"
#include "stream_kernels.cuh"
#include "tree.cuh"

namespace {


constexpr int TPB = NH_STREAM_THREADS;     // 128
constexpr int H = NH_STREAM_HALO;          // 4
constexpr int OWN = TPB - 2 * H;           // 120
constexpr int NW = TPB / 32;
// levels of the cross-warp tree over the NW warp aggregates (a level that
// merges with identities only is an exact no-op, so fewer levels are bitwise
// the same result; every caller uses this count)
constexpr int NWL = NW <= 1 ? 0 : NW <= 2 ? 1 : NW <= 4 ? 2 : NW <= 8 ? 3 : NW <= 16 ? 4 : 5;

__device__ __forceinline__ double ederiv(const nh_member& m, double v0, double v1, int i) {
  return RMUL(fma(v1, m.deriv_ref[2 * i + 1], RMUL(v0, m.deriv_ref[2 * i])), m.two_over_dx);
}

struct Q6 {
  double h0, h1, q0, q1, w0, w1;
};

// one Heun stage for the thread's element: node sides from the registers,
// left face from the left neighbour's node-1 side (exchanged through smem),
// right face from the right neighbour's left face (exchanged through smem)
template <int KIND>
__device__ __forceinline__ void stage_tend(const nh_member& m, double g, const Q6& q,
                                           const BottomTime& bt, double x0, double x1,
                                           const BottomSpace& s0, const BottomSpace& s1, int i,
                                           int e, int N, double* sh, double* sf, double t6[6],
                                           double& speed, double& d0, double& d1) {
  Bottom6 b0, b1;
  if (KIND >= 0) {
    bottom_eval_sp2<KIND>(m, bt, x0, x1, s0, s1, b0, b1);
  } else {
    b0 = bottom_eval_sp_k<KIND>(m, bt, x0, s0);
    b1 = bottom_eval_sp_k<KIND>(m, bt, x1, s1);
  }
  Side n0, n1;
  make_sides_warp(q.h0, q.q0, q.w0, b0.d, q.h1, q.q1, q.w1, b1.d, n0, n1);
  sh[0 * TPB + i] = q.h1; sh[1 * TPB + i] = q.q1; sh[2 * TPB + i] = q.w1; sh[3 * TPB + i] = b1.d;
  sh[4 * TPB + i] = n1.u;
  __syncthreads();
  Side L;
  if (NH_UNLIKELY(e == 0)) {
    L = ghost_side(n0, m.bc_left);
  } else {   // the left neighbour's node-1 side, u included (no second division)
    int k = i > 0 ? i - 1 : 0;
    L.h = sh[0 * TPB + k]; L.hu = sh[1 * TPB + k]; L.hw = sh[2 * TPB + k];
    L.d = sh[3 * TPB + k]; L.u = sh[4 * TPB + k];
#if NH_STRICT
    L.rh = 0.0;
#else
    L.rh = nh_rcp(L.h);
#endif
  }
  double sp;
  Face fl = face_flux<KIND == NH_BOTTOM_FLAT, true>(L, n0, g, sp);
  speed = nh_max(speed, sp);
  sf[0 * TPB + i] = fl.F1; sf[1 * TPB + i] = fl.F2L; sf[2 * TPB + i] = fl.F3;
  __syncthreads();
  Face fr;
  if (NH_UNLIKELY(e == N - 1)) {
    fr = face_flux<KIND == NH_BOTTOM_FLAT>(n1, ghost_side(n1, m.bc_right), g, sp);
    speed = nh_max(speed, sp);
  } else {
    int k = i < TPB - 1 ? i + 1 : i;
    fr.F1 = sf[0 * TPB + k]; fr.F2L = sf[1 * TPB + k]; fr.F3 = sf[2 * TPB + k]; fr.F2R = 0.0;
  }
  element_tendency<KIND == NH_BOTTOM_FLAT>(m, g, n0, n1, fl, fr, b0.d_x, b1.d_x, t6);
  d0 = b0.d; d1 = b1.d;
}

__device__ __forceinline__ void store_super(double* dst, const Super& s) {
  dst[0] = s.ga; dst[1] = s.aa; dst[2] = s.ba; dst[3] = s.gz; dst[4] = s.az; dst[5] = s.bz;
}
__device__ __forceinline__ Super load_super(const double* s) {
  return Super{s[0], s[1], s[2], s[3], s[4], s[5]};
}

// The element's LDG coefficients as 10 scratch planes of stride BN (K_S or
// the fused K_P store, K_C loads): s11, s12, s22, f1, f2 at nodes 0 and 1.
constexpr int NH_COEF_PLANES = 10;
__device__ __forceinline__ void store_coef(double* sc, size_t BN, const NodeCoef& c0,
                                           const NodeCoef& c1) {
  sc[0 * BN] = c0.s11; sc[1 * BN] = c1.s11; sc[2 * BN] = c0.s12; sc[3 * BN] = c1.s12;
  sc[4 * BN] = c0.s22; sc[5 * BN] = c1.s22; sc[6 * BN] = c0.f1;  sc[7 * BN] = c1.f1;
  sc[8 * BN] = c0.f2;  sc[9 * BN] = c1.f2;
}
__device__ __forceinline__ void load_coef(const double* sc, size_t BN, NodeCoef& c0,
                                          NodeCoef& c1) {
  c0.s11 = sc[0 * BN]; c1.s11 = sc[1 * BN]; c0.s12 = sc[2 * BN]; c1.s12 = sc[3 * BN];
  c0.s22 = sc[4 * BN]; c1.s22 = sc[5 * BN]; c0.f1 = sc[6 * BN];  c1.f1 = sc[7 * BN];
  c0.f2 = sc[8 * BN];  c1.f2 = sc[9 * BN];
  c0.phi = 0.0; c1.phi = 0.0;
}

// CTA-level reduction of per-element super-elements (1 per thread) into the
// tile aggregate.  Nodes are stored so that tile_down() can unwind them.
__device__ __forceinline__ Super tile_up(Super agg, bool tflag, double* wnode, double* wagg,
                                         double* bnode, int* wflag, int lane, int warp) {
  const bool wany = __any_sync(0xffffffffu, tflag);
  double* wn = wnode + warp * 31 * 6;
  if (wany) {
    agg = warp_up<false>(agg, wn, lane, 5);   // aggregate only: K_C rebuilds the trees it unwinds
  } else {
    unsigned nonid = __ballot_sync(0xffffffffu, !is_identity(agg));
    int first = nonid ? __ffs(nonid) - 1 : 0;
    agg = shfl_super(agg, first);
    if (!nonid) agg = super_identity();
  }
  if (lane == 0) {
    store_super(wagg + warp * 6, agg);
    wflag[warp] = wany ? 1 : 0;
  }
  __syncthreads();
  Super v = super_identity();
  if (warp == 0) {
    if (lane < NW) v = load_super(wagg + lane * 6);
    v = warp_up<false>(v, bnode, lane, NWL);
  }
  return v;   // valid in thread 0
}

}  // namespace

// FUSE (template argument of the K_P body): K_P also condenses its flagged
// tiles and K_S is not launched.  Used for the global mode, where every tile
// is condensed and the fusion saves K_S's state re-read (config 4 global step
// 2.30 -> 2.17 ms); the adaptive mode keeps K_S (fused: 0.82 -> 0.86 ms,
// register pressure on every tile).

// ---------------------------------------------------------------------- K_P
struct KpSmem {
  double sh[5 * TPB];
  double sf[3 * TPB];
  double sk[6 * TPB];     // k1 of this thread's element
  alignas(16) double sq[6 * TPB];   // step-start state: [3][TPB] double2 (h, hu, hw node pairs)
  unsigned long long wcfl[NW];   // per warp: max wave speed bits (CFL = speed dt / dx at the end)
  uint8_t rf[TPB];
};



// (h p) traces of the pending correction: the sf planes
#define NH_HP_TRACES(ks) ((ks).sf)

struct KsSmem {
  double wnode[NW * 31 * 6];
  double wagg[NW * 6];
  double bnode[31 * 6];
  int wflag[NW];
};
static_assert(sizeof(KsSmem) <= 12 * TPB * sizeof(double), "K_S tree nodes alias sk + sq");

// Per-thread geometry of a streaming tile.
struct TileIdx {
  int b, tile, i, lane, warp, e;
  bool valid, own;
  size_t o;
};

__device__ __forceinline__ TileIdx tile_idx(const StreamArgs& a, int b, int tile) {
  TileIdx t;
  t.b = b; t.tile = tile;
  t.i = threadIdx.x; t.lane = t.i & 31; t.warp = t.i >> 5;
  t.e = t.tile * OWN - H + t.i;
  // one unsigned compare per range test; o is only dereferenced for valid
  // slots, so it is not clamped (CTA-uniform base + slot): cheaper to
  // re-materialise, which the 64-register cap forces a dozen times
  t.valid = (unsigned)t.e < (unsigned)a.N;
  t.own = t.valid && (unsigned)(t.i - H) < (unsigned)OWN;
  t.o = (size_t)((long long)t.b * a.N + (t.tile * OWN - H) + t.i) * 2;
  return t;
}

// Per-member constants of one step, written once per member by K_X (for the
// next step) or the prep kernel (first step) so tile kernels copy them with
// the member record instead of recomputing them serially per CTA.
struct MemberConst {
  LdgConst lk;        // 8 doubles
  BottomTime bt0;     // bottom time factors at t
  BottomTime bt1;     // ... and at t + dt
  double pad[2];
};
static_assert(sizeof(MemberConst) == 16 * 8, "MemberConst is 16 doubles");

__device__ __forceinline__ void member_const(const nh_member& m, const nh_scheme& sch, double t,
                                             double* out) {
  MemberConst c;
  c.lk = make_ldg_const(m.dt, sch.g, sch.rho);
  c.bt0 = bottom_time(m, t);
  c.bt1 = bottom_time(m, t + m.dt);
  c.pad[0] = c.pad[1] = 0.0;
  *reinterpret_cast<MemberConst*>(out) = c;
}

// cooperative copy of the member record (39 words) and its step constants (16)
__device__ __forceinline__ void load_member(const StreamArgs& a, int b, nh_member& msh,
                                            MemberConst& mc) {
  constexpr int MW = (int)(sizeof(nh_member) / 8);
  const int i = threadIdx.x;
  if (i < MW)
    reinterpret_cast<unsigned long long*>(&msh)[i] =
        reinterpret_cast<const unsigned long long*>(a.members + b)[i];
  else if (i < MW + 16)
    reinterpret_cast<unsigned long long*>(&mc)[i - MW] =
        reinterpret_cast<const unsigned long long*>(a.mconst + (size_t)b * 16)[i - MW];
}

// One flagged element's LDG condensation (K_S, or the fused K_P):
// LDG coefficients at t + dt (corrector.py:100-170), the element block
// eliminated to its super-element (corrector.py:173-349 -> physics.cuh) for
// the tile aggregate, the coefficients stored for K_C (which re-eliminates
// the block for the reconstruction rows and evaluates the residual gate), and
// phi / d_x stored in the pending record of the hw update.  q = predictor
// state of the element.
template <int KIND>
__device__ __forceinline__ void condense_element(const StreamArgs& a, const nh_member& m,
                                                 const LdgConst& lk, const BottomTime& bt1, int b,
                                                 int e, const Q6& q, bool range_end, Super& S) {
  const int N = a.N;
  const double ed = (double)e;
  const double x0 = sample_xd(m, ed, 0), x1 = sample_xd(m, ed, 1);
  Bottom6 b0 = bottom_eval<KIND, true>(m, bt1, x0);
  Bottom6 b1 = bottom_eval<KIND, true>(m, bt1, x1);
  Chan ch0{b0.d, b0.d_x, b0.d_t, b0.d_tt, b0.d_xt, b0.d_xx};
  Chan ch1{b1.d, b1.d_x, b1.d_t, b1.d_tt, b1.d_xt, b1.d_xx};
  double exa = ederiv(m, q.h0 - b0.d, q.h1 - b1.d, 0);
  double exb = ederiv(m, q.h0 - b0.d, q.h1 - b1.d, 1);
  NodeCoef c0 = ldg_coefficients(q.h0, q.q0, q.w0, ederiv(m, q.h0, q.h1, 0), exa, ch0, lk);
  NodeCoef c1 = ldg_coefficients(q.h1, q.q1, q.w1, ederiv(m, q.h0, q.h1, 1), exb, ch1, lk);
  // field-major planes: each store of the warp is one coalesced run (stored
  // before the elimination, so the coefficients are dead during it)
  const size_t BN = (size_t)a.B * N, fe = (size_t)b * N + e;
  store_coef(a.scratch + fe, BN, c0, c1);
  double* pn = a.pend_out + fe;
  pn[2 * BN] = c0.phi; pn[3 * BN] = c1.phi; pn[4 * BN] = b0.d_x; pn[5 * BN] = b1.d_x;
  const int step = a.step_counter ? a.step_counter[b] : 0;
  if (!ldg_structure_ok(c0, c1)) nh_report(a.status + b, step, NH_ERR_STRUCTURE, e);
  double R[6];
  if (!local_condense(m, c0, c1, lk.rho, lk.inv_rho, a.sch.c11, range_end, S, R))
    nh_report(a.status + b, step, NH_ERR_SOLVE_PIVOT, e);
}

template <int KIND, bool FUSE, class SM>
__device__ __forceinline__ void kp_body(const StreamArgs& a, const nh_member& m,
                                        const MemberConst& mc, const TileIdx& ti, Q6 q,
                                        SM& ks, double* sq) {
  double* sh = ks.sh;
  double* sf = ks.sf;
  uint8_t* rf = ks.rf;
  double* XS = sh;
  double* XF = sf;

  const int N = a.N, T = a.tiles;
  const int b = ti.b, tile = ti.tile, i = ti.i, lane = ti.lane, e = ti.e;
  const bool valid = ti.valid, own = ti.own;
  const size_t o = ti.o;
  const nh_scheme& sch = a.sch;
  const double g = sch.g;
  nh_status* st = a.status + b;
  const int step = a.step_counter ? a.step_counter[b] : 0;

  const double dt = m.dt;
  const double ed = (double)e;
  const double x0 = sample_xd(m, ed, 0), x1 = sample_xd(m, ed, 1);
  const BottomSpace s0 = bottom_space_k<KIND>(m, x0), s1 = bottom_space_k<KIND>(m, x1);
  double speed = 0.0;

  // ---------------- Heun stage 1 at t ----------------
  // positivity (hydrostatic.py:101-103, 216-217) gathered into one report
  unsigned bad = (own && (q.h0 <= 0.0 || q.h1 <= 0.0)) ? 1u : 0u;
  {   // step-start state, one (node 0, node 1) pair per field: [3][TPB] double2
    double2* s2 = reinterpret_cast<double2*>(sq);
    s2[0 * TPB + i] = double2{q.h0, q.h1};
    s2[1 * TPB + i] = double2{q.q0, q.q1};
    s2[2 * TPB + i] = double2{q.w0, q.w1};
  }
  Q6 qs;
  {
    double k1[6], dd0, dd1;
    stage_tend<KIND>(m, g, q, mc.bt0, x0, x1, s0, s1, i, e, N, XS, XF, k1, speed, dd0, dd1);
#pragma unroll
    for (int f = 0; f < 6; ++f) ks.sk[f * TPB + i] = k1[f];
    qs = Q6{RADD(q.h0, RMUL(dt, k1[0])), RADD(q.h1, RMUL(dt, k1[1])),
            RADD(q.q0, RMUL(dt, k1[2])), RADD(q.q1, RMUL(dt, k1[3])),
            RADD(q.w0, RMUL(dt, k1[4])), RADD(q.w1, RMUL(dt, k1[5]))};
  }
  bad |= (own && !(qs.h0 > 0.0 && qs.h1 > 0.0)) ? 2u : 0u;
  // (no barrier before stage 2: its sh writes follow stage 1's sf barrier,
  // which every stage-1 sh read precedes, and its sf writes follow its own
  // sh barrier, which every stage-1 sf read precedes)

  // ---------------- Heun stage 2 at t + dt ----------------
  double k2[6], d0, d1;   // d0, d1: depth at t + dt, reused by the criterion
  {
    double dummy = 0.0;
    stage_tend<KIND>(m, g, qs, mc.bt1, x0, x1, s0, s1, i, e, N, XS, XF, k2, dummy, d0, d1);
  }
  double qv[6];
#pragma unroll
  for (int f = 0; f < 6; ++f)
    qv[f] = RADD(sq[(f >> 1) * 2 * TPB + 2 * i + (f & 1)],
                 RMUL(dt, RMUL(0.5, RADD(ks.sk[f * TPB + i], k2[f]))));
  Q6 qp{qv[0], qv[1], qv[2], qv[3], qv[4], qv[5]};
  bad |= (own && !(qp.h0 > 0.0 && qp.h1 > 0.0)) ? 4u : 0u;
  if (sch.record_cfl) {
    // max wave speed over the warp on the bit patterns (speeds are >= 0, so
    // the unsigned order is the numeric order): high words, then low words of
    // the lanes holding the maximal high word.  Halo lanes contribute 0.
    const unsigned long long u = (unsigned long long)__double_as_longlong(own ? speed : 0.0);
    const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(u >> 32));
    const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned)(u >> 32) == hi ? (unsigned)u : 0u);
    if (lane == 0) ks.wcfl[ti.warp] = ((unsigned long long)hi << 32) | lo;
  }

  // ---------------- criterion on the predictor (t + dt) ----------------
  uint8_t raw = 0;
#if NH_STRICT
  if (sch.mode == NH_MODE_ADAPTIVE && sch.criterion == NH_CRIT_ETA_OVER_D) {
    // the default criterion, evaluated by the whole warp (one vote for both
    // divisions); halo slots past the domain ends compute and discard
    const double e0 = RSUB(qp.h0, d0), e1 = RSUB(qp.h1, d1);
    // |e / d| > k decided without the division wherever that is certain:
    // with p = k d, |e| >= p (1 + 2^-50) puts e / d more than an ulp above k
    // and |e| <= p (1 - 2^-50) more than an ulp below it, so the rounded
    // quotient compares the same way.  Only an element inside that 2^-49
    // band takes the correctly rounded division (one warp vote) -- the flag
    // is the reference's bit for bit.
    const double k = sch.k_nh;
    const double a0 = fabs(e0), a1 = fabs(e1), p0 = k * d0, p1 = k * d1;
    const double up = 1.0 + 0x1p-50, dn = 1.0 - 0x1p-50;
    const bool sure = a0 >= p0 * up || a1 >= p1 * up;
    const bool amb = !sure && (a0 > p0 * dn || a1 > p1 * dn);
    bool hit = sure;
    NH_WARP_FIX(amb, (hit = sure || nh_max(fabs(RDIVP(e0, d0)), fabs(RDIVP(e1, d1))) > k));
    raw = (valid && hit) ? 1 : 0;
  } else
#endif
  if (valid && sch.mode != NH_MODE_HYDROSTATIC) {
    if (sch.mode == NH_MODE_GLOBAL) {
      raw = 1;
    } else {
      double v0, v1;
      switch (sch.criterion) {
        case NH_CRIT_ETA_OVER_D: {
          v0 = fabs(RDIVP(RSUB(qp.h0, d0), d0)); v1 = fabs(RDIVP(RSUB(qp.h1, d1), d1));
          break;
        }
        case NH_CRIT_ETA_X: {
          v0 = fabs(ederiv(m, RSUB(qp.h0, d0), RSUB(qp.h1, d1), 0));
          v1 = fabs(ederiv(m, RSUB(qp.h0, d0), RSUB(qp.h1, d1), 1));
          break;
        }
        case NH_CRIT_U:
          v0 = fabs(RDIVP(qp.q0, qp.h0)); v1 = fabs(RDIVP(qp.q1, qp.h1));
          break;
        case NH_CRIT_U_X: {
          double u0 = RDIVP(qp.q0, qp.h0), u1 = RDIVP(qp.q1, qp.h1);
          v0 = fabs(ederiv(m, u0, u1, 0)); v1 = fabs(ederiv(m, u0, u1, 1));
          break;
        }
        case NH_CRIT_W:
          v0 = fabs(RDIVP(qp.w0, qp.h0)); v1 = fabs(RDIVP(qp.w1, qp.h1));
          break;
        default: {
          double w0 = RDIVP(qp.w0, qp.h0), w1 = RDIVP(qp.w1, qp.h1);
          v0 = fabs(ederiv(m, w0, w1, 0)); v1 = fabs(ederiv(m, w0, w1, 1));
          break;
        }
      }
      raw = nh_max(v0, v1) > sch.k_nh ? 1 : 0;
    }
  }
  rf[i] = raw;
  __syncthreads();
  if (NH_UNLIKELY(bad))   // the reference raises at the first failing check: lowest code wins
    nh_report(st, step,
              (bad & 1u) ? NH_ERR_POSITIVITY_ENTRY
                         : ((bad & 2u) ? NH_ERR_POSITIVITY_STAGE1 : NH_ERR_POSITIVITY_STAGE2),
              (bad & 1u) ? e : -1);
  if (own) {
    *reinterpret_cast<double2*>(a.h_out + o) = double2{qp.h0, qp.h1};
    *reinterpret_cast<double2*>(a.hu_out + o) = double2{qp.q0, qp.q1};
    *reinterpret_cast<double2*>(a.hw_out + o) = double2{qp.w0, qp.w1};
  }
  // CFL of the tile = (max speed) dt / dx: rounding is monotone, so this is
  // the max over elements of the per-element speed dt / dx (hydrostatic.py CFL check)
  auto publish_cfl = [&]() {   // after the flags barrier: every warp's slot is written
    if (i != 0 || !sch.record_cfl) return;
    unsigned long long mx = ks.wcfl[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) mx = max(mx, ks.wcfl[w]);
    const double cfl_sh = __longlong_as_double((long long)mx);
    if (cfl_sh > 0.0) {
      const double c = cfl_sh * dt / m.dx;
      atomicMax((unsigned long long*)&st->cfl_max, (unsigned long long)__double_as_longlong(c));
    }
  };
  if (sch.mode == NH_MODE_HYDROSTATIC) {
    publish_cfl();
    return;
  }
  const bool enl = sch.mode == NH_MODE_ADAPTIVE && sch.enlarge;
  auto eff = [&](int s) -> bool {
    int ee = tile * OWN - H + s;
    if (ee < 0 || ee >= N || s < 0 || s >= TPB) return false;
    bool f = rf[s] != 0;
    if (enl) {
      if (ee > 0 && s > 0) f = f || rf[s - 1];
      if (ee < N - 1 && s + 1 < TPB) f = f || rf[s + 1];
    }
    return f;
  };
  const bool flag = own && eff(i);
  if (own) a.flags_cur[(size_t)b * N + e] = flag ? 1 : 0;
  if (flag && a.flag_bits) {
    uint32_t* fb = a.flag_bits + ((size_t)step * a.B + b) * ((N + 31) / 32);
    atomicOr(fb + (e >> 5), 1u << (e & 31));
  }

  // ---------------- per-tile flagged count; unflagged tiles aggregate to a gap ----------------
  {
    int nf = __syncthreads_count(flag);
    if (i == H) {   // first own slot
      double* ta = a.tile_agg + ((size_t)b * T + tile) * 8;
      ta[6] = (double)nf;
      if (nf == 0) store_super(ta, super_gap(qp.q0));
      if (nf) {
        atomicAdd((unsigned long long*)&st->flagged, (unsigned long long)nf);
        a.tile_list[atomicAdd(a.tile_count, 1)] = b * T + tile;   // work list of K_S / K_C
      }
    }
    if (FUSE && nf) {   // CTA-uniform: this tile's condensation and aggregate (K_S's work)
      Super S = super_identity();
      if (own) S = super_gap(qp.q0);
      if (flag) condense_element<KIND>(a, m, mc.lk, mc.bt1, b, e, qp, (e == N - 1) || !eff(i + 1), S);
      // tree nodes in the k1 / step-start planes, dead since the Heun combination
      KsSmem& kss = *reinterpret_cast<KsSmem*>(ks.sk);
      Super v = tile_up(S, flag, kss.wnode, kss.wagg, kss.bnode, kss.wflag, lane, ti.warp);
      if (i == 0) store_super(a.tile_agg + ((size_t)b * T + tile) * 8, v);
    }
    // right-end ghost outer trace (corrector.py:400-402)
    if (e == N - 1 && own) {
      double qq = qp.q1;
      a.tile_agg[((size_t)b * T + tile) * 8 + 7] = (m.bc_right == NH_BC_WALL) ? -qq : qq;
    }
  }
  publish_cfl();
}

// The previous step's pending hw correction of the thread's element (q.w
// updated in place) and the step body.  On entry the (h p) traces are in
// NH_HP_TRACES(ks), made visible by the caller's barrier.
// hw += dt/rho (6/quad p + d_x/quad (h p)_x + phi) on flagged elements
// (corrector.py:441-482); (h p)_x lifts use the neighbours' (h p) traces.
template <bool FUSE, bool FIN, class SM>
__device__ __forceinline__ void kp_correct_and_step(const StreamArgs& a, const TileIdx& ti,
                                                    const nh_member& msh, const MemberConst& mc,
                                                    SM& ks, double* sq, Q6 q, bool f, double p0,
                                                    double p1, double phi0, double phi1,
                                                    double dx0, double dx1) {
  const int N = a.N, i = ti.i, b = ti.b, e = ti.e;
  const double hp0 = q.h0 * p0, hp1 = q.h1 * p1;
  double bp0 = 0.0, bp1 = 0.0;
  if (f) {
    const double* sh = NH_HP_TRACES(ks);
    auto hp_of = [&](int ee, int node, int slot) -> double {
      if (slot >= 0 && slot < TPB) return sh[node * TPB + slot];
      // neighbour outside the CTA's slots (never needed for own elements)
      if (!a.flags_prev[(size_t)b * N + ee]) return 0.0;
      size_t oo = ((size_t)b * N + ee) * 2 + node;
      return a.h_in[oo] * a.pend[(size_t)node * a.B * N + (size_t)b * N + ee];
    };
    double hx0 = ederiv(msh, hp0, hp1, 0), hx1 = ederiv(msh, hp0, hp1, 1);
    if (e < N - 1) {
      double hr = hp_of(e + 1, 0, i + 1);
      double avg = 0.5 * (hp1 + hr);
      hx0 += (avg - hp1) * msh.lift_right[0];
      hx1 += (avg - hp1) * msh.lift_right[1];
    }
    if (e > 0) {
      double hl = hp_of(e - 1, 1, i - 1);
      double avg = 0.5 * (hl + hp0);
      hx0 -= (avg - hp0) * msh.lift_left[0];
      hx1 -= (avg - hp0) * msh.lift_left[1];
    }
    double qd0 = 4.0 + dx0 * dx0, qd1 = 4.0 + dx1 * dx1;
    bp0 = nh_div(6.0, qd0) * p0 + nh_div(dx0, qd0) * hx0 + phi0;
    bp1 = nh_div(6.0, qd1) * p1 + nh_div(dx1, qd1) * hx1 + phi1;
  }
  // (no barrier: the traces live in the sf planes, which stage 1 first
  // writes after its sh barrier, i.e. after every thread's reads here)
  if (f) {
    q.w0 += mc.lk.cdt * bp0;
    q.w1 += mc.lk.cdt * bp1;
  }
  if (FIN) {   // K_fin: only flagged elements change (the tile is on the last step's list)
    if (f && ti.own) {
      double2 vw{q.w0, q.w1};
      *reinterpret_cast<double2*>(const_cast<double*>(a.hw_in) + ti.o) = vw;
    }
    return;
  }
  if (a.finalize) {
    if (ti.own) {
      double2 vw{q.w0, q.w1};
      *reinterpret_cast<double2*>(const_cast<double*>(a.hw_in) + ti.o) = vw;
    }
    // residual gate of the last step's solve (K_X checks the earlier ones)
    if (ti.tile == 0 && i == 0 && a.step_counter)
      resid_check(a.status + b, a.step_counter[b] - 1, a.sch.residual_tol);
    return;
  }
  if (a.hw_any) {   // w / w_x criterion: member-wide any(hw != 0) of the step input
    if (__syncthreads_or(ti.own && (q.w0 != 0.0 || q.w1 != 0.0)) && i == 0) a.hw_any[b] = 1;
  }
#ifdef NH_KP_ONLY_KIND   // diagnostics: one body, for reading its SASS (cuobjdump) in isolation
  kp_body<NH_KP_ONLY_KIND, FUSE>(a, msh, mc, ti, q, ks, sq);
  return;
#endif
  switch (msh.bottom_kind) {
    case NH_BOTTOM_FLAT: kp_body<NH_BOTTOM_FLAT, FUSE>(a, msh, mc, ti, q, ks, sq); break;
    case NH_BOTTOM_PLATE: kp_body<NH_BOTTOM_PLATE, FUSE>(a, msh, mc, ti, q, ks, sq); break;
    case NH_BOTTOM_QUARTIC_SLIDE: kp_body<NH_BOTTOM_QUARTIC_SLIDE, FUSE>(a, msh, mc, ti, q, ks, sq); break;
    case NH_BOTTOM_SMOOTH_BOX: kp_body<NH_BOTTOM_SMOOTH_BOX, FUSE>(a, msh, mc, ti, q, ks, sq); break;
    default: kp_body<NH_BOTTOM_SLOPE_SLIDE, FUSE>(a, msh, mc, ti, q, ks, sq); break;
  }
}

// One K_P tile (b, tile): the body of nh_stream_kp / nh_stream_kp_fused, and
// (FIN) of nh_stream_kfin, which applies the last pending update only.
template <bool FUSE, bool FIN = false>
__device__ __forceinline__ void kp_tile(const StreamArgs& a, const TileIdx& ti, nh_member& msh,
                                        MemberConst& mc, KpSmem& ks) {
  const int N = a.N, i = ti.i, b = ti.b, e = ti.e;

  // state and the previous step's pending record are requested first so their
  // latency overlaps the member-record copy and the per-CTA constants
  Q6 q{1.0, 1.0, 0.0, 0.0, 0.0, 0.0};
  if (ti.valid) {
    double2 vh = *reinterpret_cast<const double2*>(a.h_in + ti.o);
    double2 vq = *reinterpret_cast<const double2*>(a.hu_in + ti.o);
    double2 vw = *reinterpret_cast<const double2*>(a.hw_in + ti.o);
    q = Q6{vh.x, vh.y, vq.x, vq.y, vw.x, vw.y};
  }
  const bool f = a.pend && ti.valid && a.flags_prev[(size_t)b * N + e];
  double p0 = 0.0, p1 = 0.0, phi0 = 0.0, phi1 = 0.0, dx0 = 0.0, dx1 = 0.0;
  if (f) {
    const size_t BN = (size_t)a.B * N;
    const double* pv = a.pend + (size_t)b * N + e;
    p0 = pv[0]; p1 = pv[BN]; phi0 = pv[2 * BN]; phi1 = pv[3 * BN]; dx0 = pv[4 * BN]; dx1 = pv[5 * BN];
  }
  load_member(a, b, msh, mc);
  if (a.pend) {
    NH_HP_TRACES(ks)[0 * TPB + i] = q.h0 * p0;
    NH_HP_TRACES(ks)[1 * TPB + i] = q.h1 * p1;
  }
  __syncthreads();
  kp_correct_and_step<FUSE, FIN>(a, ti, msh, mc, ks, ks.sq, q, f, p0, p1, phi0, phi1, dx0, dx1);
}
