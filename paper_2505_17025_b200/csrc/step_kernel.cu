// Fused adaptive non-hydrostatic SWE time step for B200 (sm_100a).
//
// One thread-block CLUSTER owns one ensemble member (an independent 1D
// channel of N P1 elements).  Each CTA of the cluster owns a contiguous tile
// of `tile` elements and keeps it, plus a halo of H elements on each side,
// RESIDENT IN SHARED MEMORY for all n_steps of the launch: HBM is touched
// once to load the member and once to store it, whatever n_steps is.  Per
// step the CTA runs, entirely on chip:
//
//   1. Heun stage 1 at t    (hydrostatic.py:192-209, rhs_operator :88-184)
//   2. Heun stage 2 at t+dt
//   3. criterion + optional +-1 enlargement      (adaptivity.py:75-113)
//   4. LDG coefficients and per-element condensation (corrector.py:100-349)
//   5. segmented elimination of the flagged ranges: thread chunk -> warp ->
//      CTA -> cluster merge trees (tree.cuh), the B200 replacement for
//      LAPACK dgbsv (corrector.py:352)
//   6. back-substitution, hu replacement, hw update from the bottom pressure
//      (corrector.py:427-482)
//
// and pushes the final states of its H edge elements into the neighbours'
// halo slots through distributed shared memory.  Three cluster barriers per
// step (elimination, (h p) edge traces, halo).  The body is specialised per
// bottom model (template KIND) so each cluster runs a straight-line path.
// All arithmetic is fp64.
#include <cooperative_groups.h>
#include "bathy.cuh"
#include "physics.cuh"
#include "step_kernel.cuh"
#include "tree.cuh"

#ifndef NH_STAGE_UNROLL
#define NH_STAGE_UNROLL 1
#endif

// shared-memory field indices (SoA, each S doubles)
enum { F_H0 = 0, F_H1, F_Q0, F_Q1, F_W0, F_W1 };

struct Smem {
  double* Qn;     // 6*S  state at step start -> predictor -> final state
  double* Qs;     // 6*S  stage-1 state; later phi0, phi1, dx0, dx1, hp0, hp1
  double* Fx;     // 3*T  face exchange (F1, F2L, F3) of each thread's first face
  double* SK;     // 6*S  condensed super-element of each flagged slot
  double* AZ;     // 2*S  (a_{e-1}, z_{e+1}) of each flagged slot after the elimination
  short* flist;   // S    compacted list of flagged own slots
  int* wsum;      // W+1  per-warp flagged counts (prefix)
  uint8_t* raw;   // S    raw criterion flags
  int S, T, W;
};

size_t nh_step_smem_bytes(int threads, int E) {
  int S = threads * E, W = threads / 32;
  size_t dbl = 20 * (size_t)S + 3 * threads + W * 31 * 6 + W * 6 + W * 2 + 16 + 2 * 31 * 6;
  return dbl * 8 + W * 4 + (W + 1) * 4 + 2 * (size_t)S + S + 32;
}

__device__ __forceinline__ double& fld(double* base, int S, int f, int j) { return base[f * S + j]; }

// element derivative (grid.py:214-215) of a P1 pair, node i (numpy dgemm rounding)
__device__ __forceinline__ double elem_deriv(const nh_member& m, double v0, double v1, int i) {
  return RMUL(fma(v1, m.deriv_ref[2 * i + 1], RMUL(v0, m.deriv_ref[2 * i])), m.two_over_dx);
}

struct Tend6 {
  double v[6];
};

struct SideX {
  Side s;
  double sx;   // bottom slope at the node
};

#ifndef NH_KIND_TEMPLATE
#define NH_KIND_TEMPLATE 1
#endif

// bottom evaluation specialised at compile time (KIND >= 0) or dispatched at run time
template <int KIND, bool ALL>
__device__ __forceinline__ Bottom6 bot(const nh_member& m, const BottomTime& bt, double x) {
  if constexpr (KIND < 0) return bottom_eval_rt<ALL>(m, bt, x);
  else return bottom_eval<KIND, ALL>(m, bt, x);
}
template <int KIND>
__device__ __forceinline__ BottomTime bot_time(const nh_member& m, double t) {
  if constexpr (KIND < 0) return bottom_time(m, t);
  else return bottom_time_k<KIND>(m, t);
}

template <int KIND>
__device__ __forceinline__ SideX load_side(const nh_member& m, const BottomTime& bt,
                                           const double* src, int S, int j, double ed, int node) {
  Bottom6 b = bot<KIND, false>(m, bt, sample_xd(m, ed, node));
  SideX r;
  r.s = make_side(src[(F_H0 + node) * S + j], src[(F_Q0 + node) * S + j],
                  src[(F_W0 + node) * S + j], b.d);
  r.sx = b.d_x;
  return r;
}

// -------------------------------------------------------------------------
// One Heun stage over this thread's E slots.  Faces are streamed left to
// right; each thread publishes its first face for its left neighbour, and
// after one __syncthreads() the tendency of every slot is handed to `fn`
// (so `fn` may overwrite this thread's own slots of `src`).
// -------------------------------------------------------------------------
template <int E, int KIND, class Fn>
__device__ __forceinline__ double stage(const nh_member& m, double g, const double* src,
                                        const Smem& sm, int tid, int j0, int e0, double e0d,
                                        int N, int c0, int c1, const BottomTime& bt, Fn fn) {
  // speed: max over the left faces of own elements [c0, c1) and the right
  // ghost face (halo slots past the domain ends hold no state)
  const int S = sm.S;
  double speed = 0.0, sp;
  // carried state: the previous slot's two nodes and its left face
  SideX P0, P1;
  Face PF;
  Side Lprev;
  if (e0 == 0) {
    Lprev = load_side<KIND>(m, bt, src, S, j0, e0d, 0).s;
    Lprev = ghost_side(Lprev, m.bc_left);
  } else {
    int jp = j0 > 0 ? j0 - 1 : 0;
    Lprev = load_side<KIND>(m, bt, src, S, jp, e0d - 1.0, 1).s;
  }
#if NH_STAGE_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
  for (int k = 0; k < E; ++k) {
    SideX B0 = load_side<KIND>(m, bt, src, S, j0 + k, e0d + k, 0);
    SideX B1 = load_side<KIND>(m, bt, src, S, j0 + k, e0d + k, 1);
    Side L = (e0 + k == 0) ? ghost_side(B0.s, m.bc_left) : Lprev;
    Face Fk = face_flux<KIND == NH_BOTTOM_FLAT>(L, B0.s, g, sp);
    if (e0 + k >= c0 && e0 + k < c1) speed = fmax(speed, sp);
    if (k == 0) {
      sm.Fx[0 * sm.T + tid] = Fk.F1;
      sm.Fx[1 * sm.T + tid] = Fk.F2L;
      sm.Fx[2 * sm.T + tid] = Fk.F3;
    } else {
      Face Fr = Fk;
      if (e0 + k - 1 == N - 1) {
        Fr = face_flux<KIND == NH_BOTTOM_FLAT>(P1.s, ghost_side(P1.s, m.bc_right), g, sp);
        if (N - 1 >= c0 && N - 1 < c1) speed = fmax(speed, sp);
      }
      Tend6 td;
      element_tendency<KIND == NH_BOTTOM_FLAT>(m, g, P0.s, P1.s, PF, Fr, P0.sx, P1.sx, td.v);
      fn(k - 1, td);
    }
    P0 = B0; P1 = B1; PF = Fk; Lprev = B1.s;
  }
  __syncthreads();
  {
    Face fr;
    if (e0 + E - 1 == N - 1) {
      fr = face_flux<KIND == NH_BOTTOM_FLAT>(P1.s, ghost_side(P1.s, m.bc_right), g, sp);
      if (N - 1 >= c0 && N - 1 < c1) speed = fmax(speed, sp);
    } else {
      int tn = tid + 1 < sm.T ? tid + 1 : tid;
      fr.F1 = sm.Fx[0 * sm.T + tn];
      fr.F2L = sm.Fx[1 * sm.T + tn];
      fr.F3 = sm.Fx[2 * sm.T + tn];
      fr.F2R = 0.0;
    }
    Tend6 td;
    element_tendency<KIND == NH_BOTTOM_FLAT>(m, g, P0.s, P1.s, PF, fr, P0.sx, P1.sx, td.v);
    fn(E - 1, td);
  }
  return speed;
}

__device__ __forceinline__ double dsm_read(cg::cluster_group& cl, double* local, int rank) {
  return *cl.map_shared_rank(local, rank);
}

template <int E, int KIND>
__device__ __forceinline__ void member_steps(const StepArgs& a, cg::cluster_group& cluster,
                                             const nh_member& m, Smem& sm, TreeSmem& ts,
                                             const LdgConst& lk, double t) {
  const int C = a.cluster;
  const int rank = (int)cluster.block_rank();
  const int b = blockIdx.x / C;
  const int tid = threadIdx.x, T = blockDim.x, W = T >> 5, lane = tid & 31, warp = tid >> 5;
  const int S = sm.S;
  const int N = a.N;
  const int H = NH_HALO;
  const nh_scheme& sch = a.sch;
  const int tile = a.tile;
  const int c0 = rank * tile;
  const int c1 = min(c0 + tile, N);
  nh_status* st = a.status + b;
  const size_t base = (size_t)b * N * 2;
  const int j0 = tid * E;
  const int e0 = c0 - H + j0;
  const double e0d = (double)e0;
  const bool wcrit = (sch.criterion == NH_CRIT_W || sch.criterion == NH_CRIT_W_X) &&
                     sch.mode == NH_MODE_ADAPTIVE;
  const double dt = m.dt, hdt = 0.5 * dt;
  const double g = sch.g, c11 = sch.c11;
  const bool do_pred = sch.mode != NH_MODE_CORRECT_GIVEN;
  const bool do_corr = sch.mode != NH_MODE_HYDROSTATIC;

  double cfl_max = 0.0;
  long long flagged_sum = 0;
#if NH_PROFILE_PHASES
  long long prof[NH_NPHASE];
#pragma unroll
  for (int i = 0; i < NH_NPHASE; ++i) prof[i] = 0;
  long long tlast = clock64();
#define NH_TS(i) do { long long tc_ = clock64(); prof[i] += tc_ - tlast; tlast = tc_; } while (0)
#else
#define NH_TS(i) do { } while (0)
#endif

  for (int step = 0; step < a.n_steps; ++step) {
    const double t1 = do_pred ? t + dt : t;
    const BottomTime bt0 = bot_time<KIND>(m, t);
    const BottomTime bt1 = bot_time<KIND>(m, t1);
    // member-wide any(hw != 0) of this step's input (adaptivity.py:153)
    bool hw_any = true;
    if (wcrit) {
      hw_any = false;
      for (int r = 0; r < C; ++r) hw_any |= dsm_read(cluster, ts.pub + 7, r) != 0.0;
    }

    if (do_pred) {
      // ---------------- stage 1 at t: Qs = Q* = Qn + dt k1, k1 parked in SK ----------------
      double sp = stage<E, KIND>(m, g, sm.Qn, sm, tid, j0, e0, e0d, N, c0, c1, bt0,
                                 [&](int k, const Tend6 K1) {
        const double* k1 = K1.v;
        int j = j0 + k, e = e0 + k;
        bool own = e >= c0 && e < c1;
        double hn0 = fld(sm.Qn, S, F_H0, j), hn1 = fld(sm.Qn, S, F_H1, j);
        if (own && (hn0 <= 0.0 || hn1 <= 0.0)) nh_report(st, step, NH_ERR_POSITIVITY_ENTRY, e);
#pragma unroll
        for (int f = 0; f < 6; ++f) {
          fld(sm.Qs, S, f, j) = RADD(fld(sm.Qn, S, f, j), RMUL(dt, k1[f]));
          fld(sm.SK, S, f, j) = k1[f];
        }
        if (own && !(fld(sm.Qs, S, F_H0, j) > 0.0 && fld(sm.Qs, S, F_H1, j) > 0.0))
          nh_report(st, step, NH_ERR_POSITIVITY_STAGE1, -1);
      });
      if (sch.record_cfl) cfl_max = fmax(cfl_max, sp * dt / m.dx);
      __syncthreads();
      NH_TS(0);
      // ---------------- stage 2 at t + dt: Qn = Qn + dt (k1 + k2)/2 (hydrostatic.py:208-209)
      stage<E, KIND>(m, g, sm.Qs, sm, tid, j0, e0, e0d, N, c0, c1, bt1, [&](int k, const Tend6 K2) {
        const double* k2 = K2.v;
        int j = j0 + k, e = e0 + k;
#pragma unroll
        for (int f = 0; f < 6; ++f)
          fld(sm.Qn, S, f, j) =
              RADD(fld(sm.Qn, S, f, j), RMUL(dt, RMUL(0.5, RADD(fld(sm.SK, S, f, j), k2[f]))));
        if (e >= c0 && e < c1 &&
            !(fld(sm.Qn, S, F_H0, j) > 0.0 && fld(sm.Qn, S, F_H1, j) > 0.0))
          nh_report(st, step, NH_ERR_POSITIVITY_STAGE2, -1);
      });
      NH_TS(1);
    }

    if (do_corr) {
      // ---------------- criterion on the predictor (t+dt) ----------------
      const bool all = sch.mode == NH_MODE_GLOBAL || (wcrit && !hw_any);
      if (sch.mode == NH_MODE_ADAPTIVE && !all) {
#if NH_STAGE_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
        for (int k = 0; k < E; ++k) {
          int j = j0 + k, e = e0 + k;
          uint8_t fl = 0;
          if (e >= 0 && e < N) {
            double h0 = fld(sm.Qn, S, F_H0, j), h1 = fld(sm.Qn, S, F_H1, j);
            double v0, v1;
            switch (sch.criterion) {
              case NH_CRIT_ETA_OVER_D: {
                double d0 = bot<KIND, false>(m, bt1, sample_xd(m, e0d + k, 0)).d;
                double d1 = bot<KIND, false>(m, bt1, sample_xd(m, e0d + k, 1)).d;
                v0 = fabs(RDIVP(RSUB(h0, d0), d0)); v1 = fabs(RDIVP(RSUB(h1, d1), d1));
                break;
              }
              case NH_CRIT_ETA_X: {
                double d0 = bot<KIND, false>(m, bt1, sample_xd(m, e0d + k, 0)).d;
                double d1 = bot<KIND, false>(m, bt1, sample_xd(m, e0d + k, 1)).d;
                v0 = fabs(elem_deriv(m, RSUB(h0, d0), RSUB(h1, d1), 0));
                v1 = fabs(elem_deriv(m, RSUB(h0, d0), RSUB(h1, d1), 1));
                break;
              }
              case NH_CRIT_U:
                v0 = fabs(RDIVP(fld(sm.Qn, S, F_Q0, j), h0));
                v1 = fabs(RDIVP(fld(sm.Qn, S, F_Q1, j), h1));
                break;
              case NH_CRIT_U_X: {
                double u0 = RDIVP(fld(sm.Qn, S, F_Q0, j), h0);
                double u1 = RDIVP(fld(sm.Qn, S, F_Q1, j), h1);
                v0 = fabs(elem_deriv(m, u0, u1, 0)); v1 = fabs(elem_deriv(m, u0, u1, 1));
                break;
              }
              case NH_CRIT_W:
                v0 = fabs(RDIVP(fld(sm.Qn, S, F_W0, j), h0));
                v1 = fabs(RDIVP(fld(sm.Qn, S, F_W1, j), h1));
                break;
              default: {
                double w0 = RDIVP(fld(sm.Qn, S, F_W0, j), h0);
                double w1 = RDIVP(fld(sm.Qn, S, F_W1, j), h1);
                v0 = fabs(elem_deriv(m, w0, w1, 0)); v1 = fabs(elem_deriv(m, w0, w1, 1));
                break;
              }
            }
            fl = fmax(v0, v1) > sch.k_nh ? 1 : 0;
          }
          sm.raw[j] = fl;
        }
      } else if (sch.mode == NH_MODE_CORRECT_GIVEN) {
        const uint32_t* gb = a.given + (size_t)b * a.nwords;
#pragma unroll
        for (int k = 0; k < E; ++k) {
          int e = e0 + k;
          sm.raw[j0 + k] = (e >= 0 && e < N) ? ((gb[e >> 5] >> (e & 31)) & 1u) : 0;
        }
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k) {
          int e = e0 + k;
          sm.raw[j0 + k] = (e >= 0 && e < N) ? 1 : 0;
        }
      }
      __syncthreads();
      NH_TS(2);
      const bool enl = sch.mode == NH_MODE_ADAPTIVE && !all && sch.enlarge;
      auto eff = [&](int j) -> bool {
        int e = c0 - H + j;
        if (e < 0 || e >= N || j < 0 || j >= S) return false;
        bool f = sm.raw[j] != 0;
        if (enl) {
          if (e > 0 && j > 0) f = f || (sm.raw[j - 1] != 0);
          if (e < N - 1 && j + 1 < S) f = f || (sm.raw[j + 1] != 0);
        }
        return f;
      };

      // ---------------- compaction of the flagged own elements ----------------
      // Flagged elements are spread evenly over all threads of the CTA, so a
      // CTA with F flagged elements condenses them in ceil(F/T) rounds
      // instead of E rounds on whichever threads happen to own them.
      int myf = 0, nmy = 0;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        int j = j0 + k, e = e0 + k;
        if (e >= c0 && e < c1 && eff(j)) { myf |= 1 << k; ++nmy; }
      }
      const bool tflag = myf != 0;
      int incl = nmy;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) sm.wsum[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        int v = lane < W ? sm.wsum[lane] : 0, x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (lane < W) sm.wsum[lane] = x - v;          // exclusive warp offsets
        if (lane == W - 1) sm.wsum[W] = x;            // total
      }
      __syncthreads();
      {
        int pos = sm.wsum[warp] + incl - nmy;
#pragma unroll
        for (int k = 0; k < E; ++k)
          if (myf & (1 << k)) sm.flist[pos++] = (short)(j0 + k);
      }
      const int F = sm.wsum[W];
      flagged_sum += nmy;
      __syncthreads();

      // ---------------- condensation of the compacted elements ----------------
      Super Sc[E];
      double Rc[E][6];
      int jc[E];
#pragma unroll
      for (int r = 0; r < E; ++r) {
        int i = r * T + tid;
        jc[r] = i < F ? (int)sm.flist[i] : -1;
        if (jc[r] < 0) continue;
        const int j = jc[r], e = c0 - H + j;
        const double ed = (double)e;
        bool range_end = (e == N - 1) || !eff(j + 1);
        double h0 = fld(sm.Qn, S, F_H0, j), h1 = fld(sm.Qn, S, F_H1, j);
        Bottom6 b0 = bot<KIND, true>(m, bt1, sample_xd(m, ed, 0));
        Bottom6 b1 = bot<KIND, true>(m, bt1, sample_xd(m, ed, 1));
        Chan ch0{b0.d, b0.d_x, b0.d_t, b0.d_tt, b0.d_xt, b0.d_xx};
        Chan ch1{b1.d, b1.d_x, b1.d_t, b1.d_tt, b1.d_xt, b1.d_xx};
        NodeCoef q0 = ldg_coefficients(h0, fld(sm.Qn, S, F_Q0, j), fld(sm.Qn, S, F_W0, j),
                                       elem_deriv(m, h0, h1, 0),
                                       elem_deriv(m, h0 - b0.d, h1 - b1.d, 0), ch0, lk);
        NodeCoef q1 = ldg_coefficients(h1, fld(sm.Qn, S, F_Q1, j), fld(sm.Qn, S, F_W1, j),
                                       elem_deriv(m, h0, h1, 1),
                                       elem_deriv(m, h0 - b0.d, h1 - b1.d, 1), ch1, lk);
        fld(sm.Qs, S, 0, j) = q0.phi;
        fld(sm.Qs, S, 1, j) = q1.phi;
        fld(sm.Qs, S, 2, j) = b0.d_x;
        fld(sm.Qs, S, 3, j) = b1.d_x;
        bool ok = local_condense(m, q0, q1, lk.rho, lk.inv_rho, c11, range_end, Sc[r], Rc[r]);
        if (!ok) nh_report(st, step, NH_ERR_SOLVE_PIVOT, e);
        fld(sm.SK, S, 0, j) = Sc[r].ga; fld(sm.SK, S, 1, j) = Sc[r].aa;
        fld(sm.SK, S, 2, j) = Sc[r].ba; fld(sm.SK, S, 3, j) = Sc[r].gz;
        fld(sm.SK, S, 4, j) = Sc[r].az; fld(sm.SK, S, 5, j) = Sc[r].bz;
      }
      __syncthreads();
      NH_TS(3);

      // ---------------- elimination over the slot chain ----------------
      Super Sk[E];
#pragma unroll
      for (int k = 0; k < E; ++k) {
        int j = j0 + k, e = e0 + k;
        if (!(e >= c0 && e < c1)) {
          Sk[k] = super_identity();
        } else if (!(myf & (1 << k))) {
          Sk[k] = super_gap(fld(sm.Qn, S, F_Q0, j));
        } else {
          Sk[k] = Super{fld(sm.SK, S, 0, j), fld(sm.SK, S, 1, j), fld(sm.SK, S, 2, j),
                        fld(sm.SK, S, 3, j), fld(sm.SK, S, 4, j), fld(sm.SK, S, 5, j)};
        }
      }
      Super agg = chunk_aggregate<E>(Sk, tflag);
      // right-end ghost outer trace (corrector.py:400-402)
      if (N - 1 >= e0 && N - 1 < e0 + E && N - 1 >= c0 && N - 1 < c1) {
        int j = j0 + (N - 1 - e0);
        double q = fld(sm.Qn, S, F_Q1, j);
        ts.pub[6] = (m.bc_right == NH_BC_WALL) ? -q : q;
      }
      double a_in, z_in;
#if NH_PROFILE_PHASES
      prof[14] = clock64();
      tree_solve(cluster, ts, C, rank, W, warp, lane, tflag, F > 0, agg, a_in, z_in,
                 tid == 0 ? prof + 10 : nullptr);
#else
      tree_solve(cluster, ts, C, rank, W, warp, lane, tflag, F > 0, agg, a_in, z_in);
#endif
      NH_TS(4);
      if (tflag) {
        double aprev[E], znext[E];
        chunk_unwind<E>(Sk, a_in, z_in, aprev, znext);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if (!(myf & (1 << k))) continue;
          fld(sm.AZ, S, 0, j0 + k) = aprev[k];
          fld(sm.AZ, S, 1, j0 + k) = znext[k];
        }
      }
      // unflagged own slots carry p = 0
#pragma unroll
      for (int k = 0; k < E; ++k) {
        int j = j0 + k, e = e0 + k;
        if (e >= c0 && e < c1 && !(myf & (1 << k))) {
          fld(sm.Qs, S, 4, j) = 0.0;
          fld(sm.Qs, S, 5, j) = 0.0;
          if (step == a.n_steps - 1 && a.p_out) {
            size_t o = base + (size_t)e * 2;
            a.p_out[o] = 0.0;
            a.p_out[o + 1] = 0.0;
          }
        }
      }
      __syncthreads();
      // ---------------- reconstruction of the compacted elements ----------------
      double pk[E][2];
      ResidAcc ra{0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int r = 0; r < E; ++r) {
        pk[r][0] = 0.0; pk[r][1] = 0.0;
        if (jc[r] < 0) continue;
        const int j = jc[r], e = c0 - H + j;
        double P0, P1, Q0, Q1;
        const double ap = fld(sm.AZ, S, 0, j), zn = fld(sm.AZ, S, 1, j);
        reconstruct(Sc[r], Rc[r], ap, zn, c11, P0, P1, Q0, Q1);
        if (!isfinite(P0 + P1 + Q0 + Q1)) nh_report(st, step, NH_ERR_SOLVE_NONFINITE, e);
        {   // residual rows of the element (corrector.py:355-366): its
            // coefficients again from the predictor still in shared memory
          const double ed = (double)e;
          const double h0 = fld(sm.Qn, S, F_H0, j), h1 = fld(sm.Qn, S, F_H1, j);
          Bottom6 b0 = bot<KIND, true>(m, bt1, sample_xd(m, ed, 0));
          Bottom6 b1 = bot<KIND, true>(m, bt1, sample_xd(m, ed, 1));
          Chan ch0{b0.d, b0.d_x, b0.d_t, b0.d_tt, b0.d_xt, b0.d_xx};
          Chan ch1{b1.d, b1.d_x, b1.d_t, b1.d_tt, b1.d_xt, b1.d_xx};
          NodeCoef q0 = ldg_coefficients(h0, fld(sm.Qn, S, F_Q0, j), fld(sm.Qn, S, F_W0, j),
                                         elem_deriv(m, h0, h1, 0),
                                         elem_deriv(m, h0 - b0.d, h1 - b1.d, 0), ch0, lk);
          NodeCoef q1 = ldg_coefficients(h1, fld(sm.Qn, S, F_Q1, j), fld(sm.Qn, S, F_W1, j),
                                         elem_deriv(m, h0, h1, 1),
                                         elem_deriv(m, h0 - b0.d, h1 - b1.d, 1), ch1, lk);
          const bool rs = (e == 0) || !eff(j - 1), re = (e == N - 1) || !eff(j + 1);
          ldg_residual(m, q0, q1, lk.rho, lk.inv_rho, c11, rs, re, rs ? 0.0 : ap, zn, P0, Q0,
                       P1, Q1, ra);
        }
        pk[r][0] = lk.rho * P0; pk[r][1] = lk.rho * P1;
        fld(sm.Qn, S, F_Q0, j) = Q0;
        fld(sm.Qn, S, F_Q1, j) = Q1;
        fld(sm.Qs, S, 4, j) = fld(sm.Qn, S, F_H0, j) * pk[r][0];
        fld(sm.Qs, S, 5, j) = fld(sm.Qn, S, F_H1, j) * pk[r][1];
        if (step == a.n_steps - 1 && a.p_out) {
          size_t o = base + (size_t)e * 2;
          a.p_out[o] = pk[r][0];
          a.p_out[o + 1] = pk[r][1];
        }
      }
      resid_flush_warp(st, ra);   // the member's norms of this step's solve
      NH_TS(5);
      cluster.sync();   // ---- B3: (h p) traces visible to the neighbours
      NH_TS(6);
      if (rank == 0 && tid == 0) resid_check(st, step, a.sch.residual_tol);
      // hw update from the bottom pressure (corrector.py:441-482)
#pragma unroll
      for (int r = 0; r < E; ++r) {
        if (jc[r] < 0) continue;
        const int j = jc[r], e = c0 - H + j;
        double hp0 = fld(sm.Qs, S, 4, j), hp1 = fld(sm.Qs, S, 5, j);
        double hx0 = elem_deriv(m, hp0, hp1, 0), hx1 = elem_deriv(m, hp0, hp1, 1);
        if (e < N - 1) {
          double hr;
          if (e + 1 < c1) hr = fld(sm.Qs, S, 4, j + 1);
          else hr = dsm_read(cluster, sm.Qs + 4 * S + (e + 1 - (rank + 1) * tile + H), rank + 1);
          double avg = 0.5 * (hp1 + hr);
          hx0 += (avg - hp1) * m.lift_right[0];
          hx1 += (avg - hp1) * m.lift_right[1];
        }
        if (e > 0) {
          double hl;
          if (e - 1 >= c0) hl = fld(sm.Qs, S, 5, j - 1);
          else hl = dsm_read(cluster, sm.Qs + 5 * S + (e - 1 - (rank - 1) * tile + H), rank - 1);
          double avg = 0.5 * (hl + hp0);
          hx0 -= (avg - hp0) * m.lift_left[0];
          hx1 -= (avg - hp0) * m.lift_left[1];
        }
        double dx0 = fld(sm.Qs, S, 2, j), dx1 = fld(sm.Qs, S, 3, j);
        double q0 = 4.0 + dx0 * dx0, q1 = 4.0 + dx1 * dx1;
        double bp0 = nh_div(6.0, q0) * pk[r][0] + nh_div(dx0, q0) * hx0 + fld(sm.Qs, S, 0, j);
        double bp1 = nh_div(6.0, q1) * pk[r][1] + nh_div(dx1, q1) * hx1 + fld(sm.Qs, S, 1, j);
        fld(sm.Qn, S, F_W0, j) += lk.cdt * bp0;
        fld(sm.Qn, S, F_W1, j) += lk.cdt * bp1;
        if (a.flag_bits) {
          uint32_t* fb = a.flag_bits + ((size_t)step * a.B + b) * a.nwords;
          atomicOr(fb + (e >> 5), 1u << (e & 31));
        }
      }
    }

    // ---------------- step end: halo push, member-wide any(hw) ----------------
    __syncthreads();
    // gauges: h is final once the predictor is done (the correction leaves it)
    for (int gi = tid; gi < a.n_gauges; gi += T) {
      const int node = a.gauge_nodes[gi], e = node >> 1;
      if (e >= c0 && e < c1)
        a.gauge_h[((size_t)step * a.B + b) * a.n_gauges + gi] =
            fld(sm.Qn, S, F_H0 + (node & 1), e - c0 + H);
    }
    NH_TS(7);
    if (C > 1) {
      const int per = H * 6;
      for (int idx = tid; idx < 2 * per; idx += T) {
        int side = idx / per, r6 = idx % per, q = r6 / 6, f = r6 % 6;
        if (side == 0 && rank > 0) {
          int e = c0 + q;
          if (e < c1) {
            double v = fld(sm.Qn, S, f, e - c0 + H);
            double* rp = cluster.map_shared_rank(sm.Qn, rank - 1);
            rp[f * S + (e - (rank - 1) * tile + H)] = v;
          }
        } else if (side == 1 && rank < C - 1) {
          int e = c1 - H + q;
          if (e >= c0) {
            double v = fld(sm.Qn, S, f, e - c0 + H);
            double* rp = cluster.map_shared_rank(sm.Qn, rank + 1);
            rp[f * S + (e - (rank + 1) * tile + H)] = v;
          }
        }
      }
    }
    if (wcrit) {
      bool any = false;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        int j = j0 + k, e = e0 + k;
        if (e >= c0 && e < c1)
          any |= (fld(sm.Qn, S, F_W0, j) != 0.0) || (fld(sm.Qn, S, F_W1, j) != 0.0);
      }
      any = __syncthreads_or(any);
      if (tid == 0) ts.pub[7] = any ? 1.0 : 0.0;
    }
    NH_TS(8);
    cluster.sync();   // ---- B1: halos and flags in place for the next step
    NH_TS(9);
    t = t1;
  }
#if NH_PROFILE_PHASES
  if (tid == 0 && a.prof) {
#pragma unroll
    for (int i = 0; i < NH_NPHASE; ++i) a.prof[blockIdx.x * NH_NPHASE + i] = prof[i];
  }
#endif

  // ---------------- store the member tile ----------------
  for (int j = tid; j < S; j += T) {
    int e = c0 - H + j;
    if (e < c0 || e >= c1) continue;
    size_t o = base + (size_t)e * 2;
    a.h[o] = fld(sm.Qn, S, F_H0, j);
    a.h[o + 1] = fld(sm.Qn, S, F_H1, j);
    a.hu[o] = fld(sm.Qn, S, F_Q0, j);
    a.hu[o + 1] = fld(sm.Qn, S, F_Q1, j);
    a.hw[o] = fld(sm.Qn, S, F_W0, j);
    a.hw[o + 1] = fld(sm.Qn, S, F_W1, j);
  }
  unsigned long long fs = (unsigned long long)flagged_sum;
  double cm = cfl_max;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    fs += __shfl_down_sync(0xffffffffu, fs, o);
    cm = fmax(cm, __shfl_down_sync(0xffffffffu, cm, o));
  }
  if (lane == 0) {
    atomicAdd((unsigned long long*)&st->flagged, fs);
    atomicMax((unsigned long long*)&st->cfl_max, (unsigned long long)__double_as_longlong(cm));
  }
  if (rank == 0 && tid == 0) {
    a.time[b] = t;
    st->steps_done += a.n_steps;
  }
}

template <int E, int MAXT>
__global__ void __launch_bounds__(MAXT) nh_step_kernel(StepArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int C = a.cluster;
  const int rank = (int)cluster.block_rank();
  const int b = blockIdx.x / C;
  const int tid = threadIdx.x, T = blockDim.x, W = T >> 5;
  const int S = T * E;
  const int N = a.N;
  const int H = NH_HALO;
  const int c0 = rank * a.tile;
  const int c1 = min(c0 + a.tile, N);

  __shared__ nh_member msh;
  __shared__ LdgConst ksh;
  extern __shared__ __align__(16) double smem_raw[];
  Smem sm;
  sm.S = S; sm.T = T; sm.W = W;
  sm.Qn = smem_raw;
  sm.Qs = sm.Qn + 6 * S;
  sm.Fx = sm.Qs + 6 * S;
  TreeSmem ts;
  ts.wnode = sm.Fx + 3 * T;
  ts.wagg = ts.wnode + W * 31 * 6;
  ts.wio = ts.wagg + W * 6;
  ts.pub = ts.wio + W * 2;
  ts.bnode = ts.pub + 16;
  ts.cnode = ts.bnode + 31 * 6;
  sm.SK = ts.cnode + 31 * 6;
  sm.AZ = sm.SK + 6 * S;
  ts.wflag = (int*)(sm.AZ + 2 * S);
  sm.wsum = ts.wflag + W;
  sm.flist = (short*)(sm.wsum + W + 1);
  sm.raw = (uint8_t*)(sm.flist + S);

  if (tid == 0) {
    msh = a.members[b];
    ksh = make_ldg_const(msh.dt, a.sch.g, a.sch.rho);
  }
  const size_t base = (size_t)b * N * 2;
  for (int j = tid; j < S; j += T) {
    int e = c0 - H + j;
    bool in = (e >= 0) && (e < N) && (e < c1 + H);
    size_t o = base + (size_t)(in ? e : 0) * 2;
    fld(sm.Qn, S, F_H0, j) = in ? a.h[o] : 1.0;
    fld(sm.Qn, S, F_H1, j) = in ? a.h[o + 1] : 1.0;
    fld(sm.Qn, S, F_Q0, j) = in ? a.hu[o] : 0.0;
    fld(sm.Qn, S, F_Q1, j) = in ? a.hu[o + 1] : 0.0;
    fld(sm.Qn, S, F_W0, j) = in ? a.hw[o] : 0.0;
    fld(sm.Qn, S, F_W1, j) = in ? a.hw[o + 1] : 0.0;
#pragma unroll
    for (int f = 0; f < 6; ++f) fld(sm.Qs, S, f, j) = (f < 2) ? 1.0 : 0.0;
    sm.raw[j] = 0;
  }
  const double t = a.time[b];
  __syncthreads();
  {
    bool any = false;
    for (int j = tid; j < S; j += T) {
      int e = c0 - H + j;
      if (e >= c0 && e < c1)
        any |= (fld(sm.Qn, S, F_W0, j) != 0.0) || (fld(sm.Qn, S, F_W1, j) != 0.0);
    }
    any = __syncthreads_or(any);
    if (tid == 0) { ts.pub[7] = any ? 1.0 : 0.0; ts.pub[6] = 0.0; }
  }
  cluster.sync();
#if NH_KIND_TEMPLATE
  switch (msh.bottom_kind) {
    case NH_BOTTOM_FLAT: member_steps<E, NH_BOTTOM_FLAT>(a, cluster, msh, sm, ts, ksh, t); break;
    case NH_BOTTOM_PLATE: member_steps<E, NH_BOTTOM_PLATE>(a, cluster, msh, sm, ts, ksh, t); break;
    case NH_BOTTOM_QUARTIC_SLIDE:
      member_steps<E, NH_BOTTOM_QUARTIC_SLIDE>(a, cluster, msh, sm, ts, ksh, t); break;
    case NH_BOTTOM_SMOOTH_BOX:
      member_steps<E, NH_BOTTOM_SMOOTH_BOX>(a, cluster, msh, sm, ts, ksh, t); break;
    default:
      member_steps<E, NH_BOTTOM_SLOPE_SLIDE>(a, cluster, msh, sm, ts, ksh, t); break;
  }
#else
  member_steps<E, -1>(a, cluster, msh, sm, ts, ksh, t);
#endif
}

template __global__ void nh_step_kernel<3, 384>(StepArgs);
template __global__ void nh_step_kernel<1, 1024>(StepArgs);
template __global__ void nh_step_kernel<1, 512>(StepArgs);
template __global__ void nh_step_kernel<2, 512>(StepArgs);

// variants: 0 = (E 3, <=384 threads), 1 = (E 1, <=1024), 2 = (E 1, <=512), 3 = (E 2, <=512)
void* nh_step_kernel_ptr(int v) {
  switch (v) {
    case 1: return (void*)nh_step_kernel<1, 1024>;
    case 2: return (void*)nh_step_kernel<1, 512>;
    case 3: return (void*)nh_step_kernel<2, 512>;
    default: return (void*)nh_step_kernel<3, 384>;
  }
}
int nh_step_variant_E(int v) { return v == 1 || v == 2 ? 1 : v == 3 ? 2 : 3; }
int nh_step_variant_maxt(int v) { return v == 1 ? 1024 : v == 2 || v == 3 ? 512 : 384; }
