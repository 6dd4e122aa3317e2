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

// shared-memory field indices (SoA, each S doubles)
enum { F_H0 = 0, F_H1, F_Q0, F_Q1, F_W0, F_W1 };

struct Smem {
  double* Qn;     // 6*S  state at step start -> predictor -> final state
  double* Qs;     // 6*S  stage-1 state; later phi0, phi1, dx0, dx1, hp0, hp1
  double* Fx;     // 3*T  face exchange (F1, F2L, F3) of each thread's first face
  uint8_t* raw;   // S    raw criterion flags
  int S, T, W;
};

size_t nh_step_smem_bytes(int threads, int E) {
  int S = threads * E, W = threads / 32;
  size_t dbl = 12 * (size_t)S + 3 * threads + W * 31 * 6 + W * 6 + W * 2 + 16 + 2 * 31 * 6;
  return dbl * 8 + W * 4 + S + 16;
}

__device__ __forceinline__ double& fld(double* base, int S, int f, int j) { return base[f * S + j]; }

// element derivative (grid.py:214-215) of a P1 pair, node i
__device__ __forceinline__ double elem_deriv(const nh_member& m, double v0, double v1, int i) {
  return fma(v1, m.deriv_ref[2 * i + 1], v0 * m.deriv_ref[2 * i]) * m.two_over_dx;
}

struct Tend6 {
  double v[6];
};

struct SideX {
  Side s;
  double sx;   // bottom slope at the node
};

template <int KIND>
__device__ __forceinline__ SideX load_side(const nh_member& m, const BottomTime& bt,
                                           const double* src, int S, int j, double ed, int node) {
  Bottom6 b = bottom_eval<KIND, false>(m, bt, sample_xd(m, ed, node));
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
                                        int N, const BottomTime& bt, Fn fn) {
  const int S = sm.S;
  double speed = 0.0, sp;
  Tend6 tend[E];
  SideX A0 = load_side<KIND>(m, bt, src, S, j0, e0d, 0);
  SideX A1 = load_side<KIND>(m, bt, src, S, j0, e0d, 1);
  Face FL;
  {
    Side L;
    if (e0 == 0) {
      L = ghost_side(A0.s, m.bc_left);
    } else {
      int jp = j0 > 0 ? j0 - 1 : 0;
      L = load_side<KIND>(m, bt, src, S, jp, e0d - 1.0, 1).s;
    }
    FL = face_flux(L, A0.s, g, sp);
    speed = fmax(speed, sp);
  }
  sm.Fx[0 * sm.T + tid] = FL.F1;
  sm.Fx[1 * sm.T + tid] = FL.F2L;
  sm.Fx[2 * sm.T + tid] = FL.F3;
#pragma unroll
  for (int k = 1; k < E; ++k) {
    SideX B0 = load_side<KIND>(m, bt, src, S, j0 + k, e0d + k, 0);
    SideX B1 = load_side<KIND>(m, bt, src, S, j0 + k, e0d + k, 1);
    Face Fk, Fr;
    if (e0 + k == 0) {
      Fk = face_flux(ghost_side(B0.s, m.bc_left), B0.s, g, sp);
    } else {
      Fk = face_flux(A1.s, B0.s, g, sp);
    }
    speed = fmax(speed, sp);
    Fr = Fk;
    if (e0 + k - 1 == N - 1) {
      Fr = face_flux(A1.s, ghost_side(A1.s, m.bc_right), g, sp);
      speed = fmax(speed, sp);
    }
    element_tendency(m, g, A0.s, A1.s, FL, Fr, A0.sx, A1.sx, tend[k - 1].v);
    A0 = B0; A1 = B1; FL = Fk;
  }
  __syncthreads();
  {
    Face fr;
    if (e0 + E - 1 == N - 1) {
      fr = face_flux(A1.s, ghost_side(A1.s, m.bc_right), g, sp);
      speed = fmax(speed, sp);
    } else {
      int tn = tid + 1 < sm.T ? tid + 1 : tid;
      fr.F1 = sm.Fx[0 * sm.T + tn];
      fr.F2L = sm.Fx[1 * sm.T + tn];
      fr.F3 = sm.Fx[2 * sm.T + tn];
      fr.F2R = 0.0;
    }
    element_tendency(m, g, A0.s, A1.s, FL, fr, A0.sx, A1.sx, tend[E - 1].v);
  }
#pragma unroll
  for (int k = 0; k < E; ++k) fn(k, tend[k]);
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

  for (int step = 0; step < a.n_steps; ++step) {
    const double t1 = do_pred ? t + dt : t;
    const BottomTime bt0 = bottom_time_k<KIND>(m, t);
    const BottomTime bt1 = bottom_time_k<KIND>(m, t1);
    // member-wide any(hw != 0) of this step's input (adaptivity.py:153)
    bool hw_any = true;
    if (wcrit) {
      hw_any = false;
      for (int r = 0; r < C; ++r) hw_any |= dsm_read(cluster, ts.pub + 7, r) != 0.0;
    }

    if (do_pred) {
      // ---------------- stage 1 at t: Qs = Q*, Qn += dt/2 k1 ----------------
      double sp = stage<E, KIND>(m, g, sm.Qn, sm, tid, j0, e0, e0d, N, bt0,
                                 [&](int k, const Tend6 K1) {
        const double* k1 = K1.v;
        int j = j0 + k, e = e0 + k;
        bool own = e >= c0 && e < c1;
        double hn0 = fld(sm.Qn, S, F_H0, j), hn1 = fld(sm.Qn, S, F_H1, j);
        if (own && (hn0 <= 0.0 || hn1 <= 0.0)) nh_report(st, step, NH_ERR_POSITIVITY_ENTRY, e);
#pragma unroll
        for (int f = 0; f < 6; ++f) {
          double q = fld(sm.Qn, S, f, j);
          fld(sm.Qs, S, f, j) = q + dt * k1[f];
          fld(sm.Qn, S, f, j) = q + hdt * k1[f];
        }
        if (own && !(fld(sm.Qs, S, F_H0, j) > 0.0 && fld(sm.Qs, S, F_H1, j) > 0.0))
          nh_report(st, step, NH_ERR_POSITIVITY_STAGE1, -1);
      });
      if (sch.record_cfl) cfl_max = fmax(cfl_max, sp * dt / m.dx);
      __syncthreads();
      // ---------------- stage 2 at t + dt: Qn += dt/2 k2 ----------------
      stage<E, KIND>(m, g, sm.Qs, sm, tid, j0, e0, e0d, N, bt1, [&](int k, const Tend6 K2) {
        const double* k2 = K2.v;
        int j = j0 + k, e = e0 + k;
#pragma unroll
        for (int f = 0; f < 6; ++f) fld(sm.Qn, S, f, j) += hdt * k2[f];
        if (e >= c0 && e < c1 &&
            !(fld(sm.Qn, S, F_H0, j) > 0.0 && fld(sm.Qn, S, F_H1, j) > 0.0))
          nh_report(st, step, NH_ERR_POSITIVITY_STAGE2, -1);
      });
    }

    if (do_corr) {
      // ---------------- criterion on the predictor (t+dt) ----------------
      const bool all = sch.mode == NH_MODE_GLOBAL || (wcrit && !hw_any);
      if (sch.mode == NH_MODE_ADAPTIVE && !all) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
          int j = j0 + k, e = e0 + k;
          uint8_t fl = 0;
          if (e >= 0 && e < N) {
            double h0 = fld(sm.Qn, S, F_H0, j), h1 = fld(sm.Qn, S, F_H1, j);
            double v0, v1;
            switch (sch.criterion) {
              case NH_CRIT_ETA_OVER_D: {
                double d0 = bottom_eval<KIND, false>(m, bt1, sample_xd(m, e0d + k, 0)).d;
                double d1 = bottom_eval<KIND, false>(m, bt1, sample_xd(m, e0d + k, 1)).d;
                v0 = fabs((h0 - d0) * nh_rcp(d0)); v1 = fabs((h1 - d1) * nh_rcp(d1));
                break;
              }
              case NH_CRIT_ETA_X: {
                double d0 = bottom_eval<KIND, false>(m, bt1, sample_xd(m, e0d + k, 0)).d;
                double d1 = bottom_eval<KIND, false>(m, bt1, sample_xd(m, e0d + k, 1)).d;
                v0 = fabs(elem_deriv(m, h0 - d0, h1 - d1, 0));
                v1 = fabs(elem_deriv(m, h0 - d0, h1 - d1, 1));
                break;
              }
              case NH_CRIT_U:
                v0 = fabs(fld(sm.Qn, S, F_Q0, j) * nh_rcp(h0));
                v1 = fabs(fld(sm.Qn, S, F_Q1, j) * nh_rcp(h1));
                break;
              case NH_CRIT_U_X: {
                double u0 = fld(sm.Qn, S, F_Q0, j) * nh_rcp(h0);
                double u1 = fld(sm.Qn, S, F_Q1, j) * nh_rcp(h1);
                v0 = fabs(elem_deriv(m, u0, u1, 0)); v1 = fabs(elem_deriv(m, u0, u1, 1));
                break;
              }
              case NH_CRIT_W:
                v0 = fabs(fld(sm.Qn, S, F_W0, j) * nh_rcp(h0));
                v1 = fabs(fld(sm.Qn, S, F_W1, j) * nh_rcp(h1));
                break;
              default: {
                double w0 = fld(sm.Qn, S, F_W0, j) * nh_rcp(h0);
                double w1 = fld(sm.Qn, S, F_W1, j) * nh_rcp(h1);
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

      // ---------------- per-element condensation ----------------
      Super Sk[E];
      double R[E][6];
      bool flg[E];
      bool tflag = false;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        int j = j0 + k, e = e0 + k;
        bool own = e >= c0 && e < c1;
        flg[k] = own && eff(j);
        tflag = tflag || flg[k];
        flagged_sum += flg[k] ? 1 : 0;
#pragma unroll
        for (int q = 0; q < 6; ++q) R[k][q] = 0.0;
        if (!own) {
          Sk[k] = super_identity();
        } else if (!flg[k]) {
          Sk[k] = super_gap(fld(sm.Qn, S, F_Q0, j));
        } else {
          bool range_end = (e == N - 1) || !eff(j + 1);
          double h0 = fld(sm.Qn, S, F_H0, j), h1 = fld(sm.Qn, S, F_H1, j);
          Bottom6 b0 = bottom_eval<KIND, true>(m, bt1, sample_xd(m, e0d + k, 0));
          Bottom6 b1 = bottom_eval<KIND, true>(m, bt1, sample_xd(m, e0d + k, 1));
          Chan ch0{b0.d, b0.d_x, b0.d_t, b0.d_tt, b0.d_xt, b0.d_xx};
          Chan ch1{b1.d, b1.d_x, b1.d_t, b1.d_tt, b1.d_xt, b1.d_xx};
          double hx = elem_deriv(m, h0, h1, 0);
          double ex = elem_deriv(m, h0 - b0.d, h1 - b1.d, 0);
          NodeCoef q0 = ldg_coefficients(h0, fld(sm.Qn, S, F_Q0, j), fld(sm.Qn, S, F_W0, j),
                                         hx, ex, ch0, lk);
          NodeCoef q1 = ldg_coefficients(h1, fld(sm.Qn, S, F_Q1, j), fld(sm.Qn, S, F_W1, j),
                                         elem_deriv(m, h0, h1, 1),
                                         elem_deriv(m, h0 - b0.d, h1 - b1.d, 1), ch1, lk);
          fld(sm.Qs, S, 0, j) = q0.phi;
          fld(sm.Qs, S, 1, j) = q1.phi;
          fld(sm.Qs, S, 2, j) = b0.d_x;
          fld(sm.Qs, S, 3, j) = b1.d_x;
          bool ok = local_condense(m, q0, q1, lk.rho, lk.inv_rho, c11, range_end, Sk[k], R[k]);
          if (!ok) nh_report(st, step, NH_ERR_SOLVE_PIVOT, e);
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
      tree_solve(cluster, ts, C, rank, W, warp, lane, tflag, agg, a_in, z_in);
      // chunk back-substitution and reconstruction
      double pk[E][2];
      const bool last_step = (step == a.n_steps - 1);
#pragma unroll
      for (int k = 0; k < E; ++k) { pk[k][0] = 0.0; pk[k][1] = 0.0; }
      if (tflag) {
        double aprev[E], znext[E];
        chunk_unwind<E>(Sk, a_in, z_in, aprev, znext);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if (!flg[k]) continue;
          int j = j0 + k, e = e0 + k;
          double P0, P1, Q0, Q1;
          reconstruct(Sk[k], R[k], aprev[k], znext[k], c11, P0, P1, Q0, Q1);
          if (!isfinite(P0 + P1 + Q0 + Q1)) nh_report(st, step, NH_ERR_SOLVE_NONFINITE, e);
          pk[k][0] = lk.rho * P0; pk[k][1] = lk.rho * P1;
          fld(sm.Qn, S, F_Q0, j) = Q0;
          fld(sm.Qn, S, F_Q1, j) = Q1;
        }
      }
#pragma unroll
      for (int k = 0; k < E; ++k) {
        int j = j0 + k, e = e0 + k;
        if (e >= c0 && e < c1) {
          fld(sm.Qs, S, 4, j) = fld(sm.Qn, S, F_H0, j) * pk[k][0];
          fld(sm.Qs, S, 5, j) = fld(sm.Qn, S, F_H1, j) * pk[k][1];
          if (last_step && a.p_out) {
            size_t o = base + (size_t)e * 2;
            a.p_out[o] = pk[k][0];
            a.p_out[o + 1] = pk[k][1];
          }
        }
      }
      cluster.sync();   // ---- B3: (h p) traces visible to the neighbours
      // hw update from the bottom pressure (corrector.py:441-482)
      if (tflag) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if (!flg[k]) continue;
          int j = j0 + k, e = e0 + k;
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
          double r0 = nh_rcp(4.0 + dx0 * dx0), r1 = nh_rcp(4.0 + dx1 * dx1);
          double bp0 = (6.0 * r0) * pk[k][0] + (dx0 * r0) * hx0 + fld(sm.Qs, S, 0, j);
          double bp1 = (6.0 * r1) * pk[k][1] + (dx1 * r1) * hx1 + fld(sm.Qs, S, 1, j);
          fld(sm.Qn, S, F_W0, j) += lk.cdt * bp0;
          fld(sm.Qn, S, F_W1, j) += lk.cdt * bp1;
          if (a.flag_bits) {
            uint32_t* fb = a.flag_bits + ((size_t)step * a.B + b) * a.nwords;
            atomicOr(fb + (e >> 5), 1u << (e & 31));
          }
        }
      }
    }

    // ---------------- step end: halo push, member-wide any(hw) ----------------
    __syncthreads();
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
    cluster.sync();   // ---- B1: halos and flags in place for the next step
    t = t1;
  }

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

template <int E>
__global__ void __launch_bounds__(NH_STEP_MAX_THREADS) nh_step_kernel(StepArgs a) {
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
  ts.wflag = (int*)(ts.cnode + 31 * 6);
  sm.raw = (uint8_t*)(ts.wflag + W);

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
}

template __global__ void nh_step_kernel<3>(StepArgs);

void* nh_step_kernel_ptr(int E) { return E == 3 ? (void*)nh_step_kernel<3> : nullptr; }
