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
//   5. segmented elimination of the flagged ranges: thread chunk -> warp
//      (shuffle tree) -> CTA (smem chain) -> cluster (DSMEM chain), the
//      B200 replacement for LAPACK dgbsv (corrector.py:352)
//   6. back-substitution, hu replacement, hw update from the bottom pressure
//      (corrector.py:427-482)
//
// and pushes the final states of its H edge elements into the neighbours'
// halo slots through distributed shared memory.  Three cluster barriers per
// step (halo, elimination, (h p) edge traces); everything else is
// __syncthreads.  All arithmetic is fp64.
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
  double* wnode;  // W*31*6 warp merge tree
  double* wagg;   // W*6
  double* wio;    // W*2
  double* pub;    // 16 : CTA aggregate (0..5), right ghost z (6), any_hw (7), red (8..)
  uint8_t* raw;   // S  raw criterion flags
  int S, T, W;
};

size_t nh_step_smem_bytes(int threads, int E) {
  int S = threads * E, W = threads / 32;
  size_t dbl = 12 * (size_t)S + 3 * threads + W * 31 * 6 + W * 6 + W * 2 + 16;
  return dbl * 8 + S + 16;
}

__device__ __forceinline__ double& fld(double* base, int S, int f, int j) { return base[f * S + j]; }

// element derivative (grid.py:214-215) of a P1 pair, node i
__device__ __forceinline__ double elem_deriv(const nh_member& m, double v0, double v1, int i) {
  return fma(v1, m.deriv_ref[2 * i + 1], v0 * m.deriv_ref[2 * i]) * m.two_over_dx;
}

struct SideX {
  Side s;
  double sx;   // bottom slope at the node
};

__device__ __forceinline__ SideX load_side(const nh_member& m, const BottomTime& bt,
                                           const double* src, int S, int j, int e, int node) {
  double d, sx;
  bottom_d_dx(m, bt, sample_x(m, e, node), d, sx);
  SideX r;
  r.s = make_side(src[(F_H0 + node) * S + j], src[(F_Q0 + node) * S + j],
                  src[(F_W0 + node) * S + j], d);
  r.sx = sx;
  return r;
}

// -------------------------------------------------------------------------
// One Heun stage over this thread's E slots.  Faces are streamed left to
// right; each thread publishes its first face for its left neighbour, and
// after one __syncthreads() the tendency of every slot is handed to `fn`
// (so `fn` may overwrite this thread's own slots of `src`).
// -------------------------------------------------------------------------
template <int E, class Fn>
__device__ __forceinline__ double stage(const nh_member& m, double g, const double* src,
                                        const Smem& sm, int tid, int j0, int e0, int N, double t,
                                        Fn fn) {
  const int S = sm.S;
  BottomTime bt = bottom_time(m, t);
  double speed = 0.0, sp;
  double tend[E][6];
  SideX A0 = load_side(m, bt, src, S, j0, e0, 0);
  SideX A1 = load_side(m, bt, src, S, j0, e0, 1);
  Face FL;
  {
    Side L;
    if (e0 == 0) {
      L = ghost_side(A0.s, m.bc_left);
    } else {
      int jp = j0 > 0 ? j0 - 1 : 0;
      L = load_side(m, bt, src, S, jp, e0 - 1, 1).s;
    }
    FL = face_flux(L, A0.s, g, sp);
    speed = fmax(speed, sp);
  }
  sm.Fx[0 * sm.T + tid] = FL.F1;
  sm.Fx[1 * sm.T + tid] = FL.F2L;
  sm.Fx[2 * sm.T + tid] = FL.F3;
#pragma unroll
  for (int k = 1; k < E; ++k) {
    SideX B0 = load_side(m, bt, src, S, j0 + k, e0 + k, 0);
    SideX B1 = load_side(m, bt, src, S, j0 + k, e0 + k, 1);
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
    element_tendency(m, g, A0.s, A1.s, FL, Fr, A0.sx, A1.sx, tend[k - 1]);
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
    element_tendency(m, g, A0.s, A1.s, FL, fr, A0.sx, A1.sx, tend[E - 1]);
  }
#pragma unroll
  for (int k = 0; k < E; ++k) fn(k, tend[k]);
  return speed;
}

__device__ __forceinline__ double dsm_read(cg::cluster_group& cl, double* local, int rank) {
  return *cl.map_shared_rank(local, rank);
}

template <int E>
__global__ void __launch_bounds__(NH_STEP_MAX_THREADS) nh_step_kernel(StepArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int C = a.cluster;
  const int rank = (int)cluster.block_rank();
  const int b = blockIdx.x / C;
  const int tid = threadIdx.x, T = blockDim.x, W = T >> 5, lane = tid & 31, warp = tid >> 5;
  const int S = T * E;
  const int N = a.N;
  const int H = NH_HALO;
  __shared__ nh_member msh;
  __shared__ double chain[4 * (NH_MAX_CLUSTER + 32)];
  if (tid == 0) msh = a.members[b];
  const nh_member& m = msh;
  const nh_scheme& sch = a.sch;
  const int tile = a.tile;
  const int c0 = rank * tile;
  const int c1 = min(c0 + tile, N);
  nh_status* st = a.status + b;

  extern __shared__ __align__(16) double smem_raw[];
  Smem sm;
  sm.S = S; sm.T = T; sm.W = W;
  sm.Qn = smem_raw;
  sm.Qs = sm.Qn + 6 * S;
  sm.Fx = sm.Qs + 6 * S;
  sm.wnode = sm.Fx + 3 * T;
  sm.wagg = sm.wnode + W * 31 * 6;
  sm.wio = sm.wagg + W * 6;
  sm.pub = sm.wio + W * 2;
  sm.raw = (uint8_t*)(sm.pub + 16);
  TreeSmem ts{sm.wnode, sm.wagg, sm.wio, sm.pub, chain};

  const size_t base = (size_t)b * N * 2;
  const int j0 = tid * E;              // first slot of this thread
  const int e0 = c0 - H + j0;          // its element

  // ---------------- load the member tile (+halo) ----------------
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
  double t = a.time[b];
  const bool wcrit = (sch.criterion == NH_CRIT_W || sch.criterion == NH_CRIT_W_X) &&
                     sch.mode == NH_MODE_ADAPTIVE;
  __syncthreads();
  {
    bool any = false;
    for (int j = tid; j < S; j += T) {
      int e = c0 - H + j;
      if (e >= c0 && e < c1)
        any |= (fld(sm.Qn, S, F_W0, j) != 0.0) || (fld(sm.Qn, S, F_W1, j) != 0.0);
    }
    any = __syncthreads_or(any);
    if (tid == 0) { sm.pub[7] = any ? 1.0 : 0.0; sm.pub[6] = 0.0; }
  }
  cluster.sync();

  double cfl_max = 0.0;
  long long flagged_sum = 0;
  const double dt = m.dt;
  const double g = sch.g, rho = sch.rho, c11 = sch.c11;
  const bool do_pred = sch.mode != NH_MODE_CORRECT_GIVEN;
  const bool do_corr = sch.mode != NH_MODE_HYDROSTATIC;
  const double hdt = 0.5 * dt;

  for (int step = 0; step < a.n_steps; ++step) {
    const double t1 = do_pred ? t + dt : t;
    // member-wide any(hw != 0) of this step's input (adaptivity.py:153)
    bool hw_any = true;
    if (wcrit) {
      hw_any = false;
      for (int r = 0; r < C; ++r) hw_any |= dsm_read(cluster, sm.pub + 7, r) != 0.0;
    }

    if (do_pred) {
      // ---------------- stage 1 at t: Qs = Q*, Qn += dt/2 k1 ----------------
      double sp = stage<E>(m, g, sm.Qn, sm, tid, j0, e0, N, t, [&](int k, const double* k1) {
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
      stage<E>(m, g, sm.Qs, sm, tid, j0, e0, N, t1, [&](int k, const double* k2) {
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
        BottomTime bt1 = bottom_time(m, t1);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          int j = j0 + k, e = e0 + k;
          uint8_t fl = 0;
          if (e >= 0 && e < N) {
            double h0 = fld(sm.Qn, S, F_H0, j), h1 = fld(sm.Qn, S, F_H1, j);
            double v0, v1;
            switch (sch.criterion) {
              case NH_CRIT_ETA_OVER_D: {
                double d0 = bottom_depth(m, bt1, sample_x(m, e, 0));
                double d1 = bottom_depth(m, bt1, sample_x(m, e, 1));
                v0 = fabs((h0 - d0) / d0); v1 = fabs((h1 - d1) / d1);
                break;
              }
              case NH_CRIT_ETA_X: {
                double d0 = bottom_depth(m, bt1, sample_x(m, e, 0));
                double d1 = bottom_depth(m, bt1, sample_x(m, e, 1));
                v0 = fabs(elem_deriv(m, h0 - d0, h1 - d1, 0));
                v1 = fabs(elem_deriv(m, h0 - d0, h1 - d1, 1));
                break;
              }
              case NH_CRIT_U:
                v0 = fabs(fld(sm.Qn, S, F_Q0, j) / h0); v1 = fabs(fld(sm.Qn, S, F_Q1, j) / h1);
                break;
              case NH_CRIT_U_X: {
                double u0 = fld(sm.Qn, S, F_Q0, j) / h0, u1 = fld(sm.Qn, S, F_Q1, j) / h1;
                v0 = fabs(elem_deriv(m, u0, u1, 0)); v1 = fabs(elem_deriv(m, u0, u1, 1));
                break;
              }
              case NH_CRIT_W:
                v0 = fabs(fld(sm.Qn, S, F_W0, j) / h0); v1 = fabs(fld(sm.Qn, S, F_W1, j) / h1);
                break;
              default: {
                double w0 = fld(sm.Qn, S, F_W0, j) / h0, w1 = fld(sm.Qn, S, F_W1, j) / h1;
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
      {
        BottomTime bt1 = bottom_time(m, t1);
        int nflag = 0;
#pragma unroll
        for (int k = 0; k < E; ++k) {
          int j = j0 + k, e = e0 + k;
          bool own = e >= c0 && e < c1;
          flg[k] = own && eff(j);
          nflag += flg[k] ? 1 : 0;
#pragma unroll
          for (int q = 0; q < 6; ++q) R[k][q] = 0.0;
          if (!own) {
            Sk[k] = super_identity();
          } else if (!flg[k]) {
            Sk[k] = super_gap(fld(sm.Qn, S, F_Q0, j));
          } else {
            bool range_end = (e == N - 1) || !eff(j + 1);
            double h0 = fld(sm.Qn, S, F_H0, j), h1 = fld(sm.Qn, S, F_H1, j);
            Bottom6 b0 = bottom_all(m, bt1, sample_x(m, e, 0));
            Bottom6 b1 = bottom_all(m, bt1, sample_x(m, e, 1));
            Chan ch0{b0.d, b0.d_x, b0.d_t, b0.d_tt, b0.d_xt, b0.d_xx};
            Chan ch1{b1.d, b1.d_x, b1.d_t, b1.d_tt, b1.d_xt, b1.d_xx};
            NodeCoef q0 = ldg_coefficients(h0, fld(sm.Qn, S, F_Q0, j), fld(sm.Qn, S, F_W0, j),
                                           elem_deriv(m, h0, h1, 0),
                                           elem_deriv(m, h0 - b0.d, h1 - b1.d, 0), ch0, dt, g, rho);
            NodeCoef q1 = ldg_coefficients(h1, fld(sm.Qn, S, F_Q1, j), fld(sm.Qn, S, F_W1, j),
                                           elem_deriv(m, h0, h1, 1),
                                           elem_deriv(m, h0 - b0.d, h1 - b1.d, 1), ch1, dt, g, rho);
            fld(sm.Qs, S, 0, j) = q0.phi;
            fld(sm.Qs, S, 1, j) = q1.phi;
            fld(sm.Qs, S, 2, j) = b0.d_x;
            fld(sm.Qs, S, 3, j) = b1.d_x;
            bool ok = local_condense(m, q0, q1, rho, c11, range_end, Sk[k], R[k]);
            if (!ok) nh_report(st, step, NH_ERR_SOLVE_PIVOT, e);
          }
        }
        flagged_sum += nflag;
      }
      // chunk aggregate, then the cluster-wide elimination
      Super agg = Sk[0];
#pragma unroll
      for (int k = 1; k < E; ++k) agg = merge2(agg, Sk[k]);
      // right-end ghost outer trace (corrector.py:400-402)
      if (N - 1 >= e0 && N - 1 < e0 + E && N - 1 >= c0 && N - 1 < c1) {
        int j = j0 + (N - 1 - e0);
        double q = fld(sm.Qn, S, F_Q1, j);
        sm.pub[6] = (m.bc_right == NH_BC_WALL) ? -q : q;
      }
      double a_in, z_in;
      tree_solve(cluster, ts, C, rank, W, warp, lane, tid, agg, a_in, z_in);
      // chunk back-substitution and reconstruction
      double pk[E][2];
      {
        double aprev[E], znext[E];
        chunk_unwind<E>(Sk, a_in, z_in, aprev, znext);
        const bool last_step = (step == a.n_steps - 1);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          int j = j0 + k, e = e0 + k;
          pk[k][0] = 0.0; pk[k][1] = 0.0;
          if (flg[k]) {
            double P0, P1, Q0, Q1;
            reconstruct(Sk[k], R[k], aprev[k], znext[k], c11, P0, P1, Q0, Q1);
            if (!isfinite(P0 + P1 + Q0 + Q1)) nh_report(st, step, NH_ERR_SOLVE_NONFINITE, e);
            pk[k][0] = rho * P0; pk[k][1] = rho * P1;
            fld(sm.Qn, S, F_Q0, j) = Q0;
            fld(sm.Qn, S, F_Q1, j) = Q1;
          }
          bool own = e >= c0 && e < c1;
          if (own) {
            fld(sm.Qs, S, 4, j) = fld(sm.Qn, S, F_H0, j) * pk[k][0];
            fld(sm.Qs, S, 5, j) = fld(sm.Qn, S, F_H1, j) * pk[k][1];
            if (last_step && a.p_out) {
              size_t o = base + (size_t)e * 2;
              a.p_out[o] = pk[k][0];
              a.p_out[o + 1] = pk[k][1];
            }
          }
        }
      }
      cluster.sync();   // ---- B3: (h p) traces visible to the neighbours
      // hw update from the bottom pressure (corrector.py:441-482)
      {
        const double cdt = dt / rho;
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
          double qd0 = 4.0 + dx0 * dx0, qd1 = 4.0 + dx1 * dx1;
          double bp0 = (6.0 / qd0) * pk[k][0] + (dx0 / qd0) * hx0 + fld(sm.Qs, S, 0, j);
          double bp1 = (6.0 / qd1) * pk[k][1] + (dx1 / qd1) * hx1 + fld(sm.Qs, S, 1, j);
          fld(sm.Qn, S, F_W0, j) += cdt * bp0;
          fld(sm.Qn, S, F_W1, j) += cdt * bp1;
          if (a.flag_bits) {
            uint32_t* fb = a.flag_bits + ((size_t)step * a.B + b) * a.nwords;
            atomicOr(fb + (e >> 5), 1u << (e & 31));
          }
        }
      }
    }

    // ---------------- step end: halo push, member-wide any(hw) ----------------
    __syncthreads();
    {
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
      if (tid == 0) sm.pub[7] = any ? 1.0 : 0.0;
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
  // per-member counters
  {
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
}

template __global__ void nh_step_kernel<3>(StepArgs);
template __global__ void nh_step_kernel<2>(StepArgs);

void* nh_step_kernel_ptr(int E) {
  if (E == 2) return (void*)nh_step_kernel<2>;
  if (E == 3) return (void*)nh_step_kernel<3>;
  return nullptr;
}
