// K_P with two elements per thread (NH_KP_E2=1): the same tile of
// NH_STREAM_THREADS slots as K_S / K_C, computed by half as many threads.
// Each thread owns the element pair (2i, 2i+1) of the tile, so the face
// between them is local (no exchange), one shared-memory exchange per stage
// serves two elements, and the per-thread bookkeeping (indices, loads of the
// member record, CFL reduction, flags) is paid once per pair.  Arithmetic is
// operation for operation that of kp_body (stream_kp.cuh), so results are
// bit-identical to the one-element kernel.
#pragma once
#include "stream_kp.cuh"

namespace {

constexpr int TP2 = TPB / 2;   // threads of a K_P2 CTA

struct Kp2Smem {
  double sh[5 * TP2];    // node-1 side of each thread's second element; (h p) traces
  double sf[3 * TP2];    // left-face flux of each thread's first element
  double sk[12 * TP2];   // k1 of both elements
  double sq[12 * TP2];   // step-start state of both elements
  double cfl;            // max wave speed of the tile
  uint8_t rf[TPB];       // raw criterion flags per slot
};

// One Heun stage for the element pair (A, B) = (e0, e0 + 1).
template <int KIND>
__device__ __forceinline__ void stage_pair(const nh_member& m, double g, const Q6 (&q)[2],
                                           const BottomTime& bt, const double (&x)[4],
                                           const BottomSpace (&sp)[4], int i, int e0, int N,
                                           bool own0, bool own1, double* sh, double* sf,
                                           double (&t)[2][6], double& speed, double (&d)[4]) {
  constexpr bool LEVEL = KIND == NH_BOTTOM_FLAT;
  Bottom6 bb[4];
#pragma unroll
  for (int n = 0; n < 4; ++n) bb[n] = bottom_eval_sp_k<KIND>(m, bt, x[n], sp[n]);
  Side A0, A1, B0, B1;
  make_sides_warp(q[0].h0, q[0].q0, q[0].w0, bb[0].d, q[0].h1, q[0].q1, q[0].w1, bb[1].d, A0, A1);
  make_sides_warp(q[1].h0, q[1].q0, q[1].w0, bb[2].d, q[1].h1, q[1].q1, q[1].w1, bb[3].d, B0, B1);
  sh[0 * TP2 + i] = B1.h; sh[1 * TP2 + i] = B1.hu; sh[2 * TP2 + i] = B1.hw;
  sh[3 * TP2 + i] = B1.d; sh[4 * TP2 + i] = B1.u;
  __syncthreads();
  Side L;
  if (e0 == 0) {
    L = ghost_side(A0, m.bc_left);
  } else {   // the left thread's second element, node 1 (u included)
    const int k = i > 0 ? i - 1 : 0;
    L.h = sh[0 * TP2 + k]; L.hu = sh[1 * TP2 + k]; L.hw = sh[2 * TP2 + k];
    L.d = sh[3 * TP2 + k]; L.u = sh[4 * TP2 + k];
#if NH_STRICT
    L.rh = 0.0;
#else
    L.rh = nh_rcp(L.h);
#endif
  }
  double s;
  const Face fl = face_flux<LEVEL, true>(L, A0, g, s);
  if (own0) speed = fmax(speed, s);
  Face fm = face_flux<LEVEL, true>(A1, B0, g, s);   // local face between A and B
  if (own1) speed = fmax(speed, s);
  if (e0 == N - 1) {   // odd N: A is the last element, B lies past the domain
    fm = face_flux<LEVEL>(A1, ghost_side(A1, m.bc_right), g, s);
    if (own0) speed = fmax(speed, s);
  }
  sf[0 * TP2 + i] = fl.F1; sf[1 * TP2 + i] = fl.F2L; sf[2 * TP2 + i] = fl.F3;
  __syncthreads();
  Face fr;
  if (e0 + 1 == N - 1) {
    fr = face_flux<LEVEL>(B1, ghost_side(B1, m.bc_right), g, s);
    if (own1) speed = fmax(speed, s);
  } else {
    const int k = i < TP2 - 1 ? i + 1 : i;
    fr.F1 = sf[0 * TP2 + k]; fr.F2L = sf[1 * TP2 + k]; fr.F3 = sf[2 * TP2 + k]; fr.F2R = 0.0;
  }
  element_tendency<LEVEL>(m, g, A0, A1, fl, fm, bb[0].d_x, bb[1].d_x, t[0]);
  element_tendency<LEVEL>(m, g, B0, B1, fm, fr, bb[2].d_x, bb[3].d_x, t[1]);
#pragma unroll
  for (int n = 0; n < 4; ++n) d[n] = bb[n].d;
}

__device__ __forceinline__ double q6_get(const Q6& q, int f) {
  switch (f) {
    case 0: return q.h0;
    case 1: return q.h1;
    case 2: return q.q0;
    case 3: return q.q1;
    case 4: return q.w0;
    default: return q.w1;
  }
}

template <int KIND>
__device__ __forceinline__ void kp2_body(const StreamArgs& a, const nh_member& m,
                                         const MemberConst& mc, int b, int tile, Q6 (&q)[2],
                                         Kp2Smem& ks) {
  const int N = a.N, T = a.tiles;
  const int i = threadIdx.x, lane = i & 31;
  const int s0 = 2 * i;                      // first slot of the pair
  const int e0 = tile * OWN - H + s0;        // first element of the pair
  bool valid[2], own[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int e = e0 + k, s = s0 + k;
    valid[k] = e >= 0 && e < N;
    own[k] = valid[k] && s >= H && s < H + OWN;
  }
  const nh_scheme& sch = a.sch;
  const double g = sch.g;
  nh_status* st = a.status + b;
  const int step = a.step_counter ? a.step_counter[b] : 0;
  const double dt = m.dt;
  double x[4];
  BottomSpace sp[4];
#pragma unroll
  for (int n = 0; n < 4; ++n) {
    x[n] = sample_xd(m, (double)(e0 + (n >> 1)), n & 1);
    sp[n] = bottom_space_k<KIND>(m, x[n]);
  }
  double speed = 0.0;

  // ---------------- Heun stage 1 at t ----------------
  unsigned bad[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    bad[k] = (own[k] && (q[k].h0 <= 0.0 || q[k].h1 <= 0.0)) ? 1u : 0u;
#pragma unroll
    for (int f = 0; f < 6; ++f) ks.sq[(6 * k + f) * TP2 + i] = q6_get(q[k], f);
  }
  Q6 qs[2];
  {
    double k1[2][6], dd[4];
    stage_pair<KIND>(m, g, q, mc.bt0, x, sp, i, e0, N, own[0], own[1], ks.sh, ks.sf, k1, speed,
                     dd);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
#pragma unroll
      for (int f = 0; f < 6; ++f) ks.sk[(6 * k + f) * TP2 + i] = k1[k][f];
      qs[k] = Q6{RADD(q[k].h0, RMUL(dt, k1[k][0])), RADD(q[k].h1, RMUL(dt, k1[k][1])),
                 RADD(q[k].q0, RMUL(dt, k1[k][2])), RADD(q[k].q1, RMUL(dt, k1[k][3])),
                 RADD(q[k].w0, RMUL(dt, k1[k][4])), RADD(q[k].w1, RMUL(dt, k1[k][5]))};
      bad[k] |= (own[k] && !(qs[k].h0 > 0.0 && qs[k].h1 > 0.0)) ? 2u : 0u;
    }
  }
  __syncthreads();   // every read of sh / sf of stage 1 is done

  // ---------------- Heun stage 2 at t + dt ----------------
  double d[4];   // depth at t + dt at the four nodes, reused by the criterion
  Q6 qp[2];
  {
    double k2[2][6], dummy = 0.0;
    stage_pair<KIND>(m, g, qs, mc.bt1, x, sp, i, e0, N, false, false, ks.sh, ks.sf, k2, dummy, d);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      double qv[6];
#pragma unroll
      for (int f = 0; f < 6; ++f)
        qv[f] = RADD(ks.sq[(6 * k + f) * TP2 + i],
                     RMUL(dt, RMUL(0.5, RADD(ks.sk[(6 * k + f) * TP2 + i], k2[k][f]))));
      qp[k] = Q6{qv[0], qv[1], qv[2], qv[3], qv[4], qv[5]};
      bad[k] |= (own[k] && !(qp[k].h0 > 0.0 && qp[k].h1 > 0.0)) ? 4u : 0u;
    }
  }
  double& cfl_sh = ks.cfl;
  if (sch.record_cfl) {   // as kp_body: max over the warp on the bit patterns
    const unsigned long long u = (unsigned long long)__double_as_longlong(speed);
    const unsigned hi = __reduce_max_sync(0xffffffffu, (unsigned)(u >> 32));
    const unsigned lo = __reduce_max_sync(0xffffffffu, (unsigned)(u >> 32) == hi ? (unsigned)u : 0u);
    if (lane == 0 && (hi | lo))
      atomicMax((unsigned long long*)&cfl_sh, ((unsigned long long)hi << 32) | lo);
  }

  // ---------------- criterion on the predictor (t + dt) ----------------
  uint8_t raw[2] = {0, 0};
  if (sch.mode == NH_MODE_ADAPTIVE && sch.criterion == NH_CRIT_ETA_OVER_D) {
#if NH_STRICT
    bool badc = false;
    double v[2][2], ee[2][2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      ee[k][0] = RSUB(qp[k].h0, d[2 * k]);
      ee[k][1] = RSUB(qp[k].h1, d[2 * k + 1]);
      v[k][0] = fabs(nh_div_pos_fp(ee[k][0], d[2 * k], badc));
      v[k][1] = fabs(nh_div_pos_fp(ee[k][1], d[2 * k + 1], badc));
    }
    if (__any_sync(0xffffffffu, badc)) {   // NH_WARP_FIX for the four divisions
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        v[k][0] = fabs(RDIVP(ee[k][0], d[2 * k]));
        v[k][1] = fabs(RDIVP(ee[k][1], d[2 * k + 1]));
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) raw[k] = (valid[k] && fmax(v[k][0], v[k][1]) > sch.k_nh) ? 1 : 0;
#else
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      double v0 = fabs(RDIVP(RSUB(qp[k].h0, d[2 * k]), d[2 * k]));
      double v1 = fabs(RDIVP(RSUB(qp[k].h1, d[2 * k + 1]), d[2 * k + 1]));
      raw[k] = (valid[k] && fmax(v0, v1) > sch.k_nh) ? 1 : 0;
    }
#endif
  } else if (sch.mode != NH_MODE_HYDROSTATIC) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (!valid[k]) continue;
      if (sch.mode == NH_MODE_GLOBAL) { raw[k] = 1; continue; }
      const Q6& p = qp[k];
      const double da = d[2 * k], db = d[2 * k + 1];
      double v0, v1;
      switch (sch.criterion) {
        case NH_CRIT_ETA_OVER_D:
          v0 = fabs(RDIVP(RSUB(p.h0, da), da)); v1 = fabs(RDIVP(RSUB(p.h1, db), db));
          break;
        case NH_CRIT_ETA_X:
          v0 = fabs(ederiv(m, RSUB(p.h0, da), RSUB(p.h1, db), 0));
          v1 = fabs(ederiv(m, RSUB(p.h0, da), RSUB(p.h1, db), 1));
          break;
        case NH_CRIT_U:
          v0 = fabs(RDIVP(p.q0, p.h0)); v1 = fabs(RDIVP(p.q1, p.h1));
          break;
        case NH_CRIT_U_X: {
          double u0 = RDIVP(p.q0, p.h0), u1 = RDIVP(p.q1, p.h1);
          v0 = fabs(ederiv(m, u0, u1, 0)); v1 = fabs(ederiv(m, u0, u1, 1));
          break;
        }
        case NH_CRIT_W:
          v0 = fabs(RDIVP(p.w0, p.h0)); v1 = fabs(RDIVP(p.w1, p.h1));
          break;
        default: {
          double w0 = RDIVP(p.w0, p.h0), w1 = RDIVP(p.w1, p.h1);
          v0 = fabs(ederiv(m, w0, w1, 0)); v1 = fabs(ederiv(m, w0, w1, 1));
          break;
        }
      }
      raw[k] = fmax(v0, v1) > sch.k_nh ? 1 : 0;
    }
  }
  ks.rf[s0] = raw[0];
  ks.rf[s0 + 1] = raw[1];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    if (bad[k])   // the reference raises at the first failing check: lowest code wins
      nh_report(st, step,
                (bad[k] & 1u) ? NH_ERR_POSITIVITY_ENTRY
                              : ((bad[k] & 2u) ? NH_ERR_POSITIVITY_STAGE1 : NH_ERR_POSITIVITY_STAGE2),
                (bad[k] & 1u) ? e0 + k : -1);
  }
  const size_t o = ((size_t)b * N + (valid[0] ? e0 : 0)) * 2;   // pair base (4 doubles per field)
  if (own[0] && own[1]) {
    double* hp = a.h_out + o;
    double* qp_ = a.hu_out + o;
    double* wp = a.hw_out + o;
    *reinterpret_cast<double2*>(hp) = double2{qp[0].h0, qp[0].h1};
    *reinterpret_cast<double2*>(hp + 2) = double2{qp[1].h0, qp[1].h1};
    *reinterpret_cast<double2*>(qp_) = double2{qp[0].q0, qp[0].q1};
    *reinterpret_cast<double2*>(qp_ + 2) = double2{qp[1].q0, qp[1].q1};
    *reinterpret_cast<double2*>(wp) = double2{qp[0].w0, qp[0].w1};
    *reinterpret_cast<double2*>(wp + 2) = double2{qp[1].w0, qp[1].w1};
  } else {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (!own[k]) continue;
      const size_t ok = ((size_t)b * N + e0 + k) * 2;
      *reinterpret_cast<double2*>(a.h_out + ok) = double2{qp[k].h0, qp[k].h1};
      *reinterpret_cast<double2*>(a.hu_out + ok) = double2{qp[k].q0, qp[k].q1};
      *reinterpret_cast<double2*>(a.hw_out + ok) = double2{qp[k].w0, qp[k].w1};
    }
  }
  auto publish_cfl = [&]() {
    if (i == 0 && cfl_sh > 0.0) {
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
    bool f = ks.rf[s] != 0;
    if (enl) {
      if (ee > 0 && s > 0) f = f || ks.rf[s - 1];
      if (ee < N - 1 && s + 1 < TPB) f = f || ks.rf[s + 1];
    }
    return f;
  };
  bool flag[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    flag[k] = own[k] && eff(s0 + k);
    if (own[k]) a.flags_cur[(size_t)b * N + e0 + k] = flag[k] ? 1 : 0;
    if (flag[k] && a.flag_bits) {
      const int e = e0 + k;
      uint32_t* fb = a.flag_bits + ((size_t)step * a.B + b) * ((N + 31) / 32);
      atomicOr(fb + (e >> 5), 1u << (e & 31));
    }
  }
  {
    const int nf = __syncthreads_count(flag[0]) + __syncthreads_count(flag[1]);
    if (s0 == H) {   // first own slot (H even: the pair's first element)
      double* ta = a.tile_agg + ((size_t)b * T + tile) * 8;
      ta[6] = (double)nf;
      if (nf == 0) store_super(ta, super_gap(qp[0].q0));
      if (nf) {
        atomicAdd((unsigned long long*)&st->flagged, (unsigned long long)nf);
        a.tile_list[atomicAdd(a.tile_count, 1)] = b * T + tile;
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k)   // right-end ghost outer trace (corrector.py:400-402)
      if (e0 + k == N - 1 && own[k])
        a.tile_agg[((size_t)b * T + tile) * 8 + 7] =
            (m.bc_right == NH_BC_WALL) ? -qp[k].q1 : qp[k].q1;
  }
  publish_cfl();
}

// One K_P2 tile: loads, pending hw correction of the previous step, body.
__device__ __forceinline__ void kp2_tile(const StreamArgs& a, int b, int tile, nh_member& msh,
                                         MemberConst& mc, Kp2Smem& ks) {
  static_assert(H % 2 == 0, "pairs must not straddle the halo boundary");
  const int N = a.N, i = threadIdx.x;
  const int s0 = 2 * i, e0 = tile * OWN - H + s0;
  bool valid[2];
  Q6 q[2];
  bool f[2];
  double p[2][2], phi[2][2], dxs[2][2];
  const size_t BN = (size_t)a.B * N;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int e = e0 + k;
    valid[k] = e >= 0 && e < N;
    q[k] = Q6{1.0, 1.0, 0.0, 0.0, 0.0, 0.0};
    if (valid[k]) {
      const size_t o = ((size_t)b * N + e) * 2;
      double2 vh = *reinterpret_cast<const double2*>(a.h_in + o);
      double2 vq = *reinterpret_cast<const double2*>(a.hu_in + o);
      double2 vw = *reinterpret_cast<const double2*>(a.hw_in + o);
      q[k] = Q6{vh.x, vh.y, vq.x, vq.y, vw.x, vw.y};
    }
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int e = e0 + k;
    f[k] = a.pend && valid[k] && a.flags_prev[(size_t)b * N + e];
    p[k][0] = p[k][1] = phi[k][0] = phi[k][1] = dxs[k][0] = dxs[k][1] = 0.0;
    if (f[k]) {
      const double* pv = a.pend + (size_t)b * N + e;
      p[k][0] = pv[0]; p[k][1] = pv[BN]; phi[k][0] = pv[2 * BN]; phi[k][1] = pv[3 * BN];
      dxs[k][0] = pv[4 * BN]; dxs[k][1] = pv[5 * BN];
    }
  }
  load_member(a, b, msh, mc);
  double hp[2][2];
#pragma unroll
  for (int k = 0; k < 2; ++k) { hp[k][0] = q[k].h0 * p[k][0]; hp[k][1] = q[k].h1 * p[k][1]; }
  if (a.pend) {   // (h p) at the pair's outer nodes for the neighbouring threads
    ks.sh[0 * TP2 + i] = hp[0][0];   // first element, node 0
    ks.sh[1 * TP2 + i] = hp[1][1];   // second element, node 1
  }
  if (i == 0) ks.cfl = 0.0;
  __syncthreads();

  // ---------------- pending correction of the previous step (corrector.py:441-482) ----------------
  if (f[0] || f[1]) {
    // (h p) of the neighbour element on the other side of a face: inside the
    // pair from registers, across pairs from shared memory, outside the CTA's
    // slots (halo elements only) from global memory
    auto hp_glob = [&](int ee, int node) -> double {
      if (!a.flags_prev[(size_t)b * N + ee]) return 0.0;
      size_t oo = ((size_t)b * N + ee) * 2 + node;
      return a.h_in[oo] * a.pend[(size_t)node * BN + (size_t)b * N + ee];
    };
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (!f[k]) continue;
      const int e = e0 + k;
      double hx0 = ederiv(msh, hp[k][0], hp[k][1], 0), hx1 = ederiv(msh, hp[k][0], hp[k][1], 1);
      if (e < N - 1) {
        double hr = k == 0 ? hp[1][0] : (i + 1 < TP2 ? ks.sh[0 * TP2 + i + 1] : hp_glob(e + 1, 0));
        double avg = 0.5 * (hp[k][1] + hr);
        hx0 += (avg - hp[k][1]) * msh.lift_right[0];
        hx1 += (avg - hp[k][1]) * msh.lift_right[1];
      }
      if (e > 0) {
        double hl = k == 1 ? hp[0][1] : (i > 0 ? ks.sh[1 * TP2 + i - 1] : hp_glob(e - 1, 1));
        double avg = 0.5 * (hl + hp[k][0]);
        hx0 -= (avg - hp[k][0]) * msh.lift_left[0];
        hx1 -= (avg - hp[k][0]) * msh.lift_left[1];
      }
      double qd0 = 4.0 + dxs[k][0] * dxs[k][0], qd1 = 4.0 + dxs[k][1] * dxs[k][1];
      double bp0 = nh_div(6.0, qd0) * p[k][0] + nh_div(dxs[k][0], qd0) * hx0 + phi[k][0];
      double bp1 = nh_div(6.0, qd1) * p[k][1] + nh_div(dxs[k][1], qd1) * hx1 + phi[k][1];
      q[k].w0 += mc.lk.cdt * bp0;
      q[k].w1 += mc.lk.cdt * bp1;
    }
  }
  __syncthreads();   // every read of the (h p) traces done before sh is reused
  if (a.finalize) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int s = s0 + k;
      if (valid[k] && s >= H && s < H + OWN) {
        const size_t o = ((size_t)b * N + e0 + k) * 2;
        *reinterpret_cast<double2*>(const_cast<double*>(a.hw_in) + o) = double2{q[k].w0, q[k].w1};
      }
    }
    return;
  }
  switch (msh.bottom_kind) {
    case NH_BOTTOM_FLAT: kp2_body<NH_BOTTOM_FLAT>(a, msh, mc, b, tile, q, ks); break;
    case NH_BOTTOM_PLATE: kp2_body<NH_BOTTOM_PLATE>(a, msh, mc, b, tile, q, ks); break;
    case NH_BOTTOM_QUARTIC_SLIDE: kp2_body<NH_BOTTOM_QUARTIC_SLIDE>(a, msh, mc, b, tile, q, ks); break;
    case NH_BOTTOM_SMOOTH_BOX: kp2_body<NH_BOTTOM_SMOOTH_BOX>(a, msh, mc, b, tile, q, ks); break;
    default: kp2_body<NH_BOTTOM_SLOPE_SLIDE>(a, msh, mc, b, tile, q, ks); break;
  }
}

}  // namespace
