// Streaming (HBM round-trip) time step for large ensembles.
//
// One element per thread, 128-thread CTAs over tiles of OWN = 120 elements
// plus a halo of H = 4 on each side, all CTAs independent (no clusters), so
// the SMs run many CTAs at full occupancy.  Per step:
//
//   K_P  (tile)    stream_kp.cu: load the tile + halo (coalesced double2 per
//                  field), finish the previous step's correction in registers
//                  -- the vertical-momentum update needs the solved pressure
//                  of the neighbours, so it is fused into the NEXT step's load
//                  ("corrector fused with the next predictor") -- then both
//                  Heun stages (hydrostatic.py:192-209), the criterion with
//                  +-1 enlargement (adaptivity.py:75-113), the flags, the
//                  per-tile flagged count and the work list of flagged tiles.
//   K_S  (flagged tiles, one warp per tile) LDG coefficients at t + dt
//                  (corrector.py:100-170) stored for K_C, the per-element
//                  condensation (corrector.py:173-349 -> physics.cuh) and the
//                  tile's merged super-element.  Global mode: fused into K_P.
//   K_X  (member)  one warp per member merges its tiles' super-elements and
//                  hands every tile its boundary inputs (a_in, z_in); time,
//                  step counter, next step's bottom-time constants, residual
//                  gate of the previous solve.
//   K_C  (flagged tiles) element blocks re-eliminated, warp / CTA merge trees
//                  down to the elements, hu replacement, pressure p, residual
//                  shares (corrector.py:355-366).
//   K_fin (after the loop, stream_kp.cu) the last pending hw update on the
//                  flagged tiles of the last step.
//
// The launches of a step pair and the ping-pong of buffers are captured in a
// CUDA graph by nh_stream_advance (capi.cu).
#include "stream_kp.cuh"




// ---------------------------------------------------------------------- K_S
// Tiles holding flagged elements: LDG coefficients at t+dt and the per-element
// condensation (corrector.py:100-349 -> physics.cuh), stored for K_C, and the
// tile's merged super-element for K_X.
template <int KIND>
__device__ __forceinline__ void ks_body(const StreamArgs& a, int bt, const nh_member& m,
                                        const LdgConst& lk, const BottomTime& bt1, KsSmem& ks) {
  const int N = a.N, T = a.tiles;
  const int b = bt / T, tile = bt % T;
  const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
  const int e = tile * OWN - H + i;
  const bool valid = e >= 0 && e < N;
  const bool own = valid && i >= H && i < H + OWN;
  const size_t o = ((size_t)b * N + (valid ? e : 0)) * 2;
  const size_t fe = (size_t)b * N + (valid ? e : 0);
  const bool flag = own && a.flags_cur[fe];
  Super S = super_identity();
  if (own) S = super_gap(a.hu_out[o]);
  if (flag) {
    double2 vh = *reinterpret_cast<const double2*>(a.h_out + o);
    double2 vq = *reinterpret_cast<const double2*>(a.hu_out + o);
    double2 vw = *reinterpret_cast<const double2*>(a.hw_out + o);
    const bool range_end = (e == N - 1) || !a.flags_cur[fe + 1];
    condense_element<KIND>(a, m, lk, bt1, b, e, Q6{vh.x, vh.y, vq.x, vq.y, vw.x, vw.y},
                           range_end, S);
  }
  Super v = tile_up(S, flag, ks.wnode, ks.wagg, ks.bnode, ks.wflag, lane, warp);
  if (i == 0) store_super(a.tile_agg + ((size_t)b * T + tile) * 8, v);
}

#ifndef NH_KS_WARP
#define NH_KS_WARP 1   // 1: one warp per tile, no CTA barriers (0: one CTA per tile)
#endif

#if NH_KS_WARP
// One warp per tile: the tile's NW slices of 32 elements one after another,
// each reduced by the same warp tree as tile_up's per-warp level, then the
// slice aggregates by tile_up's cross-warp tree -- the same merges in the same
// order, so the tile aggregate is bitwise the CTA version's, without a CTA
// barrier: the warps of a CTA work on different tiles independently.
struct KsWarpSmem {
  nh_member msh;
  MemberConst mc;
  double wnode[31 * 6];
  double wagg[NW * 6];
};

template <int KIND>
__device__ __forceinline__ void ks_warp_tile(const StreamArgs& a, int bt, KsWarpSmem& ws, int lane) {
  const int N = a.N, T = a.tiles;
  const int b = bt / T, tile = bt % T;
  const nh_member& m = ws.msh;
  for (int c = 0; c < NW; ++c) {
    const int i = c * 32 + lane;
    const int e = tile * OWN - H + i;
    const bool valid = e >= 0 && e < N;
    const bool own = valid && i >= H && i < H + OWN;
    const size_t o = ((size_t)b * N + (valid ? e : 0)) * 2;
    const size_t fe = (size_t)b * N + (valid ? e : 0);
    const bool flag = own && a.flags_cur[fe];
    Super S = super_identity();
    if (own) S = super_gap(a.hu_out[o]);
    if (flag) {
      double2 vh = *reinterpret_cast<const double2*>(a.h_out + o);
      double2 vq = *reinterpret_cast<const double2*>(a.hu_out + o);
      double2 vw = *reinterpret_cast<const double2*>(a.hw_out + o);
      const bool range_end = (e == N - 1) || !a.flags_cur[fe + 1];
      condense_element<KIND>(a, m, ws.mc.lk, ws.mc.bt1, b, e, Q6{vh.x, vh.y, vq.x, vq.y, vw.x, vw.y},
                             range_end, S);
    }
    Super agg = S;   // tile_up's per-warp level
    if (__any_sync(0xffffffffu, flag)) {
      agg = warp_up<false>(agg, ws.wnode, lane, 5);   // K_S never sweeps down: no tree nodes
    } else {
      unsigned nonid = __ballot_sync(0xffffffffu, !is_identity(agg));
      int first = nonid ? __ffs(nonid) - 1 : 0;
      agg = shfl_super(agg, first);
      if (!nonid) agg = super_identity();
    }
    if (lane == 0) store_super(ws.wagg + c * 6, agg);
    __syncwarp();
  }
  Super v = lane < NW ? load_super(ws.wagg + lane * 6) : super_identity();
  v = warp_up<false>(v, ws.wnode, lane, NWL);   // tile_up's cross-warp level
  if (lane == 0) store_super(a.tile_agg + ((size_t)b * T + tile) * 8, v);
}

__global__ void __launch_bounds__(TPB, NH_KS_MIN_BLOCKS) nh_stream_ks(StreamArgs a) {
  __shared__ KsWarpSmem wsm[NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  KsWarpSmem& ws = wsm[warp];
  const bool all = a.sch.mode == NH_MODE_GLOBAL;
  const int n = all ? a.B * a.tiles : *a.tile_count;
  constexpr int MW = (int)(sizeof(nh_member) / 8);
  for (int w = blockIdx.x * NW + warp; w < n; w += gridDim.x * NW) {
    const int bt = all ? w : a.tile_list[w];
    const int b = bt / a.tiles;
    __syncwarp();   // the previous tile's reads of the member record are done
    for (int k = lane; k < MW + 16; k += 32) {
      if (k < MW)
        reinterpret_cast<unsigned long long*>(&ws.msh)[k] =
            reinterpret_cast<const unsigned long long*>(a.members + b)[k];
      else
        reinterpret_cast<unsigned long long*>(&ws.mc)[k - MW] =
            reinterpret_cast<const unsigned long long*>(a.mconst + (size_t)b * 16)[k - MW];
    }
    __syncwarp();
    switch (ws.msh.bottom_kind) {
      case NH_BOTTOM_FLAT: ks_warp_tile<NH_BOTTOM_FLAT>(a, bt, ws, lane); break;
      case NH_BOTTOM_PLATE: ks_warp_tile<NH_BOTTOM_PLATE>(a, bt, ws, lane); break;
      case NH_BOTTOM_QUARTIC_SLIDE: ks_warp_tile<NH_BOTTOM_QUARTIC_SLIDE>(a, bt, ws, lane); break;
      case NH_BOTTOM_SMOOTH_BOX: ks_warp_tile<NH_BOTTOM_SMOOTH_BOX>(a, bt, ws, lane); break;
      default: ks_warp_tile<NH_BOTTOM_SLOPE_SLIDE>(a, bt, ws, lane); break;
    }
  }
}
#else
// Persistent: the grid strides over the step's list of flagged tiles (or over
// every tile in global mode, where all are flagged and the list is skipped).
__global__ void __launch_bounds__(TPB, NH_KS_MIN_BLOCKS) nh_stream_ks(StreamArgs a) {
  __shared__ nh_member msh;
  __shared__ MemberConst mc;
  __shared__ KsSmem ks;
  const bool all = a.sch.mode == NH_MODE_GLOBAL;
  const int n = all ? a.B * a.tiles : *a.tile_count;
  for (int w = blockIdx.x; w < n; w += gridDim.x) {
    const int bt = all ? w : a.tile_list[w];
    const int b = bt / a.tiles;
    load_member(a, b, msh, mc);
    __syncthreads();
    switch (msh.bottom_kind) {
      case NH_BOTTOM_FLAT: ks_body<NH_BOTTOM_FLAT>(a, bt, msh, mc.lk, mc.bt1, ks); break;
      case NH_BOTTOM_PLATE: ks_body<NH_BOTTOM_PLATE>(a, bt, msh, mc.lk, mc.bt1, ks); break;
      case NH_BOTTOM_QUARTIC_SLIDE: ks_body<NH_BOTTOM_QUARTIC_SLIDE>(a, bt, msh, mc.lk, mc.bt1, ks); break;
      case NH_BOTTOM_SMOOTH_BOX: ks_body<NH_BOTTOM_SMOOTH_BOX>(a, bt, msh, mc.lk, mc.bt1, ks); break;
      default: ks_body<NH_BOTTOM_SLOPE_SLIDE>(a, bt, msh, mc.lk, mc.bt1, ks); break;
    }
    __syncthreads();   // shared memory is reused by the next tile
  }
}
#endif

// ---------------------------------------------------------------------- K_X
// One warp per member: chain of its T tile aggregates (lane l folds tiles
// [l*cpl, (l+1)*cpl)), merge tree across lanes, back-substitution, then each
// tile's (a_in, z_in).  Also advances the member's time and step counter.
// 9 warps per CTA: warps 0-7 run the tile chains of 8 members; lanes 0-7 of
// warp 8 advance the same 8 members' time and step constants concurrently.
__global__ void __launch_bounds__(288) nh_stream_kx(StreamArgs a) {
  __shared__ double nodes[8][31 * 6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0 && a.tile_count_next) *a.tile_count_next = 0;
  if (warp == 8) {
    const int b = blockIdx.x * 8 + lane;
    if (lane >= 8 || b >= a.B) return;
    const nh_member& m = a.members[b];
    // residual gate of the previous step's solve (its K_C ran before this K_X)
    if (a.sch.mode != NH_MODE_HYDROSTATIC && a.step_counter)
      resid_check(a.status + b, a.step_counter[b] - 1, a.sch.residual_tol);
    const double tn = a.time[b] + m.dt;
    a.time[b] = tn;
    if (a.step_counter) a.step_counter[b] += 1;
    // next step's constants: its bt0 = bottom_time(tn) is this step's bt1
    // (the same call on the same argument, t + dt); only bt1 is new
    MemberConst* mc = reinterpret_cast<MemberConst*>(a.mconst + (size_t)b * 16);
    mc->bt0 = mc->bt1;
    mc->bt1 = bottom_time(m, tn + m.dt);
    return;
  }
  const int b = blockIdx.x * 8 + warp;
  if (b >= a.B) return;
  const int T = a.tiles;
  const int cpl = (T + 31) / 32;
  const double* ta = a.tile_agg + (size_t)b * T * 8;
  double* io = a.tile_io + (size_t)b * T * 2;
  // this lane's tiles: flagged counts and the folded aggregate in one pass
  const int k0 = lane * cpl, k1 = min(k0 + cpl, T);
  bool any = false;
  Super agg = super_identity();
  for (int k = k0; k < k1; ++k) {
    any |= ta[k * 8 + 6] > 0.0;
    agg = merge2(agg, load_super(ta + k * 8));
  }
  if (__any_sync(0xffffffffu, any)) {
    warp_up(agg, nodes[warp], lane, 5);
    double a_in = 0.0, z_in = ta[(T - 1) * 8 + 7];
    warp_down(a_in, z_in, nodes[warp], lane, 5);
    // unwind this lane's tiles (Riccati sweep, exact elimination)
    double s = a_in, tt = 0.0;
    double sv[NH_STREAM_MAXCPL], tv[NH_STREAM_MAXCPL], mv[NH_STREAM_MAXCPL], nv[NH_STREAM_MAXCPL];
    for (int k = k0; k < k1; ++k) {
      sv[k - k0] = s; tv[k - k0] = tt;
      riccati_step(load_super(ta + k * 8), s, tt, mv[k - k0], nv[k - k0]);
    }
    double z = z_in;
    for (int k = k1 - 1; k >= k0; --k) {
      io[k * 2 + 1] = z;
      z = fma(nv[k - k0], z, mv[k - k0]);
      io[k * 2 + 0] = fma(tv[k - k0], z, sv[k - k0]);
    }
  }
}

// ---------------------------------------------------------------------- K_F
// w / w_x criterion: a member whose step input has hw == 0 everywhere is
// corrected globally for that step (adaptivity.py:153-154), so the indicator
// can activate.  K_P flags by the criterion and records any(hw != 0) of the
// input per member (hw_any); this kernel gives the all-zero members the full
// mask before K_S: every element flagged (flags, flag bits, flagged count) and
// every tile not yet on the work list appended to it.  One warp per member.
__global__ void __launch_bounds__(256) nh_stream_kf(StreamArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * 8 + warp;
  if (b >= a.B) return;
  int any = 0;
  if (lane == 0) {
    any = a.hw_any[b];
    a.hw_any[b] = 0;   // K_P of the next step records it afresh
  }
  if (__shfl_sync(0xffffffffu, any, 0)) return;
  const int N = a.N, T = a.tiles;
  double* ta = a.tile_agg + (size_t)b * T * 8;
  unsigned long long had = 0;
  for (int k = lane; k < T; k += 32) {
    const double nf = ta[k * 8 + 6];
    had += (unsigned long long)nf;
    if (nf == 0.0) a.tile_list[atomicAdd(a.tile_count, 1)] = b * T + k;
    ta[k * 8 + 6] = (double)min(OWN, N - k * OWN);
  }
  for (int o = 16; o > 0; o >>= 1) had += __shfl_xor_sync(0xffffffffu, had, o);
  uint8_t* fl = a.flags_cur + (size_t)b * N;
  for (int e = lane; e < N; e += 32) fl[e] = 1;
  if (a.flag_bits) {
    const int nw = (N + 31) / 32, step = a.step_counter ? a.step_counter[b] : 0;
    uint32_t* fb = a.flag_bits + ((size_t)step * a.B + b) * nw;
    for (int w = lane; w < nw; w += 32)
      fb[w] = (w == nw - 1 && (N & 31)) ? ((1u << (N & 31)) - 1u) : 0xffffffffu;
  }
  if (lane == 0 && (unsigned long long)N > had)
    atomicAdd((unsigned long long*)&a.status[b].flagged, (unsigned long long)N - had);
}

// Step constants of every member at its current time (before the first step).
__global__ void __launch_bounds__(256) nh_stream_prep(StreamArgs a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < a.B) member_const(a.members[b], a.sch, a.time[b], a.mconst + (size_t)b * 16);
}

// Gauges after K_P: h of this step (the correction leaves h unchanged) at
// every gauge node of every member, into row step_counter[b] (K_X advances
// it later in the step, so graph replays need no step argument).
__global__ void __launch_bounds__(128) nh_stream_gauge(StreamArgs a) {
  const size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (k >= (size_t)a.B * a.n_gauges) return;
  const int b = (int)(k / a.n_gauges), gi = (int)(k % a.n_gauges);
  const int step = a.step_counter[b];
  a.gauge_h[((size_t)step * a.B + b) * a.n_gauges + gi] =
      a.h_out[(size_t)b * a.N * 2 + a.gauge_nodes[gi]];
}

// Members grouped by bottom kind (stable within a kind), one 1024-thread CTA.
__global__ void __launch_bounds__(1024) nh_stream_order(StreamArgs a) {
  __shared__ int wsum[32];
  __shared__ int base;
  const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
  if (i == 0) base = 0;
  __syncthreads();
  for (int kind = 0; kind <= NH_BOTTOM_SLOPE_SLIDE + 1; ++kind) {
    for (int c = 0; c < a.B; c += 1024) {
      const int b = c + i;
      int k = b < a.B ? a.members[b].bottom_kind : -1;
      if (k < 0 || k > NH_BOTTOM_SLOPE_SLIDE) k = NH_BOTTOM_SLOPE_SLIDE + 1;
      const bool mine = b < a.B && k == kind;
      const unsigned bal = __ballot_sync(0xffffffffu, mine);
      if (lane == 0) wsum[warp] = __popc(bal);
      __syncthreads();
      int pre = 0, tot = 0;
      for (int w = 0; w < 32; ++w) { pre += w < warp ? wsum[w] : 0; tot += wsum[w]; }
      if (mine) const_cast<int*>(a.order)[base + pre + __popc(bal & ((1u << lane) - 1u))] = b;
      __syncthreads();
      if (i == 0) base += tot;
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------- K_C
struct KcSmem {
  double wnode[NW * 31 * 6];
  double wagg[NW * 6];
  double bnode[31 * 6];
  double wio[NW * 2];
};

__device__ __forceinline__ void kc_tile(const StreamArgs& a, int bt, KcSmem& kc) {
  double* wnode = kc.wnode;
  double* wagg = kc.wagg;
  double* bnode = kc.bnode;
  double* wio = kc.wio;
  const int N = a.N, T = a.tiles;
  const int b = bt / T, tile = bt % T;
  const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
  const int e = tile * OWN - H + i;
  const bool valid = e >= 0 && e < N;
  const bool own = valid && i >= H && i < H + OWN;
  const size_t o = ((size_t)b * N + (valid ? e : 0)) * 2;
  const size_t fe = (size_t)b * N + (valid ? e : 0);
  // global mode flags every element: no dependent flag load before the scratch loads
  const bool gmode = a.sch.mode == NH_MODE_GLOBAL;
  const bool flag = own && (gmode || a.flags_cur[fe]);
  const nh_member& m = a.members[b];
  const double rho = a.sch.rho, inv_rho = 1.0 / rho, c11 = a.sch.c11;
  Super S = super_identity();
  double R[6] = {0, 0, 0, 0, 0, 0};
  bool range_start = false, range_end = false;
  if (flag) {
    // re-eliminate the element block from K_S's coefficients: the same
    // super-element K_S aggregated, plus the reconstruction rows
    NodeCoef c0, c1;
    load_coef(a.scratch + fe, (size_t)a.B * N, c0, c1);
    range_start = e == 0 || !(gmode || a.flags_cur[fe - 1]);
    range_end = e == N - 1 || !(gmode || a.flags_cur[fe + 1]);
    local_condense(m, c0, c1, rho, inv_rho, c11, range_end, S, R);
  } else if (own) {
    S = super_gap(a.hu_out[o]);
  }
  // up: the same trees K_S built (recomputed from the super-elements)
  const bool wany = __any_sync(0xffffffffu, flag);
  double* wn = wnode + warp * 31 * 6;
  Super agg = S;
  if (wany) {
    agg = warp_up(agg, wn, lane, 5);
  } else {
    unsigned nonid = __ballot_sync(0xffffffffu, !is_identity(agg));
    int first = nonid ? __ffs(nonid) - 1 : 0;
    agg = shfl_super(agg, first);
    if (!nonid) agg = super_identity();
  }
  if (lane == 0) store_super(wagg + warp * 6, agg);
  __syncthreads();
  if (warp == 0) {
    Super v = lane < NW ? load_super(wagg + lane * 6) : super_identity();
    warp_up(v, bnode, lane, NWL);
    const double* io = a.tile_io + ((size_t)b * T + tile) * 2;
    double ai = lane == 0 ? io[0] : 0.0, zi = lane == 0 ? io[1] : 0.0;
    warp_down(ai, zi, bnode, lane, NWL);
    if (lane < NW) { wio[lane * 2] = ai; wio[lane * 2 + 1] = zi; }
  }
  __syncthreads();
  if (!wany) return;   // warp-uniform
  double a_in = wio[warp * 2], z_in = wio[warp * 2 + 1];
  warp_down(a_in, z_in, wn, lane, 5);
  ResidAcc ra{0.0, 0.0, 0.0, 0.0};
  if (flag) {
    double P0, P1, Q0, Q1;
    reconstruct(S, R, a_in, z_in, c11, P0, P1, Q0, Q1);
    const int step = a.step_counter ? a.step_counter[b] - 1 : 0;
    if (!isfinite(P0 + P1 + Q0 + Q1)) nh_report(a.status + b, step, NH_ERR_SOLVE_NONFINITE, e);
    NodeCoef c0, c1;   // reloaded (L1 / L2) rather than held across the trees
    load_coef(a.scratch + fe, (size_t)a.B * N, c0, c1);
    ldg_residual(m, c0, c1, rho, inv_rho, c11, range_start, range_end,
                 range_start ? 0.0 : a_in, z_in, P0, Q0, P1, Q1, ra);
    *reinterpret_cast<double2*>(a.hu_out + o) = double2{Q0, Q1};
    double* pn = a.pend_out + fe;
    pn[0] = rho * P0;
    pn[(size_t)a.B * N] = rho * P1;
  }
  resid_flush_warp(a.status + b, ra);   // the member's norms of this step's solve
}

// Persistent: the grid strides over the step's list of flagged tiles.
__global__ void __launch_bounds__(TPB, NH_KS_MIN_BLOCKS) nh_stream_kc(StreamArgs a) {
  __shared__ KcSmem kc;
  const bool all = a.sch.mode == NH_MODE_GLOBAL;
  const int n = all ? a.B * a.tiles : *a.tile_count;
  // the next tile's list entry is requested while the current tile runs: one
  // dependent global load less at the head of every tile (K_C -2 %; the same
  // in K_S measured +4 % on config 5, profiles/r2_ab_tile_prefetch.txt)
  int bt = (!all && (int)blockIdx.x < n) ? a.tile_list[blockIdx.x] : 0;
  for (int w = blockIdx.x; w < n; w += gridDim.x) {
    const int wn = w + gridDim.x;
    const int nxt = (!all && wn < n) ? a.tile_list[wn] : 0;
    kc_tile(a, all ? w : bt, kc);
    bt = nxt;
    __syncthreads();   // shared memory is reused by the next tile
  }
}

__global__ void nh_gather_p_kernel(const double* pend, const uint8_t* flags, double* p, size_t n) {
  size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  bool f = flags[k];
  p[2 * k] = f ? pend[k] : 0.0;             // planes p0, p1 of the pending record
  p[2 * k + 1] = f ? pend[n + k] : 0.0;
}

int nh_launch_gather_p(const double* pend, const uint8_t* flags, double* p, size_t n,
                       cudaStream_t s) {
  nh_gather_p_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(pend, flags, p, n);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

void* nh_stream_kernel(int which) {
  switch (which) {
    case 0: return nh_stream_kp_ptr();
    case 1: return (void*)nh_stream_kx;
    case 3: return (void*)nh_stream_ks;
    case 4: return (void*)nh_stream_prep;
    case 5: return (void*)nh_stream_order;
    case 6: return (void*)nh_stream_gauge;
    case 7: return (void*)nh_stream_kf;
    default: return (void*)nh_stream_kc;
  }
}
