// Single-purpose kernels behind the reference's finer-grained entry points:
// rhs_operator, criterion_values, phi_term/assemble_coefficients,
// BathymetryModel.sample, correct_momentum and the coefficient-driven
// ldg_solve / solve_on_ranges.  The fused time step (step_kernel.cu) does not
// use these; they exist so every public function of the reference hot path
// has a device implementation of its own (no CPU fallback).
#include <algorithm>
#include <cooperative_groups.h>
#include "bathy.cuh"
#include "physics.cuh"
#include "step_kernel.cuh"
#include "tree.cuh"

namespace cg = cooperative_groups;

__device__ __forceinline__ double ed(const nh_member& m, double v0, double v1, int i) {
  return fma(v1, m.deriv_ref[2 * i + 1], v0 * m.deriv_ref[2 * i]) * m.two_over_dx;
}

// ---------------------------------------------------------------- rhs_operator
__global__ void nh_rhs_kernel(const nh_member* __restrict__ members, int B, int N,
                              const double* __restrict__ h, const double* __restrict__ hu,
                              const double* __restrict__ hw, const double* __restrict__ time,
                              double g, double* th, double* tq, double* tw, nh_status* status) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * N) return;
  int b = idx / N, e = idx % N;
  const nh_member& m = members[b];
  double t = time[b];
  BottomTime bt = bottom_time(m, t);
  size_t base = (size_t)b * N * 2;
  auto side = [&](int ee, int node, double& sx) {
    size_t o = base + (size_t)ee * 2 + node;
    double d;
    bottom_d_dx(m, bt, sample_x(m, ee, node), d, sx);
    return make_side(h[o], hu[o], hw[o], d);
  };
  double sx0, sx1, dummy, sp;
  Side n0 = side(e, 0, sx0), n1 = side(e, 1, sx1);
  if (h[base + 2 * e] <= 0.0 || h[base + 2 * e + 1] <= 0.0)
    nh_report(status + b, 0, NH_ERR_POSITIVITY_ENTRY, e);
  Side L = (e == 0) ? ghost_side(n0, m.bc_left) : side(e - 1, 1, dummy);
  Side R = (e == N - 1) ? ghost_side(n1, m.bc_right) : side(e + 1, 0, dummy);
  Face fl = face_flux(L, n0, g, sp);
  Face fr = face_flux(n1, R, g, sp);
  double t6[6];
  element_tendency(m, g, n0, n1, fl, fr, sx0, sx1, t6);
  size_t o = base + (size_t)e * 2;
  th[o] = t6[0]; th[o + 1] = t6[1];
  tq[o] = t6[2]; tq[o + 1] = t6[3];
  tw[o] = t6[4]; tw[o + 1] = t6[5];
}

// ------------------------------------------------------------ criterion_values
__global__ void nh_criterion_kernel(const nh_member* __restrict__ members, int B, int N,
                                    const double* __restrict__ h, const double* __restrict__ hu,
                                    const double* __restrict__ hw,
                                    const double* __restrict__ time, int kind, double* out) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * N) return;
  int b = idx / N, e = idx % N;
  const nh_member& m = members[b];
  size_t o = (size_t)idx * 2;
  double h0 = h[o], h1 = h[o + 1], v0, v1;
  if (kind == NH_CRIT_ETA_OVER_D || kind == NH_CRIT_ETA_X) {
    BottomTime bt = bottom_time(m, time[b]);
    double d0 = bottom_depth(m, bt, sample_x(m, e, 0));
    double d1 = bottom_depth(m, bt, sample_x(m, e, 1));
    if (kind == NH_CRIT_ETA_OVER_D) {
      v0 = fabs((h0 - d0) / d0); v1 = fabs((h1 - d1) / d1);
    } else {
      v0 = fabs(ed(m, h0 - d0, h1 - d1, 0)); v1 = fabs(ed(m, h0 - d0, h1 - d1, 1));
    }
  } else {
    const double* q = (kind == NH_CRIT_U || kind == NH_CRIT_U_X) ? hu : hw;
    double a0 = q[o] / h0, a1 = q[o + 1] / h1;
    if (kind == NH_CRIT_U || kind == NH_CRIT_W) {
      v0 = fabs(a0); v1 = fabs(a1);
    } else {
      v0 = fabs(ed(m, a0, a1, 0)); v1 = fabs(ed(m, a0, a1, 1));
    }
  }
  out[o] = v0; out[o + 1] = v1;
}

// --------------------------------------------------- phi_term + coefficients
__global__ void nh_coef_kernel(const nh_member* __restrict__ members, int B, int N,
                               const double* __restrict__ h, const double* __restrict__ hu,
                               const double* __restrict__ hw, const double* __restrict__ time,
                               double g, double rho, double* coef) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * N) return;
  int b = idx / N, e = idx % N;
  const nh_member& m = members[b];
  BottomTime bt = bottom_time(m, time[b]);
  size_t o = (size_t)idx * 2;
  size_t plane = (size_t)B * N * 2;
  double h0 = h[o], h1 = h[o + 1];
  Bottom6 b0 = bottom_all(m, bt, sample_x(m, e, 0));
  Bottom6 b1 = bottom_all(m, bt, sample_x(m, e, 1));
  Chan c[2] = {{b0.d, b0.d_x, b0.d_t, b0.d_tt, b0.d_xt, b0.d_xx},
               {b1.d, b1.d_x, b1.d_t, b1.d_tt, b1.d_xt, b1.d_xx}};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    NodeCoef q = ldg_coefficients(i ? h1 : h0, hu[o + i], hw[o + i], ed(m, h0, h1, i),
                                  ed(m, h0 - b0.d, h1 - b1.d, i), c[i], make_ldg_const(m.dt, g, rho));
    coef[0 * plane + o + i] = q.s11;
    coef[1 * plane + o + i] = q.s12;
    coef[2 * plane + o + i] = q.s22;
    coef[3 * plane + o + i] = q.f1;
    coef[4 * plane + o + i] = q.f2;
    coef[5 * plane + o + i] = q.phi;
    coef[6 * plane + o + i] = c[i].d_x;
  }
}

// ------------------------------------------------------- BathymetryModel.sample
__global__ void nh_bottom_kernel(const nh_member* __restrict__ members, int B,
                                 const double* __restrict__ x, int P,
                                 const double* __restrict__ time, double* out) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * P) return;
  int b = idx / P;
  const nh_member& m = members[b];
  BottomTime bt = bottom_time(m, time[b]);
  Bottom6 v = bottom_all(m, bt, x[idx]);
  size_t plane = (size_t)B * P;
  out[0 * plane + idx] = v.d;
  out[1 * plane + idx] = v.d_x;
  out[2 * plane + idx] = v.d_t;
  out[3 * plane + idx] = v.d_tt;
  out[4 * plane + idx] = v.d_xt;
  out[5 * plane + idx] = v.d_xx;
}

// ----------------------------------------------------------- correct_momentum
// hw += dt/rho * (6/quad p + d_x/quad (h p)_x + phi) on flagged elements,
// (h p)_x = element derivative + central-average lifting, p = 0 off ranges
// (corrector.py:427-482).
__global__ void nh_momentum_kernel(const nh_member* __restrict__ members, int B, int N,
                                   const double* __restrict__ h, const double* __restrict__ p,
                                   const double* __restrict__ coef,
                                   const uint32_t* __restrict__ flags, int nwords, double rho,
                                   const double* __restrict__ hw_in, double* hw_out) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * N) return;
  int b = idx / N, e = idx % N;
  const nh_member& m = members[b];
  size_t o = (size_t)idx * 2;
  size_t plane = (size_t)B * N * 2;
  const uint32_t* fb = flags + (size_t)b * nwords;
  bool f = (fb[e >> 5] >> (e & 31)) & 1u;
  if (!f) { hw_out[o] = hw_in[o]; hw_out[o + 1] = hw_in[o + 1]; return; }
  double hp0 = h[o] * p[o], hp1 = h[o + 1] * p[o + 1];
  double hx0 = ed(m, hp0, hp1, 0), hx1 = ed(m, hp0, hp1, 1);
  if (e < N - 1) {
    double hr = h[o + 2] * p[o + 2];
    double avg = 0.5 * (hp1 + hr);
    hx0 += (avg - hp1) * m.lift_right[0];
    hx1 += (avg - hp1) * m.lift_right[1];
  }
  if (e > 0) {
    double hl = h[o - 1] * p[o - 1];
    double avg = 0.5 * (hl + hp0);
    hx0 -= (avg - hp0) * m.lift_left[0];
    hx1 -= (avg - hp0) * m.lift_left[1];
  }
  double dx0 = coef[6 * plane + o], dx1 = coef[6 * plane + o + 1];
  double qd0 = 4.0 + dx0 * dx0, qd1 = 4.0 + dx1 * dx1;
  double bp0 = (6.0 / qd0) * p[o] + (dx0 / qd0) * hx0 + coef[5 * plane + o];
  double bp1 = (6.0 / qd1) * p[o + 1] + (dx1 / qd1) * hx1 + coef[5 * plane + o + 1];
  double cdt = m.dt / rho;
  hw_out[o] = hw_in[o] + cdt * bp0;
  hw_out[o + 1] = hw_in[o + 1] + cdt * bp1;
}

// ------------------------------------------------------------------- ldg_solve
size_t nh_solve_smem_bytes(int threads) {
  int W = threads / 32;
  return ((size_t)W * 31 * 6 + W * 6 + W * 2 + 16 + 2 * 31 * 6) * 8 + W * 4 + 16;
}

template <int E>
__global__ void __launch_bounds__(NH_STEP_MAX_THREADS) nh_solve_kernel(SolveArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  const int C = a.cluster, rank = (int)cluster.block_rank(), b = blockIdx.x / C;
  const int tid = threadIdx.x, T = blockDim.x, W = T >> 5, lane = tid & 31, warp = tid >> 5;
  const int N = a.N;
  const nh_member& m = a.members[b];
  const int c0 = rank * a.tile, c1 = min(c0 + a.tile, N);
  const int e0 = c0 + tid * E;
  extern __shared__ __align__(16) double sh[];
  TreeSmem ts;
  ts.wnode = sh;
  ts.wagg = ts.wnode + W * 31 * 6;
  ts.wio = ts.wagg + W * 6;
  ts.pub = ts.wio + W * 2;
  ts.bnode = ts.pub + 16;
  ts.cnode = ts.bnode + 31 * 6;
  ts.wflag = (int*)(ts.cnode + 31 * 6);
  const size_t plane = (size_t)a.B * N * 2;
  const uint32_t* fb = a.flags + (size_t)b * a.nwords;
  const uint32_t* sb = a.starts ? a.starts + (size_t)b * a.nwords : nullptr;
  auto flag = [&](int e) -> bool { return e >= 0 && e < N && ((fb[e >> 5] >> (e & 31)) & 1u); };
  // a range starts at e: e flagged and e - 1 not, or a caller-given start
  // inside a flagged run (adjacent ranges are separate systems, each with
  // P* = 0 at its ends -- the reference stacks them block-diagonally)
  auto start = [&](int e) -> bool {
    return flag(e) && (!flag(e - 1) || (sb && ((sb[e >> 5] >> (e & 31)) & 1u)));
  };
  const double* outer = a.outer_right + (size_t)b * N;
  const double inv_rho = 1.0 / a.rho;
  auto load_q = [&](int e, NodeCoef (&q)[2]) {
    size_t o = ((size_t)b * N + e) * 2;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      q[i].s11 = a.coef[0 * plane + o + i];
      q[i].s12 = a.coef[1 * plane + o + i];
      q[i].s22 = a.coef[2 * plane + o + i];
      q[i].f1 = a.coef[3 * plane + o + i];
      q[i].f2 = a.coef[4 * plane + o + i];
      q[i].phi = 0.0;
    }
  };
  Super Sk[E];
  double R[E][6];
  bool flg[E];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    int e = e0 + k;
    bool own = e >= c0 && e < c1;
    flg[k] = own && flag(e);
#pragma unroll
    for (int q = 0; q < 6; ++q) R[k][q] = 0.0;
    if (!own) {
      Sk[k] = super_identity();
    } else if (!flg[k]) {
      Sk[k] = super_gap(e > 0 ? outer[e - 1] : 0.0);
    } else {
      NodeCoef q[2];
      load_q(e, q);
      const bool cut_right = e < N - 1 && start(e + 1) && flag(e);   // next range starts at e + 1
      bool range_end = (e == N - 1) || !flag(e + 1) || cut_right;
      if (!local_condense(m, q[0], q[1], a.rho, inv_rho, a.c11, range_end, Sk[k], R[k]))
        nh_report(a.status + b, 0, NH_ERR_SOLVE_PIVOT, e);
      if (!ldg_structure_ok(q[0], q[1])) nh_report(a.status + b, 0, NH_ERR_STRUCTURE, e);
      if (cut_right) {   // z_{e+1} is the outer trace hu(e+1, node 0): fold it in
        const double zc = outer[e];
        Sk[k].ga += Sk[k].ba * zc; Sk[k].ba = 0.0;
        Sk[k].gz += Sk[k].bz * zc; Sk[k].bz = 0.0;
        R[k][0] += R[k][2] * zc; R[k][2] = 0.0;
        R[k][3] += R[k][5] * zc; R[k][5] = 0.0;
      }
      if (start(e) && flag(e - 1)) {   // P* = 0 at this range start: drop a_{e-1}
        Sk[k].aa = 0.0; Sk[k].az = 0.0;
        R[k][1] = 0.0; R[k][4] = 0.0;
      }
    }
  }
  bool tflag = false;
#pragma unroll
  for (int k = 0; k < E; ++k) tflag = tflag || flg[k];
  Super agg = chunk_aggregate<E>(Sk, tflag);
  if (tid == 0) ts.pub[6] = outer[N - 1];
  double a_in, z_in;
  tree_solve(cluster, ts, C, rank, W, warp, lane, tflag, true, agg, a_in, z_in);
  double aprev[E], znext[E];
  chunk_unwind<E>(Sk, a_in, z_in, aprev, znext);
  ResidAcc ra{0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < E; ++k) {
    if (!flg[k]) continue;
    int e = e0 + k;
    double P0, P1, Q0, Q1;
    reconstruct(Sk[k], R[k], aprev[k], znext[k], a.c11, P0, P1, Q0, Q1);
    if (!isfinite(P0 + P1 + Q0 + Q1)) nh_report(a.status + b, 0, NH_ERR_SOLVE_NONFINITE, e);
    size_t o = ((size_t)b * N + e) * 2;
    a.p[o] = a.rho * P0; a.p[o + 1] = a.rho * P1;
    a.hu[o] = Q0; a.hu[o + 1] = Q1;
    // residual rows of the element (the reference's gate, corrector.py:355-366)
    NodeCoef q[2];
    load_q(e, q);
    const bool rs = start(e);
    const bool cut_right = e < N - 1 && start(e + 1);
    const bool re = (e == N - 1) || !flag(e + 1) || cut_right;
    ldg_residual(m, q[0], q[1], a.rho, inv_rho, a.c11, rs, re, rs ? 0.0 : aprev[k],
                 cut_right ? outer[e] : znext[k], P0, Q0, P1, Q1, ra);
  }
  resid_flush_warp(a.status + b, ra);
  cluster.sync();   // every CTA's shares are in; also keeps shared memory alive for DSMEM reads
  if (rank == 0 && tid == 0) {
    __threadfence();
    resid_check(a.status + b, 0, a.residual_tol);
  }
}

template __global__ void nh_solve_kernel<3>(SolveArgs);

void* nh_solve_kernel_ptr(int E) { return E == 3 ? (void*)nh_solve_kernel<3> : nullptr; }

// ------------------------------------------------------------- launch helpers
// ------------------------------------------------------------ arithmetic self-test
__device__ __forceinline__ unsigned long long splitmix(unsigned long long& x) {
  unsigned long long z = (x += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// operand with a mix of exponent ranges: mostly near 1 (the solver's values),
// plus full-range, tiny, denormal, zero, huge, inf and nan operands
__device__ __forceinline__ double test_operand(unsigned long long& st) {
  unsigned long long r = splitmix(st);
  unsigned cls = (unsigned)(r & 15);
  unsigned long long mant = (r >> 4) & 0xfffffffffffffull;
  unsigned long long sign = (r >> 60) & 1ull;
  unsigned long long ex;
  switch (cls) {
    case 0: return sign ? -0.0 : 0.0;
    case 1: ex = 0; break;                                        // denormal
    case 2: ex = 1 + (splitmix(st) % 60); break;                   // tiny
    case 3: ex = 2046 - (splitmix(st) % 60); break;                // huge
    case 4: ex = (splitmix(st) & 1) ? 2047 : 1 + (splitmix(st) % 2046); break;  // inf/nan or any
    case 5: case 6: ex = 1 + (splitmix(st) % 2046); break;         // full range
    default: ex = 1023 - 40 + (splitmix(st) % 60); break;          // 1e-12 .. 1e6
  }
  return __longlong_as_double((long long)((sign << 63) | (ex << 52) | mant));
}

__device__ __forceinline__ bool same_bits(double x, double y) {
  return __double_as_longlong(x) == __double_as_longlong(y) || (isnan(x) && isnan(y));
}

__global__ void nh_selftest_kernel(long long n, unsigned long long seed, unsigned long long* bad) {
  unsigned long long nd = 0, ns = 0, np = 0;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    unsigned long long st = seed ^ ((unsigned long long)k * 0xd1b54a32d192ed03ull);
    double a = test_operand(st), b = test_operand(st);
    nd += !same_bits(nh_ddiv_rn(a, b), __ddiv_rn(a, b));
    ns += !same_bits(nh_dsqrt_rn(a), __dsqrt_rn(a));
    double bp = fabs(b);
    if (bp > 0.0 && bp < INFINITY) np += !same_bits(nh_div_pos(a, bp), __ddiv_rn(a, bp));
  }
  if (nd) atomicAdd(bad + 0, nd);
  if (ns) atomicAdd(bad + 1, ns);
  if (np) atomicAdd(bad + 2, np);
}

// evaluate_criterion's mask (adaptivity.py:99-113): flag = max nodal indicator
// of the element > k_nh, optionally dilated by one element to each side
// (clipped to the member).  One thread per element; values [B][N][m].
__global__ void nh_mask_kernel(const double* __restrict__ v, int B, int N, int m, double k_nh,
                               int enlarge, uint8_t* __restrict__ flags) {
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (idx >= (size_t)B * N) return;
  const int e = (int)(idx % N);
  auto raw = [&](size_t i) -> bool {
    double mx = v[i * m];
    for (int j = 1; j < m; ++j) mx = fmax(mx, v[i * m + j]);   // np.max: NaN-free here
    return mx > k_nh;
  };
  bool f = raw(idx);
  if (enlarge) {
    if (e > 0) f = f || raw(idx - 1);
    if (e < N - 1) f = f || raw(idx + 1);
  }
  flags[idx] = f ? 1 : 0;
}

// max_wavespeed (hydrostatic.py:187-189): max over a member's nodes of
// |hu / h| + sqrt(g h), every operation the IEEE-rounded one numpy does.
// The values are non-negative, so the maximum is taken on the bit patterns.
__global__ void nh_wavespeed_kernel(const double* __restrict__ h, const double* __restrict__ hu,
                                    int B, size_t nodes, double g,
                                    unsigned long long* __restrict__ out) {
  const int b = blockIdx.y;
  unsigned long long mx = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nodes;
       i += (size_t)gridDim.x * blockDim.x) {
    const double hh = h[(size_t)b * nodes + i], q = hu[(size_t)b * nodes + i];
    const double a = __dadd_rn(fabs(__ddiv_rn(q, hh)), __dsqrt_rn(__dmul_rn(g, hh)));
    if (a == a) mx = max(mx, (unsigned long long)__double_as_longlong(a));
  }
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out + b, mx);
}

extern "C" {

int nh_launch_mask(const double* values, int B, int N, int m, double k_nh, int enlarge,
                   uint8_t* flags, cudaStream_t s) {
  const size_t n = (size_t)B * N;
  nh_mask_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(values, B, N, m, k_nh, enlarge, flags);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int nh_launch_wavespeed(const double* h, const double* hu, int B, size_t nodes, double g,
                        double* out, cudaStream_t s) {
  if (cudaMemsetAsync(out, 0, 8 * (size_t)B, s) != cudaSuccess) return 1;
  const unsigned gx = (unsigned)std::min<size_t>((nodes + 255) / 256, 1024);
  nh_wavespeed_kernel<<<dim3(gx, B), 256, 0, s>>>(h, hu, B, nodes, g, (unsigned long long*)out);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

int nh_launch_selftest(long long n, unsigned long long seed, unsigned long long* bad,
                       cudaStream_t s) {
  nh_selftest_kernel<<<148 * 8, 256, 0, s>>>(n, seed, bad);
  return cudaGetLastError() == cudaSuccess ? 0 : NH_E_CUDA;
}

int nh_launch_rhs(const nh_member* members, int B, int N, const double* h, const double* hu,
                  const double* hw, const double* time, double g, double* th, double* tq,
                  double* tw, nh_status* status, cudaStream_t s) {
  int n = B * N, tb = 128;
  nh_rhs_kernel<<<(n + tb - 1) / tb, tb, 0, s>>>(members, B, N, h, hu, hw, time, g, th, tq, tw,
                                                 status);
  return cudaGetLastError() == cudaSuccess ? 0 : NH_E_CUDA;
}

int nh_launch_criterion(const nh_member* members, int B, int N, const double* h, const double* hu,
                        const double* hw, const double* time, int kind, double* out,
                        cudaStream_t s) {
  int n = B * N, tb = 128;
  nh_criterion_kernel<<<(n + tb - 1) / tb, tb, 0, s>>>(members, B, N, h, hu, hw, time, kind, out);
  return cudaGetLastError() == cudaSuccess ? 0 : NH_E_CUDA;
}

int nh_launch_coef(const nh_member* members, int B, int N, const double* h, const double* hu,
                   const double* hw, const double* time, double g, double rho, double* coef,
                   cudaStream_t s) {
  int n = B * N, tb = 128;
  nh_coef_kernel<<<(n + tb - 1) / tb, tb, 0, s>>>(members, B, N, h, hu, hw, time, g, rho, coef);
  return cudaGetLastError() == cudaSuccess ? 0 : NH_E_CUDA;
}

int nh_launch_bottom(const nh_member* members, int B, const double* x, int P, const double* time,
                     double* out, cudaStream_t s) {
  int n = B * P, tb = 128;
  if (n == 0) return 0;
  nh_bottom_kernel<<<(n + tb - 1) / tb, tb, 0, s>>>(members, B, x, P, time, out);
  return cudaGetLastError() == cudaSuccess ? 0 : NH_E_CUDA;
}

int nh_launch_momentum(const nh_member* members, int B, int N, const double* h, const double* p,
                       const double* coef, const uint32_t* flags, double rho,
                       const double* hw_in, double* hw_out, cudaStream_t s) {
  int n = B * N, tb = 128;
  nh_momentum_kernel<<<(n + tb - 1) / tb, tb, 0, s>>>(members, B, N, h, p, coef, flags,
                                                      (N + 31) / 32, rho, hw_in, hw_out);
  return cudaGetLastError() == cudaSuccess ? 0 : NH_E_CUDA;
}

}  // extern "C"
