// Cluster-wide elimination of a chain of super-elements (see physics.cuh).
//
// Three levels, each a 32-wide merge tree run by one warp with shuffles:
//   A. every warp merges its 32 thread chunks (nodes kept in shared memory),
//   B. warp 0 merges the CTA's warp aggregates and publishes the CTA aggregate,
//   C. after ONE cluster barrier, warp 0 of every CTA reads the cluster's CTA
//      aggregates over DSMEM and merges them (redundantly in each CTA).
// The matching back-substitution runs C -> B -> A: the left end enters with
// a_in = 0 (P* = 0 at a range start), the right end with z_in = the right
// boundary ghost of hu (published by the last CTA in pub[6]).  Warps with no
// flagged element skip their tree entirely: an unflagged chunk aggregates to
// the gap super-element of its first element.  Every merge is an exact
// Schur elimination (Thomas-like, no transfer-matrix products), which keeps
// the result as accurate as the pivoted LAPACK band solve it replaces
// (DESIGN.md §3).
#pragma once
#include <cooperative_groups.h>
#include "physics.cuh"
#include "step_kernel.cuh"

namespace cg = cooperative_groups;

struct TreeSmem {
  double* wnode;   // W*31*6  level A nodes
  double* wagg;    // W*6     warp aggregates
  double* wio;     // W*2     warp (a_in, z_in)
  double* pub;     // 16      CTA aggregate (0..5), right ghost (6), any_hw (7)
  double* bnode;   // 31*6    level B nodes
  double* cnode;   // 31*6    level C nodes
  int* wflag;      // W       warp has a flagged element
};

__device__ __forceinline__ Super shfl_down_super(const Super& v, int d) {
  Super o;
  o.ga = __shfl_down_sync(0xffffffffu, v.ga, d);
  o.aa = __shfl_down_sync(0xffffffffu, v.aa, d);
  o.ba = __shfl_down_sync(0xffffffffu, v.ba, d);
  o.gz = __shfl_down_sync(0xffffffffu, v.gz, d);
  o.az = __shfl_down_sync(0xffffffffu, v.az, d);
  o.bz = __shfl_down_sync(0xffffffffu, v.bz, d);
  return o;
}

__device__ __forceinline__ Super shfl_super(const Super& v, int src) {
  Super o;
  o.ga = __shfl_sync(0xffffffffu, v.ga, src);
  o.aa = __shfl_sync(0xffffffffu, v.aa, src);
  o.ba = __shfl_sync(0xffffffffu, v.ba, src);
  o.gz = __shfl_sync(0xffffffffu, v.gz, src);
  o.az = __shfl_sync(0xffffffffu, v.az, src);
  o.bz = __shfl_sync(0xffffffffu, v.bz, src);
  return o;
}

// Up-sweep over `levels` (count <= 2^levels lanes hold data, the rest
// identities); lane 0 ends with the aggregate.  Node (l, k) at nodes[(base_l+k)*6].
// STORE = false: the aggregate alone (a caller that never sweeps down, K_S).
template <bool STORE = true>
__device__ __forceinline__ Super warp_up(Super agg, double* nodes, int lane, int levels) {
  int base_l = 0;
  for (int l = 0; l < levels; ++l) {
    const int d = 1 << l;
    Super o = shfl_down_super(agg, d);
    if ((lane & (2 * d - 1)) == 0) {
      double AL[3], ZR[3];
      agg = merge(agg, o, AL, ZR);
      if (STORE) {
        double* nd = nodes + (base_l + (lane >> (l + 1))) * 6;
        nd[0] = AL[0]; nd[1] = AL[1]; nd[2] = AL[2];
        nd[3] = ZR[0]; nd[4] = ZR[1]; nd[5] = ZR[2];
      }
    }
    base_l += 16 >> l;
  }
  return agg;
}

// Down-sweep: lane 0 enters with the aggregate's (a_in, z_in); every lane
// leaves with its own.
__device__ __forceinline__ void warp_down(double& a_in, double& z_in, const double* nodes, int lane,
                                          int levels) {
  for (int l = levels - 1; l >= 0; --l) {
    const int d = 1 << l;
    double sa = 0.0, sz = 0.0;
    if ((lane & (2 * d - 1)) == 0) {
      const double* nd = nodes + ((32 - (32 >> l)) + (lane >> (l + 1))) * 6;
      sa = nd[0] + nd[1] * a_in + nd[2] * z_in;          // A_L -> right child's a_in
      double zl = nd[3] + nd[4] * a_in + nd[5] * z_in;   // Z_R -> left child's z_in
      sz = z_in;
      z_in = zl;
    }
    double ra = __shfl_up_sync(0xffffffffu, sa, d);
    double rz = __shfl_up_sync(0xffffffffu, sz, d);
    if ((lane & (2 * d - 1)) == d) { a_in = ra; z_in = rz; }
  }
}

__device__ __forceinline__ int tree_levels(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

// tflag: this thread's chunk holds a flagged element; agg: its aggregate.
// Returns the chunk's (a_in, z_in) in a_in / z_in (meaningful when tflag).
// pub[6] (right ghost) must be set by its owner before the call.
__device__ __forceinline__ void tree_solve(cg::cluster_group& cluster, const TreeSmem& ts, int C,
                                           int rank, int W, int warp, int lane, bool tflag,
                                           bool cta_any, Super agg, double& a_in, double& z_in,
                                           long long* tprof = nullptr) {
#define NH_TT(i) do { if (tprof) { long long c_ = clock64(); tprof[i] += c_ - tprof[4]; tprof[4] = c_; } } while (0)
  double* wn = ts.wnode + warp * 31 * 6;
  const bool wany = __any_sync(0xffffffffu, tflag);
  if (wany) {
    agg = warp_up(agg, wn, lane, 5);
  } else {
    unsigned nonid = __ballot_sync(0xffffffffu, !is_identity(agg));
    int first = nonid ? __ffs(nonid) - 1 : 0;
    agg = shfl_super(agg, first);
    if (!nonid) agg = super_identity();
  }
  if (lane == 0) {
    double* wa = ts.wagg + warp * 6;
    wa[0] = agg.ga; wa[1] = agg.aa; wa[2] = agg.ba;
    wa[3] = agg.gz; wa[4] = agg.az; wa[5] = agg.bz;
    ts.wflag[warp] = wany ? 1 : 0;
  }
  __syncthreads();
  NH_TT(0);
  const int lb = tree_levels(W), lc = tree_levels(C);
  if (warp == 0) {
    Super v = super_identity();
    if (lane < W) {
      const double* wa = ts.wagg + lane * 6;
      v = Super{wa[0], wa[1], wa[2], wa[3], wa[4], wa[5]};
    }
    // a CTA without flagged elements is the gap of its first element: no merges
    if (cta_any) v = warp_up(v, ts.bnode, lane, lb);
    if (lane == 0) {
      ts.pub[0] = v.ga; ts.pub[1] = v.aa; ts.pub[2] = v.ba;
      ts.pub[3] = v.gz; ts.pub[4] = v.az; ts.pub[5] = v.bz;
    }
  }
  NH_TT(1);
  cluster.sync();   // CTA aggregates (and the right ghost) visible cluster-wide
  NH_TT(2);
  if (warp == 0 && cta_any) {
    Super v = super_identity();
    if (lane < C) {
      const double* rp = cluster.map_shared_rank(ts.pub, lane);
      v = Super{rp[0], rp[1], rp[2], rp[3], rp[4], rp[5]};
    }
    warp_up(v, ts.cnode, lane, lc);
    double ca = 0.0;
    double cz = *cluster.map_shared_rank(ts.pub + 6, C - 1);
    warp_down(ca, cz, ts.cnode, lane, lc);
    double my_a = __shfl_sync(0xffffffffu, ca, rank);
    double my_z = __shfl_sync(0xffffffffu, cz, rank);
    double wa_ = lane == 0 ? my_a : 0.0, wz_ = lane == 0 ? my_z : 0.0;
    warp_down(wa_, wz_, ts.bnode, lane, lb);
    if (lane < W) {
      ts.wio[lane * 2 + 0] = wa_;
      ts.wio[lane * 2 + 1] = wz_;
    }
  }
  __syncthreads();
  NH_TT(3);
  if (!cta_any) { a_in = 0.0; z_in = 0.0; return; }
  a_in = ts.wio[warp * 2 + 0];
  z_in = ts.wio[warp * 2 + 1];
  if (wany) warp_down(a_in, z_in, wn, lane, 5);
#undef NH_TT
}

// Chunk back-substitution: given the chunk's (a_in, z_in) and its elements'
// super-elements, returns a_{e-1} and z_{e+1} for each element.
template <int E>
__device__ __forceinline__ void chunk_unwind(const Super (&Sk)[E], double a_in, double z_in,
                                             double (&aprev)[E], double (&znext)[E]) {
  double sk[E], tk[E], mk[E], nk[E];
  double s = a_in, tt = 0.0;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    sk[k] = s; tk[k] = tt;
    riccati_step(Sk[k], s, tt, mk[k], nk[k]);
  }
  double z = z_in;
#pragma unroll
  for (int k = E - 1; k >= 0; --k) {
    znext[k] = z;
    z = fma(nk[k], z, mk[k]);
    aprev[k] = fma(tk[k], z, sk[k]);
  }
}

// Chunk aggregate; an unflagged chunk is the gap of its first own element
// (gap (+) gap = left gap, identity (+) X = X), so no merges are needed.
template <int E>
__device__ __forceinline__ Super chunk_aggregate(const Super (&Sk)[E], bool tflag) {
  if (!tflag) {
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (!is_identity(Sk[k])) return Sk[k];
    return super_identity();
  }
  Super agg = Sk[0];
#pragma unroll
  for (int k = 1; k < E; ++k) agg = merge2(agg, Sk[k]);
  return agg;
}

// Element reconstruction from the condensed form: P0, P1 (= p/rho), Q0, Q1 (= hu).
__device__ __forceinline__ void reconstruct(const Super& Q, const double (&R)[6], double ap,
                                            double zn, double c11, double& P0, double& P1,
                                            double& Q0, double& Q1) {
  P0 = R[0] + ap * R[1] + zn * R[2];
  Q1 = R[3] + ap * R[4] + zn * R[5];
  P1 = Q.ga + Q.aa * ap + Q.ba * zn;
  Q0 = (Q.gz + Q.az * ap + Q.bz * zn) + c11 * P0;
}
