// Cluster-wide elimination of a chain of super-elements (see physics.cuh).
//
// Every thread holds the aggregate of its chunk of E consecutive elements.
// Up: warp merge tree over 32 chunks with shuffles (31 merge nodes kept in
// shared memory), then thread 0 folds the warps into the CTA aggregate and
// publishes it.  One cluster barrier.  Down: thread 0 of every CTA solves
// the short chain of CTA aggregates read over DSMEM (a_in = 0 at the left
// end because P* = 0 there, z_in = the right-end ghost hu trace published by
// the last CTA in pub[6]), then the chain of its warp aggregates, and the
// warps unwind their merge trees so that every lane ends with the
// (a_in, z_in) entering its chunk.  Elimination order is Thomas-like at every
// level (no transfer-matrix products), which is what keeps it as accurate as
// the pivoted LAPACK band solve it replaces.
#pragma once
#include <cooperative_groups.h>
#include "physics.cuh"
#include "step_kernel.cuh"

namespace cg = cooperative_groups;

struct TreeSmem {
  double* wnode;  // W*31*6
  double* wagg;   // W*6
  double* wio;    // W*2
  double* pub;    // >= 8
  double* chain;  // 4*(NH_MAX_CLUSTER+32)
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

__device__ __forceinline__ void tree_solve(cg::cluster_group& cluster, const TreeSmem& ts, int C,
                                           int rank, int W, int warp, int lane, int tid,
                                           Super agg, double& a_in, double& z_in) {
  double* wn = ts.wnode + warp * 31 * 6;
  {
    int base_l = 0;
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      const int d = 1 << l;
      Super o = shfl_down_super(agg, d);
      if ((lane & (2 * d - 1)) == 0) {
        double AL[3], ZR[3];
        agg = merge(agg, o, AL, ZR);
        double* nd = wn + (base_l + (lane >> (l + 1))) * 6;
        nd[0] = AL[0]; nd[1] = AL[1]; nd[2] = AL[2];
        nd[3] = ZR[0]; nd[4] = ZR[1]; nd[5] = ZR[2];
      }
      base_l += 16 >> l;
    }
  }
  if (lane == 0) {
    double* wa = ts.wagg + warp * 6;
    wa[0] = agg.ga; wa[1] = agg.aa; wa[2] = agg.ba;
    wa[3] = agg.gz; wa[4] = agg.az; wa[5] = agg.bz;
  }
  __syncthreads();
  if (tid == 0) {
    Super ca{ts.wagg[0], ts.wagg[1], ts.wagg[2], ts.wagg[3], ts.wagg[4], ts.wagg[5]};
    for (int w = 1; w < W; ++w) {
      const double* wa = ts.wagg + w * 6;
      ca = merge2(ca, Super{wa[0], wa[1], wa[2], wa[3], wa[4], wa[5]});
    }
    ts.pub[0] = ca.ga; ts.pub[1] = ca.aa; ts.pub[2] = ca.ba;
    ts.pub[3] = ca.gz; ts.pub[4] = ca.az; ts.pub[5] = ca.bz;
  }
  cluster.sync();   // CTA aggregates visible cluster-wide
  if (tid == 0) {
    double* sv = ts.chain; double* tv = sv + NH_MAX_CLUSTER;
    double* mv = tv + NH_MAX_CLUSTER; double* nv = mv + NH_MAX_CLUSTER;
    double s = 0.0, tt = 0.0;
    for (int r = 0; r < C; ++r) {
      const double* rp = cluster.map_shared_rank(ts.pub, r);
      Super A{rp[0], rp[1], rp[2], rp[3], rp[4], rp[5]};
      sv[r] = s; tv[r] = tt;
      riccati_step(A, s, tt, mv[r], nv[r]);
    }
    double z = *cluster.map_shared_rank(ts.pub + 6, C - 1);
    double my_a = 0.0, my_z = 0.0;
    for (int r = C - 1; r >= 0; --r) {
      double zin = z;
      z = fma(nv[r], z, mv[r]);
      if (r == rank) { my_z = zin; my_a = fma(tv[r], z, sv[r]); }
    }
    double* ws = ts.chain + 4 * NH_MAX_CLUSTER; double* wt = ws + 32;
    double* wm = wt + 32; double* wv = wm + 32;
    s = my_a; tt = 0.0;
    for (int w = 0; w < W; ++w) {
      const double* wa = ts.wagg + w * 6;
      ws[w] = s; wt[w] = tt;
      riccati_step(Super{wa[0], wa[1], wa[2], wa[3], wa[4], wa[5]}, s, tt, wm[w], wv[w]);
    }
    z = my_z;
    for (int w = W - 1; w >= 0; --w) {
      ts.wio[w * 2 + 1] = z;
      z = fma(wv[w], z, wm[w]);
      ts.wio[w * 2 + 0] = fma(wt[w], z, ws[w]);
    }
  }
  __syncthreads();
  a_in = ts.wio[warp * 2 + 0];
  z_in = ts.wio[warp * 2 + 1];
  {
    const int lbase[5] = {0, 16, 24, 28, 30};
#pragma unroll
    for (int l = 4; l >= 0; --l) {
      const int d = 1 << l;
      double sa = 0.0, sz = 0.0;
      if ((lane & (2 * d - 1)) == 0) {
        const double* nd = wn + (lbase[l] + (lane >> (l + 1))) * 6;
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

// Element reconstruction from the condensed form: P0, P1 (= p/rho), Q0, Q1 (= hu).
__device__ __forceinline__ void reconstruct(const Super& Q, const double (&R)[6], double ap,
                                            double zn, double c11, double& P0, double& P1,
                                            double& Q0, double& Q1) {
  P0 = R[0] + ap * R[1] + zn * R[2];
  Q1 = R[3] + ap * R[4] + zn * R[5];
  P1 = Q.ga + Q.aa * ap + Q.ba * zn;
  Q0 = (Q.gz + Q.az * ap + Q.bz * zn) + c11 * P0;
}
