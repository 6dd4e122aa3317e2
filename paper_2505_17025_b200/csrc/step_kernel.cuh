// Launch-side declarations shared by step_kernel.cu, solve_kernel.cu and capi.cu.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include "../../include/nhswe_b200.h"

#define NH_HALO 4
#define NH_MAX_CLUSTER 16
#define NH_STEP_MAX_THREADS 384

struct StepArgs {
  const nh_member* members;
  double* h;
  double* hu;
  double* hw;
  double* time;
  nh_status* status;
  uint32_t* flag_bits;
  double* p_out;
  const uint32_t* given;
  const int32_t* gauge_nodes;   // [n_gauges] flat node indices, or NULL
  double* gauge_h;              // [n_steps][B][n_gauges]
  int n_gauges;
  nh_scheme sch;
  int B, N, n_steps;
  int cluster, tile, nwords;
  long long* prof;   // NH_PROFILE_PHASES builds: [grid][NH_NPHASE] cycle sums (else unused)
};

#define NH_NPHASE 15

struct SolveArgs {
  const nh_member* members;
  const double* coef;         // [7][B][N][2]
  const uint32_t* flags;      // [B][nwords]
  const uint32_t* starts;     // [B][nwords] range starts inside flagged runs, or NULL
  const double* outer_right;  // [B][N]
  double* p;                  // [B][N][2]
  double* hu;                 // [B][N][2]
  nh_status* status;
  double rho, c11, residual_tol;
  int B, N, cluster, tile, nwords;
};

size_t nh_step_smem_bytes(int threads, int E);
size_t nh_solve_smem_bytes(int threads);
void* nh_step_kernel_ptr(int variant);
int nh_step_variant_E(int variant);
int nh_step_variant_maxt(int variant);
void* nh_solve_kernel_ptr(int E);
