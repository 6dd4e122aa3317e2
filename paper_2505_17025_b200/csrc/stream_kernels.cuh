// Streaming step kernels: shared declarations (stream_kernels.cu, capi.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include "../../include/nhswe_b200.h"

#ifndef NH_STREAM_THREADS
#define NH_STREAM_THREADS 128   // measured on config 4: 64 96 128 160 192 256 512 -> 128 fastest
#endif
#define NH_STREAM_HALO 4
#define NH_STREAM_OWN (NH_STREAM_THREADS - 2 * NH_STREAM_HALO)
#define NH_STREAM_MAXCPL 8   // tiles per lane in K_X: members up to 32*8*OWN elements
#ifndef NH_STREAM_MIN_BLOCKS
#define NH_STREAM_MIN_BLOCKS (1024 / NH_STREAM_THREADS)   // K_P CTAs per SM (64 registers)
#endif
#ifndef NH_KS_MIN_BLOCKS
#define NH_KS_MIN_BLOCKS (1024 / NH_STREAM_THREADS)       // K_S / K_C CTAs per SM (64 registers; measured 6 / 8 / 10 at 128 threads: 8 fastest)
#endif

struct StreamArgs {
  const nh_member* members;
  const double* h_in;
  const double* hu_in;
  const double* hw_in;
  double* h_out;
  double* hu_out;
  double* hw_out;
  const uint8_t* flags_prev;   // flags of the step whose correction is pending (or unused)
  uint8_t* flags_cur;
  const double* pend;          // [6][B*N] planes p0 p1 phi0 phi1 dx0 dx1 of the pending step, or NULL
  double* pend_out;            // same, for this step
  double* scratch;             // [10][B*N] planes: LDG coefficients of flagged elements (store_coef)
  double* tile_agg;            // [B][T][8] aggregate (6), flagged count, right ghost
  double* tile_io;             // [B][T][2] (a_in, z_in)
  double* time;                // [B]
  int* step_counter;           // [B] steps done in this call
  nh_status* status;
  uint32_t* flag_bits;         // optional [n_steps][B][nwords]
  double* mconst;              // [B][16] per-member step constants (MemberConst)
  int* tile_list;              // [B*T] tiles holding a flagged element (this step, any order)
  int* tile_count;             // entries of tile_list (K_P appends, K_S / K_C consume)
  int* tile_count_next;        // the next step's counter, zeroed by K_X
  const int* order;            // [B] K_P's member order (grouped by bottom kind), or NULL
  const int32_t* gauge_nodes;  // [n_gauges] flat node indices, or NULL
  double* gauge_h;             // [n_steps][B][n_gauges]
  int* hw_any;                 // [B] w / w_x criterion: any(hw != 0) of the step input, or NULL
  int n_gauges;
  nh_scheme sch;
  int B, N, tiles, finalize;
};

// which: 0 K_P, 1 K_X, 2 K_C, 3 K_S, 4 prep (step constants for the current time),
//        5 order (members grouped by bottom kind, one CTA), 6 gauges,
//        7 full-mask fallback of the w / w_x criteria (K_F)
void* nh_stream_kernel(int which);
void* nh_stream_kp_ptr();    // stream_kp.cu
size_t nh_stream_kp_smem();  // its dynamic shared memory
int nh_stream_kp_threads();  // its block size
void* nh_stream_kp_fused_ptr();  // K_P with the K_S condensation fused in (global mode), or NULL
void* nh_stream_kfin_ptr();      // K_fin: the last pending hw update over the flagged-tile list
int nh_stream_kp_records_hw_any();   // 1: K_P records any(hw != 0) for the w / w_x fallback
int nh_launch_gather_p(const double* pend, const uint8_t* flags, double* p, size_t n,
                       cudaStream_t s);
