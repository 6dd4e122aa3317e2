// K_P of the streaming step (body in stream_kp.cuh); its own translation unit.
#include "stream_kp.cuh"


template <bool FUSE>
__device__ __forceinline__ void kp_entry(const StreamArgs& a) {
  __shared__ nh_member msh;
  __shared__ MemberConst mc;
  extern __shared__ __align__(16) unsigned char kp_dyn[];   // KpSmem (dynamic: > 48 KB at 512 threads)
  KpSmem& ks = *reinterpret_cast<KpSmem*>(kp_dyn);
  // grid (tiles, members): no integer division (members past 65535 in z);
  // the member axis runs in bottom-kind order so the CTAs resident at one
  // time mostly execute the same kind-specialised body (instruction cache)
  int b = blockIdx.z * 65535 + blockIdx.y;
  if (b >= a.B) return;   // padding of the (tiles, 65535, z) grid
  if (a.order) b = a.order[b];
  kp_tile<FUSE>(a, tile_idx(a, b, blockIdx.x), msh, mc, ks);
}

__global__ void __launch_bounds__(TPB, NH_STREAM_MIN_BLOCKS) nh_stream_kp(StreamArgs a) {
  kp_entry<false>(a);
}
// K_P with the K_S condensation fused in (global mode)
__global__ void __launch_bounds__(TPB, NH_STREAM_MIN_BLOCKS) nh_stream_kp_fused(StreamArgs a) {
  kp_entry<true>(a);
}
void* nh_stream_kp_fused_ptr() { return (void*)nh_stream_kp_fused; }

// K_fin: the last step's pending hw update after the time loop.  Only flagged
// elements change, so the grid strides over the last step's list of flagged
// tiles (every tile in global mode) instead of streaming the whole state
// through a finalize pass of K_P; a first stride over the members evaluates
// the residual gate of the last step's solve (K_X checks the earlier ones).
__global__ void __launch_bounds__(TPB, NH_STREAM_MIN_BLOCKS) nh_stream_kfin(StreamArgs a) {
  __shared__ nh_member msh;
  __shared__ MemberConst mc;
  extern __shared__ __align__(16) unsigned char kp_dyn[];
  KpSmem& ks = *reinterpret_cast<KpSmem*>(kp_dyn);
  if (a.step_counter)
    for (int b = blockIdx.x * TPB + threadIdx.x; b < a.B; b += gridDim.x * TPB)
      resid_check(a.status + b, a.step_counter[b] - 1, a.sch.residual_tol);
  const bool all = a.sch.mode == NH_MODE_GLOBAL;
  const int n = all ? a.B * a.tiles : *a.tile_count;
  for (int w = blockIdx.x; w < n; w += gridDim.x) {
    const int bt = all ? w : a.tile_list[w];
    const int b = bt / a.tiles;
    kp_tile<false, true>(a, tile_idx(a, b, bt - b * a.tiles), msh, mc, ks);
    __syncthreads();   // shared memory is reused by the next tile
  }
}
void* nh_stream_kfin_ptr() { return (void*)nh_stream_kfin; }

size_t nh_stream_kp_smem() { return sizeof(KpSmem); }
int nh_stream_kp_threads() { return TPB; }

void* nh_stream_kp_ptr() { return (void*)nh_stream_kp; }
int nh_stream_kp_records_hw_any() { return 1; }   // w / w_x fallback (K_F)

