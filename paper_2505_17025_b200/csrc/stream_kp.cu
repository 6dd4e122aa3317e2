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

size_t nh_stream_kp_smem() { return sizeof(KpSmem); }
int nh_stream_kp_threads() { return TPB; }

void* nh_stream_kp_ptr() { return (void*)nh_stream_kp; }
int nh_stream_kp_records_hw_any() { return 1; }   // w / w_x fallback (K_F)

