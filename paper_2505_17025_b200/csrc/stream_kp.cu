// K_P of the streaming step (body in stream_kp.cuh); its own translation unit.
#include "stream_kp.cuh"
#include "stream_kp2.cuh"

#ifndef NH_KP_E2
#define NH_KP_E2 0   // 1: two elements per thread (stream_kp2.cuh); measured 20% slower (fewer warps)
#endif

#if NH_KP_E2
#ifndef NH_KP2_MIN_BLOCKS
#define NH_KP2_MIN_BLOCKS 8   // 64-thread CTAs per SM: 128 registers
#endif
__global__ void __launch_bounds__(TP2, NH_KP2_MIN_BLOCKS) nh_stream_kp(StreamArgs a) {
  __shared__ nh_member msh;
  __shared__ MemberConst mc;
  extern __shared__ __align__(16) unsigned char kp_dyn[];
  Kp2Smem& ks = *reinterpret_cast<Kp2Smem*>(kp_dyn);
  int b = blockIdx.z * 65535 + blockIdx.y;
  if (b >= a.B) return;
  if (a.order) b = a.order[b];
  kp2_tile(a, b, blockIdx.x, msh, mc, ks);
}
size_t nh_stream_kp_smem() { return sizeof(Kp2Smem); }
int nh_stream_kp_threads() { return TP2; }
#else

__global__ void __launch_bounds__(TPB, NH_STREAM_MIN_BLOCKS) nh_stream_kp(StreamArgs a) {
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
  kp_tile(a, tile_idx(a, b, blockIdx.x), msh, mc, ks);
}

size_t nh_stream_kp_smem() { return sizeof(KpSmem); }
int nh_stream_kp_threads() { return TPB; }
#endif

#ifndef NH_KP_PERSIST
// 1: steps run the persistent prefetching K_P (finalize keeps nh_stream_kp).
// Measured slower on config 4 (K_P 0.699 -> 0.854 ms; with raw-byte flag
// prefetch and no per-tile division 0.953 ms): the loop-carried prefetch
// state raises spills (176 -> 210-330 B) and instructions (+11 %) at the
// 64-register cap, more than the hidden load latency saves.  Off.
#define NH_KP_PERSIST 0
#endif
static_assert(!(NH_KP_PERSIST && NH_KP_FUSE_KS), "K_S fusion aliases sq, which the stages replace");

// Persistent K_P: the grid strides over the (member slot, tile) list with
// the next tile's copies in flight during the current tile (stream_kp.cuh).
__global__ void __launch_bounds__(TPB, NH_STREAM_MIN_BLOCKS) nh_stream_kp_pf(StreamArgs a) {
  extern __shared__ __align__(16) unsigned char kp_dyn[];
  KpSmemP& ks = *reinterpret_cast<KpSmemP*>(kp_dyn);
  const int T = a.tiles, G = gridDim.x, total = a.B * T;   // B * T < 2^31 (capi checks)
  const int gq = G / T, gr = G - gq * T;                    // stride G as (slots, tiles)
  int L = blockIdx.x;
  if (L >= total) return;
  int slot = L / T, tile = L - slot * T;
  // (slot, tile) of the tile G further on, without a division per tile
  auto advance = [&](int& sl, int& tl) {
    sl += gq; tl += gr;
    if (tl >= T) { tl -= T; ++sl; }
  };
  const int* ord = a.order;
  int b = ord ? ord[slot] : slot;
  kp_prefetch(a, b, tile, ks.st[0]);
  uint8_t f = kp_pending_flag(a, b, tile);
  int slot_n = slot, tile_n = tile;
  advance(slot_n, tile_n);
  // the member of the next tile; loads stay in flight (clamped index, no select)
  int b_next = ord ? ord[min(slot_n, a.B - 1)] : slot_n;
  for (int k = 0;; ++k) {
    const int s = k & 1;
    cp_async_wait_all();
    __syncthreads();   // stage s landed and is visible; every thread is done with stage s ^ 1
    const int Ln = L + G;
    uint8_t f_next = 0;
    int slot_a = slot_n, tile_a = tile_n;
    advance(slot_a, tile_a);
    int b_after = 0;
    if (Ln < total) {
      kp_prefetch(a, b_next, tile_n, ks.st[s ^ 1]);
      f_next = kp_pending_flag(a, b_next, tile_n);
      b_after = ord ? ord[min(slot_a, a.B - 1)] : slot_a;
    }
    kp_tile_staged(a, tile_idx(a, b, tile), ks.st[s], ks, f);
    if (Ln >= total) break;
    L = Ln; b = b_next; tile = tile_n; f = f_next;
    b_next = b_after; slot_n = slot_a; tile_n = tile_a;
  }
}

void* nh_stream_kp_pf_ptr() { return NH_KP_PERSIST ? (void*)nh_stream_kp_pf : nullptr; }
size_t nh_stream_kp_pf_smem() { return sizeof(KpSmemP); }

void* nh_stream_kp_ptr() { return (void*)nh_stream_kp; }
int nh_stream_kp_records_hw_any() { return NH_KP_E2 ? 0 : 1; }   // w / w_x fallback (K_F)
int nh_stream_kp_fuses_ks() { return (NH_KP_FUSE_KS && !NH_KP_E2) ? 1 : 0; }
