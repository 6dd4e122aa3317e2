// extern "C" boundary (include/nhswe_b200.h): argument checks, launch
// geometry, cluster launches.
#include <cuda_runtime.h>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "step_kernel.cuh"
#include "stream_kernels.cuh"

extern "C" {
int nh_launch_rhs(const nh_member*, int, int, const double*, const double*, const double*,
                  const double*, double, double*, double*, double*, nh_status*, cudaStream_t);
int nh_launch_criterion(const nh_member*, int, int, const double*, const double*, const double*,
                        const double*, int, double*, cudaStream_t);
int nh_launch_coef(const nh_member*, int, int, const double*, const double*, const double*,
                   const double*, double, double, double*, cudaStream_t);
int nh_launch_selftest(long long, unsigned long long, unsigned long long*, cudaStream_t);
int nh_launch_mask(const double*, int, int, int, double, int, uint8_t*, cudaStream_t);
int nh_launch_wavespeed(const double*, const double*, int, size_t, double, double*, cudaStream_t);
int nh_launch_bottom(const nh_member*, int, const double*, int, const double*, double*,
                     cudaStream_t);
int nh_launch_momentum(const nh_member*, int, int, const double*, const double*, const double*,
                       const uint32_t*, double, const double*, double*, cudaStream_t);
}

namespace {

constexpr int kE = 3;   // elements per thread of the coefficient-driven solve kernel

int variant() {
  static int v = [] {
    const char* e = getenv("NH_STEP_VARIANT");
    int x = e ? atoi(e) : 0;
    return (x < 0 || x > 3) ? 0 : x;
  }();
  return v;
}

struct Plan {
  int cluster, tile, threads;
  size_t smem;
};

// Launch geometry for members of n elements.  Each CTA keeps `tile` own
// elements plus NH_HALO on each side in shared memory; clusters are as small
// as the 384-thread CTA allows for large ensembles (more members in flight),
// and up to 8 CTAs for small ensembles (lower step latency).
int max_threads() {
  static int v = [] {
    const char* e = getenv("NH_MAX_THREADS");
    int cap = nh_step_variant_maxt(variant());
    int x = e ? atoi(e) : cap;
    if (x < 32 || x > cap) x = cap;
    return x;
  }();
  return v;
}

Plan make_plan(int n, int members) {
  const int H = NH_HALO;
  const int E = nh_step_variant_E(variant());
  const int tile_max = E * max_threads() - 2 * H;
  int cmin = (n + tile_max - 1) / tile_max;
  int c = cmin;
  if ((long long)members * cmin < 148) {
    int want = std::max(cmin, std::min(8, (int)((148 + members - 1) / members)));
    // keep tiles >= 64 elements so halos stay small next to the tile
    while (want > cmin && (n + want - 1) / want < 64) --want;
    c = want;
  }
  Plan p;
  p.cluster = c;
  p.tile = (n + c - 1) / c;
  int slots = p.tile + 2 * H;
  int thr = (slots + E - 1) / E;
  p.threads = std::max(32, ((thr + 31) / 32) * 32);
  p.smem = nh_step_smem_bytes(p.threads, E);
  return p;
}

bool g_attr_done = false;
long long* g_prof = nullptr;
std::mutex g_attr_mu;
std::atomic<long long> g_launches{0};   // kernels this library has enqueued (nh_launch_count)

// Optional per-kernel CUDA-event timing of the streaming path (nh_stream_timing):
// one event between consecutive launches on the caller's stream, so event i-1 -> i
// brackets exactly one kernel.
struct StreamTiming {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  size_t used = 0;
  struct Mark { int kernel; size_t a, b; };
  std::vector<Mark> marks;
  cudaEvent_t next() {
    if (used == ev.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      ev.push_back(e);
    }
    return ev[used++];
  }
} g_timing;
std::mutex g_timing_mu;

int counted(int rc) {
  if (rc == 0) ++g_launches;
  return rc;
}

// enqueue a plain launch of a streaming kernel, bracketing it with events when timing
int stream_launch(void* k, int kid, dim3 g, dim3 b, void** args, cudaStream_t s, size_t smem = 0) {
  size_t a = 0;
  if (g_timing.on) {
    if (g_timing.used == 0 || g_timing.marks.empty() || g_timing.marks.back().b != g_timing.used - 1) {
      cudaEvent_t e = g_timing.next();
      if (!e || cudaEventRecord(e, s) != cudaSuccess) return NH_E_CUDA;
    }
    a = g_timing.used - 1;
  }
  if (cudaLaunchKernel(k, g, b, args, smem, s) != cudaSuccess) return NH_E_CUDA;
  ++g_launches;
  if (g_timing.on) {
    cudaEvent_t e = g_timing.next();
    if (!e || cudaEventRecord(e, s) != cudaSuccess) return NH_E_CUDA;
    g_timing.marks.push_back({kid, a, g_timing.used - 1});
  }
  return 0;
}

int set_attrs() {
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (g_attr_done) return 0;
  void* k = nh_step_kernel_ptr(variant());
  size_t smax = nh_step_smem_bytes(nh_step_variant_maxt(variant()), nh_step_variant_E(variant()));
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax) != cudaSuccess)
    return NH_E_CUDA;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return NH_E_CUDA;
  void* ks = nh_solve_kernel_ptr(kE);
  if (cudaFuncSetAttribute(ks, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    return NH_E_CUDA;
  g_attr_done = true;
  return 0;
}

int launch_cluster(void* kernel, void* args, int grid, int block, size_t smem, int cluster,
                   cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(block, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* params[1] = {args};
  cudaError_t e = cudaLaunchKernelExC(&cfg, kernel, params);
  return e == cudaSuccess ? 0 : NH_E_CUDA;
}

}  // namespace

// the launch counter, for kernels in other translation units (pm_kernels.cu)
void nh_count_launch() { ++g_launches; }

extern "C" {

int nh_abi_version(void) { return NH_ABI_VERSION; }

int nh_plan(int n_elements, int n_members, int* cluster, int* tile, int* threads,
            int* smem_bytes) {
  if (n_elements < 2 || n_members < 1) return NH_E_ARG;
  Plan p = make_plan(n_elements, n_members);
  if (p.cluster > NH_MAX_CLUSTER) return NH_E_UNSUPPORTED;
  if (cluster) *cluster = p.cluster;
  if (tile) *tile = p.tile;
  if (threads) *threads = p.threads;
  if (smem_bytes) *smem_bytes = (int)p.smem;
  return 0;
}

int nh_advance(const nh_member* members, int n_members, int n_elements, double* h, double* hu,
               double* hw, double* time, int n_steps, const nh_scheme* scheme,
               const nh_outputs* outputs, nh_status* status, void* stream) {
  if (!members || !h || !hu || !hw || !time || !scheme || !status) return NH_E_ARG;
  if (n_members < 1 || n_elements < 2 || n_steps < 0) return NH_E_ARG;
  if (n_steps == 0) return 0;
  const nh_scheme& sc = *scheme;
  if (sc.mode < NH_MODE_HYDROSTATIC || sc.mode > NH_MODE_CORRECT_GIVEN) return NH_E_ARG;
  if (sc.mode != NH_MODE_HYDROSTATIC && (sc.c12 != -0.5 || sc.c22 != 0.0))
    return NH_E_UNSUPPORTED;   // condensed solve needs the alternating flux (physics.cuh)
  if (sc.mode == NH_MODE_CORRECT_GIVEN && (!outputs || !outputs->given_flags)) return NH_E_ARG;
  Plan p = make_plan(n_elements, n_members);
  if (p.cluster > NH_MAX_CLUSTER) return NH_E_UNSUPPORTED;
  int rc = set_attrs();
  if (rc) return rc;
  StepArgs a{};
  a.members = members;
  a.h = h; a.hu = hu; a.hw = hw; a.time = time;
  a.status = status;
  a.flag_bits = outputs ? outputs->flag_bits : nullptr;
  if (outputs && outputs->n_gauges > 0) {
    if (!outputs->gauge_nodes || !outputs->gauge_h) return NH_E_ARG;
    a.gauge_nodes = outputs->gauge_nodes; a.gauge_h = outputs->gauge_h; a.n_gauges = outputs->n_gauges;
  }
  a.p_out = outputs ? outputs->p_nh : nullptr;
  a.given = outputs ? outputs->given_flags : nullptr;
  a.sch = sc;
  a.B = n_members; a.N = n_elements; a.n_steps = n_steps;
  a.cluster = p.cluster; a.tile = p.tile; a.nwords = (n_elements + 31) / 32;
  a.prof = g_prof;
  return counted(launch_cluster(nh_step_kernel_ptr(variant()), &a, n_members * p.cluster,
                                p.threads, p.smem, p.cluster, (cudaStream_t)stream));
}

int nh_rhs(const nh_member* members, int n_members, int n_elements, const double* h,
           const double* hu, const double* hw, const double* time, double g, double* t_h,
           double* t_hu, double* t_hw, nh_status* status, void* stream) {
  if (!members || n_members < 1 || n_elements < 2) return NH_E_ARG;
  return counted(nh_launch_rhs(members, n_members, n_elements, h, hu, hw, time, g, t_h, t_hu, t_hw, status,
                       (cudaStream_t)stream));
}

int nh_criterion(const nh_member* members, int n_members, int n_elements, const double* h,
                 const double* hu, const double* hw, const double* time, int kind,
                 double* values, void* stream) {
  if (!members || n_members < 1 || n_elements < 2 || kind < 0 || kind > 5) return NH_E_ARG;
  return counted(nh_launch_criterion(members, n_members, n_elements, h, hu, hw, time, kind, values,
                             (cudaStream_t)stream));
}

int nh_mask(const double* values, int n_members, int n_elements, int nodes, double k_nh,
            int enlarge, uint8_t* flags, void* stream) {
  if (!values || !flags || n_members < 1 || n_elements < 1 || nodes < 1) return NH_E_ARG;
  return counted(nh_launch_mask(values, n_members, n_elements, nodes, k_nh, enlarge, flags,
                                (cudaStream_t)stream));
}

int nh_max_wavespeed(const double* h, const double* hu, int n_members, long long nodes_per_member,
                     double g, double* out, void* stream) {
  if (!h || !hu || !out || n_members < 1 || n_members > 65535 || nodes_per_member < 1)
    return NH_E_ARG;
  return counted(nh_launch_wavespeed(h, hu, n_members, (size_t)nodes_per_member, g, out,
                                     (cudaStream_t)stream));
}

int nh_coefficients(const nh_member* members, int n_members, int n_elements, const double* h,
                    const double* hu, const double* hw, const double* time, double g, double rho,
                    double* coef, void* stream) {
  if (!members || n_members < 1 || n_elements < 2) return NH_E_ARG;
  return counted(nh_launch_coef(members, n_members, n_elements, h, hu, hw, time, g, rho, coef,
                        (cudaStream_t)stream));
}

int nh_ldg_solve(const nh_member* members, int n_members, int n_elements, const double* coef,
                 const uint32_t* flags, const uint32_t* range_starts, const double* outer_right,
                 double rho, double c11, double c12, double c22, double residual_tol, double* p,
                 double* hu, nh_status* status, void* stream) {
  if (!members || n_members < 1 || n_elements < 2) return NH_E_ARG;
  if (c12 != -0.5 || c22 != 0.0) return NH_E_UNSUPPORTED;
  int rc = set_attrs();
  if (rc) return rc;
  const int tile_max = kE * NH_STEP_MAX_THREADS;
  int c = (n_elements + tile_max - 1) / tile_max;
  if (c > NH_MAX_CLUSTER) return NH_E_UNSUPPORTED;
  int tile = (n_elements + c - 1) / c;
  int thr = std::max(32, ((tile + kE - 1) / kE + 31) / 32 * 32);
  SolveArgs a;
  a.members = members; a.coef = coef; a.flags = flags; a.starts = range_starts;
  a.outer_right = outer_right;
  a.p = p; a.hu = hu; a.status = status; a.rho = rho; a.c11 = c11; a.residual_tol = residual_tol;
  a.B = n_members; a.N = n_elements; a.cluster = c; a.tile = tile;
  a.nwords = (n_elements + 31) / 32;
  return counted(launch_cluster(nh_solve_kernel_ptr(kE), &a, n_members * c, thr,
                                nh_solve_smem_bytes(thr), c, (cudaStream_t)stream));
}

int nh_correct_momentum(const nh_member* members, int n_members, int n_elements, const double* h,
                        const double* p, const double* coef, const uint32_t* flags, double rho,
                        const double* hw_in, double* hw_out, void* stream) {
  if (!members || n_members < 1 || n_elements < 2) return NH_E_ARG;
  return counted(nh_launch_momentum(members, n_members, n_elements, h, p, coef, flags, rho, hw_in, hw_out,
                            (cudaStream_t)stream));
}

int nh_bottom_sample(const nh_member* members, int n_members, const double* x, int n_points,
                     const double* time, double* out, void* stream) {
  if (!members || n_members < 1 || n_points < 0) return NH_E_ARG;
  return counted(nh_launch_bottom(members, n_members, x, n_points, time, out, (cudaStream_t)stream));
}

// ------------------------------------------------------------- CUDA graphs
extern "C++" {
namespace {
// NH_STREAM_GRAPH=0 disables the captured time loop (plain launches).
std::atomic<int> g_graphs{-1};
bool graphs_enabled() {
  if (g_graphs.load() < 0)
    g_graphs = (!getenv("NH_STREAM_GRAPH") || atoi(getenv("NH_STREAM_GRAPH")) != 0) ? 1 : 0;
  return g_graphs.load() != 0;
}

// Cached executable graphs of a pair of steps, keyed on the device and the
// launch arguments of both steps.  A small LRU of slots: callers that
// alternate between ensembles or buffers (e.g. the host-pipelined member
// blocks of driver.advance_host) replay their own graph instead of
// re-capturing.  Capture streams are per device.
constexpr int NH_GRAPH_SLOTS = 16;
constexpr int NH_MAX_DEVICES = 64;
struct PairGraph {
  bool valid = false;
  int device = -1;
  unsigned long long used = 0;   // LRU stamp
  unsigned char key[sizeof(StreamArgs)];
  cudaGraphExec_t exec = nullptr;
  long long nodes = 0;
};
PairGraph g_pairs[NH_GRAPH_SLOTS];
cudaStream_t g_cap[NH_MAX_DEVICES] = {};
unsigned long long g_stamp = 0;
std::mutex g_pair_mu;

template <class Capture>
int pair_graph(const StreamArgs& a, Capture capture, cudaGraphExec_t& exec, long long& nodes) {
  std::lock_guard<std::mutex> lk(g_pair_mu);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= NH_MAX_DEVICES) return NH_E_CUDA;
  if (!g_cap[dev] && cudaStreamCreateWithFlags(&g_cap[dev], cudaStreamNonBlocking) != cudaSuccess)
    return NH_E_CUDA;
  // capture (nothing executes) on a private stream: the caller's may be the
  // legacy default stream, which cannot be captured; the graph is launched
  // on the caller's stream
  const long long l0 = g_launches.load();
  if (cudaStreamBeginCapture(g_cap[dev], cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return NH_E_CUDA;
  int rc = capture(g_cap[dev]);
  cudaGraph_t graph = nullptr;
  cudaError_t ce = cudaStreamEndCapture(g_cap[dev], &graph);
  const long long n = g_launches.load() - l0;
  g_launches -= n;   // captured, not executed
  if (rc || ce != cudaSuccess || !graph) {
    if (graph) cudaGraphDestroy(graph);
    return rc ? rc : NH_E_CUDA;
  }
  // `a` now holds the even step's arguments, which fix the odd step's too
  PairGraph* hit = nullptr;
  PairGraph* victim = &g_pairs[0];
  for (PairGraph& g : g_pairs) {
    if (g.valid && g.device == dev && std::memcmp(&a, g.key, sizeof(StreamArgs)) == 0) {
      hit = &g;
      break;
    }
    if (!g.valid || (victim->valid && g.used < victim->used)) victim = &g;
  }
  if (hit) {
    cudaGraphDestroy(graph);
  } else {
    hit = victim;
    if (hit->exec) {
      int cur = dev;
      if (hit->device != dev) cudaSetDevice(hit->device);
      cudaGraphExecDestroy(hit->exec);
      if (hit->device != dev) cudaSetDevice(cur);
    }
    hit->exec = nullptr;
    hit->valid = false;
    ce = cudaGraphInstantiate(&hit->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) return NH_E_CUDA;
    std::memcpy(hit->key, &a, sizeof(StreamArgs));
    hit->device = dev;
    hit->valid = true;
    hit->nodes = n;
  }
  hit->used = ++g_stamp;
  exec = hit->exec;
  nodes = hit->nodes;
  return 0;
}

// Persistent-grid sizes of K_S / K_C (resident CTAs x SMs) and the K_P
// shared-memory opt-in, per device.
struct StreamDevice {
  int ks_grid = 0, kc_grid = 0;
};
StreamDevice g_sdev[NH_MAX_DEVICES];
std::mutex g_sdev_mu;

int stream_device_init(StreamDevice*& out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= NH_MAX_DEVICES) return NH_E_CUDA;
  std::lock_guard<std::mutex> lk(g_sdev_mu);
  StreamDevice& d = g_sdev[dev];
  if (!d.ks_grid) {
    int sms = 0, nks = 0, nkc = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nks, nh_stream_kernel(3), NH_STREAM_THREADS, 0) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nkc, nh_stream_kernel(2), NH_STREAM_THREADS, 0) != cudaSuccess)
      return NH_E_CUDA;
    if (cudaFuncSetAttribute(nh_stream_kernel(0), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)nh_stream_kp_smem()) != cudaSuccess)
      return NH_E_CUDA;
    if (void* kf = nh_stream_kp_fused_ptr())
      if (cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)nh_stream_kp_smem()) != cudaSuccess)
        return NH_E_CUDA;
    int ks = std::max(1, nks) * sms, kc = std::max(1, nkc) * sms;
    if (getenv("NH_STREAM_VERBOSE"))
      fprintf(stderr, "nh_stream: device %d K_S grid %d, K_C grid %d\n", dev, ks, kc);
    if (const char* v = getenv("NH_KS_WAVES")) {   // diagnostics: grid = waves x resident CTAs
      int wv = atoi(v);
      if (wv > 0) { ks *= wv; kc *= wv; }
    }
    d.kc_grid = kc;
    d.ks_grid = ks;
  }
  out = &d;
  return 0;
}
}  // namespace
}  // extern "C++"

// ------------------------------------------------------------- streaming path
static int stream_tiles(int n) { return (n + NH_STREAM_OWN - 1) / NH_STREAM_OWN; }

size_t nh_stream_workspace_bytes(int n_members, int n_elements) {
  size_t BN = (size_t)n_members * n_elements, BT = (size_t)n_members * stream_tiles(n_elements);
  size_t dbl = 6 * BN + 10 * BN + 12 * BN + 10 * BT + 16 * (size_t)n_members;
  return dbl * 8 + 2 * BN + 4 * (size_t)n_members + 8 + 4 * BT + 8 * (size_t)n_members + 1024;
}

int nh_stream_advance(const nh_member* members, int B, int N, double* h, double* hu, double* hw,
                      double* time, int n_steps, const nh_scheme* scheme,
                      const nh_outputs* outputs, nh_status* status, void* workspace,
                      size_t workspace_bytes, void* stream) {
  if (!members || !h || !hu || !hw || !time || !scheme || !status || !workspace) return NH_E_ARG;
  if (B < 1 || N < 2 || n_steps < 0) return NH_E_ARG;
  if (workspace_bytes < nh_stream_workspace_bytes(B, N)) return NH_E_ARG;
  const nh_scheme& sc = *scheme;
  if (sc.mode < NH_MODE_HYDROSTATIC || sc.mode > NH_MODE_ADAPTIVE) return NH_E_UNSUPPORTED;
  if (sc.mode != NH_MODE_HYDROSTATIC && (sc.c12 != -0.5 || sc.c22 != 0.0)) return NH_E_UNSUPPORTED;
  const int T = stream_tiles(N);
  if ((T + 31) / 32 > NH_STREAM_MAXCPL) return NH_E_UNSUPPORTED;
  if ((long long)B * T >= (1ll << 31)) return NH_E_UNSUPPORTED;   // tile ids are int
  if (n_steps == 0) return 0;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t BN = (size_t)B * N, BT = (size_t)B * T;
  char* w = (char*)workspace;
  double* alt = (double*)w;             w += 6 * BN * 8;
  double* scratch = (double*)w;         w += 10 * BN * 8;
  double* pend[2] = {(double*)w, (double*)w + 6 * BN};  w += 12 * BN * 8;
  double* tagg = (double*)w;            w += 8 * BT * 8;
  double* tio = (double*)w;             w += 2 * BT * 8;
  double* mconst = (double*)w;          w += 16 * (size_t)B * 8;
  uint8_t* flags[2] = {(uint8_t*)w, (uint8_t*)w + BN};  w += 2 * BN;
  int* counter = (int*)(((uintptr_t)w + 15) & ~(uintptr_t)15);
  int* tcount = counter + B;            // [2] flagged-tile counters (ping-pong by step)
  int* tlist = tcount + 2;              // [B*T] flagged-tile list
  int* order = tlist + BT;              // [B] K_P member order (by bottom kind)
  int* hw_any = order + B;              // [B] w / w_x: any(hw != 0) of the step input (K_P -> K_F)
  if (cudaMemsetAsync(counter, 0, 4 * ((size_t)B + 2), s) != cudaSuccess) return NH_E_CUDA;
  const bool w_crit = sc.mode == NH_MODE_ADAPTIVE &&
                      (sc.criterion == NH_CRIT_W || sc.criterion == NH_CRIT_W_X);
  if (w_crit && !nh_stream_kp_records_hw_any()) return NH_E_UNSUPPORTED;
  if (w_crit && cudaMemsetAsync(hw_any, 0, 4 * (size_t)B, s) != cudaSuccess) return NH_E_CUDA;
  StreamDevice* sdev = nullptr;   // persistent grids of this device
  if (int rc = stream_device_init(sdev)) return rc;
  const int ks_grid = sdev->ks_grid, kc_grid = sdev->kc_grid;
  double* A[3] = {h, hu, hw};
  double* Bb[3] = {alt, alt + 2 * BN, alt + 4 * BN};
  StreamArgs a;
  std::memset(&a, 0, sizeof a);   // padding too: the graph cache compares bytes
  a.members = members; a.time = time; a.status = status; a.step_counter = counter;
  a.scratch = scratch; a.tile_agg = tagg; a.tile_io = tio;
  a.flag_bits = outputs ? outputs->flag_bits : nullptr;
  if (outputs && outputs->n_gauges > 0) {
    if (!outputs->gauge_nodes || !outputs->gauge_h) return NH_E_ARG;
    a.gauge_nodes = outputs->gauge_nodes; a.gauge_h = outputs->gauge_h; a.n_gauges = outputs->n_gauges;
  }
  a.sch = sc; a.B = B; a.N = N; a.tiles = T; a.finalize = 0;
  a.tile_list = tlist; a.mconst = mconst;
  a.hw_any = w_crit ? hw_any : nullptr;
  static const bool use_order = !getenv("NH_STREAM_ORDER") || atoi(getenv("NH_STREAM_ORDER")) != 0;
  a.order = use_order ? order : nullptr;
  const dim3 gp(T, std::min(B, 65535), (B + 65534) / 65535), bp(NH_STREAM_THREADS),
      bpp(nh_stream_kp_threads()),
      gx((B + 7) / 8), bx(288);
  const dim3 gs((unsigned)std::min<size_t>(ks_grid, BT)), gc((unsigned)std::min<size_t>(kc_grid, BT));
  void* kp = nh_stream_kernel(0);
  const size_t kp_smem = nh_stream_kp_smem();
  void* kx = nh_stream_kernel(1);
  void* kc = nh_stream_kernel(2);
  void* ks = nh_stream_kernel(3);
  const bool corr = sc.mode != NH_MODE_HYDROSTATIC;
  // global mode: every tile is condensed, so K_P does it in the same pass
  // (no K_S launch, no state re-read); NH_KP_FUSE_GLOBAL=0 keeps K_S
  static const bool fuse_global =
      !getenv("NH_KP_FUSE_GLOBAL") || atoi(getenv("NH_KP_FUSE_GLOBAL")) != 0;
  // (adaptive mode keeps K_S at every flagged fraction: fused K_P + K_C measured
  // 6 % slower at 2 %, 7 % at 20 % and 6 % at 26 % flagged, profiles/r2_ab_fuse_adaptive.txt)
  const bool fused_ks = fuse_global && sc.mode == NH_MODE_GLOBAL && nh_stream_kp_fused_ptr();
  void* kp_step = fused_ks ? nh_stream_kp_fused_ptr() : kp;
  {
    void* args[1] = {&a};
    if (int rc = stream_launch(nh_stream_kernel(4), 5, dim3((B + 255) / 256), dim3(256), args, s))
      return rc;
    if (a.order)
      if (int rc = stream_launch(nh_stream_kernel(5), 5, dim3(1), dim3(1024), args, s)) return rc;
  }
  // step k reads the state written by step k - 1: ping-pong A <-> Bb, and
  // the pending record / flags / flagged-tile counters alternate the same way,
  // so every step's launches depend only on k's parity (k > 0)
  auto set_step = [&](int k) {
    double** in = (k & 1) ? Bb : A;
    double** out = (k & 1) ? A : Bb;
    a.h_in = in[0]; a.hu_in = in[1]; a.hw_in = in[2];
    a.h_out = out[0]; a.hu_out = out[1]; a.hw_out = out[2];
    a.pend = (corr && k > 0) ? pend[(k - 1) & 1] : nullptr;
    a.flags_prev = flags[(k - 1) & 1];
    a.pend_out = pend[k & 1];
    a.flags_cur = flags[k & 1];
    a.tile_count = tcount + (k & 1);
    a.tile_count_next = tcount + ((k + 1) & 1);
  };
  auto launch_step = [&](int k, cudaStream_t st) -> int {
    set_step(k);
    void* args[1] = {&a};
    int rc = stream_launch(kp_step, 0, gp, bpp, args, st, kp_smem);
    if (!rc && a.n_gauges > 0)
      rc = stream_launch(nh_stream_kernel(6), 5, dim3((unsigned)(((size_t)B * a.n_gauges + 127) / 128)),
                         dim3(128), args, st);
    if (!rc && w_crit)   // full mask for members whose input hw is identically zero
      rc = stream_launch(nh_stream_kernel(7), 5, dim3((B + 7) / 8), dim3(256), args, st);
    if (!rc && corr && !fused_ks) rc = stream_launch(ks, 1, gs, bp, args, st);
    if (!rc) rc = stream_launch(kx, 2, gx, bx, args, st);
    if (!rc && corr) rc = stream_launch(kc, 3, gc, bp, args, st);
    return rc;
  };
  if (graphs_enabled() && !g_timing.on && n_steps >= 5) {
    // the time loop as a CUDA graph: step 0 directly, then one captured
    // (odd, even) pair of steps replayed, then a trailing odd step if any
    if (int rc = launch_step(0, s)) return rc;
    cudaGraphExec_t exec = nullptr;
    long long nodes = 0;
    if (int rc = pair_graph(a, [&](cudaStream_t cs) -> int {
          int r = launch_step(1, cs);
          return r ? r : launch_step(2, cs);
        }, exec, nodes))
      return rc;
    const int pairs = (n_steps - 1) / 2;
    for (int r = 0; r < pairs; ++r) {
      if (cudaGraphLaunch(exec, s) != cudaSuccess) return NH_E_CUDA;
      g_launches += nodes;
    }
    if ((n_steps - 1) & 1)
      if (int rc = launch_step(n_steps - 1, s)) return rc;
  } else {
    for (int k = 0; k < n_steps; ++k)
      if (int rc = launch_step(k, s)) return rc;
  }
  const int cur = n_steps & 1;   // 1: the final state is in Bb
  double** fin = cur ? Bb : A;
  if (corr) {   // apply the last pending vertical-momentum update in place
    a.h_in = fin[0]; a.hu_in = fin[1]; a.hw_in = fin[2];
    a.pend = pend[(n_steps - 1) & 1];
    a.flags_prev = flags[(n_steps - 1) & 1];
    a.finalize = 1;
    a.tile_count = tcount + ((n_steps - 1) & 1);   // the last step's list of flagged tiles
    void* args[1] = {&a};
    static const bool fin_list = !getenv("NH_KFIN_LIST") || atoi(getenv("NH_KFIN_LIST")) != 0;
    if (fin_list) {
      if (int rc = stream_launch(nh_stream_kfin_ptr(), 4, gc, bpp, args, s, kp_smem)) return rc;
    } else if (int rc = stream_launch(kp, 4, gp, bpp, args, s, kp_smem)) {
      return rc;
    }
  }
  if (cur) {
    for (int f = 0; f < 3; ++f)
      if (cudaMemcpyAsync(A[f], Bb[f], 2 * BN * 8, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return NH_E_CUDA;
  }
  if (outputs && outputs->p_nh && corr) {   // pressure of the last step, 0 off the ranges
    // gather p from the pending record of the last step where its flag is set
    const int last = (n_steps - 1) & 1;
    if (nh_launch_gather_p(pend[last], flags[last], outputs->p_nh, BN, s)) return NH_E_CUDA;
    ++g_launches;
  }
  return 0;
}

int nh_stream_graphs(int enable) {
  const int prev = graphs_enabled() ? 1 : 0;
  if (enable >= 0) g_graphs = enable ? 1 : 0;
  return prev;
}

int nh_stream_timing(int enable) {
  std::lock_guard<std::mutex> lk(g_timing_mu);
  g_timing.on = enable != 0;
  g_timing.used = 0;
  g_timing.marks.clear();
  return 0;
}

int nh_stream_kernel_times(double* ms, long long* launches) {
  std::lock_guard<std::mutex> lk(g_timing_mu);
  for (int k = 0; k < NH_STREAM_NKERNELS; ++k) {
    if (ms) ms[k] = 0.0;
    if (launches) launches[k] = 0;
  }
  if (g_timing.used && cudaEventSynchronize(g_timing.ev[g_timing.used - 1]) != cudaSuccess)
    return NH_E_CUDA;
  for (const auto& m : g_timing.marks) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, g_timing.ev[m.a], g_timing.ev[m.b]) != cudaSuccess)
      return NH_E_CUDA;
    if (ms) ms[m.kernel] += t;
    if (launches) launches[m.kernel] += 1;
  }
  g_timing.used = 0;
  g_timing.marks.clear();
  return 0;
}

long long nh_launch_count(void) { return g_launches.load(); }

int nh_selftest_arith(long long n, unsigned long long seed, unsigned long long* mismatches,
                      void* stream) {
  if (n < 0 || !mismatches) return NH_E_ARG;
  return counted(nh_launch_selftest(n, seed, mismatches, (cudaStream_t)stream));
}

// diagnostics: device buffer [grid][NH_NPHASE] for NH_PROFILE_PHASES builds
void nh_set_profile_buffer(long long* buf) { g_prof = buf; }

const char* nh_last_cuda_error(void) { return cudaGetErrorString(cudaGetLastError()); }

}  // extern "C"
