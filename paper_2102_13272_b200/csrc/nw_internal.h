// nw_internal.h -- plan structure and launcher declarations shared by the
// library's translation units (not part of the public ABI; see include/nw.h).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <utility>
#include <vector>
#include <cstddef>
#include <cstdint>

#include "../../include/nw.h"
#include "cooktoom.cuh"

namespace nw {

constexpr int kMaxTaps = 12;
constexpr int kGranule = 16;  // tensor-core K / N granule (kind::f16 K = 16, N % 16 == 0 at M = 128)

// Geometry of one layer, computed by the planner (host) and passed by value to
// the kernels.
struct Geometry {
  // per spatial axis (square filters, same on both axes)
  int mode;          // 0 stride 1, 1 stride-2 input phases (Eq. 2.7), 2 transposed output phases
  int SR;            // input-phase stride factor (2 for mode 1, else 1)
  int n_sp;          // stride / output phases per axis (2 for modes 1, 2)
  int Kp;            // taps per phase after the split
  int off[2];        // per phase: mode 0 -pad; mode 1 p - pad; mode 2 -offset (input index offset)
  int taps[2][kMaxTaps];  // per phase tap -> original filter tap index, -1 = zero
  int adv, nph, shift[3];
  // layer
  int N, Cin, Cout, H, W, Ho, Wo;
  int Hq, Wq;        // extent of the stride-1 output grid covered by slices (per phase for mode 2)
  int tiles_h, tiles_w;
  long long T, T_pad;       // slices, padded to the GEMM M tile
  int cin_e, cout_e, cin_pad, cout_pad;
  int P, Pa;
  // path (nested / OLA comparison / direct comparison) and its slice algorithm
  int path;          // kPathNested, kPathOla, kPathDirect
  int mo, ro, mi;    // axis kernel F(mo, ro) (x) F(mi, 3): nested = the plan's; OLA = (1, 1, 3); direct: unused
  int R;             // filter taps per block and axis (3 r_o nested, 3 OLA, 1 direct)
  int nb;            // filter blocks per axis: 1 nested, ceil(Kp/3) OLA (Eq. 2.3), Kp direct (Eq. 2.1 taps)
  int nsh;           // nb^2: contraction K = nsh * cin_pad, A rows shifted per block
  int gemm_ctas;     // persistent contraction grid (0: one CTA per SM)
  int vblk;          // V in the blocked split layout [T_pad/128][P][hi, lo][128][cin_pad] (nested, bf16x3)
  int cs;            // stride 2: ce = (2p + q) * cs + ci (phase-major contraction channels)
  // streamed pipeline (api.cu forward_streamed): per-128-slice-block completion counters the
  // producing kernel releases and the consuming kernel acquires (nullptr: stream-ordered launches)
  int *sync;         // [nmb] input transform -> contraction
  int *sync2;        // [nmb] contraction -> output transform
  int it_ctas;       // persistent input-transform grid (0: every SM)
  int ot_ctas;       // persistent output-transform grid (0: every SM)
};

constexpr int kPathNested = 0, kPathOla = 1, kPathDirect = 2;
constexpr int kMaxShift = 81;

}  // namespace nw

struct nw_plan_st {
  int K, stride, m_o, m_i, Cin, Cout;
  int math = NW_MATH_BF16X3;
  int dtype = NW_DTYPE_F32;
  int transposed = 0, output_padding = 0, outer_taps = 3, pad = -1, prelu = 0, depthwise = 0;
  const float *slopes = nullptr;
  bool finalized = false;
  // derived at finalize
  int Kp = 0, r_o = 0, cin_e = 0, cout_e = 0, cin_pad = 0, cout_pad = 0;
  int cs = 0;  // per-phase channel stride of the stride-2 contraction channels (Cin rounded up to 4)
  nw::NestedAxis ax{};
  // copy streams of nw_conv_forward_host (created on first use, released by nw_plan_destroy)
  std::mutex io_mu;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  // streams of the chunk pipeline inside nw_conv_forward (input / contraction / output)
  cudaStream_t s_pipe[3] = {nullptr, nullptr, nullptr};
  int pipe_chunks = -1;  // batch chunks of the forward pipeline (-1: NW_PIPE_CHUNKS or the default)
  // ordering events of nw_conv_forward_host / the chunk pipeline, created once and reused:
  // the host path enqueues under io_mu, the pipeline under pipe_mu (a stream wait captures the
  // event's latest record when it is enqueued, so re-recording by a later call is safe)
  std::mutex pipe_mu;
  std::vector<cudaEvent_t> ev_host, ev_pipe;
  ~nw_plan_st();
};

namespace nw {

extern std::atomic<unsigned long long> g_launches;

nw_status_t finalize(nw_plan_st *p);
Geometry make_geometry(const nw_plan_st *p, int N, int H, int W, int path = kPathNested);
size_t v_bytes(const nw_plan_st *p, const Geometry &g);
size_t m_bytes(const nw_plan_st *p, const Geometry &g);
size_t u_bytes(const Geometry &g);  // P * cout_pad * nsh * cin_pad * 4
size_t filter_bytes(const nw_plan_st *p);
NestedAxis path_axis(const nw_plan_st *p, int path);
// forward pipeline: chunks of the batch and the workspace of nw_conv_forward
int forward_chunks(const nw_plan_st *p, int N, int H, int W);
size_t forward_ws_bytes(const nw_plan_st *p, int N, int H, int W);

// launchers (nested_kernels.cu)
nw_status_t launch_filter_transform(const nw_plan_st *p, const Geometry &g, const void *w, void *U,
                                    cudaStream_t s);
// direct comparison path (comparison.cu): NCHW x -> shifted-pixel-grid V; M -> y
nw_status_t launch_pack_input(const nw_plan_st *p, const Geometry &g, const void *x, void *V, cudaStream_t s);
nw_status_t launch_unpack_output(const nw_plan_st *p, const Geometry &g, const float *M, void *y, cudaStream_t s);
nw_status_t launch_input_transform(const nw_plan_st *p, const Geometry &g, const void *x, void *V,
                                   cudaStream_t s);
nw_status_t launch_output_transform(const nw_plan_st *p, const Geometry &g, const float *M, void *y,
                                    cudaStream_t s);
nw_status_t launch_gemm_simt(const nw_plan_st *p, const Geometry &g, const float *V, const float *U,
                             float *M, cudaStream_t s);
// tcgen05 contraction (tc_gemm.cu)
bool gemm_fused_eligible(const nw_plan_st *p, const Geometry &g);
nw_status_t launch_gemm_tc_fused(const nw_plan_st *p, const Geometry &g, const void *V, const void *U, float *Mp,
                                 cudaStream_t s);
// fusion level of the contraction epilogue: 0 plain (M), 1 inner output level along w (M'),
// 2 inner level along both axes (M'' = (m_i / l_i)^2 of M)
int gemm_fused_level(const nw_plan_st *p, const Geometry &g);
// wide layers (Cout_pad 128 / 256): level 1 with 128-channel CTAs (pairs multicast the A tiles)
bool gemm_fused_wide(const nw_plan_st *p, const Geometry &g);
nw_status_t launch_gemm_tc_fused1c(const nw_plan_st *p, const Geometry &g, const void *V, const void *U, float *Mp,
                                   cudaStream_t s);
nw_status_t launch_gemm_tc_fused2(const nw_plan_st *p, const Geometry &g, const void *V, const void *U, float *Mpp,
                                  cudaStream_t s);
nw_status_t launch_output_transform_pre2(const nw_plan_st *p, const Geometry &g, const float *Mpp, void *y,
                                         cudaStream_t s);
// output transform of a fused contraction: M holds M' (inner w level applied)
nw_status_t launch_output_transform_pre(const nw_plan_st *p, const Geometry &g, const float *Mp, void *y,
                                        cudaStream_t s);
nw_status_t launch_gemm_tc(const nw_plan_st *p, const Geometry &g, const void *V, const void *U,
                           float *M, cudaStream_t s);
// depthwise layers: per-channel transform-domain product (depthwise.cu)
nw_status_t launch_depthwise_product(const nw_plan_st *p, const Geometry &g, const void *V, const float *U, float *M,
                                     cudaStream_t s);
// layers with Cout_e <= 4: the whole nested pipeline in one kernel (fused_smallout.cuh); ws holds
// the compact U copy (Cin_e * P * 16 bytes)
bool fused_co_eligible(const nw_plan_st *p, const Geometry &g);
nw_status_t launch_fused_co(const nw_plan_st *p, const Geometry &g, const void *x, const void *U, void *y, void *ws,
                            cudaStream_t s);
// single-input-channel layers: the whole nested pipeline in one kernel (fused_small.cuh)
bool fused_c1_eligible(const nw_plan_st *p, const Geometry &g);
// ws (>= fused_c1_ws_bytes, or nullptr) receives the per-channel-group fp32 copy of U that the
// kernel bulk-copies into shared memory
nw_status_t launch_fused_c1(const nw_plan_st *p, const Geometry &g, const void *x, const void *U, void *y,
                            void *ws, size_t ws_bytes, cudaStream_t s);
size_t fused_c1_ws_bytes(const nw_plan_st *p, const Geometry &g);

// Launch with programmatic stream serialization (PDL): the kernel may start while the
// previous kernel in the stream drains; it calls griddepcontrol.wait before reading
// dependent data.  Opt-in with NW_PDL=1; otherwise a plain launch.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline nw_status_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...) == cudaSuccess ? NW_OK : NW_ERR_CUDA;
}

// RAII: when profiling is on, brackets one launch with CUDA events on its stream.
class LaunchScope {
 public:
  LaunchScope(const char *kind, cudaStream_t s);
  ~LaunchScope();
  LaunchScope(const LaunchScope &) = delete;
  LaunchScope &operator=(const LaunchScope &) = delete;

 private:
  const char *kind_;
  cudaStream_t s_;
  cudaEvent_t a_ = nullptr, b_ = nullptr;
};

inline nw_status_t check_launch() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError() == cudaSuccess ? NW_OK : NW_ERR_CUDA;
}

inline long long round_up(long long a, long long b) { return (a + b - 1) / b * b; }

// Raise kernel KERN's dynamic shared-memory limit once per device (function attributes are
// per device; one bit per device id, thread-safe).
template <auto KERN>
inline nw_status_t ensure_smem(int bytes) {
  static std::atomic<unsigned long long> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return NW_ERR_CUDA;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return NW_OK;
  if (cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return NW_ERR_CUDA;
  done.fetch_or(bit, std::memory_order_release);
  return NW_OK;
}

}  // namespace nw
