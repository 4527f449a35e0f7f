// fused_small.cuh -- SURVEY section 2 G7: the whole nested pipeline on chip for a layer with a
// single input channel (Cin_e = 1, e.g. FSRCNN-s conv1 5x5 1 -> 32).  With one input channel the
// contraction of P:110 degenerates to a pointwise product M_xi = V_xi * U_xi[co], so neither V
// nor M needs to leave the SM: per 32-slice chunk a persistent CTA
//   1. computes V = B^T_hat X B_hat for the 32 slices into shared memory (fp32),
//   2. for each group of CO output channels stages U (fp32: hi + lo planes of the plan's filter
//      transform for bf16x3, which makes this path at least as accurate as the split products;
//      hi alone, with V rounded to bf16, for NW_MATH_BF16) and runs the output-transform
//      consumers of output_transform.cuh on rows M = V (.) U produced on the fly.
// HBM traffic is x (once) + y; the path is bound by the CUDA-core transforms.
#pragma once
#include "output_transform.cuh"

namespace nw {

template <int MO, int RO, int MI>
constexpr int X_PA() { return Ax<MO, RO, MI>::PA; }

template <int MO, int RO, int MI, int CO_>
struct FusedC1Shape {
  using X = Ax<MO, RO, MI>;
  using O = OutCfg<MO, RO, MI, 0>;
  static constexpr int SPL = O::SPL;
  static constexpr int CO = CO_;                                // output channels per pass
  static constexpr int WARPS = CO * SPL;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int P = X::PA * X::PA;
  static constexpr int RPV = X::PA + (X::PA & 1);               // V point row padded to float2
  // slice stride in float2 units odd: conflict-free 64-bit loads across the 32 lanes
  static constexpr int VSTR = (X::PA * RPV / 2) % 2 ? X::PA * RPV : X::PA * RPV + 2;
  static constexpr int HSTR = X::L | 1;
  static constexpr size_t V_BYTES = (size_t)32 * VSTR * 4;
  static constexpr size_t H_BYTES = (size_t)32 * X::PA * HSTR * 4;  // pass-1 buffer, reused as output stage
  static constexpr size_t STAGE_BYTES = ((size_t)WARPS * O::YST * 4 + 127) / 128 * 128;
  static constexpr int RPU = X::PA + (X::PA & 1);               // U point row padded to float2
  static constexpr size_t U_BYTES = (size_t)CO * X::PA * RPU * 4;
  static constexpr size_t INFO_BYTES = (size_t)WARPS * 32 * 16;
  static constexpr size_t HS_OR_STAGE = H_BYTES > STAGE_BYTES ? H_BYTES : STAGE_BYTES;
  // U of the current and, where shared memory allows, the next channel group (bulk copies from
  // the prepped fp32 copy; one buffer: the copy is issued and awaited at the group's start)
  static constexpr size_t SMEM1 = 128 + V_BYTES + HS_OR_STAGE + U_BYTES + INFO_BYTES + 16;
  static constexpr int NUB = (SMEM1 + U_BYTES <= 227 * 1024) ? 2 : 1;
  static constexpr size_t SMEM = SMEM1 + (NUB - 1) * U_BYTES;
};

// U (plan layout [P][cout_pad][cin_pad], fp32 or bf16 hi / lo planes) -> Uc, one contiguous block
// per channel group in exactly the shared-memory layout of Us: [group][CO][p_h][RPU] fp32 (zero
// for channels >= Cout_e and the row padding), so the kernel stages a group with one bulk copy
static __global__ void fused_c1_prep_kernel(const void* __restrict__ U, int umode, float* __restrict__ Uc, int PA, int RPU,
                                     int CO, int ngroups, int cout_e, int cout_pad, int cin_pad) {
  const long long n = (long long)ngroups * CO * PA * RPU;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int pw = (int)(i % RPU);
  long long r = i / RPU;
  const int ph = (int)(r % PA);
  const int co = (int)(r / PA);  // group * CO + cl
  float u = 0.f;
  if (co < cout_e && pw < PA) {
    const long long P = (long long)PA * PA;
    const long long o = ((long long)(ph * PA + pw) * cout_pad + co) * cin_pad;  // input channel 0
    if (umode) {  // 1: bf16 hi + lo planes, 2: hi only
      const __nv_bfloat16* Ub = static_cast<const __nv_bfloat16*>(U);
      u = __bfloat162float(Ub[o]) + (umode == 1 ? __bfloat162float(Ub[P * cout_pad * cin_pad + o]) : 0.f);
    } else {
      u = static_cast<const float*>(U)[o];
    }
  }
  Uc[i] = u;
}

// Warps per CTA: the consumers are latency-bound, so as many as registers allow -- 16 (128
// registers) for the column-split 12 x 12 tile, 12 (168) for a 9 x 9 tile held whole (16 spill)
// -- and shared memory allows (F(4,3) (x) F(3,3): 12).
template <int MO, int RO, int MI>
struct FusedC1Cfg
    : FusedC1Shape<MO, RO, MI,
                   (OutCfg<MO, RO, MI, 0>::SPL == 1)
                       ? 12
                       : (FusedC1Shape<MO, RO, MI, 16 / OutCfg<MO, RO, MI, 0>::SPL>::SMEM <= 227 * 1024
                              ? 16 / OutCfg<MO, RO, MI, 0>::SPL
                              : 12 / OutCfg<MO, RO, MI, 0>::SPL)> {};

template <int MO, int RO, int MI, typename XT, typename YT>
__global__ void __launch_bounds__(FusedC1Cfg<MO, RO, MI>::THREADS, 1)
    fused_c1_kernel(const XT* __restrict__ x, const void* __restrict__ Uraw, const float* __restrict__ Uc, int umode,
                    YT* __restrict__ y, Geometry g, const float* __restrict__ slopes, int nchunks) {
  using X = Ax<MO, RO, MI>;
  using C = FusedC1Cfg<MO, RO, MI>;
  using O = OutCfg<MO, RO, MI, 0>;
  constexpr int PA = X::PA, L = X::L, P = C::P;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* base = smem_raw + ((128u - (ptx::smem_u32(smem_raw) & 127u)) & 127u);
  float* Vs = reinterpret_cast<float*>(base);
  float* Hs = reinterpret_cast<float*>(base + C::V_BYTES);      // pass 1, then the output stage
  float* Us2 = reinterpret_cast<float*>(base + C::V_BYTES + C::HS_OR_STAGE);  // NUB x U_BYTES
  long long* sinfo = reinterpret_cast<long long*>(base + C::V_BYTES + C::HS_OR_STAGE + C::NUB * C::U_BYTES);
  uint64_t* ubar =
      reinterpret_cast<uint64_t*>(base + C::V_BYTES + C::HS_OR_STAGE + C::NUB * C::U_BYTES + C::INFO_BYTES);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cw_ = warp / C::SPL, part = warp - cw_ * C::SPL;
  const long long plane = (long long)P * g.cout_pad * g.cin_pad;  // hi -> lo (bf16 elements)
  // prepped U: channel group k of the CTA's sequence (k = local chunk * groups + group) goes to
  // buffer k & 1 by a bulk copy issued one group ahead, so staging U overlaps the previous group
  const int ngroups = (g.cout_e + C::CO - 1) / C::CO;
  const int nloc = (nchunks - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;  // chunks of this CTA
  const long long nseq = (long long)nloc * ngroups;
  constexpr int NUB = C::NUB;
  auto u_issue = [&](long long k) {
    if (k >= nseq) return;
    const int grp = (int)(k % ngroups), b = (int)(k % NUB);
    const uint32_t bar = ptx::smem_u32(&ubar[b]);
    ptx::mbar_expect_tx(bar, (uint32_t)C::U_BYTES);
    ptx::bulk_g2s(ptx::smem_u32(Us2 + b * (C::U_BYTES / 4)), Uc + (long long)grp * (C::U_BYTES / 4),
                  (uint32_t)C::U_BYTES, bar);
  };
  if (Uc) {
    if (tid == 0) {
      for (int b = 0; b < NUB; ++b) ptx::mbar_init(ptx::smem_u32(&ubar[b]), 1);
      ptx::mbar_init_fence();
      if (NUB == 2) u_issue(0);
    }
    __syncthreads();
  }
  long long useq = 0;

  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
    const long long t0 = (long long)chunk * 32;
    // ---- 1. V for the chunk's 32 slices (pass 1 along h into Hs, pass 2 along w into Vs) ----
    for (int task = tid; task < 32 * L; task += C::THREADS) {
      const int s = task % 32, col = task / 32;
      const long long t = t0 + s;
      float xin[L], hv[PA];
      const bool tv = t < g.T;
      long long tt = tv ? t : 0;
      const int aw = (int)(tt % g.tiles_w);
      tt /= g.tiles_w;
      const int ah = (int)(tt % g.tiles_h);
      const int n = (int)(tt / g.tiles_h);
      const int r0 = ah * X::ADV + g.off[0], c = aw * X::ADV + g.off[0] + col;
      const bool cok = tv && c >= 0 && c < g.W;
      const XT* src = x + (long long)n * g.H * g.W + (cok ? c : 0);
#pragma unroll
      for (int r = 0; r < L; ++r) {
        const int gr = r0 + r;
        xin[r] = (cok && gr >= 0 && gr < g.H) ? to_f(src[(long long)gr * g.W]) : 0.f;
      }
      in_axis<MO, RO, MI>(xin, hv);
#pragma unroll
      for (int q = 0; q < PA; ++q) Hs[(s * PA + q) * C::HSTR + col] = hv[q];
    }
    __syncthreads();
    for (int task = tid; task < 32 * PA; task += C::THREADS) {
      const int s = task % 32, p_h = task / 32;
      float hin[L], vv[PA];
#pragma unroll
      for (int k = 0; k < L; ++k) hin[k] = Hs[(s * PA + p_h) * C::HSTR + k];
      in_axis<MO, RO, MI>(hin, vv);
#pragma unroll
      for (int p_w = 0; p_w < PA; ++p_w)
        Vs[s * C::VSTR + p_h * C::RPV + p_w] = (umode == 2) ? __bfloat162float(__float2bfloat16_rn(vv[p_w])) : vv[p_w];
    }
    __syncthreads();
    // ---- 2. output channels in groups of CO: rows of M = V (.) U on the fly ----
    for (int co0 = 0; co0 < g.cout_e; co0 += C::CO, ++useq) {
      float* Us = Us2 + (Uc ? (useq % NUB) * (C::U_BYTES / 4) : 0);
      if (Uc) {
        if (tid == 0) {  // (next) group's U into the free buffer (its readers passed the last barrier)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          u_issue(NUB == 2 ? useq + 1 : useq);
        }
        ptx::mbar_wait(ptx::smem_u32(&ubar[useq % NUB]), (uint32_t)((useq / NUB) & 1));
      } else
      for (int i = tid; i < P * C::CO; i += C::THREADS) {
        const int cl = i % C::CO, xi = i / C::CO, co = co0 + cl;
        float u = 0.f;
        if (co < g.cout_e) {
          const long long o = ((long long)xi * g.cout_pad + co) * g.cin_pad;  // input channel 0
          if (umode) {  // 1: bf16 hi + lo planes, 2: hi only
            const __nv_bfloat16* Ub = static_cast<const __nv_bfloat16*>(Uraw);
            u = __bfloat162float(Ub[o]) + (umode == 1 ? __bfloat162float(Ub[plane + o]) : 0.f);
          } else {
            u = static_cast<const float*>(Uraw)[o];
          }
        }
        Us[(cl * PA + xi / PA) * C::RPU + xi % PA] = u;
      }
      if (!Uc) __syncthreads();
      const int coe = co0 + cw_;
      float* yst = Hs + warp * O::YST;
      long long* info = sinfo + warp * 64;
      auto prod_row = [&](int r, float(&mv)[PA]) {
        // V row of the lane's slice and U row of the warp's channel (broadcast), two points
        // per 64-bit load
        const float2* vr = reinterpret_cast<const float2*>(Vs + lane * C::VSTR + r * C::RPV);
        const float2* ur = reinterpret_cast<const float2*>(Us + (cw_ * PA + r) * C::RPU);
#pragma unroll
        for (int k = 0; k < C::RPU / 2; ++k) {
          const float2 u = ur[k], v = vr[k];
          mv[2 * k] = v.x * u.x;
          if (2 * k + 1 < PA) mv[(2 * k + 1) < PA ? 2 * k + 1 : 0] = v.y * u.y;
        }
      };
      if constexpr (C::SPL == 1) {
        out_unit<MO, RO, MI, YT, 0, 0>(t0, coe, prod_row, yst, info, y, g, slopes);
      } else {
        if (part == 0) out_unit<MO, RO, MI, YT, 0, 0>(t0, coe, prod_row, yst, info, y, g, slopes);
        else out_unit<MO, RO, MI, YT, 0, 1>(t0, coe, prod_row, yst, info, y, g, slopes);
      }
      __syncthreads();  // Us and the stage are rewritten by the next group
    }
  }
}

template <int MO, int RO, int MI, typename XT, typename YT>
static nw_status_t fused_c1_launch(const nw_plan_st* p, const Geometry& g, const void* x, const void* U, void* y,
                                   void* ws, cudaStream_t s) {
  using C = FusedC1Cfg<MO, RO, MI>;
  static_assert(C::SMEM <= 227 * 1024, "fused single-channel kernel exceeds shared memory");
  if (ensure_smem<fused_c1_kernel<MO, RO, MI, XT, YT>>((int)C::SMEM) != NW_OK) return NW_ERR_CUDA;
  const int umode = p->math == NW_MATH_FP32_SIMT ? 0 : (p->math == NW_MATH_BF16 ? 2 : 1);
  float* Uc = static_cast<float*>(ws);
  if (Uc) {  // per-group fp32 copy of U (workspace), bulk-copied by the kernel
    const int ngroups = (g.cout_e + C::CO - 1) / C::CO;
    const long long n = (long long)ngroups * C::CO * X_PA<MO, RO, MI>() * C::RPU;
    LaunchScope scope_("fused_c1_prep", s);
    fused_c1_prep_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(U, umode, Uc, X_PA<MO, RO, MI>(), C::RPU, C::CO,
                                                                     ngroups, g.cout_e, g.cout_pad, g.cin_pad);
    nw_status_t st = check_launch();
    if (st != NW_OK) return st;
  }
  const long long nchunks = (g.T + 31) / 32;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(nchunks < sms ? nchunks : sms);
  LaunchScope scope_("fused_c1", s);
  fused_c1_kernel<MO, RO, MI, XT, YT><<<grid, C::THREADS, C::SMEM, s>>>(
      static_cast<const XT*>(x), U, Uc, umode, static_cast<YT*>(y), g, p->prelu ? p->slopes : nullptr, (int)nchunks);
  return check_launch();
}

template <int MO, int RO, int MI>
nw_status_t fused_c1_impl(const nw_plan_st* p, const Geometry& g, const void* x, const void* U, void* y, void* ws,
                          cudaStream_t s) {
  if constexpr (MI == 3 && Ax<MO, RO, MI>::NPH == 1 && Ax<MO, RO, MI>::PA <= 30) {
    if (p->dtype == NW_DTYPE_BF16)
      return fused_c1_launch<MO, RO, MI, __nv_bfloat16, __nv_bfloat16>(p, g, x, U, y, ws, s);
    return fused_c1_launch<MO, RO, MI, float, float>(p, g, x, U, y, ws, s);
  }
  return NW_ERR_UNSUPPORTED;
}

}  // namespace nw
