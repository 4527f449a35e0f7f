// fused_smallout.cuh -- the whole nested pipeline in one kernel for layers with at most four
// contraction outputs (Cout_e <= 4): the FSRCNN-s 9x9 stride-2 deconvolution of BASELINE
// config 5 (32 -> 1, four output phases, R11) and Table I's SRCNN 5x5 1 <- 32.
//
// With Cout_e <= 4 the contraction of P:110 / Eq. 2.1 is 4 multiply-adds per V value, so the
// transform domain never needs to leave the SM: a persistent CTA takes a chunk of S slices of
// one tile row and keeps M = sum_c V_c (.) U_c in registers -- thread (slice s, point row p_h)
// owns the P_a x 4 accumulators of its row -- while it walks the input channels:
//   loads   a ring of NSTG stages, each one channel: a TMA box {window columns, L rows} of x
//           (zero fill outside the image = the padding; start rounded down to 16 bytes) and a
//           bulk copy of U_c (a compact [Cin_e][P][4] fp32 copy the prep kernel writes into the
//           workspace), both completing on one mbarrier; a stage is refilled NSTG channels ahead
//   pass 1  thread = (slice, window column): B^T_hat along h -> Hs[s][p_h][col]
//   pass 2  thread = (slice, p_h): B^T_hat along w -> V row, acc[p_w][co] += V[p_w] U_c[p_h, p_w][co]
//           (pass 2 of channel c and pass 1 of channel c + 1 share one barrier: Hs is double
//           buffered)
//   then    A^T_hat along w in registers -> Q[s][co][p_h][q_w] (shared), A^T_hat along h per
//           (slice, co, q_w), crop / depth-to-space, store.
// HBM traffic is x (once) + y: C5's deconvolution no longer writes and reads its 4.6 GB V.
// Arithmetic is fp32 (U = hi + lo for bf16x3, exact in fp32), like fused_c1.
#pragma once
#include "ptx.cuh"
#include "transforms.cuh"

namespace nw {

template <int MO, int RO, int MI>
struct FusedCoCfg {
  using X = Ax<MO, RO, MI>;
  static constexpr int PA = X::PA, L = X::L, MA = X::MA, P = PA * PA;
  static constexpr int CO = 4;                          // output lanes of the accumulators
  static constexpr int S = 300 / PA;                    // slices per chunk (12 for P_a 25, 10 for 30)
  static constexpr int ROWS = S * PA;                   // pass-2 threads
  static constexpr int THREADS = (ROWS + 31) / 32 * 32;
  static constexpr int HSTR = L | 1;
  static constexpr int HS = S * PA * HSTR;              // floats per buffer
  static constexpr int QSTR = MA | 1;
  static constexpr int QS = S * CO * PA * QSTR;         // floats (aliases the Hs buffers)
  static constexpr size_t HS_BYTES = (size_t)2 * HS * 4;
  static constexpr size_t Q_BYTES = (size_t)QS * 4;
  static constexpr size_t BUF_BYTES = ((HS_BYTES > Q_BYTES ? HS_BYTES : Q_BYTES) + 15) / 16 * 16;
  static constexpr int NSTG = 3;                        // load ring depth (channels in flight)
  static constexpr size_t U_STAGE = (size_t)P * 16;     // one channel of U_c (float4 per point)
  static constexpr int WC = (S - 1) * X::ADV + L;       // window columns of a full chunk
  template <typename XT>
  static constexpr int bw() {                           // TMA box width: 16-byte start + multiple
    constexpr int al = 16 / (int)sizeof(XT);
    return (WC + al - 1 + al - 1) / al * al;
  }
  template <typename XT>
  static constexpr size_t win_stage() { return ((size_t)L * bw<XT>() * sizeof(XT) + 1023) / 1024 * 1024; }
  template <typename XT>
  static constexpr size_t smem() {
    return BUF_BYTES + NSTG * (U_STAGE + win_stage<XT>()) + 1024 + 64;
  }
};

// U (plan layout [P][cout_pad][cin_pad], fp32 or bf16 hi / lo planes) -> U4 [cin_e][P][4] fp32
__global__ void fused_co_prep_kernel(const void* __restrict__ U, int umode, float4* __restrict__ U4, int P,
                                     int cout_e, int cout_pad, int cin_e, int cin_pad) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)cin_e * P) return;
  const int c = (int)(i / P), xi = (int)(i % P);
  float u[4];
  const long long plane = (long long)P * cout_pad * cin_pad;
#pragma unroll
  for (int co = 0; co < 4; ++co) {
    u[co] = 0.f;
    if (co < cout_e) {
      const long long o = ((long long)xi * cout_pad + co) * cin_pad + c;
      if (umode) {
        const __nv_bfloat16* Ub = static_cast<const __nv_bfloat16*>(U);
        u[co] = __bfloat162float(Ub[o]) + __bfloat162float(Ub[plane + o]);
      } else {
        u[co] = static_cast<const float*>(U)[o];
      }
    }
  }
  U4[i] = make_float4(u[0], u[1], u[2], u[3]);
}

// The P_a x 4 channel-sum accumulators of one (slice, p_h) row.  Packed (PK): output lanes
// (0, 1) and (2, 3) in f32x2 pairs, two FFMA2 (the V value as a broadcast scalar operand) per
// V value instead of four FFMA, same per-lane rounding.  Measured 4 % SLOWER on C5's
// deconvolution (1.37 -> 1.42 ms) and Table I's SRCNN 5x5 1 <- 32 (0.123 -> 0.128 ms): the
// aligned register pairs cost moves and the kernel is not issue-bound there; so the scalar form
// runs (the packed one stays for the record, and spills at P_a = 30 under 10 warps' 168-register
// cap).
template <int PA, bool PK>
struct CoAcc {
  float a[PA][4];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int p = 0; p < PA; ++p)
#pragma unroll
      for (int k = 0; k < 4; ++k) a[p][k] = 0.f;
  }
  __device__ __forceinline__ void fma(int p, float v, const float4& u) {
    a[p][0] = fmaf(v, u.x, a[p][0]);
    a[p][1] = fmaf(v, u.y, a[p][1]);
    a[p][2] = fmaf(v, u.z, a[p][2]);
    a[p][3] = fmaf(v, u.w, a[p][3]);
  }
  __device__ __forceinline__ float get(int p, int co) const { return a[p][co]; }
};
template <int PA>
struct CoAcc<PA, true> {
  f2 a01[PA], a23[PA];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int p = 0; p < PA; ++p) a01[p] = a23[p] = f2_splat(0.f);
  }
  __device__ __forceinline__ void fma(int p, float v, const float4& u) {
    a01[p] = fmaf(v, f2_pack(u.x, u.y), a01[p]);
    a23[p] = fmaf(v, f2_pack(u.z, u.w), a23[p]);
  }
  __device__ __forceinline__ float get(int p, int co) const {
    float x0, x1;
    f2_unpack(co < 2 ? a01[p] : a23[p], x0, x1);
    return (co & 1) ? x1 : x0;
  }
};

template <int MO, int RO, int MI, typename XT, typename YT>
__global__ void __launch_bounds__(FusedCoCfg<MO, RO, MI>::THREADS, 1)
    fused_co_kernel(const __grid_constant__ CUtensorMap mapX, const float4* __restrict__ U4, YT* __restrict__ y,
                    Geometry g, int wchunks, int nchunks) {
  using X = Ax<MO, RO, MI>;
  using C = FusedCoCfg<MO, RO, MI>;
  constexpr int PA = C::PA, L = C::L, MA = C::MA, P = C::P, S = C::S, CO = C::CO, NSTG = C::NSTG;
  constexpr int BW = C::template bw<XT>(), AL = 16 / (int)sizeof(XT);
  constexpr size_t WST = C::template win_stage<XT>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* wring = base;                                            // NSTG x WST (TMA boxes)
  float4* Us = reinterpret_cast<float4*>(base + NSTG * WST);              // NSTG x P
  float* Hbuf = reinterpret_cast<float*>(base + NSTG * (WST + C::U_STAGE));  // 2 x HS, later Q
  uint64_t* full = reinterpret_cast<uint64_t*>(base + NSTG * (WST + C::U_STAGE) + C::BUF_BYTES);
  const int tid = threadIdx.x;
  // pass-2 / w-output role: (slice, p_h), slice fastest, so the 32 lanes of a warp share two or
  // three point rows p_h and their U_c row loads (LDS.128 per point) are broadcasts; with p_h
  // fastest every lane read its own U row (~0.5 ms of shared-memory wavefronts per C5 layer)
  const int ph2 = tid / S, s2 = tid - (tid / S) * S;
  const bool row_thread = tid < C::ROWS;
  const int cin = g.cin_e;

  // chunk k of this CTA -> (image n, tile row ah, first tile aw0, slices)
  auto chunk_of = [&](int chunk, int& n, int& ah, int& aw0) {
    const int wc = chunk % wchunks;
    const int r = chunk / wchunks;
    ah = r % g.tiles_h;
    n = r / g.tiles_h;
    aw0 = wc * S;
  };
  // stage q (global channel counter of this CTA: q = local chunk * cin + c) -> ring slot q % NSTG
  auto issue = [&](long long q) {
    const int lc = (int)(q / cin), c = (int)(q % cin);
    const int chunk = blockIdx.x + lc * gridDim.x;
    if (chunk >= nchunks) return;
    int n, ah, aw0;
    chunk_of(chunk, n, ah, aw0);
    const int st = (int)(q % NSTG);
    const uint32_t bar = ptx::smem_u32(&full[st]);
    ptx::mbar_expect_tx(bar, (uint32_t)(L * BW * sizeof(XT) + C::U_STAGE));
    const int col0 = (aw0 * X::ADV + g.off[0]) & ~(AL - 1);
    ptx::tma_load_3d(ptx::smem_u32(wring + st * WST), &mapX, bar, col0, ah * X::ADV + g.off[0], n * g.Cin + c);
    ptx::bulk_g2s(ptx::smem_u32(Us + st * P), U4 + (long long)c * P, (uint32_t)C::U_STAGE, bar);
  };

  if (tid == 0) {
    ptx::tma_prefetch(&mapX);
    for (int i = 0; i < NSTG; ++i) ptx::mbar_init(ptx::smem_u32(&full[i]), 1);
    ptx::mbar_init_fence();
  }
  __syncthreads();
  if (tid == 0)
    for (int i = 0; i < NSTG; ++i) issue(i);

  long long q0 = 0;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, q0 += cin) {
    int n, ah, aw0;
    chunk_of(chunk, n, ah, aw0);
    const int ns = min(S, g.tiles_w - aw0);                   // slices of this chunk
    const long long t0 = ((long long)n * g.tiles_h + ah) * g.tiles_w + aw0;
    const int sh = (aw0 * X::ADV + g.off[0]) & (AL - 1);      // window start inside the aligned box
    // pass 1 of the channel in ring stage q into Hs buffer b
    auto pass1 = [&](long long q, int b) {
      const int st = (int)(q % NSTG);
      ptx::mbar_wait(ptx::smem_u32(&full[st]), (uint32_t)((q / NSTG) & 1));
      const XT* win = reinterpret_cast<const XT*>(wring + st * WST) + sh;
      float* Hs = Hbuf + b * C::HS;
      // two window columns per thread (FADD2 / FFMA2) spill: the P_a x 4 accumulators are live
      // across pass 1 of the next channel, so pass 1 stays scalar here
      if constexpr (false && kPackedAxis<MO, RO, MI>) {
        for (int task = tid; task < S * L; task += 2 * C::THREADS) {
          const int s = task / L, col = task - (task / L) * L;
          const XT* src = win + s * X::ADV + col;
          const int tb = task + C::THREADS;
          if (tb < S * L) {
            const int sb = tb / L, colb = tb - (tb / L) * L;
            const XT* srcb = win + sb * X::ADV + colb;
            f2 xin[L], hv[PA];
#pragma unroll
            for (int r = 0; r < L; ++r) xin[r] = f2_pack(to_f(src[r * BW]), to_f(srcb[r * BW]));
            in_axis_t<MO, RO, MI, f2>(xin, hv);
#pragma unroll
            for (int p = 0; p < PA; ++p)
              f2_unpack(hv[p], Hs[(s * PA + p) * C::HSTR + col], Hs[(sb * PA + p) * C::HSTR + colb]);
          } else {
            float xin[L], hv[PA];
#pragma unroll
            for (int r = 0; r < L; ++r) xin[r] = to_f(src[r * BW]);
            in_axis<MO, RO, MI>(xin, hv);
#pragma unroll
            for (int p = 0; p < PA; ++p) Hs[(s * PA + p) * C::HSTR + col] = hv[p];
          }
        }
      } else {
        for (int task = tid; task < S * L; task += C::THREADS) {
          const int s = task / L, col = task - (task / L) * L;
          float xin[L], hv[PA];
          const XT* src = win + s * X::ADV + col;
#pragma unroll
          for (int r = 0; r < L; ++r) xin[r] = to_f(src[r * BW]);
          in_axis<MO, RO, MI>(xin, hv);
#pragma unroll
          for (int p = 0; p < PA; ++p) Hs[(s * PA + p) * C::HSTR + col] = hv[p];
        }
      }
    };
    CoAcc<PA, false> acc;
    acc.zero();
    pass1(q0, 0);
    __syncthreads();
    for (int c = 0; c < cin; ++c) {
      const long long q = q0 + c;
      const int b = c & 1;
      if (row_thread) {  // pass 2 of channel c + the channel sum
        const float* h = Hbuf + b * C::HS + (s2 * PA + ph2) * C::HSTR;
        float hin[L], v[PA];
#pragma unroll
        for (int k = 0; k < L; ++k) hin[k] = h[k];
        in_axis<MO, RO, MI>(hin, v);
        const float4* u = Us + (q % NSTG) * P + ph2 * PA;
#pragma unroll
        for (int pw = 0; pw < PA; ++pw) {
          acc.fma(pw, v[pw], u[pw]);
        }
      }
      if (c + 1 < cin) pass1(q + 1, b ^ 1);
      __syncthreads();   // stage q: window read (pass 1 of channel c) and U_c read (pass 2): free
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(q + NSTG);
      }
    }
    // ---- output transform: A^T_hat along w in registers, then along h per column ----
    float* Q = Hbuf;  // reuses the pass-1 buffers (every thread is past its last read)
    if (row_thread && s2 < ns) {
#pragma unroll
      for (int co = 0; co < CO; ++co) {
        if (co < g.cout_e) {
          float m[PA], yq[MA];
#pragma unroll
          for (int p = 0; p < PA; ++p) m[p] = acc.get(p, co);
          out_axis<MO, RO, MI>(m, yq);
          float* qd = Q + ((s2 * CO + co) * PA + ph2) * C::QSTR;
#pragma unroll
          for (int qq = 0; qq < MA; ++qq) qd[qq] = yq[qq];
        }
      }
    }
    __syncthreads();
    const long long HoWo = (long long)g.Ho * g.Wo;
    for (int task = tid; task < S * CO * MA; task += C::THREADS) {
      const int qw = task % MA, r = task / MA;
      const int co = r % CO, s = r / CO;
      if (s >= ns || co >= g.cout_e) continue;
      float col[PA], yh[MA];
#pragma unroll
      for (int p = 0; p < PA; ++p) col[p] = Q[((s * CO + co) * PA + p) * C::QSTR + qw];
      out_axis<MO, RO, MI>(col, yh);
      const int gi0 = ah * X::ADV, gj0 = (aw0 + s) * X::ADV + qw;   // m_i = 3: output q lands at q
      if (g.mode == 2) {  // transposed: output phase f = (fo_h, fo_w) of channel c (R11)
        const int f = co / g.Cout, c = co % g.Cout, fo_h = f / 2, fo_w = f % 2;
        if (2 * gj0 + fo_w >= g.Wo) continue;
        YT* dst = y + ((long long)n * g.Cout + c) * HoWo + (2 * gj0 + fo_w);
#pragma unroll
        for (int qh = 0; qh < MA; ++qh) {
          const int row = 2 * (gi0 + qh) + fo_h;
          if (row < g.Ho) dst[(long long)row * g.Wo] = from_f<YT>(yh[qh]);
        }
      } else {
        if (gj0 >= g.Wo) continue;
        YT* dst = y + ((long long)n * g.Cout + co) * HoWo + gj0;
#pragma unroll
        for (int qh = 0; qh < MA; ++qh)
          if (gi0 + qh < g.Ho) dst[(long long)(gi0 + qh) * g.Wo] = from_f<YT>(yh[qh]);
      }
    }
    (void)t0;
    __syncthreads();  // Q (the Hs buffers) is rewritten by the next chunk's pass 1
  }
}

template <int MO, int RO, int MI, typename XT, typename YT>
static nw_status_t fused_co_launch(const nw_plan_st* p, const Geometry& g, const void* x, const void* U, void* y,
                                   void* ws, cudaStream_t s) {
  using C = FusedCoCfg<MO, RO, MI>;
  constexpr size_t SMEM = C::template smem<XT>();
  static_assert(SMEM <= 227 * 1024, "fused small-output kernel exceeds shared memory");
  if (((long long)g.W * sizeof(XT)) % 16 != 0) return NW_ERR_UNSUPPORTED;  // TMA row pitch
  float4* U4 = static_cast<float4*>(ws);
  {
    const long long n = (long long)g.cin_e * C::P;
    LaunchScope scope_("fused_co_prep", s);
    fused_co_prep_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
        U, p->math == NW_MATH_FP32_SIMT ? 0 : 1, U4, C::P, g.cout_e, g.cout_pad, g.cin_e, g.cin_pad);
    nw_status_t st = check_launch();
    if (st != NW_OK) return st;
  }
  const uint64_t dims[3] = {(uint64_t)g.W, (uint64_t)g.H, (uint64_t)g.N * g.Cin};
  const uint64_t strides[2] = {(uint64_t)g.W * sizeof(XT), (uint64_t)g.H * g.W * sizeof(XT)};
  const uint32_t box[3] = {(uint32_t)C::template bw<XT>(), (uint32_t)C::L, 1u};
  alignas(64) CUtensorMap mapX;
  if (!encode_tmap(&mapX, sizeof(XT) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, x,
                   dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE))
    return NW_ERR_CUDA;
  if (ensure_smem<fused_co_kernel<MO, RO, MI, XT, YT>>((int)SMEM) != NW_OK) return NW_ERR_CUDA;
  const int wchunks = (g.tiles_w + C::S - 1) / C::S;                // row-aligned chunks
  const long long nchunks = (long long)g.N * g.tiles_h * wchunks;
  if (nchunks >= (1ll << 31)) return NW_ERR_UNSUPPORTED;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(nchunks < sms ? nchunks : sms);
  LaunchScope scope_("fused_co", s);
  fused_co_kernel<MO, RO, MI, XT, YT><<<grid, C::THREADS, SMEM, s>>>(mapX, U4, static_cast<YT*>(y), g, wchunks,
                                                                      (int)nchunks);
  return check_launch();
}

template <int MO, int RO, int MI>
nw_status_t fused_co_impl(const nw_plan_st* p, const Geometry& g, const void* x, const void* U, void* y, void* ws,
                          cudaStream_t s) {
  if constexpr (MI == 3 && Ax<MO, RO, MI>::NPH == 1 && (Ax<MO, RO, MI>::PA == 25 || Ax<MO, RO, MI>::PA == 30)) {
    if (p->dtype == NW_DTYPE_BF16)
      return fused_co_launch<MO, RO, MI, __nv_bfloat16, __nv_bfloat16>(p, g, x, U, y, ws, s);
    return fused_co_launch<MO, RO, MI, float, float>(p, g, x, U, y, ws, s);
  }
  return NW_ERR_UNSUPPORTED;
}

}  // namespace nw
