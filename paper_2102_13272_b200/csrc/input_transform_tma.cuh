// input_transform_tma.cuh -- G2 on sm_100a: nested input transform V = B^T_hat X B_hat
// as a persistent kernel fed by TMA halo-tile loads.
//
// Persistent CTAs walk tasks (image n, tile row a_h, TW = 2 adjacent tiles along w, CC = 32
// source channels -- 16 warps, one CTA per SM; CC = 16: 8 warps, two CTAs per SM), channel
// group fastest so the CTAs filling one 128-byte V row run side by side.  Per task:
//   TMA     one 3-D box {window columns (+ up to 15 bytes so it starts 16-byte aligned),
//           L rows, 16 channels} of x [N*Cin][H][W] lands in the CTA's window buffer;
//           coordinates outside the image are zero-filled by the copy engine (= the
//           convolution's zero padding), so there are no bounds tests.  The next task's box is
//           issued as soon as pass 1 has read the buffer, so it lands during pass 2 (and while
//           an SM's other CTA computes).
//   pass 1  thread = (channel, window column): B^T_hat along h (both levels, factored 1-D
//           kernels of transforms.cuh) -> Hs[p_h][channel][column], fp32.
//   pass 2  lane = (channel pair, (p_h, tile) combo): the L-long row of Hs along w -> P_a
//           values per channel, split into bf16 hi / lo (one cvt.rn.bf16x2 per plane) and
//           stored straight into the blocked V layout [T_pad/128][P][hi, lo][128][CINP] (the
//           contraction's TMA A operand) from one base pointer per lane (immediate offsets).
// Arithmetic is the same sequence of fp32 operations as input_transform_kernel, so V is
// bit-identical to it (tests/test_gpu_env_variants.py checks with NW_INPUT_TMA=0).
// Measured variants (profiles/r2_input_transform.md): a staged form (one CTA per SM, double-
// buffered window, per-warp V stage copied out with 16-byte stores) was 1.2-1.5x slower (more
// instructions, 8 warps per SM); this kernel beats the first-round one on bf16 x (C3) and
// loses on fp32 x (C2), so it runs for bf16 x only (input_tma_eligible).
#pragma once
#include <cstdlib>

#include "ptx.cuh"
#include "transforms.cuh"

namespace nw {

template <int MO, int RO, int MI, typename XT, int CC_>
struct ItCfg {
  using X = Ax<MO, RO, MI>;
  static constexpr int CC = CC_;                        // source channels per task (16 or 32)
  static constexpr int NPR = CC / 2;                    // channel pairs: lanes per combo in pass 2
  static constexpr int SUBS = 32 / NPR;                 // combos per warp pass
  static constexpr int TW = 2;                          // tiles per task along w
  static constexpr int ES = (int)sizeof(XT);
  static constexpr int WC = (TW - 1) * X::ADV + X::L;   // window columns used
  // The box starts on a 16-byte boundary of the x row (a tiled TMA load whose inner start
  // coordinate is not 16-byte aligned faults with "illegal instruction" on sm_100a, measured):
  // the start is rounded down by up to AL - 1 elements and the box widened to cover it.
  static constexpr int AL = 16 / ES;                    // elements per 16 bytes
  static constexpr int BW = (WC + AL - 1 + AL - 1) / AL * AL;  // box width: 16-byte multiple
  static constexpr int L = X::L;
  static constexpr int PA = X::PA;
  static constexpr int STAGE = (CC * L * BW * ES + 1023) / 1024 * 1024;
  static constexpr int HSTR = WC | 1;                   // odd row pitch of Hs (bank spread)
  static constexpr int HS = PA * CC * HSTR;             // floats
  static constexpr int COMBOS = PA * TW;                // (p_h, tile) rows of pass 2
  static constexpr int GROUPS = (COMBOS + SUBS - 1) / SUBS;  // SUBS combos x NPR pairs per warp pass
  // 16 channels: 8 warps, two CTAs per SM; 32 channels: 16 warps, one CTA per SM (shared memory)
  static constexpr int WARPS = CC == 16 ? 8 : 16;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int MINB = CC == 16 ? 2 : 1;         // <= 128 registers either way
  static constexpr size_t SMEM = (size_t)STAGE + (size_t)HS * 4 + 64;
  static_assert(BW <= 256 && L <= 256, "TMA box");
};

template <int MO, int RO, int MI, typename XT, int CINP, int CC_>
__global__ void __launch_bounds__(ItCfg<MO, RO, MI, XT, CC_>::THREADS, ItCfg<MO, RO, MI, XT, CC_>::MINB)
    input_transform_tma_kernel(const __grid_constant__ CUtensorMap mapX, void* __restrict__ Vout, Geometry g,
                               int cgroups, int wgroups, int ntasks) {
  using X = Ax<MO, RO, MI>;
  using C = ItCfg<MO, RO, MI, XT, CC_>;
  constexpr int PA = X::PA, L = X::L, CC = C::CC;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* stage = smem;                                   // window (one buffer)
  float* Hs = reinterpret_cast<float*>(smem + C::STAGE);         // HS floats
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGE + C::HS * 4);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grid = gridDim.x;

  auto issue = [&](int task, int s) {  // one TMA box for task -> stage s
    int b = task;
    const int cg = b % cgroups;
    b /= cgroups;
    const int wg = b % wgroups;
    b /= wgroups;
    const int ah = b % g.tiles_h;
    const int n = b / g.tiles_h;
    const int row0 = ah * X::ADV + g.off[0];
    const int col0 = (wg * C::TW * X::ADV + g.off[0]) & ~(C::AL - 1);  // 16-byte aligned start
    const uint32_t bar = ptx::smem_u32(&full[s]);
    ptx::mbar_expect_tx(bar, (uint32_t)(CC * L * C::BW * C::ES));
    ptx::tma_load_3d(ptx::smem_u32(stage + (size_t)s * C::STAGE), &mapX, bar, col0, row0, n * g.Cin + cg * CC);
  };

  if (tid == 0) {
    ptx::tma_prefetch(&mapX);
    ptx::mbar_init(ptx::smem_u32(&full[0]), 1);
    ptx::mbar_init_fence();
  }
  __syncthreads();
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();  // x may come from the previous kernel in the stream
  if (tid == 0 && blockIdx.x < ntasks) issue(blockIdx.x, 0);

  int it = 0;
#pragma unroll 1
  for (int task = blockIdx.x; task < ntasks; task += grid, ++it) {
    int b = task;
    const int cg = b % cgroups;
    b /= cgroups;
    const int wg = b % wgroups;
    b /= wgroups;
    const int ah = b % g.tiles_h;
    const int n = b / g.tiles_h;
    const int aw0 = wg * C::TW;
    const int sh = (aw0 * X::ADV + g.off[0]) & (C::AL - 1);  // window start inside the aligned box
    const XT* win = reinterpret_cast<const XT*>(stage) + sh;
    ptx::mbar_wait(ptx::smem_u32(&full[0]), (uint32_t)(it & 1));

    // ---------------- pass 1: columns along h (window -> Hs) ----------------
#pragma unroll 1
    for (int t1 = tid; t1 < CC * C::WC; t1 += C::THREADS) {
      const int col = t1 % C::WC, c = t1 / C::WC;
      const XT* src = win + (c * L) * C::BW + col;
      float xin[L], hv[PA];
#pragma unroll
      for (int r = 0; r < L; ++r) xin[r] = to_f(src[r * C::BW]);
      in_axis<MO, RO, MI>(xin, hv);
      float* dst = Hs + c * C::HSTR + col;
#pragma unroll
      for (int q = 0; q < PA; ++q) dst[q * CC * C::HSTR] = hv[q];
    }
    __syncthreads();  // window consumed, Hs complete
    if (tid == 0 && task + grid < ntasks) {  // refill: the next window lands during pass 2
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the async refill
      issue(task + grid, 0);
    }

    // ---------------- pass 2: rows along w, split, store V ----------------
    const int pair = lane % C::NPR, sub = lane / C::NPR;
#pragma unroll 1
    for (int grp = warp; grp < C::GROUPS; grp += C::WARPS) {
      const int q = grp * C::SUBS + sub;            // (p_h, tile) combo of this lane
      const int ph = q / C::TW, tile = q % C::TW;
      const bool live = q < C::COMBOS && aw0 + tile < g.tiles_w;
      if (live) {
        const float* h0 = Hs + (ph * CC + 2 * pair) * C::HSTR + tile * X::ADV;
        const float* h1 = h0 + C::HSTR;
        float za[X::LO][X::LI], zb[X::LO][X::LI];
        {
          float a[L], bb[L];
#pragma unroll
          for (int k = 0; k < L; ++k) {
            a[k] = h0[k];
            bb[k] = h1[k];
          }
          in_axis_inner<MO, RO, MI>(a, za);
          in_axis_inner<MO, RO, MI>(bb, zb);
        }
        // straight to V: one base pointer per lane, every store an immediate offset from it
        const long long t = ((long long)n * g.tiles_h + ah) * g.tiles_w + aw0 + tile;
        const long long row = (((t >> 7) * g.P + (long long)ph * PA) * 2) * 128 + (t & 127);
        char* hp = reinterpret_cast<char*>(Vout) + (row * CINP + cg * CC + 2 * pair) * 2;
        store_row_imm<MO, RO, MI, CINP>(za, zb, hp);
      }
    }
    __syncthreads();  // Hs free for the next task's pass 1 (and this task's V stores are done)
    if (g.sync && tid == 0) {  // streamed pipeline: count (slice, source channel) completions per block
      const long long t0 = ((long long)n * g.tiles_h + ah) * g.tiles_w + aw0;
      const int nt = min(C::TW, g.tiles_w - aw0);
      const long long t1 = t0 + nt - 1;
      if ((t0 >> 7) == (t1 >> 7)) {
        ptx::signal_add(g.sync + (t0 >> 7), nt * CC);
      } else {
        ptx::signal_add(g.sync + (t0 >> 7), CC);
        ptx::signal_add(g.sync + (t1 >> 7), CC);
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Warp-specialised form (round 2, NW_ITMA_WS): the two passes of a task run on different warps
// and overlap across tasks, so no warp waits at a CTA-wide barrier.  Per CTA (one per SM):
//   warp P1W+P2W        TMA producer: window boxes into an NS-deep ring (mbarrier complete_tx)
//   warps 0..P1W-1      pass 1: window s -> Hs[b] (B^T_hat along h), then release both
//   warps P1W..+P2W-1   pass 2: Hs[b] -> split -> V stores (the same code as above)
// Ring depths NS = 2 windows, NB = 2 Hs buffers, 16 source channels per task: pass 1 of task
// i+1 runs while pass 2 of task i stores.  The fp32 arithmetic is the same sequence as the
// kernels above (V bit-identical).
template <int MO, int RO, int MI, typename XT>
struct ItWsCfg {
  using B = ItCfg<MO, RO, MI, XT, 16>;
  static constexpr int P1W = 4, P2W = 12;
  static constexpr int THREADS = (P1W + P2W + 1) * 32;
  static constexpr int NS = 2, NB = 2;
  static constexpr size_t SMEM = (size_t)NS * B::STAGE + (size_t)NB * B::HS * 4 + 8 * (2 * NS + 2 * NB) + 128;
};

template <int MO, int RO, int MI, typename XT, int CINP>
__global__ void __launch_bounds__(ItWsCfg<MO, RO, MI, XT>::THREADS, 1)
    input_transform_ws_kernel(const __grid_constant__ CUtensorMap mapX, void* __restrict__ Vout, Geometry g,
                              int cgroups, int wgroups, int ntasks) {
  using X = Ax<MO, RO, MI>;
  using W = ItWsCfg<MO, RO, MI, XT>;
  using C = typename W::B;
  constexpr int PA = X::PA, L = X::L, CC = C::CC, NS = W::NS, NB = W::NB;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* stage = smem;                                            // NS windows
  float* Hsb = reinterpret_cast<float*>(smem + NS * C::STAGE);            // NB x HS floats
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * C::STAGE + NB * C::HS * 4);
  uint64_t* w_full = bars;
  uint64_t* w_empty = bars + NS;
  uint64_t* h_full = bars + 2 * NS;
  uint64_t* h_empty = bars + 2 * NS + NB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int grid = gridDim.x;
  constexpr int P1T = W::P1W * 32, P2T = W::P2W * 32;

  auto decode = [&](int task, int& n, int& ah, int& wg, int& cg) {
    int b = task;
    cg = b % cgroups;
    b /= cgroups;
    wg = b % wgroups;
    b /= wgroups;
    ah = b % g.tiles_h;
    n = b / g.tiles_h;
  };
  if (tid == 0) {
    ptx::tma_prefetch(&mapX);
    for (int i = 0; i < NS; ++i) {
      ptx::mbar_init(ptx::smem_u32(&w_full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&w_empty[i]), P1T);
    }
    for (int i = 0; i < NB; ++i) {
      ptx::mbar_init(ptx::smem_u32(&h_full[i]), P1T);
      ptx::mbar_init(ptx::smem_u32(&h_empty[i]), P2T);
    }
    ptx::mbar_init_fence();
  }
  __syncthreads();
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();  // x may come from the previous kernel in the stream

  if (warp == W::P1W + W::P2W) {  // ------------------------- TMA producer -------------------------
    if (lane == 0) {
      int it = 0;
      for (int task = blockIdx.x; task < ntasks; task += grid, ++it) {
        const int s = it % NS;
        ptx::mbar_wait(ptx::smem_u32(&w_empty[s]), (uint32_t)(((it / NS) & 1) ^ 1));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // pass-1 reads before the refill
        int n, ah, wg, cg;
        decode(task, n, ah, wg, cg);
        const int row0 = ah * X::ADV + g.off[0];
        const int col0 = (wg * C::TW * X::ADV + g.off[0]) & ~(C::AL - 1);  // 16-byte aligned start
        const uint32_t bar = ptx::smem_u32(&w_full[s]);
        ptx::mbar_expect_tx(bar, (uint32_t)(CC * L * C::BW * C::ES));
        ptx::tma_load_3d(ptx::smem_u32(stage + (size_t)s * C::STAGE), &mapX, bar, col0, row0, n * g.Cin + cg * CC);
      }
    }
    return;
  }
  if (warp < W::P1W) {  // ------------------------- pass 1: columns along h -------------------------
    int it = 0;
    for (int task = blockIdx.x; task < ntasks; task += grid, ++it) {
      const int s = it % NS, b = it % NB;
      int n, ah, wg, cg;
      decode(task, n, ah, wg, cg);
      const int sh = (wg * C::TW * X::ADV + g.off[0]) & (C::AL - 1);  // window start inside the aligned box
      const XT* win = reinterpret_cast<const XT*>(stage + (size_t)s * C::STAGE) + sh;
      float* Hs = Hsb + (size_t)b * C::HS;
      ptx::mbar_wait(ptx::smem_u32(&w_full[s]), (uint32_t)((it / NS) & 1));
      ptx::mbar_wait(ptx::smem_u32(&h_empty[b]), (uint32_t)(((it / NB) & 1) ^ 1));
      if constexpr (kPackedAxis<MO, RO, MI>) {
        // two window columns per thread in one packed register pair (FADD2 / FFMA2)
#pragma unroll 1
        for (int t1 = tid; t1 < CC * C::WC; t1 += 2 * P1T) {
          const int tb = t1 + P1T;
          const int col = t1 % C::WC, c = t1 / C::WC;
          const XT* src = win + (c * L) * C::BW + col;
          float* dst = Hs + c * C::HSTR + col;
          if (tb < CC * C::WC) {
            const int colb = tb % C::WC, cb = tb / C::WC;
            const XT* srcb = win + (cb * L) * C::BW + colb;
            float* dstb = Hs + cb * C::HSTR + colb;
            f2 xin[L], hv[PA];
#pragma unroll
            for (int r = 0; r < L; ++r) xin[r] = f2_pack(to_f(src[r * C::BW]), to_f(srcb[r * C::BW]));
            in_axis_t<MO, RO, MI, f2>(xin, hv);
#pragma unroll
            for (int q = 0; q < PA; ++q) f2_unpack(hv[q], dst[q * CC * C::HSTR], dstb[q * CC * C::HSTR]);
          } else {
            float xin[L], hv[PA];
#pragma unroll
            for (int r = 0; r < L; ++r) xin[r] = to_f(src[r * C::BW]);
            in_axis<MO, RO, MI>(xin, hv);
#pragma unroll
            for (int q = 0; q < PA; ++q) dst[q * CC * C::HSTR] = hv[q];
          }
        }
      } else {
#pragma unroll 1
        for (int t1 = tid; t1 < CC * C::WC; t1 += P1T) {
          const int col = t1 % C::WC, c = t1 / C::WC;
          const XT* src = win + (c * L) * C::BW + col;
          float xin[L], hv[PA];
#pragma unroll
          for (int r = 0; r < L; ++r) xin[r] = to_f(src[r * C::BW]);
          in_axis<MO, RO, MI>(xin, hv);
          float* dst = Hs + c * C::HSTR + col;
#pragma unroll
          for (int q = 0; q < PA; ++q) dst[q * CC * C::HSTR] = hv[q];
        }
      }
      ptx::mbar_arrive(ptx::smem_u32(&w_empty[s]));
      ptx::mbar_arrive(ptx::smem_u32(&h_full[b]));
    }
    return;
  }
  // ----------------------------- pass 2: rows along w, split, store V -----------------------------
  const int t2 = tid - P1T, w2 = warp - W::P1W;
  const int pair = lane % C::NPR, sub = lane / C::NPR;
  int it = 0;
  for (int task = blockIdx.x; task < ntasks; task += grid, ++it) {
    const int b = it % NB;
    int n, ah, wg, cg;
    decode(task, n, ah, wg, cg);
    const int aw0 = wg * C::TW;
    const float* Hs = Hsb + (size_t)b * C::HS;
    ptx::mbar_wait(ptx::smem_u32(&h_full[b]), (uint32_t)((it / NB) & 1));
#pragma unroll 1
    for (int grp = w2; grp < C::GROUPS; grp += W::P2W) {
      const int q = grp * C::SUBS + sub;            // (p_h, tile) combo of this lane
      const int ph = q / C::TW, tile = q % C::TW;
      const bool live = q < C::COMBOS && aw0 + tile < g.tiles_w;
      if (live) {
        const float* h0 = Hs + (ph * CC + 2 * pair) * C::HSTR + tile * X::ADV;
        const float* h1 = h0 + C::HSTR;
        const long long t = ((long long)n * g.tiles_h + ah) * g.tiles_w + aw0 + tile;
        const long long row = (((t >> 7) * g.P + (long long)ph * PA) * 2) * 128 + (t & 127);
        char* hp = reinterpret_cast<char*>(Vout) + (row * CINP + cg * CC + 2 * pair) * 2;
        if constexpr (kPackedAxis<MO, RO, MI>) {  // the pair's two channels in one packed lane pair
          f2 zab[X::LO][X::LI];
          {
            f2 ab[L];
#pragma unroll
            for (int k = 0; k < L; ++k) ab[k] = f2_pack(h0[k], h1[k]);
            in_axis_inner_t<MO, RO, MI, f2>(ab, zab);
          }
          store_row_imm_p<MO, RO, MI, CINP>(zab, hp);
        } else {
          float za[X::LO][X::LI], zb[X::LO][X::LI];
          {
            float a[L], bb[L];
#pragma unroll
            for (int k = 0; k < L; ++k) {
              a[k] = h0[k];
              bb[k] = h1[k];
            }
            in_axis_inner<MO, RO, MI>(a, za);
            in_axis_inner<MO, RO, MI>(bb, zb);
          }
          store_row_imm<MO, RO, MI, CINP>(za, zb, hp);
        }
      }
    }
    ptx::mbar_arrive(ptx::smem_u32(&h_empty[b]));
    if (g.sync) {  // streamed pipeline: every pass-2 thread's V stores of this task, then count them
      asm volatile("bar.sync 1, %0;" ::"n"(P2T) : "memory");
      if (t2 == 0) {
        const long long t0 = ((long long)n * g.tiles_h + ah) * g.tiles_w + aw0;
        const int nt = min(C::TW, g.tiles_w - aw0);
        const long long t1 = t0 + nt - 1;
        if ((t0 >> 7) == (t1 >> 7)) {
          ptx::signal_add(g.sync + (t0 >> 7), nt * CC);
        } else {
          ptx::signal_add(g.sync + (t0 >> 7), CC);
          ptx::signal_add(g.sync + (t1 >> 7), CC);
        }
      }
    }
  }
}

// NW_ITMA_WS=0|1: the warp-specialised kernel (default on; measured in profiles/r2u_*)
inline bool input_ws_enabled() {
  static const int on = [] {
    const char* v = getenv("NW_ITMA_WS");
    return v ? atoi(v) : 1;
  }();
  return on != 0;
}

bool encode_tmap(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base, const uint64_t* dims,
                 const uint64_t* strides_bytes, const uint32_t* box, CUtensorMapSwizzle swz);

// NW_INPUT_TMA=0 selects the first-round kernel (input_transform_kernel) everywhere.
inline bool input_tma_enabled() {
  static const int on = [] {
    const char* v = getenv("NW_INPUT_TMA");
    return v ? atoi(v) : 1;
  }();
  return on != 0;
}

// NW_ITMA_CC=16|32: source channels per task (default 32: C3 0.432 ms against 0.485 with 16,
// 0.565 with the first-round kernel; profiles/r2_input_transform.md)
inline int input_tma_cc() {
  static const int cc = [] {
    const char* v = getenv("NW_ITMA_CC");
    return v ? atoi(v) : 32;
  }();
  return cc;
}

template <int MO, int RO, int MI, typename XT, int CINP, int CC_>
static nw_status_t input_tma_launch_cc(const Geometry& g, const void* x, void* V, cudaStream_t s) {
  using C = ItCfg<MO, RO, MI, XT, CC_>;
  auto kern = input_transform_tma_kernel<MO, RO, MI, XT, CINP, CC_>;
  if (ensure_smem<input_transform_tma_kernel<MO, RO, MI, XT, CINP, CC_>>((int)C::SMEM) != NW_OK) return NW_ERR_CUDA;
  const uint64_t dims[3] = {(uint64_t)g.W, (uint64_t)g.H, (uint64_t)g.N * g.Cin};
  const uint64_t strides[2] = {(uint64_t)g.W * C::ES, (uint64_t)g.H * g.W * C::ES};
  const uint32_t box[3] = {(uint32_t)C::BW, (uint32_t)C::L, (uint32_t)C::CC};
  alignas(64) CUtensorMap mapX;
  if (!encode_tmap(&mapX, sizeof(XT) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, x,
                   dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE))
    return NW_ERR_CUDA;
  const int wgroups = (g.tiles_w + C::TW - 1) / C::TW;
  const int cgroups = g.Cin / C::CC;
  const long long ntasks = (long long)g.N * g.tiles_h * wgroups * cgroups;
  if (ntasks >= (1ll << 31)) return NW_ERR_UNSUPPORTED;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long slots = (long long)sms * C::MINB;  // persistent: every resident CTA slot
  if (g.it_ctas > 0 && g.it_ctas < slots) slots = g.it_ctas;  // streamed pipeline: its share of the SMs
  const int grid = (int)(ntasks < slots ? ntasks : slots);
  LaunchScope scope_("input_transform", s);
  if (launch_pdl(kern, dim3(grid), dim3(C::THREADS), C::SMEM, s, mapX, V, g, cgroups, wgroups, (int)ntasks) != NW_OK)
    return NW_ERR_CUDA;
  return check_launch();
}

template <int MO, int RO, int MI, typename XT, int CINP>
static nw_status_t input_ws_launch(const Geometry& g, const void* x, void* V, cudaStream_t s) {
  using W = ItWsCfg<MO, RO, MI, XT>;
  using C = typename W::B;
  auto kern = input_transform_ws_kernel<MO, RO, MI, XT, CINP>;
  if (ensure_smem<input_transform_ws_kernel<MO, RO, MI, XT, CINP>>((int)W::SMEM) != NW_OK) return NW_ERR_CUDA;
  const uint64_t dims[3] = {(uint64_t)g.W, (uint64_t)g.H, (uint64_t)g.N * g.Cin};
  const uint64_t strides[2] = {(uint64_t)g.W * C::ES, (uint64_t)g.H * g.W * C::ES};
  const uint32_t box[3] = {(uint32_t)C::BW, (uint32_t)C::L, (uint32_t)C::CC};
  alignas(64) CUtensorMap mapX;
  if (!encode_tmap(&mapX, sizeof(XT) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, x,
                   dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE))
    return NW_ERR_CUDA;
  const int wgroups = (g.tiles_w + C::TW - 1) / C::TW;
  const int cgroups = g.Cin / C::CC;
  const long long ntasks = (long long)g.N * g.tiles_h * wgroups * cgroups;
  if (ntasks >= (1ll << 31)) return NW_ERR_UNSUPPORTED;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long slots = sms;
  if (g.it_ctas > 0 && g.it_ctas < slots) slots = g.it_ctas;
  const int grid = (int)(ntasks < slots ? ntasks : slots);
  LaunchScope scope_("input_transform", s);
  if (launch_pdl(kern, dim3(grid), dim3(W::THREADS), W::SMEM, s, mapX, V, g, cgroups, wgroups, (int)ntasks) != NW_OK)
    return NW_ERR_CUDA;
  return check_launch();
}

// The warp-specialised kernel measured faster for the r_o = 3 outer kernels (c2k9 / c2k7 input
// transform 0.222 -> 0.207 ms, C3 0.478 -> 0.437 ms) and slower for the mixed F(4,2) outer kernel
// (c2k5 0.164 -> 0.168 ms, where the first-round kernel stays; profiles/r2u_workloads.md)
template <int RO>
constexpr bool ws_preferred() { return RO == 3; }

template <int MO, int RO, int MI, typename XT, int CINP>
static nw_status_t input_tma_launch(const Geometry& g, const void* x, void* V, cudaStream_t s) {
  if (input_ws_enabled() && ws_preferred<RO>() && ItWsCfg<MO, RO, MI, XT>::SMEM <= 227 * 1024)
    return input_ws_launch<MO, RO, MI, XT, CINP>(g, x, V, s);
  if (input_tma_cc() == 32 && g.Cin % 32 == 0 && ItCfg<MO, RO, MI, XT, 32>::SMEM <= 227 * 1024)
    return input_tma_launch_cc<MO, RO, MI, XT, CINP, 32>(g, x, V, s);
  return input_tma_launch_cc<MO, RO, MI, XT, CINP, 16>(g, x, V, s);
}

// The TMA kernel covers stride-1 inputs (incl. the transposed plan's input side) without
// coverage phases, bf16x3 blocked V, every source channel real (Cin = cin_pad, a multiple of
// 16) and 16-byte x row pitches (TMA).
template <int MO, int RO, int MI, typename XT>
inline bool input_tma_eligible(const Geometry& g) {
  using C = ItCfg<MO, RO, MI, XT, 16>;
  // bf16 x only: with fp32 x (C2) the first-round kernel measured as fast or faster (0.197 ms per
  // C2 layer against 0.203 with 32 channels per task, 0.243 with 16); with bf16 x (C3) this kernel
  // is faster, 0.432 against 0.565 ms (profiles/r2_input_transform.md)
  static const bool fp32_too = [] {  // NW_ITMA_F32=1: also fp32 x (measurement switch)
    const char* v = getenv("NW_ITMA_F32");
    return v && atoi(v) == 1;
  }();
  return input_tma_enabled() && (sizeof(XT) == 2 || fp32_too || g.sync || (input_ws_enabled() && ws_preferred<RO>())) && g.SR == 1 && g.nph == 1 && g.vblk && g.Cin == g.cin_pad && g.Cin % C::CC == 0 &&
         ((long long)g.W * C::ES) % 16 == 0 && 2 * C::SMEM <= 227 * 1024 && g.H < (1 << 30);
}

}  // namespace nw
