// input_transform_tma.cuh -- G2 on sm_100a: nested input transform V = B^T_hat X B_hat
// as a persistent, TMA-fed kernel with 16-byte V stores.
//
// One CTA per SM walks tasks (image n, tile row a_h, TW = 2 adjacent tiles along w, CC = 16
// source channels), channel group fastest so the four CTAs filling one 128-byte V row run
// side by side.  Per task:
//   TMA     one 3-D box {window columns (+ up to 15 bytes to start 16-byte aligned), L rows,
//           16 channels} of x [N*Cin][H][W] lands in a
//           double-buffered shared stage; coordinates outside the image are zero-filled by
//           the copy engine (= the convolution's zero padding), so there are no bounds tests.
//           The box of task i+2 is issued as soon as pass 1 of task i has consumed the stage.
//   pass 1  thread = (channel, window column): B^T_hat along h (both levels, factored 1-D
//           kernels of transforms.cuh) -> Hs[p_h][channel][column], fp32.
//   pass 2  lane = (channel pair, (p_h, tile) combo): the L-long row of Hs along w -> P_a
//           values per channel, split into bf16 hi / lo (one cvt.rn.bf16x2 per plane) and
//           staged per warp as [combo][p_w][plane][pair] words; the warp then copies its stage
//           out with 16-byte stores: every (slice, point, plane) row segment of the 16
//           channels is two aligned 16-byte pieces of the blocked V layout
//           [T_pad/128][P][hi, lo][128][CINP] (the contraction's TMA A operand).
// Arithmetic is the same sequence of fp32 operations as input_transform_kernel, so V is
// bit-identical to it (tests/test_gpu_env_variants.py checks with NW_INPUT_TMA=0).
#pragma once
#include <cstdlib>

#include "ptx.cuh"
#include "transforms.cuh"

namespace nw {

template <int MO, int RO, int MI, typename XT, bool STAGED>
struct ItCfg {
  using X = Ax<MO, RO, MI>;
  static constexpr int CC = 16;                         // source channels per task
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
  static constexpr int GROUPS = (COMBOS + 3) / 4;       // 4 combos x 8 channel pairs per warp pass
  // per-warp output stage: 4 combos x P_a points x 2 planes x 8 pairs (u32), the combo pitch
  // padded to 8 (mod 32) words so the 4 combos of a store land in distinct banks
  static constexpr int SSTR = PA * 16 + ((8 - PA * 16 % 32) + 32) % 32;
  static constexpr int WARPS = 8;
  static constexpr int THREADS = WARPS * 32;
  // STAGED: one CTA per SM, double-buffered window, per-warp output stage + 16-byte stores.
  // Direct: two CTAs per SM, one window buffer (refilled as soon as pass 1 has read it, so the
  // load overlaps pass 2 and the other CTA), 4-byte stores of bf16 channel pairs.
  static constexpr int NSTAGE = STAGED ? 2 : 1;
  static constexpr int MINB = STAGED ? 1 : 2;
  static constexpr size_t WS_BYTES = STAGED ? (size_t)WARPS * 4 * SSTR * 4 : 0;
  static constexpr size_t SMEM = (size_t)NSTAGE * STAGE + (size_t)HS * 4 + WS_BYTES + 64;
  static_assert(SSTR % 32 == 8, "stage pitch");
  static_assert(BW <= 256 && L <= 256, "TMA box");
};

template <int MO, int RO, int MI, typename XT, int CINP, bool STAGED>
__global__ void __launch_bounds__(ItCfg<MO, RO, MI, XT, STAGED>::THREADS, ItCfg<MO, RO, MI, XT, STAGED>::MINB)
    input_transform_tma_kernel(const __grid_constant__ CUtensorMap mapX, void* __restrict__ Vout, Geometry g,
                               int cgroups, int wgroups, int ntasks) {
  using X = Ax<MO, RO, MI>;
  using C = ItCfg<MO, RO, MI, XT, STAGED>;
  constexpr int PA = X::PA, L = X::L, CC = C::CC, NS = C::NSTAGE;
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* stage = smem;                                                  // NS x STAGE
  float* Hs = reinterpret_cast<float*>(smem + NS * C::STAGE);                   // HS floats
  uint32_t* Ws = reinterpret_cast<uint32_t*>(smem + NS * C::STAGE + C::HS * 4);  // per-warp out stages
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * C::STAGE + C::HS * 4 + C::WS_BYTES);
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
    ptx::mbar_init(ptx::smem_u32(&full[1]), 1);
    ptx::mbar_init_fence();
  }
  __syncthreads();
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();  // x may come from the previous kernel in the stream
  if (tid == 0) {
    for (int i = 0; i < NS; ++i)
      if (blockIdx.x + i * grid < ntasks) issue(blockIdx.x + i * grid, i);
  }

  uint32_t* ws = Ws + warp * 4 * C::SSTR;
  int it = 0;
#pragma unroll 1
  for (int task = blockIdx.x; task < ntasks; task += grid, ++it) {
    const int s = it % NS;
    int b = task;
    const int cg = b % cgroups;
    b /= cgroups;
    const int wg = b % wgroups;
    b /= wgroups;
    const int ah = b % g.tiles_h;
    const int n = b / g.tiles_h;
    const int aw0 = wg * C::TW;
    const int sh = (aw0 * X::ADV + g.off[0]) & (C::AL - 1);  // window start inside the aligned box
    const XT* win = reinterpret_cast<const XT*>(stage + (size_t)s * C::STAGE) + sh;
    ptx::mbar_wait(ptx::smem_u32(&full[s]), (uint32_t)((it / NS) & 1));

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
    __syncthreads();  // stage s consumed, Hs complete
    if (tid == 0 && task + NS * grid < ntasks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before the async refill
      issue(task + NS * grid, s);
    }

    // ---------------- pass 2: rows along w, split, stage, 16-byte stores ----------------
    const int pair = lane & 7, sub = lane >> 3;
#pragma unroll 1
    for (int grp = warp; grp < C::GROUPS; grp += C::WARPS) {
      const int q = grp * 4 + sub;                  // (p_h, tile) combo of this lane
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
        if constexpr (STAGED) {
          uint32_t* wp = ws + sub * C::SSTR + pair;
#pragma unroll
          for (int pi = 0; pi < X::LI; ++pi) {
            float oa[X::LO], ob[X::LO];
            in_axis_outer_col<MO, RO, MI>(za, pi, oa);
            in_axis_outer_col<MO, RO, MI>(zb, pi, ob);
#pragma unroll
            for (int po = 0; po < X::LO; ++po) {
              uint32_t hi, lo;
              ptx::split_bf16x2(oa[po], ob[po], hi, lo);
              const int pw = po * X::LI + pi;
              wp[(pw * 2 + 0) * 8] = hi;
              wp[(pw * 2 + 1) * 8] = lo;
            }
          }
        } else {
          // straight to V: one base pointer per lane, every store an immediate offset from it
          const long long t = ((long long)n * g.tiles_h + ah) * g.tiles_w + aw0 + tile;
          const long long row = (((t >> 7) * g.P + (long long)ph * PA) * 2) * 128 + (t & 127);
          char* hp = reinterpret_cast<char*>(Vout) + (row * CINP + cg * CC + 2 * pair) * 2;
          store_row_imm<MO, RO, MI, CINP>(za, zb, hp);
        }
      }
      if constexpr (STAGED) {
        __syncwarp();
        // copy out: lane = (half, plane, p_w parity, combo sub); the loop walks p_w by 2, so the
        // stage and V addresses advance by constants
        const int half = lane & 1, plane = (lane >> 1) & 1, pwl = (lane >> 2) & 1, sb = lane >> 3;
        const int qq = grp * 4 + sb;
        const int phq = qq / C::TW, tq = qq % C::TW;
        if (qq < C::COMBOS && aw0 + tq < g.tiles_w) {
          const long long t = ((long long)n * g.tiles_h + ah) * g.tiles_w + aw0 + tq;
          const long long row = (((t >> 7) * g.P + (long long)phq * PA + pwl) * 2 + plane) * 128 + (t & 127);
          char* dst = reinterpret_cast<char*>(Vout) + (row * CINP + cg * CC + half * 8) * 2;
          const uint32_t* src = ws + sb * C::SSTR + (pwl * 2 + plane) * 8 + half * 4;
#pragma unroll 5
          for (int j = 0; j < (PA + 1) / 2; ++j) {
            if (2 * j + pwl < PA)
              *reinterpret_cast<uint4*>(dst + (long long)j * (4 * 128 * CINP * 2)) =
                  *reinterpret_cast<const uint4*>(src + j * 32);
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();  // Hs free for the next task's pass 1
  }
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

// NW_ITMA_STAGED=1 selects the staged variant (one CTA per SM, 16-byte stores), default the
// direct variant (two CTAs per SM, 4-byte stores).
inline bool input_tma_staged() {
  static const int on = [] {
    const char* v = getenv("NW_ITMA_STAGED");
    return v ? atoi(v) : 0;
  }();
  return on != 0;
}

template <int MO, int RO, int MI, typename XT, int CINP, bool STAGED>
static nw_status_t input_tma_launch_v(const Geometry& g, const void* x, void* V, cudaStream_t s) {
  using C = ItCfg<MO, RO, MI, XT, STAGED>;
  auto kern = input_transform_tma_kernel<MO, RO, MI, XT, CINP, STAGED>;
  if (ensure_smem<input_transform_tma_kernel<MO, RO, MI, XT, CINP, STAGED>>((int)C::SMEM) != NW_OK)
    return NW_ERR_CUDA;
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
  const long long slots = (long long)sms * C::MINB;  // persistent: every resident CTA slot
  const int grid = (int)(ntasks < slots ? ntasks : slots);
  LaunchScope scope_("input_transform", s);
  if (launch_pdl(kern, dim3(grid), dim3(C::THREADS), C::SMEM, s, mapX, V, g, cgroups, wgroups, (int)ntasks) != NW_OK)
    return NW_ERR_CUDA;
  return check_launch();
}

template <int MO, int RO, int MI, typename XT, int CINP>
static nw_status_t input_tma_launch(const Geometry& g, const void* x, void* V, cudaStream_t s) {
  if (input_tma_staged() && ItCfg<MO, RO, MI, XT, true>::SMEM <= 227 * 1024)
    return input_tma_launch_v<MO, RO, MI, XT, CINP, true>(g, x, V, s);
  return input_tma_launch_v<MO, RO, MI, XT, CINP, false>(g, x, V, s);
}

// The TMA kernel covers stride-1 inputs (incl. the transposed plan's input side) without
// coverage phases, bf16x3 blocked V, every source channel real (Cin = cin_pad, a multiple of
// 16) and 16-byte x row pitches (TMA).
template <int MO, int RO, int MI, typename XT>
inline bool input_tma_eligible(const Geometry& g) {
  using C = ItCfg<MO, RO, MI, XT, false>;
  return input_tma_enabled() && g.SR == 1 && g.nph == 1 && g.vblk && g.Cin == g.cin_pad && g.Cin % C::CC == 0 &&
         ((long long)g.W * C::ES) % 16 == 0 && 2 * C::SMEM <= 227 * 1024 && g.H < (1 << 30);
}

}  // namespace nw
