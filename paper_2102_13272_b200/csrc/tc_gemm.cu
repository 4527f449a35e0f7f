// tc_gemm.cu -- G3: the per-transform-point channel contraction on 5th-gen tensor
// cores (tcgen05, sm_100a).  For every point xi of the P = P_a^2 transform points
//     M_xi[T x Cout_e] = V_xi[T x Cin_e] . U_xi[Cout_e x Cin_e]^T
// (the EWMM of P:110 summed over input channels, Eq. 2.1), the only dense
// contraction of the method.
//
// Precision (R12): BF16X3 splits both operands into bf16 hi/lo planes
// (written by the input / filter transforms) and issues three kind::f16 MMAs per
// K step into one fp32 TMEM accumulator: Vh.Uh + Vh.Ul + Vl.Uh.  BF16 issues Vh.Uh.
//
// Structure (persistent, warp-specialised, 1 CTA per SM):
//   warp 0 lane 0  TMA producer: B ring (U_xi k-block, hi+lo) and A ring (128-slice
//                  blocks of V_xi, hi+lo), 128B-swizzled, mbarrier complete_tx
//   warp 1 lane 0  MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M=128, N=Cout_pad,
//                  K=16 per instruction, accumulators double-buffered in TMEM,
//                  tcgen05.commit frees smem stages / signals the epilogue
//   warps 2..5     epilogue: tcgen05.ld 32x32b -> registers -> coalesced stores of
//                  M[xi][co][t] (each warp owns a 32-lane TMEM quarter = 32 slices)
// A work unit is (xi, group of G 128-slice blocks); one B k-block is loaded per
// unit and k-block and reused by the G A blocks (G*N <= 256 TMEM columns).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "nw_internal.h"
#include "ptx.cuh"

namespace nw {
namespace tc {

constexpr int kBM = 128;      // slices per MMA (TMEM lanes)
constexpr int kBK = 64;       // bf16 elements per 128-byte swizzle row
constexpr int kThreads = 192;
constexpr int kMaxStages = 8;

// ------------------------------- PTX wrappers --------------------------------
using namespace ::nw::ptx;
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
// one lane of a converged warp (elect.sync): ptxas knows exactly one thread is active inside the
// branch, so single-thread instructions (tcgen05.mma / commit) need no per-instruction election loop
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t"
      "}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---- cluster helpers (CTA pairs sharing the B operand) ----
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load whose box lands at the same shared offset in every CTA of ctamask, each CTA's
// mbarrier at `bar` receiving the bytes
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                               uint16_t ctamask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
      "[%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "h"(ctamask)
      : "memory");
}
// tcgen05.commit arriving on the mbarrier at `bar` in every CTA of ctamask
__device__ __forceinline__ void umma_commit_mc(uint32_t bar, uint16_t ctamask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   bar),
               "h"(ctamask)
               : "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address >> 4
  d |= (uint64_t)(0) << 16;                         // leading byte offset (unused for K-major SW128)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;      // stride byte offset: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                           // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                           // layout: SWIZZLE_128B
  return d;
}
// K-major descriptor for a K block of kbk bf16 (rows of 2*kbk bytes, swizzle span = row):
// kbk 64 -> SWIZZLE_128B, 32 -> SWIZZLE_64B, 16 -> SWIZZLE_32B; 8-row groups 16*kbk bytes apart.
// Narrow K blocks serve layers with 16 / 32 contraction channels without zero-padding to 64.
__device__ __forceinline__ uint64_t swk_desc(uint32_t saddr, int kbk) {
  const uint32_t layout = kbk == 64 ? 2u : (kbk == 32 ? 4u : 6u);
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(((16u * (uint32_t)kbk) >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
// Instruction descriptor: D fp32, A/B bf16, both K-major, M=128, N=n.
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

// Lean MMA issue for the fused kernels: the issuing lane was the bottleneck (ncu: ~26 dependent
// instructions per MMA rebuilding both descriptors, ~150 cycles per MMA).  A descriptor's upper
// word is constant per launch and its lower word is the shared address >> 4, so a k-step is one
// add per operand.
__device__ __forceinline__ uint32_t swk_desc_hi(int kbk) {
  const uint32_t layout = kbk == 64 ? 2u : (kbk == 32 ? 4u : 6u);
  return (((16u * (uint32_t)kbk) >> 4) & 0x3FFFu) | (1u << 14) | (layout << 29);
}
__device__ __forceinline__ uint64_t mk_desc(uint32_t hi, uint32_t lo) { return ((uint64_t)hi << 32) | (uint64_t)lo; }
// one k-block (KS k-steps of 16) of one point: alo / blo = (stage A / B address) >> 4, apl / bpl =
// (plane bytes) >> 4; accumulate = 0 starts the accumulator
template <int KS>
__device__ __forceinline__ void issue_kblock(uint32_t acc, uint32_t alo, uint32_t blo, uint32_t apl, uint32_t bpl,
                                             uint32_t dhi, uint32_t idesc, int lo, uint32_t accumulate) {
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    const uint64_t ah = mk_desc(dhi, alo + 2 * k), bh = mk_desc(dhi, blo + 2 * k);
    umma_f16(acc, ah, bh, idesc, k == 0 ? accumulate : 1u);
    if (lo) {
      umma_f16(acc, ah, mk_desc(dhi, blo + bpl + 2 * k), idesc, 1u);
      umma_f16(acc, mk_desc(dhi, alo + apl + 2 * k), bh, idesc, 1u);
    }
  }
}
__device__ __forceinline__ void issue_kblock_any(int kbk, uint32_t acc, uint32_t alo, uint32_t blo, uint32_t apl,
                                                 uint32_t bpl, uint32_t dhi, uint32_t idesc, int lo,
                                                 uint32_t accumulate) {
  if (kbk == 64) issue_kblock<4>(acc, alo, blo, apl, bpl, dhi, idesc, lo, accumulate);
  else if (kbk == 32) issue_kblock<2>(acc, alo, blo, apl, bpl, dhi, idesc, lo, accumulate);
  else issue_kblock<1>(acc, alo, blo, apl, bpl, dhi, idesc, lo, accumulate);
}

struct Params {
  int P;            // transform points
  int nmb;          // 128-slice blocks per point (T_pad / 128)
  int G;            // blocks per unit
  int ngrp;         // unit groups per point = ceil(nmb / G)
  int N;            // cout_pad (MMA N, <= 256)
  int Nst;          // channels stored (cout_e): rows of padded channels are never read, not written
  int KB;           // k-blocks of 64 (ceil(cin_pad / 64))
  int lo;           // 1 = bf16x3 (lo planes), 0 = plain bf16
  int nA, nB;       // ring depths
  long long T_pad;
  long long a_lo_row; // row offset of the lo plane in the V tensor map (= P * T_pad)
  long long b_lo_row; // row offset of the lo plane in the U tensor map (= P * N)
  int vblk;           // blocked split layout: rows ((mb * P + xi) * 2 + plane) * 128
  float* M;
  // shifted operands (OLA / direct comparison paths): k-block kb belongs to
  // shift s = kb / kbc and channel block kc = kb % kbc; its A rows are read at
  // t + shoff[s] and its B columns at s * cin_pad + kc * 64.  Nested: nsh = 1.
  int nsh, kbc, cin_pad;
  int kbk;           // K block width in bf16 elements (64, 32 or 16)
  int shoff[kMaxShift];
};

// CL > 1: clusters of CL CTAs work on CL consecutive 128-slice blocks of the same point;
// each CTA loads 1/CL of every B k-block and multicasts it to the whole cluster, and every
// CTA's MMA completion releases the B stage in all of them (B read from L2 once per cluster).
template <int CL>
__global__ void __launch_bounds__(kThreads, 1)
    contraction_kernel(const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapU,
                       const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment for the swizzled tiles
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sbase = smem_raw + (base - raw);

  const uint32_t a_plane = kBM * p.kbk * 2;            // 16 KB at kbk 64
  const uint32_t a_stage = a_plane * (p.lo ? 2 : 1);
  const uint32_t b_plane = (uint32_t)p.N * p.kbk * 2;  // N rows of 2 kbk bytes
  const uint32_t b_stage = b_plane * (p.lo ? 2 : 1);
  const uint32_t a_off = 0;
  const uint32_t b_off = a_off + a_stage * p.nA;
  const uint32_t bar_off = b_off + b_stage * p.nB;
  // barriers: A_full[nA], A_empty[nA], B_full[nB], B_empty[nB], T_full[2], T_empty[2], tmem addr
  uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + bar_off);
  uint64_t* A_full = bars;
  uint64_t* A_empty = bars + kMaxStages;
  uint64_t* B_full = bars + 2 * kMaxStages;
  uint64_t* B_empty = bars + 3 * kMaxStages;
  uint64_t* T_full = bars + 4 * kMaxStages;
  uint64_t* T_empty = bars + 4 * kMaxStages + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 4 * kMaxStages + 4);

  // warp index through a shuffle: provably warp-uniform (role branches and issue loops in uniform registers)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int total_units = p.P * p.ngrp;
  const int rank = (CL > 1) ? (int)cluster_rank() : 0;
  const int ustart = (CL > 1) ? (int)blockIdx.x / CL : (int)blockIdx.x;
  const int ustep = (CL > 1) ? (int)gridDim.x / CL : (int)gridDim.x;
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapV);
    tma_prefetch(&mapU);
    for (int i = 0; i < p.nA; ++i) { mbar_init(smem_u32(&A_full[i]), 1); mbar_init(smem_u32(&A_empty[i]), 1); }
    for (int i = 0; i < p.nB; ++i) { mbar_init(smem_u32(&B_full[i]), 1); mbar_init(smem_u32(&B_empty[i]), CL); }
    for (int i = 0; i < 2; ++i) { mbar_init(smem_u32(&T_full[i]), 1); mbar_init(smem_u32(&T_empty[i]), 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // whole warp allocates TMEM (512 columns: 2 accumulator buffers)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync();  // every CTA's barriers are initialised before multicasts target them
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();
  griddep_wait();  // V comes from the input transform just before in the stream

  if (warp == 0) {
    {
      // ------------------------------ TMA producer (warp-uniform loop, elected lane issues) ------------------------------
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      for (int u = ustart; u < total_units; u += ustep) {
        const int xi = u / p.ngrp, grp = u % p.ngrp;
        const int mb0 = (CL > 1) ? grp * CL + rank : grp * p.G;
        const int g_eff = (CL > 1) ? 1 : min(p.G, p.nmb - mb0);
        for (int kb = 0; kb < p.KB; ++kb) {
          mbar_wait(smem_u32(&B_empty[sb]), pb ^ 1);
          const uint32_t bfull = smem_u32(&B_full[sb]);
          const uint32_t bdst = base + b_off + sb * b_stage;
          const int sh = kb / p.kbc, kc = kb - sh * p.kbc;
          const int bcol = sh * p.cin_pad + kc * p.kbk, acol = kc * p.kbk, aoff = p.shoff[sh];
          if (elect_one()) {
          mbar_expect_tx(bfull, b_stage);
          if constexpr (CL > 1) {
            const int rows = p.N / CL;  // this CTA's slice of the B tile, multicast to the cluster
            const uint32_t so = (uint32_t)(rank * rows) * (p.kbk * 2);
            tma_load_2d_mc(bdst + so, &mapU, bfull, bcol, xi * p.N + rank * rows, kMask);
            if (p.lo)
              tma_load_2d_mc(bdst + b_plane + so, &mapU, bfull, bcol,
                             (int)(p.b_lo_row + (long long)xi * p.N) + rank * rows, kMask);
          } else {
            tma_load_2d(bdst, &mapU, bfull, bcol, xi * p.N);
            if (p.lo) tma_load_2d(bdst + b_plane, &mapU, bfull, bcol, (int)(p.b_lo_row + (long long)xi * p.N));
          }
          }
          __syncwarp();
          if (++sb == p.nB) { sb = 0; pb ^= 1; }
          for (int g = 0; g < g_eff; ++g) {
            mbar_wait(smem_u32(&A_empty[sa]), pa ^ 1);
            const uint32_t afull = smem_u32(&A_full[sa]);
            const uint32_t adst = base + a_off + sa * a_stage;
            long long row, lrow;
            if (p.vblk) {
              row = ((long long)(mb0 + g) * p.P + xi) * (2 * kBM);
              lrow = row + kBM;
            } else {
              row = (long long)xi * p.T_pad + (long long)(mb0 + g) * kBM + aoff;
              lrow = p.a_lo_row + row;
            }
            if (elect_one()) {
              mbar_expect_tx(afull, a_stage);
              tma_load_2d(adst, &mapV, afull, acol, (int)row);
              if (p.lo) tma_load_2d(adst + a_plane, &mapV, afull, acol, (int)lrow);
            }
            __syncwarp();
            if (++sa == p.nA) { sa = 0; pa ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    {
      // ------------------------------- MMA issuer (warp-uniform loop, elected lane issues) -------------------------------
      const uint32_t idesc = idesc_bf16(p.N), dhi = swk_desc_hi(p.kbk);
      int sa = 0, sb = 0;
      uint32_t pa = 0, pb = 0;
      int it = 0;
      for (int u = ustart; u < total_units; u += ustep, ++it) {
        const int grp = u % p.ngrp;
        const int g_eff = (CL > 1) ? 1 : min(p.G, p.nmb - grp * p.G);
        const int buf = it & 1;
        const uint32_t tpar = (uint32_t)((it >> 1) & 1);
        mbar_wait(smem_u32(&T_empty[buf]), tpar ^ 1);
        fence_after();
        const uint32_t acc0 = tmem_base + (uint32_t)(buf * 256);
        for (int kb = 0; kb < p.KB; ++kb) {
          mbar_wait(smem_u32(&B_full[sb]), pb);
          const uint32_t bsm = base + b_off + sb * b_stage;
          for (int g = 0; g < g_eff; ++g) {
            mbar_wait(smem_u32(&A_full[sa]), pa);
            fence_after();
            const uint32_t asm_ = base + a_off + sa * a_stage;
            const uint32_t acc = acc0 + (uint32_t)(g * p.N);
            if (elect_one()) {
              issue_kblock_any(p.kbk, acc, asm_ >> 4, bsm >> 4, a_plane >> 4, b_plane >> 4, dhi, idesc, p.lo,
                               kb > 0 ? 1u : 0u);
              umma_commit(smem_u32(&A_empty[sa]));
            }
            __syncwarp();
            if (++sa == p.nA) { sa = 0; pa ^= 1; }
          }
          if (elect_one()) {
            if constexpr (CL > 1) umma_commit_mc(smem_u32(&B_empty[sb]), kMask);  // frees the stage cluster-wide
            else umma_commit(smem_u32(&B_empty[sb]));
          }
          __syncwarp();
          if (++sb == p.nB) { sb = 0; pb ^= 1; }
        }
        if (elect_one()) umma_commit(smem_u32(&T_full[buf]));
        __syncwarp();
      }
    }
  } else {
    // -------------------------------- epilogue ---------------------------------
    const int quarter = warp & 3;                     // TMEM lanes [32q, 32q+32)
    const int row = quarter * 32 + lane;
    int it = 0;
    for (int u = ustart; u < total_units; u += ustep, ++it) {
      const int xi = u / p.ngrp, grp = u % p.ngrp;
      const int mb0 = (CL > 1) ? grp * CL + rank : grp * p.G;
      // (a cluster's last group may run past the slices: its MMAs ran on zero-filled rows, nothing is stored)
      const int g_eff = (CL > 1) ? (mb0 < p.nmb ? 1 : 0) : min(p.G, p.nmb - mb0);
      const int buf = it & 1;
      const uint32_t tpar = (uint32_t)((it >> 1) & 1);
      mbar_wait(smem_u32(&T_full[buf]), tpar);
      fence_after();
      for (int g = 0; g < g_eff; ++g) {
        const long long t = (long long)(mb0 + g) * kBM + row;
        float* dst = p.M + (long long)xi * p.N * p.T_pad + t;
        const long long ts = p.T_pad;
        for (int c0 = 0; c0 < p.Nst; c0 += 16) {
          uint32_t r[16];
          const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(buf * 256 + g * p.N + c0);
          tmem_ld16(taddr, r);
          tmem_ld_wait();
          float* d = dst + (long long)c0 * ts;
          const int nj = p.Nst - c0;
          if (nj >= 16) {
#pragma unroll
            for (int j = 0; j < 16; ++j) d[j * ts] = __uint_as_float(r[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j < nj) d[j * ts] = __uint_as_float(r[j]);
          }
        }
      }
      fence_before();
      mbar_arrive(smem_u32(&T_empty[buf]));
    }
  }
  fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync();  // no CTA leaves while its pair may still multicast into it
  fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512u));
}


// ---------------------------------------------------------------------------
// Contraction with the inner level of the output transform fused into the
// epilogue (Y = A^T_hat M A_hat, A^T_hat = A_o^T (x) A_i^T).  A unit is
// the l_i consecutive points (p_h, p_o, p_i = 0 .. l_i-1) of one 128-slice
// block; their accumulators land in a ring of NSLOT TMEM slots (N columns each),
// and 8 epilogue warps (two per TMEM lane quarter, one column half each) fold
// each slot into m_i partial sums with the compile-time A_i^T as soon as it is
// committed, so only M' = (A_i^T along w) M -- m_i/l_i of M -- reaches HBM:
//   M'[((p_h * l_o + p_o) * m_i + s)][co][t] = sum_{p_i} A_i^T[s][p_i] M[(p_h, p_o, p_i)][co][t]
// ---------------------------------------------------------------------------
constexpr int kFuseThreads = 320;  // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue
constexpr int kSlots = 8;

struct FusedParams {
  int nmb, N, KB, lo, nst;
  int kbk;                // K block width in bf16 elements (64, 32 or 16)
  int PA, LO;             // points per axis, outer points per axis
  long long T_pad;
  long long a_lo_row, b_lo_row;
  int P, vblk;
  float* Mp;
  // streamed pipeline (api.cu forward_streamed): units walk 128-slice blocks in order (sb blocks
  // per sweep of the point groups, so one U point group serves sb blocks back to back); before
  // the first V load of block mb the producer waits for ready[mb] >= rdy_per_slice * (real
  // slices of mb); each finished unit adds 1 to done[mb] for the output transform.
  const int* ready;
  int* done;
  int rdy_per_slice, sb;
  long long T;
};

// unit u -> (point group pg = p_h * l_o + p_o, 128-slice block mb)
__device__ __forceinline__ void fused_unit(const FusedParams& p, int u, int& pg, int& mb) {
  const int PG = p.PA * p.LO;
  if (p.sb <= 0) {  // point-group major (stream-ordered launches)
    pg = u / p.nmb;
    mb = u - pg * p.nmb;
    return;
  }
  const int gsz = p.sb * PG, grp = u / gsz, r = u - grp * gsz, mb0 = grp * p.sb;
  const int nb = min(p.sb, p.nmb - mb0);
  pg = r / nb;
  mb = mb0 + (r - pg * nb);
}

template <int MI, int NH>
__global__ void __launch_bounds__(kFuseThreads, 1)
    contraction_fused_kernel(const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapU,
                             const FusedParams p) {
  constexpr int LI = MI + 2;
  constexpr Kernel1D KI = make_kernel(MI, 3);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sbase = smem_raw + (base - raw);
  const uint32_t a_plane = kBM * p.kbk * 2, b_plane = (uint32_t)p.N * p.kbk * 2;
  const uint32_t a_bytes = a_plane * (p.lo ? 2 : 1), b_bytes = b_plane * (p.lo ? 2 : 1);
  const uint32_t stage = a_bytes + b_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + (size_t)stage * p.nst);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages;
  uint64_t* s_full = bars + 2 * kMaxStages;
  uint64_t* s_empty = bars + 2 * kMaxStages + kSlots;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kMaxStages + 2 * kSlots);
  // warp index through a shuffle: provably warp-uniform, so the role branches and everything the
  // MMA warp computes stay in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int units = p.nmb * p.PA * p.LO;
  const uint32_t tcols = (uint32_t)(kSlots * p.N) <= 32 ? 32u : (uint32_t)(kSlots * p.N);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapV);
    tma_prefetch(&mapU);
    for (int i = 0; i < p.nst; ++i) { mbar_init(smem_u32(&full[i]), 1); mbar_init(smem_u32(&empty[i]), 1); }
    for (int i = 0; i < kSlots; ++i) { mbar_init(smem_u32(&s_full[i]), 1); mbar_init(smem_u32(&s_empty[i]), 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();
  griddep_wait();  // V comes from the input transform just before in the stream

  if (warp == 0) {
    if (lane == 0) {  // ------------------------- TMA producer -------------------------
      int st = 0;
      uint32_t ph = 0;
      int waited = -1;  // highest block whose V is known complete
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int pg, mb;
        fused_unit(p, u, pg, mb);
        const int p_h = pg / p.LO, p_o = pg - p_h * p.LO;
        if (p.ready) {  // every block of this unit's sweep group (units walk the groups in order)
          const int gsz = p.sb * p.PA * p.LO, last = min(p.nmb, (u / gsz + 1) * p.sb) - 1;
          for (; waited < last; ++waited) {
            const long long s0 = (long long)(waited + 1) * kBM, s1 = min(p.T, s0 + kBM);
            ptx::wait_count(p.ready + waited + 1, p.rdy_per_slice * (int)(s1 - s0));
          }
        }
        for (int pi = 0; pi < LI; ++pi) {
          const int xi = p_h * p.PA + p_o * LI + pi;
          for (int kb = 0; kb < p.KB; ++kb) {
            mbar_wait(smem_u32(&empty[st]), ph ^ 1);
            const uint32_t fb = smem_u32(&full[st]);
            mbar_expect_tx(fb, stage);
            const uint32_t dst = base + (uint32_t)st * stage;
            long long row, lrow;
            if (p.vblk) {
              row = ((long long)mb * p.P + xi) * (2 * kBM);
              lrow = row + kBM;
            } else {
              row = (long long)xi * p.T_pad + (long long)mb * kBM;
              lrow = p.a_lo_row + row;
            }
            tma_load_2d(dst, &mapV, fb, kb * p.kbk, (int)row);
            if (p.lo) tma_load_2d(dst + a_plane, &mapV, fb, kb * p.kbk, (int)lrow);
            tma_load_2d(dst + a_bytes, &mapU, fb, kb * p.kbk, xi * p.N);
            if (p.lo)
              tma_load_2d(dst + a_bytes + b_plane, &mapU, fb, kb * p.kbk, (int)(p.b_lo_row + (long long)xi * p.N));
            if (++st == p.nst) { st = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------- MMA issuer ---------------------------
    // the whole warp walks the loop and waits (uniform control flow keeps the descriptors in
    // uniform registers: no per-MMA register-to-uniform broadcasts); lane 0 issues
    {
      const uint32_t idesc = idesc_bf16(p.N), dhi = swk_desc_hi(p.kbk);
      int st = 0;
      uint32_t ph = 0;
      uint32_t sc = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        for (int pi = 0; pi < LI; ++pi, ++sc) {
          const uint32_t slot = sc % kSlots, spar = (sc / kSlots) & 1;
          mbar_wait(smem_u32(&s_empty[slot]), spar ^ 1);
          fence_after();
          const uint32_t acc = tmem_base + slot * (uint32_t)p.N;
          for (int kb = 0; kb < p.KB; ++kb) {
            mbar_wait(smem_u32(&full[st]), ph);
            fence_after();
            const uint32_t asm_ = base + (uint32_t)st * stage, bsm = asm_ + a_bytes;
            if (elect_one()) {
              issue_kblock_any(p.kbk, acc, asm_ >> 4, bsm >> 4, a_plane >> 4, b_plane >> 4, dhi, idesc, p.lo,
                               kb > 0 ? 1u : 0u);
              umma_commit(smem_u32(&empty[st]));
            }
            __syncwarp();
            if (++st == p.nst) { st = 0; ph ^= 1; }
          }
          if (elect_one()) umma_commit(smem_u32(&s_full[slot]));
          __syncwarp();
        }
      }
    }
  } else {  // ------------------------------- epilogue ----------------------------------
    const int q = warp & 3, half = (warp - 2) >> 2;
    static_assert(NH == 16 || NH == 32, "16 or 32 columns per warp (N = 32 or 64)");
    uint32_t sc = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int pg, mb;
      fused_unit(p, u, pg, mb);
      float out[MI][32];
#pragma unroll
      for (int s = 0; s < MI; ++s)
#pragma unroll
        for (int c = 0; c < 32; ++c) out[s][c] = 0.f;
#pragma unroll
      for (int pi = 0; pi < LI; ++pi, ++sc) {
        const uint32_t slot = sc % kSlots, spar = (sc / kSlots) & 1;
        mbar_wait(smem_u32(&s_full[slot]), spar);
        fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + slot * (uint32_t)p.N + (uint32_t)(half * NH);
        uint32_t r0[16], r1[16];
        tmem_ld16(taddr, r0);
        if (NH == 32) tmem_ld16(taddr + 16, r1);
        tmem_ld_wait();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&s_empty[slot]));
#pragma unroll
        for (int s = 0; s < MI; ++s) {
          const float a = float(rdouble(KI.AT[s][pi]));
          if (a == 0.f) continue;
#pragma unroll
          for (int c = 0; c < 16; ++c) out[s][c] = fmaf(a, __uint_as_float(r0[c]), out[s][c]);
          if (NH == 32) {
#pragma unroll
            for (int c = 0; c < 16; ++c) out[s][16 + c] = fmaf(a, __uint_as_float(r1[c]), out[s][16 + c]);
          }
        }
      }
      const long long t = (long long)mb * kBM + q * 32 + lane;
      // one pointer walked by the channel pitch (T_pad floats): one 64-bit add per store instead
      // of a 64-bit multiply-add chain (the epilogue's address arithmetic was half of the kernel's
      // instructions and kept the MMA waiting for TMEM slots; profiles/r2u)
      float* dst = p.Mp + ((long long)(pg * MI) * p.N + half * NH) * p.T_pad + t;
      const long long pitch = p.T_pad;
      const long long skip = (long long)(p.N - NH) * p.T_pad;  // to the next s row's first column
#pragma unroll
      for (int s = 0; s < MI; ++s) {
#pragma unroll
        for (int c = 0; c < NH; ++c) {
          *dst = out[s][c];
          long long w = pitch;
          asm volatile("" : "+l"(w));  // keep the walk incremental (no hoisted per-store offsets)
          dst += w;
        }
        long long w = skip;
        asm volatile("" : "+l"(w));
        dst += w;
      }
      if (p.done) {  // streamed pipeline: the 8 epilogue warps' M' stores of this unit, then count it
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (warp == 2 && lane == 0) ptx::signal_add(p.done + mb, 1);
      }
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tcols));
}

// ---------------------------------------------------------------------------
// Contraction with the inner output level along BOTH axes fused into the epilogue
// (round 2, NW_FUSE_AI=2): Y = A^T_hat M A_hat with A^T_hat = A_o^T (x) A_i^T, and the inner
// factor acts on the l_i x l_i points (p_ih, p_iw) of one outer point (p_oh, p_ow), so
//   M''[((p_oh * m_i + j_h) * l_o + p_ow) * m_i + j_w][co][t]
//       = sum_{p_ih, p_iw} A_i^T[j_h][p_ih] A_i^T[j_w][p_iw] M[(p_oh, p_ih), (p_ow, p_iw)][co][t]
// is (m_i / l_i)^2 = 9/25 of M (M' is 15/25).  A thread must hold the m_i^2 partial sums of
// its columns across the unit's l_i^2 points, which the register file allows for 16 columns
// per thread: a unit is (outer point pair, 128-slice block, 32-channel half); the two halves
// of one (point pair, block) are consecutive units, i.e. run on two CTAs at the same time,
// so the second read of the A tiles is an L2 hit.  Accumulators rotate through 16 TMEM
// slots of 32 columns; the 8 epilogue warps (lane quarter x column half) fold each
// committed slot with the compile-time products of A_i^T entries.
// ---------------------------------------------------------------------------
constexpr int kSlots2 = 16;
constexpr int kMaxStages2 = 16;  // small-K layers (10 KB stages) need > 8 stages in flight to cover the load latency
// warpgroup 0: warp 0 TMA, warp 1 MMA (2, 3 idle); warpgroups 1, 2: epilogue.  setmaxnreg moves
// registers from warpgroup 0 to the epilogue warps, whose 144 partial sums + two slot buffers
// exceed the 168 registers a 12-warp CTA starts with.
constexpr int kFuse2Threads = 384;
constexpr int kN2 = 32;  // channels per unit

struct Fused2Params {
  int nmb, N, nhalf, KB, lo, nst;
  int kbk;
  int PA, LO;
  long long T_pad;
  long long a_lo_row, b_lo_row;
  int P, vblk;
  float* Mpp;
};

template <int MI, int CL>
__global__ void __launch_bounds__(kFuse2Threads, 1)
    contraction_fused2_kernel(const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapU,
                              const Fused2Params p) {
  constexpr int LI = MI + 2;
  constexpr Kernel1D KI = make_kernel(MI, 3);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sbase = smem_raw + (base - raw);
  const uint32_t a_plane = kBM * p.kbk * 2, b_plane = (uint32_t)kN2 * p.kbk * 2;
  const uint32_t a_bytes = a_plane * (p.lo ? 2 : 1), b_bytes = b_plane * (p.lo ? 2 : 1);
  const uint32_t stage = a_bytes + b_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + (size_t)stage * p.nst);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages2;
  uint64_t* s_full = bars + 2 * kMaxStages2;
  uint64_t* s_empty = bars + 2 * kMaxStages2 + kSlots2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kMaxStages2 + 2 * kSlots2);
  // warp index through a shuffle: provably warp-uniform, so the role branches and everything the
  // MMA warp computes stay in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  // CL = 2: the two channel halves of a (point pair, block) run on the two CTAs of a cluster; each
  // CTA loads 64 of the 128 rows of every A tile and multicasts them to both, so V is read from
  // L2 once per pair (unpaired CTAs drifted apart and the second read came from HBM)
  const int units = p.nmb * p.LO * p.LO * (CL > 1 ? 1 : p.nhalf);
  const int rank = (CL > 1) ? (int)cluster_rank() : 0;
  const int ustart = (int)blockIdx.x / CL, ustep = (int)gridDim.x / CL;
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);
  constexpr uint32_t tcols = kSlots2 * kN2;  // 512
  // 3 groups of l_i slots are in use: the epilogue releases a whole group at once (one
  // tcgen05 fence + arrive per l_i points instead of per point: the per-point release was a
  // third of the epilogue's time on small-K layers), the MMA warp waits once per group
  constexpr uint32_t kUsed = 3 * LI;
  static_assert(kUsed <= kSlots2, "slot groups");

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapV);
    tma_prefetch(&mapU);
    for (int i = 0; i < p.nst; ++i) { mbar_init(smem_u32(&full[i]), 1); mbar_init(smem_u32(&empty[i]), CL); }
    for (int i = 0; i < kSlots2; ++i) { mbar_init(smem_u32(&s_full[i]), 1); mbar_init(smem_u32(&s_empty[i]), 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync();  // every CTA's barriers are initialised before multicasts target them
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();
  griddep_wait();  // V comes from the input transform just before in the stream

  // unit u -> (outer point pair pg = p_oh * l_o + p_ow, block mb, channel half nh), half fastest
  auto decode = [&](int u, int& pg, int& mb, int& nh) {
    nh = (CL > 1) ? rank : u % p.nhalf;
    const int r = (CL > 1) ? u : u / p.nhalf;
    pg = r / p.nmb;
    mb = r - pg * p.nmb;
  };

  if (warp < 4) {  // warpgroup 0 gives registers away; its role code stays inside this branch
  asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
  if (warp == 0) {
    {  // ------------------------- TMA producer (warp-uniform loop, one elected lane issues) -------------------------
      int st = 0;
      uint32_t ph = 0;
      for (int u = ustart; u < units; u += ustep) {
        int pg, mb, nh;
        decode(u, pg, mb, nh);
        const int p_oh = pg / p.LO, p_ow = pg - p_oh * p.LO;
        for (int pt = 0; pt < LI * LI; ++pt) {
          const int pih = pt / LI, piw = pt - pih * LI;
          const int xi = (p_oh * LI + pih) * p.PA + p_ow * LI + piw;
          for (int kb = 0; kb < p.KB; ++kb) {
            mbar_wait(smem_u32(&empty[st]), ph ^ 1);
            const uint32_t fb = smem_u32(&full[st]);
            const uint32_t dst = base + (uint32_t)st * stage;
            long long row, lrow;
            if (p.vblk) {
              row = ((long long)mb * p.P + xi) * (2 * kBM);
              lrow = row + kBM;
            } else {
              row = (long long)xi * p.T_pad + (long long)mb * kBM;
              lrow = p.a_lo_row + row;
            }
            if (elect_one()) {
            mbar_expect_tx(fb, stage);
            if constexpr (CL > 1) {
              const int hr = kBM / CL;  // this CTA's rows of the A tile, multicast to the pair
              const uint32_t so = (uint32_t)(rank * hr) * (uint32_t)(p.kbk * 2);
              tma_load_2d_mc(dst + so, &mapV, fb, kb * p.kbk, (int)row + rank * hr, kMask);
              if (p.lo) tma_load_2d_mc(dst + a_plane + so, &mapV, fb, kb * p.kbk, (int)lrow + rank * hr, kMask);
            } else {
              tma_load_2d(dst, &mapV, fb, kb * p.kbk, (int)row);
              if (p.lo) tma_load_2d(dst + a_plane, &mapV, fb, kb * p.kbk, (int)lrow);
            }
            const int brow = xi * p.N + nh * kN2;
            tma_load_2d(dst + a_bytes, &mapU, fb, kb * p.kbk, brow);
            if (p.lo) tma_load_2d(dst + a_bytes + b_plane, &mapU, fb, kb * p.kbk, (int)(p.b_lo_row + brow));
            }
            __syncwarp();
            if (++st == p.nst) { st = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------- MMA issuer (warp-uniform loop, lane 0 issues) ---------------------------
    {
      const uint32_t idesc = idesc_bf16(kN2), dhi = swk_desc_hi(p.kbk);
      int st = 0;
      uint32_t ph = 0;
      uint32_t sc = 0;
      for (int u = ustart; u < units; u += ustep) {
        for (int pt = 0; pt < LI * LI; ++pt, ++sc) {
          const uint32_t slot = sc % kUsed, spar = (sc / kUsed) & 1;
          if (slot % LI == 0) {  // first slot of a group: the epilogue has drained the group's previous use
            mbar_wait(smem_u32(&s_empty[slot / LI]), spar ^ 1);
            fence_after();
          }
          const uint32_t acc = tmem_base + slot * (uint32_t)kN2;
          for (int kb = 0; kb < p.KB; ++kb) {
            mbar_wait(smem_u32(&full[st]), ph);
            fence_after();
            const uint32_t asm_ = base + (uint32_t)st * stage, bsm = asm_ + a_bytes;
            if (elect_one()) {
              issue_kblock_any(p.kbk, acc, asm_ >> 4, bsm >> 4, a_plane >> 4, b_plane >> 4, dhi, idesc, p.lo,
                               kb > 0 ? 1u : 0u);
              if constexpr (CL > 1) umma_commit_mc(smem_u32(&empty[st]), kMask);  // frees the stage in both CTAs
              else umma_commit(smem_u32(&empty[st]));
            }
            __syncwarp();
            if (++st == p.nst) { st = 0; ph ^= 1; }
          }
          if (elect_one()) umma_commit(smem_u32(&s_full[slot]));
          __syncwarp();
        }
      }
    }
  }
  } else {  // ------------------------------- epilogue (warpgroups 1 and 2) ----------------------------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
    const int q = warp & 3, half = (warp - 4) >> 2;
    uint32_t sc = 0;
    for (int u = ustart; u < units; u += ustep) {
      int pg, mb, nh;
      decode(u, pg, mb, nh);
      const int p_oh = pg / p.LO, p_ow = pg - p_oh * p.LO;
      float out[MI][MI][16];
#pragma unroll
      for (int a = 0; a < MI; ++a)
#pragma unroll
        for (int b = 0; b < MI; ++b)
#pragma unroll
          for (int c = 0; c < 16; ++c) out[a][b][c] = 0.f;
      // software pipeline over the unit's l_i^2 slots: the TMEM load of slot pt + 1 is in flight
      // while slot pt is folded (two register buffers).  A partial sum (j_h, j_w) is final after the
      // last point with non-zero A_i^T[j_h][p_ih] A_i^T[j_w][p_iw]; it is stored right then, so most
      // of the unit's 144 stores per thread overlap the remaining points instead of queueing up in
      // the load/store unit after the last one.
      const long long t = (long long)mb * kBM + q * 32 + lane;
      const int col0 = nh * kN2 + half * 16;
      const int rl = p.LO * MI;  // M'' values per row of the (p_oh, j_h) grid
      const long long pitch = p.T_pad;
      auto store_out = [&](int jh, int jw) {
        const long long R = (long long)(p_oh * MI + jh) * rl + p_ow * MI + jw;
        float* dst = p.Mpp + (R * p.N + col0) * p.T_pad + t;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          *dst = out[jh][jw][c];
          long long w = pitch;
          asm volatile("" : "+l"(w));  // keep the walk incremental (no hoisted per-store offsets)
          dst += w;
        }
      };
      uint32_t rbuf[2][16];
      const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(half * 16);
      {
        const uint32_t slot = sc % kUsed, spar = (sc / kUsed) & 1;
        mbar_wait(smem_u32(&s_full[slot]), spar);
        fence_after();
        tmem_ld16(tq + slot * (uint32_t)kN2, rbuf[0]);
      }
#pragma unroll
      for (int pt = 0; pt < LI * LI; ++pt, ++sc) {
        const int pih = pt / LI, piw = pt % LI;
        const uint32_t slot = sc % kUsed;
        tmem_ld_wait();
        if (pt % LI == LI - 1) {  // the group's last slot is in registers: release the group
          fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&s_empty[slot / LI]));
        }
        if (pt + 1 < LI * LI) {
          const uint32_t sn = (sc + 1) % kUsed, spn = ((sc + 1) / kUsed) & 1;
          mbar_wait(smem_u32(&s_full[sn]), spn);
          fence_after();
          tmem_ld16(tq + sn * (uint32_t)kN2, rbuf[(pt + 1) & 1]);
        }
#pragma unroll
        for (int jh = 0; jh < MI; ++jh) {
          const float ah = float(rdouble(KI.AT[jh][pih]));
          if (ah == 0.f) continue;
#pragma unroll
          for (int jw = 0; jw < MI; ++jw) {
            const float a = ah * float(rdouble(KI.AT[jw][piw]));
            if (a == 0.f) continue;
#pragma unroll
            for (int c = 0; c < 16; ++c)
              out[jh][jw][c] = fmaf(a, __uint_as_float(rbuf[pt & 1][c]), out[jh][jw][c]);
          }
        }
        // partial sums whose last contributing point this was
#pragma unroll
        for (int jh = 0; jh < MI; ++jh) {
#pragma unroll
          for (int jw = 0; jw < MI; ++jw) {
            int lh = 0, lw = 0;
#pragma unroll
            for (int k = 0; k < LI; ++k) {
              if (rdouble(KI.AT[jh][k]) != 0.0) lh = k;
              if (rdouble(KI.AT[jw][k]) != 0.0) lw = k;
            }
            if (pih == lh && piw == lw) store_out(jh, jw);
          }
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync();  // no CTA leaves while its pair may still multicast into it
  fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tcols));
}

// ---------------------------------------------------------------------------
// Level-1 fusion for wide layers (Cout_pad = 128 or 256, e.g. C3): the inner output level along
// w in the epilogue, 128 channels per CTA.  Five 256-column accumulators do not fit TMEM and a
// 64-channel unit would re-read every A tile four times, so the two 128-channel halves of a
// (point group, block) run on the two CTAs of a cluster that multicast the A tiles to each other
// (same scheme as contraction_fused2_kernel).  4 TMEM slots of 128 columns; 8 epilogue warps
// (lane quarter x 64 columns) hold m_i x 64 partial sums each (setmaxnreg 232).  M' is 3/5 of M.
// ---------------------------------------------------------------------------
constexpr int kSlotsC = 4;
constexpr int kNC = 128;

template <int MI, int CL>
__global__ void __launch_bounds__(kFuse2Threads, 1)
    contraction_fused1c_kernel(const __grid_constant__ CUtensorMap mapV, const __grid_constant__ CUtensorMap mapU,
                               const Fused2Params p) {
  constexpr int LI = MI + 2;
  constexpr Kernel1D KI = make_kernel(MI, 3);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* sbase = smem_raw + (base - raw);
  const uint32_t a_plane = kBM * p.kbk * 2, b_plane = (uint32_t)kNC * p.kbk * 2;
  const uint32_t a_bytes = a_plane * (p.lo ? 2 : 1), b_bytes = b_plane * (p.lo ? 2 : 1);
  const uint32_t stage = a_bytes + b_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sbase + (size_t)stage * p.nst);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages2;
  uint64_t* s_full = bars + 2 * kMaxStages2;
  uint64_t* s_empty = bars + 2 * kMaxStages2 + kSlotsC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kMaxStages2 + 2 * kSlotsC);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int units = p.nmb * p.PA * p.LO;  // (point group, block) per CTA (CL = 1) or per pair
  const int rank = (CL > 1) ? (int)cluster_rank() : 0;
  const int ustart = (int)blockIdx.x / CL, ustep = (int)gridDim.x / CL;
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);
  constexpr uint32_t tcols = kSlotsC * kNC;  // 512

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapV);
    tma_prefetch(&mapU);
    for (int i = 0; i < p.nst; ++i) { mbar_init(smem_u32(&full[i]), 1); mbar_init(smem_u32(&empty[i]), CL); }
    for (int i = 0; i < kSlotsC; ++i) { mbar_init(smem_u32(&s_full[i]), 1); mbar_init(smem_u32(&s_empty[i]), 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(tcols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  griddep_launch_dependents();
  griddep_wait();

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp == 0) {  // ------------------------- TMA producer -------------------------
      int st = 0;
      uint32_t ph = 0;
      for (int u = ustart; u < units; u += ustep) {
        const int pg = u / p.nmb, mb = u - pg * p.nmb;
        const int p_h = pg / p.LO, p_o = pg - p_h * p.LO;
        for (int pi = 0; pi < LI; ++pi) {
          const int xi = p_h * p.PA + p_o * LI + pi;
          for (int kb = 0; kb < p.KB; ++kb) {
            mbar_wait(smem_u32(&empty[st]), ph ^ 1);
            const uint32_t fb = smem_u32(&full[st]);
            const uint32_t dst = base + (uint32_t)st * stage;
            long long row, lrow;
            if (p.vblk) {
              row = ((long long)mb * p.P + xi) * (2 * kBM);
              lrow = row + kBM;
            } else {
              row = (long long)xi * p.T_pad + (long long)mb * kBM;
              lrow = p.a_lo_row + row;
            }
            if (elect_one()) {
              mbar_expect_tx(fb, stage);
              if constexpr (CL > 1) {
                const int hr = kBM / CL;
                const uint32_t so = (uint32_t)(rank * hr) * (uint32_t)(p.kbk * 2);
                tma_load_2d_mc(dst + so, &mapV, fb, kb * p.kbk, (int)row + rank * hr, kMask);
                if (p.lo) tma_load_2d_mc(dst + a_plane + so, &mapV, fb, kb * p.kbk, (int)lrow + rank * hr, kMask);
              } else {
                tma_load_2d(dst, &mapV, fb, kb * p.kbk, (int)row);
                if (p.lo) tma_load_2d(dst + a_plane, &mapV, fb, kb * p.kbk, (int)lrow);
              }
              const int brow = xi * p.N + rank * kNC;
              tma_load_2d(dst + a_bytes, &mapU, fb, kb * p.kbk, brow);
              if (p.lo) tma_load_2d(dst + a_bytes + b_plane, &mapU, fb, kb * p.kbk, (int)(p.b_lo_row + brow));
            }
            __syncwarp();
            if (++st == p.nst) { st = 0; ph ^= 1; }
          }
        }
      }
    } else if (warp == 1) {  // ------------------------- MMA issuer ---------------------------
      const uint32_t idesc = idesc_bf16(kNC), dhi = swk_desc_hi(p.kbk);
      int st = 0;
      uint32_t ph = 0;
      uint32_t sc = 0;
      for (int u = ustart; u < units; u += ustep) {
        for (int pi = 0; pi < LI; ++pi, ++sc) {
          const uint32_t slot = sc % kSlotsC, spar = (sc / kSlotsC) & 1;
          mbar_wait(smem_u32(&s_empty[slot]), spar ^ 1);
          fence_after();
          const uint32_t acc = tmem_base + slot * (uint32_t)kNC;
          for (int kb = 0; kb < p.KB; ++kb) {
            mbar_wait(smem_u32(&full[st]), ph);
            fence_after();
            const uint32_t asm_ = base + (uint32_t)st * stage, bsm = asm_ + a_bytes;
            if (elect_one()) {
              issue_kblock_any(p.kbk, acc, asm_ >> 4, bsm >> 4, a_plane >> 4, b_plane >> 4, dhi, idesc, p.lo,
                               kb > 0 ? 1u : 0u);
              if constexpr (CL > 1) umma_commit_mc(smem_u32(&empty[st]), kMask);
              else umma_commit(smem_u32(&empty[st]));
            }
            __syncwarp();
            if (++st == p.nst) { st = 0; ph ^= 1; }
          }
          if (elect_one()) umma_commit(smem_u32(&s_full[slot]));
          __syncwarp();
        }
      }
    }
  } else {  // ------------------------------- epilogue (warpgroups 1 and 2) ----------------------------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
    const int q = warp & 3, half = (warp - 4) >> 2;
    uint32_t sc = 0;
    for (int u = ustart; u < units; u += ustep) {
      const int pg = u / p.nmb, mb = u - pg * p.nmb;
      float out[MI][64];
#pragma unroll
      for (int s2 = 0; s2 < MI; ++s2)
#pragma unroll
        for (int c = 0; c < 64; ++c) out[s2][c] = 0.f;
      const long long t = (long long)mb * kBM + q * 32 + lane;
      const int col0 = rank * kNC + half * 64;
      const long long pitch = p.T_pad;
      // a partial sum is stored as soon as its last contributing point is folded (two of the three
      // rows after point l_i - 2), so most stores overlap the unit's last point
      auto store_out = [&](int s2) {
        float* dst = p.Mpp + ((long long)(pg * MI + s2) * p.N + col0) * p.T_pad + t;
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          *dst = out[s2][c];
          long long w = pitch;
          asm volatile("" : "+l"(w));
          dst += w;
        }
      };
#pragma unroll
      for (int pi = 0; pi < LI; ++pi, ++sc) {
        const uint32_t slot = sc % kSlotsC, spar = (sc / kSlotsC) & 1;
        mbar_wait(smem_u32(&s_full[slot]), spar);
        fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + slot * (uint32_t)kNC + (uint32_t)(half * 64);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t r0[16];
          tmem_ld16(taddr + ch * 16, r0);
          tmem_ld_wait();
          if (ch == 3) {  // the slot's last columns are in registers: release it
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&s_empty[slot]));
          }
#pragma unroll
          for (int s2 = 0; s2 < MI; ++s2) {
            const float a = float(rdouble(KI.AT[s2][pi]));
            if (a == 0.f) continue;
#pragma unroll
            for (int c = 0; c < 16; ++c) out[s2][ch * 16 + c] = fmaf(a, __uint_as_float(r0[c]), out[s2][ch * 16 + c]);
          }
        }
#pragma unroll
        for (int s2 = 0; s2 < MI; ++s2) {
          int last = 0;
#pragma unroll
          for (int k = 0; k < LI; ++k)
            if (rdouble(KI.AT[s2][k]) != 0.0) last = k;
          if (pi == last) store_out(s2);
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync();
  fence_after();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tcols));
}

}  // namespace tc

// ------------------------------ host side ------------------------------------
// 2-D bf16 tensor map [rows][cols] with a (64 x box_rows) box, 128-byte swizzle.
static bool make_map(CUtensorMap* m, const void* base, long long rows, long long cols, int box_rows, int kbk = 64) {
  const uint64_t dims[2] = {(uint64_t)cols, (uint64_t)rows};
  const uint64_t strides[1] = {(uint64_t)cols * 2};
  const uint32_t box[2] = {(uint32_t)kbk, (uint32_t)box_rows};
  const CUtensorMapSwizzle sw =
      kbk == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : (kbk == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  return encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, sw);
}

// K block width: the whole contraction channel pitch when it is 16 or 32 (no zero padding to
// 64 in the MMA K loop), else 64.  NW_KBK=64 forces the wide block.
static int pick_kbk(int cin_pad) {
  static const int force = [] {
    const char* v = getenv("NW_KBK");
    return v ? atoi(v) : 0;
  }();
  if (force == 64) return 64;
  return (cin_pad == 16 || cin_pad == 32) ? cin_pad : 64;
}

nw_status_t launch_gemm_tc(const nw_plan_st* p, const Geometry& g, const void* V, const void* U, float* M,
                           cudaStream_t s) {
  if (g.cout_pad > 256) return NW_ERR_UNSUPPORTED;
  tc::Params prm{};
  prm.P = g.P;
  prm.nmb = (int)(g.T_pad / tc::kBM);
  prm.N = g.cout_pad;
  prm.Nst = g.cout_e;
  // blocks per unit: fill the 256-column TMEM buffer (narrow N: up to 16 blocks share one B load
  // and one round of unit synchronisation); NW_GEMM_G caps it
  static const int g_cap = [] {
    const char* v = getenv("NW_GEMM_G");
    return v ? atoi(v) : 16;
  }();
  prm.G = 256 / prm.N;
  if (prm.G > g_cap) prm.G = g_cap;
  if (prm.G < 1) prm.G = 1;
  // small layers: keep at least two units per SM
  while (prm.G > 1 && (long long)prm.P * ((prm.nmb + prm.G - 1) / prm.G) < 2 * 148) prm.G /= 2;
  prm.ngrp = (prm.nmb + prm.G - 1) / prm.G;
  if (g.nsh < 1 || g.nsh > kMaxShift) return NW_ERR_UNSUPPORTED;
  prm.nsh = g.nsh;
  prm.kbk = pick_kbk(g.cin_pad);
  prm.kbc = (g.cin_pad + prm.kbk - 1) / prm.kbk;
  prm.cin_pad = g.cin_pad;
  prm.KB = prm.nsh * prm.kbc;
  for (int b = 0; b < g.nsh; ++b) prm.shoff[b] = (b / g.nb) * g.tiles_w + (b % g.nb);  // Eq. 2.3 block shift
  prm.lo = (p->math == NW_MATH_BF16X3) ? 1 : 0;
  prm.T_pad = g.T_pad;
  prm.a_lo_row = (long long)g.P * g.T_pad;
  prm.b_lo_row = (long long)g.P * g.cout_pad;
  prm.vblk = (g.vblk && prm.lo) ? 1 : 0;
  prm.M = M;
  const uint32_t a_stage = tc::kBM * prm.kbk * 2 * (prm.lo ? 2 : 1);
  const uint32_t b_stage = (uint32_t)prm.N * prm.kbk * 2 * (prm.lo ? 2 : 1);
  // ring depths within ~200 KB
  const uint32_t budget = 200 * 1024;
  prm.nB = 2;
  prm.nA = (int)((budget - prm.nB * b_stage) / a_stage);
  if (prm.nA > tc::kMaxStages) prm.nA = tc::kMaxStages;
  if (prm.nA < 2) {
    prm.nB = 1;
    prm.nA = (int)((budget - b_stage) / a_stage);
    if (prm.nA < 2) return NW_ERR_UNSUPPORTED;
  }
  size_t smem = 1024 + (size_t)a_stage * prm.nA + (size_t)b_stage * prm.nB + (4 * tc::kMaxStages + 8) * 8;
  if (smem < 120 * 1024) smem = 120 * 1024;  // one CTA per SM: each CTA owns all 512 TMEM columns
  const long long rowsV = (long long)g.P * g.T_pad * (prm.lo ? 2 : 1);
  const long long rowsU = (long long)g.P * g.cout_pad * (prm.lo ? 2 : 1);
  if (rowsV >= (1ll << 31)) return NW_ERR_UNSUPPORTED;
  alignas(64) CUtensorMap mapV, mapU;
  if (!make_map(&mapV, V, rowsV, g.cin_pad, tc::kBM, prm.kbk)) return NW_ERR_CUDA;
  // CTA pairs share B when one B k-block serves a single A block (N > 128) and there is more
  // than one block per point: B is then read from L2 once per pair (NW_CLUSTER=1 disables)
  static const int cl_env = [] {
    const char* v = getenv("NW_CLUSTER");
    return v ? atoi(v) : 2;
  }();
  // pairs need two CTAs: a grid cap below 2 (NW_GEMM_CTAS=1 in the chunk pipeline) runs unpaired
  const int CL = (cl_env == 2 && prm.G == 1 && prm.nmb >= 2 && g.nsh == 1 && prm.N % 16 == 0 &&
                  (g.gemm_ctas <= 0 || g.gemm_ctas >= 2)) ? 2 : 1;
  if (CL > 1) prm.ngrp = (prm.nmb + CL - 1) / CL;
  if (!make_map(&mapU, U, rowsU, (long long)g.nsh * g.cin_pad, prm.N / CL, prm.kbk)) return NW_ERR_CUDA;
  if (CL > 1 ? ensure_smem<tc::contraction_kernel<2>>(227 * 1024) != NW_OK
             : ensure_smem<tc::contraction_kernel<1>>(227 * 1024) != NW_OK)
    return NW_ERR_CUDA;
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long units = (long long)prm.P * prm.ngrp * CL;  // CTA-units
  if (g.gemm_ctas > 0 && g.gemm_ctas < sms) sms = g.gemm_ctas;
  int grid = (int)(units < sms ? units : sms);
  grid -= grid % CL;
  LaunchScope scope_("contraction_tc", s);
  if (CL > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tc::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, tc::contraction_kernel<2>, mapV, mapU, prm) != cudaSuccess) return NW_ERR_CUDA;
  } else if (launch_pdl(tc::contraction_kernel<1>, dim3(grid), dim3(tc::kThreads), smem, s, mapV, mapU, prm) !=
             NW_OK) {
    return NW_ERR_CUDA;
  }
  return check_launch();
}

// Fused contraction + inner output level (see contraction_fused_kernel).  Eligible
// for the nested path in the tensor-core modes with Cout_pad in {32, 64} and
// inner F(3,3); M' ([P_a * l_o * m_i][cout_pad][T_pad]) is written to M.
static int fuse_ai_env() {  // NW_FUSE_AI: 0 off, 1 inner level along w, 2 along both axes (default)
  static const int on = [] {
    const char* v = getenv("NW_FUSE_AI");
    return v ? atoi(v) : 2;
  }();
  return on;
}
bool gemm_fused_eligible(const nw_plan_st* p, const Geometry& g) {
  return fuse_ai_env() && !p->depthwise && g.path == kPathNested && p->math != NW_MATH_FP32_SIMT &&
         (g.cout_pad == 32 || g.cout_pad == 64) &&
         g.mi == 3 && g.nsh == 1;
}
// 0: plain contraction (M), 1: M' (inner level along w), 2: M'' (inner level along both axes;
// stream-ordered launches only: the streamed pipeline's counters belong to level 1)
// wide layers (Cout_pad 128 / 256): level 1 on 128-channel CTAs / CTA pairs (contraction_fused1c_kernel);
// NW_FUSE_WIDE=0 keeps the plain contraction
bool gemm_fused_wide(const nw_plan_st* p, const Geometry& g) {
  static const int on = [] {
    const char* v = getenv("NW_FUSE_WIDE");
    return v ? atoi(v) : 1;
  }();
  return on && fuse_ai_env() && !p->depthwise && g.path == kPathNested && p->math != NW_MATH_FP32_SIMT &&
         (g.cout_pad == 128 || g.cout_pad == 256) && g.mi == 3 && g.nsh == 1 && !g.sync && !g.sync2 &&
         (g.gemm_ctas <= 0 || g.gemm_ctas >= 2);
}
int gemm_fused_level(const nw_plan_st* p, const Geometry& g) {
  if (gemm_fused_wide(p, g)) return 1;
  if (!gemm_fused_eligible(p, g)) return 0;
  return (fuse_ai_env() >= 2 && !g.sync && !g.sync2) ? 2 : 1;
}

nw_status_t launch_gemm_tc_fused1c(const nw_plan_st* p, const Geometry& g, const void* V, const void* U, float* Mp,
                                   cudaStream_t s) {
  tc::Fused2Params prm{};
  prm.nmb = (int)(g.T_pad / tc::kBM);
  prm.N = g.cout_pad;
  prm.nhalf = g.cout_pad / tc::kNC;
  // K block width: 64 KB stages (kbk 64) leave two stages of loads in flight behind the one being
  // multiplied; narrower blocks keep more bytes in flight in the same shared memory (NW_KBK_WIDE)
  static const int kbk_env = [] {
    const char* v = getenv("NW_KBK_WIDE");
    return v ? atoi(v) : 0;
  }();
  prm.kbk = pick_kbk(g.cin_pad);
  if ((kbk_env == 16 || kbk_env == 32) && g.cin_pad % kbk_env == 0 && prm.kbk > kbk_env) prm.kbk = kbk_env;
  prm.KB = (g.cin_pad + prm.kbk - 1) / prm.kbk;
  prm.lo = (p->math == NW_MATH_BF16X3) ? 1 : 0;
  const NestedAxis ax = path_axis(p, g.path);
  prm.PA = ax.Pa;
  prm.LO = ax.l_o;
  prm.T_pad = g.T_pad;
  prm.a_lo_row = (long long)g.P * g.T_pad;
  prm.b_lo_row = (long long)g.P * g.cout_pad;
  prm.P = g.P;
  prm.vblk = (g.vblk && prm.lo) ? 1 : 0;
  prm.Mpp = Mp;
  const uint32_t stage = (tc::kBM * prm.kbk * 2 + (uint32_t)tc::kNC * prm.kbk * 2) * (prm.lo ? 2 : 1);
  prm.nst = (int)((200u * 1024u) / stage);
  if (prm.nst > tc::kMaxStages2) prm.nst = tc::kMaxStages2;
  if (prm.nst < 2) return NW_ERR_UNSUPPORTED;
  size_t smem = 1024 + (size_t)stage * prm.nst + (2 * tc::kMaxStages2 + 2 * tc::kSlotsC + 2) * 8;
  if (smem < 120 * 1024) smem = 120 * 1024;  // one CTA per SM: each CTA owns all 512 TMEM columns
  const long long rowsV = (long long)g.P * g.T_pad * (prm.lo ? 2 : 1);
  const long long rowsU = (long long)g.P * g.cout_pad * (prm.lo ? 2 : 1);
  if (rowsV >= (1ll << 31)) return NW_ERR_UNSUPPORTED;
  alignas(64) CUtensorMap mapV, mapU;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (g.gemm_ctas > 0 && g.gemm_ctas < sms) sms = g.gemm_ctas;
  const int CL = prm.nhalf;  // 1 or 2
  if (!make_map(&mapV, V, rowsV, g.cin_pad, tc::kBM / CL, prm.kbk)) return NW_ERR_CUDA;
  if (!make_map(&mapU, U, rowsU, g.cin_pad, tc::kNC, prm.kbk)) return NW_ERR_CUDA;
  if ((CL > 1 ? ensure_smem<tc::contraction_fused1c_kernel<3, 2>>(227 * 1024)
              : ensure_smem<tc::contraction_fused1c_kernel<3, 1>>(227 * 1024)) != NW_OK)
    return NW_ERR_CUDA;
  const long long units = (long long)prm.nmb * prm.PA * prm.LO * CL;  // CTA-units
  int grid = (int)(units < sms ? units : sms);
  if (grid > CL) grid -= grid % CL;
  LaunchScope scope_("contraction_tc", s);
  if (CL > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tc::kFuse2Threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, tc::contraction_fused1c_kernel<3, 2>, mapV, mapU, prm) != cudaSuccess)
      return NW_ERR_CUDA;
  } else if (launch_pdl(tc::contraction_fused1c_kernel<3, 1>, dim3(grid), dim3(tc::kFuse2Threads), smem, s, mapV,
                        mapU, prm) != NW_OK) {
    return NW_ERR_CUDA;
  }
  return check_launch();
}

nw_status_t launch_gemm_tc_fused2(const nw_plan_st* p, const Geometry& g, const void* V, const void* U, float* Mpp,
                                  cudaStream_t s) {
  tc::Fused2Params prm{};
  prm.nmb = (int)(g.T_pad / tc::kBM);
  prm.N = g.cout_pad;
  prm.nhalf = g.cout_pad / tc::kN2;
  prm.kbk = pick_kbk(g.cin_pad);
  prm.KB = (g.cin_pad + prm.kbk - 1) / prm.kbk;
  prm.lo = (p->math == NW_MATH_BF16X3) ? 1 : 0;
  const NestedAxis ax = path_axis(p, g.path);
  prm.PA = ax.Pa;
  prm.LO = ax.l_o;
  prm.T_pad = g.T_pad;
  prm.a_lo_row = (long long)g.P * g.T_pad;
  prm.b_lo_row = (long long)g.P * g.cout_pad;
  prm.P = g.P;
  prm.vblk = (g.vblk && prm.lo) ? 1 : 0;
  prm.Mpp = Mpp;
  const uint32_t stage = (tc::kBM * prm.kbk * 2 + (uint32_t)tc::kN2 * prm.kbk * 2) * (prm.lo ? 2 : 1);
  prm.nst = (int)((200u * 1024u) / stage);
  if (prm.nst > tc::kMaxStages2) prm.nst = tc::kMaxStages2;
  if (prm.nst < 2) return NW_ERR_UNSUPPORTED;
  size_t smem = 1024 + (size_t)stage * prm.nst + (2 * tc::kMaxStages2 + 2 * tc::kSlots2 + 2) * 8;
  if (smem < 120 * 1024) smem = 120 * 1024;  // one CTA per SM: each CTA owns all 512 TMEM columns
  const long long rowsV = (long long)g.P * g.T_pad * (prm.lo ? 2 : 1);
  const long long rowsU = (long long)g.P * g.cout_pad * (prm.lo ? 2 : 1);
  if (rowsV >= (1ll << 31)) return NW_ERR_UNSUPPORTED;
  alignas(64) CUtensorMap mapV, mapU;
  // CTA pairs (one channel half each, A multicast) when the layer has two halves; NW_CLUSTER=1 unpairs
  static const int cl_env = [] {
    const char* v = getenv("NW_CLUSTER");
    return v ? atoi(v) : 2;
  }();
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (g.gemm_ctas > 0 && g.gemm_ctas < sms) sms = g.gemm_ctas;
  const int CL = (prm.nhalf == 2 && cl_env == 2 && sms >= 2) ? 2 : 1;
  if (!make_map(&mapV, V, rowsV, g.cin_pad, tc::kBM / CL, prm.kbk)) return NW_ERR_CUDA;
  if (!make_map(&mapU, U, rowsU, g.cin_pad, tc::kN2, prm.kbk)) return NW_ERR_CUDA;
  if ((CL > 1 ? ensure_smem<tc::contraction_fused2_kernel<3, 2>>(227 * 1024)
              : ensure_smem<tc::contraction_fused2_kernel<3, 1>>(227 * 1024)) != NW_OK)
    return NW_ERR_CUDA;
  const long long units = (long long)prm.nmb * prm.LO * prm.LO * prm.nhalf;  // CTA-units
  int grid = (int)(units < sms ? units : sms);
  if (grid > prm.nhalf) grid -= grid % prm.nhalf;  // the halves of a (point pair, block) stay on CTA pairs
  LaunchScope scope_("contraction_tc", s);
  if (CL > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tc::kFuse2Threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, tc::contraction_fused2_kernel<3, 2>, mapV, mapU, prm) != cudaSuccess)
      return NW_ERR_CUDA;
  } else if (launch_pdl(tc::contraction_fused2_kernel<3, 1>, dim3(grid), dim3(tc::kFuse2Threads), smem, s, mapV, mapU,
                        prm) != NW_OK) {
    return NW_ERR_CUDA;
  }
  return check_launch();
}

nw_status_t launch_gemm_tc_fused(const nw_plan_st* p, const Geometry& g, const void* V, const void* U, float* Mp,
                                 cudaStream_t s) {
  tc::FusedParams prm{};
  prm.nmb = (int)(g.T_pad / tc::kBM);
  prm.N = g.cout_pad;
  prm.kbk = pick_kbk(g.cin_pad);
  prm.KB = (g.cin_pad + prm.kbk - 1) / prm.kbk;
  prm.lo = (p->math == NW_MATH_BF16X3) ? 1 : 0;
  const NestedAxis ax = path_axis(p, g.path);
  prm.PA = ax.Pa;
  prm.LO = ax.l_o;
  prm.T_pad = g.T_pad;
  prm.a_lo_row = (long long)g.P * g.T_pad;
  prm.b_lo_row = (long long)g.P * g.cout_pad;
  prm.P = g.P;
  prm.vblk = (g.vblk && prm.lo) ? 1 : 0;
  prm.Mp = Mp;
  prm.ready = g.sync;
  prm.done = g.sync2;
  prm.rdy_per_slice = g.Cin;  // the input transform counts (slice, source channel) pairs
  prm.T = g.T;
  static const int sb_env = [] {
    const char* v = getenv("NW_STREAM_SB");
    return v ? atoi(v) : 1;
  }();
  prm.sb = (g.sync || g.sync2) ? (sb_env > 0 ? sb_env : 1) : 0;
  const uint32_t stage = (tc::kBM * prm.kbk * 2 + (uint32_t)prm.N * prm.kbk * 2) * (prm.lo ? 2 : 1);
  prm.nst = (int)((200u * 1024u) / stage);
  if (prm.nst > tc::kMaxStages) prm.nst = tc::kMaxStages;
  if (prm.nst < 2) return NW_ERR_UNSUPPORTED;
  size_t smem = 1024 + (size_t)stage * prm.nst + (2 * tc::kMaxStages + 2 * tc::kSlots + 2) * 8;
  if (smem < 120 * 1024) smem = 120 * 1024;  // one CTA per SM (a second CTA would wait for TMEM columns)
  const long long rowsV = (long long)g.P * g.T_pad * (prm.lo ? 2 : 1);
  const long long rowsU = (long long)g.P * g.cout_pad * (prm.lo ? 2 : 1);
  if (rowsV >= (1ll << 31)) return NW_ERR_UNSUPPORTED;
  alignas(64) CUtensorMap mapV, mapU;
  if (!make_map(&mapV, V, rowsV, g.cin_pad, tc::kBM, prm.kbk)) return NW_ERR_CUDA;
  if (!make_map(&mapU, U, rowsU, g.cin_pad, prm.N, prm.kbk)) return NW_ERR_CUDA;
  auto kern = prm.N == 64 ? tc::contraction_fused_kernel<3, 32> : tc::contraction_fused_kernel<3, 16>;
  if ((prm.N == 64 ? ensure_smem<tc::contraction_fused_kernel<3, 32>>(227 * 1024)
                   : ensure_smem<tc::contraction_fused_kernel<3, 16>>(227 * 1024)) != NW_OK)
    return NW_ERR_CUDA;
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long units = (long long)prm.nmb * prm.PA * prm.LO;
  if (g.gemm_ctas > 0 && g.gemm_ctas < sms) sms = g.gemm_ctas;
  const int grid = (int)(units < sms ? units : sms);
  LaunchScope scope_("contraction_tc", s);
  if (launch_pdl(kern, dim3(grid), dim3(tc::kFuseThreads), smem, s, mapV, mapU, prm) != NW_OK) return NW_ERR_CUDA;
  return check_launch();
}

}  // namespace nw
