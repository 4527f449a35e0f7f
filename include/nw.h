/*
 * nw.h -- C ABI of the B200 nested-Winograd convolution library (libnw.so).
 *
 * Implements the nested Winograd convolution of Jiang, Chen & Tsui,
 * arXiv 2102.13272 ("P:n" = line n of the paper text, PAPER.md), forward pass
 * only, for sm_100a.  A K x K filter (K <= 9, or K <= 18 at stride 2) is split
 * into 3-tap tiles; an outer F(m_o, r_o) Winograd kernel runs over the tile
 * grid and an inner F(m_i, 3) kernel inside each tile (Eq. 2.4-2.6),
 * so the convolution becomes
 *     nested input transform -> per-transform-point channel contraction ->
 *     nested output transform.
 * Stride 2 uses the stride-Winograd polyphase split (Eq. 2.7);
 * a stride-2 transposed convolution uses output phases (R11).
 *
 * Conventions (all calls):
 *  - Tensors are dense, contiguous, NCHW, caller-owned device memory, 16-byte
 *    aligned.  x [N][Cin][H][W], w [Cout][Cin][K][K] (transposed plans:
 *    [Cin][Cout][K][K], PyTorch's conv_transpose2d layout), y [N][Cout][Ho][Wo].
 *    Storage dtype is fp32 or bf16 (NW_ATTR_DTYPE); arithmetic is fp32 or the
 *    split-bf16 tensor-core scheme selected by NW_ATTR_MATH.
 *  - Cross-correlation, no filter flip, zero padding `pad` on every side
 *    (Eq. 2.1 read as in DESIGN.md#R1).
 *  - Every call returning nw_status_t never throws, never exits and never
 *    synchronises the device except nw_plan_finalize (one table upload).
 *    Kernel work is enqueued on `stream` (a cudaStream_t; NULL = legacy
 *    default stream); errors from launches are reported as NW_ERR_CUDA after
 *    cudaGetLastError, asynchronous faults surface on the next sync.
 *  - A plan is immutable after its first use (finalize) and may be shared by
 *    several threads and streams; each concurrent call brings its own
 *    workspace.
 *  - Environment tunables (performance only; results are bit-identical or within
 *    rounding order, never a different algorithm): NW_FUSE_AI=0 disables the
 *    inner output level in the contraction epilogue, 1 applies it along w only (default 2:
 *    along both axes); NW_FUSE_WIDE=0 keeps the plain contraction for layers with 128 / 256
 *    padded output channels (default: inner level along w on 128-channel CTAs / CTA pairs),
 *    NW_KBK_WIDE=16|32 narrows that kernel's K block (measured slower); NW_IN_CC=16|32|64 source
 *    channels per input-transform CTA (default 32); NW_PIPE_CHUNKS=k runs
 *    nw_conv_forward as a k-chunk three-stream pipeline (default 1) and
 *    NW_GEMM_CTAS caps its contraction grid; NW_HOST_CHUNKS=k sets the chunk
 *    count of nw_conv_forward_host (default 8; read once, at the first host-path
 *    call or workspace query, so sizes stay consistent); NW_PDL=1 launches the
 *    three hot kernels with programmatic dependent launch; NW_FUSED_C1=0 turns
 *    off the single-kernel path for one-input-channel layers, NW_FUSED_CO=0 the one for
 *    layers with at most four contraction outputs; NW_CLUSTER=1
 *    disables the CTA pairs (B multicast) of the plain contraction; NW_INPUT_TMA=0 selects
 *    the first-round input transform instead of the persistent TMA-fed kernels (the
 *    warp-specialised one, NW_ITMA_WS=0 falls back to the single-role one for bf16 x;
 *    NW_ITMA_F32=1 also fp32 x, NW_ITMA_CC=32 32 channels per task);
 *    NW_STREAM=1|2|3 runs the input transform and the contraction (1), the contraction
 *    and the output transform (2) or all three (3) at the same time on disjoint SM sets,
 *    linked by per-128-slice-block completion counters in the workspace (default 0: off;
 *    measured slower), with NW_STREAM_IT / NW_STREAM_OT CTAs for the
 *    input / output transform (default 64 / 48) and NW_STREAM_SB blocks per sweep of the
 *    contraction's point groups (default 1);
 *    NW_GEMM_G=g
 *    caps its 128-slice blocks per unit (default 16); NW_KBK=64 forces 64-wide
 *    K blocks for narrow layers (default: 16 / 32 when cin_pad is 16 / 32);
 *    NW_DEBUG_SYNC=1 synchronises after every launch and names a faulting kernel on stderr.
 */
#ifndef NW_H_
#define NW_H_

#include <stddef.h>

#if defined(NW_BUILD) && defined(__GNUC__)
#define NW_API __attribute__((visibility("default")))
#else
#define NW_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nw_plan_st *nw_plan_t;  /* opaque, owned by the library */
typedef struct CUstream_st *nw_stream_t; /* == cudaStream_t */

typedef enum {
  NW_OK = 0,
  NW_ERR_INVALID = 1,     /* bad argument (null pointer, m outside [1,6], size mismatch) */
  NW_ERR_UNSUPPORTED = 2, /* valid but not built: K > 9*stride, stride not in {1,2}, no kernel for (m_o, r_o, m_i) */
  NW_ERR_NOMEM = 3,       /* host allocation failed */
  NW_ERR_CUDA = 4,        /* a CUDA runtime / driver call or a kernel launch failed */
  NW_ERR_WORKSPACE = 5,   /* ws_bytes smaller than nw_workspace_size() */
  NW_ERR_STATE = 6        /* nw_plan_set after the plan was finalized */
} nw_status_t;

typedef enum {
  NW_MATH_FP32_SIMT = 0, /* CUDA-core FP32 pipeline: the accuracy reference */
  NW_MATH_BF16X3 = 1,    /* tcgen05 kind::f16, V=Vh+Vl, U=Uh+Ul, M = Vh.Uh + Vh.Ul + Vl.Uh (default) */
  NW_MATH_BF16 = 2       /* tcgen05 kind::f16 on Vh, Uh only: speed ceiling, fails 5e-3 (R12) */
} nw_math_t;

typedef enum { NW_DTYPE_F32 = 0, NW_DTYPE_BF16 = 1 } nw_dtype_t;

typedef enum {
  NW_ATTR_MATH = 0,           /* nw_math_t, default NW_MATH_BF16X3 */
  NW_ATTR_DTYPE = 1,          /* nw_dtype_t of x, w, y; default NW_DTYPE_F32 */
  NW_ATTR_TRANSPOSED = 2,     /* 0/1: transposed convolution (stride 2 only); default 0 */
  NW_ATTR_OUTPUT_PADDING = 3, /* transposed only; default 0 */
  NW_ATTR_OUTER_TAPS = 4,     /* r_o: 3 = paper's fixed 3x3 tile grid (default); 0 = mixed ceil(K'/3) (R8) */
  NW_ATTR_PAD = 5,            /* zero padding on every side; default K/2 */
  NW_ATTR_PRELU = 6,          /* 0/1: fuse y = y >= 0 ? y : slope[c]*y into the store (slopes via nw_plan_set_prelu) */
  NW_ATTR_DEPTHWISE = 7       /* 0/1: depthwise layer (Cin == Cout == C, w [C][1][K][K], groups = C; Table I's
                                 PNASNet row): no channel contraction, the transform-domain product
                                 is per channel; stride 1; math FP32_SIMT or BF16X3 (default 0) */
} nw_attr_t;

/* Integer tables exported for bit-exact comparison with the CPU oracle
 * (DESIGN.md "Plan tables").  Rationals are (num, den) int64 pairs in lowest
 * terms, den > 0, row-major. */
typedef enum {
  NW_TABLE_BT = 0,         /* B^T_hat  P_a x L        composite input transform (B_o^T (x) B_i^T).Gather */
  NW_TABLE_G = 1,          /* G_hat    P_a x 3*r_o    composite filter transform G_o (x) G_i */
  NW_TABLE_AT = 2,         /* A^T_hat  M_a x P_a      composite output transform A_o^T (x) A_i^T */
  NW_TABLE_GATHER = 3,     /* l_o*l_i entries: reordered-column entry (j, s) -> slice input 3j + s */
  NW_TABLE_SCATTER = 4,    /* n_phase x M_a x (position, keep): output placement + redundant-term discard */
  NW_TABLE_ORIGINS = 5,    /* [advance, n_phase, shift_0 .. shift_{n_phase-1}]: slice origins per axis */
  NW_TABLE_PHASE_TAPS = 6, /* [mode, n_phase, Kp, (offset, taps[Kp]) per phase]: stride / transposed phase split, Eq. 2.7 */
  NW_TABLE_DIMS = 7        /* [K, stride, transposed, m_o, r_o, m_i, l_o, l_i, P_a, L, M_a, P, Cin, Cout, Cin_e, Cout_e, Kp, n_phase, advance] */
} nw_table_t;

typedef struct {
  int K, stride, transposed, pad, output_padding;
  int m_outer, r_outer, m_inner;
  int points_axis;   /* P_a = l_o * l_i */
  int points;        /* P = P_a^2 transform points per slice (625 for F(3,3)(x)F(3,3)) */
  int window;        /* L = 3(l_o - 1) + l_i input window per slice axis (17) */
  int tile_out;      /* advance: distinct outputs per tile axis (9) */
  int n_phase;       /* coverage phases per axis (2 for m_i = 2, else 1) */
  int Kp;            /* per-axis taps after the stride/transposed phase split */
  int cin, cout;     /* layer channels */
  int cin_e, cout_e; /* contraction K / N after phase folding (4*Cin stride 2; 4*Cout transposed) */
  int cin_pad, cout_pad; /* cin_e / cout_e rounded up to the tensor-core granule (16) */
  int math, dtype;
  size_t filter_bytes; /* bytes of U for nw_transform_filter */
  int m_rows;          /* transform-domain rows per slice the contraction writes: points, or, with the
                          inner output level fused into its epilogue, P_a * l_o * m_i (along w only)
                          or (l_o * m_i)^2 (along both axes, the default) */
  int single_kernel;   /* 1: nw_conv_forward runs the layer as ONE kernel -- one input channel (the
                          contraction is a pointwise product) or at most four contraction outputs
                          (Cout_e <= 4: the channel sum accumulates in registers, x rows of a
                          16-byte multiple); V and M stay on chip, HBM traffic is x and y -- 0:
                          input transform, contraction, output transform */
} nw_plan_info_t;

/* Create a plan for a K x K convolution with the given stride (1 or 2) using
 * the nested F(m_outer, r_o) (x) F(m_inner, 3) algorithm.
 * Errors: NW_ERR_INVALID if out is NULL, K < 1, Cin/Cout < 1, m outside [1,6];
 * NW_ERR_UNSUPPORTED if stride not in {1,2} or the per-axis filter is longer
 * than 3*r_o.  On success *out owns host memory until nw_plan_destroy. */
NW_API nw_status_t nw_plan(int K, int stride, int m_outer, int m_inner, int Cin, int Cout, nw_plan_t *out);

/* Set an attribute before first use (NW_ERR_STATE afterwards). */
NW_API nw_status_t nw_plan_set(nw_plan_t plan, nw_attr_t attr, long long value);

/* Per-output-channel PReLU slopes (device pointer, Cout floats, caller-owned,
 * must outlive every call using the plan); used when NW_ATTR_PRELU = 1. */
NW_API nw_status_t nw_plan_set_prelu(nw_plan_t plan, const float *slopes_dev);

/* Validate the attribute set, build the transform tables and upload them to the
 * current device (synchronous, once).  Called implicitly by the first GPU call;
 * host-only queries (info, tables, sizes, counts) do not need a device. */
NW_API nw_status_t nw_plan_finalize(nw_plan_t plan);

NW_API nw_status_t nw_plan_destroy(nw_plan_t plan);

/* Geometry of the plan (host only; works without a GPU). */
NW_API nw_status_t nw_plan_info(nw_plan_t plan, nw_plan_info_t *info);

/* Copy table `which` (nw_table_t) as int64 into dst[0..cap); *n receives the
 * full length (call with cap = 0 to size).  NW_ERR_INVALID if cap < length. */
NW_API nw_status_t nw_plan_tables(nw_plan_t plan, int which, long long *dst, size_t cap, size_t *n);

/* Output spatial size for an H x W input (Eq. 2.1 / transposed definition). */
NW_API nw_status_t nw_output_size(nw_plan_t plan, int H, int W, int *Ho, int *Wo);

/* Bytes of device workspace nw_conv_forward / _ola / _direct need for a batch
 * of N images of H x W (V and M transform-domain tensors, DESIGN.md layout). */
NW_API nw_status_t nw_workspace_size(nw_plan_t plan, int N, int H, int W, size_t *bytes);
NW_API nw_status_t nw_workspace_size_ola(nw_plan_t plan, int N, int H, int W, size_t *bytes);
NW_API nw_status_t nw_workspace_size_direct(nw_plan_t plan, int N, int H, int W, size_t *bytes);

/* Nested filter transform: phase split (stride / transposed),
 * zero-pad to 3r_o x 3r_o taps, U = G_hat W G_hat^T, rounded once to the math
 * mode's storage (fp32, or bf16 hi/lo planes).  w: device, layout above;
 * U: device, info.filter_bytes, layout [P][cout_pad][cin_pad] (per plane). */
NW_API nw_status_t nw_transform_filter(nw_plan_t plan, const void *w, void *U, nw_stream_t stream);

/* Nested-Winograd forward: input transform -> contraction -> output
 * transform (+ optional PReLU) into y.  x, U, y, ws device pointers;
 * NW_ERR_WORKSPACE if ws_bytes < nw_workspace_size(plan, N, H, W). */
NW_API nw_status_t nw_conv_forward(nw_plan_t plan, const void *x, const void *U, void *y,
                            int N, int H, int W, void *ws, size_t ws_bytes, nw_stream_t stream);

/* Comparison path: single-level OLA-Winograd F(3,3) (Eq. 2.3) with the
 * ceil(K'/3)^2 block sum folded into the contraction; filter transformed from
 * raw w inside the call (into ws). */
NW_API nw_status_t nw_conv_ola(nw_plan_t plan, const void *x, const void *w, void *y,
                        int N, int H, int W, void *ws, size_t ws_bytes, nw_stream_t stream);

/* Comparison path: native convolution (Eq. 2.1) as an implicit GEMM. */
NW_API nw_status_t nw_conv_direct(nw_plan_t plan, const void *x, const void *w, void *y,
                           int N, int H, int W, void *ws, size_t ws_bytes, nw_stream_t stream);

/* End-to-end form of nw_conv_forward on HOST buffers: x_host -> device copy
 * (cudaMemcpyAsync into ws), the forward pass, y -> y_host, all enqueued on
 * `stream`.  Pinned host memory makes the copies asynchronous.  ws must hold
 * nw_workspace_size_host() bytes (forward workspace + device x and y). */
NW_API nw_status_t nw_workspace_size_host(nw_plan_t plan, int N, int H, int W, size_t *bytes);
NW_API nw_status_t nw_conv_forward_host(nw_plan_t plan, const void *x_host, const void *U, void *y_host,
                                        int N, int H, int W, void *ws, size_t ws_bytes, nw_stream_t stream);

/* Per-kernel timing for the benchmark's roofline: between nw_profile_begin()
 * and nw_profile_end() every library launch is bracketed by CUDA events on its
 * stream.  nw_profile_end synchronises those events and writes, for up to
 * `cap` kernel kinds, the kind name (static string), launch count and total
 * milliseconds; *n receives the number of kinds.  Not thread-safe. */
NW_API nw_status_t nw_profile_begin(void);
NW_API nw_status_t nw_profile_end(const char **names, unsigned long long *launches, double *ms,
                                  size_t cap, size_t *n);

/* Decomposition algorithm of section IV.B, host only: the expression tree
 * of F(M, R; S) over one base kernel F(m, r) -- stride Winograd split (Eq. 2.7) while
 * S > 1, nested Winograd (III.A) while R > r, output lengths matched with
 * F(n.m, r) = n.F(m, r) -- written as its reverse-Polish token stream, NUL-terminated,
 * into rpn[0..cap) (tokens K<m>,<r> NEST<d> REP<n> SUM<k>; Eq. 4.1 is
 * "K2,2 NEST2 K2,2 REP2 SUM2"); *len receives the string length, *M the resolved output
 * length per tile.  rpn may be NULL (size query).  Errors: NW_ERR_INVALID for arguments
 * < 1 (or absurdly large) or cap too small; NW_ERR_UNSUPPORTED when nesting would need
 * m < r (holes, R6).  The GPU kernels execute the two-level plans with r = 3
 * taps and stride <= 2; deeper or stride-3 plans are planned, not executed. */
NW_API nw_status_t nw_decompose(int R, int S, int m, int r, char *rpn, size_t cap, size_t *len, int *M);

/* EWMM multiplications of one nested forward (slices * P * Cin_e * Cout_e). */
NW_API nw_status_t nw_count_mults(nw_plan_t plan, int N, int H, int W, unsigned long long *ewmm);

/* Number of kernels the library launched since load (host counter; for the
 * bench's gpu_launches claim). */
NW_API unsigned long long nw_launch_count(void);

NW_API const char *nw_status_str(nw_status_t status);

#ifdef __cplusplus
}
#endif
#endif /* NW_H_ */
