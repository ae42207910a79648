/*
 * bfly.h — C ABI of libbfly.so, the B200 (sm_100a) butterfly-factorization
 * hot path. Plain pointers and sizes only; no torch or C++ types.
 *
 * The reference (arxiv/paper_1502_01379, package `butterfly`, pure NumPy)
 * has no native boundary; every entry point here replaces one NumPy call
 * site of the reference, cited as pkg/src/butterfly/<file>:<line>.
 *
 * Conventions
 *  - Complex data is interleaved (re, im): complex128 = 2 x f64, complex64 =
 *    2 x f32. Factor arrays use the reference layout exactly
 *    (factors.py:23-203): leaf (nb, n0, r); transfer (G, 2, P, r, 2r) at
 *    splitting levels and (G, P, r, 2r) at merge-only levels; middle
 *    weights (m, m, r) f64. All row-major (C order).
 *  - Vectors are (N, k) row-major: RHS index fastest, as the reference's
 *    `g.reshape(n, -1)` (factors.py:222).
 *  - Every call returns BF_OK (0) or an error code; bf_last_error() returns
 *    the thread-local message. BF_EINVAL maps to Python ValueError,
 *    BF_EORACLE to OracleError (oracles.py:18-19), others to RuntimeError.
 *  - Device work is stream-ordered on the `stream` argument (a
 *    cudaStream_t passed as void*; NULL = legacy default stream). Nothing
 *    synchronises the device except bf_apply_host (it must return host data).
 *  - A plan is immutable after bf_plan_upload; concurrent bf_apply calls on
 *    one plan are safe with distinct out/workspace buffers.
 */
#ifndef BFLY_H_
#define BFLY_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BF_OK 0
#define BF_EINVAL 1
#define BF_ECUDA 2
#define BF_ENOMEM 3
#define BF_EORACLE 4
#define BF_ESTATE 5
#define BF_EFORMAT 6 /* malformed .bfac file: Python FormatError (storage.py:40-45) */

#define BF_C128 0 /* complex128 factors + vectors (the reference's dtype, factors.py:222) */
#define BF_C64 1  /* opt-in complex64 mode (fp32 arithmetic) */

/* factor selectors for bf_apply_factor (reference classes in factors.py) */
#define BF_FACTOR_V 0 /* right leaf V^L   BlockDiagonalFactor (factors.py:23-56)  */
#define BF_FACTOR_H 1 /* right transfer   TransferFactor      (factors.py:59-142) */
#define BF_FACTOR_M 2 /* middle           MiddleFactor        (factors.py:145-190) */
#define BF_FACTOR_G 3 /* left transfer    TransferFactor                           */
#define BF_FACTOR_U 4 /* left leaf U^L    BlockDiagonalFactor                      */

/* entry-oracle kernels for bf_entries (kernels.py:23-42; config-1 DFT) */
#define BF_KERNEL_FIO 0  /* exp(2 pi i (x xi + c(x)|xi|)), x=i/N, xi=j-N/2 (kernels.py:27-38) */
#define BF_KERNEL_DFTP 1 /* exp(+2 pi i (j k mod N)/N) — BASELINE config 1                   */
#define BF_KERNEL_DENSE 2 /* explicit n x n complex128 matrix on the device (DenseOracle)    */
#define BF_KERNEL_RADON2D 3 /* 2-D generalized Radon, n = n_side^2 Morton indices (cfg 3/4b)   */
#define BF_KERNEL_DFT 4   /* the reference's centered DftKernel exp(-2 pi i (j - N/2) k / N) (kernels.py:87-97) */
#define BF_KERNEL_TILES 5 /* per-middle-block windows of any entry oracle (bf_middle_blocks_tiled) */

typedef struct bf_plan bf_plan;

int bf_version(void);
/* Copy the calling thread's last error message (NUL-terminated, truncated). */
int bf_last_error(char* buf, size_t len);

/* Geometry of DyadicPartition(n, levels) (partition.py:18-70) with rank r,
 * mirroring construct.py:_level_geometry (216-227). max_rhs is a hint only.
 * dtype: BF_C128 or BF_C64. device: CUDA ordinal. */
int bf_plan_create(bf_plan** out, uint64_t n, uint32_t levels, uint32_t rank,
                   uint32_t max_rhs, int dtype, int device);
void bf_plan_destroy(bf_plan* plan);

/* Number of transfer levels per side (= levels - levels/2) and, per level
 * index i in [0, nlev) ascending from half, the block-array shape:
 * dims[i*5 .. i*5+4] = (G, 2, P, r, 2r) when splits[i]=1 else (G, P, r, 2r, 0).
 * leaf[3] = (nb, n0, r). Any output pointer may be NULL. */
int bf_plan_geometry(const bf_plan* plan, uint32_t* nlev, int8_t* splits,
                     uint64_t* dims, uint64_t* leaf);

/* Copy complex128 factors (host or device pointers; cudaMemcpyDefault) into
 * the plan, converting to the plan dtype. g_levels/h_levels are arrays of
 * nlev pointers ascending from level half (ButterflyFactors.g_chain/h_chain
 * order, factors.py:200-202). Replaces holding the NumPy arrays of
 * ButterflyFactors (factors.py:193-203). */
int bf_plan_upload(bf_plan* plan, const void* u_leaf, const void* const* g_levels,
                   const double* weights, const void* const* h_levels,
                   const void* v_leaf);

/* Bytes of device workspace bf_apply needs for k right-hand sides. */
uint64_t bf_apply_workspace_bytes(const bf_plan* plan, uint32_t k);

/* out = K in (adjoint=0) or K* in (adjoint=1); in/out device (N, k) in the
 * plan dtype. Replaces ButterflyFactors.apply / apply_adjoint
 * (factors.py:209-237). in and out may not alias the workspace. */
int bf_apply(const bf_plan* plan, const void* in, void* out, uint32_t k, int adjoint,
             void* workspace, uint64_t workspace_bytes, void* stream);

/* Same with HOST in/out buffers (pinned for full PCIe speed): H2D copy,
 * apply, D2H copy, stream synchronise. Allocates its own workspace. */
int bf_apply_host(const bf_plan* plan, const void* in_host, void* out_host, uint32_t k,
                  int adjoint, void* stream);

/* One factor of the chain, for per-level parity: which = BF_FACTOR_*;
 * level = transfer level (ignored for V, M, U); adjoint selects
 * forward/adjoint of that factor as in factors.py:49-56, 120-142, 180-190.
 * in/out are device (dim, k) arrays of the plan dtype. */
int bf_apply_factor(const bf_plan* plan, int which, uint32_t level, int adjoint,
                    const void* in, void* out, uint32_t k, void* stream);

/* Per-launch device timing of the apply chain (CUDA events recorded on the
 * launching stream around every kernel). A timer holds max_steps x
 * max_launches event pairs; bf_apply_timed is bf_apply recording into the
 * next step slot; bf_timer_read synchronises on the last event and returns
 * launch_ms[step * launches + i] plus the counts. For roofline reporting. */
typedef struct bf_timer bf_timer;
int bf_timer_create(bf_timer** out, uint32_t max_steps, uint32_t max_launches);
void bf_timer_destroy(bf_timer* timer);
int bf_apply_timed(const bf_plan* plan, const void* in, void* out, uint32_t k, int adjoint,
                   void* workspace, uint64_t workspace_bytes, void* stream, bf_timer* timer);
int bf_timer_read(bf_timer* timer, float* launch_ms, uint32_t* steps, uint32_t* launches);

/* ---------------------------------------------------------------------------
 * Sharded apply across GPUs. Part `part` of `nparts`
 * (nparts divides m = 2^(levels/2)) owns middle column nodes J and row nodes I
 * = [part*m/nparts, (part+1)*m/nparts): the V^L/H slices feeding J and the
 * G/U^L slices fed by I. bf_plan_upload then takes this part's slices in the
 * reference layout: leaf blocks [part*nb/P, (part+1)*nb/P) and transfer groups
 * [part*G/P, (part+1)*G/P) of every level (the leading block index carries
 * the middle node), plus the full (m, m, r) weights. Forward apply of K:
 *   bf_apply_down(in rows [part*n/P, ...)) -> mid ((m/P)*m*r, k)
 *   bf_middle_pack(mid) -> send (P, (m/P)^2 r, k), scaled by M's weights
 *   all-to-all of equal chunks (NCCL) -> recv
 *   bf_middle_unpack(recv) -> mid' ; bf_apply_up(mid') -> out rows [part*n/P, ...)
 * adjoint = 1 runs K* the same way (U*, G* down; H, V up). */
int bf_plan_create_sharded(bf_plan** out, uint64_t n, uint32_t levels, uint32_t rank, int dtype, int device,
                           uint32_t part, uint32_t nparts);
/* General tree: branching 2 (the reference's binary trees) or 4 (quadtrees
 * over Morton-ordered 2-D grids, BASELINE configs 3/4b; transfer blocks
 * (G, 4, P, r, 4r)); nparts = 1 for an unsharded plan. */
int bf_plan_create_tree(bf_plan** out, uint64_t n, uint32_t levels, uint32_t rank, uint32_t branching,
                        int dtype, int device, uint32_t part, uint32_t nparts);
int bf_apply_down(const bf_plan* plan, const void* in, void* mid, uint32_t k, int adjoint,
                  void* workspace, uint64_t workspace_bytes, void* stream);
/* Fused variant of bf_apply_down + bf_middle_pack + all-to-all: the last
 * level's epilogue applies the middle weights and stores every output straight
 * into the receive buffer of the part that owns it — peers[d] is part d's
 * receive buffer (P, (m/P)^2 r, k), mapped into this process (CUDA IPC /
 * symmetric memory over NVLink; plain device buffers when the parts share one
 * GPU). After every part's push has completed (a cross-part barrier), each part
 * runs bf_middle_unpack on its own receive buffer. */
int bf_apply_down_push(const bf_plan* plan, const void* in, void* const* peers, uint32_t k, int adjoint,
                       void* workspace, uint64_t workspace_bytes, void* stream);
int bf_middle_pack(const bf_plan* plan, const void* mid, void* send, uint32_t k, int adjoint, void* stream);
int bf_middle_unpack(const bf_plan* plan, const void* recv, void* mid, uint32_t k, int adjoint, void* stream);
int bf_apply_up(const bf_plan* plan, const void* mid, void* out, uint32_t k, int adjoint,
                void* workspace, uint64_t workspace_bytes, void* stream);

/* The reference's .bfac factor file (storage.py:1-186) straight to/from a
 * device plan: records stream through a pinned buffer; one kernel per chunk
 * checks every block header against the geometry (mismatch -> BF_EFORMAT,
 * message carries the byte offset) and transposes the column-major payloads
 * into the plan layout. save -> load -> save is byte-identical
 * (save_factors/load_factors, storage.py:79-167). bf_plan_export copies one
 * factor array (reference layout, plan dtype) to dst. */
int bf_plan_load_bfac(bf_plan** out, const char* path, int dtype, int device);
int bf_plan_save_bfac(const bf_plan* plan, const char* path);
int bf_plan_export(const bf_plan* plan, int which, uint32_t level, void* dst, uint64_t dst_bytes, void* stream);

/* Dense entry block K[rows[a], cols[b]] -> out (nr, nc) complex128 on the
 * device; rows/cols are device int64 arrays. Replaces FioKernel.block
 * (kernels.py:34-38) via BlockView (oracles.py:66-68). */
int bf_entries(int kernel_id, uint64_t n, const int64_t* rows, uint32_t nr,
               const int64_t* cols, uint32_t nc, void* out, void* stream);

/* The per-N table of row-only transcendental terms the FIO and 2-D Radon entries read:
 * FIO c(x_i) = (2 + sin 2 pi x_i)/8 for i < n (n doubles); 2-D sin and cos of 2 pi a/n_side
 * for a < n_side (2 n_side doubles: sines then cosines). Sines are correctly rounded
 * (double-double), hence equal to the reference's NumPy values. out: device, len doubles. */
int bf_entry_table(int kernel_id, uint64_t n, double* out, uint64_t len, void* stream);

/* Hankel-kernel rows (HankelKernel, kernels.py:45-84; hankel1_orders,
 * bessel.py:178-230): out[t, m] = H1_m(x[t]) = J_m + i Y_m for m = 0..max_order,
 * complex128 rows of stride ld. x: device float64 (nx), all > 0. start: the
 * backward-recurrence start the reference computes for this batch,
 * int(max(x + 10 cbrt(x) + 40)) but at least max_order + 15 (host-computed, so
 * the J sweep is bit-identical to the reference's). Synchronises `stream` (it
 * reports invalid x). */
int bf_hankel_orders(const double* x, uint32_t nx, uint32_t max_order, int64_t start, void* out, uint64_t ld,
                     void* stream);

/* ---------------------------------------------------------------------------
 * Sampling construction (construct.py:43-68, lowrank.py:219-258, construct.py:127-163).
 *
 * bf_middle_blocks: randomized sampling SVD of `nblocks` middle-level blocks
 * of DyadicPartition(n, levels) with rank r and OversamplingParams (q, iters)
 * — one CTA per block. block_ij: device int32 (nblocks, 2) block coordinates
 * (i, j); draws: device int32 (nblocks, 2*(iters+1), min(r*q, side)) — the
 * rng.choice draws of block_rng(seed, 0, i, j) in consumption order (row,
 * col, row, col, ...; lowrank.py:237-251), made on the host with the
 * reference's generator; unused (may be NULL) when r*q >= side (dense
 * branch). dense: device n x n complex128 for BF_KERNEL_DENSE, else NULL.
 * Outputs (device): u_out, v_out (nblocks, side, r) complex128 = u0*sigma0,
 * v0*sigma0; w_out (nblocks, r) f64 = floored_inverse(sigma0) — exactly what
 * construct.py:63-65 scatters into U^h, V^h and M. branching 2 (binary tree)
 * or 4 (quadtree, middle blocks = contiguous Morton ranges). Requires
 * r*(q+1) <= 128 (shared-memory small matrices up to 64, global above).
 */
uint64_t bf_middle_workspace_bytes(uint64_t n, uint32_t levels, uint32_t branching, uint32_t rank,
                                   uint32_t q_over, uint32_t nblocks);
int bf_middle_blocks(int kernel_id, uint64_t n, uint32_t levels, uint32_t branching, uint32_t rank,
                     uint32_t q_over, uint32_t iters, const void* dense, uint32_t nblocks, const int32_t* block_ij,
                     const int32_t* draws, void* u_out, void* v_out, double* w_out,
                     void* workspace, uint64_t ws_bytes, void* stream);

/* Roofline denominators measured in the caller's process (bench.py): out[0] FP64 tensor
 * pipe TF/s (mma.sync m8n8k4), out[1] FP64 FMA TF/s, out[2] streaming-read GB/s, out[3]
 * copy GB/s (read + write bytes) over `scratch` (device, >= 1 GiB, larger than L2). */
int bf_measure_peaks(double* out, void* scratch, uint64_t scratch_bytes, void* stream);  /* scratch: 4 GiB+ */

/* Diagnostics: node kernels (one launch per chain half) stamp %globaltimer per CTA into
 * dev_buf (u64, >= 2 x m x chunks x 32; NULL turns it off). Not thread-safe; tools only. */
int bf_debug_node_trace(unsigned long long* dev_buf);

/* bf_middle_blocks for any entry oracle (the BlockView protocol, oracles.py:57-68):
 * the caller evaluates each block's side x side window K[i side + a, j side + b]
 * (host oracle.block(), or a device producer) and passes the windows stacked as
 * tiles (ntiles, side, side) complex128 row-major on the device, with slot
 * (m, m) int32 on the device giving block (i, j)'s tile index (-1 for blocks not
 * in this call). Every entry a middle block's sampling SVD reads lies in its
 * window, so the results are those of bf_middle_blocks on the dense matrix. */
int bf_middle_blocks_tiled(uint64_t n, uint32_t levels, uint32_t branching, uint32_t rank, uint32_t q_over,
                           uint32_t iters, const void* tiles, const int32_t* slot, uint32_t nblocks,
                           const int32_t* block_ij, const int32_t* draws, void* u_out, void* v_out, double* w_out,
                           void* workspace, uint64_t ws_bytes, void* stream);

/* Matvec-mode middle level (middle_factorization_matvec, construct.py:89-124;
 * per block svd_from_probes, lowrank.py:204-216): the rank-r SVD of `nblocks`
 * middle blocks finished from stored probe products only. All device,
 * complex128 row-major:
 *   k_cols (n x ldc) = K @ col_probe; block (i, j) reads rows [i side, (i+1) side),
 *          columns [j width, (j+1) width)           (y_col = Z C)
 *   k_rows (n x ldr) = K^H @ row_probe; block (i, j) reads rows [j side, ...),
 *          columns [i width, ...)                    (y_row = Z* R)
 *   row_probe (m, side, width): the diagonal blocks of the row probe (R).
 * Per block: greedy pivots of y_col / y_row (k = width, rel_tol 0), the
 * orthonormal bases of the pivot columns padded with canonical columns
 * (orthonormal_columns, lowrank.py:132-154), mid = pinv_floored(R* Q_col)
 * (y_row* Q_row), its SVD truncated to r (_assemble, lowrank.py:284-293).
 * Outputs as bf_middle_blocks. Requires r <= width <= min(side, 128). */
uint64_t bf_probe_workspace_bytes(uint64_t n, uint32_t levels, uint32_t branching, uint32_t rank, uint32_t width,
                                  uint32_t nblocks);
int bf_middle_probes(uint64_t n, uint32_t levels, uint32_t branching, uint32_t rank, uint32_t width,
                     uint32_t nblocks, const int32_t* block_ij, const void* k_cols, uint64_t ldc,
                     const void* k_rows, uint64_t ldr, const void* row_probe, void* u_out, void* v_out,
                     double* w_out, void* workspace, uint64_t ws_bytes, void* stream);

/* One level of _recurse (construct.py:127-163) with branching b (2; 4 on
 * quadtrees): cur (nb, rows, groups, r) complex128 -> transfer blocks
 * (nb, b, groups/b, r, b r) when rows >= b (SVD of each (rows/b x b r) stack;
 * keep = min(r, rows/b)) or (nb, groups/b, r, b r) when rows < b, and the next
 * cur (b nb, rows/b, groups/b, r) or (nb, 1, groups/b, r). With workspace ==
 * NULL, *ws_bytes receives the scratch size. Requires b r <= 128. */
int bf_recurse_level(uint32_t rank, uint32_t branching, uint64_t nb, uint64_t rows, uint64_t groups,
                     const void* cur, void* blocks, void* next, void* workspace, uint64_t* ws_bytes,
                     void* stream);

/* Direct sampled-row sums y = K[rows, :] g (rows: device int64 (nr); g, y:
 * device complex128 (n, k) and (nr, k)) with entries evaluated on the fly:
 * the ground truth of the reference's accuracy metric eps_a
 * (RowSampledReference.rows, bench.py:44-46; estimate_eps_a_info 90-97).
 * Deterministic (fixed-order partial sums in a workspace of
 * bf_sampled_rows_workspace(n, nr, k) bytes). */
uint64_t bf_sampled_rows_workspace(uint64_t n, uint32_t nr, uint32_t k);
int bf_sampled_rows(int kernel_id, uint64_t n, const void* dense, const int64_t* rows, uint32_t nr,
                    const void* g, uint32_t k, void* out, void* workspace, uint64_t ws_bytes, void* stream);

/* Greedy pivoted column selection (select_pivot_columns, lowrank.py:102-129)
 * on a batch of device matrices a (batch, m, n) complex128 row-major with
 * m <= 64: up to k picks each, in pick order, into pivots (batch, k) and pick
 * counts into counts (batch); rel_tol as the reference's. pairwise = 1 sums
 * the initial column norms in numpy's pairwise order (the reference matrix is
 * F-ordered), 0 sequentially (C-ordered). Workspace >= 16*batch*min(k,m)*n bytes. */
int bf_select_pivots(const void* a, uint32_t batch, uint32_t m, uint32_t n, uint32_t k, double rel_tol,
                     int pairwise, int32_t* pivots, int32_t* counts, void* workspace,
                     uint64_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BFLY_H_ */
