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

/* Dense entry block K[rows[a], cols[b]] -> out (nr, nc) complex128 on the
 * device; rows/cols are device int64 arrays. Replaces FioKernel.block
 * (kernels.py:34-38) via BlockView (oracles.py:66-68). */
int bf_entries(int kernel_id, uint64_t n, const int64_t* rows, uint32_t nr,
               const int64_t* cols, uint32_t nc, void* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BFLY_H_ */
