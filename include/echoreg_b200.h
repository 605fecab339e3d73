/*
 * echoreg_b200.h -- C ABI of the B200 (sm_100a) SMC rigid-registration path.
 *
 * Drop-in boundary for the reference's kernel-module seam
 * (/root/reference/pkg/src/echoreg/backend.py:33-108 selects a module that
 * exports NAME, ncc_measure_batch, resample_trilinear, warm_up --
 * kernels_numba.py:22,192-233).  Plain pointers and sizes only: every
 * pointer named *_dev is DEVICE memory owned by the caller, every `stream`
 * is a cudaStream_t passed as void*.  All functions are asynchronous on
 * `stream` unless stated and return 0 on success or an ER_E* code; the text
 * of the last error is available from er_last_error().
 *
 * Volumes are C-order (nx, ny, nz) with k (z) fastest, the reference's
 * in-memory layout (volume.py:33).  A volume may be stored as u8 / f32 /
 * f64; the value the algorithm sees is  alpha * stored + gamma  (alpha = 1,
 * gamma = 0 for a verbatim copy; raw uint8 echo data with the z-score of
 * volume.py:119-130 folded in otherwise).
 */
#ifndef ECHOREG_B200_H
#define ECHOREG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ER_OK 0
#define ER_EINVAL 1     /* bad argument (maps to echoreg BadConfig / ValueError) */
#define ER_ECUDA 2      /* CUDA runtime error (maps to echoreg InternalError) */
#define ER_EWEIGHTS 3   /* weights failed to normalise (smc.py:139-142 check) */

#define ER_U8 0
#define ER_F32 1
#define ER_F64 2

/* Interpolation arithmetic of the measurement kernel. */
#define ER_LERP_F32 0      /* fp32 lerps on fp64 coordinates/fractions      */
#define ER_LERP_F64 1      /* fp64 lerps (FMA), fp64 everywhere             */
#define ER_LERP_EXACT 2    /* fp64 lerps in the reference's a(1-f)+bf order */
#define ER_LERP_NEAREST 3  /* nearest voxel, ties to the upper one: the north
                              star's option for binary masks (opt-in; the
                              reference itself samples masks trilinearly) */

typedef struct er_volume {
  const void *data_dev; /* device pointer */
  int32_t dtype;        /* ER_U8 / ER_F32 / ER_F64 */
  int32_t nx, ny, nz;
  double alpha, gamma;  /* value = alpha * stored + gamma */
  const void *oct_dev;  /* optional er_build_oct() re-layout of a u8 volume, or NULL */
  const void *bitoct_dev; /* optional er_build_bitoct() re-layout of a binary volume */
  const void *quad_dev;   /* optional er_build_quad() re-layout of an f32/f64 volume */
} er_volume;

int er_abi_version(void);
const char *er_last_error(void);

/* Debug builds only (-DER_BOUNDS_CHECK=1): number of out-of-range gather
 * indices the kernels have seen since load (each counted and clamped to 0).
 * Returns ER_EINVAL, *count = 0, on a normal build.  No reference
 * counterpart: this replaces compute-sanitizer memcheck, which the GPU pool
 * does not allow. */
int er_debug_bounds_faults(unsigned long long *count);

/* Measurement infrastructure (no reference counterpart): one launch reading
 * the first `bytes` of buf_dev `reps` times with 8-byte lane loads through L2
 * (every SM, 4 loads in flight per thread).  Timed by the caller with events
 * on `stream`; bench.py uses it for the live L2 roofline denominator.
 * sink_dev: 4 bytes of device scratch. */
int er_probe_read(const void *buf_dev, int64_t bytes, int32_t reps, void *sink_dev,
                  void *stream);

/* ---- volumes ---------------------------------------------------------- */

/* Stored-value moments: out_dev[0] = sum(stored), out_dev[1] = sum(stored^2),
 * deterministic fixed-order fp64 reduction.  Feeds the full-region target
 * totals of kernels_numba.py:123-130.  out_dev must hold ER_MOMENTS_DOUBLES
 * doubles (the tail is reduction scratch). */
#define ER_MOMENTS_DOUBLES 1026
int er_volume_moments(const er_volume *v, double *out_dev, void *stream);

/* Oct re-layout of a u8 volume for the measurement fast path: padded cell
 * (ci, cj, ck) holds the 8 trilinear corners of floor cell (ci-1, cj-1, ck-1),
 * clamped into the grid, as one 8-byte word.  er_oct_bytes() = (nx+1)(ny+1)
 * (nz+1) * 8.  Set er_volume.oct_dev to the result to enable the fast path
 * (used for lerp modes F32/F64; LERP_EXACT always gathers the plain copy). */
size_t er_oct_bytes(const er_volume *v);
int er_build_oct(const er_volume *v, void *oct_dev, void *stream);

/* Bit-oct re-layout of a BINARY u8 volume (values 0/1): the same padded
 * cells with the 8 corners as the 8 bits of one byte (bit b = byte b of the
 * oct word).  (nx+1)(ny+1)(nz+1) bytes.  Set er_volume.bitoct_dev to enable
 * the mask fast path (1-byte gathers; uniform cells skip the lerps). */
size_t er_bitoct_bytes(const er_volume *v);
int er_build_bitoct(const er_volume *v, void *bitoct_dev, void *stream);

/* Quad re-layout of an f32- or f64-stored volume for the fp32-lerp fast path:
 * column (ci, cj) of the padded grid, ci in [0, nx], cj in [0, ny], holds
 * nz + 2 float4 entries, entry m = the 4 corners (x[i0][j0], x[i0][j1],
 * x[i1][j0], x[i1][j1]) of plane clamp(m - 1) with i0 = clamp(ci - 1),
 * i1 = clamp(ci) (likewise j): the sample of padded cell (ci, cj, ck) reads
 * entries ck and ck + 1 (two adjacent 16-byte loads).  f64 values are
 * rounded to fp32.  er_quad_bytes() = (nx+1)(ny+1)(nz+2) * 16.  Set
 * er_volume.quad_dev to use it in ER_LERP_F32 (with the fp64 refinement of
 * ill-conditioned particles, as for the 8-bit path). */
size_t er_quad_bytes(const er_volume *v);
int er_build_quad(const er_volume *v, void *quad_dev, void *stream);

/* 256-bin histogram of a u8 volume (exact int64 counts, order-free integer
 * atomics): the z-score of volume.py:119-130 on 8-bit data is computed from
 * it (exact integer sums -> numpy-identical mean).  hist_dev: 256 int64. */
int er_histogram_u8(const er_volume *v, int64_t *hist_dev, void *stream);

/* Ingest of an 8-bit NIfTI payload (E/io.py:124-187, the reader's
 * reshape(order="F") at io.py:165-171): payload_dev holds frames x nz x ny x
 * nx bytes as on disk (x fastest, frame slowest); out_dev receives the frames
 * in the reference's memory order (each (nx, ny, nz) C order, z fastest),
 * frame f at out_dev + f*nx*ny*nz.  hist_dev (frames x 256 int64, or NULL)
 * receives each frame's exact 256-bin histogram, from which the z-score of
 * volume.py:119-130 is computed (same counts as er_histogram_u8).  One launch
 * (plus a zeroing launch when hist_dev is set).  frames <= 65535. */
int er_ingest_u8(const uint8_t *payload_dev, int64_t nx, int64_t ny, int64_t nz, int64_t frames,
                 uint8_t *out_dev, int64_t *hist_dev, void *stream);

/* Classify an f64 device volume: flags_dev[0] = 1 if every voxel is 0 or 1
 * (volume.py:138-140), flags_dev[1] = 1 if every voxel is exactly
 * representable in fp32.  Used to pick a lossless storage type. */
int er_classify_f64(const double *data_dev, int64_t n, int32_t *flags_dev, void *stream);

/* out2_dev[0] = min, out2_dev[1] = max of an f64 array (NaN-free), exact. */
int er_minmax_f64(const double *data_dev, int64_t n, double *out2_dev, void *stream);

/* Recover 8-bit data behind an affine image (e.g. the reference's z-score of
 * 8-bit echo data, volume.py:119-130, which reaches the kernel-module seam as
 * plain fp64): out_dev[i] = rint((x_i - x0) / delta); flag_dev[0] (int32)
 * stays 1 iff every byte is in 0..255 and |x_i - (x0 + k_i delta)| <= tol.
 * The volume can then be measured as u8 storage with alpha = delta,
 * gamma = x0 (the oct fast path) -- values reproduced to <= tol. */
int er_lattice_u8(const double *data_dev, int64_t n, double x0, double delta, double tol,
                  uint8_t *out_dev, int32_t *flag_dev, void *stream);

/* Convert an f64 volume to u8 (values must be integers 0..255) or f32. */
int er_convert_f64(const double *data_dev, int64_t n, int32_t dst_dtype, void *dst_dev,
                   void *stream);

/* ---- the hot path: fused pull-back trilinear resample + squared NCC ---- */
/* Replaces kernels_numba.ncc_measure_batch / _ncc_kernel
 * (kernels_numba.py:116-189, 203-223) and is what Executor.measure_ncc
 * (backend.py:78-108) dispatches to.  A_dev: P x 9 (row-major 3x3 index
 * affine, geometry.index_affine), b_dev: P x 3.  tgt_moments_dev: the
 * er_volume_moments() of the target.  Outputs: squared NCC (f64), the
 * degenerate flag, and the exact in-bounds voxel count per particle.
 * In ER_LERP_F32 on a non-binary source, particles whose fp32 samples
 * cannot resolve the likelihood to 1e-4 relative (or the degenerate test)
 * -- ill-conditioned, nearly decorrelated or nearly constant overlaps -- are
 * re-measured on the device in ER_LERP_EXACT arithmetic before return (no
 * host round trip; the workspace holds the list).  The workspace is
 * P x tiles x 48 B of partials + 16 B + 4 B per particle. */
size_t er_measure_workspace_bytes(const er_volume *tgt, int64_t P);
int er_measure_ncc(const er_volume *tgt, const er_volume *src, const double *tgt_moments_dev,
                   const double *A_dev, const double *b_dev, int64_t P, int32_t overlap_only,
                   int32_t lerp_mode, double *ncc_dev, uint8_t *degen_dev, int64_t *n_in_dev,
                   void *workspace_dev, size_t workspace_bytes, void *stream);

/* ---- SMC particle machinery (smc.py:145-259), all on device ------------ */

/* init_particles (smc.py:145-157): states_dev[N x 6] ~ uniform(-lim, lim)
 * from stream (seed, 0, 0, 0), bit-exact with numpy. */
int er_smc_init(double *states_dev, int64_t n, uint64_t seed, const double lim[6],
                void *stream);

/* predict (smc.py:160-174): out = clip(in + sigma * N(0,1)_{(seed,1,k,i)},
 * -clip, clip) for particles i in [0, n).  sigma/clip computed by the host
 * exactly as the reference does. */
int er_smc_predict(const double *states_in_dev, double *states_out_dev, int64_t n,
                   uint64_t seed, int64_t k, const double sigma[6], const double clip[6],
                   void *stream);

/* er_smc_predict fused with er_states_to_affine for this rank's shard
 * [first, first + count) of the predicted states: one launch per iteration
 * instead of two; identical outputs. */
int er_smc_predict_affine(const double *states_in_dev, double *states_out_dev, int64_t n,
                          uint64_t seed, int64_t k, const double sigma[6], const double clip[6],
                          int64_t first, int64_t count, const double center[3],
                          const double tgt_spacing[3], const double tgt_origin[3],
                          const double src_spacing[3], const double src_origin[3],
                          double *A_dev, double *b_dev, void *stream);

/* to_matrix about `center` (geometry.py:87-99) + index_affine
 * (geometry.py:136-152) for states [first, first + count). */
int er_states_to_affine(const double *states_dev, int64_t first, int64_t count,
                        const double center[3], const double tgt_spacing[3],
                        const double tgt_origin[3], const double src_spacing[3],
                        const double src_origin[3], double *A_dev, double *b_dev,
                        void *stream);

/* Exhaustive grid nodes [first, first + count) of a GridSpec
 * (exhaustive.py:25-75, lexicographic, last axis fastest) straight to
 * index affines.  axis_step[6] in internal units (radians, mm). */
int er_grid_to_affine(int64_t first, int64_t count, const int32_t half_counts[6],
                      const double axis_step[6], const double center[3],
                      const double tgt_spacing[3], const double tgt_origin[3],
                      const double src_spacing[3], const double src_origin[3],
                      double *states_dev, double *A_dev, double *b_dev, void *stream);

/* First-max argmax over z_dev[0..n) folded into a running best with a strict
 * '>' (exhaustive.py:106-109): best_dev = {value, index}, both stored as f64 (the index
 * as its numeric value, exact below 2^53). */
int er_argmax_update(const double *z_dev, int64_t n, int64_t base_index, double *best_dev,
                     void *stream);

/* One SMC update after measurement: best tracking (smc.py:203-206),
 * update_weights (210-224), ess (227-229), resample_systematic with stream
 * (seed, 2, k, 0) when ess < ess_fraction * n (232-248, 353-357), estimate
 * (251-259) and the trace row (358-364).  No host round trip: one CTA for
 * n < 16384, else a chain of whole-GPU kernels with the same per-chunk loops
 * and reduction trees (bit-identical results).  ctl_dev layout: see
 * er_smc_ctl below.  weights_dev is updated in place; states_out/z_out
 * receive the (possibly resampled) population; z_out, states_out and
 * scratch must not alias the inputs (z_out and scratch also serve as the
 * large-n path's reduction scratch). */
typedef struct er_smc_ctl {
  double best_measurement; /* running best (init -1.0) */
  double best_state[6];
  int32_t has_best;
  int32_t error;           /* ER_EWEIGHTS when |sum w - 1| > 1e-9 */
} er_smc_ctl;

#define ER_TRACE_STRIDE 12 /* estimate[6], mean, max, best, ess, fired, n_degenerate */

int er_smc_update(const double *z_dev, const uint8_t *degen_dev, double *weights_dev,
                  const double *states_in_dev, double *states_out_dev, double *z_out_dev,
                  double *scratch_dev /* n doubles: cumulative weights */, int64_t n, double beta, double ess_fraction, uint64_t seed, int64_t k,
                  int32_t estimate_best, er_smc_ctl *ctl_dev, double *trace_row_dev,
                  void *stream);

/* er_smc_update reading the result of the ONE all-gather per iteration of a
 * particle-sharded run: zd_dev holds world blocks of
 * block_bytes, rank r's block = [z: shard f64 | degenerate flags: shard u8 |
 * pad to 8 B]; particle i = r * shard + j.  Identical outputs to
 * er_smc_update on the unpacked arrays.  block_bytes >= 9 * shard, % 8 == 0. */
int er_smc_update_gathered(const void *zd_dev, int64_t shard, int64_t block_bytes,
                           double *weights_dev, const double *states_in_dev,
                           double *states_out_dev, double *z_out_dev, double *scratch_dev,
                           int64_t n, double beta, double ess_fraction, uint64_t seed, int64_t k,
                           int32_t estimate_best, er_smc_ctl *ctl_dev, double *trace_row_dev,
                           void *stream);

/* ---- warp / scoring of frames (geometry.py:188-200, metrics.py) -------- */

/* resample_trilinear (kernels_numba.py:65-85, 192-200): pull `src` through
 * the index affine onto an (nx, ny, nz) grid, fill 0, fp64 in the
 * reference's operation order.  out_dev is f64. */
int er_resample(const er_volume *src, const double A[9], const double b[3], int32_t nx,
                int32_t ny, int32_t nz, double *out_dev, void *stream);

/* dice_under_transform (metrics.py:88-93) as exact integer counts:
 * counts_dev[0] = |moved > 0.5|, [1] = |target == 1|, [2] = |both|. */
int er_warp_dice_counts(const er_volume *src_mask, const double A[9], const double b[3],
                        const er_volume *tgt_mask, int64_t *counts_dev, void *stream);

/* Two-pass squared-NCC sums of (tgt, warp(src)) over the full grid
 * (metrics.py:49-68): out_dev = {sst, sss, sts, n}; out_dev must hold
 * ER_NCC_SUMS_DOUBLES doubles (the tail is reduction scratch).  With
 * identity != 0 the source is read on the target grid unwarped. */
#define ER_NCC_SUMS_DOUBLES 1782
int er_warp_ncc_sums(const er_volume *tgt, const er_volume *src, const double A[9],
                     const double b[3], int32_t identity, double *out_dev, void *stream);

/* ---- synthetic phantoms (E/phantom.py:61-91) ------- */

/* Device scratch needed by er_phantom_speckle for n voxels. */
size_t er_phantom_scratch_bytes(int64_t n);

/* speckle_out[i] = np.exp(sigma * z_i), z = Generator(Philox(key=seed))
 * .standard_normal(n) (E/phantom.py:76-77), bit-exact: the ziggurat's
 * variable word consumption is resolved in parallel (chunked chain walk) and
 * exp is numpy's AVX512 SVML exp restated (csrc/npexp.cuh).  normals_out
 * (optional) receives z.  Synchronises the stream (checks the chain). */
int er_phantom_speckle(uint64_t seed, int64_t n, double sigma, void *scratch_dev,
                       size_t scratch_bytes, double *speckle_out_dev, double *normals_out_dev,
                       void *stream);

/* One frame of make_phantom (E/phantom.py:78-90): base intensity from the two
 * ellipsoid radii (semi-axes already scaled for the frame, as the reference
 * computes them) times the speckle -> frame_out (optional); cavity -> mask_out
 * bytes (optional).  C-order (nx, ny, nz), fp64 in the reference's op order. */
int er_phantom_frame(const double *speckle_dev, int32_t nx, int32_t ny, int32_t nz,
                     const double spacing[3], const double center[3], const double outer[3],
                     const double inner[3], double *frame_out_dev, uint8_t *mask_out_dev,
                     void *stream);

/* out = clip(round_half_even(v * scale), 0, 255) as bytes; entries at index
 * >= keep_before are 0 (make_pair's overlap crop, E/phantom.py:139-145). */
int er_quantize_u8(const double *v_dev, int64_t n, double scale, int64_t keep_before,
                   uint8_t *out_dev, void *stream);

/* out = (v > threshold) as bytes (E/volume.py:133-135), 0 at index >= keep_before. */
int er_binarize_u8(const double *v_dev, int64_t n, double threshold, int64_t keep_before,
                   uint8_t *out_dev, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ECHOREG_B200_H */
