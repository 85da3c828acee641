/*
 * mgauss_b200.h -- C ABI of the B200 (sm_100a) M-Gaussian rendering path.
 *
 * Every entry point takes raw DEVICE pointers, element counts and a
 * cudaStream_t passed as void*; none allocates (scratch comes from the
 * caller's `ws` buffer, sized by the matching *_workspace_bytes query); all
 * are asynchronous on `stream` and return 0 on success, a negative CUDA
 * error code on a launch failure, or a positive MG_E* code for an argument
 * error (message via mg_last_error()).  Domain errors raised by the
 * reference's Python wrappers (DegenerateQuaternion, InconsistentGrid,
 * OutOfMemoryRequest, ValueError) are raised by the host layer, exactly as
 * the reference raises them outside its kernels.
 *
 * Reference interfaces each group replaces (paths under
 * /root/reference/pkg/src/mgauss):
 *   mg_block_forward / mg_block_backward / mg_dense_forward (+ the strict
 *   float64 mg_block_forward_f64 / mg_block_backward_f64)
 *        -> _kernels.block_forward (_kernels.py:24-27), block_backward
 *           (_kernels.py:73-76), dense_forward (_kernels.py:147-148):
 *           same argument list and meaning, float64/int64 device arrays.
 *   mg_bin_f32 / mg_bin_f64 / mg_cell_keys_f64
 *        -> spatial.cell_index / spatial.build (spatial.py:18-66)
 *   mg_activate / mg_activate_f64
 *        -> render.activated_parameters (render.py:122-142)
 *   mg_bin_points + mg_forward + mg_forward_finish
 *        -> render.render_points (render.py:161-187), plus the slice-PSF
 *           tap expansion
 *   mg_backward_points + mg_backward + mg_backward_epilogue /
 *   mg_backward_accumulators
 *        -> render.render_backward (render.py:276-354)
 *   mg_transform_grads -> render.transform_grads_from_points (render.py:246-273)
 *   mg_sample_volume   -> render.sample_volume (render.py:379-408)
 *   mg_smooth_l1 / mg_gauss_update / mg_transform_adam / mg_upsample
 *        -> train.smooth_l1(_grad) (train.py:108-120), AdamState.step +
 *           aniso_loss_grad (train.py:128-147, 239-271), progressive_upsample
 *           (train.py:157-218)
 */
#ifndef MGAUSS_B200_H
#define MGAUSS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MG_ABI_VERSION 4
#define MG_EINVAL 1

int mg_abi_version(void);
const char *mg_last_error(void);
int mg_device_sm_count(void);
/* Kernel launches issued by this library so far (host-side counter; a CUDA
 * graph capture counts each captured launch once). */
long long mg_launch_count(void);

/* ---- binning: spatial.py:18-66 ------------------------------------------ */
/* keys[i] = (ci*G + cj)*G + ck with c = clamp(floor((x+1)*(G/2)), 0, G-1) in float64 */
int mg_cell_keys_f64(const double *pos, int64_t n, int64_t grid_res, uint32_t *keys, void *stream);
size_t mg_bin_workspace_bytes(int64_t n, int64_t grid_res);
/* Stable bucket sort: keys_sorted (n), cell_indices (n, ascending primitive id
 * within a cell), cell_starts (G^3+1).  int32 on device. */
int mg_bin_f32(const float *pos, int64_t n, int64_t grid_res, uint32_t *keys_sorted, int32_t *cell_indices,
               int32_t *cell_starts, void *ws, size_t ws_bytes, void *stream);
int mg_bin_f64(const double *pos, int64_t n, int64_t grid_res, uint32_t *keys_sorted, int32_t *cell_indices,
               int32_t *cell_starts, void *ws, size_t ws_bytes, void *stream);
/* keys_sorted[p] = the cell c with cell_starts[c] <= p < cell_starts[c+1]
 * (follows a caller-supplied CSR exactly, like the reference kernels do). */
int mg_keys_from_csr(const int32_t *cell_starts, int64_t ncell, uint32_t *keys_sorted, void *stream);
/* Device-wide exclusive scan of int32 (out may alias in); ws sized by
 * mg_scan_workspace_bytes.  Exposed for tests and the host layer. */
size_t mg_scan_workspace_bytes(int64_t n);
int mg_excl_scan_i32(const int32_t *in, int32_t *out, int64_t n, void *ws, size_t ws_bytes, void *stream);
/* int64 -> int32 copy (device CSR from the reference's int64 arrays). */
int mg_i64_to_i32(const int64_t *src, int64_t n, int32_t *dst, void *stream);
/* int32 -> int64 copies in the reference dtype (PartitionGrid fields). */
int mg_i32_to_i64(const int32_t *src, int64_t n, int64_t *dst, void *stream);

/* ---- preprocessing: render.py:122-142 ----------------------------------- */
/* Packed records in cell order (record p describes primitive cell_indices[p]),
 * structure-of-arrays in one float buffer of 12*n: float4 {mu, alpha} x n,
 * float4 {P'00, P'11, P'22, P'01} x n, float2 {P'02, P'12} x n, with
 * P' = -0.5*log2(e)*P.  err_flag |= 1 when some |q| <= 1e-12. */
int mg_activate(const float *pos, const float *quat, const float *log_scales, const float *logits, int64_t n,
                const int32_t *cell_indices, void *grec, int32_t *err_flag, void *stream);
/* Records from float64 prepared (mu (n,3), prec6 (n,6), alpha (n)) in cell order. */
int mg_pack_records(const double *mu, const double *prec6, const double *alpha, const int32_t *cell_indices,
                    int64_t n, void *grec, void *stream);
/* float64 activated_parameters: qn (n,4), rot (n,3,3), inv_var (n,3), prec6 (n,6), alpha (n) */
int mg_activate_f64(const double *quat, const double *log_scales, const double *logits, int64_t n, double *qn,
                    double *rot, double *inv_var, double *prec6, double *alpha, int32_t *err_flag, void *stream);

/* Per-slice rotations R(q/|q|) (k,3,3) from w-first quats (k,4), float64 (core.py:48-67). */
int mg_quat_to_rot_f64(const double *quats, int64_t k, double *rot, void *stream);

/* ---- sample points: transform (+ PSF taps) and bin ---------------------- */
size_t mg_points_workspace_bytes(int64_t n_sub, int64_t grid_res);
/* n_sub = b * ntaps.  tap_offsets (ntaps) and through_dirs (k,3) may be NULL
 * (no PSF, ntaps = 1).  rot (k,3,3), trans (k,3) float64; slice_ids < 0 mean
 * identity.  Outputs: pkey_sorted (n_sub), pinv (n_sub: sorted position of
 * sub-point b*ntaps+t), pstart (G^3+1), prec (n_sub float4 records), and
 * optionally transformed (n_sub,3) float64 in input order. */
int mg_bin_points(const double *coords, const int64_t *slice_ids, int64_t b, int32_t ntaps,
                  const double *tap_offsets, const double *through_dirs, const double *rot, const double *trans,
                  int64_t k, int64_t grid_res, uint32_t *pkey_sorted, int32_t *pinv, int32_t *pstart, void *prec,
                  double *transformed, void *ws, size_t ws_bytes, void *stream);

/* ---- forward: _kernels.py:24-70 ----------------------------------------- */
size_t mg_forward_workspace_bytes(int64_t n_sub);
/* out4[p] = {H.x, H.y, H.z, I} per sorted sub-point (H = sum alpha g P d,
 * only when with_h != 0); counts[p] = candidate count (sorted order). */
int mg_forward(const void *grec, int64_t n_gauss, const int32_t *gstart, int64_t grid_res, int64_t radius,
               const void *prec,
               const uint32_t *pkey_sorted, const int32_t *pstart, int64_t n_sub, int32_t with_h, void *out4,
               int32_t *counts, void *ws, size_t ws_bytes, void *stream);
/* I_b = sum_t w_t I_(b,t) (tap_weights NULL = single tap); counts summed. */
int mg_forward_finish(const void *out4, const int32_t *counts, const int32_t *pinv, int64_t b, int32_t ntaps,
                      const double *tap_weights, double *intensity, float *intensity_f32, int64_t *counts_out,
                      int64_t *pair_total, void *stream);

/* ---- backward: _kernels.py:73-144, render.py:276-354 -------------------- */
/* upstream (b) float64 (or upstream_f32) -> prec[].w and d_points (n_sub,3, input order, may be NULL) */
int mg_backward_points(const double *upstream, const float *upstream_f32, int64_t b, int32_t ntaps,
                       const double *tap_weights, const int32_t *pinv, const void *out4, void *prec,
                       double *d_points, void *stream);
size_t mg_backward_workspace_bytes(int64_t n, int64_t grid_res);
/* Gaussian-major pair pass: acc10[p] = {S, T(3), A6(6)} per sorted Gaussian.
 * For radius <= 5 strips of 16 cells stage their neighbourhood in shared
 * memory with TMA bulk copies when MGAUSS_STAGED_BWD=1 (default: L1/L2 item path). */
int mg_backward(const void *grec, const uint32_t *gkey_sorted, const int32_t *gstart, int64_t n, int64_t grid_res,
                int64_t radius, const void *prec, const int32_t *pstart, float *acc10, void *ws, size_t ws_bytes,
                void *stream);
/* RenderGradients parameter fields (float64, primitive order). */
int mg_backward_epilogue(const float *acc10, const int32_t *cell_indices, int64_t n, const float *quat,
                         const float *log_scales, const float *logits, double *d_positions, double *d_quaternions,
                         double *d_log_scales, double *d_logits, void *stream);
/* render.py:319-340 chain rule from reference-convention float64 accumulators
 * (d_mu, d_abar6, d_alpha) and float64 parameters; primitive order. */
int mg_epilogue_f64(const double *d_mu, const double *d_abar6, const double *d_alpha, const double *quat,
                    const double *log_scales, const double *logits, int64_t n, double *d_positions,
                    double *d_quaternions, double *d_log_scales, double *d_logits, void *stream);
/* Reference block_backward accumulators, ADDED into d_mu (n,3), d_abar6 (n,6), d_alpha (n). */
int mg_backward_accumulators(const float *acc10, const int32_t *cell_indices, int64_t n, const double *alpha,
                             double *d_mu, double *d_abar6, double *d_alpha, void *stream);
/* (k,7) transform gradients; scratch12 is (k,12) float64. */
/* The per-slice sums are reduced deterministically (fixed order, no float
 * atomics) when ws holds mg_transform_grads_workspace_bytes(k) bytes; with
 * ws == NULL an atomic fallback is used (not bit-reproducible). */
size_t mg_transform_grads_workspace_bytes(int64_t k);
int mg_transform_grads(const double *d_points, const double *coords, const int64_t *slice_ids, int64_t b,
                       int32_t ntaps, const double *tap_offsets, const double *through_dirs, const double *t_quats,
                       int64_t k, double *scratch12, double *out7, int32_t accumulate, void *ws, size_t ws_bytes,
                       void *stream);

/* ---- inference: render.py:357-408 --------------------------------------- */
size_t mg_volume_workspace_bytes(int64_t nx, int64_t ny, int64_t nz);
/* Slab [i0, i1) of a node-inclusive (nx,ny,nz) grid over [lo, hi]; out is
 * (i1-i0, ny, nz) float32 clipped to [0,1]; residual (same shape) optional. */
int mg_sample_volume(const void *grec, int64_t n_gauss, const int32_t *gstart, int64_t grid_res, int64_t radius,
                     int64_t nx,
                     int64_t ny, int64_t nz, const double *lo3_host, const double *hi3_host, int64_t i0, int64_t i1,
                     const float *residual, float *out, void *ws, size_t ws_bytes, void *stream);

/* ---- training: train.py ------------------------------------------------- */
/* Smooth-L1 data loss (train.py:108-120): upstream_out = dL/dpred over the b
 * predictions (mean), loss_acc += L (float64 device scalar). */
int mg_smooth_l1(const float *pred, const float *target, int64_t b, float *upstream_out, double *loss_acc,
                 void *stream);
/* Same with an explicit normaliser: upstream_out = scale * dHuber/dpred,
 * loss_acc += scale * sum Huber.  A rank holding a share of a sharded batch
 * passes scale = 1 / (global batch size), so the all-reduced partial sums
 * are exactly the global mean and its gradient. */
int mg_smooth_l1_scaled(const float *pred, const float *target, int64_t b, double scale, float *upstream_out,
                        double *loss_acc, void *stream);
/* aniso_loss_grad (train.py:128-147), float64: grad (n,3) overwritten with
 * d(loss)/d(log_scales), loss_acc += loss. */
int mg_aniso_loss_grad_f64(const double *log_scales, int64_t n, double lambda_ratio, double *grad,
                           double *loss_acc, void *stream);
/* AdamState.step on one float64 tensor (train.py:251-271); t = the group's
 * post-increment step count.  param, m, v updated in place. */
int mg_adam_f64(double *param, const double *grad, double *m, double *v, int64_t n, int64_t t, double lr,
                double beta1, double beta2, double eps, void *stream);
/* Residual field r(x) = 0.1 tanh(MLP(enc(x))) with the reference widths
 * 39-64-64-64-64-1, SiLU, 6 Fourier bands (nrf.py:23-182; ResidualField.forward /
 * backward).  w[l] are (fan_in, fan_out) row-major float32, bias[l] (fan_out).
 * Forward: r_out / pred_add (+= r) / t_out = tanh(.) / z_out = 4 x b x 64 hidden
 * pre-activations (point-major; needed by the backward), each optional except
 * t_out.  Backward: d_points (b x 3) and the parameter gradients of
 * sum_b upstream_b r(x_b), deterministic (fixed-order partial sums). */
int mg_nrf_forward(const float *x, int64_t b, const float *const *w, const float *const *bias, float *pred_add,
                   float *r_out, float *t_out, float *z_out, void *stream);
size_t mg_nrf_backward_workspace_bytes(int64_t b);
int mg_nrf_backward(const float *x, int64_t b, const float *const *w, const float *const *bias,
                    const float *upstream, const float *t, const float *z, float *d_points, float *const *dw,
                    float *const *db, void *ws, size_t ws_bytes, void *stream);

/* Adam over up to 10 float32 parameter tensors (AdamState.step, train.py:251-271):
 * reads the device step counter *tstep (float64), uses t = *tstep + 1 for the bias
 * corrections and stores it back; sizes[k] elements in params[k], grads[k], m[k], v[k]. */
int mg_nrf_adam(const float *const *grads, float *const *params, float *const *m, float *const *v,
                const int64_t *sizes, int32_t count, double *tstep, double lr, double beta1, double beta2,
                double eps, void *stream);

/* 2D SSIM (ssim.py:59-122) of an (H,W) slice: upstream_out = scale * d(1-SSIM)/dpred,
 * ssim_sum += sum of the SSIM map over the (H-10)(W-10) valid windows. */
size_t mg_ssim_workspace_bytes(int64_t h, int64_t w);
int mg_ssim_loss_grad(const float *pred, const float *target, int64_t h, int64_t w, double scale,
                      float *upstream_out, double *ssim_sum, void *ws, size_t ws_bytes, void *stream);
int mg_counter_incr(int32_t *counters, int32_t n, void *stream);
/* One step's batch rows from the resident sample pool (train.py:332-347 draws
 * pool indices; the rows are gathered on the device): coords[i] =
 * pool_coords[idx[i]] (3 doubles), slice_ids[i], target[i] likewise. */
int mg_gather_batch(const int64_t *idx, int64_t n, const double *pool_coords, const int64_t *pool_slice_ids,
                    const float *pool_target, double *coords, int64_t *slice_ids, float *target, void *stream);
/* hyper (host, 9 doubles): lr_pos, lr_quat, lr_scale, lr_logit, beta1, beta2, eps, lambda_aniso, lambda_ratio.
 * t_dev: device int32 post-increment Adam step.  Moments m, v are float32 structure-of-arrays (11, n)
 * (slot rows: position 3, quaternion 4, log-scale 3, logit 1); the Adam arithmetic is float32. */
int mg_gauss_update(const float *acc10, const int32_t *cell_indices, int64_t n, float *pos, float *quat,
                    float *log_scales, float *logits, float *m, float *v, const double *hyper_host,
                    int32_t use_aniso, const int32_t *t_dev, double *aniso_acc, void *stream);
/* Same update walking the ORIGINAL Gaussian order (coalesced parameter and
 * moment rows): inv[i] = the sorted position of Gaussian i (the inverse of
 * cell_indices, mg_invert_permutation).  Bit-identical results. */
int mg_gauss_update_inv(const float *acc10, const int32_t *inv, int64_t n, float *pos, float *quat,
                        float *log_scales, float *logits, float *m, float *v, const double *hyper_host,
                        int32_t use_aniso, const int32_t *t_dev, double *aniso_acc, void *stream);
/* inv[perm[p]] = p for a permutation of 0..n-1 (int32). */
int mg_invert_permutation(const int32_t *perm, int64_t n, int32_t *inv, void *stream);
int mg_transform_adam(double *t_quats, double *t_trans, const double *grad7, double *m7, double *v7, int64_t k,
                      double lr, double beta1, double beta2, double eps, const int32_t *t_dev, void *stream);
/* node_of_old[(i*R+j)*R+k] = primitive id at lattice node (i,j,k) */
int mg_upsample(const float *quat_old, const float *log_scales_old, const float *logits_old,
                const int32_t *node_of_old, int64_t r_old, int64_t r_new, float *pos, float *quat,
                float *log_scales, float *logits, void *stream);

/* ---- drop-in reference kernel ABI: _kernels.py -------------------------- */
size_t mg_block_workspace_bytes(int64_t b, int64_t n, int64_t grid_res);
int mg_block_forward(const double *points, const int64_t *slice_ids, int64_t b, const double *rot,
                     const double *trans, int64_t k, const double *mu, const double *prec6, const double *alpha,
                     int64_t n, const int64_t *cell_starts, const int64_t *cell_indices, int64_t grid_res,
                     int64_t radius, double *out_intensity, int64_t *out_counts, double *out_transformed, void *ws,
                     size_t ws_bytes, void *stream);
int mg_block_backward(const double *points, const int64_t *slice_ids, int64_t b, const double *rot,
                      const double *trans, int64_t k, const double *mu, const double *prec6, const double *alpha,
                      int64_t n, const int64_t *cell_starts, const int64_t *cell_indices, int64_t grid_res,
                      int64_t radius, const double *upstream, double *d_mu, double *d_abar6, double *d_alpha,
                      double *out_dpoint, void *ws, size_t ws_bytes, void *stream);
/* Self-test of the tcgen05 tensor-core path (kind::tf32, TMEM accumulator) the
 * NRF layers use: D (128 x 64) = A (128 x 64, row-major) * B where Bt (64 x 64)
 * holds B transposed; split != 0 evaluates 3xTF32 (hi*hi + hi*lo + lo*hi). */
int mg_tc_selftest(const float *A, const float *Bt, float *D, int32_t split, void *stream);
/* Strict float64 instantiation of the same two kernels (same arguments, same
 * ownership): every pair is evaluated in IEEE float64 in the reference's
 * operation order without FMA contraction, so results agree with
 * _kernels.py to ~1e-15 relative (selected by render.set_strict_fp64). */
size_t mg_block_f64_workspace_bytes(int64_t b, int64_t n, int64_t grid_res);
int mg_block_forward_f64(const double *points, const int64_t *slice_ids, int64_t b, const double *rot,
                         const double *trans, int64_t k, const double *mu, const double *prec6, const double *alpha,
                         int64_t n, const int64_t *cell_starts, const int64_t *cell_indices, int64_t grid_res,
                         int64_t radius, double *out_intensity, int64_t *out_counts, double *out_transformed,
                         void *ws, size_t ws_bytes, void *stream);
int mg_block_backward_f64(const double *points, const int64_t *slice_ids, int64_t b, const double *rot,
                          const double *trans, int64_t k, const double *mu, const double *prec6, const double *alpha,
                          int64_t n, const int64_t *cell_starts, const int64_t *cell_indices, int64_t grid_res,
                          int64_t radius, const double *upstream, double *d_mu, double *d_abar6, double *d_alpha,
                          double *out_dpoint, void *ws, size_t ws_bytes, void *stream);
/* Float64 variants of the training-step pieces for strict-float64 training
 * (train.StrictTrainer): Huber loss (train.py:108-120), SSIM loss/gradient
 * (ssim.py:82-122), progressive upsample (train.py:157-218), and the residual
 * field forward / manual backward (nrf.py:23-182) in float64 like the
 * reference's numpy code.  mg_nrf_forward_f64 fills `ws` with the forward
 * cache (encoding, activations) that mg_nrf_backward_f64 consumes, the role
 * of nrf_forward_cached's cache (nrf.py:140-145); weights are (fan_in,
 * fan_out) row-major float64; widths[0..depth] = (3 + 6 bands, hidden...,
 * 1), every width <= 64, depth <= 8 (any ResidualField.create configuration
 * of that size, nrf.py:58-83). */
int mg_smooth_l1_f64(const double *pred, const double *target, int64_t b, double *upstream_out, double *loss_acc,
                     void *stream);
int mg_ssim_loss_grad_f64(const double *pred, const double *target, int64_t h, int64_t w, double scale,
                          double *upstream_out, double *ssim_sum, void *ws, size_t ws_bytes, void *stream);
int mg_upsample_f64(const double *quat_old, const double *log_scales_old, const double *logits_old,
                    const int32_t *node_of_old, int64_t r_old, int64_t r_new, double *pos, double *quat,
                    double *log_scales, double *logits, void *stream);
size_t mg_nrf_f64_workspace_bytes(int64_t b);
int mg_nrf_forward_f64(const double *x, int64_t b, const double *const *w, const double *const *bias,
                       const int32_t *widths, int32_t depth, int32_t bands, double output_bound, double *r_out,
                       void *ws, size_t ws_bytes, void *stream);
int mg_nrf_backward_f64(const double *x, int64_t b, const double *const *w, const double *const *bias,
                        const int32_t *widths, int32_t depth, int32_t bands, double output_bound,
                        const double *upstream, double *d_points, double *const *d_w, double *const *d_b, void *ws,
                        size_t ws_bytes, void *stream);
size_t mg_dense_workspace_bytes(int64_t n);
int mg_dense_forward(const double *points, int64_t b, const double *mu, const double *prec6, const double *alpha,
                     int64_t n, double *out_intensity, void *ws, size_t ws_bytes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MGAUSS_B200_H */
