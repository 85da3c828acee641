// mg_render.cuh -- host launchers for the Gaussian path kernels.
#pragma once
#include "mg_common.cuh"

namespace mg {
int num_sms();
int fwd_qmax();
int fwd_dense_min();

// preprocessing / binning
void launch_gauss_keys(const float* pos, int64_t n, int g, uint32_t* keys, cudaStream_t st);
void launch_gauss_keys_f64(const double* pos, int64_t n, int g, uint32_t* keys, cudaStream_t st);
void launch_gauss_activate(const float* pos, const float* quat, const float* ls, const float* lg, const int* order,
                           int64_t n, float* grec, int* err, cudaStream_t st);
void launch_gauss_pack_prepared(const double* mu, const double* prec6, const double* alpha, const int* order,
                                int64_t n, float* grec, cudaStream_t st);
void launch_points_prepare(const double* coords, const int64_t* sids64, const int* sids32, int64_t b, int ntaps,
                           const double* tap_off, const double* dirs, const double* rot, const double* trans,
                           int nslices, int g, uint32_t* keys, float4* xf, double* xout, cudaStream_t st);
void launch_points_gather(const float4* xf, const int* perm, int64_t n, float4* prec, int* inv, cudaStream_t st);
size_t items_workspace_bytes(int64_t n);
void build_items_cells(const int* starts, int g, int q, int4* items, int* nitems, cudaStream_t st,
                       int dense_min = 0);
void build_items(const uint32_t* keys, const int* starts, int64_t n, int q, int4* items, int* nitems, void* ws,
                 cudaStream_t st, int dense_min = 0);

// pair kernels
void launch_forward(bool with_h, const float* grec, int64_t n_gauss, const int* gstart, int g, int r,
                    const float4* prec,
                    const uint32_t* pkey, const int* pstart, const int4* items, const int* nitems, int64_t max_items,
                    float4* out4, int* cnt, cudaStream_t st);
void launch_backward(const float* grec, int64_t n_gauss, const uint32_t* gkey, const int* gstart, int g, int r,
                     const float4* prec, const int* pstart, const int4* items, const int* nitems, int64_t max_items,
                     float* acc10, cudaStream_t st, int pair_mode = 0);

size_t backward_staged_ws_bytes(int64_t n, int g);
void launch_backward_staged(const float* grec, int64_t n_gauss, const uint32_t* gkey, const int* gstart, int g, int r,
                            const float4* prec, const int* pstart, float* acc10, void* ws, cudaStream_t st);

// epilogues / training
void launch_forward_finish(const float4* out4, const int* cnt, const int* inv, int64_t b, int ntaps,
                           const double* tap_w, double* out_i, float* out_i32, int64_t* out_cnt, int64_t* pair_total,
                           cudaStream_t st);
void launch_gather_batch(const int64_t* idx, int64_t n, const double* pc, const int64_t* ps, const float* pt,
                         double* c, int64_t* s, float* t, cudaStream_t st);
void launch_backward_points(const double* up64, const float* up32, const int* inv, int64_t b, int ntaps,
                            const double* tap_w, const float4* out4, float4* prec, double* dpoints, cudaStream_t st);
void launch_acc_to_ref(const float* acc10, const int* order, int64_t n, const double* alpha64, double* d_mu,
                       double* d_abar6, double* d_alpha, cudaStream_t st);
void launch_epilogue(const float* acc10, const int* order, int64_t n, const float* quat, const float* ls,
                     const float* lg, double* d_pos, double* d_q, double* d_s, double* d_l, cudaStream_t st);
void launch_epilogue_f64(const double* d_mu, const double* d_abar6, const double* d_alpha, const double* quat,
                         const double* ls, const double* lg, int64_t n, double* d_pos, double* d_q, double* d_s,
                         double* d_l, cudaStream_t st);
void launch_transform_grads(const double* dpoints, const double* coords, const int64_t* sids, int64_t b, int ntaps,
                            const double* tap_off, const double* dirs, const double* tq, int k, double* acc12,
                            double* out7, int accumulate, void* ws, cudaStream_t st);
size_t transform_grads_ws_bytes(int64_t k);
void launch_smooth_l1(const float* pred, const float* target, int64_t b, double scale, float* up_out,
                      double* loss_acc, cudaStream_t st);
void launch_aniso_f64(const double* ls, int64_t n, double lambda_ratio, double* grad, double* loss_acc,
                      cudaStream_t st);
void launch_adam_f64(double* p, const double* g, double* m, double* v, int64_t n, int64_t t, double lr, double b1,
                     double b2, double eps, cudaStream_t st);
// fused residual field (mg_nrf.cu)
size_t nrf_backward_ws_bytes(int64_t b);
void launch_nrf_forward(const float* x, int64_t b, const float* const* w, const float* const* bias, float* pred_add,
                        float* r_out, float* t_out, float* z_out, cudaStream_t st);
void launch_nrf_backward(const float* x, int64_t b, const float* const* w, const float* const* bias, const float* up,
                         const float* t, const float* z, float* dp, float* const* dw, float* const* db, void* ws,
                         cudaStream_t st);
void launch_nrf_adam(const float* const* g, float* const* p, float* const* m, float* const* v, const int64_t* n,
                     int count, double* tstep, double lr, double b1, double b2, double eps, cudaStream_t st);
size_t ssim_workspace_bytes(int H, int W);
void launch_ssim(const float* pred, const float* tgt, int H, int W, double scale, float* up, double* ssim_sum,
                 void* ws, cudaStream_t st);
void launch_quat_to_rot(const double* q, int64_t k, double* rot, cudaStream_t st);
void launch_counter_incr(int* c, int n, cudaStream_t st);
void launch_gauss_update(const float* acc10, const int* perm, int by_inv, int64_t n, float* pos, float* quat,
                         float* ls, float* lg, float* mom_m, float* mom_v, const double* hyper, int use_aniso,
                         const int* t_dev, double* aniso_acc, cudaStream_t st);
void launch_invert_perm(const int* perm, int64_t n, int* inv, cudaStream_t st);
void launch_transform_adam(double* tq, double* tt, const double* g7, double* m7, double* v7, int k, double lr,
                           double b1, double b2, double eps, const int* t_dev, cudaStream_t st);
void launch_upsample(const float* q_old, const float* s_old, const float* l_old, const int* node_of_old, int ro, int rn,
                     float* pos, float* q, float* s, float* l, cudaStream_t st);

// float64 variants for the strict-float64 training path
void launch_smooth_l1_f64(const double* pred, const double* target, int64_t b, double divisor, double* up_out,
                          double* loss_acc, cudaStream_t st);
void launch_ssim_f64(const double* pred, const double* tgt, int H, int W, double scale, double* up,
                     double* ssim_sum, void* ws, cudaStream_t st);
void launch_upsample_f64(const double* q_old, const double* s_old, const double* l_old, const int* node_of_old,
                         int ro, int rn, double* pos, double* q, double* s, double* l, cudaStream_t st);
size_t nrf64_workspace_bytes(int64_t b);
bool launch_nrf64_forward(const double* x, int64_t b, const double* const* w, const double* const* bias,
                          const int* widths, int depth, int bands, double bound, double* r, void* ws,
                          cudaStream_t st);
bool launch_nrf64_backward(const double* x, int64_t b, const double* const* w, const double* const* bias,
                           const int* widths, int depth, int bands, double bound, const double* up,
                           double* d_points, double* const* dw, double* const* db, void* ws, cudaStream_t st);

// tensor-core (tcgen05) NRF layers and the self-test GEMM (mg_nrf_tc.cu)
bool nrf_use_tc();
void launch_nrf_forward_tc(const float* x, int64_t b, const float* const* w, const float* const* bias,
                           float* pred_add, float* r_out, float* t_out, float* z_out, cudaStream_t st);
void launch_nrf_bwd_chain_tc(const float* x, int64_t b, const float* const* w, const float* const* bias,
                             const float* up, const float* t, const float* z, float* dz, float* d4, float* dp,
                             float* hout, float* enc, cudaStream_t st);
void launch_tc_selftest(const float* A, const float* Bt, float* D, int split, cudaStream_t st);

// strict float64 reference-order pair kernels (mg_strict.cu)
size_t strict_workspace_bytes(int64_t b, int64_t n, int64_t g);
int strict_block(const double* points, const int64_t* sids, int64_t b, const double* rot, const double* trans,
                 int64_t k, const double* mu, const double* prec6, const double* alpha, int64_t n, const int64_t* cs,
                 const int64_t* ci, int g, int r, double* out_i, int64_t* out_cnt, double* out_x,
                 const double* upstream, double* d_mu, double* d_abar6, double* d_alpha, double* out_dp, void* ws,
                 size_t wsb, cudaStream_t st);

// inference
size_t volume_workspace_bytes(int nx, int ny, int nz);
void launch_sample_volume(const float* grec, int64_t n_gauss, const int* gstart, int g, int r, const int dims[3],
                          const double lo[3],
                          const double hi[3], int i0, int i1, const float* residual, float* out, void* ws,
                          cudaStream_t st);
}  // namespace mg
