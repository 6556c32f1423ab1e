/* bnff.h -- C ABI of libbnff: the B200 (sm_100a) kernels of the restructured
 * batch-norm training path (BN fission-n-fusion, arXiv 1807.01702).
 *
 * Every entry point replaces one reference function of the Python/numpy
 * package `bnfuse` (paths relative to /root/reference/pkg/src/bnfuse/); the
 * Python mirror (paper_1807_01702_b200/kernels.py) binds them with ctypes and
 * keeps the reference names and argument meaning.
 *
 * Conventions
 *  - Feature maps are NHWC views: `ptr` points at (n=0,h=0,w=0,c=channel offset)
 *    and consecutive pixels are `row_stride` ELEMENTS apart, so a channel-offset
 *    slice of a DenseNet block buffer is just (base + offset, row_stride = C_total).
 *  - dtype BNFF_BF16: bf16 storage, bf16 tcgen05 MMA (kind::f16), fp32 accumulate.
 *    dtype BNFF_F32 : fp32 storage, 3xTF32 split tcgen05 MMA (kind::tf32, ~fp32).
 *  - Channel counts and channel offsets must be multiples of 8 (bf16) / 4 (f32).
 *  - Per-channel statistics are float64; per-tile partials are float64 and are
 *    combined in a fixed order (bitwise run-to-run deterministic, no atomics).
 *  - No allocation, no host synchronisation; all work is ordered on `stream`
 *    (a cudaStream_t, NULL = legacy default stream).
 *  - Return: 0 ok, 1 shape (ShapeError), 2 state (StateError), 3 unsupported,
 *    4 CUDA error; bnff_last_error() gives the message.
 */
#ifndef BNFF_H_
#define BNFF_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { BNFF_OK = 0, BNFF_ERR_SHAPE = 1, BNFF_ERR_STATE = 2, BNFF_ERR_UNSUPPORTED = 3,
       BNFF_ERR_CUDA = 4 };
enum { BNFF_F32 = 0, BNFF_BF16 = 1 };

/* operand transforms applied while a conv kernel reads a feature map */
enum {
  BNFF_PRO_NONE = 0,
  BNFF_PRO_RELU = 1,         /* max(x,0): RCF clip-on-read (execute.py:170, fusion.py:127-148) */
  BNFF_PRO_BN_RELU = 2,      /* max((x-mean)*scale+beta,0): sub-BN2 + ReLU (fused.py:133-135) */
  BNFF_PRO_BN_DX = 3,        /* g*(dt1-k1-xhat*k2): deferred sub-BN1' dx (ops.py:283-298) */
};
/* dgrad epilogues */
enum {
  BNFF_DG_PLAIN = 0,         /* dx (ops.py:193-202) */
  BNFF_DG_CLIP = 1,          /* dx where x>0 (execute.py:331-332) */
  BNFF_DG_NRC = 2,           /* dt1 = dx where relu(bn(x))>0, + sum dt1, sum dt1*xhat (fused.py:176-188) */
  /* NRC with the block-gradient fold (ICF): instead of storing dt1 for a
   * later split_bwd, the epilogue writes dx := (ACC ? dx : 0) + scale * dt1 into the
   * block gradient buffer (scale = gamma*invstd = x_coef.b); the per-channel remainder
   * -scale*(k1 + xhat*k2) is accumulated by bnff_dx_coeffs_acc.  Window kernels only.  */
  BNFF_DG_NRC_ACC = 3,
  BNFF_DG_NRC_SET = 4,
};

typedef struct {
  void* ptr;
  int64_t n, h, w, c;
  int64_t row_stride; /* elements between consecutive pixels */
} bnff_view;

/* Per-channel coefficient table consumed by the operand prologues:
 *   BNFF_PRO_BN_RELU: a = mean, b = scale (=gamma*invstd), c = beta
 *   BNFF_PRO_BN_DX  : a = mean, b = invstd, c = k1 (=dbeta/m), d = k2 (=dgamma/m), e = g (=gamma*invstd)
 * each array holds `c` floats (channels of the transformed tensor).            */
typedef struct {
  const float* a;
  const float* b;
  const float* c;
  const float* d;
  const float* e;
} bnff_coef;

typedef struct {
  int32_t dtype;
  int32_t kh, kw, stride, pad;
  bnff_view x;        /* conv input  (n, h, w, c_in)  */
  bnff_view y;        /* conv output (n, oh, ow, c_out) */
  const void* wpack;  /* packed weights [c_out][kh*kw*c_in (padded)] (bnff_pack_weights) */
  const float* bias;  /* c_out, nullable */
  int32_t x_pro;      /* BNFF_PRO_NONE / RELU / BN_RELU */
  bnff_coef x_coef;
  double* stat_part;  /* nullable: sum/sumsq partials [bnff_stat_rows()][2][c_out] of the stored y */
  const void* wwin;   /* nullable: window-layout weights (bnff_pack_window, fwd); selects the
                         window-shift kernel when bnff_window_ok() */
} bnff_fprop_args;

typedef struct {
  int32_t dtype;
  int32_t kh, kw, stride, pad;
  bnff_view dy;       /* grad wrt conv output (or dt1 of a deferred package) */
  bnff_view dy_x;     /* BNFF_PRO_BN_DX: the package's normalized-input tensor (conv output) */
  int32_t dy_pro;     /* BNFF_PRO_NONE / BN_DX */
  bnff_coef dy_coef;
  bnff_view dx;       /* output: grad wrt conv input (n, h, w, c_in) */
  bnff_view x;        /* conv input (for CLIP / NRC epilogues) */
  const void* wpack_t;/* packed transposed weights [c_in][kh*kw*c_out (padded)] */
  int32_t epi;        /* BNFF_DG_* */
  bnff_coef x_coef;   /* NRC: a = mean, b = scale, c = beta, d = invstd */
  double* stat_part;  /* NRC: partials [bnff_stat_rows()][2][c_in] of (sum dt1, sum dt1*xhat) */
  const void* wwin;   /* nullable: window-layout weights (bnff_pack_window, dgrad) */
} bnff_dgrad_args;

typedef struct {
  int32_t dtype;
  int32_t kh, kw, stride, pad;
  bnff_view x;        /* conv input (n, h, w, c_in) */
  int32_t x_pro;      /* NONE / RELU / BN_RELU (recompute of the saved post-ReLU input) */
  bnff_coef x_coef;
  bnff_view dy;       /* (n, oh, ow, c_out) */
  bnff_view dy_x;
  int32_t dy_pro;     /* NONE / BN_DX */
  bnff_coef dy_coef;
  int32_t splits;     /* split-K factor (0 = choose; < 0 forces the generic kernel); see
                         bnff_wgrad_workspace */
  float* workspace;   /* splits * (kh*kw*c_in) * c_out floats */
  float* dw;          /* output (c_out, dw_cin, kh, kw) fp32, reference layout */
  int32_t dw_cin;     /* real input channels (<= x.c when the input is channel-padded); 0 = x.c */
  float* dbias;       /* nullable, c_out fp32: sum of (transformed) dy */
} bnff_wgrad_args;

const char* bnff_last_error(void);
int bnff_version(void);
int bnff_device_ok(void); /* 1 if device 0 is sm_100 */

/* Rows of the per-CTA statistics partial buffers written by bnff_conv_fprop /
 * bnff_conv_dgrad (= number of SMs; one persistent CTA per SM).  The buffer
 * [rows][2][c] must be zero-initialised once; rows a launch does not use stay 0. */
int32_t bnff_stat_rows(void);

/* K1: conv2d_fwd (ops.py:151-175), fused_conv_stats_fwd (fused.py:79-100),
 *     fused_norm_relu_conv_fwd (fused.py:103-154), RCF clipped conv (execute.py:167-179) */
int bnff_conv_fprop(const bnff_fprop_args* a, void* stream);
/* K2: conv2d_bwd dx (ops.py:193-202), fused_nrc_bwd gradient pass (fused.py:176-188),
 *     fused_conv_stats_bwd dx (fused.py:203-219) */
int bnff_conv_dgrad(const bnff_dgrad_args* a, void* stream);
/* K3: conv2d_bwd dw/dbias (ops.py:195-203), fused_nrc_bwd weight pass (fused.py:190-199) */
int64_t bnff_wgrad_workspace(int32_t n, int32_t oh, int32_t ow, int32_t kh, int32_t kw,
                             int32_t c_in, int32_t c_out, int32_t splits);
int bnff_conv_wgrad(const bnff_wgrad_args* a, void* stream);
int32_t bnff_wgrad_default_splits(int32_t n, int32_t oh, int32_t ow, int32_t kh, int32_t kw,
                                  int32_t c_in, int32_t c_out);

/* weight re-layout (once per optimizer step): w (c_out, c_in, kh, kw) fp32 ->
 * forward pack [c_out][tap][c_in] and transposed pack [c_in][tap][c_out] in dtype,
 * K padded to a multiple of 64 (bf16) / 32 (f32) with zeros. c_in_store >= c_in pads
 * input channels with zeros (e.g. the 3-channel image stem).                     */
int64_t bnff_pack_size(int32_t dtype, int32_t c_out, int32_t c_in_store, int32_t kh, int32_t kw);
int bnff_pack_weights(int32_t dtype, const float* w, int32_t c_out, int32_t c_in,
                      int32_t c_in_store, int32_t kh, int32_t kw, void* wpack, void* wpack_t,
                      void* stream);

/* Window-shift tcgen05 kernels (csrc/wconv.cu) for stride-1 1x1/p0 and 3x3/p1 convs in
 * bf16: each input element is transformed once per tile and every 3x3 tap reads a
 * row-shifted window of it.  bnff_window_ok() says whether a conv qualifies; the
 * pre-swizzled weight layout is [slab][tap][n_pad][64B|128B row] (fwd: n = c_out,
 * reduction over c_in; dgrad: n = c_in, reduction over c_out, taps flipped).        */
int bnff_window_ok(int32_t dtype, int32_t c_in, int32_t c_out, int32_t kh, int32_t kw,
                   int32_t stride, int32_t pad, int32_t h, int32_t w);
/* bnff_window_ok for launches that need only some coefficient tables (bnff_window_ok = all
 * of them): the patch-matrix GEMMs (plain fprop operand, plain dgrad epilogue) reach
 * K = 4608 this way.  A conv call whose window plan is rejected falls back to the generic
 * kernel only when the caller passed generic packed weights (else BNFF_ERR_STATE). */
enum {
  BNFF_WT_FPROP_PRO = 1, /* fprop operand prologue (RELU / BN_RELU) */
  BNFF_WT_DGRAD_NRC = 2, /* dgrad NRC epilogue (and the fold variants) */
  BNFF_WT_DGRAD_PRO = 4, /* dgrad dy prologue (BN_DX) */
};
int bnff_window_ok_ex(int32_t dtype, int32_t c_in, int32_t c_out, int32_t kh, int32_t kw,
                      int32_t stride, int32_t pad, int32_t h, int32_t w, int32_t tables);
int64_t bnff_window_pack_size(int32_t dtype, int32_t c_out, int32_t c_in, int32_t kh, int32_t kw,
                              int32_t dgrad); /* elements */
int bnff_pack_window(int32_t dtype, const float* w, int32_t c_out, int32_t c_in, int32_t kh,
                     int32_t kw, void* wfwd, void* wdgrad, void* stream);
/* one launch re-packing many convs into the window layouts (after each SGD step);
 * jobs_dev points at njobs records in DEVICE memory; max_elems = largest pack (elements) */
typedef struct {
  const float* w;
  void* wfwd;
  void* wdgrad;
  int32_t c_out, c_in, kh, kw;
} bnff_pack_job;
int bnff_pack_window_multi(int32_t dtype, int32_t njobs, const bnff_pack_job* jobs_dev,
                           int64_t max_elems, void* stream);
int64_t bnff_window_wgrad_ws(int32_t n, int32_t h, int32_t w, int32_t kh, int32_t c_in,
                             int32_t c_out); /* floats of split partials */
int bnff_window_wgrad(bnff_view x, int32_t x_pro, bnff_coef x_coef, bnff_view dy, bnff_view dy_x,
                      int32_t dy_pro, bnff_coef dy_coef, int32_t kh, float* ws, float* dw,
                      int32_t dw_cin, float* dbias, void* stream);
int bnff_window_conv(int32_t dtype, int32_t mode, int32_t kh, int32_t pad, bnff_view in, bnff_view in_x,
                     int32_t pro, bnff_coef pcoef, bnff_view out, const void* wwin,
                     const float* bias, int32_t epi, bnff_view ex, bnff_coef ecoef,
                     double* stat_part, void* stream);

/* K5: channel sums over an NHWC view -> partials [tiles][2][c]:
 *   mode 0: (x, x^2)                         -- bn_stats_onepass (ops.py:231-237)
 *   mode 1: (dy, dy*xhat), xhat from x,coef(a=mean,b=invstd); optional relu mask
 *           from coef (mask_x>0 via c=... see kernels)  -- bn_bwd pass 1 (ops.py:271-274),
 *           FissionSubBN2 bwd (execute.py:381-399)
 *   mode 2: (dy, 0)                          -- conv dbias (ops.py:203)                */
int32_t bnff_sum_tiles(int64_t pixels);
int bnff_channel_sums(int32_t dtype, int32_t mode, bnff_view x, bnff_view dy, bnff_coef coef,
                      double* part, void* stream);
/* K4: partials -> float64 (sum, sumsq) and (mean, var) per channel plus the fp32
 * prologue table (mean32, scale32 = gamma*invstd, beta32, invstd32)
 * (ChannelStats.from_sums / inv_std, ops.py:109-116).  Writes sums at channel
 * offset `c_off` of the f64 arrays so per-piece stats assemble in place
 * (concat_stats, ops.py:128-143).                                               */
int bnff_stats_finalize(const double* part, int32_t tiles, int32_t c, int64_t count,
                        double* sum, double* sumsq, double* mean, double* var, void* stream);
/* two-pass centred variance for the unfused BN (ops.py:212-228): var from x and mean */
int bnff_centered_var(int32_t dtype, bnff_view x, const double* mean, double* part,
                      void* stream);
int bnff_var_finalize(const double* part, int32_t tiles, int32_t c, int64_t count, double* var,
                      void* stream);
/* var_finalize fused with bn_coeffs for the same BN (the unfused two-pass BN: var, then the
 * fp32 (mean32, scale32, beta32, inv32) tables, in one launch) */
int bnff_var_finalize_coeffs(const double* part, int32_t tiles, int32_t c, int64_t count, double* var,
                             const double* mean, const float* gamma, const float* beta, float eps,
                             float* mean32, float* scale32, float* beta32, float* inv32, void* stream);
int bnff_bn_coeffs(int32_t c, const double* mean, const double* var, const float* gamma,
                   const float* beta, float eps, float* mean32, float* scale32, float* beta32,
                   float* inv32, void* stream);
/* bnff_stats_finalize of a freshly produced piece (channels [c_off, c_off+c_new) of c_total)
 * fused with the consumer's bnff_bn_coeffs over all c_total channels (the other channels'
 * mean/var are read from mean_all/var_all): one launch per ICF concatenation step.        */
int bnff_stats_finalize_coeffs(const double* part, int32_t tiles, int32_t c_new, int64_t count,
                               double* sum, double* sumsq, double* mean, double* var, int32_t c_off,
                               int32_t c_total, const double* mean_all, const double* var_all,
                               const float* gamma, const float* beta, float eps, float* mean32,
                               float* scale32, float* beta32, float* inv32, void* stream);
/* backward coefficient table from the reduced (dgamma, dbeta) sums:
 * k1 = dbeta/m, k2 = dgamma/m, g = gamma*invstd (ops.py:287-293). Also writes
 * the fp32 parameter gradients dgamma32/dbeta32 (nullable). */
int bnff_dx_coeffs(int32_t c, const double* part, int32_t tiles, int64_t count,
                   const double* mean, const double* var, const float* gamma, float eps,
                   double* dgamma64, double* dbeta64, float* k1, float* k2, float* g,
                   float* mean32, float* inv32, float* dgamma32, float* dbeta32, void* stream);

/* bnff_dx_coeffs plus the ICF block-gradient fold: acc_a[c] (+)= g*k1, acc_b[c] (+)= g*k2
 * (acc_init = 1 overwrites), and mean32/inv32 written into the caller's block-level
 * arrays, so the block gradient resolves as G - acc_a - acc_b*xhat when its producer
 * reads it (bn_dx_from_sums ops.py:283-298 re-associated over consumers).            */
int bnff_dx_coeffs_acc(int32_t c, const double* part, int32_t tiles, int64_t count,
                       const double* mean, const double* var, const float* gamma, float eps,
                       double* dgamma64, double* dbeta64, float* k1, float* k2, float* g,
                       float* mean32, float* inv32, float* dgamma32, float* dbeta32,
                       float* acc_a, float* acc_b, int32_t acc_init, void* stream);

/* SyncBN (data parallel with global-batch statistics): bnff_stats_finalize with mean/var
 * NULL reduces partials to float64 (sum, sumsq) only; the caller all-reduces them and
 * finalizes here with the global count.  Backward likewise: reduce (dbeta, dgamma)
 * partials with bnff_stats_finalize, all-reduce, then bnff_dx_coeffs_from_sums.     */
int bnff_stats_from_sums(int32_t c, int64_t count, const double* sum, const double* sumsq,
                         double* mean, double* var, void* stream);
int bnff_dx_coeffs_from_sums(int32_t c, int64_t count, const double* dbeta64, const double* dgamma64,
                             const double* mean, const double* var, const float* gamma, float eps,
                             float* k1, float* k2, float* g, float* mean32, float* inv32, void* stream);
int bnff_sums_to_f32(int32_t c, const double* a, const double* b, float* a32, float* b32, void* stream);

/* K6: y = (x-mean)*scale+beta [relu]  (bn_fwd ops.py:240-254, FissionSubBN2 execute.py:211-217) */
int bnff_bn_apply(int32_t dtype, bnff_view x, bnff_view y, bnff_coef coef, int32_t relu,
                  void* stream);
/* K7/K8: out = [acc +] sum_i resolve(in_i) where resolve is identity or the deferred
 * BN dx transform g*(dt1 - k1 - xhat*k2) with xhat from x_i (bn_dx_from_sums
 * ops.py:283-298, DeferredBNGrad.materialize execute.py:123-126, split_bwd
 * ops.py:398-408, fused_split_bwd_bn_dx fused.py:222-230).  Up to 2 inputs.      */
typedef struct {
  bnff_view g;     /* plain gradient or dt1 */
  bnff_view x;     /* deferred: the normalized-input tensor */
  int32_t deferred;
  bnff_coef coef;  /* a=mean b=invstd c=k1 d=k2 e=g */
} bnff_grad_term;
int bnff_grad_sum(int32_t dtype, bnff_view out, int32_t accumulate, const bnff_grad_term* terms,
                  int32_t nterms, void* stream);
/* ReLU (ops.py:306-319) */
int bnff_relu_fwd(int32_t dtype, bnff_view x, bnff_view y, void* stream);
int bnff_relu_bwd(int32_t dtype, bnff_view x, bnff_view dy, bnff_view dx, void* stream);
/* K9: avgpool k x k non-overlapping (ops.py:428-454); optional fused stats partials */
int bnff_avgpool_fwd(int32_t dtype, bnff_view x, bnff_view y, int32_t k, double* stat_part,
                     void* stream);
int bnff_avgpool_bwd(int32_t dtype, bnff_view dy, bnff_view dx, int32_t k, void* stream);
/* K9b: sub-BN2 -> ReLU -> k x k average pool in one pass (a chain whose consumer is a pool,
 * e.g. the stem, graph.py:358-375): y = avgpool(relu((x-a)*b+c)) (+ partials of y), and
 * backward dt1 = [bn(x) > 0] * spread(dy)/k^2 with (sum dt1, sum dt1*xhat) partials (xhat =
 * (x-a)*d), i.e. avgpool_bwd + relu_bwd + bn_bwd sums (ops.py:271-274, 314-319, 428-454). */
int bnff_norm_relu_pool_fwd(int32_t dtype, bnff_view x, bnff_view y, int32_t k, bnff_coef coef,
                            double* stat_part, void* stream);
int bnff_pool_relu_bn_bwd(int32_t dtype, bnff_view dy, bnff_view x, bnff_view dt1, int32_t k,
                          bnff_coef coef, double* part, void* stream);
/* K10: y = a + zero-channel-padded b (execute.py:266-280) */
int bnff_ews_fwd(int32_t dtype, bnff_view a, bnff_view b, bnff_view y, void* stream);
/* K11: copy a view into another (physical concat piece / gradient slice copy) */
int bnff_copy(int32_t dtype, bnff_view src, bnff_view dst, void* stream);
/* boundary layout conversions, NCHW fp32 host-format <-> NHWC dtype (channel-padded) */
int bnff_nchw_to_nhwc(int32_t dtype, const float* src, int64_t n, int64_t c, int64_t h,
                      int64_t w, bnff_view dst, void* stream);
int bnff_nhwc_to_nchw(int32_t dtype, bnff_view src, float* dst, void* stream);
/* K13: channel-poor stem conv as a GEMM (csrc/stem.cu).  The 7x7/s2 conv over the
 * 3-channel image (graph.py:358-375) reads its input through a packed patch matrix
 * col (n, oh, ow, kpad), k = (ky*kw + kx)*c_real + ci, zero beyond kh*kw*c_real; the
 * conv is then a 1x1 conv over col (forward and weight gradient), replacing the
 * 49-chunk gather of conv2d_fwd/conv2d_bwd (ops.py:151-204) for this layer.
 * x must be stored as one 16-byte pixel (8 bf16 / 4 fp32 channels).  weight_to_cols / cols_to_weight move
 * fp32 weights between (c_out, c_in, kh, kw) and (c_out, kpad).                  */
int bnff_im2col(int32_t dtype, bnff_view x, int32_t c_real, int32_t kh, int32_t kw, int32_t stride,
                int32_t pad, bnff_view col, void* stream);
/* K13b: input gradient of a patch-matrix stem conv: dx = col2im(dcol), dcol = dgrad of the 1x1
 * GEMM over the patch matrix (ops.py:178-204 dx for the 7x7/s2 stem); deterministic gather,
 * storage channels >= c_real written as zeros */
int bnff_col2im(int32_t dtype, bnff_view dcol, int32_t c_real, int32_t kh, int32_t kw, int32_t stride,
                int32_t pad, bnff_view dx, void* stream);
/* K13c: strided convolutions (ResNet's stride-2 3x3s, ops.py:151-204 / fused.py:103-200) on the
 * window GEMM: im2col_s writes the patch matrix of pro(x) (pro = NONE / RELU / BN_RELU with the
 * (mean, scale, beta) tables of bnff_bn_coeffs; padding after the prologue); col2im_s gathers the
 * dgrad of the 1x1 GEMM back to dx with a PLAIN / CLIP / NRC-mask epilogue (x and the same
 * tables for the mask).  Channels must fill 16-byte chunks. */
int bnff_im2col_s(int32_t dtype, bnff_view x, int32_t kh, int32_t kw, int32_t stride, int32_t pad,
                  int32_t pro, bnff_coef pcoef, bnff_view col, void* stream);
int bnff_col2im_s(int32_t dtype, bnff_view dcol, int32_t kh, int32_t kw, int32_t stride, int32_t pad,
                  int32_t epi, bnff_view x, bnff_coef ecoef, bnff_view dx, void* stream);
int bnff_weight_to_cols(const float* w, int32_t c_out, int32_t c_in, int32_t kh, int32_t kw,
                        int32_t kpad, float* w2, void* stream);
int bnff_cols_to_weight(const float* dw2, int32_t c_out, int32_t c_in, int32_t kh, int32_t kw,
                        int32_t kpad, float* dw, void* stream);
/* K12: multi-tensor SGD w -= lr*g over a flat fp32 buffer */
int bnff_sgd(float* w, const float* g, int64_t n, float lr, void* stream);

/* debug: when buf != NULL (device memory, >= 16*1024 u64), window conv launches record a
 * %globaltimer timeline of CTA 0 (producer issue, TMA landed, transform done, MMA issue /
 * commit, epilogue per tile) into buf[event*1024 + index]; NULL turns it off.         */
int bnff_debug_trace(void* buf);

/* Profiling aid: an empty kernel; tools/ncu_node_ledger.py launches one before every engine
 * launch to attribute a profiler's per-kernel DRAM bytes to graph nodes. */
int bnff_debug_mark(int32_t id, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BNFF_H_ */
