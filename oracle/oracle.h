/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the dconv-b200 hot path.
 *
 * A plain-C restatement of the reference artifact's (arxiv 1808.05567,
 * /root/reference/proj) naive convolution oracles, blocked-layout
 * conversions, seeded data generator and error norms. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may
 * load this library; the product (paper_1808_05567_b200) never links it.
 *
 * Parity pinning: every function here is checked in tests/test_oracle.py
 * against (a) the reference's own known-answer tests (test_reference.cpp,
 * test_blocked.cpp, test_layer_spec.cpp, test_norms.cpp, acceptance.cpp:10)
 * restated as golden vectors in tests/golden/, and (b) the reference itself,
 * compiled from /root/reference sources into oracle/_ref/libdconv_ref.so by
 * oracle/Makefile (bitwise equality of the naive oracles).
 */
#ifndef DCONV_ORACLE_H
#define DCONV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ConvLayerSpec (layer_spec.hpp:12-38), field for field */
typedef struct {
  int N, C, K, H, W, R, S, stride, pad_h, pad_w, vlen;
} orc_spec;

/* status codes: 0 ok, 1 NonIntegralShape, 2 InvalidLayerSpec (errors.hpp) */
int orc_validate(const orc_spec* s);                         /* layer_spec.cpp:7-18 */
int orc_output_shape(const orc_spec* s, int* P, int* Q);     /* layer_spec.cpp:45-51 */
int orc_make_spec(int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h, int pad_w, int vlen,
                  orc_spec* out);                            /* layer_spec.cpp:20-43; pad<0 => "same" default */
int64_t orc_pass_flops(const orc_spec* s);                   /* harness.cpp:269-272 */

/* splitmix64 Rng (util.hpp:40-71) */
uint64_t orc_splitmix_next(uint64_t* state);
void orc_random_f32(uint64_t seed, float* out, int64_t n);   /* harness.cpp:274-278 via Rng::next_f32 */
/* stream helpers shared with the product generator */
void orc_uniform(uint64_t seed, float lo, float hi, float* out, int64_t n);
void orc_he_normal(uint64_t seed, float stddev, float* out, int64_t n);

/* naive oracles, f64 accumulation rounded once to f32 (reference.cpp:7-128).
 * threads > 1 parallelises over independent output elements only, so the
 * per-element summation order (and result) is identical to threads == 1. */
int orc_conv_forward(const orc_spec* s, const float* in, const float* wt, float* out, int threads);
int orc_conv_backward(const orc_spec* s, const float* grad_out, const float* wt, float* grad_in, int threads);
int orc_conv_update(const orc_spec* s, const float* in, const float* grad_out, float* grad_w, int threads);
int orc_conv_forward_f64(const orc_spec* s, const double* in, const double* wt, double* out);
int orc_conv_backward_f64(const orc_spec* s, const double* grad_out, const double* wt, double* grad_in);
int orc_conv_update_f64(const orc_spec* s, const double* in, const double* grad_out, double* grad_w);

/* blocked layouts (blocked.hpp:16-213); sizes in elements */
int64_t orc_act_elems(int n, int c, int h, int w, int vlen, int halo_h, int halo_w);
int64_t orc_wt_elems(int k, int c, int r, int s, int vlen);
void orc_to_blocked_act(const float* nchw, int n, int c, int h, int w, int vlen, int halo_h, int halo_w, float* out);
void orc_from_blocked_act(const float* blk, int n, int c, int h, int w, int vlen, int halo_h, int halo_w,
                          float* nchw);
void orc_to_blocked_wt(const float* kcrs, int k, int c, int r, int s, int vlen, float* out);
void orc_from_blocked_wt(const float* blk, int k, int c, int r, int s, int vlen, float* kcrs);
/* dual weights (propagation.hpp:20-33); out has (k,c) roles swapped */
void orc_transform_weight_stride1(const float* blk, int k, int c, int r, int s, int vlen, float* out);

/* error norms (norms.cpp:7-25): out[0..3] = linf_abs, l2_abs, linf_rel, l2_rel */
void orc_error_norms_f32(const float* ref, const float* got, int64_t n, double* out);

/* post-hoc fused op on canonical NKPQ (harness.cpp apply_op_canonical):
 * kind 0 RELU, 1 BIAS_ADD, 2 BIAS_RELU (kernel_streams.hpp:29) */
void orc_apply_op_canonical(float* out, int n, int k, int p, int q, int kind, const float* bias);

#ifdef __cplusplus
}
#endif
#endif
