/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for dconv-b200 (see oracle.h).
 * Restates /root/reference/proj/core (arxiv 1808.05567 artifact) in C.
 * Each function cites the reference file:line it follows.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ descriptor */

/* layer_spec.cpp:7-18 */
int orc_validate(const orc_spec* s) {
  if (s->N < 1 || s->C < 1 || s->K < 1 || s->H < 1 || s->W < 1 || s->R < 1 || s->S < 1) return 2;
  if (s->stride < 1) return 2;
  if (s->pad_h < 0 || s->pad_w < 0) return 2;
  if (s->vlen < 1) return 2;
  if (s->R > s->H + 2 * s->pad_h || s->S > s->W + 2 * s->pad_w) return 1;
  return 0;
}

/* layer_spec.cpp:45-51: floor division of the padded span */
int orc_output_shape(const orc_spec* s, int* P, int* Q) {
  int st = orc_validate(s);
  if (st) return st;
  *P = (s->H + 2 * s->pad_h - s->R) / s->stride + 1;
  *Q = (s->W + 2 * s->pad_w - s->S) / s->stride + 1;
  return 0;
}

/* layer_spec.cpp:20-43; pad_h/pad_w < 0 selects the "same" default
 * (R-1)/2 for odd R (0 for even), independently per axis */
int orc_make_spec(int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h, int pad_w, int vlen,
                  orc_spec* out) {
  if (pad_h < 0) pad_h = (R % 2 == 1) ? (R - 1) / 2 : 0;
  if (pad_w < 0) pad_w = (S % 2 == 1) ? (S - 1) / 2 : 0;
  orc_spec s = {N, C, K, H, W, R, S, stride, pad_h, pad_w, vlen};
  *out = s;
  return orc_validate(&s);
}

/* harness.cpp:269-272: 2*N*K*C*P*Q*R*S with logical C */
int64_t orc_pass_flops(const orc_spec* s) {
  int P, Q;
  if (orc_output_shape(s, &P, &Q)) return -1;
  return 2LL * s->N * s->K * s->C * P * Q * s->R * s->S;
}

/* ------------------------------------------------------------ generator */

/* util.hpp:46-52 */
uint64_t orc_splitmix_next(uint64_t* state) {
  *state += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* util.hpp:55-57 next_f32 (uniform in [-0.5, 0.5]); harness.cpp:274-278 */
void orc_random_f32(uint64_t seed, float* out, int64_t n) {
  uint64_t st = seed;
  for (int64_t i = 0; i < n; ++i)
    out[i] = (float)(orc_splitmix_next(&st) >> 40) * (1.0f / 16777216.0f) - 0.5f;
}

/* uniform(lo, hi) on the same 24-bit draw: lo + (hi-lo) * u, u in [0,1) */
void orc_uniform(uint64_t seed, float lo, float hi, float* out, int64_t n) {
  uint64_t st = seed;
  for (int64_t i = 0; i < n; ++i) {
    const float u = (float)(orc_splitmix_next(&st) >> 40) * (1.0f / 16777216.0f);
    out[i] = lo + (hi - lo) * u;
  }
}

/* He-normal N(0, stddev): one Box-Muller cosine branch per pair of draws */
void orc_he_normal(uint64_t seed, float stddev, float* out, int64_t n) {
  uint64_t st = seed;
  const double two_pi = 6.283185307179586476925286766559;
  for (int64_t i = 0; i < n; ++i) {
    const double u1 = (double)((orc_splitmix_next(&st) >> 11) + 1) * (1.0 / 9007199254740992.0);
    const double u2 = (double)(orc_splitmix_next(&st) >> 11) * (1.0 / 9007199254740992.0);
    const double z = sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
    out[i] = (float)(z * (double)stddev);
  }
}

/* ------------------------------------------------------------ naive oracles */

typedef struct {
  const orc_spec* s;
  const void* a;
  const void* b;
  void* out;
  int lo, hi; /* range of the parallel index */
  int dbl;    /* 1 = f64 in/out */
} job_t;

static double ld(const void* p, int dbl, int64_t i) {
  return dbl ? ((const double*)p)[i] : (double)((const float*)p)[i];
}

/* reference.cpp:7-33 forward_loops: per output element the order is c, r, s */
static void* fwd_job(void* arg) {
  job_t* j = (job_t*)arg;
  const orc_spec* s = j->s;
  int P, Q;
  orc_output_shape(s, &P, &Q);
  for (int n = j->lo; n < j->hi; ++n)
    for (int k = 0; k < s->K; ++k)
      for (int oj = 0; oj < P; ++oj)
        for (int oi = 0; oi < Q; ++oi) {
          const int ij = s->stride * oj - s->pad_h;
          const int ii = s->stride * oi - s->pad_w;
          double acc = 0.0;
          for (int c = 0; c < s->C; ++c)
            for (int r = 0; r < s->R; ++r)
              for (int q = 0; q < s->S; ++q) {
                const int y = ij + r, x = ii + q;
                if (y < 0 || y >= s->H || x < 0 || x >= s->W) continue;
                acc += ld(j->a, j->dbl, (((int64_t)n * s->C + c) * s->H + y) * s->W + x) *
                       ld(j->b, j->dbl, (((int64_t)k * s->C + c) * s->R + r) * s->S + q);
              }
          const int64_t o = (((int64_t)n * s->K + k) * P + oj) * Q + oi;
          if (j->dbl)
            ((double*)j->out)[o] = acc;
          else
            ((float*)j->out)[o] = (float)acc;
        }
  return NULL;
}

/* reference.cpp:35-65 backward_loops: per dI element the order is
 * k, then (oj, oi, r, s) lexicographic; f64 accumulator */
static void* bwd_job(void* arg) {
  job_t* j = (job_t*)arg;
  const orc_spec* s = j->s;
  int P, Q;
  orc_output_shape(s, &P, &Q);
  const int64_t plane = (int64_t)s->C * s->H * s->W;
  double* acc = (double*)calloc((size_t)plane, sizeof(double));
  for (int n = j->lo; n < j->hi; ++n) {
    memset(acc, 0, (size_t)plane * sizeof(double));
    for (int k = 0; k < s->K; ++k)
      for (int c = 0; c < s->C; ++c)
        for (int oj = 0; oj < P; ++oj)
          for (int oi = 0; oi < Q; ++oi) {
            const int ij = s->stride * oj - s->pad_h;
            const int ii = s->stride * oi - s->pad_w;
            const double g = ld(j->a, j->dbl, (((int64_t)n * s->K + k) * P + oj) * Q + oi);
            for (int r = 0; r < s->R; ++r)
              for (int q = 0; q < s->S; ++q) {
                const int y = ij + r, x = ii + q;
                if (y < 0 || y >= s->H || x < 0 || x >= s->W) continue;
                acc[((int64_t)c * s->H + y) * s->W + x] +=
                    g * ld(j->b, j->dbl, (((int64_t)k * s->C + c) * s->R + r) * s->S + q);
              }
          }
    for (int64_t e = 0; e < plane; ++e) {
      if (j->dbl)
        ((double*)j->out)[(int64_t)n * plane + e] = acc[e];
      else
        ((float*)j->out)[(int64_t)n * plane + e] = (float)acc[e];
    }
  }
  free(acc);
  return NULL;
}

/* reference.cpp:67-95 update_loops: per dW element the order is
 * n, then (oj, oi) lexicographic; parallel over k only */
static void* upd_job(void* arg) {
  job_t* j = (job_t*)arg;
  const orc_spec* s = j->s;
  int P, Q;
  orc_output_shape(s, &P, &Q);
  const int64_t crs = (int64_t)s->C * s->R * s->S;
  double* acc = (double*)calloc((size_t)crs, sizeof(double));
  for (int k = j->lo; k < j->hi; ++k) {
    memset(acc, 0, (size_t)crs * sizeof(double));
    for (int n = 0; n < s->N; ++n)
      for (int c = 0; c < s->C; ++c)
        for (int oj = 0; oj < P; ++oj)
          for (int oi = 0; oi < Q; ++oi) {
            const int ij = s->stride * oj - s->pad_h;
            const int ii = s->stride * oi - s->pad_w;
            const double g = ld(j->b, j->dbl, (((int64_t)n * s->K + k) * P + oj) * Q + oi);
            for (int r = 0; r < s->R; ++r)
              for (int q = 0; q < s->S; ++q) {
                const int y = ij + r, x = ii + q;
                if (y < 0 || y >= s->H || x < 0 || x >= s->W) continue;
                acc[((int64_t)c * s->R + r) * s->S + q] +=
                    ld(j->a, j->dbl, (((int64_t)n * s->C + c) * s->H + y) * s->W + x) * g;
              }
          }
    for (int64_t e = 0; e < crs; ++e) {
      if (j->dbl)
        ((double*)j->out)[(int64_t)k * crs + e] = acc[e];
      else
        ((float*)j->out)[(int64_t)k * crs + e] = (float)acc[e];
    }
  }
  free(acc);
  return NULL;
}

static int run_jobs(const orc_spec* s, void* (*fn)(void*), const void* a, const void* b, void* out, int extent,
                    int threads, int dbl) {
  int st = orc_validate(s);
  if (st) return st;
  if (threads < 1) threads = 1;
  if (threads > extent) threads = extent;
  job_t* jobs = (job_t*)calloc((size_t)threads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    /* util.hpp:112-117 split_range */
    const int base = extent / threads, rem = extent % threads;
    const int lo = t * base + (t < rem ? t : rem);
    jobs[t].s = s;
    jobs[t].a = a;
    jobs[t].b = b;
    jobs[t].out = out;
    jobs[t].lo = lo;
    jobs[t].hi = lo + base + (t < rem ? 1 : 0);
    jobs[t].dbl = dbl;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, fn, &jobs[t]);
  fn(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  free(jobs);
  free(th);
  return 0;
}

int orc_conv_forward(const orc_spec* s, const float* in, const float* wt, float* out, int threads) {
  return run_jobs(s, fwd_job, in, wt, out, s->N, threads, 0);
}
int orc_conv_backward(const orc_spec* s, const float* grad_out, const float* wt, float* grad_in, int threads) {
  return run_jobs(s, bwd_job, grad_out, wt, grad_in, s->N, threads, 0);
}
int orc_conv_update(const orc_spec* s, const float* in, const float* grad_out, float* grad_w, int threads) {
  return run_jobs(s, upd_job, in, grad_out, grad_w, s->K, threads, 0);
}
int orc_conv_forward_f64(const orc_spec* s, const double* in, const double* wt, double* out) {
  return run_jobs(s, fwd_job, in, wt, out, s->N, 1, 1);
}
int orc_conv_backward_f64(const orc_spec* s, const double* grad_out, const double* wt, double* grad_in) {
  return run_jobs(s, bwd_job, grad_out, wt, grad_in, s->N, 1, 1);
}
int orc_conv_update_f64(const orc_spec* s, const double* in, const double* grad_out, double* grad_w) {
  return run_jobs(s, upd_job, in, grad_out, grad_w, s->K, 1, 1);
}

/* ------------------------------------------------------------ blocked layouts */

static int cdiv(int a, int b) { return (a + b - 1) / b; }

/* blocked.hpp:29-34 storage extent */
int64_t orc_act_elems(int n, int c, int h, int w, int vlen, int halo_h, int halo_w) {
  return (int64_t)n * cdiv(c, vlen) * (h + 2 * halo_h) * (w + 2 * halo_w) * vlen;
}
int64_t orc_wt_elems(int k, int c, int r, int s, int vlen) {
  return (int64_t)cdiv(k, vlen) * cdiv(c, vlen) * r * s * vlen * vlen;
}

/* blocked.hpp:47-51 offset(img, block, ph, pw) */
static int64_t act_off(int c, int h, int w, int vlen, int hh, int hw, int img, int blk, int ph, int pw) {
  const int cb = cdiv(c, vlen), hp = h + 2 * hh, wp = w + 2 * hw;
  return ((((int64_t)img * cb + blk) * hp + ph) * wp + pw) * vlen;
}

/* blocked.hpp:133-155 to_blocked_activation: halo and tail lanes are zero */
void orc_to_blocked_act(const float* nchw, int n, int c, int h, int w, int vlen, int halo_h, int halo_w, float* out) {
  memset(out, 0, (size_t)orc_act_elems(n, c, h, w, vlen, halo_h, halo_w) * sizeof(float));
  for (int img = 0; img < n; ++img)
    for (int ch = 0; ch < c; ++ch)
      for (int y = 0; y < h; ++y) {
        float* lane = out + act_off(c, h, w, vlen, halo_h, halo_w, img, ch / vlen, y + halo_h, halo_w) + ch % vlen;
        for (int x = 0; x < w; ++x) lane[(int64_t)x * vlen] = nchw[(((int64_t)img * c + ch) * h + y) * w + x];
      }
}

/* blocked.hpp:157-178 from_blocked_activation (interior only) */
void orc_from_blocked_act(const float* blk, int n, int c, int h, int w, int vlen, int halo_h, int halo_w,
                          float* nchw) {
  for (int img = 0; img < n; ++img)
    for (int ch = 0; ch < c; ++ch)
      for (int y = 0; y < h; ++y) {
        const float* lane =
            blk + act_off(c, h, w, vlen, halo_h, halo_w, img, ch / vlen, y + halo_h, halo_w) + ch % vlen;
        for (int x = 0; x < w; ++x) nchw[(((int64_t)img * c + ch) * h + y) * w + x] = lane[(int64_t)x * vlen];
      }
}

/* blocked.hpp:112-115 offset(kblk, cblk, r, s) */
static int64_t wt_off(int k, int c, int r, int s, int vlen, int kb, int cb, int fr, int fs) {
  const int cbs = cdiv(c, vlen);
  (void)k;
  return ((((int64_t)kb * cbs + cb) * r + fr) * s + fs) * vlen * vlen;
}

/* blocked.hpp:180-200 to_blocked_weight: lane [c%v * v + k%v] */
void orc_to_blocked_wt(const float* kcrs, int k, int c, int r, int s, int vlen, float* out) {
  memset(out, 0, (size_t)orc_wt_elems(k, c, r, s, vlen) * sizeof(float));
  for (int ko = 0; ko < k; ++ko)
    for (int ci = 0; ci < c; ++ci)
      for (int fr = 0; fr < r; ++fr)
        for (int fs = 0; fs < s; ++fs)
          out[wt_off(k, c, r, s, vlen, ko / vlen, ci / vlen, fr, fs) + (ci % vlen) * vlen + ko % vlen] =
              kcrs[(((int64_t)ko * c + ci) * r + fr) * s + fs];
}

/* blocked.hpp:202-213 from_blocked_weight */
void orc_from_blocked_wt(const float* blk, int k, int c, int r, int s, int vlen, float* kcrs) {
  for (int ko = 0; ko < k; ++ko)
    for (int ci = 0; ci < c; ++ci)
      for (int fr = 0; fr < r; ++fr)
        for (int fs = 0; fs < s; ++fs)
          kcrs[(((int64_t)ko * c + ci) * r + fr) * s + fs] =
              blk[wt_off(k, c, r, s, vlen, ko / vlen, ci / vlen, fr, fs) + (ci % vlen) * vlen + ko % vlen];
}

/* propagation.hpp:20-33 transform_weight_stride1:
 * W'[c_b][k_b][r'][s'][k][c] = W[k_b][c_b][R-1-r'][S-1-s'][c][k] */
void orc_transform_weight_stride1(const float* blk, int k, int c, int r, int s, int vlen, float* out) {
  memset(out, 0, (size_t)orc_wt_elems(c, k, r, s, vlen) * sizeof(float));
  for (int ko = 0; ko < k; ++ko)
    for (int ci = 0; ci < c; ++ci)
      for (int fr = 0; fr < r; ++fr)
        for (int fs = 0; fs < s; ++fs)
          out[wt_off(c, k, r, s, vlen, ci / vlen, ko / vlen, fr, fs) + (ko % vlen) * vlen + ci % vlen] =
              blk[wt_off(k, c, r, s, vlen, ko / vlen, ci / vlen, r - 1 - fr, s - 1 - fs) + (ci % vlen) * vlen +
                  ko % vlen];
}

/* ------------------------------------------------------------ norms */

/* norms.cpp:7-25 error_norms_span (f64 arithmetic) */
void orc_error_norms_f32(const float* ref, const float* got, int64_t n, double* out) {
  double max_diff = 0.0, max_ref = 0.0, sq_diff = 0.0, sq_ref = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double r = (double)ref[i], g = (double)got[i];
    const double d = fabs(r - g);
    const double a = fabs(r);
    if (d > max_diff) max_diff = d;
    if (a > max_ref) max_ref = a;
    sq_diff += d * d;
    sq_ref += r * r;
  }
  out[0] = max_diff;
  out[1] = sqrt(sq_diff);
  out[2] = max_ref > 0.0 ? max_diff / max_ref : max_diff;
  const double ref_l2 = sqrt(sq_ref);
  out[3] = ref_l2 > 0.0 ? out[1] / ref_l2 : out[1];
}

/* harness.cpp apply_op_canonical (post-hoc RELU / BIAS_ADD / BIAS_RELU) */
void orc_apply_op_canonical(float* out, int n, int k, int p, int q, int kind, const float* bias) {
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < k; ++b)
      for (int y = 0; y < p; ++y)
        for (int x = 0; x < q; ++x) {
          float* v = out + (((int64_t)a * k + b) * p + y) * q + x;
          float t = *v;
          if (kind != 0) t += bias[b];
          if (kind != 1) t = t > 0.0f ? t : 0.0f;
          *v = t;
        }
}
