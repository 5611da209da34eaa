// Blocked-layout data movement on the device (HBM-bound; bitwise moves):
//  * pack / unpack NCHW <-> NCHW{v}c with physical zero halo   (blocked.hpp:133-178)
//  * pack / unpack KCRS <-> KCRS{v}c{v}k                        (blocked.hpp:180-213)
//  * dual weight transform W'[c_b][k_b][R-1-r][S-1-s][k][c]     (propagation.hpp:20-33)
//  * re-halo copy                                               (propagation.hpp:35-49)
//  * weight prep: blocked weights -> bf16 piece layout read by the tcgen05
//    kernels' weight TMA ([piece*Cb_in + cb][tap][2*Kb_out][16][8])
// Grid-stride loops over the DESTINATION so every element (halo and tail
// lanes included) is written exactly once: no separate memset.
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

namespace dconv_sm100 {

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

#define DCONV_GRID_STRIDE(i, total) \
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < (total); \
       i += static_cast<long long>(gridDim.x) * blockDim.x)

// NCHW (S) -> blocked (D); dst element e = ((((n*cb + b)*hp + y)*wp + x)*v + lane)
template <typename S, typename D>
__global__ void pack_act_kernel(const S* __restrict__ src, D* __restrict__ dst, int n, int c, int h, int w, int v,
                                int hh, int hw) {
  const int cb = (c + v - 1) / v, hp = h + 2 * hh, wp = w + 2 * hw;
  const long long total = static_cast<long long>(n) * cb * hp * wp * v;
  DCONV_GRID_STRIDE(e, total) {
    const int lane = static_cast<int>(e % v);
    long long r = e / v;
    const int x = static_cast<int>(r % wp) - hw;
    r /= wp;
    const int y = static_cast<int>(r % hp) - hh;
    r /= hp;
    const int b = static_cast<int>(r % cb);
    const int img = static_cast<int>(r / cb);
    const int ch = b * v + lane;
    float val = 0.0f;
    if (ch < c && y >= 0 && y < h && x >= 0 && x < w)
      val = to_f<S>(src[((static_cast<long long>(img) * c + ch) * h + y) * w + x]);
    dst[e] = from_f<D>(val);
  }
}

// 16 consecutive lanes of one blocked pixel
template <typename T>
struct Lanes16;
template <>
struct Lanes16<float> {
  static __device__ __forceinline__ void store(float* dst, const float (&v)[16]) {
    float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  }
  static __device__ __forceinline__ void load(const float* src, float (&v)[16]) {
    const float4* s = reinterpret_cast<const float4*>(src);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 t = s[i];
      v[4 * i] = t.x, v[4 * i + 1] = t.y, v[4 * i + 2] = t.z, v[4 * i + 3] = t.w;
    }
  }
};
template <>
struct Lanes16<__nv_bfloat16> {
  static __device__ __forceinline__ void store(__nv_bfloat16* dst, const float (&v)[16]) {
    uint4* d = reinterpret_cast<uint4*>(dst);
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const __nv_bfloat162 b = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
      w[i] = *reinterpret_cast<const uint32_t*>(&b);
    }
    d[0] = make_uint4(w[0], w[1], w[2], w[3]);
    d[1] = make_uint4(w[4], w[5], w[6], w[7]);
  }
  static __device__ __forceinline__ void load(const __nv_bfloat16* src, float (&v)[16]) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    const uint4 a = s[0], b = s[1];
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
};

// vlen 16: one thread per destination PIXEL (all 16 lanes). The 16 channel reads
// are coalesced across the warp (consecutive x), the 64 / 32 B lane row is written
// with 16 B vector stores (a warp writes one contiguous 2 / 1 KB run); halo pixels
// and tail lanes are written as zeros. Bitwise equal to pack_act_kernel.
template <typename S, typename D>
__global__ void __launch_bounds__(256) pack_act16_kernel(const S* __restrict__ src, D* __restrict__ dst, int n, int c,
                                                         int h, int w, int hh, int hw) {
  const int cb = (c + 15) / 16, hp = h + 2 * hh, wp = w + 2 * hw;
  const long long total = static_cast<long long>(n) * cb * hp * wp;
  const long long plane = static_cast<long long>(h) * w;
  DCONV_GRID_STRIDE(e, total) {
    long long r = e;
    const int x = static_cast<int>(r % wp) - hw;
    r /= wp;
    const int y = static_cast<int>(r % hp) - hh;
    r /= hp;
    const int b = static_cast<int>(r % cb);
    const int img = static_cast<int>(r / cb);
    float v[16];
    const bool in = y >= 0 && y < h && x >= 0 && x < w;
    const S* sp = src + ((static_cast<long long>(img) * c + b * 16) * h + (in ? y : 0)) * w + (in ? x : 0);
#pragma unroll
    for (int l = 0; l < 16; ++l) v[l] = (in && b * 16 + l < c) ? to_f<S>(sp[l * plane]) : 0.0f;
    Lanes16<D>::store(dst + e * 16, v);
  }
}

// vlen 16: one thread per interior pixel: 16 B vector loads of the lane row, 16
// channel writes coalesced across the warp
template <typename S, typename D>
__global__ void __launch_bounds__(256) unpack_act16_kernel(const S* __restrict__ src, D* __restrict__ dst, int n, int c,
                                                           int h, int w, int hh, int hw) {
  const int cb = (c + 15) / 16, hp = h + 2 * hh, wp = w + 2 * hw;
  const long long total = static_cast<long long>(n) * cb * h * w;
  const long long plane = static_cast<long long>(h) * w;
  DCONV_GRID_STRIDE(e, total) {
    long long r = e;
    const int x = static_cast<int>(r % w);
    r /= w;
    const int y = static_cast<int>(r % h);
    r /= h;
    const int b = static_cast<int>(r % cb);
    const int img = static_cast<int>(r / cb);
    float v[16];
    Lanes16<S>::load(src + ((((static_cast<long long>(img) * cb + b) * hp + y + hh) * wp) + x + hw) * 16, v);
    D* dp = dst + ((static_cast<long long>(img) * c + b * 16) * h + y) * w + x;
#pragma unroll
    for (int l = 0; l < 16; ++l)
      if (b * 16 + l < c) dp[l * plane] = from_f<D>(v[l]);
  }
}

// blocked (S) -> NCHW (D), interior only
template <typename S, typename D>
__global__ void unpack_act_kernel(const S* __restrict__ src, D* __restrict__ dst, int n, int c, int h, int w, int v,
                                  int hh, int hw) {
  const int cb = (c + v - 1) / v, hp = h + 2 * hh, wp = w + 2 * hw;
  const long long total = static_cast<long long>(n) * c * h * w;
  DCONV_GRID_STRIDE(e, total) {
    const int x = static_cast<int>(e % w);
    long long r = e / w;
    const int y = static_cast<int>(r % h);
    r /= h;
    const int ch = static_cast<int>(r % c);
    const int img = static_cast<int>(r / c);
    const long long so = ((((static_cast<long long>(img) * cb + ch / v) * hp + y + hh) * wp) + x + hw) * v + ch % v;
    dst[e] = from_f<D>(to_f<S>(src[so]));
  }
}

// KCRS -> blocked [kb][cb][r][s][c][k]
template <typename S, typename D>
__global__ void pack_wt_kernel(const S* __restrict__ src, D* __restrict__ dst, int k, int c, int r, int s, int v) {
  const int kb = (k + v - 1) / v, cb = (c + v - 1) / v;
  const long long total = static_cast<long long>(kb) * cb * r * s * v * v;
  DCONV_GRID_STRIDE(e, total) {
    const int kl = static_cast<int>(e % v);
    const int cl = static_cast<int>((e / v) % v);
    long long q = e / (static_cast<long long>(v) * v);
    const int fs = static_cast<int>(q % s);
    q /= s;
    const int fr = static_cast<int>(q % r);
    q /= r;
    const int cbi = static_cast<int>(q % cb);
    const int kbi = static_cast<int>(q / cb);
    const int ko = kbi * v + kl, ci = cbi * v + cl;
    float val = 0.0f;
    if (ko < k && ci < c) val = to_f<S>(src[((static_cast<long long>(ko) * c + ci) * r + fr) * s + fs]);
    dst[e] = from_f<D>(val);
  }
}

template <typename S, typename D>
__global__ void unpack_wt_kernel(const S* __restrict__ src, D* __restrict__ dst, int k, int c, int r, int s, int v) {
  const int cb = (c + v - 1) / v;
  const long long total = static_cast<long long>(k) * c * r * s;
  DCONV_GRID_STRIDE(e, total) {
    const int fs = static_cast<int>(e % s);
    long long q = e / s;
    const int fr = static_cast<int>(q % r);
    q /= r;
    const int ci = static_cast<int>(q % c);
    const int ko = static_cast<int>(q / c);
    const long long so =
        ((((static_cast<long long>(ko / v) * cb + ci / v) * r + fr) * s + fs) * v + ci % v) * v + ko % v;
    dst[e] = from_f<D>(to_f<S>(src[so]));
  }
}

// blocked(vs, halo shh/shw) -> blocked(vd, halo dhh/dhw), same channels / extents:
// the internal re-blocking of vlen != 16 tensors for the 16-lane tensor-core passes.
// Destination halo and tail lanes are written as zeros; accumulate adds into dst
// (interior lanes) instead of overwriting.
template <typename T>
__global__ void reblock_act_kernel(const T* __restrict__ src, T* __restrict__ dst, int n, int c, int h, int w, int vs,
                                   int shh, int shw, int vd, int dhh, int dhw, int accumulate) {
  const int cbs = (c + vs - 1) / vs, cbd = (c + vd - 1) / vd;
  const int shp = h + 2 * shh, swp = w + 2 * shw, dhp = h + 2 * dhh, dwp = w + 2 * dhw;
  const long long total = static_cast<long long>(n) * cbd * dhp * dwp * vd;
  DCONV_GRID_STRIDE(e, total) {
    const int lane = static_cast<int>(e % vd);
    long long r = e / vd;
    const int x = static_cast<int>(r % dwp) - dhw;
    r /= dwp;
    const int y = static_cast<int>(r % dhp) - dhh;
    r /= dhp;
    const int b = static_cast<int>(r % cbd);
    const int img = static_cast<int>(r / cbd);
    const int ch = b * vd + lane;
    const bool live = ch < c && y >= 0 && y < h && x >= 0 && x < w;
    float val = 0.0f;
    if (live)
      val = to_f<T>(src[((((static_cast<long long>(img) * cbs + ch / vs) * shp + y + shh) * swp) + x + shw) * vs +
                        ch % vs]);
    if (accumulate && live) val += to_f<T>(dst[e]);
    dst[e] = from_f<T>(val);
  }
}

// [kb][cb][r][s][c][k] at vs -> at vd (tail lanes zero); accumulate adds into dst
template <typename T>
__global__ void reblock_wt_kernel(const T* __restrict__ src, T* __restrict__ dst, int k, int c, int r, int s, int vs,
                                  int vd, int accumulate) {
  const int kbs = (k + vs - 1) / vs, cbs = (c + vs - 1) / vs, kbd = (k + vd - 1) / vd, cbd = (c + vd - 1) / vd;
  (void)kbs;
  const long long total = static_cast<long long>(kbd) * cbd * r * s * vd * vd;
  DCONV_GRID_STRIDE(e, total) {
    const int kl = static_cast<int>(e % vd);
    const int cl = static_cast<int>((e / vd) % vd);
    long long q = e / (static_cast<long long>(vd) * vd);
    const int fs = static_cast<int>(q % s);
    q /= s;
    const int fr = static_cast<int>(q % r);
    q /= r;
    const int cbi = static_cast<int>(q % cbd);
    const int kbi = static_cast<int>(q / cbd);
    const int ko = kbi * vd + kl, ci = cbi * vd + cl;
    const bool live = ko < k && ci < c;
    float val = 0.0f;
    if (live)
      val = to_f<T>(src[((((static_cast<long long>(ko / vs) * cbs + ci / vs) * r + fr) * s + fs) * vs + ci % vs) * vs +
                        ko % vs]);
    if (accumulate && live) val += to_f<T>(dst[e]);
    dst[e] = from_f<T>(val);
  }
}

// dual weights: out (k<->c roles swapped) [cb'=k_b... ] as transform_weight_stride1
template <typename T>
__global__ void dual_wt_kernel(const T* __restrict__ src, T* __restrict__ dst, int k, int c, int r, int s, int v) {
  // dst is a blocked weight with (k' = c, c' = k)
  const int kb2 = (c + v - 1) / v, cb2 = (k + v - 1) / v;  // dst blocks
  const int cb = (c + v - 1) / v;                          // src c blocks
  const long long total = static_cast<long long>(kb2) * cb2 * r * s * v * v;
  DCONV_GRID_STRIDE(e, total) {
    const int kl = static_cast<int>(e % v);         // dst k lane = src c lane
    const int cl = static_cast<int>((e / v) % v);   // dst c lane = src k lane
    long long q = e / (static_cast<long long>(v) * v);
    const int fs = static_cast<int>(q % s);
    q /= s;
    const int fr = static_cast<int>(q % r);
    q /= r;
    const int b_c2 = static_cast<int>(q % cb2);     // dst c block = src k block
    const int b_k2 = static_cast<int>(q / cb2);     // dst k block = src c block
    const int ko = b_c2 * v + cl, ci = b_k2 * v + kl;  // src (k, c)
    T val = from_f<T>(0.0f);
    if (ko < k && ci < c) {
      const long long so =
          ((((static_cast<long long>(b_c2) * cb + b_k2) * r + (r - 1 - fr)) * s + (s - 1 - fs)) * v + kl) * v + cl;
      val = src[so];
    }
    dst[e] = val;
  }
}

// copy interior into a tensor with a different halo; the new halo is zeroed
template <typename T>
__global__ void rehalo_kernel(const T* __restrict__ src, T* __restrict__ dst, int n, int cb, int h, int w, int v,
                              int sh, int sw, int dh, int dw) {
  const int hp = h + 2 * dh, wp = w + 2 * dw;
  const int shp = h + 2 * sh, swp = w + 2 * sw;
  const long long total = static_cast<long long>(n) * cb * hp * wp * v;
  DCONV_GRID_STRIDE(e, total) {
    const int lane = static_cast<int>(e % v);
    long long q = e / v;
    const int x = static_cast<int>(q % wp) - dw;
    q /= wp;
    const int y = static_cast<int>(q % hp) - dh;
    const long long plane = q / hp;
    T val = from_f<T>(0.0f);
    if (y >= 0 && y < h && x >= 0 && x < w) val = src[((plane * shp + y + sh) * swp + x + sw) * v + lane];
    dst[e] = val;
  }
}

// Weight prep for the tcgen05 kernels (vlen 16). dst layout (bf16):
//   [pc][cbi][ntile][t][ng][ci(16)][kk(8)],  ng = 2*nb groups of 8 output lanes per tile
// out channel o = (ntile*nb + ng/2)*16 + (ng%2)*8 + kk, in channel i = cbi*16 + ci; every
// (pc, cbi, ntile, phase) slice is contiguous so the kernel stages it with one bulk copy.
// tapmap[t] = source tap r*S+s (or -1 for an all-zero tap).
// dual = 0: out = k, in = c (forward). dual = 1: out = c, in = k (backward-data).
// pieces = 3 stores the exact hi/mid/lo bf16 split of each fp32 weight.
// one thread's share of a weight prep: the 8 output lanes (kk = 0..7, one 16 B store
// per piece) of prepared element group e8, 32-bit indices (host-checked: a piece has
// < 2^31 elements)
template <typename S>
__device__ __forceinline__ void weight_prep8(const S* __restrict__ src, __nv_bfloat16* __restrict__ dst, int kb_src,
                                             int cb_src, int rs_src, const int* __restrict__ tapmap, int n_taps,
                                             int cb_in, int nb, int n_ntiles, int dual, int pieces, int nt_major,
                                             int n8, int e8) {
  const int ci = e8 % 16;
  int q = e8 / 16;
  const int ng = q % (2 * nb);
  q /= (2 * nb);
  const int t = q % n_taps;
  q /= n_taps;
  // nt_major: [piece][n_tile][c_b][tap][2nb][16][8] -- one n-tile's channel blocks are
  // contiguous, so a streamed stage's kc blocks (all taps) are ONE bulk copy. Otherwise
  // [piece][c_b][n_tile][tap][..] (the fp32-activation plans keep the original layout)
  const int cbi = nt_major ? q % cb_in : q / n_ntiles;
  const int nt = nt_major ? q / cb_in : q % n_ntiles;
  const int ob = nt * nb + ng / 2, ol0 = (ng % 2) * 8;  // out block / first lane
  const int rs = tapmap[t];
  float val[8];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) val[kk] = 0.0f;
  // blocked src [kb][cb][rs][c lane][k lane]
  const int kb = dual ? cbi : ob, cb = dual ? ob : cbi;
  if (rs >= 0 && kb < kb_src && cb < cb_src) {
    const S* row = src + ((static_cast<long long>(kb) * cb_src + cb) * rs_src + rs) * 256;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk)  // forward: 8 consecutive k lanes; backward-data: 8 c lanes (stride 16)
      val[kk] = to_f<S>(dual ? row[(ol0 + kk) * 16 + ci] : row[ci * 16 + ol0 + kk]);
  }
  __align__(16) __nv_bfloat16 h[8];
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) h[kk] = __float2bfloat16_rn(val[kk]);
  uint4* d = reinterpret_cast<uint4*>(dst) + e8;
  *d = *reinterpret_cast<const uint4*>(h);
  if (pieces == 3) {
    __align__(16) __nv_bfloat16 m[8], l[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const float r1 = val[kk] - __bfloat162float(h[kk]);
      m[kk] = __float2bfloat16_rn(r1);
      l[kk] = __float2bfloat16_rn(r1 - __bfloat162float(m[kk]));
    }
    d[n8] = *reinterpret_cast<const uint4*>(m);
    d[2 * n8] = *reinterpret_cast<const uint4*>(l);
  }
}

template <typename S>
__global__ void weight_prep_kernel(const S* __restrict__ src, __nv_bfloat16* __restrict__ dst, int kb_src,
                                   int cb_src, int rs_src, const int* __restrict__ tapmap, int n_taps, int cb_in,
                                   int nb, int n_ntiles, int dual, int pieces, int nt_major) {
  // the conv kernel launched after this one (programmatic dependent launch) may
  // start its prologue and activation loads now; it waits before reading weights
  pdl_launch_dependents();
  const int n8 = cb_in * n_ntiles * n_taps * (2 * nb) * 16;
  for (int e8 = blockIdx.x * blockDim.x + threadIdx.x; e8 < n8; e8 += gridDim.x * blockDim.x)
    weight_prep8(src, dst, kb_src, cb_src, rs_src, tapmap, n_taps, cb_in, nb, n_ntiles, dual, pieces, nt_major, n8,
                 e8);
}

// Batched weight prep (dconv_prep_batch_*): many convs' preparations in one launch.
// The job table travels as a kernel parameter (graph-capturable, no device table);
// job j owns the element groups [off8, off8 + n8) of the launch.
struct PrepJob {
  const void* src;
  void* dst;
  const int* tapmap;
  int src_bf16, kb_src, cb_src, rs_src, n_taps, cb_in, nb, n_ntiles, dual, pieces, nt_major, n8, off8;
};
constexpr int kPrepBatchMax = 128;  // ~10 KB of kernel parameters (CUDA >= 12.1: up to 32 KB)
struct PrepBatch {
  int n_jobs, total8;
  PrepJob job[kPrepBatchMax];
};

__global__ void __launch_bounds__(256) weight_prep_batch_kernel(const __grid_constant__ PrepBatch b) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < b.total8; g += gridDim.x * blockDim.x) {
    int lo = 0, hi = b.n_jobs - 1;  // last job with off8 <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (b.job[mid].off8 <= g) lo = mid;
      else hi = mid - 1;
    }
    const PrepJob& j = b.job[lo];
    const int e8 = g - j.off8;
    if (j.src_bf16)
      weight_prep8(static_cast<const __nv_bfloat16*>(j.src), static_cast<__nv_bfloat16*>(j.dst), j.kb_src, j.cb_src,
                   j.rs_src, j.tapmap, j.n_taps, j.cb_in, j.nb, j.n_ntiles, j.dual, j.pieces, j.nt_major, j.n8, e8);
    else
      weight_prep8(static_cast<const float*>(j.src), static_cast<__nv_bfloat16*>(j.dst), j.kb_src, j.cb_src, j.rs_src,
                   j.tapmap, j.n_taps, j.cb_in, j.nb, j.n_ntiles, j.dual, j.pieces, j.nt_major, j.n8, e8);
  }
}

// zero one phase lattice (a, b) of a blocked tensor's interior: rows a + st*y, cols b + st*x
template <typename T>
__global__ void zero_lattice_kernel(T* __restrict__ dst, int planes, int h, int w, int hp, int wp, int hh, int hw,
                                    int st, int a, int b) {
  const int ly = a < h ? (h - a + st - 1) / st : 0, lx = b < w ? (w - b + st - 1) / st : 0;
  const long long total = static_cast<long long>(planes) * ly * lx * 16;
  DCONV_GRID_STRIDE(e, total) {
    const int lane = static_cast<int>(e % 16);
    long long q = e / 16;
    const int x = static_cast<int>(q % lx);
    q /= lx;
    const int y = static_cast<int>(q % ly);
    const long long plane = q / ly;
    dst[((plane * hp + hh + a + st * y) * wp + hw + b + st * x) * 16 + lane] = from_f<T>(0.0f);
  }
}

// zero only the halo frame of a blocked tensor (blocked.hpp:67-79 zero_halo)
template <typename T>
__global__ void zero_halo_kernel(T* __restrict__ dst, int planes, int h, int w, int hh, int hw, int v) {
  const int hp = h + 2 * hh, wp = w + 2 * hw;
  const long long frame = static_cast<long long>(hp) * wp - static_cast<long long>(h) * w;
  const long long total = static_cast<long long>(planes) * frame * v;
  DCONV_GRID_STRIDE(e, total) {
    const int lane = static_cast<int>(e % v);
    long long q = e / v;
    const long long fi = q % frame;
    const long long plane = q / frame;
    int y, x;
    const long long top = static_cast<long long>(hh) * wp;
    if (fi < top) {
      y = static_cast<int>(fi / wp);
      x = static_cast<int>(fi % wp);
    } else if (fi < 2 * top) {
      y = hh + h + static_cast<int>((fi - top) / wp);
      x = static_cast<int>((fi - top) % wp);
    } else {
      const long long side = fi - 2 * top;  // h rows x (2*hw) columns
      y = hh + static_cast<int>(side / (2 * hw));
      const int cx = static_cast<int>(side % (2 * hw));
      x = cx < hw ? cx : w + cx;
    }
    dst[((plane * hp + y) * wp + x) * v + lane] = from_f<T>(0.0f);
  }
}

// 3x3 / stride-2 / pad-1 max pool on blocked tensors (ResNet stem), halo 0.
// Stores the argmax tap (0..8, first max in row-major order) for the backward.
// 16 lanes of one pixel-block <-> registers (bf16: two 16 B vectors, fp32: four)
template <typename T>
__device__ __forceinline__ void ld16f(const T* p, float (&v)[16]) {
  if constexpr (sizeof(T) == 2) {
    const uint4 a = reinterpret_cast<const uint4*>(p)[0], b = reinterpret_cast<const uint4*>(p)[1];
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      v[2 * e] = __uint_as_float(w[e] << 16);
      v[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
    }
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float4 t = reinterpret_cast<const float4*>(p)[e];
      v[4 * e] = t.x;
      v[4 * e + 1] = t.y;
      v[4 * e + 2] = t.z;
      v[4 * e + 3] = t.w;
    }
  }
}
template <typename T>
__device__ __forceinline__ void st16f(T* p, const float (&v)[16]) {
  if constexpr (sizeof(T) == 2) {
    uint32_t w[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
      w[e] = *reinterpret_cast<const uint32_t*>(&h);
    }
    reinterpret_cast<uint4*>(p)[0] = make_uint4(w[0], w[1], w[2], w[3]);
    reinterpret_cast<uint4*>(p)[1] = make_uint4(w[4], w[5], w[6], w[7]);
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e)
      reinterpret_cast<float4*>(p)[e] = make_float4(v[4 * e], v[4 * e + 1], v[4 * e + 2], v[4 * e + 3]);
  }
}

// 3x3 / stride 2 / pad 1 max-pool (the ResNet stem pool), one thread per output
// pixel-block (16 lanes); argmax = window position dy*3+dx of the first maximum
template <typename T>
__global__ void maxpool_fwd_kernel(const T* __restrict__ in, T* __restrict__ out, uint8_t* __restrict__ arg,
                                   int planes, int h, int w, int p, int q) {
  const long long total = static_cast<long long>(planes) * p * q;
  DCONV_GRID_STRIDE(e, total) {
    const int x = static_cast<int>(e % q);
    const long long r = e / q;
    const int y = static_cast<int>(r % p);
    const long long plane = r / p;
    float best[16], v[16];
    uint32_t bc[16];  // argmax code per lane (two selects per lane and tap; packed to bytes once)
#pragma unroll
    for (int l = 0; l < 16; ++l) {
      best[l] = -INFINITY;
      bc[l] = 0;
    }
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int iy = 2 * y - 1 + dy, ix = 2 * x - 1 + dx;
        if (iy < 0 || iy >= h || ix < 0 || ix >= w) continue;
        ld16f(in + ((plane * h + iy) * w + ix) * 16, v);
        const uint32_t code = static_cast<uint32_t>(dy * 3 + dx);
#pragma unroll
        for (int l = 0; l < 16; ++l) {
          const bool gt = v[l] > best[l];
          best[l] = gt ? v[l] : best[l];
          bc[l] = gt ? code : bc[l];
        }
      }
    st16f(out + e * 16, best);
    uint32_t bi[4];  // 16 argmax bytes
#pragma unroll
    for (int k = 0; k < 4; ++k) bi[k] = bc[4 * k] | (bc[4 * k + 1] << 8) | (bc[4 * k + 2] << 16) | (bc[4 * k + 3] << 24);
    reinterpret_cast<uint4*>(arg)[e] = make_uint4(bi[0], bi[1], bi[2], bi[3]);
  }
}

// gather form of the max-pool backward (deterministic, no atomics): each input
// pixel-block sums the output gradients of the <= 4 windows whose argmax it is
template <typename T>
// pmask (nullable, gout's geometry): the POOLED output as the ReLU mask. The
// argmax element of a window holds the window's max, so "input > 0" at the
// argmax equals "pooled output > 0": the same mask as `mask` at a quarter of
// the bytes (the pooled tensor instead of the full-resolution activation).
__global__ void maxpool_bwd_kernel(const T* __restrict__ gout, const uint8_t* __restrict__ arg,
                                   T* __restrict__ gin, const T* __restrict__ mask, int planes, int h, int w, int p,
                                   int q, const T* __restrict__ pmask = nullptr) {
  const long long total = static_cast<long long>(planes) * h * w;
  DCONV_GRID_STRIDE(e, total) {
    const int ix = static_cast<int>(e % w);
    const long long r = e / w;
    const int iy = static_cast<int>(r % h);
    const long long plane = r / h;
    float acc[16], g[16];
#pragma unroll
    for (int l = 0; l < 16; ++l) acc[l] = 0.0f;
    for (int y = (iy + 1) / 2 - 1; y <= (iy + 1) / 2; ++y)
      for (int x = (ix + 1) / 2 - 1; x <= (ix + 1) / 2; ++x) {
        if (y < 0 || y >= p || x < 0 || x >= q) continue;
        const int dy = iy - (2 * y - 1), dx = ix - (2 * x - 1);
        if (dy < 0 || dy > 2 || dx < 0 || dx > 2) continue;
        const long long o = (plane * p + y) * q + x;
        const uint4 a4 = reinterpret_cast<const uint4*>(arg)[o];
        const uint32_t aw[4] = {a4.x, a4.y, a4.z, a4.w};
        const uint32_t code = static_cast<uint32_t>(dy * 3 + dx);
        ld16f(gout + o * 16, g);
        if (pmask != nullptr) {
          float pm[16];
          ld16f(pmask + o * 16, pm);
#pragma unroll
          for (int l = 0; l < 16; ++l)
            if (!(pm[l] > 0.0f)) g[l] = 0.0f;
        }
#pragma unroll
        for (int l = 0; l < 16; ++l)
          if (((aw[l / 4] >> (8 * (l % 4))) & 0xFFu) == code) acc[l] += g[l];
      }
    if (mask != nullptr) {  // ReLU backward of the pooled activation
      float m[16];
      ld16f(mask + e * 16, m);
#pragma unroll
      for (int l = 0; l < 16; ++l)
        if (!(m[l] > 0.0f)) acc[l] = 0.0f;
    }
    st16f(gin + e * 16, acc);
  }
}

// Quad form of the same backward: one thread per 2x2 input quad (2y.., 2x..), whose
// four pixels are covered by exactly the windows (y | y+1, x | x+1). Each window's
// argmax codes, gradient and pooled mask are read once for the quad instead of once
// per covered pixel; every pixel sums its windows in the same (y, x) ascending order
// as maxpool_bwd_kernel, so the result is bitwise identical.
template <typename T>
__global__ void maxpool_bwd_quad_kernel(const T* __restrict__ gout, const uint8_t* __restrict__ arg,
                                        T* __restrict__ gin, const T* __restrict__ mask, int planes, int h, int w,
                                        int p, int q, const T* __restrict__ pmask) {
  const int qh = (h + 1) / 2, qw = (w + 1) / 2;
  const long long total = static_cast<long long>(planes) * qh * qw;
  DCONV_GRID_STRIDE(e, total) {
    const int x = static_cast<int>(e % qw);
    const long long r = e / qw;
    const int y = static_cast<int>(r % qh);
    const long long plane = r / qh;
    float acc[4][16];  // pixels (2y, 2x), (2y, 2x+1), (2y+1, 2x), (2y+1, 2x+1)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int l = 0; l < 16; ++l) acc[i][l] = 0.0f;
#pragma unroll
    for (int wy = 0; wy < 2; ++wy)
#pragma unroll
      for (int wx = 0; wx < 2; ++wx) {
        const int oy = y + wy, ox = x + wx;
        if (oy >= p || ox >= q) continue;
        const long long o = (plane * p + oy) * q + ox;
        const uint4 a4 = reinterpret_cast<const uint4*>(arg)[o];
        const uint32_t aw[4] = {a4.x, a4.y, a4.z, a4.w};
        float g[16];
        ld16f(gout + o * 16, g);
        if (pmask != nullptr) {
          float pm[16];
          ld16f(pmask + o * 16, pm);
#pragma unroll
          for (int l = 0; l < 16; ++l)
            if (!(pm[l] > 0.0f)) g[l] = 0.0f;
        }
        // quad pixel (py, px) sits at (dy, dx) = (2(y - oy) + 1 + py, 2(x - ox) + 1 + px) of this window
#pragma unroll
        for (int py = 0; py < 2; ++py)
#pragma unroll
          for (int px = 0; px < 2; ++px) {
            const int dy = 2 * (y - oy) + 1 + py, dx = 2 * (x - ox) + 1 + px;
            if (dy < 0 || dx < 0) continue;  // window (y+1, .) / (., x+1) covers only the odd row / column
            const uint32_t code = static_cast<uint32_t>(dy * 3 + dx);
#pragma unroll
            for (int l = 0; l < 16; ++l)
              if (((aw[l / 4] >> (8 * (l % 4))) & 0xFFu) == code) acc[py * 2 + px][l] += g[l];
          }
      }
#pragma unroll
    for (int py = 0; py < 2; ++py)
#pragma unroll
      for (int px = 0; px < 2; ++px) {
        const int iy = 2 * y + py, ix = 2 * x + px;
        if (iy >= h || ix >= w) continue;
        const long long pe = (plane * h + iy) * w + ix;
        float* a = acc[py * 2 + px];
        if (mask != nullptr) {
          float m[16];
          ld16f(mask + pe * 16, m);
#pragma unroll
          for (int l = 0; l < 16; ++l)
            if (!(m[l] > 0.0f)) a[l] = 0.0f;
        }
        float v[16];
#pragma unroll
        for (int l = 0; l < 16; ++l) v[l] = a[l];
        st16f(gin + pe * 16, v);
      }
  }
}

// Stride-2 lattice of a halo-0 blocked tensor as its own dense tensor (the input of
// a stride-2 1x1 conv: the conv becomes stride 1 over it) and back: the full-size
// tensor with the lattice values and exact zeros elsewhere (a stride-2 1x1
// backward-data's result). One thread per destination pixel, 16-byte moves.
template <typename T>
__global__ void subsample2_kernel(const T* __restrict__ in, T* __restrict__ out, long long planes, int h, int w,
                                  int p, int q) {
  constexpr int kV = static_cast<int>(16 * sizeof(T) / 16);  // uint4 per pixel
  const long long total = planes * p * q;
  DCONV_GRID_STRIDE(e, total) {
    const int x = static_cast<int>(e % q);
    const long long r = e / q;
    const int y = static_cast<int>(r % p);
    const long long plane = r / p;
    const uint4* src = reinterpret_cast<const uint4*>(in + ((plane * h + 2 * y) * w + 2 * x) * 16);
    uint4* dst = reinterpret_cast<uint4*>(out + e * 16);
#pragma unroll
    for (int k = 0; k < kV; ++k) dst[k] = src[k];
  }
}
template <typename T>
__global__ void unsubsample2_kernel(const T* __restrict__ in, T* __restrict__ out, long long planes, int h, int w,
                                    int p, int q) {
  constexpr int kV = static_cast<int>(16 * sizeof(T) / 16);
  const long long total = planes * h * w;
  DCONV_GRID_STRIDE(e, total) {
    const int ix = static_cast<int>(e % w);
    const long long r = e / w;
    const int iy = static_cast<int>(r % h);
    const long long plane = r / h;
    uint4* dst = reinterpret_cast<uint4*>(out + e * 16);
    if (((ix | iy) & 1) == 0) {
      const uint4* src = reinterpret_cast<const uint4*>(in + ((plane * p + iy / 2) * q + ix / 2) * 16);
#pragma unroll
      for (int k = 0; k < kV; ++k) dst[k] = src[k];
    } else {
#pragma unroll
      for (int k = 0; k < kV; ++k) dst[k] = make_uint4(0, 0, 0, 0);
    }
  }
}

// Space-to-depth of a narrow (C <= 4), halo-0, one-block input for a stride-2
// conv: xs[n][i][j][(dy*2+dx)*C + c] = x[n][c][2i+dy-pad][2j+dx-pad] (zero
// outside; lanes >= 4C zero). A stride-2 RxS conv over x equals a stride-1
// ceil(R/2) x ceil(S/2) conv over xs with the filter s2d_wt_kernel builds
// (the 7x7/s2 ResNet stem becomes a 4x4/s1 conv over 12 of 16 lanes).
template <typename T, int C>
__global__ void s2d_act_kernel(const T* __restrict__ x, T* __restrict__ xs, int n, int h, int w, int hs, int ws,
                               int pad) {
  const long long total = static_cast<long long>(n) * hs * ws;
  DCONV_GRID_STRIDE(e, total) {
    const int j = static_cast<int>(e % ws);
    const long long r = e / ws;
    const int i = static_cast<int>(r % hs);
    const long long img = r / hs;
    T v[16];
#pragma unroll
    for (int l = 0; l < 16; ++l) v[l] = from_f<T>(0.0f);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int y = 2 * i + q / 2 - pad, xx = 2 * j + q % 2 - pad;
      if (y < 0 || y >= h || xx < 0 || xx >= w) continue;
      const T* px = x + ((img * h + y) * w + xx) * 16;
#pragma unroll
      for (int ch = 0; ch < C; ++ch) v[q * C + ch] = px[ch];
    }
    uint4* o = reinterpret_cast<uint4*>(xs + e * 16);
    const uint4* vv = reinterpret_cast<const uint4*>(v);
#pragma unroll
    for (int k = 0; k < static_cast<int>(16 * sizeof(T) / 16); ++k) o[k] = vv[k];
  }
}

// NCHW fp32 image straight into the space-to-depth blocked layout (the input pack
// and dconv_s2d_act in one pass: no 16-lane full-resolution intermediate)
template <typename T, int C>
__global__ void pack_s2d_kernel(const float* __restrict__ x, T* __restrict__ xs, int n, int h, int w, int hs, int ws,
                                int pad) {
  const long long total = static_cast<long long>(n) * hs * ws;
  DCONV_GRID_STRIDE(e, total) {
    const int j = static_cast<int>(e % ws);
    const long long r = e / ws;
    const int i = static_cast<int>(r % hs);
    const long long img = r / hs;
    T v[16];
#pragma unroll
    for (int l = 0; l < 16; ++l) v[l] = from_f<T>(0.0f);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int y = 2 * i + q / 2 - pad, xx = 2 * j + q % 2 - pad;
      if (y < 0 || y >= h || xx < 0 || xx >= w) continue;
#pragma unroll
      for (int ch = 0; ch < C; ++ch) v[q * C + ch] = from_f<T>(x[((img * C + ch) * h + y) * w + xx]);
    }
    uint4* o = reinterpret_cast<uint4*>(xs + e * 16);
    const uint4* vv = reinterpret_cast<const uint4*>(v);
#pragma unroll
    for (int k = 0; k < static_cast<int>(16 * sizeof(T) / 16); ++k) o[k] = vv[k];
  }
}

// W[k][c][r][s] (blocked, one c-block) -> W'[k][(dy*2+dx)*C + c][r'][s'] =
// W[k][c][2r'+dy][2s'+dx] (zero past R / S); inverse = s2d_wt_grad_kernel
__global__ void s2d_wt_kernel(const float* __restrict__ w, float* __restrict__ w2, int kb, int c, int R, int S,
                              int R2, int S2) {
  const long long total = static_cast<long long>(kb) * R2 * S2 * 256;
  DCONV_GRID_STRIDE(e, total) {
    const int lane = static_cast<int>(e % 256);
    const long long rr = e / 256;
    const int s2 = static_cast<int>(rr % S2), r2 = static_cast<int>((rr / S2) % R2);
    const long long kbi = rr / (static_cast<long long>(S2) * R2);
    const int ci = lane / 16, ki = lane % 16;  // lane [c][k]
    float v = 0.0f;
    if (ci < 4 * c) {
      const int q = ci / c, ch = ci % c, dy = q / 2, dx = q % 2;
      const int r = 2 * r2 + dy, sx = 2 * s2 + dx;
      if (r < R && sx < S) v = w[((kbi * R + r) * S + sx) * 256 + ch * 16 + ki];
    }
    w2[e] = v;
  }
}

__global__ void s2d_wt_grad_kernel(const float* __restrict__ g2, float* __restrict__ g, int kb, int c, int R, int S,
                                   int R2, int S2) {
  const long long total = static_cast<long long>(kb) * R * S * 256;
  DCONV_GRID_STRIDE(e, total) {
    const int lane = static_cast<int>(e % 256);
    const long long rr = e / 256;
    const int sx = static_cast<int>(rr % S), r = static_cast<int>((rr / S) % R);
    const long long kbi = rr / (static_cast<long long>(S) * R);
    const int ci = lane / 16, ki = lane % 16;
    float v = 0.0f;
    if (ci < c) {
      const int q = (r % 2) * 2 + (sx % 2);
      v = g2[((kbi * R2 + r / 2) * S2 + sx / 2) * 256 + (q * c + ci) * 16 + ki];
    }
    g[e] = v;
  }
}

// SGD on fp32 master weights: w -= lr * g (blocked layouts, identical shapes)
__global__ void scale_kernel(float* __restrict__ w, float s, long long n) {
  DCONV_GRID_STRIDE(i, n) w[i] *= s;
}

__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g, float lr, long long n) {
  DCONV_GRID_STRIDE(e, n) { w[e] -= lr * g[e]; }
}

// ReLU backward mask fused helper: g *= (y > 0) on blocked tensors of equal shape
template <typename T>
__global__ void relu_mask_kernel(T* __restrict__ g, const T* __restrict__ y, long long n) {
  DCONV_GRID_STRIDE(e, n) {
    if (!(to_f<T>(y[e]) > 0.0f)) g[e] = from_f<T>(0.0f);
  }
}

// Split a blocked fp32 tensor into `pieces` bf16 tensors laid out one after
// the other (piece-major): x == hi + mid + lo exactly (pieces = 3), or a
// round-to-nearest cast (pieces = 1). Halo / tail elements map 0 -> 0.
__global__ void split_pieces_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, long long n,
                                    int pieces) {
  DCONV_GRID_STRIDE(e, n) {
    const float x = src[e];
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    dst[e] = h;
    if (pieces == 3) {
      const float r1 = x - __bfloat162float(h);
      const __nv_bfloat16 m = __float2bfloat16_rn(r1);
      dst[e + n] = m;
      dst[e + 2 * n] = __float2bfloat16_rn(r1 - __bfloat162float(m));
    }
  }
}

}  // namespace dconv_sm100
