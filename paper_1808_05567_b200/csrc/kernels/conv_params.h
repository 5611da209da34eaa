// Kernel parameter blocks shared between the host launch plan and the
// sm_100a conv kernels. Plain structs so they can be passed by value.
#pragma once
#include <cuda.h>
#include <stdint.h>

// Developer build (tools/: role cycle counters and ablation bits). Product builds
// compile every dbg / dbg_mode branch out of the kernels.
#ifndef DCONV_DEV_BUILD
#define DCONV_DEV_BUILD 0
#endif

namespace dconv_sm100 {

constexpr bool kDevBuild = DCONV_DEV_BUILD != 0;

constexpr int kMaxTaps = 128;     // filter taps (R * S <= 128: up to 11 x 11)
constexpr int kMaxPhases = 16;    // stride phases (stride <= 4)
constexpr int kMaxXsSlots = 32;   // cross-stacked UPD: A slots (row / column shifted input tiles)
constexpr int kMaxTapGroups = 128;

// Implicit-GEMM forward over the "virtual row" grid: output pixel (p, q) of
// image n is virtual position v = p * wsub + q; tap t of phase ph reads the
// phase sub-image at v + tap_shift[t]. A tile is L = 128 * mb consecutive
// virtual positions of one image; the CTA computes them for 16 * nb output
// channels.
struct FwdParams {
  int n_img;
  int in_cb;           // channel blocks of the input tensor (plane index = n*in_cb + cb)
  int cb_in;           // reduction channel blocks
  int kb_out;          // output channel blocks (reduction result)
  int P, Q;            // output extents (lattice units)
  int wsub;            // virtual row pitch
  int tiles_per_img;
  int mb;              // 128-row m-blocks per tile
  int nb;              // 16-channel output blocks per CTA
  int acc_bufs;        // TMEM accumulator buffers (2 = epilogue overlaps the next tile)
  // A staging: smem chunk planes hold a_px pixels starting at virtual pixel a_px0
  int linear;          // 1: virtual index == physical pixel index of the halo'd plane
  int mimg;            // >0: multi-image tiles (1x1 stride 1, small planes): mimg whole images per tile
  // > 0 (with mimg): packed multi-tap tiles (stride-1 bf16 rows plans of small images):
  // mimg whole images along M at this pitch ((H + pad) rows of wsub), each image's
  // bottom padding the next one's top padding; one 5-D activation box of mimg + 1
  // images (images inside the channel-block planes) so the last image's is zero too
  int img_pitch;
  // 1 (bf16 linear single-tap plans with the TMA-store epilogue, planes of 4k pixels): the
  // activation stage is written as SWIZZLE_128B 128 B rows of four pixels and read through
  // the unchanged K-major SW32 descriptors -- the TMA unit moves ~1 box row per clock whatever
  // its width (27 B/clk/SM on 32 B rows, 68 on 128 B rows). MMA row q of each 32-row group
  // then holds pixel q ^ ((q >> 3) & 3) (channel halves intact); the epilogue warps undo
  // the permutation when they stage their 32-pixel slabs and fetch the fused operands.
  int a_sw128;
  int a_px;            // pixels per chunk plane per stage
  int a_load_px;       // pixels the activation TMA writes per stage
  int lin_boxes;       // linear mode: 128-pixel boxes per chunk plane
  int in_row0, in_col0;// logical input coordinate of sub-image (0, 0)
  int stride;
  int n_phases;
  int phase_row[kMaxPhases], phase_col[kMaxPhases];
  int phase_ntaps[kMaxPhases], phase_tap0[kMaxPhases];
  int tap_shift[kMaxTaps];  // phase-sorted
  int taps_box;        // max taps per phase
  int w_taps;          // taps per weight pipeline stage (<= taps_box)
  int kc;              // input channel blocks per pipeline stage (single-tap TS plans; else 1)
  int w_resident;      // 1: the CTA's whole weight slice stays in smem (loaded once)
  int w_all;           // bf16 single-phase plans, one output-channel tile: every weight stage has its own slot, loaded once
  int tma_store;       // 1: epilogue stages 32-pixel slabs in smem and TMA-stores them (dense outputs)
  int out_fill;        // 1: stride-2 lattice output that also writes the zero pixels it owns
  int split_acc;       // fp32-accurate: 1 = hi*hi and corrections in separate accumulators (long reductions)
  int ts_epi2;         // TS plans with one stage per tile: warps 12..15 are a second epilogue group
  int epi_groups;      // bf16 smem-staged plans with the lean epilogue: epilogue warp groups (1..3)
  int fill_h_end, fill_w_end;  // interior row / column ends (padded coordinates) for out_fill
  int n_taps;          // total taps (phase-sorted) in the prepared weights
  int n_ntiles;        // output-channel tiles (prepared weights are tiled by nb)
  const void* wprep;   // prepared bf16 weights [pc][cb][ntile][tap][2nb][16][8]
  // output surface (blocked, may be a strided lattice)
  void* out;
  int out_bf16;
  int out_cb;          // channel blocks of the output tensor
  int out_hp, out_wp;  // physical extents
  int out_y0, out_x0;  // physical position of lattice point (0, 0)
  int out_scale;       // physical pixels per lattice step
  int out_halo_h, out_halo_w;  // halo frame to zero (0 = none)
  const float* bias;   // kb_out*16 lanes or null
  int relu;
  // fused graph epilogue (executor): v += add[px]; v = relu(v); v *= (mask[px] > 0).
  // add / mask share the output surface's geometry and dtype (null = off)
  const void* add;
  const void* mask;
  long long* dbg;      // optional per-CTA role cycle counters (16 per CTA), null in production
  int dbg_mode;        // ablation bits (debug only): 1 skip global stores, 2 skip TMEM loads
};

// Weight update: per (c-tile x tap group, k-tile, split) CTA, fp32 partial
// dW[tap][c][k] over a contiguous range of stages. Operands are bf16 piece
// tensors read by TMA: plane index = piece * (n_img * cb) + n * cb + block.
struct UpdParams {
  int n_img;
  int in_cb, do_cb;    // channel blocks of the input / dO tensors
  int cb_in, kb_out;
  int P, Q;
  int wsub;            // virtual row pitch (dO box width)
  int linear;          // 1: both operands are dense planes (1x1, stride 1, pad 0, no halos)
  int rows_ps;         // rows mode: output rows per stage
  int vs;              // virtual pixels per stage (multiple of 16)
  int a_px;            // input pixels per chunk plane per stage
  int in_rows;         // rows mode: input sub-image rows per stage
  int in_row0, in_col0;
  int stride;
  int stages_per_img;
  int stages_total;
  int splits;
  int nb;              // K blocks per CTA (N = 16 * nb)
  int tg;              // max taps per CTA
  int n_tgroups;
  int tg_phase[kMaxTapGroups];
  int tg_tap0[kMaxTapGroups];
  int tg_ntaps[kMaxTapGroups];
  int phase_row[kMaxPhases], phase_col[kMaxPhases];
  int tap_shift[kMaxTaps];
  int tap_src[kMaxTaps];   // phase-sorted tap -> r*S + s
  // tap stacking (layers with < 8 input channel blocks): the 128 MMA rows hold
  // `stack` taps x cb_eff channel blocks, each slot staged by its own shifted box
  int stack;               // 1 = shared-tile mode (taps via descriptor shifts)
  // cross-stacking (xs >= 2; stride-1 bf16 stacked plans): the N dimension also holds
  // xs copies of the dO tile, copy j shifted by j columns (TMA box at column -j, zero
  // fill), and A slot i is the input tile shifted by (xs_slot_r[i], xs_slot_s[i]):
  // accumulator block (i, j) is the weight gradient of tap (r_i, s_i + j). The A
  // slots of a tap group are xs_slot[tg_tap0 ..] (their columns are multiples of xs)
  int xs, xs_S;            // B copies (0 / 1: off), filter width (tap = r * xs_S + s)
  // packed image planes (pimg >= 1; stride-1 bf16 rows plans of small images): a stage
  // holds pimg whole images along K at a pitch of img_pitch pixels ((H + pad) rows of
  // wsub): each image's bottom padding is the next image's top padding (zero fill), so
  // the 7x7 3x3 update spends 98 of 144 K rows on real pixels instead of 49 of 144.
  // One 5-D box per operand (images inside the channel-block planes); the A box
  // carries pimg + 1 images so that the last image's bottom padding is zero too.
  int pimg, img_pitch;
  int xs_slot_r[kMaxXsSlots], xs_slot_s[kMaxXsSlots];
  int cb_eff;
  int half;                // stacked with C <= 8: a tap slot is one 8-channel chunk (16 taps per 128 rows)
  // bf16 operands read through MN-major SWIZZLE_32B descriptors. 1: staged as SWIZZLE_32B
  // 32 B pixel rows; 2 (linear single-tap plans, planes of 4k pixels): staged as
  // SWIZZLE_128B 128 B rows of four pixels -- the TMA unit moves ~1 box row per clock
  // whatever its width, so this stages 2.5x the bytes per clock. Read back through the
  // SW32 descriptors the rows come out with their halves intact and the pixels of each
  // 32-pixel group permuted (q -> q ^ ((q >> 3) & 3)); both operands of the K = pixel
  // reduction carry the same permutation, so every MMA sums the same products.
  int sw32;
  int mc;                  // single-tap sw32 plans: 128-channel c-tiles per CTA (2: the dO tile is staged once for both)
  // lsu = 1: the operand rows are staged by cp.async from loader warps (the TMA
  // unit moves 32 B rows at ~27 B/clk/SM; 16 B cp.async from six warps ~2x that)
  int lsu;
  const void* in_ptr;      // interior pixel (0, 0) of plane 0 (halo offset applied)
  const void* do_ptr;
  int in_h, in_w, in_wp;   // interior extents, physical row pitch (pixels)
  long long in_plane;      // pixels per physical plane
  int do_h, do_w, do_wp;
  long long do_plane;
  int tap_ph[kMaxTaps], tap_r2[kMaxTaps], tap_s2[kMaxTaps];
  int n_taps;
  float* partial;      // [split][tap(RS)][c_pad][k_pad]
  int dbg_mode;        // ablation bits (debug only): 4 skip conversion, 8 skip MMAs
  int c_pad, k_pad;
  // fp32-accurate accumulation periods: the tensor core's fp32 accumulate truncates
  // per MMA, so a long chain drifts (~ chain x 2^-24 relative, biased). Every `drain`
  // stages the TMEM accumulator is added (RNE, fp32) into the CTA's partial slice
  // and restarted; `drain_bufs` = 2 alternates two accumulators so the MMA never
  // waits on the drain. drain = 0: one period (no drains).
  int drain;
  int drain_bufs;
  // 1: the partials leave through TMA stores (bf16 single-period plans whose warps own
  // 32 consecutive partial rows): each epilogue warp stages 32 rows x 16 columns in
  // shared memory (the idle operand ring) -- full-line writes instead of one 16 B
  // segment per lane per store
  int epi_tma;
};

}  // namespace dconv_sm100
