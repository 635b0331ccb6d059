// tb_kernels.cuh -- the BST filtered-backprojection kernels (sm_100a).
//
//   K1   k1_radial   per row pair: [ramp FFT -> x2 pi|f| -> IFFT] -> x(1-bump)
//                    -> FFT_L -> split the two packed rows -> true-origin phase,
//                    rect split and 1/max(|f|, sigma_min)      (fourier_bp.py:302-373, 469-505)
//   K1b  k1b_common  per slice: angular mean row over the window support ->
//                    common row Chat and coef.mean()          (fourier_bp.py:336-341, 452-458)
//   K2   k2_columns  per Cartesian column k1: bilinear polar->Cartesian gather of
//                    the Hermitian half plane (+ modulation) -> IFFT_L along k2,
//                    pruned to the n output rows              (fourier_bp.py:376-431)
//   K3   k3_rows     per output row pair: C2R along k1, crop, amplitude scale,
//                    coverage add-back, 1/(2 pi), finite flag (fourier_bp.py:431-460, 530)
//   KR   kr_ramp     standalone ramp filter                   (fourier_bp.py:490-505)
//   K5   k5_slant    slant-stack comparator                   (projector.py:126-158)
//
// Layouts in HBM (fp32 / complex64):
//   sino    [B][A][n_t]        A = input angles (n_theta, or 2 n_theta full turn)
//   polar   [B][rows][H]       rows = processed angles = A, H = L/2 radial bins
//   part    [B][groups][S]     per-CTA partial column sums over the KB support
//   rowcoef [B][rows], common [B][H], coefmean [B]
//   columns [B][ceil(n/4)][H+1][4]  K2 output in 4-row tiles (k1-major inside a tile)
//   image   [B][n][n]
#pragma once
#include "fft.cuh"

namespace tb {

struct DevPlan {
  int n_t, n_theta, rows, L, H, n, npad;
  int lo, S;          // KB window support [lo, lo+S)
  int full_turn, interp, nyq;
  int has_mod;
  int n_half;         // n/2 (crop offset)
  float inv_nt;
  float inv_rows2;    // 1 / (2 V)
  float img_scale;    // amplitude_scale / L^2
  float ss_weight;    // span / A (slant stack)
  float ss_inv_dt;    // 1 / dt
  const float2* tw_L;   // [L]   exp(-2 pi i j / L)
  const float2* tw_np;  // [npad]
  const float* ramp_g;  // [npad] 2 pi |f| taper / npad
  const float* omb;     // [n_t]  1 - bump
  const float* bump_s;  // [S]    bump over the support
  const float2* psi;    // [H]    exp(2 pi i f_k) / den_k
  const float2* rho;    // [H]    ref_k / den_k
  const float2* modt;   // [L]    half-node modulation (or null)
  const float2* twm;    // per-pass twiddle bases of fft_mod for alpha = pi / L (the
                        // half-node modulation of an n = L/2 crop), K2's column IFFT
  const double2* ss_cs; // [A]    (cos, sin) of the input angles
  const uint2* gridtab; // [(H+1)^2] first-quadrant gridding table
  // [(H+1)][(H+1)] first-quadrant gridding table of the half-turn bilinear
  // path: per node (a, b), a, b >= 0, the TLD4 texel coordinates (r0 + 1,
  // t0 + 1) and the fp32 radial / angular weights, or null
  const float4* gridtab2;
  const int* colext;    // [H+1] per column a: largest b' whose gridtab2 entry is inside the disc (-1: none)
  int c2pitch;          // elements per slice of Work::common2 (>= H + 1; [H..] = 0)
  int prow;             // polar rows per slice: V + 1 (half turn, row V = conj row 0) or 2V + 1 (full turn, row 2V = row 0)
  size_t col_slice;     // complex elements per slice of the K2 output (tiled)
};

struct Work {
  float2* polar;
  float* rowcoef;
  float* part;
  float2* common;
  float2* common2;  // [B][c2pitch] (Re C[r], Re C[min(r+1, H-1)]) for the half-turn fast path, 0 for r >= H
  float* coefmean;
  float2* columns;
  float* filtered;
  int* status;  // [0] non-finite input, [1] non-finite output
  // transmission-count input (NORM kernels): per input row and detector
  // (dark D, 1 / max(I0 - D, eps)) and eps
  const float2* normtab;  // null with NORM: constant frames, norm_c = (D, 1 / max(I0 - D, eps))
  float norm_eps;
  float2 norm_c;
  // input addressing (elements): row j of slice q at q * in_slice + j * in_row
  // (slice-major [B][A][n_t]: A n_t, n_t; a frame-major slab [A][B][n_t]: n_t, B n_t)
  long long in_slice, in_row;
  int groups;   // K1 CTAs per slice (partial-sum groups)
  int pairs_per_cta;
  // texture view of this lane's polar region (pitch 2D, float2 texels,
  // width H, height B*(V+1)); 0 = use plain loads
  cudaTextureObject_t polar_tex;
  // fused centre / ring stages (preprocess.py:119-154) on K1's load, or null:
  // per slice (floor(beta), frac(beta)) of the detector shift and the stripe
  // profile [B][n_t] subtracted after it (k_pre_params)
  const float2* pre_shift;
  const float* pre_stripe;
};

#ifndef TB_K1_SLOTS
// K1 TMA staging slots (row pairs).  0 = coalesced direct row loads: the
// measured default (2048^3 equal within noise, 1024^3 -1.6 %, 512^3 -2 %):
// the 16 KB staging slot cost more in L1 / co-residency with the other
// lane than the latency it hid
#define TB_K1_SLOTS 0
#endif
#define K1_STAGE_ROWS (2 * TB_K1_SLOTS)

template <int L>
struct KShape {
  using S = FftShape<L>;
  static constexpr int RPT = S::RPT;
  static constexpr int TPF = S::TPF;
  static constexpr int THREADS = TPF < 32 ? 32 : TPF;
  // smem buffer (float2) for the FFT passes and the K1 Z_k / Z_{L-k} exchange
  static constexpr int BUF = S::SMEM > 0 ? S::SMEM : L;
  static constexpr int K1B_THREADS = THREADS < 512 ? 512 : THREADS;
  // CTAs per SM asked of ptxas (register cap 64K / (THREADS * MINB))
#ifndef TB_MINB
#define TB_MINB 3
#endif
  static constexpr int MINB = THREADS <= 256 ? TB_MINB : 1;
};

// K1's transform shape: TB_K1_RPT = 64 puts 64 points in each thread's
// registers (4096 = 64 x 64: one shared-memory exchange per transform instead
// of two, 64 threads per row pair); default 16 as everywhere else
#ifndef TB_K1_RPT
#define TB_K1_RPT 16
#endif
template <int L>
struct K1Shape {
  static constexpr int RPT = (TB_K1_RPT == 64 && L >= 4096) ? 64 : default_rpt(L);
  using S = FftShape<L, RPT>;
  static constexpr int TPF = S::TPF;
  static constexpr int THREADS = TPF < 32 ? 32 : TPF;
  static constexpr int BUF = S::SMEM > 0 ? S::SMEM : L;
  static constexpr int PB = S::PB;
  static constexpr int LPB = ilog2(PB);
#ifndef TB_K1_MINB64
#define TB_K1_MINB64 4
#endif
  static constexpr int MINB = THREADS <= 64 ? TB_K1_MINB64 : (THREADS <= 256 ? 4 : 1);
};

// ---------------------------------------------------------------------------
// Normalisation prologue (preprocess.py:59-74): transmission counts to line
// integrals, y = -ln(max(I - D, eps) / max(I0 - D, eps)).  nt = (D, 1 /
// max(I0 - D, eps)) per input row and detector (k_norm_table).  A NaN
// difference stays NaN (np.maximum propagates it; fmaxf would not).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float norm_line(float I, float2 nt, float eps) {
  const float num = I - nt.x;
  return -__logf((num != num ? num : fmaxf(num, eps)) * nt.y);
}

// ---------------------------------------------------------------------------
// K1: radial kernel (fused ramp when npad == L; fused normalisation when NORM)
// ---------------------------------------------------------------------------
// K1 at 4 CTAs per SM: 64 registers without spills; with K2 also at 4 the
// step drops 179.6 -> 178.6 ms at 2048^3 (neutral at 1024^3 / 512^3)
#ifndef TB_K1_MINB
#define TB_K1_MINB 4
#endif
// one K1 block: row pairs of partial-sum group g of slice q (every thread of
// the CTA; smem = the dynamic shared memory of smem_k1)
template <int L, bool RAMP, bool NORM, bool PRE = false>
__device__ __forceinline__ void k1_block(const DevPlan& p, const float* __restrict__ sino, const Work& w, int g, int q,
                                         float2* smem) {
  using K = K1Shape<L>;
  constexpr int RPT = K::RPT, TPF = K::TPF, PB = K::PB;
  float2* buf = smem;
  float* sacc = reinterpret_cast<float*>(smem + K::BUF);
  // staging for the row pair (TMA bulk copies, TB_K1_SLOTS > 0), 16-B
  // aligned: one slot, refilled with the next pair as soon as every thread
  // holds its samples (the copy then hides behind three FFTs)
  float* stage = sacc + ((p.S + 3) & ~3);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage + K1_STAGE_ROWS * p.n_t);
  const int t = threadIdx.x;
  // blocks are exactly TPF threads once TPF >= 32: compile-time true there
  const bool active = TPF >= 32 || t < TPF;
  const int npairs = (p.rows + 1) >> 1;
  const int pr_begin = g * w.pairs_per_cta;
  const int pr_end = min(npairs, pr_begin + w.pairs_per_cta);
  const int H = L / 2;
  const float* slice = sino + (size_t)q * w.in_slice;
  // bulk copies need 16-byte aligned rows; otherwise read rows directly
  const bool bulk = TB_K1_SLOTS > 0 && !w.pre_shift && (p.n_t & 3) == 0 && ((reinterpret_cast<uintptr_t>(sino) & 15) == 0) && (w.in_row & 3) == 0 &&
                    (w.in_slice & 3) == 0;
  auto issue = [&](int pr, int slot) {
    // the slot was last read by generic-proxy loads (ordered before this
    // thread by the barrier); order them before the async-proxy refill
    fence_proxy_async_smem();
    const int j0 = 2 * pr;
    const int nrow = (2 * pr + 1 < p.rows) ? 2 : 1;
    const uint32_t bytes = (uint32_t)(nrow * p.n_t * 4);
    mbar_expect_tx(&bars[slot], bytes);
    if (w.in_row == p.n_t) {  // the pair is one contiguous run
      bulk_g2s(stage + slot * 2 * p.n_t, slice + (size_t)j0 * p.n_t, bytes, &bars[slot]);
    } else {
      const uint32_t rb = (uint32_t)(p.n_t * 4);
      bulk_g2s(stage + slot * 2 * p.n_t, slice + (size_t)j0 * w.in_row, rb, &bars[slot]);
      if (nrow == 2) bulk_g2s(stage + slot * 2 * p.n_t + p.n_t, slice + (size_t)(j0 + 1) * w.in_row, rb, &bars[slot]);
    }
  };

  for (int i = t; i < p.S; i += blockDim.x) sacc[i] = 0.f;
  if (bulk && t == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (bulk && t == 0 && pr_begin < pr_end) issue(pr_begin, 0);
  bool bad = false;
  uint32_t phase[2] = {0u, 0u};

  for (int pr = pr_begin; pr < pr_end; ++pr) {
    const int j0 = 2 * pr, j1 = 2 * pr + 1;
    const bool has1 = j1 < p.rows;
    const int slot = TB_K1_SLOTS == 2 ? (pr - pr_begin) & 1 : 0;
    float2 v[RPT];
    if (bulk) {
#if TB_K1_SLOTS == 2
      // prefetch the next pair into the other slot (freed by the barrier that
      // closed the previous iteration), then wait for this pair's rows
      if (t == 0 && pr + 1 < pr_end) issue(pr + 1, slot ^ 1);
#endif
      mbar_wait(&bars[slot], phase[slot]);
      phase[slot] ^= 1u;
      const float* r0 = stage + slot * 2 * p.n_t;
      const float* r1 = r0 + p.n_t;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int idx = t + i * TPF;
        float a = 0.f, b = 0.f;
        if (i < RPT / 2 && active && idx < p.n_t) {
          a = r0[idx];
          if (has1) b = r1[idx];
          if constexpr (NORM) {
            if (w.normtab) {
              const float2* nt = w.normtab + (size_t)j0 * p.n_t + idx;
              a = norm_line(a, __ldg(nt), w.norm_eps);
              if (has1) b = norm_line(b, __ldg(nt + p.n_t), w.norm_eps);
            } else {
              a = norm_line(a, w.norm_c, w.norm_eps);
              if (has1) b = norm_line(b, w.norm_c, w.norm_eps);
            }
          }
        }
        v[i] = make_float2(a, b);
      }
#if TB_K1_SLOTS == 1
      __syncthreads();  // every thread holds its samples: the slot is free
      if (t == 0 && pr + 1 < pr_end) issue(pr + 1, 0);
#endif
    } else {
      const float* y0 = slice + (size_t)j0 * w.in_row;
      const float* y1 = y0 + w.in_row;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int idx = t + i * TPF;
        float a = 0.f, b = 0.f;
        // n_t <= L/2 always (L >= pad_factor * n_t, pad_factor >= 2): the upper
        // half of every padded row is a compile-time zero (pruned first pass)
        if (i < RPT / 2 && active && idx < p.n_t) {
          if constexpr (PRE) {
            // apply_center (linear interpolation at idx + beta, 0 outside the
            // detector) then the ring stripe: preprocess.py:119-154
            const float2 sh = __ldg(w.pre_shift + q);
            const int j = idx + (int)sh.x;
            const bool ok0 = j >= 0 && j <= p.n_t - 1, ok1 = j + 1 >= 0 && j + 1 <= p.n_t - 1;
            const float w0 = 1.f - sh.y, w1 = sh.y;
            const float st = w.pre_stripe ? __ldg(w.pre_stripe + (size_t)q * p.n_t + idx) : 0.f;
            a = (ok0 ? w0 * __ldg(y0 + j) : 0.f) + (ok1 ? w1 * __ldg(y0 + j + 1) : 0.f) - st;
            if (has1) b = (ok0 ? w0 * __ldg(y1 + j) : 0.f) + (ok1 ? w1 * __ldg(y1 + j + 1) : 0.f) - st;
          } else {
            a = __ldg(y0 + idx);
            if (has1) b = __ldg(y1 + idx);
          }
          if constexpr (NORM) {
            if (w.normtab) {
              const float2* nt = w.normtab + (size_t)j0 * p.n_t + idx;
              a = norm_line(a, __ldg(nt), w.norm_eps);
              if (has1) b = norm_line(b, __ldg(nt + p.n_t), w.norm_eps);
            } else {
              a = norm_line(a, w.norm_c, w.norm_eps);
              if (has1) b = norm_line(b, w.norm_c, w.norm_eps);
            }
          }
        }
        v[i] = make_float2(a, b);
      }
    }
    if constexpr (RAMP) {
      fft_half<L, false, CtaSync, RPT>(v, buf, t, active, p.tw_np);
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const float gk = active ? __ldg(p.ramp_g + t + i * TPF) : 0.f;
        v[i] = cscale(v[i], gk);
      }
      fft<L, true, CtaSync, RPT>(v, buf, t, active, p.tw_np);
    }
    // v[i] = (h_j0, h_j1)(t_idx) for idx < n_t: support sums, window, zero pad
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int idx = t + i * TPF;
      if (i >= RPT / 2) {
        v[i] = make_float2(0.f, 0.f);  // crop to n_t + zero pad: outputs i >= RPT/2 are dead
      } else if (active) {
        const int s = idx - p.lo;
        if (s >= 0 && s < p.S) sacc[s] += v[i].x + v[i].y;
        const float m = idx < p.n_t ? __ldg(p.omb + idx) : 0.f;
        v[i] = cscale(v[i], m);
      }
    }
    fft_half<L, false, CtaSync, RPT>(v, buf, t, active, p.tw_L);
    // exchange Z_k / Z_{L-k} through smem to separate the two real rows
    constexpr bool XALIGN = K::S::SMEM > 0 && (TPF % PB == 0);
    if constexpr (XALIGN) {
      const int sp_t = spadb<PB>(t);
      if (active) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) buf[sp_t + i * TPF + (i * TPF) / PB] = v[i];
      }
    } else if constexpr (K::S::SMEM > 0) {
      if (active) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) buf[spadb<PB>(t + i * TPF)] = v[i];
      }
    } else {
      if (active) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) buf[t + i * TPF] = v[i];
      }
    }
    __syncthreads();
    const float2 z0 = buf[0];
    const float a0 = z0.x * p.inv_nt, a1 = z0.y * p.inv_nt;
    // a non-finite sample anywhere in the pair reaches the DC bin through the
    // ramp / window / FFT chain (x * 0 and inf - inf are NaN; the count
    // normalisation propagates NaN), so the rect coefficients carry the
    // input finiteness check (one test per pair instead of one per sample)
    bad |= !(isfinite(a0) && isfinite(a1));
    float2* out0 = w.polar + ((size_t)q * p.prow + j0) * H;
    float2* out1 = out0 + H;
    // half turn: row V holds conj(row 0), the angle-pi mirror (fourier_bp.py:310);
    // full turn: row 2V repeats row 0 (angle 2 pi), so the texture gathers
    // of K2_TEXF never wrap
    float2* outm = j0 == 0 ? w.polar + ((size_t)q * p.prow + p.rows) * H : nullptr;
    const float mconj = p.full_turn ? 1.f : -1.f;
    if (active) {
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int k = t + i * TPF;
        if (k < H) {
          const int km = (L - k) & (L - 1);
          const float2 zk = v[i];
          float2 zm;
          if constexpr (XALIGN) {
            // spadb(L - t - i TPF) = spadb(-t) + (L - i TPF) (PB + 1) / PB for k > 0
            const int c = L - i * TPF;
            zm = k == 0 ? buf[0] : buf[(-t) + ((-t) >> K::LPB) + c + c / PB];
          } else {
            zm = buf[K::S::SMEM > 0 ? spadb<PB>(km) : km];
          }
          const float2 X = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
          const float2 Y = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
          const float2 ps = __ldg(p.psi + k), rh = __ldg(p.rho + k);
          float2 A0 = cmul(ps, X), A1 = cmul(ps, Y);
          A0 = make_float2(fmaf(-a0, rh.x, A0.x), fmaf(-a0, rh.y, A0.y));
          A1 = make_float2(fmaf(-a1, rh.x, A1.x), fmaf(-a1, rh.y, A1.y));
          if (k == 0) { A0 = make_float2(0.f, 0.f); A1 = A0; }
          out0[k] = A0;
          if (has1) out1[k] = A1;
          if (outm) outm[k] = make_float2(A0.x, mconj * A0.y);
        }
      }
    }
    if (t == 0) {
      w.rowcoef[(size_t)q * p.rows + j0] = a0;
      if (has1) w.rowcoef[(size_t)q * p.rows + j1] = a1;
    }
    __syncthreads();
  }
  if (bad) atomicOr(&w.status[0], 1);
  float* part = w.part + ((size_t)q * w.groups + g) * p.S;
  for (int i = t; i < p.S; i += blockDim.x) part[i] = sacc[i];
}

// PRE: the fused centre / ring stages on the row load (its own
// instantiation: the plain load keeps its schedule, 0.45 ms per 2048^3)
template <int L, bool RAMP, bool NORM, bool PRE = false>
__global__ void __launch_bounds__(K1Shape<L>::THREADS, K1Shape<L>::THREADS <= 64 ? TB_K1_MINB64
                                                    : (K1Shape<L>::THREADS <= 256 ? TB_K1_MINB : 1))
    k1_radial(DevPlan p, const float* __restrict__ sino, Work w) {
  extern __shared__ float2 smem[];
  k1_block<L, RAMP, NORM, PRE>(p, sino, w, blockIdx.x, blockIdx.y, smem);
}

// ---------------------------------------------------------------------------
// KR: standalone ramp filter (rows -> rows), fourier_bp.py:469-505
// ---------------------------------------------------------------------------
template <int NP, bool NORM>
__global__ void __launch_bounds__(KShape<NP>::THREADS) kr_ramp(DevPlan p, const float* __restrict__ sino,
                                                               float* __restrict__ out, int total_rows, Work w) {
  using K = KShape<NP>;
  constexpr int RPT = K::RPT, TPF = K::TPF;
  extern __shared__ float2 smem[];
  const int t = threadIdx.x;
  // blocks are exactly TPF threads once TPF >= 32: compile-time true there
  const bool active = TPF >= 32 || t < TPF;
  const int j0 = 2 * blockIdx.x, j1 = j0 + 1;
  const bool has1 = j1 < total_rows;
  // global row index j over B slices -> (slice j / rows, row j % rows)
  const float* y0 = sino + (size_t)(j0 / p.rows) * w.in_slice + (size_t)(j0 % p.rows) * w.in_row;
  const float* y1 = sino + (size_t)(j1 / p.rows) * w.in_slice + (size_t)(j1 % p.rows) * w.in_row;
  float2 v[RPT];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int idx = t + i * TPF;
    float a = 0.f, b = 0.f;
    if (active && idx < p.n_t) {
      a = __ldg(y0 + idx);
      if (has1) b = __ldg(y1 + idx);
      bad |= !isfinite(a) || !isfinite(b);
      if constexpr (NORM) {
        // input row j0 of slice (j0 / rows) -> frame row j0 % rows
        const float2 c0 = w.normtab ? __ldg(w.normtab + (size_t)(j0 % p.rows) * p.n_t + idx) : w.norm_c;
        a = norm_line(a, c0, w.norm_eps);
        if (has1) {
          const float2 c1 = w.normtab ? __ldg(w.normtab + (size_t)(j1 % p.rows) * p.n_t + idx) : w.norm_c;
          b = norm_line(b, c1, w.norm_eps);
        }
      }
    }
    v[i] = make_float2(a, b);
  }
  fft<NP, false>(v, smem, t, active, p.tw_np);
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const float gk = active ? __ldg(p.ramp_g + t + i * TPF) : 0.f;
    v[i] = cscale(v[i], gk);
  }
  fft<NP, true>(v, smem, t, active, p.tw_np);
  if (active) {
    float* o0 = out + (size_t)j0 * p.n_t;
    float* o1 = o0 + p.n_t;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int idx = t + i * TPF;
      if (idx < p.n_t) {
        o0[idx] = v[i].x;
        if (has1) o1[idx] = v[i].y;
      }
    }
  }
  if (bad && w.status) atomicOr(&w.status[0], 1);
}

// ---------------------------------------------------------------------------
// K1b: common (angle-independent) row and coef.mean() per slice
// ---------------------------------------------------------------------------
// smem: [BUF float2][S][S][2 blockDim][H] floats.  The K1 partials are read
// through L2 (__ldcg): touched once, no reuse for L1.
template <int L>
__device__ __forceinline__ void k1b_slice(const DevPlan& p, const Work& w, int q, float2* smem) {
  using K = KShape<L>;
  constexpr int RPT = K::RPT, TPF = K::TPF;
  constexpr int H = L / 2;
  float2* buf = smem;
  float* cs = reinterpret_cast<float*>(smem + K::BUF);
  float* bm = cs + p.S;
  float* red = bm + p.S;  // [2 * blockDim]
  float* buf2 = red + 2 * blockDim.x;  // [H] real part of the common row
  const int t = threadIdx.x;
  const bool active = t < TPF;  // launched with K1B_THREADS >= TPF threads
  const float* part = w.part + (size_t)q * w.groups * p.S;
  __syncthreads();  // smem of the previous item released
  {
    // deterministic two-level sum over the K1 partial groups: warp wi sums
    // groups wi, wi + nw, ... (independent loads in flight) into the FFT buffer,
    // then a fixed-order sum over the nw warp partials
    float* wsum = reinterpret_cast<float*>(buf);
    const int nw = max(1, min((int)(blockDim.x >> 5), (2 * K::BUF) / max(p.S, 1)));
    const int wi = t >> 5, lane = t & 31;
    if (wi < nw) {
      for (int i = lane; i < p.S; i += 32) {
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
        int g = wi;
        for (; g + 3 * nw < w.groups; g += 4 * nw) {
          s0 += __ldcg(part + (size_t)g * p.S + i);
          s1 += __ldcg(part + (size_t)(g + nw) * p.S + i);
          s2 += __ldcg(part + (size_t)(g + 2 * nw) * p.S + i);
          s3 += __ldcg(part + (size_t)(g + 3 * nw) * p.S + i);
        }
        for (; g < w.groups; g += nw) s0 += __ldcg(part + (size_t)g * p.S + i);
        wsum[wi * p.S + i] = (s0 + s1) + (s2 + s3);
      }
    }
    __syncthreads();
    for (int i = t; i < p.S; i += blockDim.x) {
      float s = 0.f;
      for (int k = 0; k < nw; ++k) s += wsum[k * p.S + i];
      cs[i] = s;
    }
  }
  __syncthreads();
  float csum = 0.f;
  for (int i = t; i < p.S; i += blockDim.x) {
    const float m = (p.full_turn ? cs[i] : cs[i] + cs[p.S - 1 - i]) * p.inv_rows2;
    const float b = __ldg(p.bump_s + i) * m;
    bm[i] = b;
    csum += b;
  }
  // rect coefficient of the common row and mean of the per-row coefficients
  float asum = 0.f;
  for (int j = t; j < p.rows; j += blockDim.x) asum += __ldcg(w.rowcoef + (size_t)q * p.rows + j);
  red[t] = csum;
  red[t + blockDim.x] = asum;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (t < s) {
      red[t] += red[t + s];
      red[t + blockDim.x] += red[t + s + blockDim.x];
    }
    __syncthreads();
  }
  const float c = red[0] * p.inv_nt;
  const float amean = red[blockDim.x] / (float)p.rows;
  float2 v[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int idx = t + i * TPF;
    const int s = idx - p.lo;
    v[i] = make_float2((active && s >= 0 && s < p.S) ? bm[s] : 0.f, 0.f);
  }
  __syncthreads();
  fft<L, false>(v, buf, t, active, p.tw_L);
  if (active) {
    float2* out = w.common + (size_t)q * H;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int k = t + i * TPF;
      if (k < H) {
        const float2 ps = __ldg(p.psi + k), rh = __ldg(p.rho + k);
        float2 C = cmul(ps, v[i]);
        C = make_float2(fmaf(-c, rh.x, C.x), fmaf(-c, rh.y, C.y));
        if (k == 0) C = make_float2(0.f, 0.f);
        // half turn: the windowed mean row is symmetric in t, so C is real
        if (!p.full_turn) C.y = 0.f;
        out[k] = C;
        buf2[k] = C.x;
      }
    }
  }
  if (t == 0) w.coefmean[q] = amean + c;
  __syncthreads();
  float2* out2 = w.common2 + (size_t)q * p.c2pitch;
  for (int k = t; k < p.c2pitch; k += blockDim.x)
    out2[k] = k < H ? make_float2(buf2[k], buf2[min(k + 1, H - 1)]) : make_float2(0.f, 0.f);
}

template <int L>
__global__ void __launch_bounds__(KShape<L>::K1B_THREADS) k1b_common(DevPlan p, Work w) {
  extern __shared__ float2 smem[];
  k1b_slice<L>(p, w, blockIdx.x, smem);
}

// ---------------------------------------------------------------------------
// gridding table (fourier_bp.py:222-249): built once per plan in fp64.
// One entry per first-quadrant lattice node (|a|, |b|) in [0, H]^2, stored
// [|a|][|b|] so a Cartesian column reads it contiguously:
//   x = r0 (16 bits, 0xFFFF = outside the disc) | floor(tq) << 16
//   y = unorm16 frac(ri) | unorm16 frac(tq) << 16
// with ri = hypot(nu1, nu2)/df and tq = atan2(|nu2|, |nu1|) * 2V / (2 pi).
// The quantised fractions carry <= 2^-17 absolute weight error.
// ---------------------------------------------------------------------------
#ifdef TB_API_KERNELS  // non-template kernels: emitted by tb_api.cu only
__global__ void __launch_bounds__(256) build_grid_table(uint2* __restrict__ tab, int H, double dnu, double df,
                                                        double tscale, int nearest) {
  const long long count = (long long)(H + 1) * (H + 1);
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int a = (int)(i / (H + 1)), b = (int)(i % (H + 1));
  const int L = 2 * H;
  // numpy: fftfreq(L)[k] * L * dnu with index L/2 -> -L/2 (magnitude H)
  const double nu1 = ((double)a * (1.0 / L)) * L * dnu;
  const double nu2 = ((double)b * (1.0 / L)) * L * dnu;
  const double ri = hypot(nu1, nu2) / df;
  const double tq = atan2(nu2, nu1) * tscale;
  const int top = H - 1;
  int r0, qr, t0, qt;
  if (nearest) {
    // np.rint (half to even) decided here in fp64 (fourier_bp.py:234-236):
    // the entry holds the rounded indices with zero fractions
    r0 = (int)rint(ri);
    t0 = (int)rint(tq);
    qr = qt = 0;
  } else {
    const double rfl = floor(ri);
    r0 = (int)rfl;
    qr = (int)rint((ri - rfl) * 65536.0);
    if (qr >= 65536) { qr = 0; ++r0; }
    const double tfl = floor(tq);
    t0 = (int)tfl;
    qt = (int)rint((tq - tfl) * 65536.0);
    if (qt >= 65536) { qt = 0; ++t0; }
  }
  const bool inside = nearest ? (r0 <= top) : (ri <= (double)top);
  uint2 e;
  e.x = (uint32_t)(inside ? (r0 & 0xFFFF) : 0xFFFF) | ((uint32_t)t0 << 16);
  e.y = (uint32_t)qr | ((uint32_t)qt << 16);
  tab[i] = e;
}

// First-quadrant table of the half-turn bilinear path (fourier_bp.py:222-249
// per node, fp64): entry [a][b] for a, b in [0, H] (angle in [0, pi/2], polar
// rows t <= V/2).  K2 reads each entry for the node (a, b) and for the mirror
// (-a, b) (angle pi - theta: row coordinate V + 1 - y, angular weights
// swapped), the point reflection of the lower-half-plane node (a, -b):
//   x = ra + 1   texel coordinate of the 2x2 TLD4 footprint (ra, ra + 1);
//                H + 1 outside the disc (border texels: the gather is 0, and
//                common2[H] = 0)
//   y = t0 + 1   row coordinate within the slice's V + 1 rows
//   z, w = rf, tf  bilinear fractions, fp64-computed, rounded to fp32
//   nearest (K2_TEXN): x = ir + 0.5, y = it + 0.5 (texel centres, np.rint
//   of fourier_bp.py:234-236 in fp64), z = the row of the mirror node (a, -b)
//   as the reference rounds it (angle 2 pi - theta, minus V: the
//   conjugated half-turn row), w = 0; x = H + 0.5 outside the disc
__global__ void __launch_bounds__(256) build_grid_table2(float4* __restrict__ tab, int H, int V, double dnu,
                                                         double df, double tscale, int nearest) {
  const long long count = (long long)(H + 1) * (H + 1);
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int a = (int)(i / (H + 1)), b = (int)(i % (H + 1));
  const int L = 2 * H;
  const double nu1 = ((double)a * (1.0 / L)) * L * dnu;
  const double nu2 = ((double)b * (1.0 / L)) * L * dnu;
  const double ri = hypot(nu1, nu2) / df;
  const double ti = atan2(nu2, nu1) * tscale;  // angle in [0, pi/2]
  float4 e;
  if (nearest) {
    const int ir = (int)rint(ri);
    double pm = atan2(-nu2, nu1);  // the mirror node's own angle, np.mod(., 2 pi)
    if (pm < 0.0) pm += 2.0 * 3.14159265358979323846;
    int itm = (int)rint(pm * tscale) % (2 * V);
    itm = itm == 0 ? V : itm - V;  // extended row 2V (= 0) is the conjugate of texture row V
    if (ir <= H - 1)
      e = make_float4((float)ir + 0.5f, (float)rint(ti) + 0.5f, (float)itm + 0.5f, 0.f);
    else
      e = make_float4((float)H + 0.5f, 0.5f, 0.5f, 0.f);
  } else if (ri <= (double)(H - 1)) {
    const double rfl = floor(ri);
    const double tfl = floor(ti);
    e = make_float4((float)(rfl + 1.0), (float)(tfl + 1.0), (float)(ri - rfl), (float)(ti - tfl));
  } else {
    e = make_float4((float)(H + 1), 1.f, 0.f, 0.f);
  }
  tab[i] = e;
}

// Per column a of the first-quadrant table: the largest b whose node lies
// inside the disc (x <= H), -1 if none.  One CTA per column.
__global__ void __launch_bounds__(256) build_col_extent(const float4* __restrict__ tab, int* __restrict__ ext, int H) {
  const int a = blockIdx.x;
  int m = -1;
  for (int b = threadIdx.x; b <= H; b += blockDim.x)
    if (tab[(size_t)a * (H + 1) + b].x <= (float)H) m = max(m, b);
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ int red[8];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) m = max(m, red[i]);
    ext[a] = max(m, red[0]);
  }
}
#endif

// polar sample P(t, r) of the full circle; rows t >= V of half-turn input are
// the conjugate mirror (fourier_bp.py:302-311; SURVEY.md finding 2)
__device__ __forceinline__ float2 polar_at(const DevPlan& p, const float2* __restrict__ pol, int t, int r) {
  const bool mirror = !p.full_turn && t >= p.n_theta;
  const int row = mirror ? t - p.n_theta : t;
  float2 v = __ldg(pol + (size_t)row * p.H + r);
  if (mirror) v.y = -v.y;
  return v;
}

// interpolated, modulated lattice value C(as, bs) (fourier_bp.py:389-407, 427-430)
__device__ __forceinline__ float2 lattice_value(const DevPlan& p, const uint2* __restrict__ tab,
                                                const float2* __restrict__ pol, const float2* __restrict__ com,
                                                int as, int bs) {
  const int aa = as < 0 ? -as : as, ab = bs < 0 ? -bs : bs;
  const uint2 e = __ldg(tab + (size_t)aa * (p.H + 1) + ab);
  const int r0 = (int)(e.x & 0xFFFFu);
  if (r0 == 0xFFFF) return make_float2(0.f, 0.f);
  const int I = (int)(e.x >> 16);
  const int qr = (int)(e.y & 0xFFFFu);
  int qt = (int)(e.y >> 16);
  // full angle from the first-quadrant angle tq = I + qt/65536
  const int V = p.n_theta, rows2 = 2 * V;
  int t0;
  if ((as < 0) == (bs < 0)) {
    t0 = as < 0 ? V + I : I;               // quadrants 1 and 3: base + tq
  } else {
    const int base = as < 0 ? V : rows2;   // quadrants 2 and 4: base - tq
    if (qt == 0) t0 = base - I;
    else { t0 = base - I - 1; qt = 65536 - qt; }
  }
  if (t0 >= rows2) t0 -= rows2;
  const int top = p.H - 1;
  float2 val;
  if (p.interp == 0) {
    const float rf = (float)qr * (1.f / 65536.f), tf = (float)qt * (1.f / 65536.f);
    const int ra = r0, rb = min(r0 + 1, top);
    const int t1 = t0 + 1 == rows2 ? 0 : t0 + 1;
    const float2 p00 = polar_at(p, pol, t0, ra), p01 = polar_at(p, pol, t0, rb);
    const float2 p10 = polar_at(p, pol, t1, ra), p11 = polar_at(p, pol, t1, rb);
    const float2 c0 = __ldg(com + ra), c1 = __ldg(com + rb);
    const float2 r0v = make_float2(fmaf(rf, p01.x - p00.x, p00.x), fmaf(rf, p01.y - p00.y, p00.y));
    const float2 r1v = make_float2(fmaf(rf, p11.x - p10.x, p10.x), fmaf(rf, p11.y - p10.y, p10.y));
    const float2 cv = make_float2(fmaf(rf, c1.x - c0.x, c0.x), fmaf(rf, c1.y - c0.y, c0.y));
    val = make_float2(fmaf(tf, r1v.x - r0v.x, r0v.x) + cv.x, fmaf(tf, r1v.y - r0v.y, r0v.y) + cv.y);
  } else {
    // np.rint (half to even) on both coordinates (fourier_bp.py:234-238)
    const int ir = r0 + ((qr > 32768 || (qr == 32768 && (r0 & 1))) ? 1 : 0);
    int it = t0 + ((qt > 32768 || (qt == 32768 && (t0 & 1))) ? 1 : 0);
    if (it >= rows2) it -= rows2;
    const float2 pv = polar_at(p, pol, it, ir);
    const float2 cv = __ldg(com + ir);
    val = make_float2(pv.x + cv.x, pv.y + cv.y);
  }
  if (p.has_mod) {
    const int L = p.L;
    val = cmul(val, cmul(__ldg(p.modt + (as & (L - 1))), __ldg(p.modt + (bs & (L - 1)))));
  }
  return val;
}

// Decoded gridding node: polar corners (t0|t1, ra|rb) and bilinear weights.
struct GridNode {
  int t0, t1, ra, rb;
  float rf, tf;
  bool inside;
};

// full-angle node from a first-quadrant table entry (see build_grid_table)
__device__ __forceinline__ GridNode decode_node(const DevPlan& p, uint2 e, int as, int bs) {
  GridNode g;
  const int r0 = (int)(e.x & 0xFFFFu);
  g.inside = r0 != 0xFFFF;
  const int I = (int)(e.x >> 16);
  int qt = (int)(e.y >> 16);
  const int V = p.n_theta, rows2 = 2 * V;
  int t0;
  if ((as < 0) == (bs < 0)) {
    t0 = as < 0 ? V + I : I;
  } else {
    const int base = as < 0 ? V : rows2;
    if (qt == 0) t0 = base - I;
    else { t0 = base - I - 1; qt = 65536 - qt; }
  }
  if (t0 >= rows2) t0 -= rows2;
  g.t0 = t0;
  g.t1 = t0 + 1 == rows2 ? 0 : t0 + 1;
  g.ra = g.inside ? r0 : 0;
  g.rb = g.inside ? min(r0 + 1, p.H - 1) : 0;
  g.rf = (float)(e.y & 0xFFFFu) * (1.f / 65536.f);
  g.tf = (float)qt * (1.f / 65536.f);
  return g;
}

// K2 -> K3 intermediate: [B][ceil(n/4)][H+1][4] complex (4-row tiles = one
// 32-byte sector per (tile, column)), so K2's column stores and K3's row-pair
// loads both move whole sectors.
#ifndef TB_COL_TILE
#define TB_COL_TILE 4
#endif
constexpr int kColTile = TB_COL_TILE;  // rows per (tile, column) group of the K2 -> K3 intermediate
__device__ __forceinline__ size_t col_index(int H, int m2, int a) {
  return ((size_t)(m2 / kColTile) * (H + 1) + a) * kColTile + (m2 % kColTile);
}

// ---------------------------------------------------------------------------
// K2: gather + IFFT along k2 for one Cartesian column a in [0, H]
// (device body; every thread of the CTA must call it -- FFT barriers)
// ---------------------------------------------------------------------------
// table entry, streamed past L1 (read once per column; keeps L1 for polar texels)
__device__ __forceinline__ uint2 ld_table(const uint2* p) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}

// half-plane table entry (16 B), streamed past L1
__device__ __forceinline__ float4 ld_table4(const float4* p) {
  float4 v;
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p));
  return v;
}

// K2 kernel: CTA of G column groups (G*TPF = 512 threads for L <= 8192)
// sweeping a contiguous run of columns G at a time.  Adjacent columns read
// nearly the same polar lines, so the SM's L1 keeps the shared footprint of
// the G concurrent columns and of the next step resident.
#ifndef TB_K2_RPT
#define TB_K2_RPT 16
#endif
// A/B instrumentation only (results are wrong when set): 1 = no gather, 2 = no column
// transform, 3 = one TLD4 per node (real part reused), 4 = 3 without the transform,
// 5 = every TLD4 on border texels
#ifndef TB_K2_DBG
#define TB_K2_DBG 0
#endif
template <int L>
struct K2Shape {
  // points per thread of the column transform (TB_K2_RPT, capped at the
  // default for small L)
  static constexpr int RPT = TB_K2_RPT < default_rpt(L) ? TB_K2_RPT : default_rpt(L);
  using S = FftShape<L, RPT>;
  static constexpr int TPF = S::TPF;
#ifndef TB_K2_THREADS
#define TB_K2_THREADS 256
#endif
  static constexpr int G = TPF >= TB_K2_THREADS ? 1 : TB_K2_THREADS / TPF;
  static constexpr int THREADS = G * TPF;
// CTAs per SM asked of ptxas for <= 256-thread K2 CTAs: 4 (64 registers),
// 5 at L = 4096 (48 registers).  Round 1: a fourth resident column hid more
// gather latency than its spills cost (K2 101.5 -> 95.3 ms at 2048^3); with
// the leaner pair gather a fifth pays at 2048^3 only (below)
#ifndef TB_K2_MINB
#define TB_K2_MINB 4
#endif
// L = 4096 (2048^3): 5 CTAs per SM (48 registers, no spills with the pair
// gather): step 160.1-160.4 -> 159.1-159.4 ms; at 1024^3 / 512^3 the fifth
// CTA costs (19.79 -> 20.21, 2.52 -> 2.56 ms), so 4 there
#ifndef TB_K2_MINB_4096
#define TB_K2_MINB_4096 5
#endif
#define TB_K2_MINB_L(L) ((L) == 4096 ? TB_K2_MINB_4096 : TB_K2_MINB)
#ifndef TB_K2_NAMED
#define TB_K2_NAMED 1
#endif
#ifndef TB_K2_MINB512
#define TB_K2_MINB512 2
#endif
  static constexpr int MINB = THREADS <= 256 ? TB_K2_MINB_L(L) : (THREADS <= 512 ? TB_K2_MINB512 : 1);
  static constexpr int SMEM_PER_GROUP = KShape<L>::BUF;  // float2 FFT buffer (+ gather staging)
};

// Finished nodes are staged in the FFT buffer (thread-private slots: node i
// of thread t at smem[i * TPF + t]) so they leave registers during the
// latency-bound gather; a barrier separates the reload from the first FFT
// pass, which rewrites the buffer.
// K2 gather variants, chosen per plan on the host (each its own kernel so
// ptxas allocates registers for one path only):
//   K2_TEX   half-turn bilinear, TLD4 gathers driven by the half-plane table
//   K2_PLAIN half-turn bilinear, plain loads (polar texture view unavailable)
//   K2_ANY   nearest interpolation, or no texture view (lattice_value)
//   K2_TEXF  full-turn bilinear, TLD4 gathers of both half planes
//   K2_TEXN  half-turn nearest, one point-sampled texel per node
enum { K2_ANY = 0, K2_PLAIN = 1, K2_TEX = 2, K2_TEXF = 3, K2_TEXN = 4 };

template <int L, bool CROP_HALF, int PATH, class Sync>
__device__ __forceinline__ void k2_column(const DevPlan& p, const Work& w, int a, int q, int t, bool active,
                                          float2* smem, Sync sync) {
  float2* stg = smem;
  using K2 = K2Shape<L>;
  constexpr int RPT = K2::RPT, TPF = K2::TPF;
  constexpr int H = L / 2;
  const int as = a < H ? a : -H;
  const float2* pol = w.polar + (size_t)q * p.prow * H;
  const float2* com = w.common + (size_t)q * H;
  const uint2* tab = p.gridtab;
  float2 v[RPT];
  // TLD4 paths: K2_TEX (half turn), K2_TEXF (full turn)
  constexpr bool TEXP = PATH == K2_TEX || PATH == K2_TEXF || PATH == K2_TEXN;
  constexpr bool FULL = PATH == K2_TEXF;
  constexpr bool NEAR = PATH == K2_TEXN;
  if constexpr (PATH != K2_ANY) {
    // Bilinear fast paths.  A node in the lower half plane (b < 0) is the
    // conjugate of its point reflection (-a, -b), which lies in the upper
    // half plane (the lattice is Hermitian: .real of ifft2; for full-turn
    // input the Hermitian part is formed explicitly), so no per-corner
    // mirror logic.
    const float2* com2 = w.common2 + (size_t)q * p.c2pitch;
    const uint2* trow = tab + (size_t)a * (H + 1);
    const int V = p.n_theta;
    // M[a] M[b] with M[b] = M[t] M[TPF i]: the column factor M[a] folds into
    // the per-thread factor once per column
    // CROP_HALF with the TLD4 path: the half-node modulation M[a] M[b] is
    // exp(i pi (a + b) / L); its per-thread part rides in the column IFFT's
    // twiddles (fft_mod), its per-slot part is a constant 32nd root below,
    // and M[a] multiplies the kept outputs
    constexpr bool MODF = CROP_HALF && TEXP;
    const float2 m_t = (p.has_mod && active && !MODF) ? cmul(__ldg(p.modt + t), __ldg(p.modt + (as & (L - 1))))
                                                      : make_float2(1.f, 0.f);
#ifndef TB_K2_NB
#define TB_K2_NB 4
#endif
    constexpr int NB = TB_K2_NB < RPT ? TB_K2_NB : RPT;
    if constexpr (PATH == K2_TEX && TB_K2_DBG == 1) {
      // A/B only: no gather (time the column transform alone)
#pragma unroll
      for (int i = 0; i < RPT; ++i) if (active) stg[i * TPF + t] = make_float2((float)i, (float)t);
    } else if constexpr (TEXP) {
    // Mirrored-pair gather over the first-quadrant table.  Entry b' = t +
    // TPF j of column a drives two nodes: the direct node (a, b') and the
    // lower-half-plane node b = L - b', whose point reflection (-a, b') is
    // the entry's mirror about the k2 axis: angle pi - theta, i.e. texel row
    // V + 1 - y with the angular weights swapped, same radius (same common
    // row pair).  So one table load and one common-row load serve two nodes.
    // The mirror node lands in slot RPT-1-j of thread TPF - t (thread 0's
    // first mirror is b' = H instead: b' = 0 has no mirror and b = H no
    // direct node), so a barrier precedes the reload.
    // Software pipeline over the RPT nodes d0, m0, d1, m1, ...: TLD4 gathers
    // AH nodes ahead, the table entry of a pair before its first gather.
    // Nodes outside the disc read border texels (0) and common2[H] (0).
    // Full turn (K2_TEXF): a node is the Hermitian part 0.5 (C(k) + conj
    // C(-k)) (fourier_bp.py:431): its polar sample at angle theta and the
    // one at theta + pi (rows y + V), and for the mirror node at pi - theta
    // and 2 pi - theta (rows V + 1 - y and 2V + 1 - y; row 2V repeats row 0),
    // four TLD4s per node; the common row's Hermitian part is its real part.
#ifdef TB_K2_AHEAD
    constexpr int AH = TB_K2_AHEAD;
#else
    constexpr int AH = FULL ? 1 : 2;
#endif
    constexpr int NJ = RPT / 2;
    const float4* qrow = p.gridtab2 + (size_t)a * (H + 1);
    const float fyoff = (float)(q * p.prow);
    const float fymir = fyoff + (float)(V + 1);
    const float fyhalf = fyoff + (float)V, fymir2 = fyoff + (float)(2 * V + 1);  // full turn
    const int mb0 = t == 0 ? H : L - t;  // staging index of pair 0's mirror node
    // per-slot part of the half-node modulation (fft_mod input): slot s holds
    // b = t + TPF s, b_signed = b - L for s >= RPT/2: exp(i pi TPF s / L) =
    // exp(2 pi i (16 s / RPT) / 32), times -1 in the lower half
    auto slot_e = [](int s) { return 16 * s / RPT + (s >= RPT / 2 ? 16 : 0); };
    const float2 ma = (!MODF && p.has_mod) ? __ldg(p.modt + (as & (L - 1))) : make_float2(1.f, 0.f);
    float4 e[NJ];
    float4 em0;
    float4 fre[RPT], fim[RPT];
    float4 fre2[FULL ? RPT : 1], fim2[FULL ? RPT : 1];
    float2 cc[NJ], ccm0;
    auto tload = [&](int j) {
      e[j] = ld_table4(qrow + t + j * TPF);
      if (j == 0) em0 = t == 0 ? ld_table4(qrow + H) : e[0];
    };
    auto entry = [&](int k) { return k == 1 ? em0 : e[k >> 1]; };
#ifndef TB_K2_SKIP
#define TB_K2_SKIP 2
#endif
    // Outside-disc skip: a TLD4 on border texels costs the TEX path nearly
    // as much as a real one (all-border A/B: K2 67 vs 79 ms), so a warp whose
    // 32 entries b' = (t & ~31) + lane + TPF j all lie beyond the column's
    // inside extent (colext, largest inside b') gathers nothing and stages
    // zeros.  The predicate is warp-uniform arithmetic (no vote).  1 =
    // predicated TLD4s only (measured slower: 82.0 vs 78.9 ms), 2 = leave
    // the pipeline after the warp's last live pair (78.3-78.8 ms), 0 = off.
    const int bext = TB_K2_SKIP ? __ldg(p.colext + a) : L;
    const int wb = t & ~31;
    auto live = [&](int j) { return wb + j * TPF <= bext; };
    auto fetch = [&](int k) {
      float4 d = entry(k);
      if (TB_K2_DBG == 5) d.x = (float)(H + 1);  // A/B: every gather on border texels
      const float y = (k & 1) ? fymir - d.y : d.y + fyoff;
      if (live(k >> 1)) {
        if constexpr (NEAR) {
          // the entry's z is the mirror's own rounded row (np.rint in fp64)
          const float2 v = tex2D<float2>(w.polar_tex, d.x, (k & 1) ? d.z + fyoff : d.y + fyoff);
          fre[k] = make_float4(v.x, v.y, 0.f, 0.f);
        } else {
          fre[k] = tex2Dgather<float4>(w.polar_tex, d.x, y, 0);
          if (TB_K2_DBG == 3 || TB_K2_DBG == 4) fim[k] = fre[k];
          else fim[k] = tex2Dgather<float4>(w.polar_tex, d.x, y, 1);
        }
        if constexpr (FULL) {
          const float y2 = (k & 1) ? fymir2 - d.y : d.y + fyhalf;
          fre2[k] = tex2Dgather<float4>(w.polar_tex, d.x, y2, 0);
          fim2[k] = tex2Dgather<float4>(w.polar_tex, d.x, y2, 1);
        }
        // common-row pair at r0 (bilinear: x = r0 + 1; nearest: x = ir + 0.5)
        const int rc = NEAR ? (int)d.x : (int)d.x - 1;
        if ((k & 1) == 0) cc[k >> 1] = __ldg(com2 + rc);
        if (k == 1) ccm0 = __ldg(com2 + rc);
      } else {
        fre[k] = fim[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if constexpr (FULL) fre2[k] = fim2[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if ((k & 1) == 0) cc[k >> 1] = make_float2(0.f, 0.f);
        if (k == 1) ccm0 = make_float2(0.f, 0.f);
      }
    };
    auto consume = [&](int k) {
      const int j = k >> 1;
      const bool mir = k & 1;
      const float4 d = entry(k);
      const float2 c = k == 1 ? ccm0 : cc[j];
      const float r = d.z, u = d.w;
      // bilinear value of a TLD4 pair; mirror: the lower texel row carries
      // the weight u of the entry
      auto bil = [&](const float4 re, const float4 im) {
        const float2 p00 = make_float2(re.w, im.w), p01 = make_float2(re.z, im.z);
        const float2 p10 = make_float2(re.x, im.x), p11 = make_float2(re.y, im.y);
        const float2 r0v = make_float2(fmaf(r, p01.x - p00.x, p00.x), fmaf(r, p01.y - p00.y, p00.y));
        const float2 r1v = make_float2(fmaf(r, p11.x - p10.x, p10.x), fmaf(r, p11.y - p10.y, p10.y));
        const float2 lo = mir ? r1v : r0v, hi = mir ? r0v : r1v;
        return make_float2(fmaf(u, hi.x - lo.x, lo.x), fmaf(u, hi.y - lo.y, lo.y));
      };
      float2 val;
      if constexpr (NEAR) {
        // the sample at (it, ir) plus the real common row at ir
        const float2 v = make_float2(fre[k].x, fre[k].y);
        val = mir ? cconj(v) : v;
        val.x += c.x;
      } else if constexpr (FULL) {
        const float2 b1 = bil(fre[k], fim[k]);
        // direct: 0.5 (C(theta) + conj C(theta + pi)); mirror (conjugate of
        // the reflection): 0.5 (conj C(pi - theta) + C(2 pi - theta))
        const float2 b2 = bil(fre2[k], fim2[k]);
        val = make_float2(0.5f * (b1.x + b2.x), mir ? 0.5f * (b2.y - b1.y) : 0.5f * (b1.y - b2.y));
        val.x += fmaf(r, c.y - c.x, c.x);
      } else {
        const float2 b1 = bil(fre[k], fim[k]);
        val = mir ? cconj(b1) : b1;  // lower half plane: conjugate of the reflection
        val.x += fmaf(r, c.y - c.x, c.x);
      }
      const int idx = mir ? (j == 0 ? mb0 : (L - t) - j * TPF) : t + j * TPF;
      if constexpr (MODF)  // exp(i pi b_signed / L) / exp(i pi t_owner / L), slot j or RPT-1-j
        val = mul_e32(val, slot_e(mir ? RPT - 1 - j : j));
      else if (p.has_mod)
        val = cmul(val, cmul(ma, __ldg(p.modt + idx)));
      if (active) stg[idx] = val;
    };
#pragma unroll
    for (int j = 0; 2 * j <= AH && j < NJ; ++j) tload(j);
#pragma unroll
    for (int k = 0; k < AH && k < RPT; ++k) fetch(k);
#if TB_K2_SKIP == 2
    // the warp's live pairs are j < nlive (entries increase with j): leave
    // the pipeline after the last one (a warp-uniform branch, so the dead
    // pairs issue no TLD4 at all) and stage zeros for the rest
    const int nlive = bext < wb ? 0 : min(NJ, (bext - wb) / TPF + 1);
    int jdone = NJ;
#endif
#pragma unroll
    for (int g = 0; g < RPT; ++g) {
      const int kt = g + AH + 1;
      if (kt < RPT && (kt & 1) == 0) tload(kt >> 1);
      if (g + AH < RPT) fetch(g + AH);
      consume(g);
#if TB_K2_SKIP == 2
      if ((g & 1) && g + 1 < RPT && ((g + 1) >> 1) >= nlive) {
        jdone = (g + 1) >> 1;
        break;
      }
#endif
    }
#if TB_K2_SKIP == 2
    if (active)
      for (int j = jdone; j < NJ; ++j) {
        stg[t + j * TPF] = make_float2(0.f, 0.f);
        stg[j == 0 ? mb0 : (L - t) - j * TPF] = make_float2(0.f, 0.f);
      }
#endif
    sync();  // mirror nodes went to other threads' slots
    if (MODF && t == 0 && active) {
      // thread 0 owns the mirrors of its own entries b' = TPF j (slot RPT - j,
      // not RPT-1-j) and of b' = H (slot RPT/2): fix their slot constants
      stg[(RPT / 2) * TPF] = mul_e32(stg[(RPT / 2) * TPF], slot_e(RPT / 2) - slot_e(RPT - 1) + 32);
#pragma unroll
      for (int i = RPT / 2 + 1; i < RPT; ++i) stg[i * TPF] = mul_e32(stg[i * TPF], slot_e(i) - slot_e(i - 1));
    }
    } else {  // plain-load gathers (no texture view: too many rows, or TB_NOTEX)
    uint2 en[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      const int b = t + j * TPF;
      const int ab = b <= H ? b : L - b;
      en[j] = active ? ld_table(trow + ab) : make_uint2(0xFFFFu, 0u);
    }
#pragma unroll
    for (int c = 0; c < RPT; c += NB) {
      uint2 e[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) e[j] = en[j];
      if (c + NB < RPT) {
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          const int b = t + (c + NB + j) * TPF;
          const int ab = b <= H ? b : L - b;
          en[j] = active ? ld_table(trow + ab) : make_uint2(0xFFFFu, 0u);
        }
      }
      float2 p00[NB], p01[NB], p10[NB], p11[NB], cc[NB], mb[NB];
      float rf[NB], tf[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int b = t + (c + j) * TPF;
        const int bs = b < H ? b : b - L;
        const uint2 ej = e[j];
        const int r0 = (int)(ej.x & 0xFFFFu);
        const int ra = r0 == 0xFFFF ? 0 : r0;
        const int rb = min(ra + 1, H - 1);
        const int I = (int)(ej.x >> 16);
        int qt = (int)(ej.y >> 16);
        const bool flip = (as < 0) != (bs < 0);  // effective a < 0 after reflection
        int t0 = I;
        if (flip) {
          t0 = qt ? V - I - 1 : V - I;
          qt = qt ? 65536 - qt : 0;
        }
        const float2 z = make_float2(0.f, 0.f);
        const bool in = r0 != 0xFFFF;  // nodes outside the disc are masked below
        const float2* row0 = pol + (size_t)t0 * H;
        p00[j] = in ? __ldg(row0 + ra) : z;
        p01[j] = in ? __ldg(row0 + rb) : z;
        p10[j] = in ? __ldg(row0 + H + ra) : z;
        p11[j] = in ? __ldg(row0 + H + rb) : z;
        cc[j] = __ldg(com2 + ra);
        // M[b] = M[t] * M[TPF*i] (linear phase in the signed index): one
        // per-thread load plus a warp-uniform one instead of a load per node
        mb[j] = p.has_mod ? cmul(m_t, __ldg(p.modt + (c + j) * TPF)) : make_float2(1.f, 0.f);
        rf[j] = (float)(ej.y & 0xFFFFu) * (1.f / 65536.f);
        tf[j] = (float)qt * (1.f / 65536.f);
      }
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const int b = t + (c + j) * TPF;
        const bool lower = b >= H;  // bs < 0 (index H is -L/2)
        const float r = rf[j], u = tf[j];
        const float2 r0v = make_float2(fmaf(r, p01[j].x - p00[j].x, p00[j].x), fmaf(r, p01[j].y - p00[j].y, p00[j].y));
        const float2 r1v = make_float2(fmaf(r, p11[j].x - p10[j].x, p10[j].x), fmaf(r, p11[j].y - p10[j].y, p10[j].y));
        float2 val = make_float2(fmaf(u, r1v.x - r0v.x, r0v.x) + fmaf(r, cc[j].y - cc[j].x, cc[j].x),
                                 fmaf(u, r1v.y - r0v.y, r0v.y));
        if (lower) val.y = -val.y;
        if (p.has_mod) val = cmul(val, mb[j]);
        if (active) stg[(c + j) * TPF + t] = ((e[j].x & 0xFFFFu) == 0xFFFFu) ? make_float2(0.f, 0.f) : val;
      }
    }
    }
    if (p.nyq && active) {
      // Nyquist lines: Hermitian part 0.5 (C[k] + conj C[-k mod L]) of the fully
      // modulated lattice (.real of ifft2, fourier_bp.py:431)
#pragma unroll 1
      for (int i = 0; i < RPT; ++i) {
        const int b = t + i * TPF;
        if (a == H || b == H) {
          const int bs = b < H ? b : b - L;
          const int pa = as == -H ? -H : -as;
          const int pb = bs == -H ? -H : -bs;
          const float2 c0 = lattice_value(p, tab, pol, com, as, bs);
          const float2 m = lattice_value(p, tab, pol, com, pa, pb);
          float2 hv = make_float2(0.5f * (c0.x + m.x), 0.5f * (c0.y - m.y));
          if (TEXP && CROP_HALF)  // fft_mod input: without M[a] M[t]
            hv = cmul(hv, cconj(cmul(__ldg(p.modt + t), __ldg(p.modt + (as & (L - 1))))));
          stg[i * TPF + t] = hv;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < RPT; ++i) v[i] = active ? stg[i * TPF + t] : make_float2(0.f, 0.f);
    sync();  // every thread holds its nodes before the FFT rewrites the buffer
  } else {
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      float2 val = make_float2(0.f, 0.f);
      if (active) {
        const int b = t + i * TPF;
        const int bs = b < H ? b : b - L;
        val = lattice_value(p, tab, pol, com, as, bs);
        // Hermitian part: 0.5 (C[k] + conj C[-k mod L]) (.real of ifft2, fourier_bp.py:431)
        if (p.full_turn || (p.nyq && (a == H || b == H))) {
          const int pa = as == -H ? -H : -as;
          const int pb = bs == -H ? -H : -bs;
          const float2 m = lattice_value(p, tab, pol, com, pa, pb);
          val = make_float2(0.5f * (val.x + m.x), 0.5f * (val.y - m.y));
        }
      }
      v[i] = val;
    }
  }
  if constexpr (TEXP && CROP_HALF) {
    if (TB_K2_DBG != 2 && TB_K2_DBG != 4) fft_mod<L, true, Sync, RPT>(v, smem, t, active, p.twm, sync);
    const float2 ma = __ldg(p.modt + (as & (L - 1)));
#pragma unroll
    for (int i = 0; i < RPT; ++i)
      if (i < RPT / 4 || i >= 3 * RPT / 4) v[i] = cmul(v[i], ma);  // the kept rows
  } else {
    fft<L, true, Sync, RPT>(v, smem, t, active, p.tw_L, sync);
  }
  if (active) {
    float2* out = w.columns + (size_t)q * p.col_slice;
    if constexpr (CROP_HALF) {
      // n = L/2: the kept rows are i < RPT/4 (m2 = t + i TPF + L/4) and
      // i >= 3 RPT/4 (m2 = t + (i - 3 RPT/4) TPF); m2 = t + c_i with c_i a
      // multiple of 4, so col_index is one per-thread base plus a
      // compile-time tile offset (the other slots are DCE'd)
      float2* ob = out + (((size_t)(t / kColTile) * (H + 1) + a) * kColTile + (t % kColTile));
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        if (i < RPT / 4 || i >= 3 * RPT / 4) {
          const int c = i < RPT / 4 ? i * TPF + L / 4 : (i - 3 * RPT / 4) * TPF;
          ob[(size_t)(c / kColTile) * (H + 1) * kColTile] = v[i];
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int m2 = (t + i * TPF + p.n_half) & (L - 1);
        if (m2 < p.n) out[col_index(H, m2, a)] = v[i];
      }
    }
  }
}

// one K2 block: column group cg x slice group sg
template <int L, bool CROP_HALF, int PATH>
__device__ __forceinline__ void k2_block(const DevPlan& p, const Work& w, int cg, int sg, int cols_per_cta,
                                         int slices_per_cta, int n_slices, float2* smem) {
  using K2 = K2Shape<L>;
  constexpr int TPF = K2::TPF;
  constexpr int H = L / 2;
  const int g = threadIdx.x / TPF;
  const int t = threadIdx.x % TPF;
  float2* buf = smem + g * K2::SMEM_PER_GROUP;
  const int q0 = sg * slices_per_cta;
  const int q1 = min(n_slices, q0 + slices_per_cta);
  const int c0 = cg * cols_per_cta;
  const int c1 = min(H + 1, c0 + cols_per_cta);
  if constexpr (K2::G == 1) {
    for (int a = c0; a < c1; ++a)
      for (int q = q0; q < q1; ++q) {
        k2_column<L, CROP_HALF, PATH>(p, w, a, q, t, true, buf, CtaSync());
        __syncthreads();  // buffer reuse by the next column
      }
  } else if constexpr (TPF % 32 == 0 && K2::G < 16 && TB_K2_NAMED) {
    // G column groups side by side on one SM (adjacent columns at the same
    // time share their polar lines in L1), each synchronising only itself
    // through its own named barrier: no coupling between the groups
    const GroupSync gs{1 + g, TPF};
    for (int a = c0 + g; a < c1; a += K2::G)
      for (int q = q0; q < q1; ++q) {
        k2_column<L, CROP_HALF, PATH>(p, w, a, q, t, true, buf, gs);
        gs();  // buffer reuse by the next column
      }
  } else {
    // sub-warp groups (small L): CTA-wide barriers, idle groups on the tail
    for (int base = c0; base < c1; base += K2::G) {
      const int a = base + g;
      const bool valid = a < c1;
      for (int q = q0; q < q1; ++q) {
        k2_column<L, CROP_HALF, PATH>(p, w, valid ? a : c1 - 1, q, t, valid, buf, CtaSync());
        __syncthreads();  // buffer reuse by the next column
      }
    }
  }
}

template <int L, bool CROP_HALF, int PATH>
// the fifth CTA per SM at L = 4096 only for the lean TLD4 paths (half-turn
// bilinear / nearest); the full-turn and plain paths keep 4 (they spill at 48
// registers: full turn 0.128 -> 0.133 ms per 2048^2 slice)
__global__ void __launch_bounds__(K2Shape<L>::THREADS,
                                  (PATH == K2_TEX || PATH == K2_TEXN) ? K2Shape<L>::MINB
                                                                      : (K2Shape<L>::MINB > 4 ? 4 : K2Shape<L>::MINB))
    k2_columns(DevPlan p, Work w, int cols_per_cta, int slices_per_cta, int n_slices, int slice_fast) {
  extern __shared__ float2 smem[];
  // CTA = a run of columns x a run of slices; slice_fast puts the slice runs
  // on blockIdx.x so the resident CTAs share their columns' table rows
  const int cg = slice_fast ? blockIdx.y : blockIdx.x;
  const int sg = slice_fast ? blockIdx.x : blockIdx.y;
  k2_block<L, CROP_HALF, PATH>(p, w, cg, sg, cols_per_cta, slices_per_cta, n_slices, smem);
}

// ---------------------------------------------------------------------------
// K3: C2R along k1 for a tile of 4 output rows (two packed pairs) + epilogue
// ---------------------------------------------------------------------------

// atan(s) for s in [0, 1] (s <= 1: pixel centres satisfy r^2 < 2): s P(s^2)
// with a degree-8 least-max-error fit, 1.1e-7 max abs error in fp32 (as good
// as asinf; 9 FMAs instead of asinf's branches and square root)
__device__ __forceinline__ float atan01(float s) {
  const float z = s * s;
  float q = 0.0024567015934735537f;
  q = fmaf(q, z, -0.014401277527213097f);
  q = fmaf(q, z, 0.0397811196744442f);
  q = fmaf(q, z, -0.07234852015972137f);
  q = fmaf(q, z, 0.10498946160078049f);
  q = fmaf(q, z, -0.14161230623722076f);
  q = fmaf(q, z, 0.19985906779766083f);
  q = fmaf(q, z, -0.33332598209381104f);
  q = fmaf(q, z, 0.9999998807907104f);
  return s * q;
}

// One 4-row output tile (two packed row pairs) of the slice in workspace
// slot q, written to img_slice [n][n].  The K2 columns
// already carry the full half-node modulation M[a] M[b].  `chk` accumulates
// out * 0 (NaN for any non-finite output) for the caller's status flag.
template <int L, bool CROP_HALF>
__device__ __forceinline__ void k3_tile(const DevPlan& p, const Work& w, float* __restrict__ img_slice, float out_scale,
                                        int q, int tile, float2* smem, float& chk) {
  using K = KShape<L>;
  constexpr int RPT = K::RPT, TPF = K::TPF;
  constexpr int H = L / 2;
  const int t = threadIdx.x;
  // blocks are exactly TPF threads once TPF >= 32: compile-time true there
  const bool active = TPF >= 32 || t < TPF;
  const int n = p.n;
  const float2* Gs = w.columns + (size_t)q * p.col_slice;
  const float cm = __ldcg(w.coefmean + q);  // written by another CTA (K1b)
  const float inv_n = 2.f / (float)n;
  const float A = p.img_scale * out_scale;       // amplitude / L^2 / (2 pi)
  const float cmo = cm * out_scale;               // coef_mean / (2 pi)
  const float Bpi = cmo * 3.14159265358979323846f;  // inside the unit circle
  const float cm2 = -2.f * cmo;
  const float xt = fmaf((float)t, inv_n, 0.5f * inv_n - 1.f);  // x of column t (+ i TPF inv_n)
  for (int pair = 0; pair < 2; ++pair) {
    const int m2a = 4 * tile + 2 * pair, m2b = m2a + 1;
    // n = L/2 (CROP_HALF) is a multiple of 4: every tile holds 4 rows
    if (!CROP_HALF && m2a >= n) break;  // uniform across the CTA
    const bool hasb = CROP_HALF || m2b < n;
    // the pair's two rows: 16 B per column at stride kColTile complex
    const float2* G = Gs + (size_t)(m2a / kColTile) * (H + 1) * kColTile + (m2a % kColTile);
    float2 v[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      float2 z = make_float2(0.f, 0.f);
      if (active) {
        // a = t + i TPF; bins a > H are the conjugates of L - a (i >= RPT/2)
        const int ar = (i < RPT / 2) ? t + i * TPF : L - (t + i * TPF);
        const float4 g = __ldg(reinterpret_cast<const float4*>(G + (size_t)ar * kColTile));
        float2 ga = make_float2(g.x, g.y);
        float2 gb = hasb ? make_float2(g.z, g.w) : make_float2(0.f, 0.f);
        if (i >= RPT / 2) { ga.y = -ga.y; gb.y = -gb.y; }
        if (i == 0 || i == RPT / 2) {
          // C2R ignores the imaginary part of the DC and Nyquist bins
          if (t == 0) { ga.y = 0.f; gb.y = 0.f; }
        }
        z = make_float2(ga.x - gb.y, ga.y + gb.x);  // ga + i gb
      }
      v[i] = z;
    }
    fft<L, true>(v, smem, t, active, p.tw_L);
    if (active) {
      const float x2a = -1.f + ((float)m2a + 0.5f) * inv_n;
      const float x2b = -1.f + ((float)m2b + 0.5f) * inv_n;
      float* oa = img_slice + (size_t)m2a * n;
      float* ob = oa + n;
#pragma unroll
      for (int i = 0; i < RPT; ++i) {
        const int idx = t + i * TPF;
        int m1;
        bool keep;
        if constexpr (CROP_HALF) {
          // n = L/2, offset L/4: rows i < RPT/4 -> m1 = idx + L/4,
          // i >= 3 RPT/4 -> m1 = idx - 3L/4 (others cropped, DCE'd)
          keep = i < RPT / 4 || i >= 3 * RPT / 4;
          m1 = i < RPT / 4 ? idx + L / 4 : idx - 3 * L / 4;
        } else {
          m1 = (idx + p.n_half) & (L - 1);
          keep = m1 < n;
        }
        if (keep) {
          // x1 of output column m1 (coverage add-back, fourier_bp.py:204-220, 458)
          const float x1 = CROP_HALF ? fmaf((float)(m1 - t), inv_n, xt) : -1.f + ((float)m1 + 0.5f) * inv_n;
          float ra = fmaf(v[i].x, A, Bpi);
          float rb = fmaf(v[i].y, A, Bpi);
          const float r2a = fmaf(x1, x1, x2a * x2a), r2b = fmaf(x1, x1, x2b * x2b);
          // outside the unit circle 2 asin(1/r) - pi = -2 atan(sqrt(r^2 - 1))
          if (r2a > 1.f) { const float d = r2a - 1.f; ra = fmaf(cm2, atan01(d * rsqrtf(d)), ra); }
          if (r2b > 1.f) { const float d = r2b - 1.f; rb = fmaf(cm2, atan01(d * rsqrtf(d)), rb); }
          oa[m1] = ra;
          chk = fmaf(ra, 0.f, chk);
          if (hasb) {
            ob[m1] = rb;
            chk = fmaf(rb, 0.f, chk);
          }
        }
      }
    }
    __syncthreads();  // smem reuse by the next pair
  }
}

#ifndef TB_K3_MINB
#define TB_K3_MINB TB_MINB
#endif
template <int L, bool CROP_HALF>
__global__ void __launch_bounds__(KShape<L>::THREADS, KShape<L>::THREADS <= 256 ? TB_K3_MINB : 1)
    k3_rows(DevPlan p, Work w, float* __restrict__ img, float out_scale) {
  extern __shared__ float2 smem[];
  float chk = 0.f;
  k3_tile<L, CROP_HALF>(p, w, img + (size_t)blockIdx.y * p.n * p.n, out_scale, blockIdx.y, blockIdx.x, smem, chk);
  if (chk != 0.f) atomicOr(&w.status[1], 1);
}

// ---------------------------------------------------------------------------
// Horizontally fused launch (one kernel, three kinds of independent CTAs):
// K2 of launch group g, K1 of group g + 1 and K3 of group g - 1, whose
// workspaces are disjoint (two lanes).  The idea: K2's gathers are bound by
// TLD4 latency (~53 % issue active on its own) while K1 and K3 are FFT
// arithmetic, so an SM holding a mix could fill K2's idle issue slots.
// Measured at 2048^3 it does not (TB_FUSE=1: 176.9 ms, =2: 189.3 ms, per-group
// launches 166.6 ms): each kernel's throughput is linear in its
// resident CTAs, so sharing the SM only splits it, and the mix costs L1.
// Kept (off by default, bitwise equal, tested) as the scaffold for kernels
// that saturate a unit with fewer CTAs.  Block x maps to a task by
// two nested Bresenham splits, so each kind's tasks are spread evenly over
// the grid (and over time, as CTAs dispatch roughly in index order) and each
// kind keeps its own task order (K2 slice-fast, K1 / K3 slice-major).
// ---------------------------------------------------------------------------
struct FusedArgs {
  Work w2;                // K2 (group g)
  int n2, kc2, spc2, B2, nsg2;
  const float* sino1;     // K1 (group g + 1)
  Work w1;
  int n1, groups1;
  Work w3;                // K3 (group g - 1)
  float* img3;
  float scale3;
  int n3, tiles3;
};

// is position x of T one of the n items spread evenly over [0, T)?  idx =
// its index if so, else the number of those items before x
__device__ __forceinline__ bool bres_take(long long x, long long n, long long T, long long& idx) {
  const long long a = (x * n) / T, b = ((x + 1) * n) / T;
  idx = a;
  return b > a;
}

#ifndef TB_KF_MINB
#define TB_KF_MINB 4
#endif
template <int L, bool CROP_HALF, bool NORM>
__global__ void __launch_bounds__(KShape<L>::THREADS, KShape<L>::THREADS <= 256 ? TB_KF_MINB : 1)
    kf_fused(DevPlan p, FusedArgs a) {
  static_assert(K1Shape<L>::THREADS == K2Shape<L>::THREADS, "fused CTAs share one block size");
  extern __shared__ float2 smem[];
  const long long x = blockIdx.x;
  long long i3, i1;
  if (bres_take(x, a.n3, (long long)a.n1 + a.n2 + a.n3, i3)) {
    const int q = (int)(i3 / a.tiles3), tile = (int)(i3 % a.tiles3);
    float chk = 0.f;
    k3_tile<L, CROP_HALF>(p, a.w3, a.img3 + (size_t)q * p.n * p.n, a.scale3, q, tile, smem, chk);
    if (chk != 0.f) atomicOr(&a.w3.status[1], 1);
    return;
  }
  const long long y = x - i3;  // position among the K1 + K2 tasks
  if (bres_take(y, a.n1, (long long)a.n1 + a.n2, i1)) {
    k1_block<L, true, NORM>(p, a.sino1, a.w1, (int)(i1 % a.groups1), (int)(i1 / a.groups1), smem);
    return;
  }
  const long long i2 = y - i1;
  k2_block<L, CROP_HALF, K2_TEX>(p, a.w2, (int)(i2 / a.nsg2), (int)(i2 % a.nsg2), a.kc2, a.spc2, a.B2, smem);
}

// ---------------------------------------------------------------------------
// K5: slant-stack backprojection (projector.py:126-158)
// ---------------------------------------------------------------------------
#ifdef TB_API_KERNELS
// (D, 1 / max(I0 - D, eps)) per input row and detector
__global__ void __launch_bounds__(256) k_norm_table(const float* __restrict__ flat, const float* __restrict__ dark,
                                                    float eps, float2* __restrict__ tab, int count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const float d = dark[i];
  const float den = flat[i] - d;
  tab[i] = make_float2(d, 1.f / (den != den ? den : fmaxf(den, eps)));
}

// ---------------------------------------------------------------------------
// Centering and ring suppression (preprocess.py:77-154), fp64 arithmetic on
// fp32 rows like the reference's float64 on float32-valued data.
// ---------------------------------------------------------------------------
// one CTA per slice: full cross-correlation of row 0 and the reversed last
// row (means removed), first argmax, parabolic refinement; out[q] = (beta,
// confidence), st[q] = 0 ok / 1 constant / 2 implausible.  smem: 4 n_t - 1
// doubles + the reduction scratch.
__global__ void __launch_bounds__(512) k_center_estimate(const float* __restrict__ sino, int rows, int n_t,
                                                         double2* __restrict__ out, int* __restrict__ st) {
  extern __shared__ double cs_mem[];
  double* a = cs_mem;
  double* b = a + n_t;
  double* corr = b + n_t;               // 2 n_t - 1
  double* red = corr + 2 * n_t - 1;     // [2 blockDim]
  int* redi = reinterpret_cast<int*>(red + 2 * blockDim.x);
  const int q = blockIdx.x, t = threadIdx.x, T = blockDim.x;
  const float* y = sino + (size_t)q * rows * n_t;
  double sa = 0.0, sb = 0.0;
  for (int i = t; i < n_t; i += T) {
    a[i] = (double)y[i];
    b[i] = (double)y[(size_t)(rows - 1) * n_t + (n_t - 1 - i)];
    sa += a[i];
    sb += b[i];
  }
  auto block_sum2 = [&](double& x, double& z) {
    red[t] = x;
    red[t + T] = z;
    __syncthreads();
    for (int s = T / 2; s > 0; s >>= 1) {
      if (t < s) {
        red[t] += red[t + s];
        red[t + T] += red[t + T + s];
      }
      __syncthreads();
    }
    x = red[0];
    z = red[T];
    __syncthreads();
  };
  block_sum2(sa, sb);
  const double ma = sa / n_t, mb = sb / n_t;
  double na = 0.0, nb = 0.0;
  for (int i = t; i < n_t; i += T) {
    a[i] -= ma;
    b[i] -= mb;
    na += a[i] * a[i];
    nb += b[i] * b[i];
  }
  block_sum2(na, nb);
  const double norm = sqrt(na) * sqrt(nb);
  // corr[k] = sum_n a[n + k - (n_t - 1)] b[n]   (np.correlate "full")
  double best = -INFINITY;
  int bk = 0x7fffffff;
  for (int k = t; k < 2 * n_t - 1; k += T) {
    const int s = k - (n_t - 1);
    const int n0 = max(0, -s), n1 = min(n_t, n_t - s);
    double c = 0.0;
    for (int n = n0; n < n1; ++n) c = fma(a[n + s], b[n], c);
    corr[k] = c;
    if (c > best) { best = c; bk = k; }  // k increases: ties keep the first
  }
  red[t] = best;
  redi[t] = bk;
  __syncthreads();
  for (int s = T / 2; s > 0; s >>= 1) {
    if (t < s) {
      const double o = red[t + s];
      const int oi = redi[t + s];
      if (o > red[t] || (o == red[t] && oi < redi[t])) { red[t] = o; redi[t] = oi; }
    }
    __syncthreads();
  }
  if (t == 0) {
    const int k = redi[0];
    double pk = (double)k;
    if (k > 0 && k < 2 * n_t - 2) {
      const double y0 = corr[k - 1], y1 = corr[k], y2 = corr[k + 1];
      const double den = y0 - 2.0 * y1 + y2;
      if (den != 0.0) pk = k + 0.5 * (y0 - y2) / den;
    }
    const double beta = (pk - (n_t - 1)) / 2.0;
    const double conf = norm > 0.0 ? fmin(fmax(corr[k] / norm, 0.0), 1.0) : 0.0;
    out[q] = make_double2(beta, conf);
    st[q] = norm == 0.0 ? 1 : (fabs(beta) > n_t / 2.0 ? 2 : 0);
  }
}

// out = apply_center(in, beta[q].x): linear interpolation at i + beta, zero
// out of range (preprocess.py:121-138)
__global__ void __launch_bounds__(256) k_center_apply(const float* __restrict__ in, float* __restrict__ out,
                                                      const double2* __restrict__ beta, int rows, int n_t) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y, q = blockIdx.z;
  if (i >= n_t) return;
  const double idx = (double)i + beta[q].x;
  const double fl = floor(idx);
  const long long i0 = (long long)fl;
  const double fr = idx - fl;
  const bool ok0 = i0 >= 0 && i0 <= n_t - 1, ok1 = i0 + 1 >= 0 && i0 + 1 <= n_t - 1;
  const long long i0c = i0 < 0 ? 0 : (i0 > n_t - 1 ? n_t - 1 : i0);
  const long long i1c = i0 + 1 < 0 ? 0 : (i0 + 1 > n_t - 1 ? n_t - 1 : i0 + 1);
  const float* r = in + ((size_t)q * rows + j) * n_t;
  out[((size_t)q * rows + j) * n_t + i] =
      (float)((double)r[i0c] * (ok0 ? 1.0 - fr : 0.0) + (double)r[i1c] * (ok1 ? fr : 0.0));
}

// per-detector mean over angles (fp64), mean[q][i]: a (32, 8) block per 32
// detector columns of one slice, 8 row groups summed in parallel (coalesced
// 128-B row segments) and combined in shared memory.  Launch: grid
// (ceil(n_t / 32), slices), block (32, 8).
__global__ void __launch_bounds__(256) k_col_mean(const float* __restrict__ in, double* __restrict__ mean, int rows,
                                                  int n_t) {
  __shared__ double part[8][33];
  const int i = blockIdx.x * 32 + threadIdx.x;
  const int q = blockIdx.y;
  double s = 0.0;
  if (i < n_t) {
    const float* y = in + (size_t)q * rows * n_t + i;
    for (int j = threadIdx.y; j < rows; j += 8) s += (double)__ldg(y + (size_t)j * n_t);
  }
  part[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && i < n_t) {
    double t = 0.0;
    for (int g = 0; g < 8; ++g) t += part[g][threadIdx.x];
    mean[(size_t)q * n_t + i] = t / rows;
  }
}

// out = in - (mean - movavg_window(reflect-pad(mean)))  (preprocess.py:141-154)
__global__ void __launch_bounds__(256) k_rings_apply(const float* __restrict__ in, float* __restrict__ out,
                                                     const double* __restrict__ mean, int rows, int n_t, int window) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int q = blockIdx.y;
  if (i >= n_t) return;
  const double* m = mean + (size_t)q * n_t;
  const int h = window / 2;
  double acc = 0.0;
  for (int d = -h; d <= h; ++d) {
    int k = i + d;
    // np.pad(mode="reflect"): mirror about the edge samples (edge not repeated)
    while (k < 0 || k > n_t - 1) k = k < 0 ? -k : 2 * (n_t - 1) - k;
    acc += m[k] * (1.0 / window);
  }
  const double stripe = m[i] - acc;
  const float* y = in + (size_t)q * rows * n_t + i;
  float* o = out + (size_t)q * rows * n_t + i;
  for (int j = 0; j < rows; ++j) o[(size_t)j * n_t] = (float)((double)y[(size_t)j * n_t] - stripe);
}

// Fused centre / ring parameters per slice (one CTA each): the shift
// (floor(beta), frac(beta)) of apply_center and, with window > 0, the
// stripe profile of suppress_rings computed from the column means of the
// CENTRED data, which are the centred column means of the raw data (the
// interpolation is the same linear map on every row): stripe = c - movavg(
// reflect-pad(c)), c = apply_center(mean).  preprocess.py:119-154.
__global__ void __launch_bounds__(256) k_pre_params(const double* __restrict__ beta_conf, const double* __restrict__ mean,
                                                    int n_t, int window, float2* __restrict__ shift,
                                                    float* __restrict__ stripe) {
  const int q = blockIdx.x;
  const double beta = beta_conf ? beta_conf[2 * q] : 0.0;
  const double bf = floor(beta);
  const double fr = beta - bf;
  const int bi = (int)bf;
  if (threadIdx.x == 0) shift[q] = make_float2((float)bi, (float)fr);
  if (window <= 0) return;
  const double* m = mean + (size_t)q * n_t;
  auto centred = [&](int k) {
    const int j = k + bi;
    const bool ok0 = j >= 0 && j <= n_t - 1, ok1 = j + 1 >= 0 && j + 1 <= n_t - 1;
    return (ok0 ? m[j] * (1.0 - fr) : 0.0) + (ok1 ? m[j + 1] * fr : 0.0);
  };
  const int h = window / 2;
  for (int i = threadIdx.x; i < n_t; i += blockDim.x) {
    double acc = 0.0;
    for (int d = -h; d <= h; ++d) {
      int k = i + d;
      while (k < 0 || k > n_t - 1) k = k < 0 ? -k : 2 * (n_t - 1) - k;  // np.pad(mode="reflect")
      acc += centred(k) * (1.0 / window);
    }
    stripe[(size_t)q * n_t + i] = (float)(centred(i) - acc);
  }
}

// standalone normalize over n slices of [rows][n_t] counts
__global__ void __launch_bounds__(256) k_normalize(const float* __restrict__ counts, const float* __restrict__ flat,
                                                   const float* __restrict__ dark, float eps, float* __restrict__ out,
                                                   long long total, int frame) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(i % frame);
    const float d = __ldg(dark + f);
    const float den = __ldg(flat + f) - d;
    out[i] = norm_line(counts[i], make_float2(d, 1.f / (den != den ? den : fmaxf(den, eps))), eps);
  }
}

// ---------------------------------------------------------------------------
// K6: forward projector (projector.py:94-123): line integral of an n x n
// image (pixel-centre convention, zero outside) along each (theta_j, t_i)
// ray, midpoint rule with step h over the circumscribed diameter, samples
// bilinear (or nearest, np.rint half-even) in the image.  One thread per
// (slice, angle, detector); coordinates and the sum in fp64 like the
// reference; the sample loop is clipped to the ray's intersection with the
// one-pixel-padded image square (samples outside contribute exactly 0).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k6_forward(DevPlan p, const float* __restrict__ img, float* __restrict__ sino,
                                                  int n_ang, double h, int m, int nearest) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int q = blockIdx.z;
  if (i >= p.n_t) return;
  const int n = p.n;
  const double2 cs = __ldg(p.ss_cs + j);
  const double t = -1.0 + 2.0 * (double)i / (double)(p.n_t - 1);
  const double du = 2.0 / n, inv_du = 0.5 * n;
  const double half = 1.4142135623730951;  // sqrt(2)
  const float* im = img + (size_t)q * n * n;
  // ray point at ell: u = t (c, s) + ell (-s, c); keep |u1|, |u2| <= 1 + 1.5 du
  double lo = -half, hi = half;
  const double lim = 1.0 + 1.5 * du;
  auto clip = [&](double base, double dir) {
    if (fabs(dir) < 1e-300) {
      if (fabs(base) > lim) { lo = 1.0; hi = -1.0; }
      return;
    }
    double a = (-lim - base) / dir, b = (lim - base) / dir;
    if (a > b) { const double x = a; a = b; b = x; }
    lo = fmax(lo, a);
    hi = fmin(hi, b);
  };
  clip(t * cs.x, -cs.y);
  clip(t * cs.y, cs.x);
  double acc = 0.0;
  if (hi >= lo) {
    // samples ell_k = -sqrt2 + (k + 1/2) h inside [lo, hi] (one extra each side)
    const int k0 = max(0, (int)floor((lo + half) / h - 0.5) - 1);
    const int k1 = min(m - 1, (int)ceil((hi + half) / h - 0.5) + 1);
    for (int k = k0; k <= k1; ++k) {
      const double ell = -half + ((double)k + 0.5) * h;
      const double u1 = t * cs.x - ell * cs.y;
      const double u2 = t * cs.y + ell * cs.x;
      const double fx = (u1 + 1.0) * inv_du - 0.5;
      const double fy = (u2 + 1.0) * inv_du - 0.5;
      if (nearest) {
        const int ix = (int)rint(fx), iy = (int)rint(fy);
        if (ix >= 0 && ix < n && iy >= 0 && iy < n) acc += (double)__ldg(im + (size_t)iy * n + ix);
      } else {
        const double x0f = floor(fx), y0f = floor(fy);
        const int x0 = (int)x0f, y0 = (int)y0f;
        const double wx = fx - x0f, wy = fy - y0f;
        const bool xa = x0 >= 0 && x0 < n, xb = x0 + 1 >= 0 && x0 + 1 < n;
        const bool ya = y0 >= 0 && y0 < n, yb = y0 + 1 >= 0 && y0 + 1 < n;
        const float* r0 = im + (size_t)y0 * n;
        double v = 0.0;
        if (ya) {
          if (xa) v += (1.0 - wx) * (1.0 - wy) * (double)__ldg(r0 + x0);
          if (xb) v += wx * (1.0 - wy) * (double)__ldg(r0 + x0 + 1);
        }
        if (yb) {
          if (xa) v += (1.0 - wx) * wy * (double)__ldg(r0 + n + x0);
          if (xb) v += wx * wy * (double)__ldg(r0 + n + x0 + 1);
        }
        acc += v;
      }
    }
  }
  sino[((size_t)q * n_ang + j) * p.n_t + i] = (float)(acc * h);
}

// K6, texture path (bilinear; pitch-2D float texture over a run of image
// slices, border addressing in x): one TLD4 gathers a sample's 2 x 2
// footprint (exact fp32 pixels) instead of four scattered loads; the
// coordinates stay fp64 as in projector.py:111-117, the footprint weights
// are rounded to fp32 (<= 6e-8) and the sum runs in fp64.  Rows outside the
// slice (y0 = -1 or y0 + 1 = n lie in the neighbouring slice of the
// texture) are masked explicitly.
// NEAREST: one point fetch per sample at np.rint of the fp64 position (4 B
// of texture return instead of the 16 B footprint)
template <bool NEAREST>
__global__ void __launch_bounds__(128) k6_forward_tex(DevPlan p, cudaTextureObject_t tex, float* __restrict__ sino,
                                                      int n_ang, double h, int m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = blockIdx.y;
  const int q = blockIdx.z;
  if (i >= p.n_t) return;
  const int n = p.n;
  const double2 cs = __ldg(p.ss_cs + j);
  const double t = -1.0 + 2.0 * (double)i / (double)(p.n_t - 1);
  const double du = 2.0 / n, inv_du = 0.5 * n;
  const double half = 1.4142135623730951;  // sqrt(2)
  double lo = -half, hi = half;
  const double lim = 1.0 + 1.5 * du;
  auto clip = [&](double base, double dir) {
    if (fabs(dir) < 1e-300) {
      if (fabs(base) > lim) { lo = 1.0; hi = -1.0; }
      return;
    }
    double a = (-lim - base) / dir, b = (lim - base) / dir;
    if (a > b) { const double x = a; a = b; b = x; }
    lo = fmax(lo, a);
    hi = fmin(hi, b);
  };
  clip(t * cs.x, -cs.y);
  clip(t * cs.y, cs.x);
  double acc = 0.0;
  if (hi >= lo) {
    const int k0 = max(0, (int)floor((lo + half) / h - 0.5) - 1);
    const int k1 = min(m - 1, (int)ceil((hi + half) / h - 0.5) + 1);
    const float ybase = (float)(q * n + 1);
    for (int k = k0; k <= k1; ++k) {
      const double ell = -half + ((double)k + 0.5) * h;
      const double fx = (t * cs.x - ell * cs.y + 1.0) * inv_du - 0.5;
      const double fy = (t * cs.y + ell * cs.x + 1.0) * inv_du - 0.5;
      if constexpr (NEAREST) {
        const double ixf = rint(fx), iyf = rint(fy);
        const int iy = (int)iyf;
        // columns outside read the border (0); rows outside the slice are masked
        const float v = tex2D<float>(tex, (float)(ixf + 0.5), ybase - 0.5f + (float)iy);
        if (iy >= 0 && iy < n) acc += (double)v;
        continue;
      }
      const double x0f = floor(fx), y0f = floor(fy);
      const int y0 = (int)y0f;
      const float wx = (float)(fx - x0f), wy = (float)(fy - y0f);
      // texel (x0, q n + y0) .. (x0 + 1, q n + y0 + 1)
      const float4 g = tex2Dgather<float4>(tex, (float)(x0f + 1.0), ybase + (float)y0, 0);
      const bool ya = y0 >= 0 && y0 < n, yb = y0 + 1 >= 0 && y0 + 1 < n;
      const float a00 = ya ? g.w : 0.f, a01 = ya ? g.z : 0.f;
      const float a10 = yb ? g.x : 0.f, a11 = yb ? g.y : 0.f;
      const float r0 = fmaf(wx, a01 - a00, a00), r1 = fmaf(wx, a11 - a10, a10);
      acc += (double)fmaf(wy, r1 - r0, r0);
    }
  }
  sino[((size_t)q * n_ang + j) * p.n_t + i] = (float)(acc * h);
}

// Slant stack, tiled: a CTA owns a 32 x 32 pixel tile, a thread 4 pixels of
// one column (m2 = ty + 8 k).  The detector coordinate fi = (x c + y s + 1) /
// dt of pixel (M1 + d1, M2 + d2) is split as fi = bi + (bf + d1 B + d2 C):
// the tile-origin term in fp64 once per (tile, angle), rounded to an integer
// bi plus an fp32 remainder bf, then only small fp32 offsets per pixel
// (|remainder| < ~50 samples: 2^-18 absolute error, vs 2^-52 relative in the
// reference), so the inner loop has no fp64.  The detector-range test and the
// clamp follow projector.py:149-155 on fi = bi + f exactly (bi is an integer).
constexpr int kSsTile = 32, kSsChunk = 256;
__global__ void __launch_bounds__(256) k5_slant(DevPlan p, const float* __restrict__ rows, int n_ang,
                                                float* __restrict__ img, float scale, Work w) {
  __shared__ float4 ang[kSsChunk];  // (bf, B, C, bi) per angle of the chunk
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int M1 = blockIdx.x * kSsTile, M2 = blockIdx.y * kSsTile;
  const int q = blockIdx.z;
  const int n = p.n;
  const float* base = rows + (size_t)q * n_ang * p.n_t;
  const double inv_dt = (double)p.ss_inv_dt;
  const double x0 = -1.0 + 2.0 * ((double)M1 + 0.5) / (double)n;
  const double y0 = -1.0 + 2.0 * ((double)M2 + 0.5) / (double)n;
  const int top = p.n_t - 1;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const float d1 = (float)tx;
  for (int j0 = 0; j0 < n_ang; j0 += kSsChunk) {
    const int cnt = min(kSsChunk, n_ang - j0);
    __syncthreads();  // the previous chunk is consumed
    for (int jj = threadIdx.x; jj < cnt; jj += blockDim.x) {
      const double2 cs = __ldg(p.ss_cs + j0 + jj);
      const double fi0 = (fma(x0, cs.x, y0 * cs.y) + 1.0) * inv_dt;
      const double bi = floor(fi0);
      ang[jj] = make_float4((float)(fi0 - bi), (float)(2.0 * cs.x / n * inv_dt), (float)(2.0 * cs.y / n * inv_dt),
                            __int_as_float((int)bi));
    }
    __syncthreads();
    for (int jj = 0; jj < cnt; ++jj) {
      const float4 g = ang[jj];
      const int bi = __float_as_int(g.w);
      const float* r = base + (size_t)(j0 + jj) * p.n_t;
      const float f0 = fmaf(d1, g.y, g.x);
      const float lo = (float)(-bi), hi = (float)(top - bi);  // fi in [0, n_t - 1]
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float f = fmaf((float)(ty + 8 * k), g.z, f0);
        const float fl = floorf(f);
        const float fr = f - fl;
        const int i0 = min(max(bi + (int)fl, 0), p.n_t - 2);
        const float r0 = __ldg(r + i0), r1 = __ldg(r + i0 + 1);
        acc[k] += (f >= lo && f <= hi) ? fmaf(fr, r1 - r0, r0) : 0.f;
      }
    }
  }
  const int m1 = M1 + tx;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int m2 = M2 + ty + 8 * k;
    if (m1 < n && m2 < n) {
      const float out = acc[k] * p.ss_weight * scale;
      img[((size_t)q * n + m2) * n + m1] = out;
      if (w.status && !isfinite(out)) atomicOr(&w.status[1], 1);
    }
  }
}
#endif

}  // namespace tb
