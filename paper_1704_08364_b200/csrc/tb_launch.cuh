// tb_launch.cuh -- host-side per-L launchers shared by tb_api.cu (plan, ABI,
// dispatch) and the per-L instantiation units tb_inst.cu (compiled once per
// radial length with -DTB_L=<L>, so the sm_100a build parallelises).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tb_bst.h"
#include "tb_kernels.cuh"

using tb::DevPlan;
using tb::Work;

// last error message of the calling thread (defined in tb_api.cu)
extern thread_local std::string tb_g_err;

inline int fail(int code, const std::string& msg) {
  tb_g_err = msg;
  return code;
}

#define TB_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(TB_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));        \
  } while (0)

struct tb_plan {
  tb_plan_desc desc;
  int device;
  int n_t, V, rows, L, H, n, npad, lo, hi, S;
  double amp;
  int groups, pairs_per_cta;
  bool bst_ok = true;  // standard angle layout and gridding tables present
  DevPlan dp;
  void* blob = nullptr;   // all small device tables in one allocation
  void* table = nullptr;  // gridding table [(H+1)^2] uint2
  void* table2 = nullptr; // first-quadrant gridding table [(H+1)][(H+1)] float4 + column extents (half-turn bilinear)
  // texture objects over workspace polar regions, keyed by (pointer, rows);
  // kept until the plan is destroyed (kernels may still be using them)
  struct Tex {
    const void* ptr;
    int rows;
    cudaTextureObject_t obj;
  };
  mutable std::mutex tex_mu;
  mutable std::vector<Tex> texs;
  mutable std::vector<Tex> itexs;  // image views of the forward projector (bounded cache)
};

// ---------------------------------------------------------------------------
// per-L launchers
// ---------------------------------------------------------------------------
template <int L>
struct Launch {
  using K = tb::KShape<L>;
  static size_t smem_k1(const tb_plan* p) {
    // FFT buffer + support sums + TB_K1_SLOTS TMA staging slots of a row pair + 2 mbarriers
    return tb::K1Shape<L>::BUF * sizeof(float2) + (size_t)((std::max(p->S, 1) + 3) & ~3) * 4 +
           (size_t)K1_STAGE_ROWS * p->n_t * 4 + 16;
  }
  static size_t smem_k1b(const tb_plan* p) {
    return K::BUF * sizeof(float2) + (size_t)2 * std::max(p->S, 1) * 4 + (size_t)2 * K::K1B_THREADS * 4 +
           (size_t)(L / 2) * 4;
  }
  static size_t smem_fft() { return K::BUF * sizeof(float2); }
  using K2 = tb::K2Shape<L>;
  static size_t smem_k2() { return (size_t)K2::G * K2::SMEM_PER_GROUP * sizeof(float2); }
  // columns per K2 CTA: one resident CTA per SM sweeping G columns at a time
  static int k2_cols(const tb_plan* p, bool tex) {
    if (const char* e = std::getenv("TB_K2_COLS"))  // tuning: columns swept per CTA
      if (std::atoi(e) > 0) return K2::G * std::atoi(e);
    // half-plane-table path: slice-fast grid, one column group per CTA (the
    // resident CTAs cover a few columns of every slice of the launch group,
    // so each 16 B-per-node table row is read from DRAM once per group)
    if (tex) return K2::G;
    const int resident = std::min(K2::MINB, 4);  // CTAs per SM of the plain / general paths
    int steps = ((p->H + 1 + K2::G - 1) / K2::G + 148 * resident - 1) / (148 * resident);
    // L = 4096: the resident CTAs should cover a little less than one slice,
    // so the slice's polar spectrum and the gridding table stay in L2
    // (measured at 2048^3: 4 columns per CTA 101.9 ms, 5 columns 103.3 ms)
    if (L == 4096 && steps > 1) steps -= 1;
    return K2::G * std::max(1, steps);
  }

  // slices per K2 CTA (TB_K2_SPC, tuning; default 1) and the grid order
  // (TB_K2_ORDER=1: slice runs on blockIdx.x, resident CTAs share columns)
  static int k2_slices(int B) {
    if (const char* e = std::getenv("TB_K2_SPC"))
      if (std::atoi(e) > 0) return std::min(B, std::atoi(e));
    return 1;
  }
  static int k2_slice_fast(bool tex) {
    if (const char* e = std::getenv("TB_K2_ORDER")) return std::atoi(e) == 1 ? 1 : 0;
    return tex ? 1 : 0;
  }

  template <bool CH>
  static cudaError_t set_k2_smem() {
    const auto a = cudaFuncAttributeMaxDynamicSharedMemorySize;
    cudaError_t e = cudaFuncSetAttribute(tb::k2_columns<L, CH, tb::K2_ANY>, a, (int)smem_k2());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tb::k2_columns<L, CH, tb::K2_PLAIN>, a, (int)smem_k2());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tb::k2_columns<L, CH, tb::K2_TEX>, a, (int)smem_k2());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tb::k2_columns<L, CH, tb::K2_TEXF>, a, (int)smem_k2());
    if (e == cudaSuccess) e = cudaFuncSetAttribute(tb::k2_columns<L, CH, tb::K2_TEXN>, a, (int)smem_k2());
    return e;
  }
  template <bool CH>
  static void launch_k2(const DevPlan& dp, const Work& w, dim3 g2, cudaStream_t st, int kc, int spc, int B, int sf) {
    const bool tex = w.polar_tex && dp.gridtab2;  // the plan built the table for its interp / turn
    if (tex && dp.interp != 0)
      tb::k2_columns<L, CH, tb::K2_TEXN><<<g2, K2::THREADS, smem_k2(), st>>>(dp, w, kc, spc, B, sf);
    else if (tex && dp.full_turn)
      tb::k2_columns<L, CH, tb::K2_TEXF><<<g2, K2::THREADS, smem_k2(), st>>>(dp, w, kc, spc, B, sf);
    else if (tex)
      tb::k2_columns<L, CH, tb::K2_TEX><<<g2, K2::THREADS, smem_k2(), st>>>(dp, w, kc, spc, B, sf);
    else if (dp.full_turn || dp.interp != 0)
      tb::k2_columns<L, CH, tb::K2_ANY><<<g2, K2::THREADS, smem_k2(), st>>>(dp, w, kc, spc, B, sf);
    else
      tb::k2_columns<L, CH, tb::K2_PLAIN><<<g2, K2::THREADS, smem_k2(), st>>>(dp, w, kc, spc, B, sf);
  }

  static int configure(tb_plan* p) {
    // The dynamic shared-memory limit is a per-kernel (process-wide)
    // attribute while K1 / K1b need space for the plan's window support S:
    // size it for the largest S any plan of this L can have (S <= n_t <=
    // L/2) so a later plan never lowers it below what an earlier one needs
    // (the limit does not change occupancy; the launch's request does)
    tb_plan worst;
    worst.S = L / 2;
    worst.n_t = L / 2;
    int dev = 0, smax = 0;
    TB_CUDA(cudaGetDevice(&dev));
    TB_CUDA(cudaDeviceGetAttribute(&smax, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if ((int)smem_k1(p) > smax || (int)smem_k1b(p) > smax)
      return fail(TB_ERR_UNSUPPORTED, "the origin-window support needs more shared memory than the device has");
    const int s1 = std::min((int)smem_k1(&worst), smax), s1b = std::min((int)smem_k1b(&worst), smax);
    TB_CUDA(cudaFuncSetAttribute(tb::k1_radial<L, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1));
    TB_CUDA(cudaFuncSetAttribute(tb::k1_radial<L, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1));
    TB_CUDA(cudaFuncSetAttribute(tb::k1_radial<L, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1));
    TB_CUDA(cudaFuncSetAttribute(tb::k1_radial<L, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1));
    TB_CUDA(cudaFuncSetAttribute(tb::k1b_common<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, s1b));
    TB_CUDA(set_k2_smem<false>());
    TB_CUDA(cudaFuncSetAttribute(tb::k3_rows<L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fft()));
    if constexpr (tb::KShape<L>::THREADS == tb::K2Shape<L>::THREADS && tb::K1Shape<L>::THREADS == tb::K2Shape<L>::THREADS && L >= 64) {
      const int sf = (int)std::max({smem_k1(&worst), smem_k2(), smem_fft()});
      const int sfm = std::min(sf, smax);
      TB_CUDA(cudaFuncSetAttribute(tb::kf_fused<L, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sfm));
      TB_CUDA(cudaFuncSetAttribute(tb::kf_fused<L, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sfm));
      TB_CUDA(cudaFuncSetAttribute(tb::kf_fused<L, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sfm));
      TB_CUDA(cudaFuncSetAttribute(tb::kf_fused<L, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sfm));
    }
    if constexpr (L >= 64) {
      TB_CUDA(set_k2_smem<true>());
      TB_CUDA(cudaFuncSetAttribute(tb::k3_rows<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fft()));
    }
    TB_CUDA(cudaFuncSetAttribute(tb::kr_ramp<L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fft()));
    TB_CUDA(cudaFuncSetAttribute(tb::kr_ramp<L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_fft()));
    // tuning: shared-memory carveout (percent of the SM's 228 KB; the rest is
    // L1) for K1 / K2 / K3 as "k1,k2,k3"; unset = the driver's choice
    if (const char* e = std::getenv("TB_CARVEOUT")) {
      int c1 = -1, c2 = -1, c3 = -1;
      if (std::sscanf(e, "%d,%d,%d", &c1, &c2, &c3) == 3) {
        const auto co = cudaFuncAttributePreferredSharedMemoryCarveout;
        TB_CUDA(cudaFuncSetAttribute(tb::k1_radial<L, true, false>, co, c1));
        TB_CUDA(cudaFuncSetAttribute(tb::k1_radial<L, true, true>, co, c1));
        TB_CUDA(cudaFuncSetAttribute(tb::k1_radial<L, true, false, true>, co, c1));
        TB_CUDA(cudaFuncSetAttribute(tb::k2_columns<L, (L >= 64), tb::K2_TEX>, co, c2));
        TB_CUDA(cudaFuncSetAttribute(tb::k3_rows<L, (L >= 64)>, co, c3));
      }
    }
    return TB_OK;
  }

  // one launch group of B slices through K1 -> K1b -> K2 -> K3.  `ev`, when
  // given, receives start/stop events around each stage: [stage][2] with
  // stages 0 ramp (unfused path), 1 K1, 2 K1b, 3 K2, 4 K3.
  static int bst_group(const tb_plan* p, const float* sino, float* img, int B, const Work& w, bool ramp,
                       float out_scale, cudaStream_t st, cudaEvent_t* ev) {
    const DevPlan& dp = p->dp;
    const float* k1_in = sino;
    Work wk = w;  // K1's view of its input (the filtered rows are slice-major)
    bool fused = false;
    auto mark = [&](int stage, int which) {
      if (ev) cudaEventRecord(ev[2 * stage + which], st);
    };
    if (ramp) {
      if (p->npad == L) {
        fused = true;
      } else {
        mark(0, 0);
        int rc = ramp_rows(p, sino, w.filtered, B * p->rows, w, st);
        mark(0, 1);
        if (rc) return rc;
        k1_in = w.filtered;
        wk.in_slice = (long long)p->rows * p->n_t;
        wk.in_row = p->n_t;
        wk.normtab = nullptr;  // normalised by the ramp pass
        wk.norm_eps = 0.f;
      }
    }
    dim3 g1(p->groups, B);
    mark(1, 0);
    if (fused && wk.norm_eps > 0.f)  // transmission counts: normalisation fused into the load
      tb::k1_radial<L, true, true><<<g1, tb::K1Shape<L>::THREADS, smem_k1(p), st>>>(dp, k1_in, wk);
    else if (fused && wk.pre_shift)  // centre / ring stages fused into the load (tb_fbp_pre)
      tb::k1_radial<L, true, false, true><<<g1, tb::K1Shape<L>::THREADS, smem_k1(p), st>>>(dp, k1_in, wk);
    else if (fused)
      tb::k1_radial<L, true, false><<<g1, tb::K1Shape<L>::THREADS, smem_k1(p), st>>>(dp, k1_in, wk);
    else
      tb::k1_radial<L, false, false><<<g1, tb::K1Shape<L>::THREADS, smem_k1(p), st>>>(dp, k1_in, wk);
    mark(1, 1);
    mark(2, 0);
    tb::k1b_common<L><<<B, K::K1B_THREADS, smem_k1b(p), st>>>(dp, w);
    mark(2, 1);
    const bool half = L >= 64 && 2 * p->n == L;
    mark(3, 0);
    const bool tex = w.polar_tex && dp.gridtab2;
    const int kc = k2_cols(p, tex);
    const int spc = k2_slices(B);
    const int ncg = (p->H + 1 + kc - 1) / kc, nsg = (B + spc - 1) / spc;
    const int sf = k2_slice_fast(tex);
    const dim3 g2(sf ? nsg : ncg, sf ? ncg : nsg);
    if (half)
      launch_k2<(L >= 64)>(dp, w, g2, st, kc, spc, B, sf);
    else
      launch_k2<false>(dp, w, g2, st, kc, spc, B, sf);
    mark(3, 1);
    mark(4, 0);
    if (half)
      tb::k3_rows<L, (L >= 64)><<<dim3((p->n + 3) / 4, B), K::THREADS, smem_fft(), st>>>(dp, w, img, out_scale);
    else
      tb::k3_rows<L, false><<<dim3((p->n + 3) / 4, B), K::THREADS, smem_fft(), st>>>(dp, w, img, out_scale);
    mark(4, 1);
    TB_CUDA(cudaGetLastError());
    return TB_OK;
  }

  static int ramp_rows(const tb_plan* p, const float* in, float* out, int total_rows, const Work& w,
                       cudaStream_t st);

  // The fused schedule on one stream, launch groups alternating between the
  // two workspace lanes:
  //   K1(0) K1b(0) | F(K2(0) + K1(1)) K1b(1) | F(K2(1) + K1(2) + K3(0)) K1b(2) | ... | K3(G-1)
  // (with_k3 = false: K3(g) runs alone right after F(g)).  F(g)'s three parts
  // touch disjoint lanes: K2(g) reads lane g&1's polar rows and writes its
  // columns, K1(g+1) writes lane (g+1)&1's polar rows (read by K2(g-1) in the
  // previous launch), K3(g-1) reads lane (g+1)&1's columns and coef mean
  // (rewritten only by K2(g+1) / K1b(g+1), both after F(g) on the stream).
  // lanes[]: the two lanes' Work with the input addressing set.  Returns
  // TB_ERR_UNSUPPORTED (nothing enqueued) where the fused kernel does not
  // apply; the caller then runs the per-group path.
  static int fused_pipeline(const tb_plan* p, const float* sino, float* img, int n_slices, int batch,
                            const Work* lanes, size_t in_stride, size_t out_stride, float scale, bool with_k3,
                            cudaStream_t st) {
    if constexpr (tb::K1Shape<L>::THREADS != tb::K2Shape<L>::THREADS || tb::KShape<L>::THREADS != tb::K2Shape<L>::THREADS || L < 64) {
      return TB_ERR_UNSUPPORTED;
    } else {
      const DevPlan& dp = p->dp;
      const bool tex = !dp.full_turn && dp.interp == 0 && lanes[0].polar_tex && lanes[1].polar_tex && dp.gridtab2;
      if (!tex || p->npad != L || n_slices <= batch) return TB_ERR_UNSUPPORTED;
      const bool norm = lanes[0].norm_eps > 0.f;
      const bool half = 2 * p->n == L;
      const int G = (n_slices + batch - 1) / batch;
      auto nb = [&](int g) { return std::min(batch, n_slices - g * batch); };
      const int tiles = (p->n + 3) / 4;
      const int kc = K2::G;
      const int ncg = (p->H + 1 + kc - 1) / kc;
      // K1(0), K1b(0)
      {
        const dim3 g1(p->groups, nb(0));
        if (norm)
          tb::k1_radial<L, true, true><<<g1, tb::K1Shape<L>::THREADS, smem_k1(p), st>>>(dp, sino, lanes[0]);
        else
          tb::k1_radial<L, true, false><<<g1, tb::K1Shape<L>::THREADS, smem_k1(p), st>>>(dp, sino, lanes[0]);
        tb::k1b_common<L><<<nb(0), K::K1B_THREADS, smem_k1b(p), st>>>(dp, lanes[0]);
      }
      const size_t smem = std::max({smem_k1(p), smem_k2(), smem_fft()});
      for (int g = 0; g < G; ++g) {
        tb::FusedArgs a{};
        a.w2 = lanes[g & 1];
        a.B2 = nb(g);
        a.nsg2 = nb(g);
        a.n2 = ncg * a.nsg2;
        a.kc2 = kc;
        a.spc2 = 1;
        if (g + 1 < G) {
          a.w1 = lanes[(g + 1) & 1];
          a.sino1 = sino + (size_t)(g + 1) * batch * in_stride;
          a.groups1 = p->groups;
          a.n1 = p->groups * nb(g + 1);
        }
        if (with_k3 && g >= 1) {
          a.w3 = lanes[(g - 1) & 1];
          a.img3 = img + (size_t)(g - 1) * batch * out_stride;
          a.scale3 = scale;
          a.tiles3 = tiles;
          a.n3 = tiles * nb(g - 1);
        }
        const unsigned blocks = (unsigned)(a.n1 + a.n2 + a.n3);
        if (half) {
          if (norm) tb::kf_fused<L, true, true><<<blocks, K::THREADS, smem, st>>>(dp, a);
          else tb::kf_fused<L, true, false><<<blocks, K::THREADS, smem, st>>>(dp, a);
        } else {
          if (norm) tb::kf_fused<L, false, true><<<blocks, K::THREADS, smem, st>>>(dp, a);
          else tb::kf_fused<L, false, false><<<blocks, K::THREADS, smem, st>>>(dp, a);
        }
        if (g + 1 < G) tb::k1b_common<L><<<nb(g + 1), K::K1B_THREADS, smem_k1b(p), st>>>(dp, lanes[(g + 1) & 1]);
        if (!with_k3 || g == G - 1) {
          const int g3 = g;  // K3(g) alone: every group without K3 fusion, the last group with it
          float* im = img + (size_t)g3 * batch * out_stride;
          const dim3 gk3(tiles, nb(g3));
          if (half)
            tb::k3_rows<L, true><<<gk3, K::THREADS, smem_fft(), st>>>(dp, lanes[g3 & 1], im, scale);
          else
            tb::k3_rows<L, false><<<gk3, K::THREADS, smem_fft(), st>>>(dp, lanes[g3 & 1], im, scale);
        }
      }
      TB_CUDA(cudaGetLastError());
      return TB_OK;
    }
  }
};

template <int NP>
int launch_ramp(const tb_plan* p, const float* in, float* out, int total_rows, const Work& w, cudaStream_t st) {
  using K = tb::KShape<NP>;
  if (w.norm_eps > 0.f)  // unfused ramp on transmission counts: normalisation in its load
    tb::kr_ramp<NP, true><<<(total_rows + 1) / 2, K::THREADS, K::BUF * sizeof(float2), st>>>(p->dp, in, out, total_rows, w);
  else
    tb::kr_ramp<NP, false><<<(total_rows + 1) / 2, K::THREADS, K::BUF * sizeof(float2), st>>>(p->dp, in, out, total_rows, w);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int ramp_dispatch(const tb_plan* p, const float* in, float* out, int total_rows, const Work& w, cudaStream_t st);

template <int L>
int Launch<L>::ramp_rows(const tb_plan* p, const float* in, float* out, int total_rows, const Work& w,
                         cudaStream_t st) {
  return ramp_dispatch(p, in, out, total_rows, w, st);
}

// per-L entry points, defined in tb_inst.cu for each supported L
#define TB_FOR_EACH_L(X) X(4) X(8) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(8192) X(16384)
#define TB_DECLARE_L(N)                                                                                    \
  int tb_configure_##N(tb_plan* p);                                                                      \
  int tb_group_##N(const tb_plan* p, const float* sino, float* img, int B, const Work& w, bool ramp,       \
                   float scale, cudaStream_t st, cudaEvent_t* ev);                                       \
  int tb_ramp_##N(const tb_plan* p, const float* in, float* out, int total_rows, const Work& w,           \
                  cudaStream_t st);                                                                      \
  int tb_pipe_##N(const tb_plan* p, const float* sino, float* img, int n_slices, int batch,               \
                  const Work* lanes, size_t in_stride, size_t out_stride, float scale, bool with_k3,       \
                  cudaStream_t st);
TB_FOR_EACH_L(TB_DECLARE_L)
