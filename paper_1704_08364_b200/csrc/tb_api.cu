// tb_api.cu -- host side of the C ABI declared in include/tb_bst.h.
//
// Plan creation restates the reference's BstPlan / FilterPlan derived tables
// (fourier_bp.py:97-267) in float64 on the host and uploads them once; the
// execute functions only enqueue kernels on the caller's stream.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <vector>

#define TB_API_KERNELS
#include "../../include/tb_bst.h"
#include "tb_kernels.cuh"
#include "tb_launch.cuh"

using tb::DevPlan;
using tb::Work;

thread_local std::string tb_g_err;

namespace {

constexpr double kPi = 3.14159265358979323846;
constexpr int kMaxL = 16384;

int next_pow2(long n) {
  long m = 1;
  while (m < n) m *= 2;
  return (int)m;
}

// Modified Bessel I0 by its power series (scipy.special.i0 in the reference,
// fourier_bp.py:187); converges to fp64 accuracy for the betas of interest.
double bessel_i0(double x) {
  const double y = 0.25 * x * x;
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 500; ++k) {
    term *= y / ((double)k * (double)k);
    sum += term;
    if (term < sum * 1e-17) break;
  }
  return sum;
}

size_t align_up(size_t x) { return (x + 511) & ~(size_t)511; }  // textureAlignment
}  // namespace

namespace {

// fused schedule (Launch<L>::fused_pipeline): 0 off (the measured best), 1
// K2(g) + K1(g+1), 2 K2(g) + K1(g+1) + K3(g-1); TB_FUSE selects (tuning)
int fuse_cfg() {
  const char* e = std::getenv("TB_FUSE");  // read per call: tests compare the schedules in one process
  const int x = e ? std::atoi(e) : 0;
  return (x >= 0 && x <= 2) ? x : 0;
}

// concurrent launch groups (streams) per call; TB_LANES overrides (tuning)
int lanes_cfg() {
  static const int v = [] {
    const char* e = std::getenv("TB_LANES");
    const int x = e ? std::atoi(e) : 0;
    return (x >= 1 && x <= 8) ? x : 2;
  }();
  return v;
}

struct Layout {
  size_t polar, rowcoef, part, common, common2, coefmean, columns, filtered, status, normtab, total;
  size_t lane_bytes;  // stride between the per-lane regions (all but status / normtab)
};

Layout layout_for(const tb_plan* p, int B) {
  Layout l;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  l.status = take(2 * sizeof(int));  // first: its offset does not depend on the batch
  l.normtab = take((size_t)p->rows * p->n_t * sizeof(float2));  // count-input frames table
  l.polar = take((size_t)B * p->dp.prow * p->H * sizeof(float2));
  l.rowcoef = take((size_t)B * p->rows * sizeof(float));
  l.part = take((size_t)B * p->groups * std::max(p->S, 1) * sizeof(float));
  l.common = take((size_t)B * p->H * sizeof(float2));
  l.common2 = take((size_t)B * p->dp.c2pitch * sizeof(float2));
  l.coefmean = take((size_t)B * sizeof(float));
  l.columns = take((size_t)B * p->dp.col_slice * sizeof(float2));
  l.filtered = take((size_t)B * p->rows * p->n_t * sizeof(float));
  l.lane_bytes = off - l.polar;
  l.total = off + (size_t)(lanes_cfg() - 1) * l.lane_bytes;
  return l;
}

cudaTextureObject_t polar_texture(const tb_plan* p, const void* ptr, int rows);

Work work_for(const tb_plan* p, int B, void* ws, int lane = 0) {
  Layout l = layout_for(p, B);
  char* base = static_cast<char*>(ws) + (size_t)lane * l.lane_bytes;
  Work w;
  w.polar = reinterpret_cast<float2*>(base + l.polar);
  w.rowcoef = reinterpret_cast<float*>(base + l.rowcoef);
  w.part = reinterpret_cast<float*>(base + l.part);
  w.common = reinterpret_cast<float2*>(base + l.common);
  w.common2 = reinterpret_cast<float2*>(base + l.common2);
  w.coefmean = reinterpret_cast<float*>(base + l.coefmean);
  w.columns = reinterpret_cast<float2*>(base + l.columns);
  w.filtered = reinterpret_cast<float*>(base + l.filtered);
  w.status = reinterpret_cast<int*>(static_cast<char*>(ws) + l.status);
  w.normtab = nullptr;
  w.pre_shift = nullptr;
  w.pre_stripe = nullptr;
  w.norm_eps = 0.f;
  w.norm_c = make_float2(0.f, 0.f);
  w.in_slice = (long long)p->rows * p->n_t;  // slice-major input by default
  w.in_row = p->n_t;
  w.groups = p->groups;
  w.pairs_per_cta = p->pairs_per_cta;
  w.polar_tex = polar_texture(p, w.polar, B * p->dp.prow);
  return w;
}

// Texture object viewing `rows` polar rows of H float2 texels at `ptr`
// (0 when the view does not fit the device's pitch-2D limits).
cudaTextureObject_t polar_texture(const tb_plan* p, const void* ptr, int rows) {
  // bilinear (half or full turn: K2_TEX / K2_TEXF) and half-turn nearest (K2_TEXN)
  if (p->desc.interp != TB_INTERP_BILINEAR && p->desc.full_turn) return 0;
  if (rows > 65000 || p->H > 65000) return 0;
  if (const char* e = std::getenv("TB_NOTEX")) if (std::atoi(e) == 1) return 0;  // A/B: plain gathers
  std::lock_guard<std::mutex> lk(p->tex_mu);
  for (const auto& t : p->texs)
    if (t.ptr == ptr && t.rows == rows) return t.obj;
  cudaResourceDesc res{};
  res.resType = cudaResourceTypePitch2D;
  res.res.pitch2D.devPtr = const_cast<void*>(ptr);
  res.res.pitch2D.desc = cudaCreateChannelDesc<float2>();
  res.res.pitch2D.width = (size_t)p->H;
  res.res.pitch2D.height = (size_t)rows;
  res.res.pitch2D.pitchInBytes = (size_t)p->H * sizeof(float2);
  cudaTextureDesc td{};
  // radial texels beyond H - 1 read as 0: nodes outside the disc (table x = H + 1)
  // gather zeros, and the clamp r1c = min(r0 + 1, H - 1) only matters at
  // r0 = H - 1, where the radial fraction is exactly 0
  td.addressMode[0] = cudaAddressModeBorder;
  td.addressMode[1] = cudaAddressModeClamp;
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  cudaTextureObject_t obj = 0;
  if (cudaCreateTextureObject(&obj, &res, &td, nullptr) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  p->texs.push_back({ptr, rows, obj});
  return obj;
}

// Texture object over `rows` image rows of n floats at `ptr` (forward
// projector), 0 when the pitch-2D view is not possible (alignment / size).
// Cached per plan like the polar views; the cache is bounded: evicting an
// entry waits for the device (kernels may still be reading it).
cudaTextureObject_t image_texture(const tb_plan* p, const void* ptr, int rows) {
  if (rows > 65000 || p->n > 65000) return 0;
  if (const char* e = std::getenv("TB_NOTEX")) if (std::atoi(e) == 1) return 0;
  int talign = 0, palign = 0;  // cudaDeviceGetAttribute: cheap, unlike cudaGetDeviceProperties
  if (cudaDeviceGetAttribute(&talign, cudaDevAttrTextureAlignment, p->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&palign, cudaDevAttrTexturePitchAlignment, p->device) != cudaSuccess || talign <= 0 ||
      palign <= 0) {
    cudaGetLastError();
    return 0;
  }
  const size_t pitch = (size_t)p->n * sizeof(float);
  if ((reinterpret_cast<uintptr_t>(ptr) % (uintptr_t)talign) != 0 || pitch % (size_t)palign != 0) return 0;
  std::lock_guard<std::mutex> lk(p->tex_mu);
  for (const auto& t : p->itexs)
    if (t.ptr == ptr && t.rows == rows) return t.obj;
  if (p->itexs.size() >= 16) {
    cudaDeviceSynchronize();
    for (auto& t : p->itexs) cudaDestroyTextureObject(t.obj);
    p->itexs.clear();
  }
  cudaResourceDesc res{};
  res.resType = cudaResourceTypePitch2D;
  res.res.pitch2D.devPtr = const_cast<void*>(ptr);
  res.res.pitch2D.desc = cudaCreateChannelDesc<float>();
  res.res.pitch2D.width = (size_t)p->n;
  res.res.pitch2D.height = (size_t)rows;
  res.res.pitch2D.pitchInBytes = pitch;
  cudaTextureDesc td{};
  td.addressMode[0] = cudaAddressModeBorder;  // columns -1 and n read 0 (projector.py zero padding)
  td.addressMode[1] = cudaAddressModeClamp;   // rows outside the slice are masked in the kernel
  td.filterMode = cudaFilterModePoint;
  td.readMode = cudaReadModeElementType;
  td.normalizedCoords = 0;
  cudaTextureObject_t obj = 0;
  if (cudaCreateTextureObject(&obj, &res, &td, nullptr) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  p->itexs.push_back({ptr, rows, obj});
  return obj;
}

}  // namespace

int ramp_dispatch(const tb_plan* p, const float* in, float* out, int total_rows, const Work& w, cudaStream_t st) {
  switch (p->npad) {
#define TB_CASE(N) \
  case N:          \
    return tb_ramp_##N(p, in, out, total_rows, w, st);
    TB_CASE(4) TB_CASE(8) TB_CASE(16) TB_CASE(32) TB_CASE(64) TB_CASE(128) TB_CASE(256) TB_CASE(512)
    TB_CASE(1024) TB_CASE(2048) TB_CASE(4096) TB_CASE(8192) TB_CASE(16384)
#undef TB_CASE
  }
  return fail(TB_ERR_UNSUPPORTED, "ramp length not supported on the GPU path");
}


namespace {

#define TB_CASE_CFG(N) case N: return tb_configure_##N(p);
#define TB_CASE_GRP(N) case N: return tb_group_##N(p, sino, img, B, w, ramp, scale, st, ev);
#define TB_CASE_PIPE(N) \
  case N: return tb_pipe_##N(p, sino, img, n_slices, batch, lanes, in_stride, out_stride, scale, with_k3, st);

int configure_dispatch(tb_plan* p) {
  switch (p->L) { TB_FOR_EACH_L(TB_CASE_CFG) }
  return fail(TB_ERR_UNSUPPORTED, "radial_samples not supported on the GPU path");
}

int bst_dispatch(const tb_plan* p, const float* sino, float* img, int B, const Work& w, bool ramp, float scale,
                 cudaStream_t st, cudaEvent_t* ev = nullptr) {
  switch (p->L) { TB_FOR_EACH_L(TB_CASE_GRP) }
  return fail(TB_ERR_UNSUPPORTED, "radial_samples not supported on the GPU path");
}

int pipe_dispatch(const tb_plan* p, const float* sino, float* img, int n_slices, int batch, const Work* lanes,
                  size_t in_stride, size_t out_stride, float scale, bool with_k3, cudaStream_t st) {
  switch (p->L) { TB_FOR_EACH_L(TB_CASE_PIPE) }
  return TB_ERR_UNSUPPORTED;
}

int check_exec_args(const tb_plan* p, const void* a, const void* b, int n_slices, int batch, const void* ws,
                    size_t ws_bytes) {
  if (!p) return fail(TB_ERR_INVALID, "null plan");
  if (n_slices < 0) return fail(TB_ERR_INVALID, "n_slices must be >= 0");
  if (n_slices > 0 && (!a || !b)) return fail(TB_ERR_INVALID, "null data pointer");
  if (batch < 1) return fail(TB_ERR_INVALID, "batch must be >= 1");
  if (ws) {
    size_t need = layout_for(p, batch).total;
    if (ws_bytes < need)
      return fail(TB_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need) + " bytes, got " +
                                        std::to_string(ws_bytes));
  } else {
    return fail(TB_ERR_WORKSPACE, "null workspace");
  }
  return TB_OK;
}

int set_device(const tb_plan* p) {
  int cur = -1;
  TB_CUDA(cudaGetDevice(&cur));
  if (cur != p->device) TB_CUDA(cudaSetDevice(p->device));
  return TB_OK;
}

// transmission-count input (tb_fbp_counts): flat / dark frames [rows][n_t]
struct NormFrames {
  const float* flat;  // null: constant frames i0 / d below
  const float* dark;
  double eps;
  double i0, d;
};

int run_bst_like(const tb_plan* p, const float* sino, float* img, int n_slices, int batch, void* ws,
                 size_t ws_bytes, void* stream, bool ramp, float scale, double* stage_ms = nullptr,
                 const NormFrames* norm = nullptr, bool frame_major = false, const float2* pre_shift = nullptr,
                 const float* pre_stripe = nullptr) {
  int rc = check_exec_args(p, sino, img, n_slices, batch, ws, ws_bytes);
  if (rc) return rc;
  if (!p->bst_ok)
    return fail(TB_ERR_INVALID, p->rows != (p->desc.full_turn ? 2 * p->V : p->V)
                                    ? "sinogram dimensions do not match the plan"
                                    : "plan was created without gridding tables (TB_PLAN_NO_GRID)");
  if ((rc = set_device(p))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float2* normtab = nullptr;
  float2 norm_c = make_float2(0.f, 0.f);
  if (norm && norm->flat) {  // (D, 1 / max(I0 - D, eps)) once per call, read by every slice's K1
    normtab = reinterpret_cast<float2*>(static_cast<char*>(ws) + layout_for(p, batch).normtab);
    const int cnt = p->rows * p->n_t;
    tb::k_norm_table<<<(cnt + 255) / 256, 256, 0, st>>>(norm->flat, norm->dark, (float)norm->eps, normtab, cnt);
    TB_CUDA(cudaGetLastError());
  } else if (norm) {  // constant frames: the same pair for every sample, no table loads
    const double den = norm->i0 - norm->d;
    norm_c = make_float2((float)norm->d, (float)(1.0 / (den != den ? den : std::max(den, norm->eps))));
  }
  // frame-major input [A][n_slices][n_t] (a TOMOVOL1 layout-0 slab): slice
  // q, row j at q n_t + j n_slices n_t -- read in place, no transpose
  const size_t in_stride = frame_major ? (size_t)p->n_t : (size_t)p->rows * p->n_t;
  const long long in_row = frame_major ? (long long)n_slices * p->n_t : (long long)p->n_t;
  const size_t out_stride = (size_t)p->n * p->n;
  const int ngroups = (n_slices + batch - 1) / batch;
  // the fused schedule (one stream, two workspace lanes) where it applies
  if (!stage_ms && ramp && !pre_shift && fuse_cfg() > 0 && lanes_cfg() >= 2 && ngroups >= 2) {
    Work lw[2];
    for (int l = 0; l < 2; ++l) {
      lw[l] = work_for(p, batch, ws, l);
      lw[l].in_slice = (long long)in_stride;
      lw[l].in_row = in_row;
      if (norm) {
        lw[l].normtab = normtab;
        lw[l].norm_eps = (float)norm->eps;
        lw[l].norm_c = norm_c;
      }
    }
    rc = pipe_dispatch(p, sino, img, n_slices, batch, lw, in_stride, out_stride, scale, fuse_cfg() == 2, st);
    if (rc != TB_ERR_UNSUPPORTED) return rc;
    rc = TB_OK;
  }
  std::vector<cudaEvent_t> evs;
  if (stage_ms) {
    for (int i = 0; i < 5; ++i) stage_ms[i] = 0.0;
    evs.resize((size_t)ngroups * 10);
    for (auto& e : evs) TB_CUDA(cudaEventCreate(&e));
  }
  // lanes: launch group g runs on lane g % lanes (lane 0 = the caller's
  // stream, the others auxiliary streams forked from it), each lane with its
  // own workspace region, so one group's serial K1b / kernel tails overlap
  // the other groups' work.  The profiled variant stays on one lane so
  // per-kernel times are clean.
  const int lanes = (stage_ms || ngroups < 2) ? 1 : std::min(lanes_cfg(), ngroups);
  cudaStream_t aux[8] = {};
  cudaEvent_t fork = nullptr, join = nullptr;
  if (lanes > 1) {
    TB_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    TB_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    TB_CUDA(cudaEventRecord(fork, st));
    for (int l = 1; l < lanes; ++l) {
      TB_CUDA(cudaStreamCreateWithFlags(&aux[l], cudaStreamNonBlocking));
      TB_CUDA(cudaStreamWaitEvent(aux[l], fork, 0));
    }
  }
  for (int g = 0; g < ngroups; ++g) {
    const int s0 = g * batch;
    const int B = std::min(batch, n_slices - s0);
    const int lane = g % lanes;
    Work w = work_for(p, batch, ws, lane);
    w.in_slice = (long long)in_stride;
    w.in_row = in_row;
    if (norm) {
      w.normtab = normtab;
      w.norm_eps = (float)norm->eps;
      w.norm_c = norm_c;
    }
    w.pre_shift = pre_shift ? pre_shift + s0 : nullptr;
    w.pre_stripe = pre_stripe ? pre_stripe + (size_t)s0 * p->n_t : nullptr;
    cudaStream_t ls = lane ? aux[lane] : st;
    rc = bst_dispatch(p, sino + s0 * in_stride, img + s0 * out_stride, B, w, ramp, scale, ls,
                      stage_ms ? evs.data() + (size_t)g * 10 : nullptr);
    if (rc) break;
  }
  if (lanes > 1) {
    for (int l = 1; l < lanes; ++l) {
      cudaEventRecord(join, aux[l]);
      cudaStreamWaitEvent(st, join, 0);
      cudaStreamDestroy(aux[l]);  // released once its queued work completes
    }
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
  }
  if (stage_ms) {
    if (!rc) {
      cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) rc = fail(TB_ERR_CUDA, cudaGetErrorString(e));
    }
    const bool unfused = ramp && p->npad != p->L;
    for (int g = 0; g < ngroups && !rc; ++g)
      for (int k = 0; k < 5; ++k) {
        if (k == 0 && !unfused) continue;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, evs[(size_t)g * 10 + 2 * k], evs[(size_t)g * 10 + 2 * k + 1]) == cudaSuccess)
          stage_ms[k] += ms;
      }
    for (auto& e : evs) cudaEventDestroy(e);
  }
  return rc;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int tb_abi_version(void) { return TB_ABI_VERSION; }

const char* tb_last_error(void) { return tb_g_err.c_str(); }

int tb_plan_create(const tb_plan_desc* d, int device, tb_plan** out) {
  if (!d || !out) return fail(TB_ERR_INVALID, "null argument");
  *out = nullptr;
  // --- validation: same rules and messages as BstPlan.__post_init__
  //     (fourier_bp.py:88-109) and FilterPlan.__post_init__ (:259-263)
  if (d->n_t < 2 || d->n_theta < 1) return fail(TB_ERR_INVALID, "need n_t >= 2 and n_theta >= 1");
  if (d->pad_factor < 2)
    return fail(TB_ERR_INVALID, "pad_factor must be >= 2, got " + std::to_string(d->pad_factor));
  if (d->sigma_min_bins < 1)
    return fail(TB_ERR_INVALID, "sigma_min_bins must be >= 1, got " + std::to_string(d->sigma_min_bins));
  if (d->interp != TB_INTERP_BILINEAR && d->interp != TB_INTERP_NEAREST)
    return fail(TB_ERR_INVALID, "unknown interp mode");
  long L = d->radial_samples > 0 ? d->radial_samples : next_pow2((long)d->pad_factor * d->n_t);
  if ((L & (L - 1)) || L < (long)d->pad_factor * d->n_t)
    return fail(TB_ERR_INVALID, "radial_samples must be a power of two >= pad_factor * n_t, got " +
                                    std::to_string(L));
  const int n = d->output_n > 0 ? d->output_n : d->n_t;
  if (n < 1 || n > L) return fail(TB_ERR_INVALID, "output_n must be in [1, radial_samples]");
  if (d->filter_kind != TB_FILTER_RAMP && d->filter_kind != TB_FILTER_RAMP_APODIZED)
    return fail(TB_ERR_INVALID, "unknown filter kind");
  if (!(d->rolloff > 0.0 && d->rolloff <= 1.0))
    return fail(TB_ERR_INVALID, "rolloff must be in (0, 1]");
  if (!(d->kb_support > 0.0)) return fail(TB_ERR_INVALID, "kb_support must be > 0");
  if (L > kMaxL) return fail(TB_ERR_UNSUPPORTED, "radial_samples > 16384 is not supported on the GPU path");
  const int rows_std = d->full_turn ? 2 * d->n_theta : d->n_theta;
  if (d->n_angles < 0) return fail(TB_ERR_INVALID, "n_angles must be >= 0");
  if (d->flags & ~TB_PLAN_NO_GRID) return fail(TB_ERR_INVALID, "unknown plan flags");

  tb_plan* p = new tb_plan();
  p->desc = *d;
  p->device = device;
  p->n_t = d->n_t;
  p->V = d->n_theta;
  p->rows = d->n_angles > 0 ? d->n_angles : rows_std;
  // the BST chain needs the standard layout and the gridding tables
  p->bst_ok = p->rows == rows_std && !(d->flags & TB_PLAN_NO_GRID);
  p->L = (int)L;
  p->H = (int)L / 2;
  p->n = n;
  p->npad = 2 * next_pow2(d->n_t);
  const int n_t = p->n_t, V = p->V, H = p->H;
  const int npad = p->npad;

  // --- scalar geometry (fourier_bp.py:119-152)
  const double dt = 2.0 / (n_t - 1);
  const double df = 1.0 / (L * dt);
  const double sigma_min = d->sigma_min_bins * df;
  const double du = 2.0 / n;
  const double dnu = 1.0 / (L * du);
  p->amp = (dnu * L) * (dnu * L) * dt;

  // --- KB window (fourier_bp.py:180-190) and its support, closed under i -> n_t-1-i
  std::vector<double> bump(n_t, 0.0);
  const double i0b = bessel_i0(d->kb_beta);
  int lo = n_t, hi = -1;
  for (int i = 0; i < n_t; ++i) {
    const double t = -1.0 + 2.0 * i / (n_t - 1);
    if (std::fabs(t) <= d->kb_support) {
      const double x = std::max(1.0 - (t / d->kb_support) * (t / d->kb_support), 0.0);
      bump[i] = bessel_i0(d->kb_beta * std::sqrt(x)) / i0b;
      lo = std::min(lo, i);
      hi = std::max(hi, i);
    }
  }
  if (hi >= lo) {
    const int lo2 = std::min(lo, n_t - 1 - hi), hi2 = std::max(hi, n_t - 1 - lo);
    lo = lo2;
    hi = hi2;
  } else {
    lo = 0;
    hi = -1;
  }
  p->lo = lo;
  p->hi = hi;
  p->S = hi - lo + 1;

  // --- K1 work split: <= 256 CTAs (partial-sum groups) per slice
  const int npairs = (p->rows + 1) / 2;
  p->pairs_per_cta = std::max(1, (npairs + 255) / 256);
  if (const char* e = std::getenv("TB_K1_PAIRS"))  // tuning: row pairs per K1 CTA
    if (std::atoi(e) > 0) p->pairs_per_cta = std::atoi(e);
  p->groups = (npairs + p->pairs_per_cta - 1) / p->pairs_per_cta;

  // --- host tables
  auto tw = [](int N) {
    std::vector<float2> v(N);
    for (int j = 0; j < N; ++j) {
      const double a = 2.0 * kPi * (double)j / N;
      v[j] = make_float2((float)std::cos(a), (float)-std::sin(a));
    }
    return v;
  };
  std::vector<float2> twL = tw((int)L), twN = tw(npad);

  // ramp multiplier 2 pi |f| (x raised-cosine taper) / npad (fourier_bp.py:477-487)
  std::vector<float> g(npad);
  {
    const double val = 1.0 / (npad * dt);
    const double fnyq = (npad / 2) * val;
    const bool apod = d->filter_kind == TB_FILTER_RAMP_APODIZED && d->rolloff < 1.0;
    for (int k = 0; k < npad; ++k) {
      const int kk = std::min(k, npad - k);
      const double f = kk * val;
      double m = 2.0 * kPi * std::fabs(f);
      if (apod) {
        const double start = d->rolloff * fnyq;
        if (f > start) {
          const double frac = (f - start) / ((1.0 - d->rolloff) * fnyq);
          m *= 0.5 * (1.0 + std::cos(kPi * frac));
        }
      }
      g[k] = (float)(m / npad);
    }
  }
  std::vector<float> omb(n_t), bump_s(std::max(p->S, 1), 0.f);
  for (int i = 0; i < n_t; ++i) omb[i] = (float)(1.0 - bump[i]);
  for (int s = 0; s < p->S; ++s) bump_s[s] = (float)bump[lo + s];

  // true-origin phase, reference spectrum and kernel denominator over k < H
  // (fourier_bp.py:164-202, 372): S_k = exp(2 pi i f_k) sum_i w_i exp(-2 pi i k i / L)
  std::vector<float2> psi(H), rho(H);
  {
    const double val = 1.0 / (L * dt);
    for (int k = 0; k < H; ++k) {
      const double f = k * val;
      const double den = std::max(std::fabs(f), sigma_min);
      const double ph = 2.0 * kPi * f;
      const double pr = std::cos(ph), pim = std::sin(ph);
      double sr, si;
      if (k == 0) {
        sr = n_t;
        si = 0.0;
      } else {
        // sum_{i<n_t} z^i with z = exp(-2 pi i k / L)
        const double a1 = -2.0 * kPi * (double)k / L;
        const double an = -2.0 * kPi * (double)(((long long)k * n_t) % L) / L;
        const double nr = 1.0 - std::cos(an), ni = -std::sin(an);
        const double dr = 1.0 - std::cos(a1), di = -std::sin(a1);
        const double dd = dr * dr + di * di;
        sr = (nr * dr + ni * di) / dd;
        si = (ni * dr - nr * di) / dd;
      }
      psi[k] = make_float2((float)(pr / den), (float)(pim / den));
      rho[k] = make_float2((float)((pr * sr - pim * si) / den), (float)((pr * si + pim * sr) / den));
    }
  }
  // half-node modulation (fourier_bp.py:424-430)
  std::vector<float2> modt(L, make_float2(1.f, 0.f));
  int has_mod = 0;
  {
    const long m0 = L / 2 - n / 2;
    const double delta = (-1.0 + 1.0 / n) - (double)(m0 - L / 2) * du;
    if (delta != 0.0) {
      has_mod = 1;
      for (long k = 0; k < L; ++k) {
        const long ks = k < L / 2 ? k : k - L;
        const double a = 2.0 * kPi * ((double)ks * dnu) * delta;
        modt[k] = make_float2((float)std::cos(a), (float)std::sin(a));
      }
    }
  }
  // per-pass twiddle bases of fft_mod (fft.cuh) for the column IFFT of an
  // n = L/2 crop, whose half-node modulation is exp(i alpha k), alpha = pi/L:
  // pass p >= 1 (radix-16 passes, then one remainder) holds ns(p) entries
  // W_L^{k s_p} exp(-i alpha s_p), s_p = L / (ns(p) radix(p))
  std::vector<float2> twm;
  {
    int P = 0;
    while ((1L << P) < L) ++P;
    const int rpt = L < 16 ? (int)L : 16;
    int lr = 0;
    while ((1 << lr) < rpt) ++lr;
    const int nfull = lr ? P / lr : 0, rem = lr ? 1 << (P % lr) : 1;
    const int npass = nfull + (rem > 1 ? 1 : 0);
    long ns = 1;
    for (int q = 0; q < npass; ++q) {
      const long radix = q < nfull ? rpt : rem;
      if (q >= 1) {
        const long stride = L / (ns * radix);
        for (long k = 0; k < ns; ++k) {
          const double a = -2.0 * kPi * (double)(k * stride) / L - kPi * (double)stride / L;
          twm.push_back(make_float2((float)std::cos(a), (float)std::sin(a)));
        }
      }
      ns *= radix;
    }
    if (twm.empty()) twm.push_back(make_float2(1.f, 0.f));
  }
  // slant-stack angles (grids.py:85-95; projector.py:137-141)
  const int A = p->rows;
  const double span = d->full_turn ? 2.0 * kPi : kPi;
  std::vector<double2> sscs(A);
  for (int j = 0; j < A; ++j) {
    const double th = (double)j * (span / A);
    sscs[j] = make_double2(std::cos(th), std::sin(th));
  }

  // --- upload everything in one allocation
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  const size_t o_twL = take(twL.size() * sizeof(float2));
  const size_t o_twN = take(twN.size() * sizeof(float2));
  const size_t o_g = take(g.size() * sizeof(float));
  const size_t o_omb = take(omb.size() * sizeof(float));
  const size_t o_bs = take(bump_s.size() * sizeof(float));
  const size_t o_psi = take(psi.size() * sizeof(float2));
  const size_t o_rho = take(rho.size() * sizeof(float2));
  const size_t o_mod = take(modt.size() * sizeof(float2));
  const size_t o_ss = take(sscs.size() * sizeof(double2));
  const size_t o_twm = take(twm.size() * sizeof(float2));
  std::vector<char> host(off, 0);
  auto put = [&](size_t o, const void* src, size_t bytes) { std::memcpy(host.data() + o, src, bytes); };
  put(o_twL, twL.data(), twL.size() * sizeof(float2));
  put(o_twN, twN.data(), twN.size() * sizeof(float2));
  put(o_g, g.data(), g.size() * sizeof(float));
  put(o_omb, omb.data(), omb.size() * sizeof(float));
  put(o_bs, bump_s.data(), bump_s.size() * sizeof(float));
  put(o_psi, psi.data(), psi.size() * sizeof(float2));
  put(o_rho, rho.data(), rho.size() * sizeof(float2));
  put(o_mod, modt.data(), modt.size() * sizeof(float2));
  put(o_ss, sscs.data(), sscs.size() * sizeof(double2));
  put(o_twm, twm.data(), twm.size() * sizeof(float2));

  int prev = -1;
  cudaGetDevice(&prev);
  auto cleanup = [&](int code, const std::string& msg) {
    if (p->blob) cudaFree(p->blob);
    if (p->table) cudaFree(p->table);
    if (p->table2) cudaFree(p->table2);
    delete p;
    if (prev >= 0) cudaSetDevice(prev);
    return fail(code, msg);
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cleanup(TB_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  e = cudaMalloc(&p->blob, off);
  if (e != cudaSuccess) return cleanup(TB_ERR_CUDA, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  e = cudaMemcpy(p->blob, host.data(), off, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cleanup(TB_ERR_CUDA, std::string("cudaMemcpy: ") + cudaGetErrorString(e));
  char* b = static_cast<char*>(p->blob);

  DevPlan& dp = p->dp;
  dp.n_t = n_t;
  dp.n_theta = V;
  dp.rows = p->rows;
  dp.L = (int)L;
  dp.H = H;
  dp.n = n;
  dp.npad = npad;
  dp.lo = lo;
  dp.S = p->S;
  dp.full_turn = d->full_turn ? 1 : 0;
  dp.interp = d->interp;
  const double cr = dnu / df;
  // Nyquist lines can hold in-disc nodes only if H*cr <= H - 1 (+1/2 for rounding)
  dp.nyq = (H * cr <= (H - 1) + 0.5 + 1e-9) ? 1 : 0;
  dp.has_mod = has_mod;
  dp.n_half = n / 2;
  dp.inv_nt = (float)(1.0 / n_t);
  dp.inv_rows2 = (float)(1.0 / (2.0 * V));
  dp.img_scale = (float)(p->amp / ((double)L * (double)L));
  dp.ss_weight = (float)(span / A);
  dp.ss_inv_dt = (float)(1.0 / dt);
  dp.tw_L = reinterpret_cast<const float2*>(b + o_twL);
  dp.tw_np = reinterpret_cast<const float2*>(b + o_twN);
  dp.ramp_g = reinterpret_cast<const float*>(b + o_g);
  dp.omb = reinterpret_cast<const float*>(b + o_omb);
  dp.bump_s = reinterpret_cast<const float*>(b + o_bs);
  dp.psi = reinterpret_cast<const float2*>(b + o_psi);
  dp.rho = reinterpret_cast<const float2*>(b + o_rho);
  dp.modt = reinterpret_cast<const float2*>(b + o_mod);
  dp.twm = reinterpret_cast<const float2*>(b + o_twm);
  // per-slice K2 output padded to 128 B: slices never share a cache line
  dp.col_slice = (((size_t)((n + 3) / 4) * (H + 1) * 4 + 15) / 16) * 16;
  // polar rows per slice: the V (2V) measured angles plus the angle-pi
  // (angle-2 pi) mirror of row 0 that the TLD4 gathers read
  dp.prow = d->full_turn ? 2 * V + 1 : V + 1;
  dp.c2pitch = H + 16;  // 128-B aligned rows; entries >= H are zero (outside-disc nodes)
  dp.ss_cs = reinterpret_cast<const double2*>(b + o_ss);

  // gridding table (fourier_bp.py:222-249), built on the device in fp64
  if (p->bst_ok && (long long)V / 2 >= 65535)
    return cleanup(TB_ERR_UNSUPPORTED, "n_theta too large for the gridding table");
  dp.gridtab = nullptr;
  if (p->bst_ok) {
    const long long cnt = (long long)(H + 1) * (H + 1);
    e = cudaMalloc(&p->table, cnt * sizeof(uint2));
    if (e != cudaSuccess) return cleanup(TB_ERR_CUDA, std::string("cudaMalloc(table): ") + cudaGetErrorString(e));
    tb::build_grid_table<<<(unsigned)((cnt + 255) / 256), 256>>>(static_cast<uint2*>(p->table), H, dnu, df,
                                                                  (2.0 * V) / (2.0 * kPi), d->interp);
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cleanup(TB_ERR_CUDA, std::string("build_grid_table: ") + cudaGetErrorString(e));
    dp.gridtab = static_cast<const uint2*>(p->table);
  }
  dp.gridtab2 = nullptr;
  dp.colext = nullptr;
  if (p->bst_ok && (d->interp == TB_INTERP_BILINEAR || !d->full_turn)) {
    const long long cnt = (long long)(H + 1) * (H + 1);
    // the table, then the per-column inside extents ((H + 1) ints)
    e = cudaMalloc(&p->table2, cnt * sizeof(float4) + (size_t)(H + 1) * sizeof(int));
    if (e != cudaSuccess) return cleanup(TB_ERR_CUDA, std::string("cudaMalloc(table2): ") + cudaGetErrorString(e));
    float4* t2 = static_cast<float4*>(p->table2);
    int* ext = reinterpret_cast<int*>(t2 + cnt);
    tb::build_grid_table2<<<(unsigned)((cnt + 255) / 256), 256>>>(t2, H, V, dnu, df, (2.0 * V) / (2.0 * kPi),
                                                                   d->interp == TB_INTERP_NEAREST ? 1 : 0);
    tb::build_col_extent<<<(unsigned)(H + 1), 256>>>(t2, ext, H);
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cleanup(TB_ERR_CUDA, std::string("build_grid_table2: ") + cudaGetErrorString(e));
    dp.gridtab2 = t2;
    dp.colext = ext;
  }

  int rc = configure_dispatch(p);
  if (rc) {
    std::string m = tb_g_err;
    return cleanup(rc, m);
  }
  if (prev >= 0 && prev != device) cudaSetDevice(prev);
  *out = p;
  return TB_OK;
}

int tb_plan_destroy(tb_plan* p) {
  if (!p) return TB_OK;
  if (p->blob) {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(p->device);
    // calls are asynchronous: kernels enqueued with this plan (on any
    // stream) may still read its tables and texture objects
    cudaDeviceSynchronize();
    for (auto& t : p->texs) cudaDestroyTextureObject(t.obj);
    for (auto& t : p->itexs) cudaDestroyTextureObject(t.obj);
    cudaFree(p->blob);
    if (p->table) cudaFree(p->table);
    if (p->table2) cudaFree(p->table2);
    if (prev >= 0) cudaSetDevice(prev);
  }
  delete p;
  return TB_OK;
}

int tb_plan_get_info(const tb_plan* p, tb_plan_info* info) {
  if (!p || !info) return fail(TB_ERR_INVALID, "null argument");
  info->n_t = p->n_t;
  info->n_theta = p->V;
  info->n_angles = p->rows;
  info->radial_samples = p->L;
  info->ramp_samples = p->npad;
  info->output_n = p->n;
  info->support_lo = p->lo;
  info->support_hi = p->hi;
  info->amplitude_scale = p->amp;
  return TB_OK;
}

int tb_workspace_bytes(const tb_plan* p, int batch, size_t* bytes) {
  if (!p || !bytes) return fail(TB_ERR_INVALID, "null argument");
  if (batch < 1) return fail(TB_ERR_INVALID, "batch must be >= 1");
  *bytes = layout_for(p, batch).total;
  return TB_OK;
}

int tb_workspace_get_layout(const tb_plan* p, int batch, tb_workspace_layout* out) {
  if (!p || !out) return fail(TB_ERR_INVALID, "null argument");
  if (batch < 1) return fail(TB_ERR_INVALID, "batch must be >= 1");
  Layout l = layout_for(p, batch);
  out->total = l.total;
  out->polar = l.polar;
  out->rowcoef = l.rowcoef;
  out->common = l.common;
  out->coefmean = l.coefmean;
  out->columns = l.columns;
  out->filtered = l.filtered;
  out->status = l.status;
  return TB_OK;
}

int tb_fbp(const tb_plan* p, const float* sino, float* image, int n_slices, int batch, void* ws, size_t ws_bytes,
           void* stream) {
  return run_bst_like(p, sino, image, n_slices, batch, ws, ws_bytes, stream, true, (float)(1.0 / (2.0 * kPi)));
}

int tb_fbp_profiled(const tb_plan* p, const float* sino, float* image, int n_slices, int batch, void* ws,
                    size_t ws_bytes, void* stream, double* stage_ms) {
  if (!stage_ms) return fail(TB_ERR_INVALID, "null stage_ms");
  return run_bst_like(p, sino, image, n_slices, batch, ws, ws_bytes, stream, true, (float)(1.0 / (2.0 * kPi)),
                      stage_ms);
}

int tb_fbp_counts(const tb_plan* p, const float* counts, const float* flat, const float* dark, double eps,
                  float* image, int n_slices, int batch, void* ws, size_t ws_bytes, void* stream) {
  if (!(eps > 0.0)) return fail(TB_ERR_INVALID, "eps must be positive");
  if (n_slices > 0 && (!flat || !dark)) return fail(TB_ERR_INVALID, "null flat/dark frame");
  const NormFrames nf{flat, dark, eps, 0.0, 0.0};
  return run_bst_like(p, counts, image, n_slices, batch, ws, ws_bytes, stream, true, (float)(1.0 / (2.0 * kPi)),
                      nullptr, &nf);
}

int tb_fbp_counts_const(const tb_plan* p, const float* counts, double i0, double dark, double eps, float* image,
                        int n_slices, int batch, void* ws, size_t ws_bytes, void* stream) {
  if (!(eps > 0.0)) return fail(TB_ERR_INVALID, "eps must be positive");
  const NormFrames nf{nullptr, nullptr, eps, i0, dark};
  return run_bst_like(p, counts, image, n_slices, batch, ws, ws_bytes, stream, true, (float)(1.0 / (2.0 * kPi)),
                      nullptr, &nf);
}

int tb_fbp_frames(const tb_plan* p, const float* frames, float* image, int n_slices, int batch, void* ws,
                  size_t ws_bytes, void* stream) {
  return run_bst_like(p, frames, image, n_slices, batch, ws, ws_bytes, stream, true, (float)(1.0 / (2.0 * kPi)),
                      nullptr, nullptr, true);
}

int tb_normalize(const tb_plan* p, const float* counts, const float* flat, const float* dark, double eps, float* out,
                 int n_slices, void* stream) {
  if (!p) return fail(TB_ERR_INVALID, "null plan");
  if (!(eps > 0.0)) return fail(TB_ERR_INVALID, "eps must be positive");
  if (n_slices < 0) return fail(TB_ERR_INVALID, "n_slices must be >= 0");
  if (n_slices == 0) return TB_OK;
  if (!counts || !flat || !dark || !out) return fail(TB_ERR_INVALID, "null data pointer");
  int rc = set_device(p);
  if (rc) return rc;
  const int frame = p->rows * p->n_t;
  const long long total = (long long)n_slices * frame;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
  tb::k_normalize<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(counts, flat, dark, (float)eps, out, total,
                                                                         frame);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_bst(const tb_plan* p, const float* sino, float* image, int n_slices, int batch, void* ws, size_t ws_bytes,
           void* stream) {
  return run_bst_like(p, sino, image, n_slices, batch, ws, ws_bytes, stream, false, 1.0f);
}

int tb_bst_scaled(const tb_plan* p, const float* sino, float* image, int n_slices, int batch, void* ws,
                  size_t ws_bytes, float scale, void* stream) {
  return run_bst_like(p, sino, image, n_slices, batch, ws, ws_bytes, stream, false, scale);
}

int tb_ramp(const tb_plan* p, const float* sino, float* out, int n_slices, void* stream) {
  if (!p) return fail(TB_ERR_INVALID, "null plan");
  if (n_slices < 0) return fail(TB_ERR_INVALID, "n_slices must be >= 0");
  if (n_slices == 0) return TB_OK;
  if (!sino || !out) return fail(TB_ERR_INVALID, "null data pointer");
  int rc = set_device(p);
  if (rc) return rc;
  Work w{};
  w.status = nullptr;
  w.in_slice = (long long)p->rows * p->n_t;
  w.in_row = p->n_t;
  return ramp_dispatch(p, sino, out, n_slices * p->rows, w, static_cast<cudaStream_t>(stream));
}

int tb_ss(const tb_plan* p, const float* sino, float* image, int n_slices, float scale, void* stream) {
  if (!p) return fail(TB_ERR_INVALID, "null plan");
  if (n_slices < 0) return fail(TB_ERR_INVALID, "n_slices must be >= 0");
  if (n_slices == 0) return TB_OK;
  if (!sino || !image) return fail(TB_ERR_INVALID, "null data pointer");
  int rc = set_device(p);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Work w{};
  w.status = nullptr;  // no workspace: the caller validates finiteness
  const int n = p->n;
  dim3 grid((n + tb::kSsTile - 1) / tb::kSsTile, (n + tb::kSsTile - 1) / tb::kSsTile, 1);
  for (int s = 0; s < n_slices; s += 65535) {
    const int B = std::min(65535, n_slices - s);
    grid.z = B;
    tb::k5_slant<<<grid, 256, 0, st>>>(p->dp, sino + (size_t)s * p->rows * p->n_t, p->rows,
                                       image + (size_t)s * n * n, scale, w);
  }
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_forward(const tb_plan* p, const float* image, float* sino, int n_slices, double step_length, int interp,
               void* stream) {
  if (!p) return fail(TB_ERR_INVALID, "null plan");
  if (!(step_length > 0.0 && step_length <= 1.0))
    return fail(TB_ERR_INVALID, "step_length must be in (0, 1], got " + std::to_string(step_length));
  if (interp != TB_INTERP_BILINEAR && interp != TB_INTERP_NEAREST) return fail(TB_ERR_INVALID, "unknown interpolation");
  if (n_slices < 0) return fail(TB_ERR_INVALID, "n_slices must be >= 0");
  if (n_slices == 0) return TB_OK;
  if (!image || !sino) return fail(TB_ERR_INVALID, "null data pointer");
  int rc = set_device(p);
  if (rc) return rc;
  // projector.py:106-110: h = step x pixel size, m = ceil(2 sqrt2 / h)
  const double h = step_length * (2.0 / p->n);
  const int m = (int)std::ceil(2.0 * std::sqrt(2.0) / h);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t nn = (size_t)p->n * p->n;
  // TLD4 gathers (bilinear) or point fetches (nearest) from a pitch-2D
  // texture over runs of slices (image_texture; rows <= the pitch-2D height
  // limit); an image the texture unit cannot view takes the plain-load kernel
  const int per_tex = std::max(1, 65000 / p->n);
  for (int s = 0; s < n_slices;) {
    const int B = std::min(std::min(65535, per_tex), n_slices - s);
    const float* im = image + (size_t)s * nn;
    dim3 grid((p->n_t + 127) / 128, p->rows, B);
    cudaTextureObject_t tex = image_texture(p, im, B * p->n);
    if (tex && interp == TB_INTERP_NEAREST)
      tb::k6_forward_tex<true><<<grid, 128, 0, st>>>(p->dp, tex, sino + (size_t)s * p->rows * p->n_t, p->rows, h, m);
    else if (tex)
      tb::k6_forward_tex<false><<<grid, 128, 0, st>>>(p->dp, tex, sino + (size_t)s * p->rows * p->n_t, p->rows, h, m);
    else
      tb::k6_forward<<<grid, 128, 0, st>>>(p->dp, im, sino + (size_t)s * p->rows * p->n_t, p->rows, h, m,
                                            interp == TB_INTERP_NEAREST ? 1 : 0);
    s += B;
  }
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

namespace {
int check_rows_call(const tb_plan* p, const void* a, const void* b, int n_slices) {
  if (!p) return fail(TB_ERR_INVALID, "null plan");
  if (n_slices < 0) return fail(TB_ERR_INVALID, "n_slices must be >= 0");
  if (n_slices > 0 && (!a || !b)) return fail(TB_ERR_INVALID, "null data pointer");
  return TB_OK;
}
}  // namespace

int tb_center_estimate(const tb_plan* p, const float* sino, int n_slices, double* beta_conf, int* status,
                       void* stream) {
  int rc = check_rows_call(p, sino, beta_conf, n_slices);
  if (rc) return rc;
  if (n_slices > 0 && !status) return fail(TB_ERR_INVALID, "null status pointer");
  if (p->rows < 2) return fail(TB_ERR_INVALID, "need at least two projection angles");
  if (n_slices == 0) return TB_OK;
  if ((rc = set_device(p))) return rc;
  const int T = 512;
  const size_t sm = (size_t)(4 * p->n_t - 1) * sizeof(double) + (size_t)2 * T * sizeof(double) + (size_t)T * sizeof(int);
  TB_CUDA(cudaFuncSetAttribute(tb::k_center_estimate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  tb::k_center_estimate<<<n_slices, T, sm, static_cast<cudaStream_t>(stream)>>>(
      sino, p->rows, p->n_t, reinterpret_cast<double2*>(beta_conf), status);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_center_apply(const tb_plan* p, const float* sino, const double* beta_conf, float* out, int n_slices,
                    void* stream) {
  int rc = check_rows_call(p, sino, out, n_slices);
  if (rc) return rc;
  if (n_slices > 0 && !beta_conf) return fail(TB_ERR_INVALID, "null beta pointer");
  if (n_slices == 0) return TB_OK;
  if ((rc = set_device(p))) return rc;
  for (int s = 0; s < n_slices; s += 65535) {
    const int B = std::min(65535, n_slices - s);
    dim3 grid((p->n_t + 255) / 256, p->rows, B);
    tb::k_center_apply<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        sino + (size_t)s * p->rows * p->n_t, out + (size_t)s * p->rows * p->n_t,
        reinterpret_cast<const double2*>(beta_conf) + s, p->rows, p->n_t);
  }
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_rings(const tb_plan* p, const float* sino, float* out, int window, double* scratch, int n_slices,
             void* stream) {
  int rc = check_rows_call(p, sino, out, n_slices);
  if (rc) return rc;
  if (window < 3 || window % 2 == 0)
    return fail(TB_ERR_INVALID, "window must be an odd integer >= 3, got " + std::to_string(window));
  if (n_slices > 0 && !scratch) return fail(TB_ERR_INVALID, "null scratch pointer");
  if (n_slices == 0) return TB_OK;
  if ((rc = set_device(p))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int s = 0; s < n_slices; s += 65535) {
    const int B = std::min(65535, n_slices - s);
    dim3 grid((p->n_t + 255) / 256, B);
    const float* in = sino + (size_t)s * p->rows * p->n_t;
    tb::k_col_mean<<<dim3((p->n_t + 31) / 32, B), dim3(32, 8), 0, st>>>(in, scratch, p->rows, p->n_t);
    tb::k_rings_apply<<<grid, 256, 0, st>>>(in, out + (size_t)s * p->rows * p->n_t, scratch, p->rows, p->n_t,
                                             window);
  }
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_pre_params(const tb_plan* p, const float* sino, int n_slices, const double* beta_conf, int window,
                  double* mean_scratch, float* shift, float* stripe, void* stream) {
  int rc = check_rows_call(p, sino, shift, n_slices);
  if (rc) return rc;
  if (window != 0 && (window < 3 || window % 2 == 0))
    return fail(TB_ERR_INVALID, "window must be an odd integer >= 3, got " + std::to_string(window));
  if (n_slices > 0 && window && (!mean_scratch || !stripe)) return fail(TB_ERR_INVALID, "null scratch / stripe pointer");
  if (n_slices == 0) return TB_OK;
  if ((rc = set_device(p))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int s = 0; s < n_slices; s += 65535) {
    const int B = std::min(65535, n_slices - s);
    if (window)
      tb::k_col_mean<<<dim3((p->n_t + 31) / 32, B), dim3(32, 8), 0, st>>>(sino + (size_t)s * p->rows * p->n_t,
                                                                          mean_scratch, p->rows, p->n_t);
    tb::k_pre_params<<<B, 256, 0, st>>>(beta_conf ? beta_conf + 2 * (size_t)s : nullptr, mean_scratch, p->n_t, window,
                                        reinterpret_cast<float2*>(shift) + s,
                                        window ? stripe + (size_t)s * p->n_t : nullptr);
  }
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_fbp_pre(const tb_plan* p, const float* sino, float* image, int n_slices, int batch, void* ws,
               size_t ws_bytes, const float* shift, const float* stripe, void* stream) {
  if (!p) return fail(TB_ERR_INVALID, "null plan");
  if (n_slices > 0 && !shift) return fail(TB_ERR_INVALID, "null shift pointer");
  // the stages act on the raw rows, so K1 must run the ramp filter itself
  if (p->npad != p->L) return fail(TB_ERR_UNSUPPORTED, "fused centre / rings need the ramp fused into K1 (npad == L)");
  return run_bst_like(p, sino, image, n_slices, batch, ws, ws_bytes, stream, true, (float)(1.0 / (2.0 * kPi)),
                      nullptr, nullptr, false, reinterpret_cast<const float2*>(shift), stripe);
}

int tb_fbp_ss(const tb_plan* p, const float* sino, float* image, int n_slices, int batch, void* ws,
              size_t ws_bytes, void* stream) {
  int rc = check_exec_args(p, sino, image, n_slices, batch, ws, ws_bytes);
  if (rc) return rc;
  if ((rc = set_device(p))) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int n = p->n;
  for (int s0 = 0; s0 < n_slices; s0 += batch) {
    const int B = std::min(batch, n_slices - s0);
    Work w = work_for(p, batch, ws);
    rc = ramp_dispatch(p, sino + (size_t)s0 * p->rows * p->n_t, w.filtered, B * p->rows, w, st);
    if (rc) return rc;
    dim3 grid((n + tb::kSsTile - 1) / tb::kSsTile, (n + tb::kSsTile - 1) / tb::kSsTile, B);
    tb::k5_slant<<<grid, 256, 0, st>>>(p->dp, w.filtered, p->rows, image + (size_t)s0 * n * n,
                                       (float)(1.0 / (2.0 * kPi)), w);
    TB_CUDA(cudaGetLastError());
  }
  return TB_OK;
}

int tb_reset_status(const tb_plan* p, void* ws, void* stream) {
  if (!p || !ws) return fail(TB_ERR_INVALID, "null argument");
  int rc = set_device(p);
  if (rc) return rc;
  Layout l = layout_for(p, 1);
  TB_CUDA(cudaMemsetAsync(static_cast<char*>(ws) + l.status, 0, 2 * sizeof(int),
                          static_cast<cudaStream_t>(stream)));
  return TB_OK;
}

int tb_copy_polar(const tb_plan* p, const void* ws, int batch, void* dst, void* stream) {
  if (!p || !ws || !dst || batch < 1) return fail(TB_ERR_INVALID, "tb_copy_polar: bad argument");
  int rc = set_device(p);
  if (rc) return rc;
  const Layout l = layout_for(p, batch);
  const size_t bytes = (size_t)batch * p->dp.prow * p->H * sizeof(float2);
  TB_CUDA(cudaMemcpyAsync(dst, static_cast<const char*>(ws) + l.polar, bytes, cudaMemcpyDeviceToDevice,
                          static_cast<cudaStream_t>(stream)));
  return TB_OK;
}

int tb_read_status(const tb_plan* p, const void* ws, void* stream) {
  if (!p || !ws) return fail(TB_ERR_INVALID, "null argument");
  int rc = set_device(p);
  if (rc) return rc;
  Layout l = layout_for(p, 1);
  int h[2] = {0, 0};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  TB_CUDA(cudaMemcpyAsync(h, static_cast<const char*>(ws) + l.status, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  TB_CUDA(cudaStreamSynchronize(st));
  if (h[0]) return fail(TB_ERR_NONFINITE_INPUT, "sinogram contains non-finite values");
  if (h[1]) return fail(TB_ERR_NONFINITE_OUTPUT, "non-finite values in backprojection output");
  return TB_OK;
}

}  // extern "C"
