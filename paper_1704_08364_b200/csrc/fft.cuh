// fft.cuh -- register/shared-memory Stockham FFT building blocks for sm_100a.
//
// One length-N complex transform is owned by TPF = N/RPT threads, each holding
// RPT = min(16, N) points in registers.  Layout contract (in and out):
//
//     thread t holds x[t + i*TPF] in v[i],  i < RPT
//
// Passes are radix-16 (two radix-4 stages with constant inner twiddles) with one
// radix-2/4/8 remainder pass last.  The first pass reads its butterfly inputs
// straight from registers and the last pass leaves its outputs in registers in
// the same layout, so an N=4096 transform makes exactly two shared-memory round
// trips.  Between passes data goes through a padded smem buffer
// (index i -> i + i/16: conflict-free for the strided Stockham stores).
//
// Forward = exp(-2 pi i jk/N) (numpy.fft.fft), inverse = exp(+2 pi i jk/N)
// without the 1/N (callers fold normalisation into their epilogues).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tb {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }

// multiply by W^{N/4}: -i (forward) / +i (inverse)
template <bool INV>
__device__ __forceinline__ float2 mul_q1(float2 a) {
  return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }

// cos/sin(2 pi k / 16)
struct Trig16 {
  static constexpr float c[16] = {1.0f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                                  0.0f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                                  -1.0f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f,
                                  0.0f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f};
  static constexpr float s[16] = {0.0f, 0.38268343236508977f, 0.70710678118654752f, 0.92387953251128674f,
                                  1.0f, 0.92387953251128674f, 0.70710678118654752f, 0.38268343236508977f,
                                  0.0f, -0.38268343236508977f, -0.70710678118654752f, -0.92387953251128674f,
                                  -1.0f, -0.92387953251128674f, -0.70710678118654752f, -0.38268343236508977f};
};

// cos/sin(2 pi k / 64) (64-point transforms, 64 points per thread)
struct Trig64 {
  static constexpr float c[64] = {1.0f, 0.99518472667219693f, 0.98078528040323043f, 0.95694033573220882f, 0.92387953251128674f, 0.88192126434835505f, 0.83146961230254524f, 0.77301045336273699f, 0.70710678118654757f, 0.63439328416364549f, 0.55557023301960229f, 0.47139673682599781f, 0.38268343236508984f, 0.29028467725446233f, 0.19509032201612833f, 0.09801714032956077f, 0.0f, -0.098017140329560645f, -0.19509032201612819f, -0.29028467725446216f, -0.38268343236508973f, -0.4713967368259977f, -0.55557023301960196f, -0.63439328416364538f, -0.70710678118654746f, -0.77301045336273699f, -0.83146961230254535f, -0.88192126434835494f, -0.92387953251128674f, -0.95694033573220882f, -0.98078528040323043f, -0.99518472667219682f, -1.0f, -0.99518472667219693f, -0.98078528040323043f, -0.95694033573220894f, -0.92387953251128685f, -0.88192126434835505f, -0.83146961230254546f, -0.7730104533627371f, -0.70710678118654768f, -0.63439328416364593f, -0.55557023301960218f, -0.47139673682599786f, -0.38268343236509034f, -0.29028467725446244f, -0.19509032201612866f, -0.098017140329560451f, 0.0f, 0.09801714032956009f, 0.1950903220161283f, 0.29028467725446205f, 0.38268343236509f, 0.47139673682599759f, 0.55557023301960184f, 0.6343932841636456f, 0.70710678118654735f, 0.77301045336273666f, 0.83146961230254524f, 0.88192126434835483f, 0.92387953251128652f, 0.95694033573220882f, 0.98078528040323032f, 0.99518472667219693f};
  static constexpr float s[64] = {0.0f, 0.098017140329560604f, 0.19509032201612825f, 0.29028467725446233f, 0.38268343236508978f, 0.47139673682599764f, 0.55557023301960218f, 0.63439328416364549f, 0.70710678118654746f, 0.77301045336273699f, 0.83146961230254524f, 0.88192126434835494f, 0.92387953251128674f, 0.95694033573220894f, 0.98078528040323043f, 0.99518472667219682f, 1.0f, 0.99518472667219693f, 0.98078528040323043f, 0.95694033573220894f, 0.92387953251128674f, 0.88192126434835505f, 0.83146961230254546f, 0.7730104533627371f, 0.70710678118654757f, 0.63439328416364549f, 0.55557023301960218f, 0.47139673682599786f, 0.38268343236508989f, 0.29028467725446239f, 0.19509032201612861f, 0.098017140329560826f, 0.0f, -0.09801714032956059f, -0.19509032201612836f, -0.29028467725446211f, -0.38268343236508967f, -0.47139673682599764f, -0.55557023301960196f, -0.63439328416364527f, -0.70710678118654746f, -0.77301045336273666f, -0.83146961230254524f, -0.88192126434835494f, -0.92387953251128652f, -0.95694033573220882f, -0.98078528040323032f, -0.99518472667219693f, -1.0f, -0.99518472667219693f, -0.98078528040323043f, -0.95694033573220894f, -0.92387953251128663f, -0.88192126434835505f, -0.83146961230254546f, -0.77301045336273688f, -0.70710678118654768f, -0.63439328416364593f, -0.55557023301960218f, -0.47139673682599792f, -0.38268343236509039f, -0.2902846772544625f, -0.19509032201612872f, -0.098017140329560506f};
};

// v * W_R^E with compile-time R | 64 and E (forward sign unless INV)
template <int R, int E, bool INV>
__device__ __forceinline__ float2 twc(float2 v) {
  constexpr int e = ((E % R) + R) % R;
  if constexpr (e == 0) {
    return v;
  } else if constexpr (2 * e == R) {
    return make_float2(-v.x, -v.y);
  } else if constexpr (4 * e == R) {
    return mul_q1<INV>(v);
  } else if constexpr (4 * e == 3 * R) {
    return mul_q1<!INV>(v);
  } else if constexpr (8 * e == R || 8 * e == 3 * R || 8 * e == 5 * R || 8 * e == 7 * R) {
    // odd multiples of pi/4: (+-1 +- i)/sqrt2 -> 2 adds + 2 muls
    constexpr int k = e * (64 / R);
    constexpr float c = Trig64::c[k];
    constexpr float s = INV ? Trig64::s[k] : -Trig64::s[k];
    // (x + iy)(c + is) with |c| = |s| = 1/sqrt2
    constexpr float h = 0.70710678118654752f;
    constexpr float sc = c > 0 ? 1.0f : -1.0f;
    constexpr float ss = s > 0 ? 1.0f : -1.0f;
    return make_float2((sc * v.x - ss * v.y) * h, (ss * v.x + sc * v.y) * h);
  } else {
    constexpr int k = e * (64 / R);
    constexpr float c = Trig64::c[k];
    constexpr float s = INV ? Trig64::s[k] : -Trig64::s[k];
    return make_float2(fmaf(v.x, c, -v.y * s), fmaf(v.x, s, v.y * c));
  }
}

template <bool INV>
__device__ __forceinline__ void dft2(float2& a, float2& b) {
  float2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(float2& x0, float2& x1, float2& x2, float2& x3) {
  float2 a = cadd(x0, x2), b = csub(x0, x2), c = cadd(x1, x3), d = mul_q1<INV>(csub(x1, x3));
  x0 = cadd(a, c);
  x2 = csub(a, c);
  x1 = cadd(b, d);
  x3 = csub(b, d);
}

// In-register DFT of size R in natural order: v[k] <- sum_j v[j] W_R^{jk}.
template <int R, bool INV>
struct Dft;

template <bool INV>
struct Dft<1, INV> {
  __device__ __forceinline__ static void run(float2*) {}
};
template <bool INV>
struct Dft<2, INV> {
  __device__ __forceinline__ static void run(float2* v) { dft2<INV>(v[0], v[1]); }
};
template <bool INV>
struct Dft<4, INV> {
  __device__ __forceinline__ static void run(float2* v) { dft4<INV>(v[0], v[1], v[2], v[3]); }
};
// R = 4*B: n = B*n1 + n2 ; k = k1 + 4*k2
template <int R, bool INV>
struct Dft {
  static constexpr int B = R / 4;
  __device__ __forceinline__ static void run(float2* v) {
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) dft4<INV>(v[n2], v[B + n2], v[2 * B + n2], v[3 * B + n2]);
    // now v[B*k1 + n2] = Y[n2][k1]; twiddle by W_R^{n2*k1}
    twiddle_all(v);
    float2 o[R];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      float2 w[B];
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) w[n2] = v[B * k1 + n2];
      Dft<B, INV>::run(w);
#pragma unroll
      for (int k2 = 0; k2 < B; ++k2) o[k1 + 4 * k2] = w[k2];
    }
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = o[k];
  }
  template <int I = 0>
  __device__ __forceinline__ static void twiddle_all(float2* v) {
    if constexpr (I < R) {
      constexpr int k1 = I / B, n2 = I % B;
      v[I] = twc<R, n2 * k1, INV>(v[I]);
      twiddle_all<I + 1>(v);
    }
  }
};

// In-register DFT of size R whose inputs v[R/2 .. R-1] are zero (a
// zero-padded first pass): the first radix-4 layer of R = 4B sees (x0, x1,
// 0, 0) and costs 8 instead of 16 adds per butterfly.  Spelled out because
// IEEE signed zeros forbid the compiler from folding x + 0 to x.
template <int R, bool INV>
struct DftHalf {
  static constexpr int B = R / 4;
  __device__ __forceinline__ static void run(float2* v) {
    if constexpr (R < 4) {
      Dft<R, INV>::run(v);  // R = 2: (x0, 0) -> (x0, x0); R = 1: nothing
    } else if constexpr (R == 4) {
      const float2 x0 = v[0], x1 = v[1], d = mul_q1<INV>(x1);
      v[0] = cadd(x0, x1);
      v[1] = cadd(x0, d);
      v[2] = csub(x0, x1);
      v[3] = csub(x0, d);
    } else {
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) {
        const float2 x0 = v[n2], x1 = v[B + n2];
        const float2 d = mul_q1<INV>(x1);
        v[n2] = cadd(x0, x1);
        v[B + n2] = cadd(x0, d);
        v[2 * B + n2] = csub(x0, x1);
        v[3 * B + n2] = csub(x0, d);
      }
      Dft<R, INV>::twiddle_all(v);
      float2 o[R];
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) {
        float2 w[B];
#pragma unroll
        for (int n2 = 0; n2 < B; ++n2) w[n2] = v[B * k1 + n2];
        Dft<B, INV>::run(w);
#pragma unroll
        for (int k2 = 0; k2 < B; ++k2) o[k1 + 4 * k2] = w[k2];
      }
#pragma unroll
      for (int k = 0; k < R; ++k) v[k] = o[k];
    }
  }
};

__device__ __forceinline__ int spad(int i) { return i + (i >> 4); }
// padding of the exchange buffer: one element per PB (16, or the radix when
// it is larger), conflict-free for the strided Stockham stores
template <int PB>
__device__ __forceinline__ int spadb(int i) { return i + i / PB; }
// spad(i + c) for a compile-time c that is a multiple of 16: spad(i) + 17 c / 16
// (lets every buffer access share one per-thread base + an immediate offset)
template <int C>
__device__ __forceinline__ int spad_add(int sp_i) {
  static_assert(C % 16 == 0, "offset must be a multiple of 16");
  return sp_i + C + C / 16;
}

// --- bulk async copy (TMA 1D: cp.async.bulk) with mbarrier completion -------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// arrive (count 1) and announce `bytes` of transaction to come
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// orders this CTA's earlier generic-proxy shared-memory accesses (made
// visible to this thread by a barrier) before its later async-proxy ones
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// global -> shared bulk copy; dst/src 16-byte aligned, bytes % 16 == 0
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__host__ __device__ constexpr int default_rpt(int n) { return n < 16 ? n : 16; }

// RPT_ points per thread (a power of two <= 16; default 16): full radix-RPT_
// passes, then one remainder pass
template <int N, int RPT_ = default_rpt(N)>
struct FftShape {
  static_assert((N & (N - 1)) == 0 && N >= 2, "power of two");
  static_assert((RPT_ & (RPT_ - 1)) == 0 && RPT_ >= 2 && (RPT_ <= 16 || RPT_ == 64) && RPT_ <= N,
                "points per thread");
  static constexpr int RPT = RPT_;             // points per thread
  static constexpr int TPF = N / RPT;          // threads per transform
  static constexpr int P = ilog2(N);
  static constexpr int LR = ilog2(RPT);
  static constexpr int NFULL = P / LR;                              // radix-RPT passes
  static constexpr int REM = 1 << (P % LR);                         // remainder radix (last)
  static constexpr int NPASS = NFULL + (REM > 1 ? 1 : 0);
  static constexpr int PB = RPT > 16 ? RPT : 16;                    // exchange-buffer pad block
  static constexpr int SMEM = NPASS > 1 ? N + N / PB : 0;          // float2 elements
  __host__ __device__ static constexpr int radix(int p) { return p < NFULL ? RPT : REM; }
  __host__ __device__ static constexpr int ns(int p) { return p == 0 ? 1 : ns(p - 1) * radix(p - 1); }
};

// Barrier policies for the passes: the whole CTA, or one named barrier per
// group of threads that owns its own transform (several independent
// transforms in one CTA, decoupled from each other).
struct CtaSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
struct GroupSync {
  int id, count;  // bar.sync id (1..15; 0 is __syncthreads), threads in the group
  __device__ __forceinline__ void operator()() const {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
  }
};

// Offset of pass PASS's entries in a per-pass twiddle table (fft_mod):
// passes 1.. hold ns(p) entries each.
template <class S>
__host__ __device__ constexpr int mod_offset(int p) { return p <= 1 ? 0 : mod_offset<S>(p - 1) + S::ns(p - 1); }

// One Stockham pass.  tw[j] = exp(-2 pi i j / N) for j < N (fp32).  MOD:
// pass p >= 1 takes its twiddle base from twm[mod_offset(p) + k] instead
// (tables with a per-pass rotation folded in, see fft_mod).
template <int N, int PASS, bool INV, class Sync = CtaSync, int RP = default_rpt(N), bool MOD = false,
          bool HALF = false>
__device__ __forceinline__ void fft_pass(float2 (&v)[FftShape<N, RP>::RPT], float2* buf, int t, bool active,
                                         const float2* __restrict__ tw, Sync sync = Sync(),
                                         const float2* __restrict__ twm = nullptr) {
  using S = FftShape<N, RP>;
  constexpr int R = S::radix(PASS);
  constexpr int NS = S::ns(PASS);
  constexpr int NB = N / R;
  constexpr int PER = S::RPT / R;
  constexpr bool FIRST = PASS == 0;
  constexpr bool LAST = PASS == S::NPASS - 1;
  float2 x[PER][R];
  // loads t + b TPF + m NB: one padded base per thread when TPF and NB are
  // multiples of 16 (N >= 256), else the padding per element
  constexpr int PB = S::PB;
  constexpr bool ALIGNED = (S::TPF % PB == 0) && (NB % PB == 0);
  const int sp_t = spadb<PB>(t);
#pragma unroll
  for (int b = 0; b < PER; ++b)
#pragma unroll
    for (int m = 0; m < R; ++m) {
      if constexpr (FIRST) {
        x[b][m] = v[b + m * PER];
      } else if constexpr (ALIGNED) {
        x[b][m] = active ? buf[sp_t + (b * S::TPF + m * NB) + (b * S::TPF + m * NB) / PB] : make_float2(0.f, 0.f);
      } else {
        x[b][m] = active ? buf[spadb<PB>(t + b * S::TPF + m * NB)] : make_float2(0.f, 0.f);
      }
    }
  if constexpr (!FIRST) sync();
#pragma unroll
  for (int b = 0; b < PER; ++b) {
    const int j = t + b * S::TPF;
    const int k = j & (NS - 1);
    if constexpr (NS > 1) {
      float2 w;
      if constexpr (MOD)
        w = active ? __ldg(&twm[mod_offset<S>(PASS) + k]) : make_float2(1.f, 0.f);
      else
        w = active ? __ldg(&tw[k * (N / (NS * R))]) : make_float2(1.f, 0.f);
      if (INV) w.y = -w.y;
      // powers w^m, m < R, from w, w^2, w^3 and w^{4k} (<= 3 roundings each,
      // ~10 live registers instead of R)
      const float2 w2 = cmul(w, w);
      const float2 w3 = cmul(w2, w);
      x[b][1] = cmul(x[b][1], w);
      if constexpr (R > 2) x[b][2] = cmul(x[b][2], w2);
      if constexpr (R > 3) x[b][3] = cmul(x[b][3], w3);
      if constexpr (R > 16) {
        // 64-point passes: w^(4a) by a running product
        const float2 w4 = cmul(w2, w2);
        float2 w4k = w4;
#pragma unroll
        for (int k = 4; k < R; k += 4) {
          if (k > 4) w4k = cmul(w4k, w4);
          x[b][k] = cmul(x[b][k], w4k);
          x[b][k + 1] = cmul(x[b][k + 1], cmul(w4k, w));
          x[b][k + 2] = cmul(x[b][k + 2], cmul(w4k, w2));
          x[b][k + 3] = cmul(x[b][k + 3], cmul(w4k, w3));
        }
      } else if constexpr (R > 4) {
        float2 w4k = cmul(w2, w2);
#pragma unroll
        for (int k = 4; k < R; k += 4) {
          if (k == 8) w4k = cmul(w4k, w4k);
          if (k == 12) w4k = cmul(w4k, cmul(w2, w2));
          x[b][k] = cmul(x[b][k], w4k);
          x[b][k + 1] = cmul(x[b][k + 1], cmul(w4k, w));
          x[b][k + 2] = cmul(x[b][k + 2], cmul(w4k, w2));
          x[b][k + 3] = cmul(x[b][k + 3], cmul(w4k, w3));
        }
      }
    }
    // HALF: the upper half of the input is zero; in the first pass (NS = 1,
    // PER = 1) that is exactly x[m], m >= R/2
    if constexpr (HALF && FIRST && PER == 1 && R >= 4)
      DftHalf<R, INV>::run(x[b]);
    else
      Dft<R, INV>::run(x[b]);
    if constexpr (LAST) {
#pragma unroll
      for (int m = 0; m < R; ++m) v[b + m * PER] = x[b][m];
    } else if (active) {
      const int base = (j / NS) * NS * R + k;
      if constexpr (NS % PB == 0 || (NS == 1 && R == PB)) {
        // base + m NS never carries into the padding index beyond m NS / PB
        // (NS % PB == 0), or base is a multiple of PB and m < PB (NS == 1)
        const int sp_b = spadb<PB>(base);
#pragma unroll
        for (int m = 0; m < R; ++m) buf[sp_b + m * NS + (m * NS) / PB] = x[b][m];
      } else {
#pragma unroll
        for (int m = 0; m < R; ++m) buf[spadb<PB>(base + m * NS)] = x[b][m];
      }
    }
  }
  if constexpr (!LAST) sync();
}

template <int N, bool INV, int PASS = 0, class Sync = CtaSync, int RP = default_rpt(N), bool MOD = false,
          bool HALF = false>
__device__ __forceinline__ void fft_passes(float2 (&v)[FftShape<N, RP>::RPT], float2* buf, int t, bool active,
                                           const float2* __restrict__ tw, Sync sync = Sync(),
                                           const float2* __restrict__ twm = nullptr) {
  if constexpr (PASS < FftShape<N, RP>::NPASS) {
    // every thread runs the same instruction stream (bar.sync is .aligned:
    // no barrier may sit under a thread-divergent branch); idle threads only
    // mask their shared-memory and table traffic
    fft_pass<N, PASS, INV, Sync, RP, MOD, HALF>(v, buf, t, active, tw, sync, twm);
    fft_passes<N, INV, PASS + 1, Sync, RP, MOD, HALF>(v, buf, t, active, tw, sync, twm);
  }
}

// Full transform.  Must be called by every thread of the CTA (barriers);
// threads with !active compute on zeros and touch no memory.  On return the
// buffer may be reused only after a __syncthreads().
template <int N, bool INV, class Sync = CtaSync, int RP = default_rpt(N)>
__device__ __forceinline__ void fft(float2 (&v)[FftShape<N, RP>::RPT], float2* buf, int t, bool active,
                                    const float2* __restrict__ tw, Sync sync = Sync()) {
  fft_passes<N, INV, 0, Sync, RP>(v, buf, t, active, tw, sync);
}

// fft of a zero-padded input: v[i] = 0 for i >= RPT/2 (x[j] = 0 for j >= N/2)
template <int N, bool INV, class Sync = CtaSync, int RP = default_rpt(N)>
__device__ __forceinline__ void fft_half(float2 (&v)[FftShape<N, RP>::RPT], float2* buf, int t, bool active,
                                         const float2* __restrict__ tw, Sync sync = Sync()) {
  fft_passes<N, INV, 0, Sync, RP, false, true>(v, buf, t, active, tw, sync);
}

// Transform of a linearly modulated input without the modulation multiplies:
// computes FFT(x[j] * exp(i alpha j)) given y[j] = x[j] * exp(i alpha N/R0 m)
// in register slot m (the caller applies the per-slot constants of pass 0;
// the per-thread factor exp(i alpha t) is never formed).  Writing the element
// index e = j + m NB of pass p, the pending factor of an element read by pass
// p is exp(i alpha (e >> 4p)), geometric in m with ratio exp(i alpha
// stride_p) (stride_p = N / (ns(p) radix(p)), the pass's twiddle stride), so
// it folds into the twiddle base: twm holds, for p >= 1 and k < ns(p),
// W_N^{k stride_p} * exp(-i alpha stride_p) (forward sign; inverse passes
// conjugate it), and the last pass leaves no factor.
template <int N, bool INV, class Sync = CtaSync, int RP = default_rpt(N)>
__device__ __forceinline__ void fft_mod(float2 (&v)[FftShape<N, RP>::RPT], float2* buf, int t, bool active,
                                        const float2* __restrict__ twm, Sync sync = Sync()) {
  static_assert(RP == 16 || FftShape<N, RP>::NPASS == 1, "pending-factor algebra assumes radix-16 passes");
  fft_passes<N, INV, 0, Sync, RP, true>(v, buf, t, active, nullptr, sync, twm);
}

// cos(2 pi e / 32), e in [0, 32): a switch, so a constant e folds to an
// immediate in device code
__host__ __device__ constexpr float cos32(int e) {
  switch (e & 31) {
    case 0: return 1.0f;
    case 1: case 31: return 0.98078528040323043f;
    case 2: case 30: return 0.92387953251128674f;
    case 3: case 29: return 0.83146961230254524f;
    case 4: case 28: return 0.70710678118654752f;
    case 5: case 27: return 0.55557023301960218f;
    case 6: case 26: return 0.38268343236508977f;
    case 7: case 25: return 0.19509032201612826f;
    case 8: case 24: return 0.0f;
    case 9: case 23: return -0.19509032201612826f;
    case 10: case 22: return -0.38268343236508977f;
    case 11: case 21: return -0.55557023301960218f;
    case 12: case 20: return -0.70710678118654752f;
    case 13: case 19: return -0.83146961230254524f;
    case 14: case 18: return -0.92387953251128674f;
    case 15: case 17: return -0.98078528040323043f;
    default: return -1.0f;
  }
}

// v * exp(2 pi i e / 32) for an e that folds to a constant after unrolling
// (quarter turns and odd eighths take the cheap forms)
__device__ __forceinline__ float2 mul_e32(float2 v, int e) {
  e &= 31;
  if (e == 0) return v;
  if (e == 8) return make_float2(-v.y, v.x);
  if (e == 16) return make_float2(-v.x, -v.y);
  if (e == 24) return make_float2(v.y, -v.x);
  const float c = cos32(e), s = cos32(e + 24);  // sin(x) = cos(x - pi/2)
  if ((e & 7) == 4) {
    const float h = 0.70710678118654752f;
    const float sc = c > 0.f ? h : -h, ss = s > 0.f ? h : -h;
    return make_float2(sc * v.x - ss * v.y, ss * v.x + sc * v.y);
  }
  return make_float2(fmaf(v.x, c, -v.y * s), fmaf(v.x, s, v.y * c));
}

}  // namespace tb
