// Microbenchmark: texture return path cost of the K2 gather forms.
//  (a) 2 x TLD4 (re, im channels) on a float2 pitch-2D texture (the shipped K2)
//  (b) 2 x point tex2D<float4> on a float4 texture holding (P[r], P[r+1]) per texel
//      (a "pair-duplicated" polar layout), one fetch per angular row
// Each thread walks a column-like curve of polar coordinates (as K2's nodes do).
// usage: tex_fetch  -> prints ms per variant
#include <cstdio>
#include <cuda_runtime.h>
#include <cmath>

__global__ void k_tld4(cudaTextureObject_t tex, float* out, int H, int V, int iters) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const float a = (float)(blockIdx.x % 2048);
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
    const float b = (float)((t % 256) + 256 * (i % 8));
    const float r = sqrtf(a * a + b * b), th = atan2f(b, a) * (V / 3.14159265f);
    const float x = fminf(floorf(r), (float)(H - 2)) + 1.f, y = floorf(th) + 1.f;
    const float4 re = tex2Dgather<float4>(tex, x, y, 0);
    const float4 im = tex2Dgather<float4>(tex, x, y, 1);
    acc += re.x + re.y + re.z + re.w + im.x + im.y + im.z + im.w;
  }
  out[t] = acc;
}

__global__ void k_pt4(cudaTextureObject_t tex4, float* out, int H, int V, int iters) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const float a = (float)(blockIdx.x % 2048);
  float acc = 0.f;
  for (int i = 0; i < iters; ++i) {
    const float b = (float)((t % 256) + 256 * (i % 8));
    const float r = sqrtf(a * a + b * b), th = atan2f(b, a) * (V / 3.14159265f);
    const float x = fminf(floorf(r), (float)(H - 2)) + 0.5f, y = floorf(th) + 0.5f;
    const float4 p0 = tex2D<float4>(tex4, x, y);
    const float4 p1 = tex2D<float4>(tex4, x, y + 1.f);
    acc += p0.x + p0.y + p0.z + p0.w + p1.x + p1.y + p1.z + p1.w;
  }
  out[t] = acc;
}

int main() {
  const int H = 2048, V = 2048, rows = 31 * (V + 1);
  float2* d2; float4* d4; float* out;
  cudaMalloc(&d2, (size_t)rows * H * sizeof(float2));
  cudaMalloc(&d4, (size_t)rows * H * sizeof(float4));
  cudaMemset(d2, 0, (size_t)rows * H * sizeof(float2));
  cudaMemset(d4, 0, (size_t)rows * H * sizeof(float4));
  const int blocks = 148 * 5 * 40, threads = 256, iters = 64;
  cudaMalloc(&out, (size_t)blocks * threads * sizeof(float));
  auto mk = [&](void* ptr, cudaChannelFormatDesc cd, size_t pitch, int rowsv) {
    cudaResourceDesc res{}; res.resType = cudaResourceTypePitch2D; res.res.pitch2D.devPtr = ptr;
    res.res.pitch2D.desc = cd; res.res.pitch2D.width = H; res.res.pitch2D.height = rowsv;
    res.res.pitch2D.pitchInBytes = pitch;
    cudaTextureDesc td{}; td.addressMode[0] = cudaAddressModeBorder; td.addressMode[1] = cudaAddressModeClamp;
    td.filterMode = cudaFilterModePoint; td.readMode = cudaReadModeElementType;
    cudaTextureObject_t o = 0; cudaCreateTextureObject(&o, &res, &td, nullptr); return o;
  };
  cudaTextureObject_t t2 = mk(d2, cudaCreateChannelDesc<float2>(), H * sizeof(float2), rows);
  cudaTextureObject_t t4 = mk(d4, cudaCreateChannelDesc<float4>(), H * sizeof(float4), rows);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    float ms;
    cudaEventRecord(e0); k_tld4<<<blocks, threads>>>(t2, out, H, V, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("tld4x2 (float2 texture)     %.3f ms\n", ms);
    cudaEventRecord(e0); k_pt4<<<blocks, threads>>>(t4, out, H, V, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("point float4 x2 (pair texels) %.3f ms\n", ms);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
