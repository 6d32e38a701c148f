// Microbenchmark: cycles per contract() call of the register-weight engine
// (TreeLSTM level phase, H=256) for T = 1, 4, 8; and FFMA vs FFMA2 issue rate.
#include <cstdio>
#include "../../paper_2011_01383_b200/csrc/rw_engine.cuh"
using namespace cx;
using namespace cx::rw;

template <int T>
__global__ void __launch_bounds__(512, 1) k_contract(long long *out, float *sink, int iters) {
  constexpr int H = 256, KC = RShape<H>::KC;
  extern __shared__ __align__(16) float smem[];
  float *X = smem, *red = X + 8 * 2 * H, *red2 = red + 16 * 5 * 8 * 16, *cv = red2 + 5 * 8 * 16;
  for (int i = threadIdx.x; i < 8 * 2 * H; i += blockDim.x) X[i] = 0.001f * (i % 97);
  float w[4][KC];
  for (int g = 0; g < 4; g++)
    for (int j = 0; j < KC; j++) w[g][j] = 0.01f * (g + j + threadIdx.x % 7);
  RCtx c;
  c.a = nullptr; c.X = X; c.red = red; c.red2 = red2; c.cv = cv; c.bias = nullptr;
  c.tslot = -1;
  __syncthreads();
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    float s[5];
    contract<RLstmLevel<2>, H, T>(c, X, w, s);
    acc += s[0] + s[4];
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[T] = (t1 - t0) / iters;
  sink[threadIdx.x] = acc;
}

__global__ void k_ffma(long long *out, float *sink, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float b = 1.0001f, c = 0.999f;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 16; r++) {
      a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
      a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[10] = t1 - t0;
  sink[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_ffma2(long long *out, float *sink, int iters) {
  float2 a0 = make_float2(threadIdx.x, 1), a1 = make_float2(2, 3), a2 = make_float2(4, 5), a3 = make_float2(6, 7);
  const float2 b = make_float2(1.0001f, 1.0002f), c = make_float2(0.999f, 0.998f);
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int r = 0; r < 16; r++) {
      a0 = ffma2(a0, b, c); a1 = ffma2(a1, b, c); a2 = ffma2(a2, b, c); a3 = ffma2(a3, b, c);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[11] = t1 - t0;
  sink[threadIdx.x] = a0.x + a1.x + a2.x + a3.x + a0.y + a1.y + a2.y + a3.y;
}

// variants: FMA part only (MODE 1), reduction only (MODE 2)
template <int T, int MODE>
__global__ void __launch_bounds__(512, 1) k_part(long long *out, float *sink, int iters) {
  constexpr int H = 256, KC = RShape<H>::KC, NA = 5, NV = 2;
  extern __shared__ __align__(16) float smem[];
  float *X = smem, *red = X + 8 * 2 * H, *red2 = red + 16 * 5 * 8 * 16;
  for (int i = threadIdx.x; i < 8 * 2 * H; i += blockDim.x) X[i] = 0.001f * (i % 97);
  float w[4][KC];
  for (int g = 0; g < 4; g++)
    for (int j = 0; j < KC; j++) w[g][j] = 0.01f * (g + j + threadIdx.x % 7);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, u = lane & 15, ksub = lane >> 4;
  const int k0 = (warp * 2 + ksub) * KC;
  float tot = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    float acc[NA][T];
    for (int a = 0; a < NA; a++) for (int t = 0; t < T; t++) acc[a][t] = 0.f;
    if (MODE == 1) {
#pragma unroll
      for (int t = 0; t < T; t++) {
#pragma unroll
        for (int q = 0; q < KC; q += 4) {
          float4 h0 = *reinterpret_cast<const float4 *>(X + (t * NV + 0) * H + k0 + q);
          float4 h1 = *reinterpret_cast<const float4 *>(X + (t * NV + 1) * H + k0 + q);
          float hx[4] = {h0.x, h0.y, h0.z, h0.w}, hy[4] = {h1.x, h1.y, h1.z, h1.w};
#pragma unroll
          for (int e = 0; e < 4; e++) {
            float ht = hx[e] + hy[e];
            acc[0][t] = fmaf(w[0][q + e], ht, acc[0][t]);
            acc[1][t] = fmaf(w[1][q + e], ht, acc[1][t]);
            acc[2][t] = fmaf(w[2][q + e], ht, acc[2][t]);
            acc[3][t] = fmaf(w[3][q + e], hx[e], acc[3][t]);
            acc[4][t] = fmaf(w[3][q + e], hy[e], acc[4][t]);
          }
        }
      }
      for (int a = 0; a < NA; a++) for (int t = 0; t < T; t++) tot += acc[a][t];
    } else {
      for (int a = 0; a < NA; a++) for (int t = 0; t < T; t++) acc[a][t] = it + a + t;
#pragma unroll
      for (int a = 0; a < NA; a++)
#pragma unroll
        for (int t = 0; t < T; t++) acc[a][t] += __shfl_xor_sync(0xffffffffu, acc[a][t], 16);
#pragma unroll
      for (int a = 0; a < NA; a++) {
        if ((a & 1) != ksub) continue;
        float *dst = red + ((warp * NA + a) * 16 + u) * T;
#pragma unroll
        for (int t = 0; t < T; t += 4) *reinterpret_cast<float4 *>(dst + t) = make_float4(acc[a][t], acc[a][t+1], acc[a][t+2], acc[a][t+3]);
      }
      __syncthreads();
      constexpr int G = NA * 16 * T / 4, WS = NA * 16 * T;
      for (int g = threadIdx.x; g < G; g += blockDim.x) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int ww = 0; ww < 16; ww++) { float4 x = *reinterpret_cast<const float4 *>(red + ww * WS + 4 * g); v.x += x.x; v.y += x.y; v.z += x.z; v.w += x.w; }
        *reinterpret_cast<float4 *>(red2 + 4 * g) = v;
      }
      __syncthreads();
      tot += red2[(threadIdx.x & 63)];
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[12 + MODE] = (t1 - t0) / iters;
  sink[threadIdx.x] = tot;
}

int main() {
  long long *d, h[16] = {0};
  float *sink;
  cudaMalloc(&d, 16 * 8);
  cudaMalloc(&sink, 4096 * 4);
  const int smem = 4 * (8 * 2 * 256 + 16 * 5 * 8 * 16 + 5 * 8 * 16 + 8 * 4 * 16);
  cudaFuncSetAttribute(k_contract<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_contract<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_contract<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_contract<1><<<1, 512, smem>>>(d, sink, 200);
  k_contract<4><<<1, 512, smem>>>(d, sink, 200);
  k_contract<8><<<1, 512, smem>>>(d, sink, 200);
  cudaFuncSetAttribute(k_part<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_part<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_part<8, 1><<<1, 512, smem>>>(d, sink, 200);
  k_part<8, 2><<<1, 512, smem>>>(d, sink, 200);
  const int it = 1000;
  k_ffma<<<1, 512>>>(d, sink, it);   // 16 warps, 8 independent chains each
  k_ffma2<<<1, 512>>>(d, sink, it);  // same FMA count as 4 float2 chains
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d, 16 * 8, cudaMemcpyDeviceToHost);
  printf("contract<LstmLevel, H=256> cycles/call: T=1 %lld  T=4 %lld  T=8 %lld  (%s)\n", h[1], h[4], h[8], cudaGetErrorString(e));
  printf("T=8 parts: FMA only (scalar FFMA) %lld cycles, reduction only %lld cycles\n", h[13], h[14]);
  double fl = 16.0 * 8 * it * 512;  // FMAs in k_ffma (per SM)
  printf("FFMA : %.1f FMA/cycle/SM  | FFMA2: %.1f FMA/cycle/SM\n", fl / h[10], fl / h[11]);
  return 0;
}
