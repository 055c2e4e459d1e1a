// Microbenchmark: fixed-order sum of per-CTA gradient partials [ncta][P]
// (the k_train_adam reduction) -- scalar rows of 32 params per 256-thread
// block vs float2 / float4 rows, partials freshly written with streaming
// stores (as the training kernel's flush leaves them).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o reduce reduce.cu && ./reduce
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_fill(float* p, size_t n, float s) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, s * (float)(i & 1023));
}

// V: params per lane (1, 2, 4); block = 8 warps, 32 * V params
template <int V, int INFL>
__global__ void __launch_bounds__(256) k_red(const float* __restrict__ part, int ncta, long long P,
                                             float* __restrict__ out) {
  __shared__ float s[8][32 * V];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const long long q = (long long)blockIdx.x * 32 * V + (long long)l * V;
  float g0[V], g1[V];
#pragma unroll
  for (int j = 0; j < V; ++j) g0[j] = g1[j] = 0.f;
  if (q < P) {
    int c = w;
    for (; c + 8 * (INFL - 1) < ncta; c += 8 * INFL) {
      float v[INFL][V];
#pragma unroll
      for (int i = 0; i < INFL; ++i) {
        const float* src = part + (size_t)(c + 8 * i) * P + q;
        if constexpr (V == 4) {
          const float4 t = *reinterpret_cast<const float4*>(src);
          v[i][0] = t.x; v[i][1] = t.y; v[i][2] = t.z; v[i][3] = t.w;
        } else if constexpr (V == 2) {
          const float2 t = *reinterpret_cast<const float2*>(src);
          v[i][0] = t.x; v[i][1] = t.y;
        } else {
          v[i][0] = *src;
        }
      }
#pragma unroll
      for (int i = 0; i < INFL; i += 2)
#pragma unroll
        for (int j = 0; j < V; ++j) {
          g0[j] += v[i][j];
          if (i + 1 < INFL) g1[j] += v[i + 1][j];
        }
    }
    for (; c < ncta; c += 8)
#pragma unroll
      for (int j = 0; j < V; ++j) g0[j] += part[(size_t)c * P + q + j];
  }
#pragma unroll
  for (int j = 0; j < V; ++j) s[w][l * V + j] = g0[j] + g1[j];
  __syncthreads();
  for (int i = threadIdx.x; i < 32 * V; i += 256) {
    const long long qq = (long long)blockIdx.x * 32 * V + i;
    if (qq < P) out[qq] = ((s[0][i] + s[1][i]) + (s[2][i] + s[3][i])) + ((s[4][i] + s[5][i]) + (s[6][i] + s[7][i]));
  }
}

__global__ void k_read(const float4* __restrict__ p, size_t n4, float* out) {
  float a = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    const float4 t = p[i];
    a += t.x + t.y + t.z + t.w;
  }
  if (a == 1234.5f) out[0] = a;
}

template <class F>
float timeit(F f, float* part, size_t n) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9f;
  for (int r = 0; r < 6; ++r) {
    k_fill<<<1184, 256>>>(part, n, 0.5f + r);
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < best) best = ms;
  }
  return best * 1e3f;
}

int main() {
  const int ncta = 148;
  const long long P = 55200;
  const size_t n = (size_t)ncta * P;
  float *part, *out;
  cudaMalloc(&part, n * 4);
  cudaMalloc(&out, P * 4 + 64);
  printf("partials %.1f MB\n", n * 4 / 1e6);
  printf("plain float4 read   %7.2f us\n", timeit([&] { k_read<<<1184, 256>>>((const float4*)part, n / 4, out); }, part, n));
  auto grid = [&](int V) { return (int)((P + 32 * V - 1) / (32 * V)); };
  printf("V1 INFL2 (current)  %7.2f us\n", timeit([&] { k_red<1, 2><<<grid(1), 256>>>(part, ncta, P, out); }, part, n));
  printf("V1 INFL8            %7.2f us\n", timeit([&] { k_red<1, 8><<<grid(1), 256>>>(part, ncta, P, out); }, part, n));
  printf("V2 INFL4            %7.2f us\n", timeit([&] { k_red<2, 4><<<grid(2), 256>>>(part, ncta, P, out); }, part, n));
  printf("V2 INFL8            %7.2f us\n", timeit([&] { k_red<2, 8><<<grid(2), 256>>>(part, ncta, P, out); }, part, n));
  printf("V4 INFL4            %7.2f us\n", timeit([&] { k_red<4, 4><<<grid(4), 256>>>(part, ncta, P, out); }, part, n));
  printf("V4 INFL8            %7.2f us\n", timeit([&] { k_red<4, 8><<<grid(4), 256>>>(part, ncta, P, out); }, part, n));
  printf("V4 INFL2            %7.2f us\n", timeit([&] { k_red<4, 2><<<grid(4), 256>>>(part, ncta, P, out); }, part, n));
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
