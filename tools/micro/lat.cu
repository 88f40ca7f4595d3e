// Microbenchmarks: FP64 dependent latency, LDS->DADD->STS chain, barrier cost (B200 calibration)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dadd_chain(double* out, int n, double a) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + a; x = x + a; x = x + a; x = x + a; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) out[1000] = (double)(t1 - t0) / (4.0 * n);
}
__global__ void dmul_chain(double* out, int n, double a) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x * a; x = x * a; x = x * a; x = x * a; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) out[1001] = (double)(t1 - t0) / (4.0 * n);
}
__global__ void ddiv_chain(double* out, int n, double a) {
  double x = out[threadIdx.x] + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x / a; x = x / a; x = x / a; x = x / a; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) out[1002] = (double)(t1 - t0) / (4.0 * n);
}
__global__ void lds_chain(double* out, int n) {
  __shared__ double s[32 * 64];
  double* S = s + (threadIdx.x & 31);
  for (int k = 0; k < 64; ++k) S[k * 32] = k;
  __syncwarp();
  int o = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { double v = S[o * 32]; S[((o + 1) & 63) * 32] = v + 1.0; o = (o + 1) & 63; }
  long long t1 = clock64();
  out[threadIdx.x] = S[0]; if (threadIdx.x == 0) out[1003] = (double)(t1 - t0) / n;
}
__global__ void bar_cost(double* out, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[1004 + (blockDim.x / 128)] = (double)(t1 - t0) / n;
}
__constant__ double kc[64];
__global__ void task_chain(double* out, int n) {  // SRL-like task, dependent through smem
  __shared__ double s[32 * 64];
  double* S = s + (threadIdx.x & 31);
  for (int k = 0; k < 64; ++k) S[k * 32] = 0.001 * k;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const int a = (i * 3) & 63, b = (i * 5 + 1) & 63, c = (i * 7 + 2) & 63, h = (i * 11 + 3) & 63;
    const double vs = S[b * 32] - S[a * 32];
    S[h * 32] = kc[1] * S[c * 32] + kc[0] * vs;
  }
  long long t1 = clock64();
  out[threadIdx.x] = S[0]; if (threadIdx.x == 0) out[1010] = (double)(t1 - t0) / n;
}
int main() {
  double* d; cudaMalloc(&d, 2048 * 8); cudaMemset(d, 0, 2048 * 8);
  double h0[64]; for (int i = 0; i < 64; ++i) h0[i] = 0.5 + i; cudaMemcpyToSymbol(kc, h0, sizeof h0);
  for (int rep = 0; rep < 2; ++rep) {
    dadd_chain<<<1, 32>>>(d, 10000, 1.0000001);
    dmul_chain<<<1, 32>>>(d, 10000, 1.0000001);
    ddiv_chain<<<1, 32>>>(d, 10000, 1.0000001);
    lds_chain<<<1, 32>>>(d, 10000);
    bar_cost<<<1, 128>>>(d, 10000);
    bar_cost<<<1, 256>>>(d, 10000);
    bar_cost<<<1, 512>>>(d, 10000);
    task_chain<<<1, 32>>>(d, 10000);
  }
  double h[2048]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("DADD dep latency %.1f cyc\nDMUL dep %.1f\nDDIV dep %.1f\nLDS->DADD->STS chain %.1f\nbar 4w %.1f 8w %.1f 16w %.1f\nSRL task chain %.1f\n",
         h[1000], h[1001], h[1002], h[1003], h[1005], h[1006], h[1008], h[1010]);
  return 0;
}
