// Segment-loop microbenchmark: plain vs software-pipelined vs straight-line SRL-type tasks.
#include <cstdio>
#include <cuda_runtime.h>
#define NT 64
__constant__ int kRi[NT * 4];
__constant__ double kRd[NT * 2];
#define LD(o) (*(const double*)(Sb + (o)))
#define ST(o, v) (*(double*)(Sb + (o)) = (v))
__global__ void plain(double* out, int nsteps) {
  extern __shared__ double sm[]; char* Sb = (char*)(sm + (threadIdx.x & 31));
  for (int k = 0; k < 256; ++k) sm[k * 32 + (threadIdx.x & 31)] = 0.001 * k;
  long long t0 = clock64();
  for (int it = 0; it < nsteps; ++it) {
    #pragma unroll 1
    for (int q = 0; q < NT; ++q) {
      const int* r = kRi + q * 4; const double* d = kRd + q * 2;
      const double vs = LD(r[1]) - LD(r[0]);
      ST(r[3], d[1] * LD(r[2]) + d[0] * vs);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / nsteps / NT;
  out[1 + threadIdx.x] = sm[threadIdx.x];
}
__global__ void piped(double* out, int nsteps) {
  extern __shared__ double sm[]; char* Sb = (char*)(sm + (threadIdx.x & 31));
  for (int k = 0; k < 256; ++k) sm[k * 32 + (threadIdx.x & 31)] = 0.001 * k;
  long long t0 = clock64();
  for (int it = 0; it < nsteps; ++it) {
    double a = LD(kRi[1]), b = LD(kRi[0]), c = LD(kRi[2]);
    #pragma unroll 1
    for (int q = 0; q < NT - 1; ++q) {
      const int* r = kRi + q * 4; const double* d = kRd + q * 2; const int* rn = r + 4;
      const double an = LD(rn[1]), bn = LD(rn[0]), cn = LD(rn[2]);
      const double vs = a - b;
      ST(r[3], d[1] * c + d[0] * vs);
      a = an; b = bn; c = cn;
    }
    { const int* r = kRi + (NT - 1) * 4; const double* d = kRd + (NT - 1) * 2; ST(r[3], d[1] * c + d[0] * (a - b)); }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / nsteps / NT;
  out[1 + threadIdx.x] = sm[threadIdx.x];
}
__global__ void piped2(double* out, int nsteps) {  // two tasks ahead
  extern __shared__ double sm[]; char* Sb = (char*)(sm + (threadIdx.x & 31));
  for (int k = 0; k < 256; ++k) sm[k * 32 + (threadIdx.x & 31)] = 0.001 * k;
  long long t0 = clock64();
  for (int it = 0; it < nsteps; ++it) {
    double a = LD(kRi[1]), b = LD(kRi[0]), c = LD(kRi[2]);
    double a1 = LD(kRi[5]), b1 = LD(kRi[4]), c1 = LD(kRi[6]);
    #pragma unroll 1
    for (int q = 0; q < NT - 2; ++q) {
      const int* r = kRi + q * 4; const double* d = kRd + q * 2; const int* rn = r + 8;
      const double an = LD(rn[1]), bn = LD(rn[0]), cn = LD(rn[2]);
      ST(r[3], d[1] * c + d[0] * (a - b));
      a = a1; b = b1; c = c1; a1 = an; b1 = bn; c1 = cn;
    }
    { const int* r = kRi + (NT - 2) * 4; const double* d = kRd + (NT - 2) * 2; ST(r[3], d[1] * c + d[0] * (a - b)); }
    { const int* r = kRi + (NT - 1) * 4; const double* d = kRd + (NT - 1) * 2; ST(r[3], d[1] * c1 + d[0] * (a1 - b1)); }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / nsteps / NT;
  out[1 + threadIdx.x] = sm[threadIdx.x];
}
int main() {
  int hr[NT * 4]; double hd[NT * 2];
  for (int q = 0; q < NT; ++q) { hr[4*q] = ((q*3)%120)*256; hr[4*q+1] = ((q*5+1)%120)*256; hr[4*q+2] = ((q*7+2)%120)*256; hr[4*q+3] = (128 + q)*256; hd[2*q] = 0.5; hd[2*q+1] = 0.25; }
  cudaMemcpyToSymbol(kRi, hr, sizeof hr); cudaMemcpyToSymbol(kRd, hd, sizeof hd);
  double* d; cudaMalloc(&d, 4096 * 8); double h[2];
  cudaFuncSetAttribute(plain, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(piped, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(piped2, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int w : {32, 64, 128, 256}) {
    plain<<<1, w, 256 * 32 * 8>>>(d, 1000); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost); printf("threads %d plain %.1f cyc/task", w, h[0]);
    piped<<<1, w, 256 * 32 * 8>>>(d, 1000); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost); printf("  piped %.1f", h[0]);
    piped2<<<1, w, 256 * 32 * 8>>>(d, 1000); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost); printf("  piped2 %.1f\n", h[0]);
  }
  return 0;
}
