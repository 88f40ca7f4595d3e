// Where do the CTAs of a 32-CTA, 221 KB-shared-memory launch land? (placement study)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int* out) {
    extern __shared__ double sm[];
    unsigned smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (threadIdx.x == 0) { sm[0] = smid; out[blockIdx.x] = (int)smid; }
}
int main() {
    int* d; cudaMalloc(&d, 256 * sizeof(int));
    const int smem = 221184;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int grid : {32, 128}) {
        probe<<<grid, 256, smem>>>(d);
        int h[256]; cudaMemcpy(h, d, grid * sizeof(int), cudaMemcpyDeviceToHost);
        printf("grid %d smids:", grid);
        for (int i = 0; i < grid; ++i) printf(" %d", h[i]);
        printf("\n");
    }
    return 0;
}
