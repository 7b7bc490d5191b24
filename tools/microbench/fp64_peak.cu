// FP64 roofs on the B200: DFMA (CUDA-core FP64 pipe), DMMA (mma.sync
// m8n8k4 f64 on the tensor cores) and both interleaved in the same warps.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu -o fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
    double a[8], b = 1.0000001, c = 1e-9;
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.0) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b, const double (&c)[2]) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
                 : "=d"(d[0]), "=d"(d[1])
                 : "d"(a), "d"(b), "d"(c[0]), "d"(c[1]));
}

__global__ void dmma_kernel(double* out, int iters) {
    double acc[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = threadIdx.x;
    double a = 1.0000001, b = 0.999999;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) dmma(acc[k], a, b, acc[k]);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s += acc[k][0] + acc[k][1];
    if (s == 12345.0) out[threadIdx.x] = s;
}

__global__ void both_kernel(double* out, int iters) {
    double acc[4][2];
    double x[8], bb = 1.0000001, cc = 1e-9;
#pragma unroll
    for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    double a = 1.0000001, b = 0.999999;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 4; ++k) dmma(acc[k], a, b, acc[k]);
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], bb, cc);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) s += acc[k][0] + acc[k][1];
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 20);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int blocks = sms * 8, threads = 256, iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8 * iters * double(blocks) * threads;
        printf("dfma: %.3f ms  %.2f TFLOP/s\n", ms, fl / ms / 1e9);
        cudaEventRecord(e0);
        dmma_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double fl2 = 2.0 * 8 * 8 * 4 * 4 * iters * double(blocks) * (threads / 32);
        printf("dmma: %.3f ms  %.2f TFLOP/s\n", ms, fl2 / ms / 1e9);
        cudaEventRecord(e0);
        both_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("both: %.3f ms  %.2f TFLOP/s combined (dfma part %.2f + dmma part %.2f)\n", ms, (fl + fl2) / ms / 1e9,
               fl / ms / 1e9, fl2 / ms / 1e9);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
