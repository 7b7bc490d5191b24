// DFMA throughput with constant-table operands (LDCU + DFMA R, R, UR, R)
// vs register operands, and a matrix-vector contraction shaped like the
// element kernel's trace phase.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 dfma_const.cu
#include <cstdio>
#include <cuda_runtime.h>

__constant__ double TABLE[256];

template <int NCH>
__global__ void dfma_reg(double* out, int iters) {
    double a[NCH], b = 1.0000001, c = 1e-9;
#pragma unroll
    for (int k = 0; k < NCH; ++k) a[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < NCH; ++k) a[k] = fma(a[k], b, c);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < NCH; ++k) s += a[k];
    if (s == 12345.0) out[threadIdx.x] = s;
}

// y[q] = sum_i T[q][i] x[i] for 14 x 10, table from constant memory, the
// outputs fed back as inputs (like repeated trace evaluations)
__global__ void matvec_const(double* out, int iters) {
    double x[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) x[k] = threadIdx.x * 1e-3 + k;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        double y[14];
#pragma unroll
        for (int q = 0; q < 14; ++q) {
            double u = 0;
#pragma unroll
            for (int i = 0; i < 10; ++i) u = fma(TABLE[q * 10 + i], x[i], u);
            y[q] = u;
        }
#pragma unroll
        for (int k = 0; k < 10; ++k) x[k] = y[k] * 1e-3 + y[k + 4];
        acc += y[13];
    }
    if (acc == 12345.0) out[threadIdx.x] = acc;
}

// same with the table in registers (loaded once)
__global__ void matvec_reg(double* out, int iters) {
    double x[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) x[k] = threadIdx.x * 1e-3 + k;
    double t[20];
#pragma unroll
    for (int k = 0; k < 20; ++k) t[k] = TABLE[k] + threadIdx.x * 1e-12;
    double acc = 0;
    for (int it = 0; it < iters; ++it) {
        double y[14];
#pragma unroll
        for (int q = 0; q < 14; ++q) {
            double u = 0;
#pragma unroll
            for (int i = 0; i < 10; ++i) u = fma(t[(q * 10 + i) % 20], x[i], u);
            y[q] = u;
        }
#pragma unroll
        for (int k = 0; k < 10; ++k) x[k] = y[k] * 1e-3 + y[k + 4];
        acc += y[13];
    }
    if (acc == 12345.0) out[threadIdx.x] = acc;
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 20);
    double h[256];
    for (int i = 0; i < 256; ++i) h[i] = 1e-3 * (i % 17) - 0.007;
    cudaMemcpyToSymbol(TABLE, h, sizeof(h));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    const int iters = 4000;
    for (int warps = 4; warps <= 32; warps *= 2) {
        const int threads = 128, blocks = sms * warps / 4;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            dfma_reg<8><<<blocks, threads>>>(out, iters * 10);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            double f1 = 2.0 * 8 * iters * 10.0 * blocks * threads / (ms * 1e-3) / 1e12;
            cudaEventRecord(e0);
            matvec_const<<<blocks, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            double f2 = 2.0 * (140 + 20) * iters * double(blocks) * threads / (ms * 1e-3) / 1e12;
            cudaEventRecord(e0);
            matvec_reg<<<blocks, threads>>>(out, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            double f3 = 2.0 * (140 + 20) * iters * double(blocks) * threads / (ms * 1e-3) / 1e12;
            if (rep) printf("warps/SM %2d: dfma_reg %.1f  matvec_const %.1f  matvec_reg %.1f TFLOP/s\n", warps, f1, f2, f3);
        }
    }
    return 0;
}
