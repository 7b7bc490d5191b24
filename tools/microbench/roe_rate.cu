// Attainable rate of the device Roe flux (csrc/hodg_common.cuh) in isolation:
// states in registers, one or two solves in flight per thread.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 roe_rate.cu -o roe_rate
#include <cstdio>
#include "../../paper_2209_01877_b200/csrc/hodg_common.cuh"

template <int ILP>
__global__ void __launch_bounds__(128) roe_kernel(double* out, int iters) {
    double qL[ILP][5], qR[ILP][5], n[3] = {0.6, 0.64, 0.48};
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
        const double s = 1.0 + 1e-3 * (threadIdx.x + k);
        qL[k][0] = s; qL[k][1] = 0.3; qL[k][2] = 0.1; qL[k][3] = -0.2; qL[k][4] = 2.5 * s;
        qR[k][0] = 1.1 * s; qR[k][1] = 0.2; qR[k][2] = -0.1; qR[k][3] = 0.1; qR[k][4] = 2.6 * s;
    }
    double acc = 0.0;
    for (int i = 0; i < iters; ++i) {
        double f[ILP][5];
        bool ok = true;
#pragma unroll
        for (int k = 0; k < ILP; ++k) ok &= hodg::roe(qL[k], qR[k], n, 1.4, f[k]);
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            acc += f[k][0] + f[k][4];
            // every input loop-carried so nothing is hoisted
#pragma unroll
            for (int v = 0; v < 5; ++v) {
                qL[k][v] += 1e-13 * f[k][v];
                qR[k][v] -= 1e-13 * f[k][4 - v];
            }
            n[0] += 1e-14 * f[k][2];
        }
        if (!ok) acc = -1.0;
    }
    if (acc == 12345.0) out[threadIdx.x] = acc;
}

template <int ILP>
void run(double* out, int blocks_per_sm, int sms) {
    const int blocks = sms * blocks_per_sm, iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    roe_kernel<ILP><<<blocks, 128>>>(out, 10);
    cudaEventRecord(e0);
    roe_kernel<ILP><<<blocks, 128>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double solves = double(blocks) * 128 * iters * ILP;
    printf("ILP %d, %2d CTAs/SM: %.3e Roe solves/s\n", ILP, blocks_per_sm, solves / (ms * 1e-3));
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 20);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int b : {4, 8, 16}) {
        run<1>(out, b, sms);
        run<2>(out, b, sms);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
