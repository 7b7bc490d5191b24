// DFMA dependent-issue latency and per-scheduler throughput vs ILP on one SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 dfma_lat.cu -o dfma_lat
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void chain(double* out, long long* cyc, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = threadIdx.x + k;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < ILP; ++k) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int ILP>
void run(int warps) {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 20);
    cudaMalloc(&cyc, 1024);
    const int iters = 4096;
    chain<ILP><<<1, 32 * warps>>>(out, cyc, iters, 0.999999, 1e-9);
    chain<ILP><<<1, 32 * warps>>>(out, cyc, iters, 0.999999, 1e-9);
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double per = double(c) / (iters * ILP);
    // warps per scheduler = warps/4; pipe time per warp-DFMA = 2 cycles at 16 lanes/SMSP
    printf("ILP %2d warps %2d: %.2f cycles per warp-DFMA per warp; SMSP pipe utilisation %.0f%%\n", ILP, warps,
           per, 100.0 * 2.0 * (warps / 4.0 > 1 ? warps / 4.0 : 1) / per);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<1>(1);
    run<1>(4);
    run<2>(4);
    run<4>(4);
    run<8>(4);
    run<1>(16);
    run<2>(16);
    run<4>(16);
    run<2>(8);
    run<4>(8);
    run<8>(8);
    return 0;
}
