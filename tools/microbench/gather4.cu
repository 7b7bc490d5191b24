// TMA row gather: one cp.async.bulk per row vs cp.async.bulk.tensor tile::gather4
// (four rows of a 2-D tensor map per instruction).  Checks the gathered
// rows (and zero fill of out-of-range row indices) and times each variant
// over the same random row list, persistent CTAs of 128 threads gathering
// 64 rows per tile -- the face kernel's pattern.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather4 gather4.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
                     su32(b)),
                 "r"(ph)
                 : "memory");
}

constexpr int ROWS = 64;  // rows per tile
constexpr int THREADS = 128;

template <int MODE>  // 0: bulk copy per row; 1: gather4
__global__ void __launch_bounds__(THREADS) gather(const __grid_constant__ CUtensorMap tm, const double* src, int cols,
                                                  const int* idx, int ntiles, double* out, int check, int n) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm);
    double* rows = reinterpret_cast<double*>(sm + 128);
    const int t = threadIdx.x;
    if (t == 0) {
        bar_init(bar, THREADS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double acc = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int* ix = idx + tile * ROWS;
        if (MODE == 0) {
            if (t < ROWS) {
                bar_expect(bar, cols * 8);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        su32(rows + t * cols)),
                    "l"(src + int64_t(min(max(ix[t], 0), n - 1)) * cols), "r"(cols * 8), "r"(su32(bar))
                    : "memory");
            } else {
                bar_arrive(bar);
            }
        } else {
            if (t < ROWS / 4) {
                const int4 r = reinterpret_cast<const int4*>(ix)[t];
                bar_expect(bar, 4 * cols * 8);
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(rows + 4 * t * cols)),
                    "l"(&tm), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(su32(bar))
                    : "memory");
            } else {
                bar_arrive(bar);
            }
        }
        bar_wait(bar, it & 1);
        if (check) {
            for (int k = t; k < ROWS * cols; k += THREADS) out[int64_t(tile) * ROWS * cols + k] = rows[k];
        } else {
            for (int k = t; k < ROWS * cols; k += THREADS) acc += rows[k];
        }
        __syncthreads();
    }
    if (!check && acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
    const int n = 1000000, cols = argc > 1 ? atoi(argv[1]) : 50;
    const int ntiles = 4000000 / ROWS;
    std::vector<double> h(size_t(n) * cols);
    for (size_t k = 0; k < h.size(); ++k) h[k] = double(k % 1000003) * 0.5 + 1;
    std::vector<int> ix(size_t(ntiles) * ROWS);
    uint64_t s = 88172645463325252ull;
    for (auto& x : ix) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        x = int(s % n);
    }
    ix[5] = -1;   // out of range below
    ix[9] = n;    // out of range above
    double *src, *out;
    int* idx;
    cudaMalloc(&src, h.size() * 8);
    cudaMalloc(&idx, ix.size() * 4);
    cudaMalloc(&out, size_t(ntiles) * ROWS * cols * 8);
    cudaMemcpy(src, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(idx, ix.data(), ix.size() * 4, cudaMemcpyHostToDevice);

    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
    CUtensorMap tm;
    cuuint64_t gdim[2] = {cuuint64_t(cols), cuuint64_t(n)};
    cuuint64_t gstride[1] = {cuuint64_t(cols) * 8};
    cuuint32_t box[2] = {cuuint32_t(cols), 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, src, gdim, gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode cols=%d: %d\n", cols, int(r));
    if (r != CUDA_SUCCESS) return 1;
    const size_t smem = 128 + ROWS * cols * 8;
    cudaFuncSetAttribute(gather<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(gather<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    std::vector<double> o(size_t(ntiles) * ROWS * cols);
    for (int mode = 0; mode < 2; ++mode) {
        const int tiles_chk = 64;
        if (mode == 0) gather<0><<<sms, THREADS, smem>>>(tm, src, cols, idx, tiles_chk, out, 1, n);
        else gather<1><<<sms, THREADS, smem>>>(tm, src, cols, idx, tiles_chk, out, 1, n);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(o.data(), out, size_t(tiles_chk) * ROWS * cols * 8, cudaMemcpyDeviceToHost);
        long bad = 0, oobz = 0;
        for (int rr = 0; rr < tiles_chk * ROWS; ++rr) {
            const int row = ix[rr];
            for (int c = 0; c < cols; ++c) {
                const int rc = row < 0 ? 0 : (row >= n ? n - 1 : row);
                const double want = (mode == 1 && (row < 0 || row >= n)) ? 0.0 : h[size_t(rc) * cols + c];
                if (o[size_t(rr) * cols + c] != want) ++bad;
                if ((row < 0 || row >= n) && o[size_t(rr) * cols + c] == 0.0) ++oobz;
            }
        }
        printf("mode %d check: %ld mismatches (oob rows zero: %ld of %d; mode 0 clamps)\n", mode, bad,
               oobz, 2 * cols);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int occ = 1; occ <= 4; occ *= 2) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (mode == 0) gather<0><<<sms * occ, THREADS, smem>>>(tm, src, cols, idx, ntiles, out, 0, n);
                else gather<1><<<sms * occ, THREADS, smem>>>(tm, src, cols, idx, ntiles, out, 0, n);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep) printf("mode %d ctas/sm %d: %.3f ms, %.1f GB/s rows\n", mode, occ, ms,
                                double(ntiles) * ROWS * cols * 8 / ms / 1e6);
            }
        }
    }
    return 0;
}
