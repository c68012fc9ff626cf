// mb_lds.cu -- diagnostic microbenchmark (not product code): throughput of
// dependent shared-memory table-lookup chains, the inner loop of the SFA scan
// without any text traffic.  A bank-private u16 table (lane L's copy in bank
// L) is walked by K independent chains per thread; per step the "byte" comes
// from a register word (PRMT), is clamped to a column (VIADDMNMX) and turned
// into the next address (IMAD), as in k_scan_tma.  Prints lookups/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mb_lds scripts/mb_lds.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

extern __shared__ __align__(1024) uint8_t dsm[];

__device__ __forceinline__ uint32_t lds16(uint32_t off) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(dsm)) + off));
    return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t off) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(dsm)) + off));
    return v;
}

template <int MODE>
__device__ __forceinline__ uint32_t step(uint32_t st, uint32_t w, int k, uint32_t X) {
    uint32_t b;
    if (MODE == 0) {  // PRMT + VIADDMNMX + IMAD + LDS.U16 (the product's step)
        asm("prmt.b32 %0, %1, 0, %2;" : "=r"(b) : "r"(w), "r"(0x4440 | k));
        b = __viaddmin_u32(b, 0u - 48u, 10u);
        return lds16(b * X + st);
    } else if (MODE == 1) {  // IDP4A + LDS.U16 (byte * 128 + st), no clamp
        b = __dp4a(w, 0x80u << (8 * k), st);
        return lds16(b);
    } else if (MODE == 2) {  // IMAD + LDS.U16 only (column from a fixed register)
        return lds16((w & 3) * X + st);
    } else {  // PRMT + VIADDMNMX + IMAD + LDS.U32
        asm("prmt.b32 %0, %1, 0, %2;" : "=r"(b) : "r"(w), "r"(0x4440 | k));
        b = __viaddmin_u32(b, 0u - 48u, 10u);
        return lds32(b * X + (st & ~3u)) & 0xffffu;
    }
}

template <int MODE, int K>
__global__ void __launch_bounds__(1024, 1) k_lds(int iters, uint32_t X, uint32_t tbytes, uint32_t* out) {
    const uint32_t lane = threadIdx.x & 31;
    // table: every cell of lane L's copy points to a pseudo-random state in bank L
    for (uint32_t i = threadIdx.x; i < tbytes / 4; i += blockDim.x) {
        const uint32_t L = i & 31, h = (i * 2654435761u) >> 7;
        const uint32_t row = X / 128, s0 = h % row, s1 = (h >> 11) % row;
        reinterpret_cast<uint32_t*>(dsm)[i] = (s0 * 128 + 4 * L) | ((s1 * 128 + 4 * L + 2) << 16);
    }
    __syncthreads();
    uint32_t st[K];
#pragma unroll
    for (int k = 0; k < K; ++k) st[k] = 4 * lane + 128 * k;
    uint32_t w = 0x35343332u + threadIdx.x * 0x01000100u;  // digits
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int k = 0; k < K; ++k) st[k] = step<MODE>(st[k], w, j, X);
        w = (w << 8) | (w >> 24);
    }
    uint32_t acc = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) acc ^= st[k];
    if (acc == static_cast<uint32_t>(iters) + 7u) out[0] = acc;  // runtime-opaque: keeps the chains live
}

template <int MODE, int K>
void run(int threads, uint32_t* out) {
    const uint32_t X = 128 * 55, tbytes = 11 * X;  // cfg2's private table: 11 columns x 55 state pairs
    const int iters = 4096;
    cudaFuncSetAttribute(k_lds<MODE, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, tbytes + 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_lds<MODE, K><<<148, threads, tbytes + 1024>>>(iters, X, tbytes, out);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) {
        printf("mode=%d K=%d threads=%d: %s\n", MODE, K, threads, cudaGetErrorString(e));
        return;
    }
    cudaEventRecord(a);
    k_lds<MODE, K><<<148, threads, tbytes + 1024>>>(iters, X, tbytes, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double lookups = 148.0 * threads * K * iters * 4;
    const double per_clk_sm = lookups / 148 / (ms * 1e-3 * clk * 1e3);
    printf("mode=%d K=%d threads=%d: %.2f lookups/clk/SM (at %d MHz nominal), %.1f G lookups/s (%s)\n", MODE, K, threads,
           per_clk_sm, clk / 1000, lookups / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    uint32_t* out;
    cudaMalloc(&out, 4);
    run<0, 1>(1024, out);
    run<0, 2>(1024, out);
    run<0, 4>(1024, out);
    run<0, 1>(512, out);
    run<0, 2>(512, out);
    run<1, 1>(1024, out);
    run<1, 2>(1024, out);
    run<2, 1>(1024, out);
    run<2, 2>(1024, out);
    run<3, 1>(1024, out);
    run<3, 2>(1024, out);
    return 0;
}
