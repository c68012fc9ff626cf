// mb_tma.cu -- diagnostic microbenchmark (not product code): the TMA access
// pattern of k_scan_tma without the SFA lookups.  One CTA per SM, 31 consumer
// warps + 1 producer; the text is viewed as [rows x L] and every stage loads
// ROWB bytes of each of the CTA's R rows.  Consumers XOR the bytes (so the
// loads stay live).  Prints GB/s for a sweep of (K, ROWB, ring, promo).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mb_tma scripts/mb_tma.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t par) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok) : "r"(bar), "r"(par) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const void* tmap, uint32_t bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(tmap), "r"(bar), "r"(x), "r"(y) : "memory");
}
extern __shared__ __align__(1024) uint8_t dsm[];

template <int ROWB>
__global__ void __launch_bounds__(1024, 1)
k_mb(const __grid_constant__ CUtensorMap map, int R, int L, int nring, int K, uint32_t* out, int Lseg, int nseg) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, NB = (R + 255) / 256, br = R / NB;
    uint64_t* bars = (uint64_t*)dsm;
    const uint32_t full0 = smem_u32(bars), empty0 = full0 + 64;
    const uint32_t ring0 = smem_u32(dsm) + 1024;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nring; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 31);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // Lseg == 0: rows span the CTA's whole share (k_scan_tma today);
    // Lseg > 0: the share is nseg segments of R rows x Lseg bytes (segment-major)
    const int per_seg = Lseg ? Lseg / ROWB : L / ROWB;
    const int nst = Lseg ? per_seg * nseg : L / ROWB;
    const int y0 = blockIdx.x * R * (Lseg ? nseg : 1);
    if (warp == 31) {
        if (lane == 0) {
            uint32_t slot = 0, ph = 0;
            for (int i = 0; i < nst; ++i) {
                if (i >= nring) mbar_wait(empty0 + 8 * slot, ph ^ 1);
                mbar_expect_tx(full0 + 8 * slot, R * ROWB);
                const int sg = i / per_seg, x = (i % per_seg) * ROWB;
                for (int j = 0; j < NB; ++j)
                    tma_load_2d(ring0 + slot * R * ROWB + j * br * ROWB, &map, full0 + 8 * slot, x, y0 + sg * R + j * br);
                if (++slot == nring) {
                    slot = 0;
                    ph ^= 1;
                }
            }
        }
        return;
    }
    uint32_t acc = 0, slot = 0, ph = 0;
    for (int i = 0; i < nst; ++i) {
        mbar_wait(full0 + 8 * slot, ph);
        for (int k = 0; k < K; ++k) {
            const uint32_t r = k * 992 + warp * 32 + lane;
            if (r < (uint32_t)R)
                for (int c = 0; c < ROWB / 16; ++c) {
                    uint4 v;
                    uint32_t o = r * ROWB + c * 16;
                    o ^= ((o >> 7) & (ROWB / 16 - 1)) << 4;
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(ring0 + slot * R * ROWB + o));
                    acc ^= v.x ^ v.y ^ v.z ^ v.w;
                }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty0 + 8 * slot);
        if (++slot == nring) {
            slot = 0;
            ph ^= 1;
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// P3: warp-major.  Warp w of CTA b owns a contiguous share; it is cut into
// segments of 32 rows x Lr bytes (Lr = 16 x odd, so the lanes' LDS.128 of
// one piece index fall in distinct bank groups), each loaded by ONE 1-D bulk
// copy issued by the warp itself into its own ring of D slots.
__global__ void __launch_bounds__(1024, 1) k_mb_warp(const uint8_t* text, int Lr, int nseg, int D, int nw, uint32_t* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t segb = 32u * Lr;
    uint64_t* bars = (uint64_t*)dsm + warp * 8;
    const uint32_t full0 = smem_u32(bars);
    const uint32_t ring = smem_u32(dsm) + 4096 + warp * D * segb;
    if (lane == 0) {
        for (int s = 0; s < D; ++s) mbar_init(full0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const uint8_t* base = text + ((size_t)blockIdx.x * nw + warp) * (size_t)nseg * segb;
    if (lane == 0)
        for (int s = 0; s < D && s < nseg; ++s) {
            mbar_expect_tx(full0 + 8 * s, segb);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(ring + s * segb), "l"(base + (size_t)s * segb), "r"(segb), "r"(full0 + 8 * s) : "memory");
        }
    uint32_t acc = 0;
    for (int s = 0; s < nseg; ++s) {
        const int slot = s % D;
        mbar_wait(full0 + 8 * slot, (s / D) & 1);
        const uint32_t row = ring + slot * segb + lane * Lr;
        for (int j = 0; j < Lr / 16; ++j) {
            uint4 v;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(row + 16 * j));
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
        __syncwarp();
        if (lane == 0 && s + D < nseg) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(full0 + 8 * slot, segb);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(ring + slot * segb), "l"(base + (size_t)(s + D) * segb), "r"(segb), "r"(full0 + 8 * slot) : "memory");
        }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

void run_warp(uint8_t* d, size_t n, int nw, int Lr, int D, uint32_t* out) {
    const int G = 148;
    const size_t segb = 32ull * Lr;
    const int nseg = (int)(n / ((size_t)G * nw * segb));
    const size_t smem = 4096 + (size_t)nw * D * segb;
    if (smem > 227 * 1024) {
        printf("warp nw=%d Lr=%d D=%d: no fit\n", nw, Lr, D);
        return;
    }
    cudaFuncSetAttribute(k_mb_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) k_mb_warp<<<G, nw * 32, smem>>>(d, Lr, nseg, D, nw, out);
    cudaEventRecord(a);
    const int it = 20;
    for (int w = 0; w < it; ++w) k_mb_warp<<<G, nw * 32, smem>>>(d, Lr, nseg, D, nw, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)G * nw * nseg * segb;
    printf("1D-warp nw=%d Lr=%d D=%d nseg=%d: %.1f GB/s (%s)\n", nw, Lr, D, nseg, bytes * it / (ms * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int ROWB>
void run(EncFn enc, uint8_t* d, size_t n, int K, int nring, int promo, uint32_t* out, int Lseg = 0) {
    const int G = 148, R = 992 * K;
    const int L = (int)(n / ((size_t)G * R)) / 256 * 256;
    const int nseg = Lseg ? L / Lseg : 0;
    const size_t rows = Lseg ? (size_t)G * R * nseg : (size_t)G * R;
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)(Lseg ? Lseg : L), rows}, str[1] = {(cuuint64_t)(Lseg ? Lseg : L)};
    const int NB = (R + 255) / 256;
    cuuint32_t box[2] = {ROWB, (cuuint32_t)(R / NB)}, es[2] = {1, 1};
    CUtensorMapSwizzle sw = ROWB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : ROWB == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE;
    CUtensorMapL2promotion pr = promo == 0    ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                              : promo == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                              : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                             : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, pr,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        return;
    }
    const size_t smem = 1024 + (size_t)nring * R * ROWB;
    if (smem > 227 * 1024) {
        printf("K=%d ROWB=%d ring=%d: no fit\n", K, ROWB, nring);
        return;
    }
    cudaFuncSetAttribute(k_mb<ROWB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) k_mb<ROWB><<<G, 1024, smem>>>(m, R, L, nring, K, out, Lseg, nseg);
    cudaEventRecord(a);
    const int it = 20;
    for (int w = 0; w < it; ++w) k_mb<ROWB><<<G, 1024, smem>>>(m, R, L, nring, K, out, Lseg, nseg);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)(Lseg ? Lseg : L) * rows;
    printf("2D K=%d ROWB=%d ring=%d promo=%d L=%d Lseg=%d: %.1f GB/s (%s)\n", K, ROWB, nring, promo, L, Lseg,
           bytes * it / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? strtoull(argv[1], 0, 0) : (256ull << 20);
    void* p;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncFn enc = (EncFn)p;
    uint8_t* d;
    cudaMalloc(&d, n);
    cudaMemset(d, 1, n);
    uint32_t* out;
    cudaMalloc(&out, 4);
    if (argc > 2 && !strcmp(argv[2], "ring")) {  // the product's pattern per ring depth
        for (int ring : {2, 3, 4, 5, 6, 7}) run<32>(enc, d, n, 1, ring, 0, out);
        for (int ring : {2, 3}) run<64>(enc, d, n, 1, ring, 0, out);
        for (int ring : {4, 6, 8}) run<16>(enc, d, n, 1, ring, 0, out);  // (the barrier block holds 8 slots)
        return 0;
    }
    for (int promo : {0, 256}) {
        run<32>(enc, d, n, 1, 6, promo, out);
        run<64>(enc, d, n, 1, 3, promo, out);
        for (int Lseg : {256, 512, 1024}) {
            run<32>(enc, d, n, 1, 6, promo, out, Lseg);
            run<64>(enc, d, n, 1, 3, promo, out, Lseg);
            run<32>(enc, d, n, 2, 3, promo, out, Lseg);
        }
    }
    for (int nw : {32, 16}) {
        for (int Lr : {48, 80, 112, 144, 208}) {
            for (int D : {2, 3, 4}) run_warp(d, n, nw, Lr, D, out);
        }
    }
    return 0;
}
