// kernels_lazy.cu -- the device half of the on-the-fly SFA construction
// (lazy.hpp): chunk runs that stop at the first transition
// the host has not built yet, the gather of the text windows the host needs to
// build more, and the composition of the chunk states as mapping vectors
// (f . g)(q) = g(f(q)) in a pairwise tree.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "device.cuh"
#include "kernels.hpp"

namespace sfa {

namespace {

constexpr uint32_t kLazyUnknown = 0xffffffffu;

__device__ __forceinline__ uint64_t lazy_piece(uint64_t g, uint64_t n, uint64_t p) {
    const uint64_t q = n / p, r = n % p;
    return g * q + (g < r ? g : r);
}

__global__ void k_lazy_init(uint64_t n, uint64_t p, uint32_t* state, uint64_t* pos) {
    for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < p;
         g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        state[g] = 0;  // f_I
        pos[g] = lazy_piece(g, n, p);
    }
}

// Chunk g = [piece(g), piece(g+1)) resumes at pos[g] from state[g] (Alg. 5
// lines 3-5 with the table in global memory / L2) and stops before the first
// byte whose transition is not built (kLazyUnknown).
__global__ void __launch_bounds__(256) k_lazy_scan(const uint32_t* __restrict__ T, const uint8_t* __restrict__ cls_g,
                                                   uint32_t C, const uint8_t* __restrict__ text, uint64_t n, uint64_t p,
                                                   uint32_t* __restrict__ state, uint64_t* __restrict__ pos) {
    __shared__ uint8_t cls[256];
    cls[threadIdx.x] = cls_g[threadIdx.x];
    __syncthreads();
    const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= p) return;
    const uint64_t end = lazy_piece(g + 1, n, p);
    uint64_t a = pos[g];
    if (a >= end) return;
    uint32_t s = state[g];
    while (a < end) {
        if ((a & 15) == 0 && a + 16 <= end) {
            const uint4 v = ldg_stream(text + a);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t c = cls[(w[j >> 2] >> (8 * (j & 3))) & 0xffu];
                const uint32_t t = __ldg(T + static_cast<uint64_t>(s) * C + c);
                if (t == kLazyUnknown) {
                    state[g] = s;
                    pos[g] = a + j;
                    return;
                }
                s = t;
            }
            a += 16;
        } else {
            const uint32_t t = __ldg(T + static_cast<uint64_t>(s) * C + cls[__ldg(text + a)]);
            if (t == kLazyUnknown) break;
            s = t;
            ++a;
        }
    }
    state[g] = s;
    pos[g] = a;
}

// out[j * K ..] <- text[pos[idx[j]], +min(K, end - pos)) for the stalled chunks idx[j]
__global__ void k_lazy_gather(const uint8_t* __restrict__ text, uint64_t n, uint64_t p, const uint64_t* __restrict__ pos,
                              const uint32_t* __restrict__ idx, uint32_t K, uint8_t* __restrict__ out) {
    const uint32_t j = blockIdx.x;
    const uint64_t g = idx[j];
    const uint64_t a = pos[g], end = lazy_piece(g + 1, n, p);
    const uint64_t len = end - a < K ? end - a : K;
    for (uint64_t i = threadIdx.x; i < len; i += blockDim.x) out[static_cast<uint64_t>(j) * K + i] = text[a + i];
}

// vec[g] <- f_{state[g]} (nD u16 per vector)
__global__ void k_lazy_vec(const uint16_t* __restrict__ maps, const uint32_t* __restrict__ state, uint64_t p, uint32_t nD,
                           uint16_t* __restrict__ vec) {
    const uint64_t total = p * nD;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t g = i / nD, q = i - g * nD;
        vec[i] = maps[static_cast<uint64_t>(state[g]) * nD + q];
    }
}

// out[j] <- in[2j] . in[2j+1], i.e. out[j][q] = in[2j+1][in[2j][q]] (or in[2j] alone)
__global__ void k_lazy_pairs(const uint16_t* __restrict__ in, uint64_t cnt, uint32_t nD, uint16_t* __restrict__ out) {
    const uint64_t half = (cnt + 1) / 2, total = half * nD;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t j = i / nD, q = i - j * nD;
        const uint32_t f = in[2 * j * nD + q];
        out[i] = 2 * j + 1 < cnt ? in[(2 * j + 1) * nD + f] : static_cast<uint16_t>(f);
    }
}

unsigned grid_for(uint64_t work, int sm_count) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, 16ull * sm_count)));
}

}  // namespace

cudaError_t lazy_init(uint64_t n, uint64_t p, uint32_t* state, uint64_t* pos, int sm_count, cudaStream_t s) {
    k_lazy_init<<<grid_for(p, sm_count), 256, 0, s>>>(n, p, state, pos);
    return cudaGetLastError();
}

cudaError_t lazy_scan(const uint32_t* T, const uint8_t* cls, uint32_t C, const uint8_t* text, uint64_t n, uint64_t p,
                      uint32_t* state, uint64_t* pos, cudaStream_t s) {
    k_lazy_scan<<<static_cast<unsigned>((p + 255) / 256), 256, 0, s>>>(T, cls, C, text, n, p, state, pos);
    return cudaGetLastError();
}

cudaError_t lazy_gather(const uint8_t* text, uint64_t n, uint64_t p, const uint64_t* pos, const uint32_t* idx,
                        uint32_t count, uint32_t K, uint8_t* out, cudaStream_t s) {
    k_lazy_gather<<<count, 256, 0, s>>>(text, n, p, pos, idx, K, out);
    return cudaGetLastError();
}

// f_fin = f_{state[0]} . ... . f_{state[p-1]} by a pairwise tree over the
// vectors (buf: 2 * p * nD u16 scratch); writes f_fin to out (nD u16, device).
cudaError_t lazy_fold(const uint16_t* maps, const uint32_t* state, uint64_t p, uint32_t nD, uint16_t* buf,
                      uint16_t* out, int sm_count, cudaStream_t s) {
    uint16_t* a = buf;
    uint16_t* b = buf + p * nD;
    k_lazy_vec<<<grid_for(p * nD, sm_count), 256, 0, s>>>(maps, state, p, nD, a);
    uint64_t cnt = p;
    while (cnt > 1) {
        k_lazy_pairs<<<grid_for((cnt + 1) / 2 * nD, sm_count), 256, 0, s>>>(a, cnt, nD, b);
        std::swap(a, b);
        cnt = (cnt + 1) / 2;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(out, a, nD * sizeof(uint16_t), cudaMemcpyDeviceToDevice, s);
}

}  // namespace sfa
