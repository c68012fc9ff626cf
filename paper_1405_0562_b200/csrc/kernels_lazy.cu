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
constexpr uint32_t kFactBitDev = 0x80000000u;  // lazy.hpp kFactBit

__device__ __forceinline__ uint64_t lazy_piece(uint64_t g, uint64_t n, uint64_t p) {
    const uint64_t q = n / p, r = n % p;
    return g * q + (g < r ? g : r);
}

__global__ void k_lazy_init(uint64_t n, uint64_t p, uint32_t* state, uint64_t* pos, uint32_t* fd) {
    for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < p;
         g += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        state[g] = 0;  // f_I
        pos[g] = lazy_piece(g, n, p);
        fd[g] = kLazyUnknown;
    }
}

// Chunk g = [piece(g), piece(g+1)) resumes at pos[g] from state[g] (Alg. 5
// lines 3-5 with the table in global memory / L2) and stops before the first
// byte whose transition is not built (kLazyUnknown).  With a.factor, at the
// first factorable state s (T entry flagged kFactBit) it keeps s and runs the
// DFA from g_s over the rest of the chunk, the DFA table in shared memory
// (C24): the chunk ends as (s, d) and never stalls again.
// Returns the chunk's status after the run: 0 finished factored, 1 finished
// as a plain SFA state, 2 stalled.
__device__ __noinline__ int lazy_chunk(const LazyScanArgs& a, const uint8_t* cls, uint64_t g) {
    const uint64_t end = lazy_piece(g + 1, a.n, a.p);
    uint64_t at = a.pos[g];
    if (at >= end) return a.fd[g] == kLazyUnknown ? 1 : 0;
    const uint8_t* text = a.text;
    const uint32_t C = a.C;
    uint32_t s = a.state[g];
    uint32_t d = a.factor ? __ldg(a.fg + s) : kLazyUnknown;
    // one SFA byte: 0 = stepped, 1 = not built (stall), 2 = reached a factorable state
    auto sfa_byte = [&](uint32_t b) -> int {
        const uint32_t t = __ldg(a.T + static_cast<uint64_t>(s) * C + cls[b]);
        if (t == kLazyUnknown) return 1;
        s = t & ~kFactBitDev;
        if (a.factor && (t & kFactBitDev)) {
            d = __ldg(a.fg + s);
            return 2;
        }
        return 0;
    };
    if (d == kLazyUnknown) {
        int r = 0;
        while (at < end && r == 0) {
            if ((at & 15) == 0 && at + 16 <= end) {
                const uint4 v = ldg_stream(text + at);
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                uint32_t j = 0;
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    if (r == 0) {
                        r = sfa_byte((w[k >> 2] >> (8 * (k & 3))) & 0xffu);
                        j += r != 1;
                    }
                at += j;
            } else {
                r = sfa_byte(__ldg(text + at));
                at += r != 1;
            }
        }
        if (r == 1) {
            a.state[g] = s;
            a.pos[g] = at;
            return 2;
        }
    }
    if (d != kLazyUnknown) {  // factored: the DFA alone to the chunk's end
        // the table's entries are shared-window addresses of rows (the base
        // added at load): per byte a class lookup off the chain, then one
        // IADD3 and one LDS on it
        const uint32_t base = smem_u32(dsmem);
        uint32_t off = base + d * 2 * C;
        auto step1 = [&](uint32_t b) {
            const uint32_t c = cls[b];
            off = lds_u16(off + c + c);
        };
        auto dstep = [&](uint32_t w) {
#pragma unroll
            for (int k = 0; k < 4; ++k) step1((w >> (8 * k)) & 0xffu);
        };
        while (at < end && (at & 15)) step1(__ldg(text + at++));
        if (at + 16 <= end) {  // 16-byte blocks, the next two in flight
            uint4 v0 = ldg_stream(text + at);
            uint4 v1 = at + 32 <= end ? ldg_stream(text + at + 16) : v0;
            while (at + 48 <= end) {
                const uint4 v2 = ldg_stream(text + at + 32);
                dstep(v0.x), dstep(v0.y), dstep(v0.z), dstep(v0.w);
                v0 = v1, v1 = v2, at += 16;
            }
            dstep(v0.x), dstep(v0.y), dstep(v0.z), dstep(v0.w);
            at += 16;
            if (at + 16 <= end) {
                dstep(v1.x), dstep(v1.y), dstep(v1.z), dstep(v1.w);
                at += 16;
            }
        }
        while (at < end) step1(__ldg(text + at++));
        d = (off - base) / (2 * C);
        a.fd[g] = d;
    }
    a.state[g] = s;
    a.pos[g] = end;
    return d == kLazyUnknown ? 1 : 0;
}

__global__ void __launch_bounds__(256) k_lazy_scan(LazyScanArgs a) {
    uint16_t* dfa_s = reinterpret_cast<uint16_t*>(dsmem);  // the window table
    __shared__ uint8_t cls[256];
    cls[threadIdx.x] = a.cls[threadIdx.x];
    if (a.factor) {
        const uint32_t base = smem_u32(dsmem);  // < 64 KiB: the entries stay u16
        for (uint32_t i = threadIdx.x; i < a.nD * a.C; i += blockDim.x)
            dfa_s[i] = static_cast<uint16_t>(a.drow[i] + base);
    }
    __syncthreads();
    const uint64_t g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int r = g < a.p ? lazy_chunk(a, cls, g) : 0;
    // counts[0]: chunks stalled, counts[1]: chunks finished as plain SFA states
    const uint32_t st = __popc(__ballot_sync(0xffffffffu, r == 2)), pl = __popc(__ballot_sync(0xffffffffu, r == 1));
    if ((threadIdx.x & 31) == 0) {
        if (st) atomicAdd(a.counts, st);
        if (pl) atomicAdd(a.counts + 1, pl);
    }
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

// vec[g] <- the chunk's mapping: f_{state[g]}, or for a factored chunk
// f(q) = absorbing[f_s(q)] ? f_s(q) : fd[g]
__global__ void k_lazy_vec(const uint16_t* __restrict__ maps, const uint32_t* __restrict__ state,
                           const uint32_t* __restrict__ fd, const uint8_t* __restrict__ absorbing, uint64_t p, uint32_t nD,
                           uint16_t* __restrict__ vec) {
    const uint64_t total = p * nD;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t g = i / nD, q = i - g * nD;
        const uint32_t m = maps[static_cast<uint64_t>(state[g]) * nD + q], e = fd[g];
        vec[i] = static_cast<uint16_t>(e == kLazyUnknown || absorbing[m] ? m : e);
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

// The compact fold when every chunk is factored (C24): (s1, d1) . e2 =
// (s1, e2(d1)), e2(x) = absorbing[f_{s2}(x)] ? f_{s2}(x) : d2 -- one lookup
// per composition instead of an |D| vector.  Each block folds 1024 adjacent
// elements in order (a tree in shared memory).
__global__ void __launch_bounds__(1024) k_lazy_cfold(const uint16_t* __restrict__ maps, const uint8_t* __restrict__ absorbing,
                                                     uint32_t nD, const uint32_t* __restrict__ s_in,
                                                     const uint32_t* __restrict__ d_in, uint64_t cnt,
                                                     uint32_t* __restrict__ s_out, uint32_t* __restrict__ d_out) {
    __shared__ uint32_t ss[1024], sd[1024];
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * 1024;
    const uint32_t i = threadIdx.x;
    const uint32_t m = static_cast<uint32_t>(cnt - base < 1024 ? cnt - base : 1024);
    if (i < m) ss[i] = s_in[base + i], sd[i] = d_in[base + i];
    __syncthreads();
    for (uint32_t w = 1; w < m; w *= 2) {
        if ((i % (2 * w)) == 0 && i + w < m) {
            const uint32_t x = sd[i], y = maps[static_cast<uint64_t>(ss[i + w]) * nD + x];
            sd[i] = absorbing[y] ? y : sd[i + w];
        }
        __syncthreads();
    }
    if (i == 0) s_out[blockIdx.x] = ss[0], d_out[blockIdx.x] = sd[0];
}

// q_final = (s, d)(q0 = 0)
__global__ void k_lazy_capply(const uint16_t* __restrict__ maps, const uint8_t* __restrict__ absorbing, uint32_t nD,
                              const uint32_t* s, const uint32_t* d, uint16_t* out) {
    const uint32_t y = maps[static_cast<uint64_t>(s[0]) * nD];
    *out = static_cast<uint16_t>(absorbing[y] ? y : d[0]);
}

unsigned grid_for(uint64_t work, int sm_count) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((work + 255) / 256, 16ull * sm_count)));
}

}  // namespace

cudaError_t lazy_init(uint64_t n, uint64_t p, uint32_t* state, uint64_t* pos, uint32_t* fd, int sm_count,
                      cudaStream_t s) {
    k_lazy_init<<<grid_for(p, sm_count), 256, 0, s>>>(n, p, state, pos, fd);
    return cudaGetLastError();
}

cudaError_t lazy_scan(const LazyScanArgs& a, cudaStream_t s) {
    const size_t smem = a.factor ? static_cast<size_t>(a.nD) * a.C * sizeof(uint16_t) : 0;
    if (smem > kLazyFactorSmem) return cudaErrorInvalidValue;
    k_lazy_scan<<<static_cast<unsigned>((a.p + 255) / 256), 256, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t lazy_gather(const uint8_t* text, uint64_t n, uint64_t p, const uint64_t* pos, const uint32_t* idx,
                        uint32_t count, uint32_t K, uint8_t* out, cudaStream_t s) {
    k_lazy_gather<<<count, 256, 0, s>>>(text, n, p, pos, idx, K, out);
    return cudaGetLastError();
}

// f_fin = f_{state[0]} . ... . f_{state[p-1]} by a pairwise tree over the
// vectors (buf: 2 * p * nD u16 scratch); writes f_fin to out (nD u16, device).
cudaError_t lazy_fold(const uint16_t* maps, const uint32_t* state, const uint32_t* fd, const uint8_t* absorbing,
                      uint64_t p, uint32_t nD, uint16_t* buf, uint16_t* out, int sm_count, cudaStream_t s) {
    uint16_t* a = buf;
    uint16_t* b = buf + p * nD;
    k_lazy_vec<<<grid_for(p * nD, sm_count), 256, 0, s>>>(maps, state, fd, absorbing, p, nD, a);
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

// The compact fold (every chunk factored): f_fin(q0) with q0 = 0 into *out.
// buf: 4 * ceil(p / 1024) u32 scratch.
cudaError_t lazy_cfold(const uint16_t* maps, const uint8_t* absorbing, uint32_t nD, const uint32_t* state,
                       const uint32_t* fd, uint64_t p, uint32_t* buf, uint16_t* out, cudaStream_t s) {
    const uint64_t half = (p + 1023) / 1024;
    uint32_t *s0 = buf, *d0 = buf + half, *s1 = buf + 2 * half, *d1 = buf + 3 * half;
    const uint32_t* si = state;
    const uint32_t* di = fd;
    uint64_t cnt = p;
    do {
        const uint64_t blocks = (cnt + 1023) / 1024;
        k_lazy_cfold<<<static_cast<unsigned>(blocks), 1024, 0, s>>>(maps, absorbing, nD, si, di, cnt, s0, d0);
        si = s0, di = d0;
        std::swap(s0, s1), std::swap(d0, d1);
        cnt = blocks;
    } while (cnt > 1);
    k_lazy_capply<<<1, 1, 0, s>>>(maps, absorbing, nD, si, di, out);
    return cudaGetLastError();
}

}  // namespace sfa
