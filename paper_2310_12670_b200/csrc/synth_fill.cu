// synth_fill.cu -- harness: seeded synthetic state on the GPU (see include/reft_synth.h).
// Not part of the method and not linked into libreft_ckpt.
#include <cuda_runtime.h>
#include <stdint.h>

#pragma GCC visibility push(default)  // the C ABI is the only exported surface
#include "../../include/reft_synth.h"
#pragma GCC visibility pop

namespace {
__device__ __forceinline__ uint64_t sm64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// one thread per 8-byte word of the tensor; byte-wise stores at the (rare) unaligned ends
__global__ void fill_kernel(uint8_t *dst, uint64_t nbytes, uint64_t base, int xor_mode) {
    const uint64_t nwords = (nbytes + 7) / 8;
    const bool aligned8 = ((uintptr_t)dst & 7) == 0;
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwords;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = sm64(base ^ w);
        const uint64_t b0 = w * 8;
        if (aligned8 && b0 + 8 <= nbytes) {
            uint64_t *p = reinterpret_cast<uint64_t *>(dst + b0);
            *p = xor_mode ? (*p ^ v) : v;
        } else {
            for (int i = 0; i < 8 && b0 + i < nbytes; ++i) {
                const uint8_t byte = (uint8_t)(v >> (8 * i));
                dst[b0 + i] = xor_mode ? (uint8_t)(dst[b0 + i] ^ byte) : byte;
            }
        }
    }
}
}  // namespace

extern "C" int reft_synth_fill(void *dst, uint64_t nbytes, uint64_t seed, uint64_t rank, uint64_t tensor,
                               int xor_mode, void *stream) {
    if (!dst || nbytes == 0) return nbytes == 0 ? 0 : -1;
    // base(j, t) on the host: three finaliser calls
    auto h = [](uint64_t x) {
        uint64_t z = x + 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    };
    const uint64_t base = h(h(h(seed) ^ rank) ^ tensor);
    const uint64_t nwords = (nbytes + 7) / 8;
    uint64_t grid = (nwords + 255) / 256;
    if (grid > 148 * 16) grid = 148 * 16;
    fill_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>((uint8_t *)dst, nbytes, base, xor_mode);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : -(int)e;
}
