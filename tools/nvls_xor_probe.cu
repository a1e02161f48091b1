// tools/nvls_xor_probe.cu -- feasibility probe for parity by in-switch XOR.
//
// One process, n GPUs: a multicast object (cuMulticastCreate) bound to one buffer per GPU
// (cuMemCreate); GPU 0 runs `multimem.ld_reduce.relaxed.sys.global.xor.b64` over the
// multicast mapping, so NVSwitch returns XOR_j buf_j[i] -- one value per address.  Checks the
// result against a host XOR of the buffers and reports the reduce rate (output bytes / time)
// and the NVLink ingress it implies (one unit per output unit instead of n).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvls tools/nvls_xor_probe.cu -lcuda
//   /tmp/nvls [n_gpus] [MiB per GPU]
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CU(x)                                                                              \
    do {                                                                                   \
        CUresult r_ = (x);                                                                 \
        if (r_ != CUDA_SUCCESS) {                                                          \
            const char *s_ = nullptr;                                                      \
            cuGetErrorString(r_, &s_);                                                     \
            fprintf(stderr, "%s:%d %s -> %d %s\n", __FILE__, __LINE__, #x, (int)r_, s_ ? s_ : ""); \
            return 2;                                                                      \
        }                                                                                  \
    } while (0)
#define RT(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            return 2;                                                                      \
        }                                                                                  \
    } while (0)

__global__ void fill(uint64_t *p, uint64_t n, uint64_t seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = (i + seed * 0x9E3779B97F4A7C15ull) * 0xBF58476D1CE4E5B9ull;
        p[i] = z ^ (z >> 31);
    }
}

template <int U>
__global__ void __launch_bounds__(256) xor_reduce(const uint64_t *mc, uint64_t *out, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t base = (blockIdx.x * (uint64_t)blockDim.x) * U + threadIdx.x; base < n; base += stride) {
        uint64_t v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint64_t i = base + (uint64_t)k * blockDim.x;
            v[k] = 0;
            if (i < n)
                asm volatile("multimem.ld_reduce.relaxed.sys.global.xor.b64 %0, [%1];"
                             : "=l"(v[k]) : "l"(mc + i) : "memory");
        }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const uint64_t i = base + (uint64_t)k * blockDim.x;
            if (i < n) out[i] = v[k];
        }
    }
}

int main(int argc, char **argv) {
    int n = argc > 1 ? atoi(argv[1]) : 2;
    const uint64_t mib = argc > 2 ? strtoull(argv[2], nullptr, 10) : 1024;
    int ndev = 0;
    RT(cudaGetDeviceCount(&ndev));
    if (n > ndev) n = ndev;
    CU(cuInit(0));
    std::vector<CUdevice> dev(n);
    for (int d = 0; d < n; ++d) {
        RT(cudaSetDevice(d));
        RT(cudaFree(0));  // primary context
        CU(cuDeviceGet(&dev[d], d));
        int mc = 0;
        CU(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev[d]));
        if (!mc) {
            printf("{\"nvls\": false, \"why\": \"device %d: CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0\"}\n", d);
            return 0;
        }
    }
    RT(cudaSetDevice(0));
    CUmulticastObjectProp prop;
    memset(&prop, 0, sizeof prop);
    prop.numDevices = (unsigned)n;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
    prop.size = mib << 20;
    size_t gran = 0;
    CU(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    const size_t size = (prop.size + gran - 1) / gran * gran;
    prop.size = size;
    CUmemGenericAllocationHandle mc;
    CU(cuMulticastCreate(&mc, &prop));
    for (int d = 0; d < n; ++d) CU(cuMulticastAddDevice(mc, dev[d]));
    std::vector<CUmemGenericAllocationHandle> h(n);
    std::vector<CUdeviceptr> va(n);
    for (int d = 0; d < n; ++d) {
        RT(cudaSetDevice(d));
        CUmemAllocationProp ap;
        memset(&ap, 0, sizeof ap);
        ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ap.location.id = d;
        size_t g2 = 0;
        CU(cuMemGetAllocationGranularity(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
        if (size % g2) {
            fprintf(stderr, "size %zu not a multiple of %zu\n", size, g2);
            return 2;
        }
        CU(cuMemCreate(&h[d], size, &ap, 0));
        CU(cuMulticastBindMem(mc, 0, h[d], 0, size, 0));
        CU(cuMemAddressReserve(&va[d], size, 0, 0, 0));
        CU(cuMemMap(va[d], size, 0, h[d], 0));
        CUmemAccessDesc ad;
        ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ad.location.id = d;
        ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        CU(cuMemSetAccess(va[d], size, &ad, 1));
        fill<<<1184, 256>>>((uint64_t *)va[d], size / 8, (uint64_t)d + 1);
        RT(cudaDeviceSynchronize());
    }
    RT(cudaSetDevice(0));
    CUdeviceptr mcva;
    CU(cuMemAddressReserve(&mcva, size, 0, 0, 0));
    CU(cuMemMap(mcva, size, 0, mc, 0));
    std::vector<CUmemAccessDesc> ads(n);
    for (int d = 0; d < n; ++d) {
        ads[d].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        ads[d].location.id = d;
        ads[d].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    CU(cuMemSetAccess(mcva, size, ads.data(), n));
    uint64_t *out = nullptr;
    RT(cudaMalloc(&out, size));
    const uint64_t words = size / 8;
    cudaEvent_t e0, e1;
    RT(cudaEventCreate(&e0));
    RT(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        RT(cudaEventRecord(e0));
        xor_reduce<8><<<148 * 8, 256>>>((const uint64_t *)mcva, out, words);
        RT(cudaEventRecord(e1));
        RT(cudaEventSynchronize(e1));
        float ms = 0;
        RT(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    // every GPU reduces its own 1/n of the buffer at once (the parity pattern: each rank
    // produces one row): the multicast mapping is made accessible on every device above
    std::vector<uint64_t *> outs(n, nullptr);
    std::vector<cudaEvent_t> a0(n), a1(n);
    for (int d = 0; d < n; ++d) {
        RT(cudaSetDevice(d));
        RT(cudaMalloc(&outs[d], size / n + 8));
        RT(cudaEventCreate(&a0[d]));
        RT(cudaEventCreate(&a1[d]));
    }
    float all_best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        for (int d = 0; d < n; ++d) {
            RT(cudaSetDevice(d));
            RT(cudaDeviceSynchronize());
        }
        auto t0 = std::chrono::steady_clock::now();
        for (int d = 0; d < n; ++d) {
            RT(cudaSetDevice(d));
            const uint64_t w0 = words * d / n, w1 = words * (d + 1) / n;
            RT(cudaEventRecord(a0[d]));
            xor_reduce<8><<<148 * 8, 256>>>((const uint64_t *)mcva + w0, outs[d], w1 - w0);
            RT(cudaEventRecord(a1[d]));
        }
        for (int d = 0; d < n; ++d) {
            RT(cudaSetDevice(d));
            RT(cudaEventSynchronize(a1[d]));
        }
        const float wall = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
        float mx = 0;
        for (int d = 0; d < n; ++d) {
            float ms = 0;
            RT(cudaEventElapsedTime(&ms, a0[d], a1[d]));
            mx = ms > mx ? ms : mx;
        }
        (void)wall;
        if (mx < all_best) all_best = mx;
    }
    RT(cudaSetDevice(0));
    // check a sample against the host XOR of the unicast buffers
    const uint64_t sample = std::min<uint64_t>(words, 1 << 20);
    std::vector<uint64_t> got(sample), acc(sample, 0), tmp(sample);
    RT(cudaMemcpy(got.data(), out, sample * 8, cudaMemcpyDeviceToHost));
    for (int d = 0; d < n; ++d) {
        RT(cudaSetDevice(d));
        RT(cudaMemcpy(tmp.data(), (void *)va[d], sample * 8, cudaMemcpyDeviceToHost));
        for (uint64_t i = 0; i < sample; ++i) acc[i] ^= tmp[i];
    }
    const bool ok = memcmp(got.data(), acc.data(), sample * 8) == 0;
    printf("{\"nvls\": true, \"gpus\": %d, \"bytes_per_gpu\": %zu, \"granularity\": %zu, \"reduce_ms\": %.3f, "
           "\"output_gbs\": %.1f, \"xor_of_n_inputs_gbs\": %.1f, \"all_gpus_each_1_over_n_ms\": %.3f, "
           "\"all_gpus_output_gbs_per_gpu\": %.1f, \"bit_exact_sampled\": %s}\n",
           n, size, gran, best, size / (best * 1e6), (double)size * n / (best * 1e6), all_best,
           (double)size / n / (all_best * 1e6), ok ? "true" : "false");
    return ok ? 0 : 1;
}
