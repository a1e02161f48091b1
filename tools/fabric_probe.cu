// tools/fabric_probe.cu -- all-concurrent NVLink probe for the XOR encode's roofline
// ("NVLink ... to be measured P2P, all ranks concurrent").
//
// One process drives m GPUs.  Every GPU moves n bytes to/from EACH of its m-1 peers at
// the same time -- the encode's all-to-all pattern (every rank pulls L*/(m-1) from every
// peer) -- with one of these mechanisms:
//   ce_pull   copy engines: one cudaMemcpyAsync per peer (peer -> local), own stream each
//   ce_push   copy engines: local -> peer
//   sm_pull   kernel: cp.async.bulk G->S from the peers (16 KiB pieces, 3 stages per warp),
//             data discarded -- the load side of xor_tma_kernel
//   sm_push   kernel: cp.async.bulk G->S locally, cp.async.bulk S->G into the peers
//   sm_red    kernel: cp.async.bulk G->S locally, cp.reduce.async.bulk .xor.b64 into the
//             peers (the push-mode encode's transfer); checked: dst ^= src
//   lsu_push  kernel: 128-bit ld.global.nc locally, st.global into the peers
//   xorpat4k / xorpat16k (m = 4): the encode's load pattern -- each stage holds one segment
//             from EVERY peer (unit sigma(me, j) of a stripe), one mbarrier for all three --
//             with xor_tma_kernel's 4 KiB x 4 warps or 16 KiB x 1 warp geometry, no arithmetic
// Reports per GPU: GB/s of NVLink bytes out (push) or in (pull), min over GPUs, and the
// aggregate.  Timing: CUDA events per GPU, best of `reps`, all GPUs launched back to back.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/fabric tools/fabric_probe.cu
//   /tmp/fabric <m> <MiB per peer> <mode> [ctas per GPU] [reps]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#define RT(x)                                                                                      \
    do {                                                                                           \
        cudaError_t e_ = (x);                                                                      \
        if (e_ != cudaSuccess) {                                                                   \
            fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));   \
            exit(2);                                                                               \
        }                                                                                          \
    } while (0)

constexpr int kW = 4, kNS = 3;
constexpr uint32_t kT = 16384;
constexpr int kMaxPeers = 7;

struct Args {
    const uint8_t *src[kMaxPeers];  // per peer q: where item (q, c) is read from
    uint8_t *dst[kMaxPeers];        // per peer q: where it goes (nullptr: discard)
    int npeers;
    uint64_t n;                     // bytes per peer
    int op;                         // 0 copy 1 xor-reduce
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
                     smem_u32(bar)),
                 "r"(parity)
                 : "memory");
}
__device__ __forceinline__ void g2s(void *s, const void *g, uint32_t b, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(s)),
                 "l"(g), "r"(b), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void s2g(void *g, const void *s, uint32_t b) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(s)), "r"(b) : "memory");
}
__device__ __forceinline__ void s2g_xor(void *g, const void *s, uint32_t b) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.xor.b64 [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(s)), "r"(b)
                 : "memory");
}

// Items: (q, c) for peer q < npeers and piece c < n / kT, interleaved over peers.
__global__ void __launch_bounds__(32 * kW) bulk_kernel(const __grid_constant__ Args a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[kW][kNS];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane) return;
    uint8_t *ring = smem + (size_t)w * kNS * kT;
    for (int i = 0; i < kNS; ++i) mbar_init(&bars[w][i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint64_t per = a.n / kT, items = per * a.npeers;
    const uint64_t step = (uint64_t)gridDim.x * kW;
    auto src_of = [&](uint64_t it) { return a.src[it % a.npeers] + (it / a.npeers) * kT; };
    auto dst_of = [&](uint64_t it) { return a.dst[it % a.npeers] + (it / a.npeers) * kT; };
    const uint64_t first = (uint64_t)blockIdx.x * kW + w;
    int k = 0;
    for (uint64_t it = first; it < items && k < kNS; it += step, ++k) {
        mbar_expect_tx(&bars[w][k], kT);
        g2s(ring + (size_t)k * kT, src_of(it), kT, &bars[w][k]);
    }
    uint32_t phase = 0;
    int st = 0;
    uint64_t prev = UINT64_MAX;
    int prev_st = 0;
    for (uint64_t it = first; it < items; it += step) {
        mbar_wait(&bars[w][st], (phase >> st) & 1);
        phase ^= 1u << st;
        if (a.dst[0] == nullptr) {  // pull, discard: refill this stage at once
            const uint64_t nx = it + (uint64_t)kNS * step;
            if (nx < items) {
                mbar_expect_tx(&bars[w][st], kT);
                g2s(ring + (size_t)st * kT, src_of(nx), kT, &bars[w][st]);
            }
        } else {
            if (a.op) s2g_xor(dst_of(it), ring + (size_t)st * kT, kT);
            else s2g(dst_of(it), ring + (size_t)st * kT, kT);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (prev != UINT64_MAX) {  // the previous item's store has read its stage: refill it
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                const uint64_t nx = prev + (uint64_t)kNS * step;
                if (nx < items) {
                    mbar_expect_tx(&bars[w][prev_st], kT);
                    g2s(ring + (size_t)prev_st * kT, src_of(nx), kT, &bars[w][prev_st]);
                }
            }
            prev = it;
            prev_st = st;
        }
        st = st + 1 == kNS ? 0 : st + 1;
    }
    if (a.dst[0] != nullptr) {
        const uint64_t nx = prev == UINT64_MAX ? items : prev + (uint64_t)kNS * step;
        (void)nx;
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}


// The encode's load pattern without its arithmetic: tile t of unit-space (stripe s, piece w
// of a unit) needs one T-byte segment from EACH peer (unit sigma(me, j) of stripe s) in one
// stage, completed by one mbarrier (all m-1 must land before the stage is reused) -- as in
// xor_tma_kernel.  Data discarded.
template <int NIN, uint32_t T, int NS, int W>
__global__ void __launch_bounds__(32 * W) xorpat_kernel(const __grid_constant__ Args a, uint64_t unit, uint32_t me) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[W][NS];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane) return;
    uint8_t *ring = smem + (size_t)w * NS * NIN * T;
    for (int i = 0; i < NS; ++i) mbar_init(&bars[w][i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    // every peer's staging holds n * NIN bytes = n / unit stripes of NIN units
    const uint64_t stripe = unit * NIN, nstripes = a.n * NIN / stripe, tpu = unit / T;
    const uint64_t items = nstripes * tpu, step = (uint64_t)gridDim.x * W;
    auto issue = [&](uint64_t it, int st) {
        const uint64_t sidx = it / tpu, off = (it - sidx * tpu) * T;
        mbar_expect_tx(&bars[w][st], T * NIN);
        for (int k = 0; k < NIN; ++k) {
            const uint32_t j = (uint32_t)k + ((uint32_t)k >= me ? 1u : 0u);  // peer j (skip me)
            const uint32_t sig = me - (me > j ? 1u : 0u);                     // sigma(me, j)
            g2s(ring + ((size_t)st * NIN + k) * T, a.src[k] + sidx * stripe + sig * unit + off, T, &bars[w][st]);
        }
    };
    const uint64_t first = (uint64_t)blockIdx.x * W + w;
    int k = 0;
    for (uint64_t it = first; it < items && k < NS; it += step, ++k) issue(it, k);
    uint32_t phase = 0;
    int st = 0;
    for (uint64_t it = first; it < items; it += step) {
        mbar_wait(&bars[w][st], (phase >> st) & 1);
        phase ^= 1u << st;
        const uint64_t nx = it + (uint64_t)NS * step;
        if (nx < items) issue(nx, st);
        st = st + 1 == NS ? 0 : st + 1;
    }
}

__global__ void __launch_bounds__(256) lsu_push_kernel(const Args a) {
    const uint64_t words = a.n / 16;
    const uint64_t total = words * a.npeers;
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += (uint64_t)gridDim.x * 256 * 4) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t x = i + (uint64_t)u * gridDim.x * 256;
            if (x < total) {
                const uint4 *p = reinterpret_cast<const uint4 *>(a.src[x % a.npeers]) + x / a.npeers;
                asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t x = i + (uint64_t)u * gridDim.x * 256;
            if (x < total) reinterpret_cast<uint4 *>(a.dst[x % a.npeers])[x / a.npeers] = v[u];
        }
    }
}

__global__ void fill_kernel(uint64_t *p, uint64_t n, uint64_t seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = (i ^ (seed * 0x9E3779B97F4A7C15ull)) * 0xBF58476D1CE4E5B9ull;
        p[i] = z ^ (z >> 29);
    }
}

int main(int argc, char **argv) {
    int m = argc > 1 ? atoi(argv[1]) : 2;
    const uint64_t n = (uint64_t)(argc > 2 ? atoll(argv[2]) : 1024) << 20;
    const std::string mode = argc > 3 ? argv[3] : "sm_pull";
    int ctas = argc > 4 ? atoi(argv[4]) : 32;
    const int reps = argc > 5 ? atoi(argv[5]) : 5;
    int ng = 0;
    RT(cudaGetDeviceCount(&ng));
    if (m > ng || m < 2 || m > kMaxPeers + 1) {
        fprintf(stderr, "need 2 <= m <= %d GPUs (have %d)\n", ng, ng);
        return 2;
    }
    // buffers: src[d] holds m regions of n (region r: read by / pushed to rank r); dst[d] m regions
    std::vector<uint8_t *> src(m), dst(m);
    std::vector<cudaStream_t> st(m * m);
    std::vector<cudaEvent_t> e0(m), e1(m);
    for (int d = 0; d < m; ++d) {
        RT(cudaSetDevice(d));
        for (int p = 0; p < m; ++p)
            if (p != d) {
                cudaError_t e = cudaDeviceEnablePeerAccess(p, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) RT(e);
                cudaGetLastError();
            }
        RT(cudaMalloc(&src[d], n * m));
        RT(cudaMalloc(&dst[d], n * m));
        fill_kernel<<<1184, 256>>>((uint64_t *)src[d], n * m / 8, 1 + d);
        fill_kernel<<<1184, 256>>>((uint64_t *)dst[d], n * m / 8, 100 + d);
        for (int q = 0; q < m; ++q) RT(cudaStreamCreateWithFlags(&st[d * m + q], cudaStreamNonBlocking));
        RT(cudaEventCreate(&e0[d]));
        RT(cudaEventCreate(&e1[d]));
        RT(cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kW * kNS * (int)kT));
    }
    for (int d = 0; d < m; ++d) {
        RT(cudaSetDevice(d));
        RT(cudaDeviceSynchronize());
    }
    // sm_red correctness: keep a host copy of one destination region and of the source
    std::vector<uint64_t> before, srcv;
    const bool red = mode == "sm_red";
    const uint64_t chk = std::min<uint64_t>(n, 1 << 20);
    if (red) {  // GPU 1 receives GPU 0's region 1 into its dst region 0
        before.resize(chk / 8);
        srcv.resize(chk / 8);
        RT(cudaSetDevice(1));
        RT(cudaMemcpy(before.data(), dst[1] + 0 * n, chk, cudaMemcpyDeviceToHost));
        RT(cudaSetDevice(0));
        RT(cudaMemcpy(srcv.data(), src[0] + 1 * n, chk, cudaMemcpyDeviceToHost));
    }
    double best_min = 0, best_agg = 0;
    std::vector<double> best_dev(m, 0);
    for (int r = 0; r < (red ? 1 : reps); ++r) {
        for (int d = 0; d < m; ++d) {
            RT(cudaSetDevice(d));
            RT(cudaEventRecord(e0[d], st[d * m]));
            Args a;
            memset(&a, 0, sizeof a);
            a.n = n;
            a.op = red ? 1 : 0;
            for (int p = 0; p < m; ++p) {
                if (p == d) continue;
                const int q = a.npeers++;
                if (mode == "sm_pull") {
                    a.src[q] = src[p] + (uint64_t)d * n;
                    a.dst[q] = nullptr;
                } else {  // push: my region p -> peer p's dst region d
                    a.src[q] = src[d] + (uint64_t)p * n;
                    a.dst[q] = dst[p] + (uint64_t)d * n;
                }
                if (mode == "ce_pull" || mode == "ce_push") {
                    cudaStream_t s = st[d * m + 1 + q];
                    RT(cudaStreamWaitEvent(s, e0[d], 0));
                    if (mode == "ce_pull") RT(cudaMemcpyAsync(dst[d] + (uint64_t)p * n, src[p] + (uint64_t)d * n, n, cudaMemcpyDeviceToDevice, s));
                    else RT(cudaMemcpyAsync(dst[p] + (uint64_t)d * n, src[d] + (uint64_t)p * n, n, cudaMemcpyDeviceToDevice, s));
                    cudaEvent_t j;
                    RT(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
                    RT(cudaEventRecord(j, s));
                    RT(cudaStreamWaitEvent(st[d * m], j, 0));
                    RT(cudaEventDestroy(j));
                }
            }
            if (mode == "xorpat4k" || mode == "xorpat16k") {  // needs m = 4; src[q] = peer staging base
                Args b = a;
                int q2 = 0;
                for (int p = 0; p < m; ++p)
                    if (p != d) b.src[q2++] = src[p];
                b.n = n;  // per peer: n bytes pulled; each peer's buffer holds n*m >= n*(m-1) bytes
                if (mode == "xorpat4k") {
                    RT(cudaFuncSetAttribute(xorpat_kernel<3, 4096, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 4 * 3 * 4096));
                    xorpat_kernel<3, 4096, 4, 4><<<ctas, 128, 4 * 4 * 3 * 4096, st[d * m]>>>(b, 65536, (uint32_t)d);
                } else {
                    RT(cudaFuncSetAttribute(xorpat_kernel<3, 16384, 4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 3 * 16384));
                    xorpat_kernel<3, 16384, 4, 1><<<ctas, 32, 4 * 3 * 16384, st[d * m]>>>(b, 65536, (uint32_t)d);
                }
            } else if (mode == "sm_pull" || mode == "sm_push" || mode == "sm_red")
                bulk_kernel<<<ctas, 32 * kW, kW * kNS * kT, st[d * m]>>>(a);
            else if (mode == "lsu_push")
                lsu_push_kernel<<<ctas, 256, 0, st[d * m]>>>(a);
            RT(cudaGetLastError());
            RT(cudaEventRecord(e1[d], st[d * m]));
        }
        double mn = 1e30, mx_ms = 0;
        for (int d = 0; d < m; ++d) {
            RT(cudaSetDevice(d));
            RT(cudaEventSynchronize(e1[d]));
            float ms = 0;
            RT(cudaEventElapsedTime(&ms, e0[d], e1[d]));
            const double gbs = (double)n * (m - 1) / (ms * 1e-3) / 1e9;
            best_dev[d] = std::max(best_dev[d], gbs);
            mn = std::min(mn, gbs);
            mx_ms = std::max(mx_ms, (double)ms);
        }
        best_min = std::max(best_min, mn);
        best_agg = std::max(best_agg, (double)n * (m - 1) * m / (mx_ms * 1e-3) / 1e9);
    }
    bool ok = true;
    if (red) {
        std::vector<uint64_t> after(chk / 8);
        RT(cudaSetDevice(1));
        RT(cudaMemcpy(after.data(), dst[1] + 0 * n, chk, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < after.size(); ++i)
            if (after[i] != (before[i] ^ srcv[i])) {
                ok = false;
                fprintf(stderr, "sm_red mismatch at word %zu\n", i);
                break;
            }
    }
    printf("{\"tool\": \"fabric_probe\", \"m\": %d, \"mode\": \"%s\", \"bytes_per_peer\": %llu, \"ctas\": %d, "
           "\"gbs_per_gpu_min\": %.1f, \"gbs_aggregate\": %.1f, \"gbs_per_gpu\": [",
           m, mode.c_str(), (unsigned long long)n, ctas, best_min, best_agg);
    for (int d = 0; d < m; ++d) printf("%s%.1f", d ? ", " : "", best_dev[d]);
    printf("], \"check\": \"%s\"}\n", red ? (ok ? "ok" : "FAIL") : "n/a");
    return ok ? 0 : 1;
}
