// ckpt_kernels.cu -- sm_100a kernels of libreft_ckpt (product code).
//
//  * pack/unpack: gather the registered tensors into a bucket of the packed image
//    (or scatter it back).  HBM-bound: 1 read + 1 write per state byte.  128-bit
//    LDG/STG with UNROLL independent loads in flight per thread; a funnel-shift path
//    keeps 128-bit stores when source and destination are misaligned mod 16 (bf16
//    views can start at any 2-byte offset).
//  * xor_gather: the AEC parity encode (Eq 1, P.476) and the rebuild
//    decode (Eq 2, P.483) as one kernel: every 16-byte output word is the XOR of up
//    to 8 input words, each from its own (possibly NVLink-peer) stream.  NVLink-bound
//    for the encode: (m-1) peer units in per parity unit out.
//
// No tensor cores: the path is pure data movement.
#include <algorithm>
#include <cstdlib>

#include "ckpt_kernels.cuh"

namespace reft {
namespace {

constexpr int kPackThreads = 512;
constexpr int kPackUnroll = 4;
constexpr int kXorThreads = 256;

__device__ __forceinline__ uint4 ld_stream(const void *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Coherent (non-.nc) 128-bit load, L2 only: used for peer slots, which are rewritten
// between launches by their owners.
__device__ __forceinline__ uint4 ld_cg(const void *p) {
    uint4 r;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_stream(void *p, const uint4 &v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// 16 bytes starting at byte `sh` (1..15) of the 32-byte pair (a, b).
__device__ __forceinline__ uint4 funnel16(const uint4 &a, const uint4 &b, uint32_t sh) {
    const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const uint32_t q = sh >> 2, bs = (sh & 3) * 8;
    uint4 o;
    // q is uniform per chunk; the selects compile to predicated moves, no local memory
    uint32_t v0 = q == 0 ? w[0] : q == 1 ? w[1] : q == 2 ? w[2] : w[3];
    uint32_t v1 = q == 0 ? w[1] : q == 1 ? w[2] : q == 2 ? w[3] : w[4];
    uint32_t v2 = q == 0 ? w[2] : q == 1 ? w[3] : q == 2 ? w[4] : w[5];
    uint32_t v3 = q == 0 ? w[3] : q == 1 ? w[4] : q == 2 ? w[5] : w[6];
    uint32_t v4 = q == 0 ? w[4] : q == 1 ? w[5] : q == 2 ? w[6] : w[7];
    o.x = __funnelshift_r(v0, v1, bs);
    o.y = __funnelshift_r(v1, v2, bs);
    o.z = __funnelshift_r(v2, v3, bs);
    o.w = __funnelshift_r(v3, v4, bs);
    return o;
}

// Block-cooperative copy of n bytes (any alignment).
__device__ __forceinline__ void block_copy(uint8_t *__restrict__ dst, const uint8_t *__restrict__ src,
                                           uint64_t n, uint32_t tid, uint32_t nt) {
    uint64_t head = (16 - ((uintptr_t)dst & 15)) & 15;
    if (head > n) head = n;
    if (tid < head) dst[tid] = src[tid];
    dst += head;
    src += head;
    n -= head;
    const uint64_t nw = n >> 4;
    uint4 *__restrict__ d4 = reinterpret_cast<uint4 *>(dst);
    const uint32_t sh = (uintptr_t)src & 15;
    if (sh == 0) {
        const uint4 *__restrict__ s4 = reinterpret_cast<const uint4 *>(src);
        uint64_t i = tid;
        for (; i + (kPackUnroll - 1) * nt < nw; i += kPackUnroll * nt) {
            uint4 v[kPackUnroll];
#pragma unroll
            for (int u = 0; u < kPackUnroll; ++u) v[u] = ld_stream(s4 + i + u * nt);
#pragma unroll
            for (int u = 0; u < kPackUnroll; ++u) st_stream(d4 + i + u * nt, v[u]);
        }
        for (; i < nw; i += nt) st_stream(d4 + i, ld_stream(s4 + i));
    } else {
        // aligned 16-byte source blocks a = floor16(src) + 16 i, b = a + 16; every block
        // read holds at least one byte of the source range, so it never crosses a page
        const uint4 *__restrict__ s4 = reinterpret_cast<const uint4 *>(src - sh);
        uint64_t i = tid;
        for (; i + (kPackUnroll - 1) * nt < nw; i += kPackUnroll * nt) {
            uint4 a[kPackUnroll], b[kPackUnroll];
#pragma unroll
            for (int u = 0; u < kPackUnroll; ++u) {
                a[u] = ld_stream(s4 + i + u * nt);
                b[u] = ld_stream(s4 + i + u * nt + 1);
            }
#pragma unroll
            for (int u = 0; u < kPackUnroll; ++u) st_stream(d4 + i + u * nt, funnel16(a[u], b[u], sh));
        }
        for (; i < nw; i += nt) st_stream(d4 + i, funnel16(ld_stream(s4 + i), ld_stream(s4 + i + 1), sh));
    }
    const uint64_t tail = n & 15, t0 = nw << 4;
    if (tid < tail) dst[t0 + tid] = src[t0 + tid];
}

__device__ __forceinline__ void block_zero(uint8_t *dst, uint64_t n, uint32_t tid, uint32_t nt) {
    uint64_t head = (16 - ((uintptr_t)dst & 15)) & 15;
    if (head > n) head = n;
    if (tid < head) dst[tid] = 0;
    dst += head;
    n -= head;
    const uint64_t nw = n >> 4;
    uint4 *d4 = reinterpret_cast<uint4 *>(dst);
    for (uint64_t i = tid; i < nw; i += nt) st_stream(d4 + i, make_uint4(0, 0, 0, 0));
    const uint64_t tail = n & 15, t0 = nw << 4;
    if (tid < tail) dst[t0 + tid] = 0;
}

// whole-CTA versions
__device__ __forceinline__ void block_copy(uint8_t *__restrict__ dst, const uint8_t *__restrict__ src, uint64_t n) {
    block_copy(dst, src, n, threadIdx.x, blockDim.x);
}
__device__ __forceinline__ void block_zero(uint8_t *dst, uint64_t n) { block_zero(dst, n, threadIdx.x, blockDim.x); }

// This CTA's share of the bucket: tiles split evenly over gridDim.x, then mapped to
// the contiguous chunk index range [c_begin, c_end).
__device__ __forceinline__ void cta_chunk_range(const PackArgs &a, uint64_t &c_begin, uint64_t &c_end) {
    const uint64_t t_lo = a.bucket_begin / kTile;
    const uint64_t t_hi = (a.bucket_end + kTile - 1) / kTile;
    const uint64_t nt = t_hi - t_lo, g = gridDim.x, b = blockIdx.x;
    const uint64_t q = nt / g, r = nt % g;
    const uint64_t ta = t_lo + b * q + (b < r ? b : r);
    const uint64_t tb = ta + q + (b < r ? 1 : 0);
    c_begin = a.tile_first[ta];
    c_end = a.tile_first[tb];
}

// Clip chunk c to the bucket; returns bytes (0 = nothing) and the from/to addresses.
__device__ __forceinline__ uint64_t clip_chunk(const PackArgs &a, const PackChunk &ch, const uint8_t *&from,
                                               uint8_t *&to) {
    const uint64_t lo = ch.dst > a.bucket_begin ? ch.dst : a.bucket_begin;
    const uint64_t end = ch.dst + ch.nbytes;
    const uint64_t hi = end < a.bucket_end ? end : a.bucket_end;
    if (lo >= hi) return 0;
    uint8_t *slot = a.slot + (lo - a.bucket_begin);
    if (ch.src == 0) {  // zero gap: written on pack, skipped on unpack
        from = nullptr;
        to = a.unpack ? nullptr : slot;
        return a.unpack ? 0 : hi - lo;
    }
    uint8_t *tensor = reinterpret_cast<uint8_t *>(ch.src) + (lo - ch.dst);
    from = a.unpack ? slot : tensor;
    to = a.unpack ? tensor : slot;
    return hi - lo;
}

// LSU pack.  The CTA stages up to kBatch chunk descriptors in SMEM, then streams the
// 16-byte words of all 16-B-aligned chunks of the batch as ONE flat index space, so
// every thread keeps kPackUnroll independent 128-bit loads in flight across chunk
// boundaries (chunks are <= 16 KiB).  Unaligned chunks (views misaligned mod 16,
// odd-sized tails, small gaps) take the block-cooperative funnel-shift path.
constexpr int kBatch = 128;

// Flat copy of the chunks [cb, ce) (clipped to a's bucket): descriptors staged in
// SMEM by batches of kBatch, the 16-B-aligned chunks streamed as one flat word space.
__device__ __forceinline__ void copy_chunks(const PackArgs &a, uint64_t cb, uint64_t ce) {
    __shared__ const uint8_t *s_from[kBatch];
    __shared__ uint8_t *s_to[kBatch];
    __shared__ uint64_t s_n[kBatch];
    __shared__ uint32_t s_pre[kBatch + 1];
    __shared__ uint32_t s_nslow;
    __shared__ uint8_t s_slow[kBatch];
    const uint32_t tid = threadIdx.x, nt = blockDim.x;
    for (uint64_t c0 = cb; c0 < ce; c0 += kBatch) {
        const uint32_t nb = (uint32_t)((ce - c0) < kBatch ? (ce - c0) : kBatch);
        if (tid == 0) s_nslow = 0;
        __syncthreads();
        if (tid < nb) {
            const uint8_t *from;
            uint8_t *to;
            const uint64_t n = clip_chunk(a, a.chunks[c0 + tid], from, to);
            const bool vec = n && ((((uintptr_t)from | (uintptr_t)to | n) & 15) == 0);
            s_from[tid] = from;
            s_to[tid] = to;
            s_n[tid] = n;
            s_pre[tid + 1] = vec ? (uint32_t)(n >> 4) : 0;
            if (n && !vec) s_slow[atomicAdd(&s_nslow, 1u)] = (uint8_t)tid;
        }
        __syncthreads();
        if (tid == 0) {
            s_pre[0] = 0;
            for (uint32_t i = 1; i <= nb; ++i) s_pre[i] += s_pre[i - 1];
        }
        __syncthreads();
        const uint32_t total = s_pre[nb];
        uint32_t k = 0;  // per-thread chunk cursor (word indices only grow)
        for (uint32_t base = 0; base < total; base += nt * kPackUnroll) {
            uint4 v[kPackUnroll];
            uint4 *dst[kPackUnroll];
#pragma unroll
            for (int u = 0; u < kPackUnroll; ++u) {
                const uint32_t w = base + u * nt + tid;
                dst[u] = nullptr;
                if (w < total) {
                    while (s_pre[k + 1] <= w) ++k;
                    const uint32_t off = w - s_pre[k];
                    const uint8_t *f = s_from[k];
                    dst[u] = reinterpret_cast<uint4 *>(s_to[k]) + off;
                    v[u] = f ? ld_stream(reinterpret_cast<const uint4 *>(f) + off) : make_uint4(0, 0, 0, 0);
                }
            }
#pragma unroll
            for (int u = 0; u < kPackUnroll; ++u)
                if (dst[u]) st_stream(dst[u], v[u]);
        }
        for (uint32_t i = 0; i < s_nslow; ++i) {
            const uint32_t j = s_slow[i];
            if (s_from[j])
                block_copy(s_to[j], s_from[j], s_n[j]);
            else
                block_zero(s_to[j], s_n[j]);
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kPackThreads, 2) pack_kernel(const PackArgs a) {
    uint64_t cb, ce;
    cta_chunk_range(a, cb, ce);
    copy_chunks(a, cb, ce);
}

__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Publish bucket k: count this CTA's `cnt` finished groups; the CTA completing the
// bucket stores its flag (release, system scope) locally and into every peer's page.
__device__ __noinline__ void publish_bucket(const PackAllArgs &g, uint32_t k, uint32_t cnt, uint32_t need) {
    if (g.unpack) return;
    // this CTA's stores (ordered by the preceding barrier) before the count: acq_rel at
    // gpu scope is enough here (__threadfence is the heavier fence.sc)
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (atomicAdd(&g.counters[k], cnt) + cnt == need) {
        const uint32_t v = g.seq_base + k + 1;
        const uint32_t i = v % g.maxb;
        st_release_sys(g.ready_local + i, v);
        for (int p = 0; p < g.npeers; ++p) st_release_sys(g.ready_peer[p] + i, v);
    }
}

__global__ void __launch_bounds__(kPackThreads, 2) pack_all_kernel(const __grid_constant__ PackAllArgs g) {
    PackArgs a;
    a.chunks = g.chunks;
    a.tile_first = g.tile_first;
    a.bucket_begin = 0;
    a.bucket_end = g.L;
    a.slot = g.image;
    a.unpack = g.unpack;
    const uint32_t ntiles = (uint32_t)((g.L + kTile - 1) / kTile);
    const uint32_t ngroups = (uint32_t)((g.L + kGroup - 1) / kGroup);
    const uint32_t gpb = (uint32_t)(g.bucket / kGroup);  // groups per bucket
    constexpr uint32_t tpg = (uint32_t)(kGroup / kTile);
    // Completion accounting batched per bucket: a CTA's groups of bucket k are consecutive
    // in its walk, so it publishes once per bucket it touched.
    uint32_t cur = 0, pending = 0;
    for (uint32_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const uint32_t k = grp / gpb;
        if (threadIdx.x == 0 && pending && k != cur) {
            publish_bucket(g, cur, pending, min(gpb, ngroups - cur * gpb));
            pending = 0;
        }
        cur = k;
        const uint32_t t0 = grp * tpg;
        const uint32_t t1 = t0 + tpg < ntiles ? t0 + tpg : ntiles;
        copy_chunks(a, g.tile_first[t0], g.tile_first[t1]);  // ends with __syncthreads()
        ++pending;
    }
    if (threadIdx.x == 0 && pending) publish_bucket(g, cur, pending, min(gpb, ngroups - cur * gpb));
}

// ---------------------------------------------------------------------------------
// TMA pack: 1-D bulk copies (cp.async.bulk) global -> SMEM -> global issued by one
// thread per CTA, kTmaStages stages of kTmaStage bytes in flight.  A 32-thread CTA
// with 64 KiB of SMEM moves as many bytes per SM as the 512-thread LSU kernel while
// holding 16x fewer threads/registers -- the low-SM-footprint variant for co-running
// with a training GEMM.  Chunks whose source and destination differ mod 16 (and the
// < 16-byte heads/tails) go through the warp's LSU path.
constexpr int kTmaThreads = 32;
constexpr int kTmaStages = 4;
constexpr uint32_t kTmaStage = 16 * 1024;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *smem, const void *gmem, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(smem)),
        "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *gmem, const void *smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem), "r"(smem_u32(smem)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_read_n(uint32_t n) {
    switch (n) {
        case 0: bulk_wait_read<0>(); break;
        case 1: bulk_wait_read<1>(); break;
        case 2: bulk_wait_read<2>(); break;
        case 3: bulk_wait_read<3>(); break;
        case 4: bulk_wait_read<4>(); break;
        case 5: bulk_wait_read<5>(); break;
        case 6: bulk_wait_read<6>(); break;
        default: bulk_wait_read<7>(); break;
    }
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// One bulk piece: up to kTmaStage bytes of one chunk body.
struct Piece {
    const uint8_t *src;
    uint8_t *dst;
    uint32_t bytes;
};

__global__ void __launch_bounds__(kTmaThreads) pack_tma_kernel(const PackArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[kTmaStages];
    const uint32_t lane = threadIdx.x;
    if (lane == 0) {
        for (int i = 0; i < kTmaStages; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    uint32_t phase = 0;      // bit i = parity to wait for on stage i
    uint32_t issued = 0, done = 0;  // pieces loaded / stored (lane 0 only)
    Piece ring[kTmaStages];
    uint64_t cb, ce;
    cta_chunk_range(a, cb, ce);
    for (uint64_t c = cb; c < ce; ++c) {
        const uint8_t *src;
        uint8_t *dst;
        const uint64_t n = clip_chunk(a, a.chunks[c], src, dst);
        if (n == 0) continue;
        if (!src) {
            block_zero(dst, n);
            continue;
        }
        if ((((uintptr_t)dst ^ (uintptr_t)src) & 15) || n < 64) {
            block_copy(dst, src, n);
            continue;
        }
        uint64_t head = (16 - ((uintptr_t)dst & 15)) & 15;
        uint64_t body = (n - head) & ~(uint64_t)15;
        uint64_t tail = n - head - body;
        if (lane < head) dst[lane] = src[lane];
        if (lane < tail) dst[head + body + lane] = src[head + body + lane];
        if (lane == 0) {
            const uint8_t *s = src + head;
            uint8_t *d = dst + head;
            for (uint64_t o = 0; o < body;) {
                const uint32_t bytes = (uint32_t)((body - o) < kTmaStage ? (body - o) : kTmaStage);
                // at most kTmaStages-1 loads in flight: retire the oldest (wait for its
                // load, issue its store) so one store can drain while the next loads fly
                if (issued - done == kTmaStages - 1) {
                    const uint32_t so = done % kTmaStages;
                    mbar_wait(&bars[so], (phase >> so) & 1);
                    phase ^= 1u << so;
                    bulk_s2g(ring[so].dst, smem + so * kTmaStage, ring[so].bytes);
                    bulk_commit();
                    ++done;
                }
                const uint32_t st = issued % kTmaStages;
                // the store of piece issued-kTmaStages (same stage) must have finished
                // reading SMEM; stores committed after it may stay in flight
                if (issued >= kTmaStages) bulk_wait_read_n(done + kTmaStages - 1 - issued);
                ring[st] = Piece{s + o, d + o, bytes};
                mbar_expect_tx(&bars[st], bytes);
                bulk_g2s(smem + st * kTmaStage, s + o, bytes, &bars[st]);
                ++issued;
                o += bytes;
            }
        }
    }
    if (lane == 0) {
        while (done < issued) {
            const uint32_t st = done % kTmaStages;
            mbar_wait(&bars[st], (phase >> st) & 1);
            phase ^= 1u << st;
            bulk_s2g(ring[st].dst, smem + st * kTmaStage, ring[st].bytes);
            bulk_commit();
            ++done;
        }
        bulk_wait_all();
    }
    __syncwarp();
}


// ---------------------------------------------------------------------------------
// TMA single-launch pack.  One elected lane per CTA drives a ring of NS SMEM stages of
// up to 16 KiB: bulk loads (cp.async.bulk G->S, mbarrier complete_tx) run NS-1 deep and
// every retired stage is written back with a bulk store (S->G, bulk_group).  A 32-thread
// CTA keeps ~(NS-1) x 16 KiB in flight -- several times the LSU kernel's bytes per SM,
// so the same HBM bandwidth costs fewer SM-seconds (the co-running GEMM loses less).
// Bucket publication as in pack_all_kernel, after draining the CTA's bulk stores and a
// proxy fence (async-proxy writes before the generic-proxy flag store).
template <int NS>
struct BulkRing {
    uint8_t *smem;
    uint64_t *bars;
    uint32_t phase, issued, done;
    Piece ring[NS];
    __device__ __forceinline__ void retire() {
        const uint32_t so = done % NS;
        mbar_wait(&bars[so], (phase >> so) & 1);
        phase ^= 1u << so;
        bulk_s2g(ring[so].dst, smem + so * kTmaStage, ring[so].bytes);
        bulk_commit();
        ++done;
    }
    __device__ __forceinline__ void push(const uint8_t *s, uint8_t *d, uint32_t bytes) {
        if (issued - done == NS - 1) retire();
        const uint32_t st = issued % NS;
        if (issued >= NS) bulk_wait_read_n(done + NS - 1 - issued);
        ring[st] = Piece{s, d, bytes};
        mbar_expect_tx(&bars[st], bytes);
        bulk_g2s(smem + st * kTmaStage, s, bytes, &bars[st]);
        ++issued;
    }
    __device__ __forceinline__ void drain() {
        while (done < issued) retire();
        bulk_wait_all();
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
};

template <int NS, int W>
__global__ void __launch_bounds__(32 * W) pack_all_tma_kernel(const __grid_constant__ PackAllArgs g) {
    // W warps, each an independent producer with its own ring of NS SMEM stages: a CTA
    // keeps W x (NS-1) x 16 KiB of bulk loads in flight, so a few dozen SMs saturate HBM
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[W][NS];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    BulkRing<NS> R;
    R.smem = smem + (size_t)w * NS * kTmaStage;
    R.bars = bars[w];
    R.phase = R.issued = R.done = 0;
    if (lane == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&bars[w][i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    PackArgs a;
    a.chunks = g.chunks;
    a.tile_first = g.tile_first;
    a.bucket_begin = 0;
    a.bucket_end = g.L;
    a.slot = g.image;
    a.unpack = g.unpack;
    const uint32_t ntiles = (uint32_t)((g.L + kTile - 1) / kTile);
    const uint32_t ngroups = (uint32_t)((g.L + kGroup - 1) / kGroup);
    const uint32_t gpb = (uint32_t)(g.bucket / kGroup);
    constexpr uint32_t tpg = (uint32_t)(kGroup / kTile);
    uint32_t cur = 0, pending = 0;
    for (uint32_t grp = blockIdx.x * W + w; grp < ngroups; grp += gridDim.x * W) {
        const uint32_t k = grp / gpb;
        if (pending && k != cur) {
            __syncwarp();
            if (lane == 0) {
                R.drain();
                publish_bucket(g, cur, pending, min(gpb, ngroups - cur * gpb));
            }
            pending = 0;
        }
        cur = k;
        const uint32_t t0 = grp * tpg;
        const uint32_t t1 = t0 + tpg < ntiles ? t0 + tpg : ntiles;
        const uint32_t cb = g.tile_first[t0], ce = g.tile_first[t1];
        for (uint32_t c = cb; c < ce; ++c) {
            const uint8_t *src;
            uint8_t *dst;
            const uint64_t n = clip_chunk(a, g.chunks[c], src, dst);
            if (n == 0) continue;
            if (!src) {
                block_zero(dst, n, lane, 32);
                continue;
            }
            if ((((uintptr_t)dst ^ (uintptr_t)src) & 15) || n < 64) {
                block_copy(dst, src, n, lane, 32);
                continue;
            }
            const uint64_t head = (16 - ((uintptr_t)dst & 15)) & 15;
            const uint64_t body = (n - head) & ~(uint64_t)15;
            const uint64_t tail = n - head - body;
            if (lane < head) dst[lane] = src[lane];
            if (lane < tail) dst[head + body + lane] = src[head + body + lane];
            if (lane == 0)  // chunks never exceed a 16 KiB tile: one stage each
                R.push(src + head, dst + head, (uint32_t)body);
        }
        ++pending;
    }
    __syncwarp();
    if (lane == 0) {
        R.drain();
        if (pending) publish_bucket(g, cur, pending, min(gpb, ngroups - cur * gpb));
    }
}

// ---------------------------------------------------------------------------------
// XOR gather.  Work is split into tiles of kXorThreads * U 16-byte words
// inside one unit, so the stripe index needs one 32-bit division per tile.
// NIN input streams, U words per thread per tile: NIN * U independent 128-bit loads in
// flight per thread (8..14), enough to cover NVLink latency (~2 us) for any m.
template <int NIN, int U>
__global__ void __launch_bounds__(kXorThreads) xor_kernel(const XorArgs a) {
    const uint32_t words_per_unit = (uint32_t)(a.unit >> 4);
    constexpr uint32_t kTileW = kXorThreads * U;
    const uint32_t tiles_per_unit = (words_per_unit + kTileW - 1) / kTileW;
    const uint64_t ntiles = a.nstripes * tiles_per_unit;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t s = t / tiles_per_unit;
        const uint32_t w0 = (uint32_t)(t - s * tiles_per_unit) * kTileW + threadIdx.x;
        uint4 v[NIN][U];
#pragma unroll
        for (int k = 0; k < NIN; ++k) {
            const uint64_t base = s * a.in[k].stride + a.in[k].off;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t w = w0 + u * kXorThreads;
                const uint64_t pos = base + ((uint64_t)w << 4);
                v[k][u] = (w < words_per_unit && pos < a.in[k].valid) ? ld_cg(a.in[k].base + pos)
                                                                       : make_uint4(0, 0, 0, 0);
            }
        }
        const uint64_t obase = s * a.out_stride + a.out_off;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            uint4 acc = v[0][u];
#pragma unroll
            for (int k = 1; k < NIN; ++k) {
                acc.x ^= v[k][u].x;
                acc.y ^= v[k][u].y;
                acc.z ^= v[k][u].z;
                acc.w ^= v[k][u].w;
            }
            const uint32_t w = w0 + u * kXorThreads;
            const uint64_t pos = obase + ((uint64_t)w << 4);
            if (w < words_per_unit && pos < a.out_valid) *reinterpret_cast<uint4 *>(a.out + pos) = acc;
        }
    }
}

template <int N>
constexpr int xor_unroll() { return N == 1 ? 8 : N == 2 ? 4 : N == 3 ? 3 : 2; }

// ---------------------------------------------------------------------------------
// TMA XOR gather.  Same contract as xor_kernel.  W warps per CTA (one CTA per SM), each an
// independent pipeline over tiles of T bytes of one unit: lane 0 loads the NIN input
// segments of a tile with cp.async.bulk (peer staging over NVLink for the encode; an
// mbarrier counts the bytes) into one of NS SMEM stages, the 32 lanes XOR the segments out
// of SMEM and store the result with 128-bit stores.  Each warp keeps NS tiles = NS*NIN*T
// bytes of peer reads in flight (~48 KiB, ~190 KiB per SM) with one instruction per
// segment instead of one per 16 B.  Segments past an input's `valid` are not loaded and
// read as zero (reading Q5).
// Tile T, NS stages, W = 4 warps per CTA: NS * NIN * T <= 48 KiB per warp.  Round-2 A/B
// (tools/r02_xor_ab.sh, m = 4, C2): 16 KiB pieces on 1-2 warps per CTA moved the same
// 606-614 GB/s as these 4 KiB pieces on 4 warps (611-614), and 64 CTAs the same as 32.
template <int NIN>
struct XorTmaCfg {
    static constexpr uint32_t T = NIN == 1 ? 16384 : NIN == 2 ? 8192 : NIN <= 4 ? 4096 : 2048;
    static constexpr int NS = (int)((48u * 1024u) / (T * NIN)) > 6 ? 6 : (int)((48u * 1024u) / (T * NIN));
    static constexpr int W = 4;
    static constexpr int smem = W * NS * NIN * (int)T;
};

template <int NIN>
__device__ __forceinline__ void xor_tile_geometry(const XorArgs &a, uint64_t t, uint64_t tpu, uint32_t T,
                                                  uint64_t &s, uint64_t &uoff, uint32_t &len, uint32_t (&n)[NIN],
                                                  uint64_t (&pos)[NIN]) {
    s = t / tpu;
    uoff = (t - s * tpu) * T;
    len = (uint32_t)((a.unit - uoff) < T ? (a.unit - uoff) : T);
#pragma unroll
    for (int k = 0; k < NIN; ++k) {
        pos[k] = s * a.in[k].stride + a.in[k].off + uoff;
        const uint64_t v = a.in[k].valid;
        n[k] = pos[k] >= v ? 0u : (uint32_t)((v - pos[k]) < len ? (v - pos[k]) : len);
    }
}

template <int NIN>
__global__ void __launch_bounds__(32 * XorTmaCfg<NIN>::W) xor_tma_kernel(const __grid_constant__ XorArgs a) {
    using Cfg = XorTmaCfg<NIN>;
    constexpr uint32_t T = Cfg::T;
    constexpr int NS = Cfg::NS, W = Cfg::W;
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[W][NS];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint8_t *ring = smem + (size_t)w * NS * NIN * T;
    if (lane == 0) {
        for (int i = 0; i < NS; ++i) mbar_init(&bars[w][i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    const uint64_t tpu = (a.unit + T - 1) / T;
    const uint64_t ntiles = a.nstripes * tpu;
    const uint64_t step = (uint64_t)gridDim.x * W;
    auto issue = [&](uint64_t t, int st) {  // lane 0 only
        uint64_t s, uoff;
        uint32_t len, n[NIN];
        uint64_t pos[NIN];
        xor_tile_geometry<NIN>(a, t, tpu, T, s, uoff, len, n, pos);
        uint32_t total = 0;
#pragma unroll
        for (int k = 0; k < NIN; ++k) total += n[k];
        mbar_expect_tx(&bars[w][st], total);  // total = 0 completes the phase at once
#pragma unroll
        for (int k = 0; k < NIN; ++k)
            if (n[k]) bulk_g2s(ring + ((size_t)st * NIN + k) * T, a.in[k].base + pos[k], n[k], &bars[w][st]);
    };
    uint64_t t_issue = (uint64_t)blockIdx.x * W + w, t = t_issue;
    if (lane == 0)
        for (int i = 0; i < NS && t_issue < ntiles; ++i, t_issue += step) issue(t_issue, i);
    t_issue = t + (uint64_t)NS * step;  // every lane tracks the issue cursor
    uint32_t phase = 0;
    for (int st = 0; t < ntiles; t += step, st = (st + 1 == NS) ? 0 : st + 1) {
        uint64_t s, uoff;
        uint32_t len, n[NIN];
        uint64_t pos[NIN];
        xor_tile_geometry<NIN>(a, t, tpu, T, s, uoff, len, n, pos);
        mbar_wait(&bars[w][st], (phase >> st) & 1);
        phase ^= 1u << st;
        const uint4 *seg = reinterpret_cast<const uint4 *>(ring + (size_t)st * NIN * T);
        const uint64_t obase = s * a.out_stride + a.out_off + uoff;
        for (uint32_t i = lane; i < (len >> 4); i += 32) {
            uint4 acc = make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int k = 0; k < NIN; ++k) {
                if ((i << 4) < n[k]) {
                    const uint4 v = seg[(size_t)k * (T >> 4) + i];
                    acc.x ^= v.x;
                    acc.y ^= v.y;
                    acc.z ^= v.z;
                    acc.w ^= v.w;
                }
            }
            const uint64_t o = obase + ((uint64_t)i << 4);
            if (o < a.out_valid) *reinterpret_cast<uint4 *>(a.out + o) = acc;
        }
        __syncwarp();  // every lane is done reading stage st
        if (lane == 0 && t_issue < ntiles) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(t_issue, st);
        }
        t_issue += step;
    }
}

template <int N>
cudaError_t launch_xor_n(const XorArgs &a, int max_ctas, cudaStream_t s) {
    constexpr int U = xor_unroll<N>();
    const uint64_t wpu = a.unit >> 4;
    const uint64_t tpu = (wpu + kXorThreads * U - 1) / (kXorThreads * U);
    const uint64_t ntiles = a.nstripes * tpu;
    const int grid = (int)(ntiles < (uint64_t)max_ctas ? ntiles : (uint64_t)max_ctas);
    xor_kernel<N, U><<<grid, kXorThreads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int N>
cudaError_t launch_xor_tma_n(const XorArgs &a, int ctas, cudaStream_t s) {
    using Cfg = XorTmaCfg<N>;
    static unsigned long long attr_set = 0;  // bit d: attribute set on device d
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set & (1ull << dev))) {
        cudaError_t e = cudaFuncSetAttribute(xor_tma_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::smem);
        if (e != cudaSuccess) return e;
        attr_set |= 1ull << dev;
    }
    const uint64_t ntiles = a.nstripes * ((a.unit + Cfg::T - 1) / Cfg::T);
    const uint64_t need = (ntiles + Cfg::W - 1) / Cfg::W;
    const int grid = (int)(need < (uint64_t)ctas ? need : (uint64_t)ctas);
    xor_tma_kernel<N><<<grid, 32 * Cfg::W, Cfg::smem, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------
// Fabric probe (ckpt_probe_fabric): the load side of xor_tma_kernel alone -- W warps per
// CTA, lane 0 of each keeps NS 16 KiB cp.async.bulk loads in flight, pieces interleaved
// over the peers; nothing is stored.
constexpr int kProbeW = 4, kProbeNS = 3;
constexpr uint32_t kProbeT = 16384;

__global__ void __launch_bounds__(32 * kProbeW) probe_pull_kernel(const __grid_constant__ ProbeArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[kProbeW][kProbeNS];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane) return;
    uint8_t *ring = smem + (size_t)w * kProbeNS * kProbeT;
    for (int i = 0; i < kProbeNS; ++i) mbar_init(&bars[w][i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint64_t items = a.n / kProbeT * a.npeers, step = (uint64_t)gridDim.x * kProbeW;
    const uint64_t first = (uint64_t)blockIdx.x * kProbeW + w;
    int k = 0;
    for (uint64_t it = first; it < items && k < kProbeNS; it += step, ++k) {
        mbar_expect_tx(&bars[w][k], kProbeT);
        bulk_g2s(ring + (size_t)k * kProbeT, a.src[it % a.npeers] + (it / a.npeers) * kProbeT, kProbeT, &bars[w][k]);
    }
    uint32_t phase = 0;
    int st = 0;
    for (uint64_t it = first; it < items; it += step) {
        mbar_wait(&bars[w][st], (phase >> st) & 1);
        phase ^= 1u << st;
        const uint64_t nx = it + (uint64_t)kProbeNS * step;
        if (nx < items) {
            mbar_expect_tx(&bars[w][st], kProbeT);
            bulk_g2s(ring + (size_t)st * kProbeT, a.src[nx % a.npeers] + (nx / a.npeers) * kProbeT, kProbeT, &bars[w][st]);
        }
        st = st + 1 == kProbeNS ? 0 : st + 1;
    }
}

// ---------------------------------------------------------------------------------
// Push-mode XOR encode (XorPushArgs).  W warps per CTA; lane 0 of each runs a pipeline over
// tiles of T bytes of the image in order: cp.async.bulk G->S of the tile from local
// staging (mbarrier), then ONE cp.reduce.async.bulk .xor.b64 S->G into the row owner's
// parity (over NVLink for a peer), committed as a bulk group; a stage is refilled once the
// previous tile's reduction has read it (wait_group.read 1), so NS-1 loads and up to two
// reductions are in flight per warp.  The warp waits for full completion of its reductions
// before it exits: kernel completion then means every XOR has been performed at the row
// owners (the REL signal that follows on the stream publishes it).
constexpr int kPushW = 4, kPushNS = 3;
constexpr uint32_t kPushT = 16384;

__device__ __forceinline__ void bulk_s2g_xor(void *gmem, const void *smem, uint32_t bytes) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.xor.b64 [%0], [%1], %2;" ::"l"(gmem),
                 "r"(smem_u32(smem)), "r"(bytes)
                 : "memory");
}

__global__ void __launch_bounds__(32 * kPushW) xor_push_kernel(const __grid_constant__ XorPushArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ __align__(8) uint64_t bars[kPushW][kPushNS];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane) return;
    uint8_t *ring = smem + (size_t)w * kPushNS * kPushT;
    for (int i = 0; i < kPushNS; ++i) mbar_init(&bars[w][i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint64_t u = a.unit, T = u < kPushT ? u : kPushT;
    const uint64_t tpu = (u + T - 1) / T;
    const uint64_t rem = a.L % u;
    // tiles in image order; tile offsets grow monotonically, so those below L are a prefix
    const uint64_t items = a.L / u * tpu + (rem + T - 1) / T;
    const uint64_t step = (uint64_t)gridDim.x * kPushW;
    const uint32_t n1 = a.m - 1;
    auto geom = [&](uint64_t it, uint64_t &o, uint32_t &len) {
        const uint64_t q = it / tpu, t = it - q * tpu;
        o = q * u + t * T;
        uint64_t l = u - t * T < T ? u - t * T : T;
        if (o + l > a.L) l = a.L - o;
        len = (uint32_t)l;
    };
    auto load = [&](uint64_t it, int st) {
        uint64_t o;
        uint32_t len;
        geom(it, o, len);
        mbar_expect_tx(&bars[w][st], len);
        bulk_g2s(ring + (size_t)st * kPushT, a.src + o, len, &bars[w][st]);
    };
    const uint64_t first = (uint64_t)blockIdx.x * kPushW + w;
    int k = 0;
    for (uint64_t it = first; it < items && k < kPushNS; it += step, ++k) load(it, k);
    uint32_t phase = 0;
    int st = 0, prev_st = 0;
    uint64_t prev = UINT64_MAX;
    for (uint64_t it = first; it < items; it += step) {
        uint64_t o;
        uint32_t len;
        geom(it, o, len);
        const uint64_t q = o / u, s = q / n1;
        const uint32_t i = (uint32_t)(q - s * n1);
        const uint32_t r = i < a.me ? i : i + 1;  // sigma(r, me) = i
        mbar_wait(&bars[w][st], (phase >> st) & 1);
        phase ^= 1u << st;
        bulk_s2g_xor(a.dst[r] + s * u + (o - q * u), ring + (size_t)st * kPushT, len);
        bulk_commit();
        if (prev != UINT64_MAX) {
            bulk_wait_read<1>();  // the previous tile's reduction has read its stage
            const uint64_t nx = prev + (uint64_t)kPushNS * step;
            if (nx < items) load(nx, prev_st);
        }
        prev = it;
        prev_st = st;
        st = st + 1 == kPushNS ? 0 : st + 1;
    }
    bulk_wait_all();
}


}  // namespace

template <int NS, int W>
static cudaError_t launch_pack_all_tma(const PackAllArgs &a, uint64_t ngroups, int ctas, cudaStream_t s) {
    static unsigned long long attr_set = 0;  // bit d: attribute set on device d
    const int smem = NS * W * kTmaStage;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set & (1ull << dev))) {
        cudaError_t e = cudaFuncSetAttribute(pack_all_tma_kernel<NS, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_set |= 1ull << dev;
    }
    const uint64_t need = (ngroups + W - 1) / W;
    const uint64_t g = need < (uint64_t)ctas ? need : (uint64_t)ctas;
    pack_all_tma_kernel<NS, W><<<(unsigned)g, 32 * W, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_pack_all(const PackAllArgs &a, int max_ctas, cudaStream_t s, bool tma) {
    const uint64_t ngroups = (a.L + kGroup - 1) / kGroup;
    if (ngroups == 0) return cudaSuccess;
    if (tma) {
        // one CTA per SM (192 KiB of SMEM) on max_ctas/2 SMs: 4 producer warps x 3 stages
        // Short-lived CTAs (k per SM in the grid) beat one persistent CTA per SM in the step
        // (C2 rank, D2H running): k = 1: 5.74-5.86 TB/s, k = 8: 5.76-5.95, k = 16: 5.91,
        // k = 32: 6.25, k = 64: 6.44-6.50 TB/s.  They also hurt a co-running GEMM LESS: a
        // CTA holds its SM for ~pack/k, and the GEMM's next kernel waits for it, so the
        // GEMMs overlapping the pack run 55% / 26% / 15% / 11% slower at k = 8 / 16 / 32 /
        // 64 (round 2, 12 ABBA pairs, profiles/r02/r02f_waves*.jsonl; round 1's opposite
        // reading was within the whole-window noise).  k = 64 for the snapshot and the
        // unpack of a load; CKPT_PACK_WAVES=k overrides both.
        static int waves_env = -1;
        if (waves_env < 0) {
            const char *e = getenv("CKPT_PACK_WAVES");
            waves_env = e ? std::max(1, atoi(e)) : 0;
        }
        const int waves = waves_env ? waves_env : 64;
        const int ctas = (max_ctas / 2 > 0 ? max_ctas / 2 : 1) * waves;
        return launch_pack_all_tma<3, 4>(a, ngroups, ctas, s);
    }
    const uint64_t g = ngroups < (uint64_t)max_ctas ? ngroups : (uint64_t)max_ctas;
    pack_all_kernel<<<(unsigned)g, kPackThreads, 0, s>>>(a);
    return cudaGetLastError();
}

// CUDA lazy loading would load each kernel at its first launch, and loading can wait for
// work in flight on the device (e.g. a background D2H); load them all up front instead.
cudaError_t preload_kernels() {
    cudaFuncAttributes fa;
    const void *fns[] = {
        (const void *)pack_kernel, (const void *)pack_all_kernel, (const void *)pack_tma_kernel,
        (const void *)pack_all_tma_kernel<3, 4>,
        (const void *)xor_kernel<1, xor_unroll<1>()>, (const void *)xor_kernel<2, xor_unroll<2>()>,
        (const void *)xor_kernel<3, xor_unroll<3>()>, (const void *)xor_kernel<4, xor_unroll<4>()>,
        (const void *)xor_kernel<5, xor_unroll<5>()>, (const void *)xor_kernel<6, xor_unroll<6>()>,
        (const void *)xor_kernel<7, xor_unroll<7>()>, (const void *)xor_kernel<8, xor_unroll<8>()>,
        (const void *)xor_tma_kernel<1>, (const void *)xor_tma_kernel<2>, (const void *)xor_tma_kernel<3>,
        (const void *)xor_tma_kernel<4>, (const void *)xor_tma_kernel<5>, (const void *)xor_tma_kernel<6>,
        (const void *)xor_tma_kernel<7>, (const void *)xor_tma_kernel<8>,
        (const void *)probe_pull_kernel, (const void *)xor_push_kernel};
    for (const void *f : fns) {
        cudaError_t e = cudaFuncGetAttributes(&fa, f);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_probe_pull(const ProbeArgs &a, int ctas, cudaStream_t s) {
    const int smem = kProbeW * kProbeNS * (int)kProbeT;
    cudaError_t e = cudaFuncSetAttribute(probe_pull_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    probe_pull_kernel<<<ctas, 32 * kProbeW, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_xor_push(const XorPushArgs &a, int ctas, cudaStream_t s) {
    if (a.m < 2 || a.m > kMaxTerms + 1 || (a.unit & 15) || a.unit == 0 || (a.L & 15) || ((uintptr_t)a.src & 15))
        return cudaErrorInvalidValue;
    if (a.L == 0) return cudaSuccess;
    static unsigned long long attr_set = 0;  // bit d: attribute set on device d
    const int smem = kPushW * kPushNS * (int)kPushT;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(attr_set & (1ull << dev))) {
        cudaError_t e = cudaFuncSetAttribute(xor_push_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_set |= 1ull << dev;
    }
    xor_push_kernel<<<ctas, 32 * kPushW, smem, s>>>(a);
    return cudaGetLastError();
}


cudaError_t launch_pack(const PackArgs &a, int max_ctas, cudaStream_t s, bool tma) {
    if (a.bucket_end <= a.bucket_begin) return cudaSuccess;
    const uint64_t ntiles = (a.bucket_end + kTile - 1) / kTile - a.bucket_begin / kTile;
    if (tma) {
        static unsigned long long attr_set = 0;  // bit d: attribute set on device d
        const int smem = kTmaStages * kTmaStage;
        int dev = 0;
        cudaGetDevice(&dev);
        if (!(attr_set & (1ull << dev))) {
            cudaError_t e = cudaFuncSetAttribute(pack_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
            attr_set |= 1ull << dev;
        }
        // 3 CTAs of 64 KiB SMEM per SM: 1.5x the LSU CTA budget
        const uint64_t cap = (uint64_t)max_ctas * 3 / 2;
        const uint64_t g = ntiles < cap ? ntiles : cap;
        pack_tma_kernel<<<(unsigned)g, kTmaThreads, smem, s>>>(a);
        return cudaGetLastError();
    }
    const uint64_t g = ntiles < (uint64_t)max_ctas ? ntiles : (uint64_t)max_ctas;
    pack_kernel<<<(unsigned)g, kPackThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_xor(const XorArgs &a, int max_ctas, cudaStream_t s) {
    if (a.nstripes == 0 || a.nin < 1 || a.nin > kMaxTerms || (a.unit & 15)) return cudaErrorInvalidValue;
    static int cap = -1;  // CKPT_XOR_CTAS: CTA budget of the XOR kernel (0 = the pack's)
    if (cap < 0) {
        const char *e = getenv("CKPT_XOR_CTAS");
        cap = e ? std::max(0, atoi(e)) : 0;
    }
    if (cap > 0) max_ctas = cap;
    static int impl = -1;  // CKPT_XOR_IMPL: tma (default) | lsu
    if (impl < 0) {
        const char *e = getenv("CKPT_XOR_IMPL");
        impl = (e && !strcmp(e, "lsu")) ? 0 : 1;
    }
    bool aligned = ((uintptr_t)a.out & 15) == 0 && (a.out_stride & 15) == 0 && (a.out_off & 15) == 0;
    for (int k = 0; k < a.nin; ++k)
        aligned = aligned && ((uintptr_t)a.in[k].base & 15) == 0 && (a.in[k].stride & 15) == 0 &&
                  (a.in[k].off & 15) == 0 && (a.in[k].valid & 15) == 0;
    if (impl == 1 && aligned) {
        // one CTA (4 warps, ~190 KiB of loads in flight) per SM; 32 SMs already pull what
        // NVLink delivers (m=2: 673 vs 678 GB/s on 148 SMs; m=4: 611 vs 607), so the
        // default leaves the other SMs to the training kernels (CKPT_XOR_CTAS overrides)
        const int ctas = cap > 0 ? std::max(1, max_ctas / 2) : std::max(1, std::min(32, max_ctas / 2));
        switch (a.nin) {
            case 1: return launch_xor_tma_n<1>(a, ctas, s);
            case 2: return launch_xor_tma_n<2>(a, ctas, s);
            case 3: return launch_xor_tma_n<3>(a, ctas, s);
            case 4: return launch_xor_tma_n<4>(a, ctas, s);
            case 5: return launch_xor_tma_n<5>(a, ctas, s);
            case 6: return launch_xor_tma_n<6>(a, ctas, s);
            case 7: return launch_xor_tma_n<7>(a, ctas, s);
            default: return launch_xor_tma_n<8>(a, ctas, s);
        }
    }
    switch (a.nin) {
        case 1: return launch_xor_n<1>(a, max_ctas, s);
        case 2: return launch_xor_n<2>(a, max_ctas, s);
        case 3: return launch_xor_n<3>(a, max_ctas, s);
        case 4: return launch_xor_n<4>(a, max_ctas, s);
        case 5: return launch_xor_n<5>(a, max_ctas, s);
        case 6: return launch_xor_n<6>(a, max_ctas, s);
        case 7: return launch_xor_n<7>(a, max_ctas, s);
        default: return launch_xor_n<8>(a, max_ctas, s);
    }
}

}  // namespace reft
