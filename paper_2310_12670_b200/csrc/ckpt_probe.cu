// ckpt_probe.cu -- ckpt_probe_fabric: the all-concurrent NVLink pull figure that is the
// XOR encode's roofline denominator (include/ckpt.h).
#include "ckpt_internal.cuh"

using namespace reft;

extern "C" int ckpt_probe_fabric(ckpt_ctx *c, int mode, uint64_t bytes_per_peer, uint32_t ctas, void *stream,
                                 double *gbs) {
    NvtxRange nvtx_("ckpt_probe_fabric");
    if (!c || !gbs) return fail(CKPT_EINVAL, "probe: null argument");
    if (mode != CKPT_PROBE_SM_PULL && mode != CKPT_PROBE_CE_PULL) return fail(CKPT_EINVAL, "probe: unknown mode %d", mode);
    if (!c->grouped || c->m < 2) return fail(CKPT_ESTATE, "probe: needs a protected group of m >= 2");
    if (c->pending_id || c->requested) return fail(CKPT_ESTATE, "probe: a snapshot is in flight");
    if (bytes_per_peer == 0 || bytes_per_peer % 16384) return fail(CKPT_EINVAL, "probe: bytes_per_peer must be a positive multiple of 16 KiB");
    for (uint32_t j = 0; j < c->m; ++j)
        if (j != c->me && bytes_per_peer * (c->m - 1) > c->staging_bytes)
            return fail(CKPT_EINVAL, "probe: %llu bytes from each of %u peers exceed the staging (%llu)",
                        (unsigned long long)bytes_per_peer, c->m - 1, (unsigned long long)c->staging_bytes);
    int rc = set_dev(c);
    if (rc) return rc;
    rc = check_sticky(c);
    if (rc) return rc;
    // peer j's staging region read by member `me`: disjoint per reader, like the encode's
    // units sigma(r, j) of one stripe
    auto region = [&](uint32_t j) { return (const uint8_t *)c->peer_staging[j] + (uint64_t)sigma(c->me, j) * bytes_per_peer; };
    cudaStream_t s = (cudaStream_t)stream;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    std::vector<cudaStream_t> ss;
    std::vector<cudaEvent_t> joins;
    uint8_t *scratch = nullptr;
    cudaError_t e = cudaSuccess;
    float ms = 0;
    auto cleanup = [&]() {
        for (auto x : ss) cudaStreamDestroy(x);
        for (auto x : joins) cudaEventDestroy(x);
        if (scratch) cudaFree(scratch);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    };
    if ((e = cudaEventCreate(&e0)) != cudaSuccess || (e = cudaEventCreate(&e1)) != cudaSuccess) goto out;
    if (mode == CKPT_PROBE_CE_PULL) {
        if ((e = cudaMalloc(&scratch, bytes_per_peer * (c->m - 1))) != cudaSuccess) goto out;
        for (uint32_t q = 0; q + 1 < c->m; ++q) {
            cudaStream_t x;
            cudaEvent_t j;
            if ((e = cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking)) != cudaSuccess) goto out;
            ss.push_back(x);
            if ((e = cudaEventCreateWithFlags(&j, cudaEventDisableTiming)) != cudaSuccess) goto out;
            joins.push_back(j);
        }
    }
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) goto out;
    if ((e = cudaEventRecord(e0, s)) != cudaSuccess) goto out;
    if (mode == CKPT_PROBE_SM_PULL) {
        ProbeArgs a;
        memset(&a, 0, sizeof a);
        for (uint32_t j = 0; j < c->m; ++j)
            if (j != c->me) a.src[a.npeers++] = region(j);
        a.n = bytes_per_peer;
        const int n = ctas ? (int)ctas : std::max(1, std::min(32, c->xor_ctas / 2));
        if ((e = launch_probe_pull(a, n, s)) != cudaSuccess) goto out;
    } else {
        uint32_t q = 0;
        for (uint32_t j = 0; j < c->m; ++j) {
            if (j == c->me) continue;
            if ((e = cudaStreamWaitEvent(ss[q], e0, 0)) != cudaSuccess) goto out;
            if ((e = cudaMemcpyAsync(scratch + (uint64_t)q * bytes_per_peer, region(j), bytes_per_peer,
                                     cudaMemcpyDeviceToDevice, ss[q])) != cudaSuccess)
                goto out;
            if ((e = cudaEventRecord(joins[q], ss[q])) != cudaSuccess) goto out;
            if ((e = cudaStreamWaitEvent(s, joins[q], 0)) != cudaSuccess) goto out;
            ++q;
        }
    }
    if ((e = cudaEventRecord(e1, s)) != cudaSuccess) goto out;
    if ((e = cudaEventSynchronize(e1)) != cudaSuccess) goto out;
    if ((e = cudaEventElapsedTime(&ms, e0, e1)) != cudaSuccess) goto out;
    *gbs = ms > 0 ? (double)bytes_per_peer * (c->m - 1) / (ms * 1e-3) / 1e9 : 0.0;
out:
    cleanup();
    if (e != cudaSuccess) return fail(CKPT_ECUDA, "probe: %s", cudaGetErrorString(e));
    return CKPT_OK;
}
