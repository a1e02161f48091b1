/* examples/drill_from_c.c -- snapshot-and-protect and a loss drill through the C ABI alone
 * (include/ckpt.h), on one GPU: m members of a CKPT_GROUP_LOCAL group, each with a few
 * separately allocated tensors of ragged sizes.  Snapshot + AEC parity (Eq 1), commit,
 * then member `lost` loses its tensors and host image (ckpt_forget), every member calls
 * ckpt_rebuild (Eq 2) and ckpt_load, and every tensor must hold its snapshotted bytes.
 * Exit code 0 and a final "ok" line on success.  tests/test_gpu_parity.py builds and runs it.
 *
 *   gcc -std=c99 -I include -I /usr/local/cuda/include examples/drill_from_c.c \
 *       -L paper_2310_12670_b200 -lreft_ckpt -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2310_12670_b200:/usr/local/cuda/lib64 -o /tmp/drill && /tmp/drill 4 1
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>

#include <cuda_runtime_api.h>

#include "ckpt.h"

#define M_MAX 8
#define T_PER 4

#define CHECK(call)                                                                         \
    do {                                                                                    \
        int rc_ = (call);                                                                   \
        if (rc_ != 0) {                                                                     \
            fprintf(stderr, "%s:%d %s -> %d (%s) %s\n", __FILE__, __LINE__, #call, rc_,     \
                    ckpt_strerror(rc_), ckpt_last_error());                                 \
            return 1;                                                                       \
        }                                                                                   \
    } while (0)

static uint64_t next(uint64_t *s) { /* xorshift64*: test input only */
    *s ^= *s >> 12; *s ^= *s << 25; *s ^= *s >> 27;
    return *s * 2685821657736338717ull;
}

int main(int argc, char **argv)
{
    const int m = argc > 1 ? atoi(argv[1]) : 4, lost = argc > 2 ? atoi(argv[2]) : 1;
    ckpt_ctx *ctx[M_MAX];
    void *dev[M_MAX][T_PER];
    uint8_t *want[M_MAX][T_PER];
    uint64_t nb[M_MAX][T_PER], seed = 12670;
    int j, t;
    if (m < 2 || m > M_MAX || lost < 0 || lost >= m) return 2;
    if (cudaSetDevice(0) != cudaSuccess) return 3;
    for (j = 0; j < m; j++) {
        ckpt_options o;
        ckpt_tensor ten[T_PER];
        ckpt_layout lay = {j, m, j, m, j, m, 0, 1, 0, 1};
        ckpt_options_default(&o);
        o.n_slots = 0;                 /* full-copy staging */
        o.stripe_unit = 4096;
        o.bucket_bytes = 1 << 16;
        CHECK(ckpt_create(0, &o, &ctx[j]));
        for (t = 0; t < T_PER; t++) {
            uint64_t i;
            nb[j][t] = 1 + next(&seed) % 200000;
            want[j][t] = malloc(nb[j][t]);
            for (i = 0; i < nb[j][t]; i++) want[j][t][i] = (uint8_t)next(&seed);
            if (cudaMalloc(&dev[j][t], nb[j][t]) != cudaSuccess) return 3;
            cudaMemcpy(dev[j][t], want[j][t], nb[j][t], cudaMemcpyHostToDevice);
            memset(&ten[t], 0, sizeof ten[t]);
            ten[t].dev_ptr = dev[j][t];
            ten[t].nbytes = nb[j][t];
            ten[t].dtype = CKPT_DTYPE_BYTES;
            ten[t].role = CKPT_ROLE_OTHER;
        }
        CHECK(ckpt_register(ctx[j], ten, T_PER, &lay));
    }
    for (j = 0; j < m; j++) {
        ckpt_group g;
        memset(&g, 0, sizeof g);
        g.m = (uint32_t)m;
        g.my_index = (uint32_t)j;
        g.transport = CKPT_GROUP_LOCAL;
        g.scheme = CKPT_SCHEME_AEC;
        g.members = ctx;
        CHECK(ckpt_protect(ctx[j], &g));
    }
    {
        uint64_t id[M_MAX];
        for (j = 0; j < m; j++) CHECK(ckpt_snapshot(ctx[j], 0, NULL, &id[j]));
        for (j = 0; j < m; j++) CHECK(ckpt_wait(ctx[j], id[j]));
    }
    /* later training steps change every tensor; member `lost` loses everything */
    for (j = 0; j < m; j++)
        for (t = 0; t < T_PER; t++) cudaMemset(dev[j][t], j == lost ? 0xA5 : 0x3C, nb[j][t]);
    CHECK(ckpt_forget(ctx[lost], 0xA5));
    for (j = 0; j < m; j++) CHECK(ckpt_rebuild(ctx[j], lost, NULL));
    for (j = 0; j < m; j++) CHECK(ckpt_load(ctx[j], NULL));
    if (cudaDeviceSynchronize() != cudaSuccess) return 3;
    for (j = 0; j < m; j++)
        for (t = 0; t < T_PER; t++) {
            uint8_t *got = malloc(nb[j][t]);
            cudaMemcpy(got, dev[j][t], nb[j][t], cudaMemcpyDeviceToHost);
            if (memcmp(got, want[j][t], nb[j][t]) != 0) {
                fprintf(stderr, "member %d tensor %d differs after the drill\n", j, t);
                return 4;
            }
            free(got);
        }
    for (j = 0; j < m; j++) CHECK(ckpt_destroy(ctx[j]));
    printf("ok m=%d lost=%d\n", m, lost);
    return 0;
}
