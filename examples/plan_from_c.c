/* examples/plan_from_c.c -- the C ABI used from plain C (no Python, no GPU needed):
 * the host-only planner entries of include/ckpt.h (the packing rule of reading Q6 and
 * L* of reading Q4/Q5), Alg 1's estimators, and AOR's Eq 4 routine of include/ckpt_aor.h.
 * Prints one line per result; tests/test_abi_cpu.py compiles it against libreft_ckpt.so
 * and checks the output against the oracle.
 *
 *   gcc -std=c99 -I include examples/plan_from_c.c -L paper_2310_12670_b200 -lreft_ckpt \
 *       -Wl,-rpath,$PWD/paper_2310_12670_b200 -o /tmp/plan_from_c && /tmp/plan_from_c
 */
#include <stdio.h>
#include <stdint.h>
#include <string.h>

#include "ckpt_aor.h"

int main(void)
{
    const uint64_t nbytes[5] = {1000, 4096, 1, 70000, 255};
    uint64_t off[5], L = 0, Ls[3], Lstar = 0, ueff = 0;
    int rc = ckpt_plan_layout(nbytes, 5, 256, off, &L);
    printf("layout rc=%d L=%llu off=%llu,%llu,%llu,%llu,%llu\n", rc, (unsigned long long)L,
           (unsigned long long)off[0], (unsigned long long)off[1], (unsigned long long)off[2],
           (unsigned long long)off[3], (unsigned long long)off[4]);
    Ls[0] = L; Ls[1] = 1280; Ls[2] = 99840;
    rc = ckpt_plan_common(Ls, 3, 4096, &Lstar, &ueff);
    printf("common rc=%d Lstar=%llu unit=%llu\n", rc, (unsigned long long)Lstar, (unsigned long long)ueff);
    ckpt_has_plan_t h;
    rc = ckpt_has_plan(0, 3, 1.0, 100, 10.0, &h);
    printf("has rc=%d t_ss=%.3f t_bubble=%.3f bubble=%llu compute=%llu\n", rc, h.t_ss, h.t_bubble,
           (unsigned long long)h.bubble_bytes, (unsigned long long)h.compute_bytes);
    {
        float w[3] = {1.0f, -3.5f, 1024.0f};
        const float g[3] = {0.5f, -0.25f, 8.0f};
        uint32_t bits[3];
        rc = ckpt_aor_apply(w, g, CKPT_DTYPE_FP32, 3, 0.25f);
        memcpy(bits, w, sizeof bits);
        printf("aor rc=%d w=%08x,%08x,%08x\n", rc, bits[0], bits[1], bits[2]);
    }
    rc = ckpt_plan_common(Ls, 0, 4096, &Lstar, &ueff);
    printf("bad rc=%d (%s) msg=%s\n", rc, ckpt_strerror(rc), ckpt_last_error());
    printf("version %s\n", ckpt_version());
    return 0;
}
