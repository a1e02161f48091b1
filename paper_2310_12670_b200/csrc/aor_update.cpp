// aor_update.cpp -- Eq 4 on the host (PAPER.md P.502-504; reading Q22):
//     w[i] = w[i] - fl(eta * g[i])      fp32, the product rounded before the subtraction.
// Built by the host compiler with -ffp-contract=off (build.py), so neither the scalar loop
// nor the AVX-512 intrinsics are contracted into a fused multiply-add; tests/test_abi_cpu.py
// checks the disassembly for FMA instructions.  The update is host-memory-bound
// (12 B/element for fp32 gradients, 10 B for bf16); AVX-512 keeps one core well above
// its share of DRAM bandwidth.
#include <cstdint>
#include <cstring>

#include <immintrin.h>

namespace reft {
namespace {

void sgd_f32_scalar(float *w, const float *g, uint64_t n, float eta) {
    for (uint64_t i = 0; i < n; ++i) {
        const float p = eta * g[i];
        w[i] = w[i] - p;
    }
}

void sgd_bf16_scalar(float *w, const uint16_t *g, uint64_t n, float eta) {
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t u = (uint32_t)g[i] << 16;  // bf16 -> fp32 is exact
        float gf;
        memcpy(&gf, &u, sizeof gf);
        const float p = eta * gf;
        w[i] = w[i] - p;
    }
}

__attribute__((target("avx512f"))) void sgd_f32_avx512(float *w, const float *g, uint64_t n, float eta) {
    const __m512 e = _mm512_set1_ps(eta);
    uint64_t i = 0;
    for (; i + 32 <= n; i += 32) {
        const __m512 p0 = _mm512_mul_ps(e, _mm512_loadu_ps(g + i));
        const __m512 p1 = _mm512_mul_ps(e, _mm512_loadu_ps(g + i + 16));
        _mm512_storeu_ps(w + i, _mm512_sub_ps(_mm512_loadu_ps(w + i), p0));
        _mm512_storeu_ps(w + i + 16, _mm512_sub_ps(_mm512_loadu_ps(w + i + 16), p1));
    }
    sgd_f32_scalar(w + i, g + i, n - i, eta);
}

__attribute__((target("avx512f"))) void sgd_bf16_avx512(float *w, const uint16_t *g, uint64_t n, float eta) {
    const __m512 e = _mm512_set1_ps(eta);
    uint64_t i = 0;
    for (; i + 16 <= n; i += 16) {
        const __m256i h = _mm256_loadu_si256((const __m256i *)(g + i));
        const __m512 gf = _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(h), 16));
        const __m512 p = _mm512_mul_ps(e, gf);
        _mm512_storeu_ps(w + i, _mm512_sub_ps(_mm512_loadu_ps(w + i), p));
    }
    sgd_bf16_scalar(w + i, g + i, n - i, eta);
}

}  // namespace

bool aor_simd() {
    static const bool ok = __builtin_cpu_supports("avx512f");
    return ok;
}

// dtype: 3 = fp32, 1 = bf16 (CKPT_DTYPE_*).  simd = false forces the scalar loop.
void aor_sgd(float *w, const void *g, uint32_t dtype, uint64_t n, float eta, bool simd) {
    if (dtype == 1) {
        if (simd && aor_simd()) sgd_bf16_avx512(w, (const uint16_t *)g, n, eta);
        else sgd_bf16_scalar(w, (const uint16_t *)g, n, eta);
    } else {
        if (simd && aor_simd()) sgd_f32_avx512(w, (const float *)g, n, eta);
        else sgd_f32_scalar(w, (const float *)g, n, eta);
    }
}

}  // namespace reft
