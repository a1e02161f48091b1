/*
 * reft_synth.h -- seeded synthetic-state generator on the GPU (HARNESS, not the
 * method).  Independent CUDA implementation of the counter-based generator of
 * SURVEY.md 8(c) / DESIGN.md section 4 (SplitMix64 finaliser sm):
 *   base(j, t) = sm(sm(sm(seed) ^ j) ^ t); word w of tensor t = sm(base ^ w), stored
 *   little-endian at byte 8w of the tensor, tail truncated.
 * The oracle (oracle/reft_oracle.c) and synth/__init__.py carry their own copies;
 * tests pin all three to each other and to the published SplitMix64 sequence.
 */
#ifndef REFT_SYNTH_H
#define REFT_SYNTH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
/* Fill (xor_mode = 0) or XOR into (xor_mode = 1, "later training step" mutation for
 * drills) nbytes at device address dst (any alignment) with the bytes of tensor
 * `tensor` of rank `rank`, ordered on `stream` (a cudaStream_t; NULL = legacy).
 * Returns 0 or a negative value (cudaError_t negated) on a launch error. */
int reft_synth_fill(void *dst, uint64_t nbytes, uint64_t seed, uint64_t rank, uint64_t tensor,
                    int xor_mode, void *stream);
#ifdef __cplusplus
}
#endif
#endif
