/*
 * ckpt_aor.h -- C ABI of REFT's Asynchronous Optimizer Recomputing (AOR) in libreft_ckpt.
 *
 * PAPER.md P.494-505: under ZeRO-1 data parallelism the optimizer
 * state is sharded over the DP members and has no inherent redundancy, but "model
 * parameters and gradients remain complete on each member".  Each member therefore keeps,
 * in HOST memory, a replica of a peer's optimizer shard and updates it asynchronously from
 * that shard's gradient with Eq 4 (P.502-504):
 *
 *     W_opt,shard^(t+1) = W_opt,shard^(t) - eta * grad W_model,shard^(t)
 *
 * "This update uses the redundant host FLOPs and is asynchronous to training.  On failures,
 * the system retrieves optimizer parameters from host memory with redundant parameters."
 *
 * B200 design:
 *   - group = the m GPUs of the node acting as ZeRO-1 DP members (reading Q25); member i
 *     holds the replica of member h = (i+1) mod m (ring placement as ARC, reading Q23);
 *   - ckpt_aor_step reads the gradient slice of member h from member i's OWN device (the
 *     gradient is complete there): copy-engine D2H on a least-priority stream, chunk by
 *     chunk, into pinned staging -- zero SMs, no NVLink, no collective;
 *   - a host worker applies Eq 4 chunk by chunk as chunks land (thread pool, AVX-512),
 *     overlapping the D2H of the next chunks;
 *   - the replica lives in a POSIX shared-memory object /dev/shm/reft-aor-<key>-<i>
 *     (4 KiB header + fp32[n_h]), so the owner can seed it and a replacement process of
 *     the owner can restore from it after the owner's GPU or process is lost.
 *
 * Arithmetic (reading Q22): fp32, element order irrelevant (elementwise), the product
 * eta * g rounded to fp32 before the subtraction -- no fused multiply-add; a bf16 gradient
 * is widened exactly.  The replica is BIT-IDENTICAL to the owner's shard when the owner's
 * device update computes the same two roundings (e.g. torch: master.sub_(grad * eta)).
 *
 * Conventions as ckpt.h: CKPT_OK or a negative CKPT_E* code, never throws, thread-local
 * ckpt_last_error(); a context is not thread-safe (its internal worker is).  The caller
 * owns the device master shard and gradient (borrowed until ckpt_aor_destroy).
 *
 * Recovery protocol (the caller orders the phases with its process-group barriers; the
 * Python binding's aor_recover does this):
 *   1. survivors: ckpt_aor_wait(last step)          -- replicas quiescent
 *   2. lost x (new context, same key):  ckpt_aor_restore -> its master from holder x-1
 *   3. member x+1 of every lost x:      ckpt_aor_seed    -> re-creates x's held replica
 * Two adjacent losses (x and its holder x-1) are unrecoverable (the oracle's
 * oracle_aor_recover).
 */
#ifndef REFT_CKPT_AOR_H
#define REFT_CKPT_AOR_H

#include "ckpt.h"

#ifdef __cplusplus
extern "C" {
#endif

#define CKPT_AOR_PERSIST 0x1u   /* keep this member's replica object at destroy: a restarted
                                   process (same key and index) re-attaches it             */

/* Replica states (ckpt_aor_view): the header's state word = (step << 8) | code. */
#define CKPT_AOR_EMPTY    0u    /* created, never seeded                                   */
#define CKPT_AOR_CLEAN    1u    /* holds W^(step) of its owner                             */
#define CKPT_AOR_UPDATING 2u    /* an Eq 4 update to `step` is being applied (torn if the
                                   holder died now: not restorable)                        */
#define CKPT_AOR_POISONED 3u    /* ckpt_aor_forget (failure drills)                        */
#define CKPT_AOR_SEEDING  4u    /* the owner's seed copy is in flight                      */

typedef struct ckpt_aor_options {
    uint32_t struct_size;   /* sizeof(ckpt_aor_options); set by ckpt_aor_options_default   */
    uint32_t grad_dtype;    /* CKPT_DTYPE_FP32 (default) or CKPT_DTYPE_BF16                 */
    uint64_t chunk_bytes;   /* gradient bytes per D2H/update chunk: multiple of 4096 and
                               >= 64 KiB; default 16 MiB                                    */
    uint32_t n_slots;       /* pinned gradient staging: 0 (default) = whole shard (one slot
                               per chunk); >= 2 = a ring of n_slots chunks (the D2H of chunk
                               k waits for the host update of chunk k - n_slots)           */
    uint32_t threads;       /* host threads applying Eq 4; 0 = min(8, cores / 2)            */
    int32_t  priority;      /* copy stream priority; default = the device's least          */
    uint32_t flags;         /* CKPT_AOR_*                                                   */
    uint64_t key;           /* != 0: names the group's replica objects (all members agree)  */
    uint32_t reserved[4];
} ckpt_aor_options;

typedef struct ckpt_aor_shard {
    float          *master;    /* device: this member's fp32 optimizer shard,
                                  bounds[my_index+1] - bounds[my_index] elements           */
    const void     *grad;      /* device: the COMPLETE flat gradient, bounds[m] elements of
                                  grad_dtype (ZeRO-1: complete on every member, P.495)      */
    const uint64_t *bounds;    /* m+1 non-decreasing element offsets, bounds[0] = 0: member
                                  j owns the flat range [bounds[j], bounds[j+1]) (copied)   */
    uint32_t        m;         /* DP group size, 1 <= m <= CKPT_MAX_GROUP (m = 1: a host
                                  replica of the member's own shard, no loss tolerance)     */
    uint32_t        my_index;  /* in [0, m)                                                 */
} ckpt_aor_shard;

typedef struct ckpt_aor_stats {
    uint64_t steps;            /* ckpt_aor_step calls applied                              */
    uint64_t chunks;           /* chunks applied                                           */
    uint64_t d2h_bytes;        /* gradient bytes copied device -> host                      */
    uint64_t h2d_bytes;        /* restore bytes                                             */
    double   update_s;         /* host wall time inside Eq 4 (all chunks, worker's clock)   */
    double   stall_s;          /* worker time waiting for chunks to land                    */
    double   last_step_ms;     /* ckpt_aor_step call -> replica CLEAN at that step         */
} ckpt_aor_stats;

typedef struct ckpt_aor ckpt_aor;

/* Defaults: fp32 gradients, 16 MiB chunks, whole-shard staging, default threads, least
 * priority, no flags, key 0 (must be set). */
void ckpt_aor_options_default(ckpt_aor_options *o);

/* Create member my_index's AOR context on `device`: validates the shard, allocates the
 * pinned gradient staging, creates (or, with the same key, re-attaches) its replica object
 * /dev/shm/reft-aor-<key>-<my_index> for member (my_index+1) mod m and starts the worker.
 * A re-attached object keeps its contents and state (e.g. after a process restart).
 * Errors: EINVAL (bad option/shard, key 0, pointers not on the device), EMISMATCH (an
 * existing object of this key describes another geometry), ENOMEM, ECUDA. */
int ckpt_aor_create(int device, const ckpt_aor_options *o, const ckpt_aor_shard *s,
                    ckpt_aor **out);

/* Drain outstanding updates, stop the worker, free staging, unmap (and, without
 * CKPT_AOR_PERSIST, unlink) this member's replica object.  NULL is a no-op. */
int ckpt_aor_destroy(ckpt_aor *a);

/* Seed: copy this member's master shard, as of the current position of `stream`, into
 * the replica its holder (my_index-1) mod m keeps, marking it CLEAN at `step`.  Host-
 * blocking.  Call on every member at attach (after the holders' contexts exist; the
 * object is awaited up to CKPT_TIMEOUT_S) and in recovery phase 3.  The holder must have
 * no update in flight.  Errors: EPEER (holder object missing), EMISMATCH, ECUDA. */
int ckpt_aor_seed(ckpt_aor *a, uint64_t step, void *stream);

/* One Eq 4 step of the held replica with learning rate eta, from the gradient as of the
 * current position of `stream`.  Asynchronous: enqueues the D2H chunks (copy engine) and
 * hands them to the host worker; returns the step id t+1 the replica will reach (t = the
 * replica's step, or the last id returned while updates are pending).  Local only.
 * Errors: ESTATE (replica not CLEAN and nothing pending: never seeded / poisoned), ECUDA. */
int ckpt_aor_step(ckpt_aor *a, float eta, void *stream, uint64_t *step);

/* Make `stream` wait until step `step`'s gradient has been copied out (it may then be
 * overwritten by the next backward pass).  Stream-ordered, zero SMs (stream memory op). */
int ckpt_aor_fence(ckpt_aor *a, uint64_t step, void *stream);

/* Host-block until the replica holds step `step` (or a later one).  Errors: ECUDA (sticky
 * asynchronous failure), ESTATE (timeout after CKPT_TIMEOUT_S or no such step). */
int ckpt_aor_wait(ckpt_aor *a, uint64_t step);

/* Restore this member's master shard from the replica held by (my_index-1) mod m (H2D,
 * ordered before later work on `stream`; host-blocking).  *step receives the replica's
 * step.  Errors: EUNRECOVERABLE (holder object missing, or not CLEAN: lost too, torn,
 * never seeded), EMISMATCH, ECUDA. */
int ckpt_aor_restore(ckpt_aor *a, void *stream, uint64_t *step);

/* Failure injection (drills): drain, overwrite the held replica with `poison`, mark it
 * POISONED. */
int ckpt_aor_forget(ckpt_aor *a, uint8_t poison);

/* The replica this member holds (of member (my_index+1) mod m): pointer into the shared
 * object, element count, step and state code.  Drains outstanding updates first unless
 * the worker is idle.  Any out pointer may be NULL. */
int ckpt_aor_view(ckpt_aor *a, const float **replica, uint64_t *n, uint64_t *step,
                  uint32_t *state);

int ckpt_aor_get_stats(const ckpt_aor *a, ckpt_aor_stats *out);

/* Remove the replica objects of `key` for members [0, m).  Host-only. */
int ckpt_aor_unlink(uint64_t key, uint32_t m);

/* Host-only: one Eq 4 step on a host buffer, w[i] = w[i] - fl(eta * g[i]), with the
 * library's own update routine (the one the worker runs), single-threaded.  For CPU tests
 * of the host arithmetic.  Errors: EINVAL. */
int ckpt_aor_apply(float *w, const void *grad, uint32_t grad_dtype, uint64_t n, float eta);

#ifdef __cplusplus
}
#endif
#endif /* REFT_CKPT_AOR_H */
