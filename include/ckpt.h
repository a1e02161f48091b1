/*
 * ckpt.h -- C ABI of libreft_ckpt: REFT snapshot-and-protect on B200 (sm_100a).
 *
 * REFT (arXiv 2310.12670) keeps training state in host memory as an in-memory
 * checkpoint ("snapshot", PAPER.md P.553-554) and protects it against the loss of
 * one member of a group with XOR parity ("Asynchronous Erasure Coding", Eq 1,
 * P.474-477; decode Eq 2, P.481-484; REFT-load, P.543-546).  This library is the
 * data-parallel hot path of that method, B200-native:
 *
 *   ckpt_register  -> plan: every registered tensor gets an A-aligned offset in a
 *                     packed image of L_j bytes (reading Q6)
 *   ckpt_protect   -> bind a node group of m ranks (one GPU each); later snapshots
 *                     also build rotated XOR parity (Q3/Q4) over NVLink P2P
 *   ckpt_snapshot  -> gather-pack (kernel) -> [parity encode (kernel, peer reads)]
 *                     -> copy-engine D2H into the ONGOING pinned host image
 *   ckpt_wait      -> completion on every member, then commit ongoing -> completed
 *                     (P.553 "the completed snapshot is replaced by the new copy")
 *   ckpt_rebuild   -> rebuild a lost member's completed image from the survivors'
 *                     completed images and parity (Eq 2; REFT-load step 3, P.545)
 *   ckpt_load      -> H2D of the completed image + unpack into the tensors (P.545
 *                     step 1, "load its checkpoint shard from local Host memory")
 *
 * Layout of the images (identical to the oracle):
 *   D_j  : uint8[L*]        packed image of rank j; tensor t at off_j(t); zero pad.
 *   P_r  : uint8[L* /(m-1)]  parity of rank r; for stripe s (= (m-1) units of u bytes)
 *          P_r[s*u + i] = XOR_{j != r} D_j[s*(m-1)*u + sigma(r,j)*u + i],
 *          sigma(r,j) = r - [r > j].   L* = align_up(max_j L_j, (m-1)*u).
 *
 * Conventions.  Every function returns CKPT_OK (0) or a negative CKPT_E* code and
 * never throws.  ckpt_last_error() returns a thread-local message for the last
 * failure on the calling thread.  A context is not thread-safe.  The caller owns
 * the registered device tensors (borrowed: they must stay allocated and unmoved
 * until ckpt_destroy) and the process group; the library owns its device staging,
 * parity buffers, peer mappings and the pinned host arena.  Asynchronous CUDA
 * errors are sticky on the context and surface at ckpt_wait / ckpt_load /
 * ckpt_rebuild as CKPT_ECUDA.  There is no CPU fallback: without a CUDA device
 * every device-touching call returns CKPT_ECUDA.
 */
#ifndef REFT_CKPT_H
#define REFT_CKPT_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---------------------------------------------------------------- */
#define CKPT_OK               0
#define CKPT_EINVAL          (-1)  /* bad argument (null, zero size, misaligned option)   */
#define CKPT_ECUDA           (-2)  /* CUDA runtime/driver error (sticky once async)       */
#define CKPT_ENOMEM          (-3)  /* device or pinned host allocation failed             */
#define CKPT_ESTATE          (-4)  /* call not valid in the context's current state       */
#define CKPT_EUNAVAIL        (-5)  /* protection unavailable: m = 1 (SPEC S.314)          */
#define CKPT_EMISMATCH       (-6)  /* group members disagree on geometry (digest)         */
#define CKPT_EPEER           (-7)  /* peer mapping (CUDA IPC open / P2P) failed           */
#define CKPT_EBUSY           (-8)  /* previous snapshot not yet waited                    */
#define CKPT_ENOSNAP         (-9)  /* no completed snapshot to load or rebuild from       */
#define CKPT_EUNRECOVERABLE  (-10) /* more losses than the code tolerates (P.460, S.334)  */

/* ---- options ---------------------------------------------------------------------- */
#define CKPT_OPT_TIMING      0x1u  /* time every pack/xor launch with CUDA events (stats) */
#define CKPT_OPT_TMA_PACK    0x2u  /* pack via cp.async.bulk (TMA 1-D) through SMEM; the
                                      default of the full-copy single-launch pack, opt-in
                                      for per-bucket (ring) packs                         */
#define CKPT_OPT_LSU_PACK    0x4u  /* force the 128-bit LDG/STG pack                      */
#define CKPT_OPT_CE_PACK     0x8u  /* pack/unpack with copy-engine D2D copies (zero SMs)  */
#define CKPT_OPT_CE_GATHER   0x10u /* parity: copy engines pull the m-1 peer units over
                                      NVLink (2-D copies) into local HBM, then the XOR
                                      kernel runs locally at HBM speed (few SM-seconds);
                                      at m = 2 (a mirror, P.459) the pull lands in the
                                      parity buffer itself: no kernel, zero SMs           */
#define CKPT_OPT_DEVICE_ONLY 0x20u /* keep the image in HBM only: snapshot = pack + parity
                                      into the full device staging (n_slots must be 0), no
                                      D2H, no host arena; load/rebuild work from HBM.  A
                                      single device image: a failed snapshot destroys the
                                      previous one.  Measures the device-side protect path. */
#define CKPT_OPT_HOST_LOAD   0x80u /* always restore (load / rebuild sources) from the host
                                      image, never from a still-valid device copy (the
                                      paper's REFT-load after a full restart, P.545)       */
#define CKPT_OPT_WINDOWED    0x100u /* HAS placement (Alg 1, P.377-429): each bucket's D2H
                                      waits until the caller's training stream has opened
                                      the snapshot window (ckpt_window)                   */
#define CKPT_OPT_REBUILD_SHARES 0x200u /* rebuild: the m-1 survivors each encode 1/(m-1) of
                                      the lost member's parity row into its parity buffer
                                      (reading Q27): the lost GPU receives L*.m/(m-1) instead
                                      of 2.L* over NVLink.  The DEFAULT for m >= 3 (measured
                                      C5 m = 4: 54.5 vs 70.7 ms); this flag forces it at m = 2
                                      too.  Every member must agree (else ckpt_protect
                                      returns EMISMATCH)                                   */
#define CKPT_OPT_REBUILD_SELF 0x800u /* rebuild: the lost member re-encodes its own parity
                                      row from the survivors' data (2.L* into the lost GPU;
                                      the default at m = 2).  Must agree like the above     */
#define CKPT_OPT_XOR_PUSH    0x400u /* parity encode in push mode (full-copy staging only;
                                      otherwise ignored): every member sends each unit of its
                                      own image to its row owner as a bulk XOR reduction
                                      (cp.reduce.async.bulk .xor) into that owner's parity,
                                      which the owner zeroes before its pack -- posted NVLink
                                      writes instead of round-trip peer reads.  Same bytes as
                                      the pull encode (Eq 1).  Every member must agree (else
                                      ckpt_protect returns EMISMATCH)                      */
#define CKPT_OPT_SHM_ARENA   0x40u /* host arena in POSIX shared memory (/dev/shm), one file
                                      per member and host buffer: peers (ARC) and a restarted
                                      process can reach it; required by the ARC schemes     */

typedef struct ckpt_options {
    uint32_t struct_size;   /* sizeof(ckpt_options); set by ckpt_options_default       */
    uint32_t align;         /* A: packed segment alignment, power of 2 in [16, 4096];
                               default 256 (reading Q6)                                  */
    uint64_t stripe_unit;   /* u: bytes, multiple of 16; default 1 MiB (Q4: at m = 4 the
                               encode's strided peer reads run at 612 GB/s with 16-64 KiB
                               units and at the all-to-all pull rate, 672, from 1 MiB);
                               0 = one stripe, u = L* /(m-1) (SPEC S.378).  The image is
                               padded to whole stripes ((m-1)u): small shards want a
                               smaller u                                                 */
    uint64_t bucket_bytes;  /* ring slot capacity / default bucket size; default 64 MiB */
    uint32_t n_slots;       /* device staging ring slots (>= 2); 0 = full device copy:
                               staging holds the whole image, the fence releases the
                               tensors after the pack alone                              */
    uint32_t host_buffers;  /* 2 = ongoing + completed (P.553-554, default); 1 = single
                               buffer (commit still atomic w.r.t. ckpt_wait, but a
                               failed snapshot destroys the previous image)              */
    int32_t  priority;      /* CUDA stream priority of the library's streams; default
                               = the device's LEAST priority (so training runs first)   */
    uint32_t max_ctas;      /* CTA budget of one pack/xor launch; 0 = 2 x SM count      */
    uint32_t flags;         /* CKPT_OPT_*                                               */
    uint32_t reserved0;
    uint64_t arena_key;     /* with CKPT_OPT_SHM_ARENA: 0 = private arena (unlinked at
                               destroy); != 0 = PERSISTENT arena named by this key and
                               the member index (= layout.local_rank): it outlives the
                               process like the paper's tmpfs copies (P.553-555), and a
                               process registering the same key, layout and geometry
                               re-attaches the last committed image (ckpt_load restores
                               it).  Remove it with ckpt_arena_unlink.                   */
    uint32_t reserved[4];
} ckpt_options;

/* ---- registered tensors and layout -------------------------------------------------- */
#define CKPT_DTYPE_BYTES 0u
#define CKPT_DTYPE_BF16  1u
#define CKPT_DTYPE_FP16  2u
#define CKPT_DTYPE_FP32  3u
#define CKPT_ROLE_PARAM      0u
#define CKPT_ROLE_MASTER     1u
#define CKPT_ROLE_EXP_AVG    2u
#define CKPT_ROLE_EXP_AVG_SQ 3u
#define CKPT_ROLE_OTHER      4u
#define CKPT_TENSOR_REPLICATED 0x1u  /* TP-replicated (e.g. RMSNorm); saved anyway (Q9) */

typedef struct ckpt_tensor {
    void       *dev_ptr;   /* device address on the context's device; any alignment   */
    uint64_t    nbytes;    /* > 0                                                       */
    uint32_t    dtype;     /* CKPT_DTYPE_*: informational; bytes are copied raw (Q7)   */
    uint32_t    role;      /* CKPT_ROLE_*: informational                                */
    uint32_t    flags;     /* CKPT_TENSOR_*                                             */
    uint32_t    reserved;
    const char *name;      /* optional, copied                                          */
} ckpt_tensor;

typedef struct ckpt_layout {   /* the hybrid-parallel position of this rank (P.359-371) */
    int32_t rank, world, local_rank, local_world;
    int32_t tp_rank, tp_size, pp_rank, pp_size, dp_rank, dp_size;
} ckpt_layout;

/* ---- groups --------------------------------------------------------------------------- */
#define CKPT_HANDLE_BYTES 1024u   /* size of one exported handle blob                   */
#define CKPT_MAX_GROUP    8u      /* m <= 8: one 8 x B200 node (reading Q1)   */
#define CKPT_GROUP_IPC    0u      /* one process per GPU; peers mapped with CUDA IPC,
                                     per-bucket ordering by stream memory operations    */
#define CKPT_GROUP_LOCAL  1u      /* all m contexts in this process (possibly the same
                                     device); ordering by CUDA events; the group's
                                     snapshot is issued by the last member's call        */

typedef struct ckpt_ctx ckpt_ctx;

/* Protection schemes (P.349, P.435-508).  AEC: rotated XOR parity, one parity row per
 * member (tolerates 1 loss).  ARC: member i's host arena also holds a copy of member
 * (i+1) mod m's image (ring placement, SPEC S.313; volume 2 W_n/m, P.459; tolerates 1
 * loss).  ARC_AEC: both, with the ARC copy carrying the neighbour's parity row too
 * (reading Q20) -- "collaborative protection" tolerating any 2 losses for m >= 3 (P.507). */
#define CKPT_SCHEME_DEFAULT  0u   /* = AEC                                               */
#define CKPT_SCHEME_AEC      1u
#define CKPT_SCHEME_ARC      2u
#define CKPT_SCHEME_ARC_AEC  3u

typedef struct ckpt_group {
    uint32_t         m;          /* group size, 1 <= m <= CKPT_MAX_GROUP                 */
    uint32_t         my_index;   /* this context's member index in [0, m)               */
    uint32_t         transport;  /* CKPT_GROUP_IPC or CKPT_GROUP_LOCAL                  */
    uint32_t         scheme;     /* CKPT_SCHEME_*; ARC schemes need CKPT_OPT_SHM_ARENA
                                    and full-copy staging (n_slots = 0)                  */
    const void      *handles;    /* IPC: m * CKPT_HANDLE_BYTES blobs from
                                    ckpt_export_handle, in member order                 */
    ckpt_ctx *const *members;    /* LOCAL: the m contexts, in member order              */
} ckpt_group;

typedef struct ckpt_stats {      /* cumulative since ckpt_stats_reset                    */
    uint64_t snapshots, loads, rebuilds;
    uint64_t pack_launches, xor_launches, unpack_launches, rebuild_launches;
    uint64_t pack_bytes;         /* algorithmic: bytes read + written by pack kernels    */
    uint64_t xor_bytes_in;       /* algorithmic: peer bytes read by encode kernels       */
    uint64_t xor_bytes_out;      /* parity bytes written                                 */
    uint64_t d2h_bytes, h2d_bytes;
    uint64_t ce_copies;          /* copy-engine operations issued (pack/gather/D2H/H2D)  */
    uint64_t rebuild_bytes_in;   /* algorithmic: peer + parity bytes read by rebuild rows */
    uint64_t rebuild_bytes_out;  /* rebuilt bytes stored into the lost rank (NVLink)      */
    double   pack_ms, xor_ms, unpack_ms, rebuild_ms; /* summed launch durations
                                    (only with CKPT_OPT_TIMING)                          */
    double   last_snapshot_ms;   /* capture event -> last D2H event of the last snapshot
                                    (only with CKPT_OPT_TIMING)                          */
    uint64_t gather_ops;         /* m = 2 with CKPT_OPT_CE_GATHER: copy-engine mirror
                                    pulls (one per bucket), no XOR kernel                */
    double   gather_ms;          /* their summed durations (only with CKPT_OPT_TIMING)   */
} ckpt_stats;

/* ---- lifecycle ------------------------------------------------------------------------- */

/* Fill *o with defaults (A = 256, u = 64 KiB, bucket = 64 MiB, n_slots = 4, two host
 * buffers, least stream priority).  Never fails for a non-null o. */
void ckpt_options_default(ckpt_options *o);

/* Create a context bound to CUDA device `device` (one context per rank).  o may be
 * NULL for defaults.  Errors: EINVAL (bad option), ECUDA (no such device / no CUDA),
 * ENOMEM. */
int ckpt_create(int device, const ckpt_options *o, ckpt_ctx **out);

/* Destroy: waits for outstanding work, unmaps peers, frees everything the library
 * owns.  NULL is a no-op. */
int ckpt_destroy(ckpt_ctx *ctx);

/* Register the rank's state (PAPER.md "Global Parameter Sharding", P.369-371: this
 * rank's shard W_n/m -- here the TP/PP shard it holds).  Builds the packing plan:
 * tensor t at off(t) = align_up(off(t-1) + nbytes(t-1), A), L_j = align_up(end, A)
 * (reading Q6), and allocates the device staging.  `tensors` is copied; the device
 * buffers are borrowed.  Registration is once per context.
 * Errors: EINVAL (null, n = 0, nbytes = 0, pointer not on the device), ESTATE
 * (already registered), ENOMEM. */
int ckpt_register(ckpt_ctx *ctx, const ckpt_tensor *tensors, uint64_t n,
                  const ckpt_layout *layout);

/* Packed length L_j of this rank (after ckpt_register) and, after ckpt_protect, the
 * group's common length L* and effective stripe unit.  Any out pointer may be NULL. */
int ckpt_geometry(const ckpt_ctx *ctx, uint64_t *L_local, uint64_t *L_star,
                  uint64_t *unit, uint32_t *m);

/* Offset of registered tensor t in the packed image (for host-image inspection). */
int ckpt_tensor_offset(const ckpt_ctx *ctx, uint64_t t, uint64_t *offset);

/* IPC groups: write this rank's handle blob (device ordinal, geometry digest, L_j,
 * CUDA IPC handles of its staging and flag page) to buf; *len is in/out (>=
 * CKPT_HANDLE_BYTES).  The caller all-gathers the blobs (e.g. torch.distributed over
 * NCCL) and passes them to ckpt_protect.  Errors: ESTATE (not registered), EINVAL. */
int ckpt_export_handle(ckpt_ctx *ctx, void *buf, uint64_t *len);

/* Bind the group ("sharding group", P.359/P.371; here the node group, Q1).
 * COLLECTIVE over the m members.  Computes L* and the stripe geometry, checks
 * every member's geometry digest (A, u, ring shape), maps peers (IPC) or links
 * contexts (LOCAL), allocates parity buffers and the host arena.  Afterwards every
 * ckpt_snapshot also builds parity.  m = 1 allocates the arena and returns
 * EUNAVAIL (no redundancy possible).  Errors: EINVAL, ESTATE, EMISMATCH, EPEER,
 * ENOMEM, EUNAVAIL. */
int ckpt_protect(ckpt_ctx *ctx, const ckpt_group *g);

/* Snapshot (REFT-save).  Captures the registered tensors as of the current position
 * of `stream` (Q10) and asynchronously packs them bucket by bucket, builds parity
 * (if protected) and copies data and parity into the ONGOING host image on the
 * library's low-priority streams.  bucket_bytes = 0 uses the option; it is rounded
 * down to whole stripes ((m-1)*u bytes; A bytes when unprotected) and must not
 * exceed the ring slot capacity.  COLLECTIVE when protected: every member passes the
 * same bucket_bytes.  *id receives the snapshot id.  Errors: EBUSY (previous
 * snapshot not waited), EINVAL, ESTATE (not registered), ECUDA. */
int ckpt_snapshot(ckpt_ctx *ctx, uint64_t bucket_bytes, void *stream, uint64_t *id);

/* Make `stream` wait until snapshot `id` no longer reads the registered tensors
 * (all buckets packed) -- call before the next optimizer step mutates them.
 * With CKPT_OPT_WINDOWED and ring staging (n_slots > 0) the packs of later buckets are
 * enqueued only as earlier buckets reach host memory inside the HAS windows (their ring
 * slots are reused), so until every pack is issued this returns EBUSY: keep opening
 * windows (ckpt_window) and call ckpt_test / ckpt_wait, or use full-copy staging. */
int ckpt_fence(ckpt_ctx *ctx, uint64_t id, void *stream);

/* Host-block until snapshot `id`'s data and parity have landed in host memory on
 * EVERY member, then commit: ongoing -> completed (P.551-554; SPEC S.427-435).  A
 * snapshot that failed is never committed; the previous completed image stays.
 * Errors: ECUDA (sticky async error; commit refused), ESTATE (no such snapshot). */
int ckpt_wait(ckpt_ctx *ctx, uint64_t id);

/* Non-blocking: *done = 1 when snapshot `id` has landed everywhere ckpt_wait waits for
 * (ckpt_wait then returns at once and commits), else 0.  Never commits by itself.  With
 * CKPT_OPT_WINDOWED it also enqueues the next window-gated copies (see ckpt_window).
 * Errors: EINVAL, ESTATE (unknown id), ECUDA. */
int ckpt_test(ckpt_ctx *ctx, uint64_t id, int *done);

/* Restore every registered tensor from the last COMPLETED image (H2D + unpack),
 * ordered on `stream`; returns after enqueueing (stream-ordered, host-async).
 * Local only: no communication.  With full-copy staging the library's device copy of
 * the completed image is used directly (no H2D) while it is still valid -- from the
 * commit until the next snapshot starts packing, unless ckpt_forget declared the device
 * lost; CKPT_OPT_HOST_LOAD forces the host path.  Errors: ENOSNAP, ESTATE, ECUDA. */
int ckpt_load(ckpt_ctx *ctx, void *stream);

/* Rebuild lost member `lost_rank`'s completed image (data and its parity row) from
 * the survivors' completed images (Eq 2, P.481-484; REFT-load step 3, P.545;
 * reading Q11: never from live device state).  COLLECTIVE over the group and
 * host-blocking; every member passes the same lost_rank.  Survivors H2D their
 * completed data and parity, each row owner r != k XORs its parity with the other
 * survivors' units (NVLink reads) and writes the result into rank k's staging (P2P
 * stores); survivor i of the m-1 then encodes stripes [i*n/(m-1), (i+1)*n/(m-1)) of
 * rank k's parity row (Eq 1 for row k: every term is a survivor's unit) into rank k's
 * parity buffer (reading Q27; IPC: mapped from the handle rank k published in its flag
 * page at ckpt_protect), and rank k D2Hs both into its completed image.
 * Follow with ckpt_load on every member to restore tensors.
 * Errors: EUNRECOVERABLE (m = 1, or a survivor has no completed image -- more than
 * one loss), EINVAL, ENOSNAP, EPEER (rank k's parity handle cannot be mapped), ECUDA. */
int ckpt_rebuild(ckpt_ctx *ctx, int32_t lost_rank, void *stream);

/* REFT-load step 3 for up to two losses (P.545; collaborative protection P.507-508).
 * COLLECTIVE and host-blocking; every member passes the same lost_mask (bit j = member
 * j lost both its tensors and its host image).  Order (the oracle's oracle_recover):
 * (1) every lost member x whose ARC holder x-1 survived takes its completed image (and
 * parity row) from the holder's ARC copy; (2) a single remaining loss is rebuilt from
 * parity as in ckpt_rebuild; (3) the ARC copies held by lost members are re-created from
 * their neighbours' completed images.  Follow with ckpt_load on every member.  With
 * full-copy staging (and without CKPT_OPT_HOST_LOAD) step (1) goes device-first: an H2D
 * of the holder's copy into the member's staging, so ckpt_load unpacks from HBM, while
 * the member's own host image and the copy it holds are re-written by host threads in
 * the background (ckpt_sync waits for them; every call that reads the host image does).
 * Errors: EUNRECOVERABLE (the losses exceed what the scheme restores), EINVAL, ENOSNAP,
 * ECUDA, EPEER. */
int ckpt_recover(ckpt_ctx *ctx, uint32_t lost_mask, void *stream);

/* Host-block until every asynchronous host-image write of this context is complete:
 * after ckpt_rebuild with full-copy staging the lost member's call returns once its
 * DEVICE image is rebuilt (ckpt_load can run at once) while its host image is re-written
 * in the background; the next snapshot, ckpt_load from host, ckpt_host_view and
 * ckpt_forget wait for it implicitly. */
int ckpt_sync(ckpt_ctx *ctx);

/* Failure injection for drills (Q12, hardware-loss semantics): overwrite this
 * member's completed and ongoing host images with `poison` and mark it as having no
 * completed snapshot (it can only be restored by ckpt_rebuild). */
int ckpt_forget(ckpt_ctx *ctx, uint8_t poison);

/* Read-only view of the completed (which = 0) or ongoing (which = 1) host image:
 * data (L* bytes) and parity (L* /(m-1) bytes, NULL/0 when unprotected).  which = 2 / 3:
 * the ARC copy (completed / ongoing) this member holds of member (i+1) mod m: data and,
 * for ARC_AEC, that member's parity row.
 * Errors: EINVAL, ENOSNAP (which = 0 and nothing committed). */
int ckpt_host_view(const ckpt_ctx *ctx, int which, const void **data, uint64_t *dlen,
                   const void **parity, uint64_t *plen);

/* Counters and (with CKPT_OPT_TIMING) per-kernel launch durations. */
int ckpt_get_stats(const ckpt_ctx *ctx, ckpt_stats *out);
int ckpt_stats_reset(ckpt_ctx *ctx);

/* Messages.  ckpt_strerror never returns NULL; ckpt_last_error returns "" when the
 * calling thread has no error recorded. */
const char *ckpt_strerror(int code);
const char *ckpt_last_error(void);

/* Host-only planner entry (no device needed): offsets and L for a tensor list, the
 * same rule ckpt_register applies.  Used by CPU tests of the host logic. */
int ckpt_plan_layout(const uint64_t *nbytes, uint64_t n, uint32_t align,
                     uint64_t *offsets, uint64_t *L);

/* Host-only: L* and effective u for a group with packed lengths Lj[0..m). */
int ckpt_plan_common(const uint64_t *Lj, uint32_t m, uint64_t unit, uint64_t *L_star,
                     uint64_t *unit_eff);

/* Remove the persistent arena of `key` (members [0, m), host buffers [0, nbuf)) from
 * /dev/shm.  Host-only; missing objects are ignored. */
int ckpt_arena_unlink(uint64_t key, uint32_t m, uint32_t nbuf);

/* ---- Hierarchical Asynchronous Snapshotting (Alg 1, P.377-429) ------------------------
 * Placement of the snapshot's host traffic relative to training.  With copy engines the
 * D2H can overlap anything; what it still disturbs is HBM-bound training work (measured:
 * a concurrent 57 GB/s D2H slows an HBM-bound kernel by 10-35%, tools/ce_interference.py).
 * ckpt_window(ctx, open, stream) enqueues on the TRAINING stream a write of the context's
 * window word: a mask of CKPT_WINDOW_BUBBLE (pipeline bubbles, Alg 1 lines 9-12) and
 * CKPT_WINDOW_COMPUTE (compute-bound phases, layers 1-2, P.419-425); 0 closes both (both
 * are open at creation).  With CKPT_OPT_WINDOWED every bucket's D2H (data and parity)
 * first waits, on the copy engine's stream (zero SMs), until its window is open.  Which
 * buckets wait for which window is Alg 1's SplitParameter, applied by ckpt_has_apply:
 * the first bubble_bytes of the image (whole buckets) go out only in bubbles, the rest
 * alongside computation or in a bubble (reading Q26); by default every bucket is a bubble
 * bucket.  Buckets leave in image order.  A snapshot whose windows are
 * never reopened does not complete (ckpt_wait times out; ckpt_destroy opens every window
 * before it drains).  With one process per member (IPC groups, or no group) the gated
 * copies are enqueued progressively -- at most 32 beyond the last one that completed --
 * so ckpt_snapshot never blocks the training thread on a full stream queue; ckpt_window,
 * ckpt_test and ckpt_wait enqueue the next ones, so call them while the snapshot is in
 * flight (a training loop that opens windows does). */
#define CKPT_WINDOW_BUBBLE  0x1u
#define CKPT_WINDOW_COMPUTE 0x2u
#define CKPT_WINDOW_COMM    0x4u  /* Layer 3 (P.425): a communication phase of training on
                                     another interconnect than the snapshot's (NVLink
                                     collectives while the D2H uses PCIe); used only by the
                                     buckets ckpt_has_apply_layers assigns to it            */
int ckpt_window(ckpt_ctx *ctx, int open, void *stream);

/* Alg 1 SplitParameter into the scheduler (lines 10-12): image bytes [0, bubble_bytes),
 * rounded up to whole buckets at each snapshot, are snapshotted in CKPT_WINDOW_BUBBLE
 * windows, the rest in CKPT_WINDOW_COMPUTE (or bubble) windows (use ckpt_has_plan's
 * bubble_bytes).
 * UINT64_MAX (the default) = all in bubbles.  Takes effect at the next snapshot.
 * Errors: EINVAL. */
int ckpt_has_apply(ckpt_ctx *ctx, uint64_t bubble_bytes);

/* The three layers of HAS (P.419-425) in the scheduler: image bytes [0, bubble_bytes) go
 * out only in bubbles (Layer 1), [bubble_bytes, bubble_bytes + compute_bytes) in bubble or
 * compute windows (Layer 2), the rest in bubble, compute or communication windows (Layer 3:
 * "not used unless the previous layers are not enough").  Whole buckets, rounded up at each
 * snapshot.  ckpt_has_apply(ctx, b) is ckpt_has_apply_layers(ctx, b, UINT64_MAX).
 * Errors: EINVAL. */
int ckpt_has_apply_layers(ckpt_ctx *ctx, uint64_t bubble_bytes, uint64_t compute_bytes);

/* Alg 1's estimators, host-only.  EstimateSnapshotTime = bytes / B_io; EstimateBubbleTime
 * = (0.8 p + 2|P| - p - 2) * C_FB,BP (1F1B, stage p of |P|, clamped at 0); SplitParameter:
 * if t_ss >= t_bubble the first floor(n * t_bubble / t_ss) of n bytes go into bubbles and
 * the rest alongside computation, else all n bytes go into bubbles. */
typedef struct ckpt_has_plan_t {
    double t_ss, t_bubble;        /* seconds                                             */
    uint64_t bubble_bytes;        /* W_bubble (Alg 1 line 10/12)                          */
    uint64_t compute_bytes;       /* W_* (snapshotted during computation)                 */
} ckpt_has_plan_t;
int ckpt_has_plan(uint32_t stage, uint32_t num_stages, double c_fb_bp_s, uint64_t snapshot_bytes,
                  double b_io_bytes_per_s, ckpt_has_plan_t *out);

/* Alg 1 extended to Layers 2 and 3 (reading Q28): the bubble part is ckpt_has_plan's
 * W_bubble exactly; of the rest W_*, the first floor(n * t_compute / t_ss) bytes (at most
 * W_*) go alongside computation -- t_compute_s is the computation time per iteration in
 * which the caller opens compute windows -- and whatever is left goes to Layer 3.
 * Host-only.  Errors: EINVAL (as ckpt_has_plan, or t_compute_s < 0). */
typedef struct ckpt_has_plan3_t {
    double t_ss, t_bubble, t_compute;  /* seconds                                           */
    uint64_t bubble_bytes;             /* Layer 1 (= ckpt_has_plan's W_bubble)              */
    uint64_t compute_bytes;            /* Layer 2                                           */
    uint64_t comm_bytes;               /* Layer 3                                           */
} ckpt_has_plan3_t;
int ckpt_has_plan3(uint32_t stage, uint32_t num_stages, double c_fb_bp_s, uint64_t snapshot_bytes,
                   double b_io_bytes_per_s, double t_compute_s, ckpt_has_plan3_t *out);

/* ---- fabric probe (measurement; "NVLink ... to be measured P2P, all
 * ranks concurrent") --------------------------------------------------------------------
 * Every member of a protected group reads `bytes_per_peer` bytes from EACH of its m-1
 * peers' device staging at once: the encode's all-to-all pattern (row r pulls L* /(m-1)
 * from every peer, Eq 1 P.474-477), so the result is the denominator of the XOR kernel's
 * roofline.  mode CKPT_PROBE_SM_PULL: the XOR kernel's own load mechanism (cp.async.bulk
 * peer -> SMEM, 16 KiB pieces, 3 stages per warp, data discarded) on `ctas` CTAs (0 = the
 * XOR kernel's CTA budget); CKPT_PROBE_CE_PULL: one copy-engine cudaMemcpyAsync per peer,
 * each on its own stream, into a scratch buffer the call allocates and frees.
 * Read-only: no staging or image is modified.  Not a collective protocol, but every member
 * must call it at the same time for the figure to mean anything (the caller aligns them,
 * e.g. with a barrier).  *gbs = bytes_per_peer * (m-1) / elapsed time between CUDA events
 * on `stream` (host-synchronous: returns after the copies finished).
 * Errors: EINVAL (bytes_per_peer 0, not a multiple of 16 KiB, or beyond a peer's staging),
 * ESTATE (not protected, m < 2, or a snapshot in flight), ECUDA. */
#define CKPT_PROBE_SM_PULL 0
#define CKPT_PROBE_CE_PULL 1
int ckpt_probe_fabric(ckpt_ctx *ctx, int mode, uint64_t bytes_per_peer, uint32_t ctas, void *stream,
                      double *gbs);

/* Library version string, e.g. "reft-ckpt 0.1 sm_100a". */
const char *ckpt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* REFT_CKPT_H */
