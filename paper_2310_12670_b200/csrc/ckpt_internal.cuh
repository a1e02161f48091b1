// ckpt_internal.cuh -- shared internals of libreft_ckpt (planner, arena, pipeline, recovery).
// Product code: nothing here is part of the C ABI (symbols are hidden; see build.py).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdarg>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <random>

#include <nvtx3/nvToolsExt.h>

#pragma GCC visibility push(default)  // the C ABI is the only exported surface
#include "../../include/ckpt.h"
#pragma GCC visibility pop
#include "ckpt_kernels.cuh"

using namespace reft;

// NVTX ranges around the public calls (host-side enqueue/wait), for nsys timelines.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};


// ------------------------------------------------------------------ errors ----------
extern thread_local std::string g_last_error;
int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
#define CUDA_TRY(expr)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (expr);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            return fail(CKPT_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                              \
    } while (0)
extern PFN_cuStreamWaitValue32_v8000 p_wait32;
extern PFN_cuStreamWriteValue32_v8000 p_write32;
int load_memops();

// ------------------------------------------------------------------ constants -------
namespace reft {
constexpr uint32_t kMagic = 0x52454654u;  // "REFT"
constexpr uint32_t kAbiVersion = 2;  // 2: HandleBlob.opt_flags (CKPT_OPT_REBUILD_SHARES, CKPT_OPT_XOR_PUSH)
// flag page: 3 arrays of CKPT_MAX_GROUP uint32, each on its own 128-B line
enum Stage { kReady = 0, kRel = 1, kDone = 2, kNumStages = 3 };
constexpr uint64_t kFlagStride = 32;  // uint32 per stage line
constexpr uint64_t kFlagBytes = 4096;  // REL and DONE lines (READY line unused)
// READY is per bucket: row j (written by member j) holds the flag of bucket seq at index
// seq % kMaxB -- per-bucket because the single-launch pack completes buckets out of order.
constexpr uint32_t kMaxB = 16384;
constexpr uint64_t kFlagAlloc = kFlagBytes + (uint64_t)CKPT_MAX_GROUP * kMaxB * 4;
inline uint32_t *ready_row(uint32_t *flags, uint32_t j) { return flags + kFlagBytes / 4 + (uint64_t)j * kMaxB; }
// IPC handle of the member's parity buffer, written into its own flag page by
// ckpt_protect (the parity is allocated after the handle blobs were exchanged); a survivor
// reads the lost member's copy there and maps it for the rebuild (rebuild_map_parity).
constexpr uint64_t kParityHandleOff = 2048;
// Group abort word (u32 at this byte offset of every member's flag page): a member whose
// collective operation fails writes (its index + 1) into every peer's page; a peer blocked
// in a host-side wait sees it within ~20 ms and fails with EPEER instead of waiting out
// CKPT_TIMEOUT_S.  After an abort the group must be re-created.
constexpr uint64_t kAbortOff = 1024;
static_assert(kNumStages * kFlagStride * 4 <= kAbortOff && kAbortOff + 4 <= kParityHandleOff, "abort word placement");
static_assert(kNumStages * kFlagStride * 4 <= kParityHandleOff, "flag lines overlap the parity handle");
static_assert(kParityHandleOff + sizeof(cudaIpcMemHandle_t) <= kFlagBytes, "parity handle beyond the flag page");

struct HandleBlob {  // exported by ckpt_export_handle; fixed layout, <= CKPT_HANDLE_BYTES
    uint32_t magic, version;
    int32_t device;
    int32_t pid;
    uint64_t L;             // this rank's packed length L_j
    uint64_t align, unit;   // options that must agree
    uint64_t slot_bytes;    // ring slot capacity
    uint32_t n_slots;       // 0 = full copy
    uint32_t full_copy;
    uint64_t staging_bytes;
    uint64_t nonce;         // random per context; member 0's names the group's shm arena
    uint64_t arena_key;     // persistent arena key (0 = none); all members must agree
    uint64_t attached_id;   // committed snapshot id found in this member's persistent arena
    char host[64];
    uint32_t opt_flags;     // CKPT_OPT_REBUILD_SHARES must agree
    uint32_t reserved0;
    cudaIpcMemHandle_t staging_h;
    cudaIpcMemHandle_t flags_h;
};
static_assert(sizeof(HandleBlob) <= CKPT_HANDLE_BYTES, "blob too large");

inline uint64_t align_up(uint64_t x, uint64_t a) { return a ? (x + a - 1) / a * a : x; }
inline uint32_t sigma(uint32_t r, uint32_t j) { return r - (r > j ? 1u : 0u); }

struct Segment {
    uint64_t dev, nbytes, off;
    uint32_t dtype, role, flags;
    std::string name;
};

struct TimedLaunch {
    cudaEvent_t a, b;
    int kind;  // 0 pack 1 xor 2 unpack 3 rebuild 4 CE mirror gather
};

enum HostKind { kNone = 0, kCudaHost = 1, kAnon = 2, kShmOwn = 3, kShmPeer = 4, kView = 5 };
struct HostBuf {
    uint8_t *p = nullptr;
    uint64_t bytes = 0;
    int kind = kNone;
    bool registered = false;
    std::string name;  // shm object name (kShmOwn: unlinked at free)
};
// Persistent-arena metadata (its own 4 KiB shm object per member): geometry + the
// committed version, published with one atomic 64-bit store after the image is complete.
struct ArenaMeta {
    uint32_t magic, version;
    uint64_t L, Lstar, unit;
    uint32_t m, me, scheme, nbuf, align, reserved;
    uint64_t state;  // (completed_id << 8) | (completed_index + 1); 0 = nothing committed
};
constexpr uint32_t kMetaMagic = 0x41464552u;  // "REFA"
}  // namespace reft

struct ckpt_ctx {
    int device = -1;
    ckpt_options opt{};
    int sm_count = 148;
    int max_ctas = 296;
    int xor_ctas = 296;  // CTA budget of the XOR kernels (CKPT_XOR_CTAS overrides)
    int xor_ctas_push = 32;  // CTAs of the push-mode encode (CKPT_XOR_CTAS overrides)
    int sticky = CKPT_OK;
    std::string sticky_msg;

    // registration / plan
    bool registered = false;
    std::vector<Segment> segs;
    uint64_t L = 0;  // L_j
    std::vector<PackChunk> chunks;
    PackChunk *d_chunks = nullptr;
    const uint32_t *d_tile_first = nullptr;  // inside the d_chunks allocation
    std::vector<uint32_t> tile_first;        // host copy (CE pack)
    ckpt_layout layout{};

    // device staging (exported)
    bool full_copy = false;
    uint32_t n_slots = 0;
    uint64_t slot_bytes = 0;
    uint8_t *staging = nullptr;
    uint64_t staging_bytes = 0;
    uint32_t *flags = nullptr;  // local flag page (device), written by peers
    uint32_t *counters = nullptr;  // per-bucket CTA completion counters (single-launch pack)
    uint32_t *window = nullptr;    // HAS window word (device, CKPT_WINDOW_* mask), written by memops
    uint64_t has_bubble_bytes = UINT64_MAX;  // Alg 1 split: image bytes snapshotted in bubbles
    uint64_t has_compute_bytes = UINT64_MAX; // Layer 2 share after them; the rest is Layer 3

    // group
    bool grouped = false;  // ckpt_protect succeeded (m >= 2) or m == 1 arena set up
    uint32_t m = 1, me = 0, transport = CKPT_GROUP_IPC;
    uint64_t Lstar = 0, unit = 0;
    uint64_t peer_L[CKPT_MAX_GROUP] = {};
    uint8_t *peer_staging[CKPT_MAX_GROUP] = {};
    uint32_t *peer_flags[CKPT_MAX_GROUP] = {};
    bool peer_opened[CKPT_MAX_GROUP] = {};
    uint8_t *peer_parity[CKPT_MAX_GROUP] = {};  // mapped on first rebuild of that member
    bool peer_parity_opened[CKPT_MAX_GROUP] = {};
    bool parity_peers_mapped = false;
    bool abort_sent = false;  // this member wrote its abort word into every peer's page
    ckpt_ctx *members[CKPT_MAX_GROUP] = {};

    // CE gather buffer (CKPT_OPT_CE_GATHER; local): m-1 unit streams per bucket
    uint8_t *gather = nullptr;
    uint64_t gather_bytes = 0;
    // parity (local, not exported)
    uint8_t *parity = nullptr;
    uint64_t parity_bytes = 0, parity_slot_bytes = 0;

    // host arena
    HostBuf hdata[2], hpar[2];
    // protection scheme and the shared-memory arena (CKPT_OPT_SHM_ARENA): one file per
    // member and host buffer, [data L*][parity P][ARC copy data L*][ARC copy parity P]
    uint32_t scheme = CKPT_SCHEME_AEC;
    bool arc = false, aec = true;
    uint64_t my_nonce = 0, group_nonce = 0;
    HostBuf shm_own[2], shm_hold[2], shm_next[2];  // mine, my ARC holder's, member me+1's
    uint8_t *harc[2] = {}, *harcp[2] = {};          // the ARC copy I hold (of member me+1)
    bool arc_dirty[2] = {false, false};             // its zero pad was poisoned
    // persistent arena (options.arena_key != 0)
    HostBuf meta_buf;
    ArenaMeta *meta = nullptr;
    uint32_t arena_member = 0;
    uint64_t attached_id = 0;  // committed id found at registration (0 = none)
    int attached_idx = -1;
    uint64_t group_version = 0;  // max committed id over the group at ckpt_protect
    int nbuf = 2;
    int completed = -1, ongoing = 0;
    bool pad_dirty[2] = {false, false};  // zero pad [L, L*) overwritten by ckpt_forget
    uint64_t completed_id = 0;
    uint64_t staging_id = 0;  // id of the image the device staging + parity hold (0: none)
    bool staging_poisoned = false;  // ckpt_forget wrote over the staging's zero gaps
    bool host_pending = false;      // a rebuilt image is still being copied to host (ev_done)
    bool done_enqueued = false;     // the snapshot's completion waits already sit on sW
    std::vector<std::thread> host_bg;  // background host copies of an ARC restore (host_sync joins)

    // streams / events
    cudaStream_t sP = nullptr, sX = nullptr, sC = nullptr, sW = nullptr, sG = nullptr;
    cudaEvent_t ev_capture = nullptr, ev_pack_all = nullptr, ev_done = nullptr, ev_t0 = nullptr,
                ev_t1 = nullptr;
    std::vector<cudaEvent_t> ev_packed, ev_xored, ev_d2h_data, ev_d2h_par, ev_h2d, ev_kdone, ev_gathered;
    // LOCAL transport: per-stage per-slot signal events
    std::vector<cudaEvent_t> ev_sig[kNumStages];

    // op state
    uint32_t seq = 0;
    uint64_t next_id = 1;
    uint64_t pending_id = 0;   // issued snapshot not yet waited
    bool requested = false;    // LOCAL: ckpt_snapshot called, group not yet issued
    bool issued = false;
    // HAS windows (CKPT_OPT_WINDOWED, IPC / single member): the window-gated copies are
    // enqueued progressively, at most kGatedAhead beyond the last completed one, so the
    // caller's thread never blocks on a full stream queue while the windows it is about to
    // open are still closed (see issue_gated)
    uint64_t gate_next = 0, gate_total = 0;
    bool gate_tail = false;    // stage_finish still to issue
    uint64_t req_bucket = 0;
    uint64_t op_B = 0, op_NB = 0;
    uint32_t op_seq_base = 0;
    bool rebuild_requested = false;
    int32_t rebuild_lost = -1;
    bool recover_requested = false;
    uint32_t recover_mask = 0;
    void *recover_stream = nullptr;

    // stats
    ckpt_stats st{};
    std::vector<TimedLaunch> timed;
    size_t timed_used = 0;
};


// ------------------------------------------------------------------ helpers -------
static inline bool device_only(const ckpt_ctx *c) { return (c->opt.flags & CKPT_OPT_DEVICE_ONLY) != 0; }

// The device staging (and parity buffer) still hold the completed image: true in
// DEVICE_ONLY mode, and with full-copy staging from a commit until the next snapshot
// packs over it (or ckpt_forget declares the device lost).
static inline bool device_image_valid(const ckpt_ctx *c) {
    if (device_only(c)) return true;
    return c->full_copy && !(c->opt.flags & CKPT_OPT_HOST_LOAD) && c->staging_id != 0 &&
           c->staging_id == c->completed_id && c->completed >= 0;
}

static inline uint64_t parity_bytes_of(const ckpt_ctx *c) { return c->m >= 2 && c->aec ? c->Lstar / (c->m - 1) : 0; }

static inline uint64_t shm_bytes(const ckpt_ctx *c) {
    const uint64_t P = parity_bytes_of(c);
    return c->Lstar + P + (c->arc ? c->Lstar + P : 0);
}

static inline bool use_shm(const ckpt_ctx *c) { return (c->opt.flags & CKPT_OPT_SHM_ARENA) != 0; }

// ------------------------------------------------------------------ geometry helpers
static inline uint64_t bucket_begin(const ckpt_ctx *c, uint64_t k) { return k * c->op_B; }

static inline uint64_t bucket_end(const ckpt_ctx *c, uint64_t k) { return std::min((k + 1) * c->op_B, c->Lstar); }

static inline uint64_t valid_in_bucket(uint64_t Lj, uint64_t bb, uint64_t be) {
    return Lj <= bb ? 0 : std::min(Lj, be) - bb;
}

static inline uint32_t slot_of(const ckpt_ctx *c, uint64_t k) { return c->full_copy ? (uint32_t)k : (uint32_t)(k % c->n_slots); }

static inline uint8_t *slot_ptr(const ckpt_ctx *c, uint8_t *base, uint64_t k) {
    return c->full_copy ? base + bucket_begin(c, k) : base + (uint64_t)(k % c->n_slots) * c->slot_bytes;
}

static inline uint8_t *parity_slot_ptr_at(const ckpt_ctx *c, uint8_t *parity, uint64_t k) {
    return c->full_copy ? parity + bucket_begin(c, k) / (c->m - 1)
                        : parity + (uint64_t)(k % c->n_slots) * c->parity_slot_bytes;
}

static inline uint8_t *parity_slot_ptr(const ckpt_ctx *c, uint64_t k) { return parity_slot_ptr_at(c, c->parity, k); }

// Alg 1 placement of bucket k (ckpt_has_apply_layers): the buckets that start below the
// split go out only in bubbles; the next compute_bytes alongside computation -- or in a
// bubble, which is never worse (reading Q26); the rest also in communication windows
// (Layer 3, reading Q28).  The wait passes when (window & mask) != 0.
static inline uint32_t window_of(const ckpt_ctx *c, uint64_t k) {
    const uint64_t b = bucket_begin(c, k);
    if (b < c->has_bubble_bytes) return CKPT_WINDOW_BUBBLE;
    const uint64_t l2 = c->has_compute_bytes > UINT64_MAX - c->has_bubble_bytes ? UINT64_MAX
                                                                               : c->has_bubble_bytes + c->has_compute_bytes;
    return b < l2 ? (CKPT_WINDOW_BUBBLE | CKPT_WINDOW_COMPUTE)
                  : (CKPT_WINDOW_BUBBLE | CKPT_WINDOW_COMPUTE | CKPT_WINDOW_COMM);  // Layer 3 (P.425)
}

static inline uint32_t bucket_seq(const ckpt_ctx *c, uint64_t k) { return c->op_seq_base + (uint32_t)k + 1; }

static inline bool ring_reuse(const ckpt_ctx *c, uint64_t k) { return !c->full_copy && k >= c->n_slots; }

// CE gather (CKPT_OPT_CE_GATHER): copy engines pull unit sigma(me, j) of every stripe
// of peer j's slot (a 2-D copy: width u, source pitch (m-1)u) into local stream jj;
// bytes beyond the peer's L_j are zero-filled (Q5).  Zero SMs on NVLink.
static inline uint64_t gather_stride(const ckpt_ctx *c, uint64_t k) {
    return c->full_copy ? (bucket_end(c, k) - bucket_begin(c, k)) / (c->m - 1) : c->parity_slot_bytes;
}

static inline uint8_t *gather_slot_ptr(const ckpt_ctx *c, uint64_t k) {
    return c->full_copy ? c->gather + bucket_begin(c, k)
                        : c->gather + (uint64_t)(k % c->n_slots) * c->parity_slot_bytes * (c->m - 1);
}

// The buffer the survivors' completed image sits in: every member flips its double
// buffer at the same commits, so the lost member rebuilds into that index and keeps its
// `ongoing` in step with the group (ARC pushes rely on identical indices).
static inline int rb_target(const ckpt_ctx *c) { return c->nbuf == 2 ? c->ongoing ^ 1 : 0; }

// Background host restore: with full-copy staging (and no ARC copies to re-create from
// it) the lost member's rebuild returns as soon as its DEVICE image is complete -- the
// REL waits sit on the kernel stream, DONE is signalled from there -- while the D2H that
// re-protects its host image keeps running on the copy stream (host_sync waits for it).
static inline bool async_host_restore(const ckpt_ctx *c) { return c->full_copy && !device_only(c) && !c->arc; }

// ------------------------------------------------------------------ recover (1-2 losses)
// The oracle's oracle_recover, step by step: (1) ARC restore of every lost member whose
// holder survived (the member copies its image out of the holder's shared file), (2)
// AEC rebuild of one remaining loss (collective, rebuild_aec), (3) every lost member
// re-creates the ARC copy it holds from member me+1's completed image.
static inline uint32_t holder_of(const ckpt_ctx *c, uint32_t x) { return (x + c->m - 1) % c->m; }

// ------------------------------------------------------------------ internal API --
int set_dev(ckpt_ctx *c);
int ensure_events(std::vector<cudaEvent_t> &v, size_t n);
void destroy_events(std::vector<cudaEvent_t> &v);
int timed_begin(ckpt_ctx *c, cudaStream_t s, int kind, TimedLaunch **out);
int timed_end(TimedLaunch *t, cudaStream_t s);
int harvest_timing(ckpt_ctx *c);
void prefault(uint8_t *p, uint64_t len);
void parallel_memcpy(uint8_t *dst, const uint8_t *src, uint64_t n);
int host_alloc(HostBuf &b, uint64_t bytes);
std::string shm_name(uint64_t nonce, uint32_t member, int buf);
int shm_create(HostBuf &b, const std::string &name, uint64_t bytes, bool reg = true);
int shm_map(HostBuf &b, const std::string &name, uint64_t bytes, bool reg);
int shm_attach(HostBuf &b, const std::string &name, uint64_t bytes, bool reg);
std::string meta_name(uint64_t key, uint32_t member);
void host_free(HostBuf &b);
int alloc_arena(ckpt_ctx *c);
void meta_commit(ckpt_ctx *c);
int ensure_holder_mapped(ckpt_ctx *c);
int ensure_next_mapped(ckpt_ctx *c);
int setup_ungrouped(ckpt_ctx *c);
int sig_signal(ckpt_ctx *c, cudaStream_t s, int stage, uint32_t seq, uint32_t slot);
int sig_wait(ckpt_ctx *c, cudaStream_t s, uint32_t j, int stage, uint32_t seq, uint32_t slot);
int wait_all(ckpt_ctx *c, cudaStream_t s, int stage, uint32_t seq, uint32_t slot, int32_t skip = -1);
int do_pack_ce(ckpt_ctx *c, uint64_t k, uint8_t *slot, cudaStream_t s, bool unpack);
int do_pack(ckpt_ctx *c, uint64_t k, uint8_t *slot, cudaStream_t s, bool unpack);
int do_encode_range(ckpt_ctx *c, uint64_t k, uint64_t bb, uint64_t be, cudaStream_t s);
int do_encode(ckpt_ctx *c, uint64_t k, cudaStream_t s);
int do_rebuild_row(ckpt_ctx *c, uint64_t k, uint32_t kl, cudaStream_t s);
int do_encode_lost_share(ckpt_ctx *c, uint64_t k, uint32_t kl, cudaStream_t s);
int rebuild_map_parity(ckpt_ctx *c, uint32_t kl, bool wait = false);
bool xor_push(const ckpt_ctx *c);
int push_issue(ckpt_ctx *c);
int push_collect(ckpt_ctx *c);
// Who re-encodes the lost member's parity row (Q27): the survivors in shares (the default
// for m >= 3, forced at any m by CKPT_OPT_REBUILD_SHARES) or the lost member itself,
// pulling L* more over NVLink (the default at m = 2, forced by CKPT_OPT_REBUILD_SELF).
// Round-2 A/B (tools/rb_share_ab.sh): C5 m = 4 54.5 / 55.0 ms in shares vs 70.7 / 70.4 ms
// self; C2 m = 2 35.6 / 34.6 ms vs 32.8 / 32.9 ms.
static inline bool rebuild_self_encode(const ckpt_ctx *c) {
    if (c->opt.flags & CKPT_OPT_REBUILD_SELF) return true;
    return !(c->opt.flags & CKPT_OPT_REBUILD_SHARES) && c->m <= 2;
}
void clean_pad(ckpt_ctx *c, int buf);
int check_sticky(ckpt_ctx *c);
void make_sticky(ckpt_ctx *c, int rc);
void group_abort(ckpt_ctx *c);
uint32_t peer_aborted(ckpt_ctx *c);
int host_sync(ckpt_ctx *c);
int issue_gated_more(ckpt_ctx *c);  // HAS windows: enqueue more window-gated copies
uint64_t effective_bucket(const ckpt_ctx *c, uint64_t req);
bool single_launch(const ckpt_ctx *c);
int issue_pack_all(ckpt_ctx *c);
int prepare_op(ckpt_ctx *c, uint64_t B);
int stage_pack(ckpt_ctx *c, uint64_t k);
int do_gather_ce(ckpt_ctx *c, uint64_t k, cudaStream_t s);
int do_encode_gathered(ckpt_ctx *c, uint64_t k, cudaStream_t s);
int stage_xor_all(ckpt_ctx *c);
bool xor_in_one_launch(const ckpt_ctx *c);
int stage_xor(ckpt_ctx *c, uint64_t k);
int stage_copy_parity(ckpt_ctx *c, uint64_t k);
int stage_copy(ckpt_ctx *c, uint64_t k, bool with_parity = true);
int stage_finish(ckpt_ctx *c);
int begin_member(ckpt_ctx *c, cudaStream_t caller, uint64_t B);
int sync_stream_timeout(ckpt_ctx *c, cudaStream_t s, const char *what);
int wait_done_all(ckpt_ctx *c, uint32_t done_seq);
int rb_stage1(ckpt_ctx *c, uint64_t b, uint32_t kl);
int rb_stage2(ckpt_ctx *c, uint64_t b, uint32_t kl);
int rb_stage3(ckpt_ctx *c, uint64_t b, uint32_t kl);
int rb_finish(ckpt_ctx *c, uint32_t kl);
int rb_commit(ckpt_ctx *c, uint32_t kl, uint64_t version);
int rebuild_aec(ckpt_ctx *c, int32_t lost, void *stream);
int recover_plan(const ckpt_ctx *c, uint32_t mask, int32_t *remaining);
int recover_step1(ckpt_ctx *c, uint32_t mask, uint64_t version);
int recover_step3(ckpt_ctx *c, uint32_t mask);
