// ckpt_lib.cu -- host side of libreft_ckpt: C ABI, planner, pinned host arena, peer
// mapping (CUDA IPC / in-process), and the bucket pipeline scheduler.
//
// Pipeline of one snapshot, per bucket k (slot s = k mod n_slots):
//   stream P (pack)  : [slot reuse: own D2H(k-n) done, every peer's XOR(k-n) done]
//                      pack(k) -> READY(k) to every peer
//   stream X (xor)   : own pack(k), every peer's READY(k), [parity slot D2H(k-n)]
//                      xor_encode(k) over NVLink -> REL(k) to every peer
//   stream C (copy)  : D2H data slot(k) ; D2H parity slot(k)   (copy engine, no SMs)
//   end              : DONE to every peer; ckpt_wait waits DONE from all, commits.
// Cross-rank signals are 32-bit sequence numbers.  IPC groups write them into the
// peers' flag pages with stream memory operations (cuStreamWriteValue32 /
// cuStreamWaitValue32: zero SMs, no NCCL on the data path); LOCAL groups (all
// members in this process) use CUDA events instead.
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

#include "../../include/ckpt.h"
#include "ckpt_kernels.cuh"

using namespace reft;

// NVTX ranges around the public calls (host-side enqueue/wait), for nsys timelines.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// ------------------------------------------------------------------ errors ----------
static thread_local std::string g_last_error;

static int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
static int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

#define CUDA_TRY(expr)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (expr);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            return fail(CKPT_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                              \
    } while (0)

// ------------------------------------------------------------------ driver memops ---
static PFN_cuStreamWaitValue32_v8000 p_wait32 = nullptr;
static PFN_cuStreamWriteValue32_v8000 p_write32 = nullptr;
static std::once_flag g_memop_once;
static int g_memop_status = CKPT_ECUDA;

static int load_memops() {
    std::call_once(g_memop_once, [] {
        cudaDriverEntryPointQueryResult q1, q2;
        void *f1 = nullptr, *f2 = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f1, cudaEnableDefault, &q1) == cudaSuccess &&
            cudaGetDriverEntryPoint("cuStreamWriteValue32", &f2, cudaEnableDefault, &q2) == cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && f1 && f2) {
            p_wait32 = (PFN_cuStreamWaitValue32_v8000)f1;
            p_write32 = (PFN_cuStreamWriteValue32_v8000)f2;
            g_memop_status = CKPT_OK;
        }
    });
    return g_memop_status;
}

// ------------------------------------------------------------------ constants -------
namespace {
constexpr uint32_t kMagic = 0x52454654u;  // "REFT"
constexpr uint32_t kAbiVersion = 1;
// flag page: 3 arrays of CKPT_MAX_GROUP uint32, each on its own 128-B line
enum Stage { kReady = 0, kRel = 1, kDone = 2, kNumStages = 3 };
constexpr uint64_t kFlagStride = 32;  // uint32 per stage line
constexpr uint64_t kFlagBytes = 4096;  // REL and DONE lines (READY line unused)
// READY is per bucket: row j (written by member j) holds the flag of bucket seq at index
// seq % kMaxB -- per-bucket because the single-launch pack completes buckets out of order.
constexpr uint32_t kMaxB = 16384;
constexpr uint64_t kFlagAlloc = kFlagBytes + (uint64_t)CKPT_MAX_GROUP * kMaxB * 4;
inline uint32_t *ready_row(uint32_t *flags, uint32_t j) { return flags + kFlagBytes / 4 + (uint64_t)j * kMaxB; }

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
    int kind;  // 0 pack 1 xor 2 unpack 3 rebuild
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
}  // namespace

struct ckpt_ctx {
    int device = -1;
    ckpt_options opt{};
    int sm_count = 148;
    int max_ctas = 296;
    int xor_ctas = 296;  // CTA budget of the XOR kernels (CKPT_XOR_CTAS overrides)
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
    uint32_t *window = nullptr;    // HAS window flag (device, bit 0 = open), written by memops

    // group
    bool grouped = false;  // ckpt_protect succeeded (m >= 2) or m == 1 arena set up
    uint32_t m = 1, me = 0, transport = CKPT_GROUP_IPC;
    uint64_t Lstar = 0, unit = 0;
    uint64_t peer_L[CKPT_MAX_GROUP] = {};
    uint8_t *peer_staging[CKPT_MAX_GROUP] = {};
    uint32_t *peer_flags[CKPT_MAX_GROUP] = {};
    bool peer_opened[CKPT_MAX_GROUP] = {};
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

// ------------------------------------------------------------------ small helpers ---
static int set_dev(ckpt_ctx *c) {
    CUDA_TRY(cudaSetDevice(c->device));
    return CKPT_OK;
}

static int ensure_events(std::vector<cudaEvent_t> &v, size_t n) {
    while (v.size() < n) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        v.push_back(e);
    }
    return CKPT_OK;
}

static void destroy_events(std::vector<cudaEvent_t> &v) {
    for (auto e : v) cudaEventDestroy(e);
    v.clear();
}

// Timed launch bracket (CKPT_OPT_TIMING): events on the launching stream.
static int timed_begin(ckpt_ctx *c, cudaStream_t s, int kind, TimedLaunch **out) {
    *out = nullptr;
    if (!(c->opt.flags & CKPT_OPT_TIMING)) return CKPT_OK;
    if (c->timed_used == c->timed.size()) {
        TimedLaunch t;
        CUDA_TRY(cudaEventCreate(&t.a));
        CUDA_TRY(cudaEventCreate(&t.b));
        c->timed.push_back(t);
    }
    TimedLaunch *t = &c->timed[c->timed_used++];
    t->kind = kind;
    CUDA_TRY(cudaEventRecord(t->a, s));
    *out = t;
    return CKPT_OK;
}

static int timed_end(TimedLaunch *t, cudaStream_t s) {
    if (t) CUDA_TRY(cudaEventRecord(t->b, s));
    return CKPT_OK;
}

static int harvest_timing(ckpt_ctx *c) {
    for (size_t i = 0; i < c->timed_used; ++i) {
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, c->timed[i].a, c->timed[i].b));
        switch (c->timed[i].kind) {
            case 0: c->st.pack_ms += ms; break;
            case 1: c->st.xor_ms += ms; break;
            case 2: c->st.unpack_ms += ms; break;
            default: c->st.rebuild_ms += ms; break;
        }
    }
    c->timed_used = 0;
    return CKPT_OK;
}

// ------------------------------------------------------------------ host arena ------
// Pinned host memory: anonymous mmap with transparent huge pages, pre-faulted by a few
// threads, then cudaHostRegister (page-locked, device-mapped).  Falls back to
// cudaHostAlloc.  Zero-filled (the pad of the image must read as zero, Q5).
static void prefault(uint8_t *p, uint64_t len) {
    unsigned nt = std::min(16u, std::max(1u, std::thread::hardware_concurrency() / 2));
    std::vector<std::thread> th;
    const uint64_t per = align_up(len / nt + 1, 2ull << 20);
    for (unsigned i = 0; i < nt; ++i)
        th.emplace_back([=] {
            for (uint64_t o = i * per; o < std::min(len, (i + 1) * per); o += 4096) p[o] = 0;
        });
    for (auto &t : th) t.join();
}

// Host copies of whole images (ARC restore): a few threads, large pieces.
static void parallel_memcpy(uint8_t *dst, const uint8_t *src, uint64_t n) {
    unsigned nt = std::min(16u, std::max(1u, std::thread::hardware_concurrency() / 2));
    if (n < (64ull << 20)) nt = 1;
    std::vector<std::thread> th;
    const uint64_t per = align_up(n / nt + 1, 4096);
    for (unsigned i = 0; i < nt; ++i)
        th.emplace_back([=] {
            const uint64_t lo = i * per, hi = std::min(n, (i + 1) * per);
            if (lo < hi) memcpy(dst + lo, src + lo, hi - lo);
        });
    for (auto &t : th) t.join();
}

static int host_alloc(HostBuf &b, uint64_t bytes) {
    b = HostBuf{};
    if (bytes == 0) return CKPT_OK;
    uint64_t len = align_up(bytes, 2ull << 20);
    void *p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
    if (p != MAP_FAILED) {
#ifdef MADV_HUGEPAGE
        madvise(p, len, MADV_HUGEPAGE);
#endif
        prefault((uint8_t *)p, len);
        if (cudaHostRegister(p, len, cudaHostRegisterPortable) == cudaSuccess) {
            b.p = (uint8_t *)p;
            b.bytes = len;
            b.kind = kAnon;
            b.registered = true;
            return CKPT_OK;
        }
        cudaGetLastError();
        munmap(p, len);
    }
    void *q = nullptr;
    if (cudaHostAlloc(&q, bytes, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return fail(CKPT_ENOMEM, "pinned host allocation of %llu bytes failed", (unsigned long long)bytes);
    }
    memset(q, 0, bytes);
    b.p = (uint8_t *)q;
    b.bytes = bytes;
    b.kind = kCudaHost;
    return CKPT_OK;
}

// POSIX shared memory: create (owner) or map (peer, waiting up to CKPT_TIMEOUT_S for the
// owner to create it at full size).  Pinned with cudaHostRegister when `reg`.
static std::string shm_name(uint64_t nonce, uint32_t member, int buf) {
    char s[64];
    snprintf(s, sizeof s, "/reft-%016llx-%u-%d", (unsigned long long)nonce, member, buf);
    return s;
}

static int shm_create(HostBuf &b, const std::string &name, uint64_t bytes) {
    b = HostBuf{};
    const uint64_t len = align_up(std::max<uint64_t>(bytes, 1), 2ull << 20);
    int fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) return fail(CKPT_ENOMEM, "shm_open(%s) failed: %s", name.c_str(), strerror(errno));
    if (ftruncate(fd, (off_t)len) != 0) {
        close(fd);
        shm_unlink(name.c_str());
        return fail(CKPT_ENOMEM, "ftruncate(%s, %llu) failed: %s", name.c_str(), (unsigned long long)len, strerror(errno));
    }
    void *p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) {
        shm_unlink(name.c_str());
        return fail(CKPT_ENOMEM, "mmap(%s) failed: %s", name.c_str(), strerror(errno));
    }
#ifdef MADV_HUGEPAGE
    madvise(p, len, MADV_HUGEPAGE);
#endif
    prefault((uint8_t *)p, len);  // allocates the tmpfs pages (zero-filled)
    if (cudaHostRegister(p, len, cudaHostRegisterPortable) != cudaSuccess) {
        cudaGetLastError();
        munmap(p, len);
        shm_unlink(name.c_str());
        return fail(CKPT_ENOMEM, "cudaHostRegister of shm %s (%llu bytes) failed", name.c_str(), (unsigned long long)len);
    }
    b.p = (uint8_t *)p;
    b.bytes = len;
    b.kind = kShmOwn;
    b.registered = true;
    b.name = name;
    return CKPT_OK;
}

static int shm_map(HostBuf &b, const std::string &name, uint64_t bytes, bool reg) {
    b = HostBuf{};
    const uint64_t len = align_up(std::max<uint64_t>(bytes, 1), 2ull << 20);
    double limit = 600.0;
    if (const char *e = getenv("CKPT_TIMEOUT_S")) limit = atof(e);
    auto t0 = std::chrono::steady_clock::now();
    int fd = -1;
    for (;;) {
        fd = shm_open(name.c_str(), O_RDWR, 0600);
        if (fd >= 0) {
            struct stat st;
            if (fstat(fd, &st) == 0 && (uint64_t)st.st_size >= len) break;
            close(fd);
            fd = -1;
        }
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit)
            return fail(CKPT_EPEER, "shm %s did not appear within %.0f s", name.c_str(), limit);
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
    void *p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) return fail(CKPT_EPEER, "mmap(%s) failed: %s", name.c_str(), strerror(errno));
    if (reg && cudaHostRegister(p, len, cudaHostRegisterPortable) != cudaSuccess) {
        cudaGetLastError();
        munmap(p, len);
        return fail(CKPT_EPEER, "cudaHostRegister of peer shm %s failed", name.c_str());
    }
    b.p = (uint8_t *)p;
    b.bytes = len;
    b.kind = kShmPeer;
    b.registered = reg;
    b.name = name;
    return CKPT_OK;
}

// Re-attach an existing shared-memory object of at least `bytes` (persistent arena): the
// contents are kept (MAP_POPULATE touches the pages without writing them).
static int shm_attach(HostBuf &b, const std::string &name, uint64_t bytes, bool reg) {
    b = HostBuf{};
    const uint64_t len = align_up(std::max<uint64_t>(bytes, 1), 2ull << 20);
    int fd = shm_open(name.c_str(), O_RDWR, 0600);
    if (fd < 0) return CKPT_ENOSNAP;
    struct stat st;
    if (fstat(fd, &st) != 0 || (uint64_t)st.st_size < len) {
        close(fd);
        return CKPT_ENOSNAP;
    }
    void *p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_POPULATE, fd, 0);
    close(fd);
    if (p == MAP_FAILED) return fail(CKPT_ENOMEM, "mmap(%s) failed: %s", name.c_str(), strerror(errno));
    if (reg && cudaHostRegister(p, len, cudaHostRegisterPortable) != cudaSuccess) {
        cudaGetLastError();
        munmap(p, len);
        return fail(CKPT_ENOMEM, "cudaHostRegister of persistent shm %s failed", name.c_str());
    }
    b.p = (uint8_t *)p;
    b.bytes = len;
    b.kind = kShmPeer;  // persistent: unmapped but never unlinked by this process
    b.registered = reg;
    b.name = name;
    return CKPT_OK;
}

static std::string meta_name(uint64_t key, uint32_t member) {
    char s[64];
    snprintf(s, sizeof s, "/reft-%016llx-%u-meta", (unsigned long long)key, member);
    return s;
}

extern "C" int ckpt_arena_unlink(uint64_t key, uint32_t m, uint32_t nbuf) {
    if (key == 0 || m == 0 || m > CKPT_MAX_GROUP || nbuf == 0 || nbuf > 2)
        return fail(CKPT_EINVAL, "arena_unlink: bad args");
    for (uint32_t j = 0; j < m; ++j) {
        shm_unlink(meta_name(key, j).c_str());
        for (uint32_t b = 0; b < nbuf; ++b) shm_unlink(shm_name(key, j, (int)b).c_str());
    }
    return CKPT_OK;
}

static void host_free(HostBuf &b) {
    if (!b.p) return;
    switch (b.kind) {
        case kCudaHost: cudaFreeHost(b.p); break;
        case kAnon:
        case kShmOwn:
        case kShmPeer:
            if (b.registered) cudaHostUnregister(b.p);
            munmap(b.p, b.bytes);
            if (b.kind == kShmOwn) shm_unlink(b.name.c_str());
            break;
        default: break;  // kView: not owned
    }
    b = HostBuf{};
}

// ------------------------------------------------------------------ planner ---------
extern "C" int ckpt_plan_layout(const uint64_t *nbytes, uint64_t n, uint32_t align, uint64_t *offsets,
                                uint64_t *L) {
    if (!L || (n && (!nbytes || !offsets)) || align == 0) return fail(CKPT_EINVAL, "plan_layout: bad args");
    uint64_t end = 0;
    for (uint64_t t = 0; t < n; ++t) {
        offsets[t] = align_up(end, align);
        end = offsets[t] + nbytes[t];
    }
    *L = align_up(end, align);
    return CKPT_OK;
}

extern "C" int ckpt_plan_common(const uint64_t *Lj, uint32_t m, uint64_t unit, uint64_t *L_star,
                                uint64_t *unit_eff) {
    if (!Lj || !L_star || !unit_eff || m < 1 || m > CKPT_MAX_GROUP)
        return fail(CKPT_EINVAL, "plan_common: bad args");
    uint64_t mx = 0;
    for (uint32_t j = 0; j < m; ++j) mx = std::max(mx, Lj[j]);
    if (m == 1) {
        *L_star = Lj[0];
        *unit_eff = unit;
    } else if (unit == 0) {  // SPEC S.378 whole-shard split: one stripe
        *L_star = align_up(mx, (uint64_t)(m - 1) * 256);
        *unit_eff = *L_star / (m - 1);
    } else {
        *L_star = align_up(mx, (uint64_t)(m - 1) * unit);
        *unit_eff = unit;
    }
    return CKPT_OK;
}

// ------------------------------------------------------------------ lifecycle -------
extern "C" void ckpt_options_default(ckpt_options *o) {
    if (!o) return;
    memset(o, 0, sizeof *o);
    o->struct_size = sizeof(ckpt_options);
    o->align = 256;
    o->stripe_unit = 64 * 1024;
    o->bucket_bytes = 64ull << 20;
    o->n_slots = 4;
    o->host_buffers = 2;
    o->priority = INT32_MAX;  // resolved to the least priority at create
    o->max_ctas = 0;
    o->flags = 0;
}

extern "C" const char *ckpt_version(void) { return "reft-ckpt 0.1 sm_100a"; }

extern "C" const char *ckpt_strerror(int code) {
    switch (code) {
        case CKPT_OK: return "ok";
        case CKPT_EINVAL: return "invalid argument";
        case CKPT_ECUDA: return "CUDA error";
        case CKPT_ENOMEM: return "out of memory";
        case CKPT_ESTATE: return "invalid state for this call";
        case CKPT_EUNAVAIL: return "protection unavailable (group of one)";
        case CKPT_EMISMATCH: return "group geometry mismatch";
        case CKPT_EPEER: return "peer mapping failed";
        case CKPT_EBUSY: return "previous snapshot not waited";
        case CKPT_ENOSNAP: return "no completed snapshot";
        case CKPT_EUNRECOVERABLE: return "unrecoverable: more losses than tolerated";
        default: return "unknown error";
    }
}

extern "C" const char *ckpt_last_error(void) { return g_last_error.c_str(); }

extern "C" int ckpt_create(int device, const ckpt_options *o, ckpt_ctx **out) {
    if (!out) return fail(CKPT_EINVAL, "create: out is NULL");
    *out = nullptr;
    ckpt_options opt;
    ckpt_options_default(&opt);
    if (o) {
        if (o->struct_size != sizeof(ckpt_options)) return fail(CKPT_EINVAL, "create: struct_size mismatch");
        opt = *o;
    }
    if (opt.align < 16 || opt.align > 4096 || (opt.align & (opt.align - 1)))
        return fail(CKPT_EINVAL, "create: align must be a power of two in [16, 4096]");
    if (opt.stripe_unit % 16) return fail(CKPT_EINVAL, "create: stripe_unit must be a multiple of 16");
    if (opt.host_buffers != 1 && opt.host_buffers != 2) return fail(CKPT_EINVAL, "create: host_buffers must be 1 or 2");
    if (opt.n_slots == 1) return fail(CKPT_EINVAL, "create: n_slots must be 0 (full copy) or >= 2");
    if (opt.bucket_bytes < 4096) return fail(CKPT_EINVAL, "create: bucket_bytes must be >= 4096");
    if ((opt.flags & CKPT_OPT_DEVICE_ONLY) && opt.n_slots != 0)
        return fail(CKPT_EINVAL, "create: DEVICE_ONLY needs n_slots = 0 (the whole image in HBM)");
    if ((opt.flags & CKPT_OPT_TMA_PACK) && (opt.flags & CKPT_OPT_LSU_PACK))
        return fail(CKPT_EINVAL, "create: TMA_PACK and LSU_PACK are exclusive");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(CKPT_ECUDA, "create: no CUDA device available (no CPU fallback)");
    }
    if (device < 0 || device >= ndev) return fail(CKPT_EINVAL, "create: device %d out of range", device);
    ckpt_ctx *c = new ckpt_ctx();
    c->device = device;
    {
        std::random_device rd;
        c->my_nonce = ((uint64_t)rd() << 32) ^ rd() ^ ((uint64_t)getpid() << 16) ^
                      (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count();
    }
    c->opt = opt;
    c->nbuf = (int)opt.host_buffers;
    int rc = set_dev(c);
    if (rc) {
        delete c;
        return rc;
    }
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    if (cudaError_t e = preload_kernels(); e != cudaSuccess) {
        delete c;
        return fail(CKPT_ECUDA, "create: loading the kernels failed: %s", cudaGetErrorString(e));
    }
    c->max_ctas = opt.max_ctas ? (int)opt.max_ctas : 2 * c->sm_count;
    // measured: at m = 2 half the SMs read peers as fast as 2 x SMs (660 vs 671 GB/s), at
    // m = 4 they do not (497 vs 590 GB/s) -- the XOR keeps the full budget
    c->xor_ctas = c->max_ctas;
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    int prio = opt.priority == INT32_MAX ? least : std::min(least, std::max(greatest, (int)opt.priority));
    c->opt.priority = prio;
    cudaError_t e = cudaSuccess;
    cudaStream_t *ss[5] = {&c->sP, &c->sX, &c->sC, &c->sW, &c->sG};
    for (auto s : ss)
        if (e == cudaSuccess) e = cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, prio);
    cudaEvent_t *es[3] = {&c->ev_capture, &c->ev_pack_all, &c->ev_done};
    for (auto ev : es)
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev_t0);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev_t1);
    if (e == cudaSuccess) e = cudaMalloc(&c->window, 256);
    if (e == cudaSuccess) {
        const uint32_t one = 1;  // windows start open
        e = cudaMemcpy(c->window, &one, sizeof one, cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {
        ckpt_destroy(c);
        return fail(CKPT_ECUDA, "create: %s", cudaGetErrorString(e));
    }
    *out = c;
    return CKPT_OK;
}

extern "C" int ckpt_destroy(ckpt_ctx *c) {
    if (!c) return CKPT_OK;
    cudaSetDevice(c->device);
    cudaStream_t ss[5] = {c->sP, c->sX, c->sC, c->sW, c->sG};
    for (auto s : ss)
        if (s) cudaStreamSynchronize(s);
    for (uint32_t j = 0; j < CKPT_MAX_GROUP; ++j) {
        if (c->peer_opened[j]) {
            if (c->peer_staging[j]) cudaIpcCloseMemHandle(c->peer_staging[j]);
            if (c->peer_flags[j]) cudaIpcCloseMemHandle(c->peer_flags[j]);
        }
    }
    for (auto s : ss)
        if (s) cudaStreamDestroy(s);
    cudaEvent_t es[5] = {c->ev_capture, c->ev_pack_all, c->ev_done, c->ev_t0, c->ev_t1};
    for (auto e : es)
        if (e) cudaEventDestroy(e);
    destroy_events(c->ev_packed);
    destroy_events(c->ev_xored);
    destroy_events(c->ev_d2h_data);
    destroy_events(c->ev_d2h_par);
    destroy_events(c->ev_h2d);
    destroy_events(c->ev_kdone);
    destroy_events(c->ev_gathered);
    for (auto &v : c->ev_sig) destroy_events(v);
    for (auto &t : c->timed) {
        cudaEventDestroy(t.a);
        cudaEventDestroy(t.b);
    }
    if (c->d_chunks) cudaFree(c->d_chunks);
    if (c->staging) cudaFree(c->staging);
    if (c->flags) cudaFree(c->flags);
    if (c->counters) cudaFree(c->counters);
    if (c->window) cudaFree(c->window);
    if (c->parity) cudaFree(c->parity);
    if (c->gather) cudaFree(c->gather);
    for (int i = 0; i < 2; ++i) {
        host_free(c->hdata[i]);
        host_free(c->hpar[i]);
        host_free(c->shm_own[i]);
        host_free(c->shm_hold[i]);
        host_free(c->shm_next[i]);
    }
    host_free(c->meta_buf);
    cudaGetLastError();
    delete c;
    return CKPT_OK;
}

// ------------------------------------------------------------------ register --------
extern "C" int ckpt_register(ckpt_ctx *c, const ckpt_tensor *t, uint64_t n, const ckpt_layout *layout) {
    if (!c || !t || n == 0) return fail(CKPT_EINVAL, "register: null context/tensors or n == 0");
    if (c->registered) return fail(CKPT_ESTATE, "register: already registered");
    int rc = set_dev(c);
    if (rc) return rc;
    std::vector<Segment> segs(n);
    for (uint64_t i = 0; i < n; ++i) {
        if (!t[i].dev_ptr || t[i].nbytes == 0) return fail(CKPT_EINVAL, "register: tensor %llu null or empty", (unsigned long long)i);
        cudaPointerAttributes pa;
        if (cudaPointerGetAttributes(&pa, t[i].dev_ptr) != cudaSuccess || pa.type != cudaMemoryTypeDevice ||
            pa.device != c->device) {
            cudaGetLastError();
            return fail(CKPT_EINVAL, "register: tensor %llu is not device memory on device %d", (unsigned long long)i, c->device);
        }
        segs[i] = Segment{(uint64_t)(uintptr_t)t[i].dev_ptr, t[i].nbytes, 0, t[i].dtype, t[i].role, t[i].flags,
                          t[i].name ? t[i].name : ""};
    }
    // plan (reading Q6): registration order, A-aligned offsets, zero gaps.  Every
    // piece (data or zero gap) is cut at multiples of kTile bytes of image so that the
    // chunks of image tile i are exactly [tile_first[i], tile_first[i+1]).
    uint64_t end = 0;
    std::vector<PackChunk> ch;
    auto emit = [&ch](uint64_t src, uint64_t img, uint64_t nbytes, uint64_t seg) {
        for (uint64_t o = 0; o < nbytes;) {
            const uint64_t at = img + o;
            const uint64_t lim = std::min(nbytes - o, align_up(at + 1, kTile) - at);
            ch.push_back(PackChunk{src ? src + o : 0, at, lim, seg});
            o += lim;
        }
    };
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t off = align_up(end, c->opt.align);
        if (off > end) emit(0, end, off - end, i);  // zero gap
        segs[i].off = off;
        emit(segs[i].dev, off, segs[i].nbytes, i);
        end = off + segs[i].nbytes;
    }
    uint64_t L = align_up(end, c->opt.align);
    if (L > end) emit(0, end, L - end, n);
    if (ch.size() >= (1ull << 32)) return fail(CKPT_EINVAL, "register: state too large (chunk index overflow)");
    const uint64_t ntiles = (L + kTile - 1) / kTile;
    std::vector<uint32_t> tf(ntiles + 1);
    for (uint64_t t = 0, ci = 0; t <= ntiles; ++t) {
        while (ci < ch.size() && ch[ci].dst < t * kTile) ++ci;
        tf[t] = (uint32_t)ci;
    }
    // device staging: full image (n_slots == 0) or a ring of n_slots buckets
    c->full_copy = c->opt.n_slots == 0;
    c->n_slots = c->opt.n_slots;
    c->slot_bytes = align_up(c->opt.bucket_bytes, 4096);
    c->staging_bytes = c->full_copy ? std::max<uint64_t>(L, 4096) : (uint64_t)c->n_slots * c->slot_bytes;
    PackChunk *dch = nullptr;
    const uint64_t tbytes = ch.size() * sizeof(PackChunk), fbytes = tf.size() * sizeof(uint32_t);
    if (cudaMalloc(&dch, tbytes + fbytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(CKPT_ENOMEM, "register: chunk table allocation failed");
    }
    CUDA_TRY(cudaMemcpy(dch, ch.data(), tbytes, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy((uint8_t *)dch + tbytes, tf.data(), fbytes, cudaMemcpyHostToDevice));
    c->d_tile_first = (const uint32_t *)((uint8_t *)dch + tbytes);
    if (cudaMalloc(&c->staging, c->staging_bytes) != cudaSuccess ||
        cudaMalloc(&c->flags, kFlagAlloc) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(dch);
        if (c->staging) cudaFree(c->staging);
        c->staging = nullptr;
        return fail(CKPT_ENOMEM, "register: device staging of %llu bytes failed", (unsigned long long)c->staging_bytes);
    }
    CUDA_TRY(cudaMemset(c->flags, 0, kFlagAlloc));
    if (cudaMalloc(&c->counters, kMaxB * sizeof(uint32_t)) != cudaSuccess) {
        cudaGetLastError();
        return fail(CKPT_ENOMEM, "register: bucket counters allocation failed");
    }
    CUDA_TRY(cudaMemset(c->staging, 0, c->staging_bytes));
    c->d_chunks = dch;
    c->tile_first = std::move(tf);
    c->chunks = std::move(ch);
    c->segs = std::move(segs);
    c->L = L;
    if (layout) c->layout = *layout;
    if ((c->opt.flags & CKPT_OPT_SHM_ARENA) && c->opt.arena_key) {
        // persistent arena: look for this member's committed image (REFT-load after an
        // elastic restart, P.551-555).  Geometry is checked again at ckpt_protect.
        c->arena_member = layout ? (uint32_t)std::max(0, layout->local_rank) : 0;
        HostBuf mb;
        if (shm_attach(mb, meta_name(c->opt.arena_key, c->arena_member), 4096, false) == CKPT_OK) {
            ArenaMeta *mt = (ArenaMeta *)mb.p;
            const uint64_t st = __atomic_load_n(&mt->state, __ATOMIC_ACQUIRE);
            if (mt->magic == kMetaMagic && mt->L == L && st != 0) {
                c->attached_id = st >> 8;
                c->attached_idx = (int)(st & 0xff) - 1;
            }
            c->meta_buf = mb;
            c->meta = mt;
        }
    }
    c->registered = true;
    return CKPT_OK;
}

extern "C" int ckpt_geometry(const ckpt_ctx *c, uint64_t *Ll, uint64_t *Ls, uint64_t *u, uint32_t *m) {
    if (!c) return fail(CKPT_EINVAL, "geometry: null context");
    if (!c->registered) return fail(CKPT_ESTATE, "geometry: not registered");
    if (Ll) *Ll = c->L;
    if (Ls) *Ls = c->grouped ? c->Lstar : c->L;
    if (u) *u = c->grouped ? c->unit : c->opt.stripe_unit;
    if (m) *m = c->m;
    return CKPT_OK;
}

extern "C" int ckpt_tensor_offset(const ckpt_ctx *c, uint64_t t, uint64_t *off) {
    if (!c || !off) return fail(CKPT_EINVAL, "tensor_offset: null");
    if (!c->registered || t >= c->segs.size()) return fail(CKPT_EINVAL, "tensor_offset: bad index");
    *off = c->segs[t].off;
    return CKPT_OK;
}

// ------------------------------------------------------------------ group -----------
extern "C" int ckpt_export_handle(ckpt_ctx *c, void *buf, uint64_t *len) {
    if (!c || !buf || !len || *len < CKPT_HANDLE_BYTES) return fail(CKPT_EINVAL, "export_handle: bad args");
    if (!c->registered) return fail(CKPT_ESTATE, "export_handle: not registered");
    int rc = set_dev(c);
    if (rc) return rc;
    HandleBlob b;
    memset(&b, 0, sizeof b);
    b.magic = kMagic;
    b.version = kAbiVersion;
    b.device = c->device;
    b.pid = (int32_t)getpid();
    b.L = c->L;
    b.align = c->opt.align;
    b.unit = c->opt.stripe_unit;
    b.slot_bytes = c->slot_bytes;
    b.n_slots = c->n_slots;
    b.full_copy = c->full_copy;
    b.staging_bytes = c->staging_bytes;
    b.nonce = c->my_nonce;
    b.arena_key = c->opt.arena_key;
    b.attached_id = c->attached_id;
    gethostname(b.host, sizeof b.host - 1);
    CUDA_TRY(cudaIpcGetMemHandle(&b.staging_h, c->staging));
    CUDA_TRY(cudaIpcGetMemHandle(&b.flags_h, c->flags));
    memset(buf, 0, CKPT_HANDLE_BYTES);
    memcpy(buf, &b, sizeof b);
    *len = CKPT_HANDLE_BYTES;
    return CKPT_OK;
}

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

static int alloc_arena(ckpt_ctx *c) {
    c->completed = -1;
    c->ongoing = 0;
    if (device_only(c)) return CKPT_OK;  // the image lives in the device staging
    const uint64_t pbytes = parity_bytes_of(c);
    int rc = CKPT_OK;
    // persistent arena: re-attach this member's files if their metadata matches the
    // group's geometry, else start them fresh
    const bool keyed = use_shm(c) && c->opt.arena_key;
    bool reuse = false;
    if (keyed) {
        if (!c->meta) {
            int r2 = shm_create(c->meta_buf, meta_name(c->opt.arena_key, c->me), 4096);
            if (r2 == CKPT_OK) {
                cudaHostUnregister(c->meta_buf.p);
                c->meta_buf.registered = false;
                c->meta_buf.kind = kShmPeer;  // persistent
                c->meta = (ArenaMeta *)c->meta_buf.p;
            } else {
                return r2;
            }
        }
        ArenaMeta *mt = c->meta;
        reuse = mt->magic == kMetaMagic && mt->L == c->L && mt->Lstar == c->Lstar && mt->unit == c->unit &&
                mt->m == c->m && mt->me == c->me && mt->scheme == c->scheme && mt->nbuf == (uint32_t)c->nbuf &&
                mt->align == c->opt.align;
        if (!reuse) {
            __atomic_store_n(&mt->state, 0ull, __ATOMIC_RELEASE);
            mt->magic = kMetaMagic;
            mt->version = kAbiVersion;
            mt->L = c->L;
            mt->Lstar = c->Lstar;
            mt->unit = c->unit;
            mt->m = c->m;
            mt->me = c->me;
            mt->scheme = c->scheme;
            mt->nbuf = (uint32_t)c->nbuf;
            mt->align = c->opt.align;
            for (int i = 0; i < c->nbuf; ++i) shm_unlink(shm_name(c->opt.arena_key, c->me, i).c_str());
            c->attached_id = 0;
            c->attached_idx = -1;
        }
    }
    for (int i = 0; i < c->nbuf && !rc; ++i) {
        if (use_shm(c)) {
            const std::string nm = shm_name(c->group_nonce, c->me, i);
            if (reuse) {
                rc = shm_attach(c->shm_own[i], nm, shm_bytes(c), true);
                if (rc == CKPT_ENOSNAP) {  // file gone (lost host memory): fresh
                    reuse = false;
                    c->attached_id = 0;
                    c->attached_idx = -1;
                    __atomic_store_n(&c->meta->state, 0ull, __ATOMIC_RELEASE);
                    rc = CKPT_OK;
                }
            }
            if (!c->shm_own[i].p) {
                rc = shm_create(c->shm_own[i], nm, shm_bytes(c));
                if (!rc && keyed) c->shm_own[i].kind = kShmPeer;  // persistent: never unlinked here
            }
            if (rc) break;
            uint8_t *base = c->shm_own[i].p;
            c->hdata[i] = HostBuf{base, c->Lstar, kView, true, ""};
            if (pbytes) c->hpar[i] = HostBuf{base + c->Lstar, pbytes, kView, true, ""};
            if (c->arc) {
                c->harc[i] = base + c->Lstar + pbytes;
                c->harcp[i] = pbytes ? base + 2 * c->Lstar + pbytes : nullptr;
            }
        } else {
            rc = host_alloc(c->hdata[i], c->Lstar);
            if (!rc && pbytes) rc = host_alloc(c->hpar[i], pbytes);
        }
    }
    if (rc) {
        for (int k = 0; k < 2; ++k) {
            host_free(c->hdata[k]);
            host_free(c->hpar[k]);
            host_free(c->shm_own[k]);
        }
        return rc;
    }
    // snapshot id n lives in host buffer (n-1) % nbuf on every member: continue from the
    // group's committed version (max over members' attached ids, 0 for a fresh group)
    c->next_id = c->group_version + 1;
    c->ongoing = (int)(c->group_version % (uint64_t)c->nbuf);
    c->completed = -1;
    c->completed_id = 0;
    if (keyed && reuse && c->attached_id == c->group_version && c->attached_idx >= 0 &&
        c->attached_idx == (int)((c->group_version - 1) % (uint64_t)c->nbuf)) {
        c->completed = c->attached_idx;
        c->completed_id = c->attached_id;
    }
    return CKPT_OK;
}

// Publish the committed version in the persistent arena's metadata (one atomic store,
// after every byte of the image is in host memory).
static void meta_commit(ckpt_ctx *c) {
    if (!c->meta) return;
    const uint64_t st = c->completed < 0 ? 0 : (c->completed_id << 8) | (uint64_t)(c->completed + 1);
    __atomic_store_n(&c->meta->state, st, __ATOMIC_RELEASE);
}

// ARC push targets: the files of my holder (member me-1), pinned so that my copy engine
// can D2H straight into the holder's ARC-copy region.  Mapped at first use (the holder
// creates them in its own ckpt_protect).
static int ensure_holder_mapped(ckpt_ctx *c) {
    if (!c->arc) return CKPT_OK;
    const uint32_t h = (c->me + c->m - 1) % c->m;
    for (int i = 0; i < c->nbuf; ++i) {
        if (c->shm_hold[i].p) continue;
        int rc = shm_map(c->shm_hold[i], shm_name(c->group_nonce, h, i), shm_bytes(c), true);
        if (rc) return rc;
    }
    return CKPT_OK;
}

// Member me+1's own files (recovery re-creates the ARC copy I hold from them; CPU only).
static int ensure_next_mapped(ckpt_ctx *c) {
    const uint32_t nx = (c->me + 1) % c->m;
    for (int i = 0; i < c->nbuf; ++i) {
        if (c->shm_next[i].p) continue;
        int rc = shm_map(c->shm_next[i], shm_name(c->group_nonce, nx, i), shm_bytes(c), false);
        if (rc) return rc;
    }
    return CKPT_OK;
}

static int setup_ungrouped(ckpt_ctx *c) {
    c->m = 1;
    c->me = 0;
    c->group_nonce = (use_shm(c) && c->opt.arena_key) ? c->opt.arena_key : c->my_nonce;
    c->group_version = c->attached_id;
    c->scheme = CKPT_SCHEME_AEC;
    c->arc = false;
    c->aec = true;
    c->Lstar = c->L;
    c->unit = c->opt.stripe_unit;
    c->peer_L[0] = c->L;
    c->peer_staging[0] = c->staging;
    c->members[0] = c;
    int rc = alloc_arena(c);
    if (rc) return rc;
    c->grouped = true;
    return CKPT_OK;
}

extern "C" int ckpt_protect(ckpt_ctx *c, const ckpt_group *g) {
    if (!c || !g) return fail(CKPT_EINVAL, "protect: null");
    if (!c->registered) return fail(CKPT_ESTATE, "protect: not registered");
    if (c->grouped) return fail(CKPT_ESTATE, "protect: group already bound");
    if (g->m < 1 || g->m > CKPT_MAX_GROUP || g->my_index >= g->m)
        return fail(CKPT_EINVAL, "protect: m must be in [1, %u] and my_index < m", CKPT_MAX_GROUP);
    int rc = set_dev(c);
    if (rc) return rc;
    if (g->m == 1) {
        rc = setup_ungrouped(c);
        return rc ? rc : fail(CKPT_EUNAVAIL, "protect: a group of one has no redundancy (SPEC S.314)");
    }
    const uint32_t m = g->m;
    const uint32_t scheme = g->scheme == CKPT_SCHEME_DEFAULT ? CKPT_SCHEME_AEC : g->scheme;
    if (scheme > CKPT_SCHEME_ARC_AEC) return fail(CKPT_EINVAL, "protect: unknown scheme %u", g->scheme);
    const bool arc = scheme == CKPT_SCHEME_ARC || scheme == CKPT_SCHEME_ARC_AEC;
    if (arc && (!use_shm(c) || !c->full_copy || device_only(c)))
        return fail(CKPT_EINVAL, "protect: ARC schemes need CKPT_OPT_SHM_ARENA and full-copy staging (n_slots = 0)");
    uint64_t Ls[CKPT_MAX_GROUP];
    if (g->transport == CKPT_GROUP_IPC) {
        if (!g->handles) return fail(CKPT_EINVAL, "protect: IPC group without handles");
        if (load_memops()) return fail(CKPT_ECUDA, "protect: stream memory operations unavailable");
        const HandleBlob *hb[CKPT_MAX_GROUP];
        for (uint32_t j = 0; j < m; ++j)
            hb[j] = (const HandleBlob *)((const uint8_t *)g->handles + (uint64_t)j * CKPT_HANDLE_BYTES);
        for (uint32_t j = 0; j < m; ++j) {
            if (hb[j]->magic != kMagic || hb[j]->version != kAbiVersion)
                return fail(CKPT_EINVAL, "protect: handle %u is not a reft-ckpt v%u blob", j, kAbiVersion);
            if (hb[j]->align != c->opt.align || hb[j]->unit != c->opt.stripe_unit ||
                hb[j]->slot_bytes != c->slot_bytes || hb[j]->n_slots != c->n_slots || hb[j]->full_copy != (uint32_t)c->full_copy)
                return fail(CKPT_EMISMATCH, "protect: member %u geometry differs (align/unit/slots)", j);
            if (strncmp(hb[j]->host, hb[g->my_index]->host, sizeof hb[j]->host) != 0)
                return fail(CKPT_EMISMATCH, "protect: member %u is on another host '%.64s' vs '%.64s' (node group only, Q1)",
                            j, hb[j]->host, hb[g->my_index]->host);
            Ls[j] = hb[j]->L;
        }
        if (hb[g->my_index]->pid != (int32_t)getpid() || hb[g->my_index]->L != c->L)
            return fail(CKPT_EINVAL, "protect: my_index does not point at this context's handle");
        c->group_nonce = hb[0]->nonce;
        c->group_version = 0;
        for (uint32_t j = 0; j < m; ++j) {
            if (hb[j]->arena_key != c->opt.arena_key)
                return fail(CKPT_EMISMATCH, "protect: member %u uses another arena key", j);
            c->group_version = std::max(c->group_version, hb[j]->attached_id);
        }
        for (uint32_t j = 0; j < m; ++j) {
            c->peer_L[j] = Ls[j];
            if (j == g->my_index) {
                c->peer_staging[j] = c->staging;
                c->peer_flags[j] = c->flags;
                continue;
            }
            void *ps = nullptr, *pf = nullptr;
            cudaError_t e1 = cudaIpcOpenMemHandle(&ps, hb[j]->staging_h, cudaIpcMemLazyEnablePeerAccess);
            cudaError_t e2 = e1 == cudaSuccess ? cudaIpcOpenMemHandle(&pf, hb[j]->flags_h, cudaIpcMemLazyEnablePeerAccess)
                                               : e1;
            if (e1 != cudaSuccess || e2 != cudaSuccess) {
                cudaGetLastError();
                if (ps) cudaIpcCloseMemHandle(ps);
                for (uint32_t k = 0; k < j; ++k)
                    if (c->peer_opened[k]) {
                        cudaIpcCloseMemHandle(c->peer_staging[k]);
                        cudaIpcCloseMemHandle(c->peer_flags[k]);
                        c->peer_opened[k] = false;
                    }
                return fail(CKPT_EPEER, "protect: cudaIpcOpenMemHandle of member %u failed: %s", j,
                            cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
            }
            c->peer_staging[j] = (uint8_t *)ps;
            c->peer_flags[j] = (uint32_t *)pf;
            c->peer_opened[j] = true;
        }
    } else if (g->transport == CKPT_GROUP_LOCAL) {
        if (!g->members) return fail(CKPT_EINVAL, "protect: LOCAL group without members");
        if (g->members[g->my_index] != c) return fail(CKPT_EINVAL, "protect: members[my_index] is not this context");
        if (!g->members[0]) return fail(CKPT_EINVAL, "protect: LOCAL group member 0 is NULL");
        c->group_nonce = g->members[0]->my_nonce;
        c->group_version = 0;
        for (uint32_t j = 0; j < m; ++j) {
            if (!g->members[j]) return fail(CKPT_EINVAL, "protect: LOCAL group member %u is NULL", j);
            if (g->members[j]->opt.arena_key != c->opt.arena_key)
                return fail(CKPT_EMISMATCH, "protect: member %u uses another arena key", j);
            c->group_version = std::max(c->group_version, g->members[j]->attached_id);
        }
        for (uint32_t j = 0; j < m; ++j) {
            ckpt_ctx *o = g->members[j];
            if (!o || !o->registered) return fail(CKPT_ESTATE, "protect: member %u not registered", j);
            if (o->opt.align != c->opt.align || o->opt.stripe_unit != c->opt.stripe_unit ||
                o->slot_bytes != c->slot_bytes || o->n_slots != c->n_slots || o->full_copy != c->full_copy)
                return fail(CKPT_EMISMATCH, "protect: member %u geometry differs", j);
            if (o->device != c->device) {
                int can = 0;
                cudaDeviceCanAccessPeer(&can, c->device, o->device);
                if (!can) return fail(CKPT_EPEER, "protect: device %d cannot access device %d", c->device, o->device);
                cudaError_t e = cudaDeviceEnablePeerAccess(o->device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    return fail(CKPT_EPEER, "protect: enable peer access: %s", cudaGetErrorString(e));
                cudaGetLastError();
            }
            Ls[j] = o->L;
            c->peer_L[j] = o->L;
            c->peer_staging[j] = o->staging;
            c->members[j] = o;
        }
    } else {
        return fail(CKPT_EINVAL, "protect: unknown transport %u", g->transport);
    }
    uint64_t Lstar = 0, ue = 0;
    rc = ckpt_plan_common(Ls, m, c->opt.stripe_unit, &Lstar, &ue);
    if (rc) return rc;
    const uint64_t stripe = (uint64_t)(m - 1) * ue;
    if (!c->full_copy && stripe > c->slot_bytes)
        return fail(CKPT_EINVAL, "protect: stripe of %llu bytes exceeds ring slot capacity %llu (use n_slots=0 or a smaller unit)",
                    (unsigned long long)stripe, (unsigned long long)c->slot_bytes);
    c->m = m;
    c->me = g->my_index;
    c->transport = g->transport;
    c->Lstar = Lstar;
    c->unit = ue;
    c->scheme = scheme;
    c->arc = arc;
    c->aec = scheme == CKPT_SCHEME_AEC || scheme == CKPT_SCHEME_ARC_AEC;
    if (use_shm(c) && c->opt.arena_key) {
        if (c->arena_member != c->me)
            return fail(CKPT_EINVAL, "protect: persistent arena member %u (layout.local_rank) != group index %u",
                        c->arena_member, c->me);
        c->group_nonce = c->opt.arena_key;
    }
    // parity buffer (local)
    if (!c->aec) {
        c->parity_bytes = 0;
    } else if (c->full_copy) {
        c->parity_slot_bytes = 0;
        c->parity_bytes = std::max<uint64_t>(Lstar / (m - 1), 4096);
    } else {
        c->parity_slot_bytes = (c->slot_bytes / stripe) * ue;
        c->parity_bytes = c->parity_slot_bytes * c->n_slots;
    }
    if (c->aec && cudaMalloc(&c->parity, c->parity_bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(CKPT_ENOMEM, "protect: parity buffer of %llu bytes failed", (unsigned long long)c->parity_bytes);
    }
    if (c->aec && (c->opt.flags & CKPT_OPT_CE_GATHER)) {
        c->gather_bytes = c->full_copy ? std::max<uint64_t>(Lstar, 4096) : c->parity_bytes * (m - 1);
        if (cudaMalloc(&c->gather, c->gather_bytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(CKPT_ENOMEM, "protect: CE gather buffer of %llu bytes failed", (unsigned long long)c->gather_bytes);
        }
    }
    rc = alloc_arena(c);
    if (rc) return rc;
    c->seq = 0;
    c->grouped = true;
    return CKPT_OK;
}

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
static inline uint8_t *parity_slot_ptr(const ckpt_ctx *c, uint64_t k) {
    return c->full_copy ? c->parity + bucket_begin(c, k) / (c->m - 1)
                        : c->parity + (uint64_t)(k % c->n_slots) * c->parity_slot_bytes;
}
static inline uint32_t bucket_seq(const ckpt_ctx *c, uint64_t k) { return c->op_seq_base + (uint32_t)k + 1; }
static inline bool ring_reuse(const ckpt_ctx *c, uint64_t k) { return !c->full_copy && k >= c->n_slots; }

// ------------------------------------------------------------------ signals ---------
// IPC signals: cuStreamWriteValue32 into the peer's flag page (default, zero SMs) or a
// one-warp st.release.sys kernel (CKPT_SIGNAL=kernel).  Waits are always
// cuStreamWaitValue32 on the local flag page.
static bool signal_by_kernel() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("CKPT_SIGNAL");
        v = (e && strcmp(e, "kernel") == 0) ? 1 : 0;
    }
    return v == 1;
}

// signal(stage, seq): tell every other member that this member reached `seq`.
static int sig_signal(ckpt_ctx *c, cudaStream_t s, int stage, uint32_t seq, uint32_t slot) {
    if (c->m < 2) return CKPT_OK;
    if (c->transport == CKPT_GROUP_IPC) {
        auto addr = [&](uint32_t j) {
            return stage == kReady ? ready_row(c->peer_flags[j], c->me) + seq % kMaxB
                                   : c->peer_flags[j] + stage * kFlagStride + c->me;
        };
        if (signal_by_kernel()) {
            SignalArgs a;
            memset(&a, 0, sizeof a);
            for (uint32_t j = 0; j < c->m; ++j)
                if (j != c->me) a.addr[a.n++] = addr(j);
            a.value = seq;
            CUDA_TRY(launch_signal(a, s));
            return CKPT_OK;
        }
        for (uint32_t j = 0; j < c->m; ++j) {
            if (j == c->me) continue;
            CUdeviceptr a = (CUdeviceptr)(uintptr_t)addr(j);
            CUresult r = p_write32((CUstream)s, a, seq, CU_STREAM_WRITE_VALUE_DEFAULT);
            if (r != CUDA_SUCCESS) return fail(CKPT_ECUDA, "cuStreamWriteValue32 failed (%d)", (int)r);
        }
        return CKPT_OK;
    }
    int rc = ensure_events(c->ev_sig[stage], slot + 1);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(c->ev_sig[stage][slot], s));
    return CKPT_OK;
}

// wait(stage, seq): stream s waits until member j signalled >= seq.
static int sig_wait(ckpt_ctx *c, cudaStream_t s, uint32_t j, int stage, uint32_t seq, uint32_t slot) {
    if (c->transport == CKPT_GROUP_IPC) {
        CUdeviceptr a = (CUdeviceptr)(uintptr_t)(stage == kReady ? ready_row(c->flags, j) + seq % kMaxB
                                                                   : c->flags + stage * kFlagStride + j);
        CUresult r = p_wait32((CUstream)s, a, seq, CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) return fail(CKPT_ECUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
        return CKPT_OK;
    }
    ckpt_ctx *o = c->members[j];
    if (o->ev_sig[stage].size() <= slot) return fail(CKPT_ESTATE, "internal: LOCAL wait before signal");
    CUDA_TRY(cudaStreamWaitEvent(s, o->ev_sig[stage][slot], 0));
    return CKPT_OK;
}

static int wait_all(ckpt_ctx *c, cudaStream_t s, int stage, uint32_t seq, uint32_t slot, int32_t skip = -1) {
    for (uint32_t j = 0; j < c->m; ++j) {
        if (j == c->me || (int32_t)j == skip) continue;
        int rc = sig_wait(c, s, j, stage, seq, slot);
        if (rc) return rc;
    }
    return CKPT_OK;
}

// ------------------------------------------------------------------ kernels ---------
// Copy-engine pack/unpack (CKPT_OPT_CE_PACK): one D2D cudaMemcpyAsync per contiguous
// piece of a tensor inside the bucket; zero SMs.  Gaps must read as zero: the full
// staging image was zeroed at registration and gaps are never written; a ring slot is
// cleared with one memset before its copies.
static int do_pack_ce(ckpt_ctx *c, uint64_t k, uint8_t *slot, cudaStream_t s, bool unpack) {
    const uint64_t bb = bucket_begin(c, k), be = std::min(bucket_end(c, k), c->L);
    const uint64_t t_lo = bb / kTile, t_hi = (be + kTile - 1) / kTile;
    uint64_t ci = c->tile_first[t_lo], ce = c->tile_first[t_hi];
    if (!unpack && (!c->full_copy || c->staging_poisoned)) {
        CUDA_TRY(cudaMemsetAsync(slot, 0, be - bb, s));
        c->st.ce_copies++;
    }
    while (ci < ce) {
        const PackChunk &a = c->chunks[ci];
        uint64_t cj = ci + 1;  // merge the contiguous pieces of one tensor
        while (cj < ce && c->chunks[cj].seg == a.seg && c->chunks[cj].src != 0 && a.src != 0) ++cj;
        const PackChunk &z = c->chunks[cj - 1];
        ci = cj;
        if (a.src == 0) continue;
        const uint64_t lo = std::max(a.dst, bb), hi = std::min(z.dst + z.nbytes, be);
        if (lo >= hi) continue;
        uint8_t *tensor = (uint8_t *)(uintptr_t)(a.src + (lo - a.dst));
        uint8_t *sl = slot + (lo - bb);
        CUDA_TRY(cudaMemcpyAsync(unpack ? tensor : sl, unpack ? sl : tensor, hi - lo, cudaMemcpyDeviceToDevice, s));
        c->st.ce_copies++;
    }
    if (!unpack) c->st.pack_bytes += 2 * (be - bb);  // CE pieces are counted in ce_copies
    return CKPT_OK;
}

static int do_pack(ckpt_ctx *c, uint64_t k, uint8_t *slot, cudaStream_t s, bool unpack) {
    const uint64_t bb = bucket_begin(c, k), be = std::min(bucket_end(c, k), c->L);
    if (be <= bb) return CKPT_OK;
    if (c->opt.flags & CKPT_OPT_CE_PACK) return do_pack_ce(c, k, slot, s, unpack);
    PackArgs a;
    a.chunks = c->d_chunks;
    a.tile_first = c->d_tile_first;
    a.bucket_begin = bb;
    a.bucket_end = be;
    a.slot = slot;
    a.unpack = unpack ? 1 : 0;
    TimedLaunch *t;
    int rc = timed_begin(c, s, unpack ? 2 : 0, &t);
    if (rc) return rc;
    CUDA_TRY(launch_pack(a, c->max_ctas, s, (c->opt.flags & CKPT_OPT_TMA_PACK) != 0));
    rc = timed_end(t, s);
    if (rc) return rc;
    if (unpack) {
        c->st.unpack_launches++;
    } else {
        c->st.pack_launches++;
        c->st.pack_bytes += 2 * (be - bb);
    }
    return CKPT_OK;
}

// Encode row r = c->me over image bytes [bb, be) (Eq 1): terms are every peer j's data
// slot.  k is the bucket holding bb (a full-copy encode may span every bucket).
static int do_encode_range(ckpt_ctx *c, uint64_t k, uint64_t bb, uint64_t be, cudaStream_t s);
static int do_encode(ckpt_ctx *c, uint64_t k, cudaStream_t s) {
    return do_encode_range(c, k, bucket_begin(c, k), bucket_end(c, k), s);
}
static int do_encode_range(ckpt_ctx *c, uint64_t k, uint64_t bb, uint64_t be, cudaStream_t s) {
    const uint64_t stripe = (uint64_t)(c->m - 1) * c->unit;
    XorArgs a;
    memset(&a, 0, sizeof a);
    a.nin = 0;
    uint64_t in_bytes = 0;
    for (uint32_t j = 0; j < c->m; ++j) {
        if (j == c->me) continue;
        XorTerm &t = a.in[a.nin++];
        t.base = slot_ptr(c, c->peer_staging[j], k);
        t.valid = valid_in_bucket(c->peer_L[j], bb, be);
        t.stride = stripe;
        t.off = (uint64_t)sigma(c->me, j) * c->unit;
        in_bytes += (be - bb) / (c->m - 1);
    }
    a.out = parity_slot_ptr(c, k);
    a.out_valid = UINT64_MAX;
    a.out_stride = c->unit;
    a.out_off = 0;
    a.nstripes = (be - bb) / stripe;
    a.unit = c->unit;
    TimedLaunch *t;
    int rc = timed_begin(c, s, 1, &t);
    if (rc) return rc;
    CUDA_TRY(launch_xor(a, c->xor_ctas, s));
    rc = timed_end(t, s);
    if (rc) return rc;
    c->st.xor_launches++;
    c->st.xor_bytes_in += in_bytes;
    c->st.xor_bytes_out += (be - bb) / (c->m - 1);
    return CKPT_OK;
}

// Rebuild row r = c->me (a survivor) of bucket k into lost rank kl's slot (Eq 2).
static int do_rebuild_row(ckpt_ctx *c, uint64_t k, uint32_t kl, cudaStream_t s) {
    const uint64_t bb = bucket_begin(c, k), be = bucket_end(c, k);
    const uint64_t stripe = (uint64_t)(c->m - 1) * c->unit;
    XorArgs a;
    memset(&a, 0, sizeof a);
    XorTerm &p = a.in[a.nin++];
    p.base = parity_slot_ptr(c, k);
    p.valid = UINT64_MAX;
    p.stride = c->unit;
    p.off = 0;
    for (uint32_t j = 0; j < c->m; ++j) {
        if (j == c->me || j == kl) continue;
        XorTerm &t = a.in[a.nin++];
        t.base = slot_ptr(c, c->peer_staging[j], k);
        t.valid = valid_in_bucket(c->peer_L[j], bb, be);
        t.stride = stripe;
        t.off = (uint64_t)sigma(c->me, j) * c->unit;
    }
    a.out = slot_ptr(c, c->peer_staging[kl], k);
    a.out_valid = valid_in_bucket(c->peer_L[kl], bb, be);
    a.out_stride = stripe;
    a.out_off = (uint64_t)sigma(c->me, kl) * c->unit;
    a.nstripes = (be - bb) / stripe;
    a.unit = c->unit;
    TimedLaunch *t;
    int rc = timed_begin(c, s, 3, &t);
    if (rc) return rc;
    CUDA_TRY(launch_xor(a, c->xor_ctas, s));
    rc = timed_end(t, s);
    if (rc) return rc;
    c->st.rebuild_launches++;
    const uint64_t unit_bytes = (be - bb) / (c->m - 1);  // one unit per stripe per term
    c->st.rebuild_bytes_in += (uint64_t)a.nin * unit_bytes;
    c->st.rebuild_bytes_out += unit_bytes;
    return CKPT_OK;
}

// ------------------------------------------------------------------ snapshot --------
// The image's zero pad [L, L*) is structural (Q5) and never written by a D2H (which
// covers [0, L)); after ckpt_forget poisoned a buffer, re-zero it before it commits.
static void clean_pad(ckpt_ctx *c, int buf) {
    if (buf < 0) return;
    if (c->pad_dirty[buf] && c->hdata[buf].p) {
        if (c->Lstar > c->L) memset(c->hdata[buf].p + c->L, 0, c->Lstar - c->L);
        c->pad_dirty[buf] = false;
    }
    if (c->arc_dirty[buf] && c->harc[buf]) {  // pad of the ARC copy I hold (of member me+1)
        const uint64_t Ln = c->peer_L[(c->me + 1) % c->m];
        if (c->Lstar > Ln) memset(c->harc[buf] + Ln, 0, c->Lstar - Ln);
        c->arc_dirty[buf] = false;
    }
}

static int check_sticky(ckpt_ctx *c) {
    if (c->sticky) return fail(c->sticky, "context has a sticky error: %s", c->sticky_msg.c_str());
    return CKPT_OK;
}

static void make_sticky(ckpt_ctx *c, int rc) {
    if (!c->sticky) {
        c->sticky = rc;
        c->sticky_msg = g_last_error;
    }
}

// Bucket = whole stripes ((m-1)u; A when unprotected).  With full-copy staging the
// single-launch pack also needs whole 64 KiB tile groups: B is rounded down to a
// multiple of lcm(stripe, kGroup).
static int host_sync(ckpt_ctx *c);

static uint64_t effective_bucket(const ckpt_ctx *c, uint64_t req) {
    uint64_t B = req ? req : c->opt.bucket_bytes;
    uint64_t q = c->m >= 2 ? (uint64_t)(c->m - 1) * c->unit : (uint64_t)c->opt.align;
    if (c->full_copy) q = q / std::gcd(q, kGroup) * kGroup;
    return std::max<uint64_t>(q, B / q * q);
}

static bool single_launch(const ckpt_ctx *c) {
    return c->full_copy && !(c->opt.flags & CKPT_OPT_CE_PACK) &&
           (c->transport == CKPT_GROUP_LOCAL && c->m >= 2 ? true : load_memops() == CKPT_OK);
}

// The whole snapshot's pack as one launch (full-copy staging); the kernel publishes each
// bucket's READY flag itself (see PackAllArgs).  Buckets past this rank's L hold no data
// and are published up front.
static int issue_pack_all(ckpt_ctx *c) {
    const uint64_t nb_data = (c->L + c->op_B - 1) / c->op_B;
    int rc;
    CUDA_TRY(cudaMemsetAsync(c->counters, 0, std::max<uint64_t>(nb_data, 1) * sizeof(uint32_t), c->sP));
    if (c->m >= 2)
        for (uint64_t k = nb_data; k < c->op_NB; ++k)
            if ((rc = sig_signal(c, c->sP, kReady, bucket_seq(c, k), slot_of(c, k)))) return rc;
    PackAllArgs a;
    memset(&a, 0, sizeof a);
    a.chunks = c->d_chunks;
    a.tile_first = c->d_tile_first;
    a.L = c->L;
    a.image = c->staging;
    a.bucket = c->op_B;
    a.counters = c->counters;
    a.ready_local = ready_row(c->flags, c->me);
    if (c->m >= 2 && c->transport == CKPT_GROUP_IPC)
        for (uint32_t j = 0; j < c->m; ++j)
            if (j != c->me) a.ready_peer[a.npeers++] = ready_row(c->peer_flags[j], c->me);
    a.seq_base = c->op_seq_base;
    a.maxb = kMaxB;
    TimedLaunch *t;
    if ((rc = timed_begin(c, c->sP, 0, &t))) return rc;
    // default single-launch pack: the multi-producer TMA kernel (same HBM bandwidth as the
    // LSU kernel from ~2.5x fewer SM-seconds); CKPT_OPT_LSU_PACK selects the LSU kernel
    CUDA_TRY(launch_pack_all(a, c->max_ctas, c->sP, !(c->opt.flags & CKPT_OPT_LSU_PACK)));
    if ((rc = timed_end(t, c->sP))) return rc;
    c->st.pack_launches++;
    c->st.pack_bytes += 2 * c->L;
    CUDA_TRY(cudaEventRecord(c->ev_pack_all, c->sP));
    if (c->transport == CKPT_GROUP_LOCAL && c->m >= 2) {
        for (uint64_t k = 0; k < nb_data; ++k) {
            CUDA_TRY(cudaEventRecord(c->ev_packed[slot_of(c, k)], c->sP));
            if ((rc = sig_signal(c, c->sP, kReady, bucket_seq(c, k), slot_of(c, k)))) return rc;
        }
    }
    return CKPT_OK;
}

static int prepare_op(ckpt_ctx *c, uint64_t B) {
    const uint64_t nb = c->Lstar ? (c->Lstar + B - 1) / B : 0;
    if (nb >= kMaxB) return fail(CKPT_EINVAL, "bucket of %llu bytes gives %llu buckets (max %u): use larger buckets",
                                 (unsigned long long)B, (unsigned long long)nb, kMaxB - 1);
    c->op_B = B;
    c->op_NB = nb;
    c->op_seq_base = c->seq;
    c->seq += (uint32_t)c->op_NB + 1;
    const size_t ne = c->full_copy ? (size_t)std::max<uint64_t>(c->op_NB, 1) : c->n_slots;
    int rc = 0;
    for (auto *v : {&c->ev_packed, &c->ev_xored, &c->ev_d2h_data, &c->ev_d2h_par, &c->ev_h2d, &c->ev_kdone,
                    &c->ev_gathered})
        if (!rc) rc = ensure_events(*v, ne);
    return rc;
}

// Stage 1 of bucket k on member c: pack into its slot, then READY.
static int stage_pack(ckpt_ctx *c, uint64_t k) {
    const uint32_t s = slot_of(c, k);
    int rc;
    if (ring_reuse(c, k)) {
        CUDA_TRY(cudaStreamWaitEvent(c->sP, c->ev_d2h_data[s], 0));
        if (c->m >= 2 && (rc = wait_all(c, c->sP, kRel, bucket_seq(c, k - c->n_slots), s))) return rc;
    }
    if ((rc = do_pack(c, k, slot_ptr(c, c->staging, k), c->sP, false))) return rc;
    CUDA_TRY(cudaEventRecord(c->ev_packed[s], c->sP));
    if (c->m >= 2 && (rc = sig_signal(c, c->sP, kReady, bucket_seq(c, k), s))) return rc;
    return CKPT_OK;
}

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

static int do_gather_ce(ckpt_ctx *c, uint64_t k, cudaStream_t s) {
    const uint64_t bb = bucket_begin(c, k), be = bucket_end(c, k);
    const uint64_t u = c->unit, pitch = (uint64_t)(c->m - 1) * u, nst = (be - bb) / pitch;
    const uint64_t gs = gather_stride(c, k);
    uint8_t *g = gather_slot_ptr(c, k);
    uint32_t jj = 0;
    for (uint32_t j = 0; j < c->m; ++j) {
        if (j == c->me) continue;
        uint8_t *dst = g + (uint64_t)jj++ * gs;
        const uint8_t *src = slot_ptr(c, c->peer_staging[j], k);
        const uint64_t v = valid_in_bucket(c->peer_L[j], bb, be), off = (uint64_t)sigma(c->me, j) * u;
        const uint64_t full = v >= off + u ? std::min(nst, (v - off - u) / pitch + 1) : 0;
        if (full == 1 || (full && nst == 1)) {
            CUDA_TRY(cudaMemcpyAsync(dst, src + off, u, cudaMemcpyDeviceToDevice, s));
        } else if (full) {
            CUDA_TRY(cudaMemcpy2DAsync(dst, u, src + off, pitch, u, full, cudaMemcpyDeviceToDevice, s));
        }
        uint64_t done = full * u;
        if (full < nst) {
            const uint64_t start = full * pitch + off;
            if (v > start) {
                CUDA_TRY(cudaMemcpyAsync(dst + done, src + start, v - start, cudaMemcpyDeviceToDevice, s));
                done += v - start;
                c->st.ce_copies++;
            }
            CUDA_TRY(cudaMemsetAsync(dst + done, 0, nst * u - done, s));
            c->st.ce_copies++;
        }
        if (full) c->st.ce_copies++;
        c->st.xor_bytes_in += (be - bb) / (c->m - 1);
    }
    return CKPT_OK;
}

static int do_encode_gathered(ckpt_ctx *c, uint64_t k, cudaStream_t s) {
    const uint64_t bb = bucket_begin(c, k), be = bucket_end(c, k);
    const uint64_t gs = gather_stride(c, k);
    XorArgs a;
    memset(&a, 0, sizeof a);
    for (uint32_t jj = 0; jj + 1 < c->m; ++jj) {
        XorTerm &t = a.in[a.nin++];
        t.base = gather_slot_ptr(c, k) + (uint64_t)jj * gs;
        t.valid = UINT64_MAX;
        t.stride = c->unit;
        t.off = 0;
    }
    a.out = parity_slot_ptr(c, k);
    a.out_valid = UINT64_MAX;
    a.out_stride = c->unit;
    a.out_off = 0;
    a.nstripes = (be - bb) / ((uint64_t)(c->m - 1) * c->unit);
    a.unit = c->unit;
    TimedLaunch *t;
    int rc = timed_begin(c, s, 1, &t);
    if (rc) return rc;
    CUDA_TRY(launch_xor(a, c->xor_ctas, s));
    rc = timed_end(t, s);
    if (rc) return rc;
    c->st.xor_launches++;
    c->st.xor_bytes_out += (be - bb) / (c->m - 1);
    return CKPT_OK;
}

// Stage 2: parity of bucket k once every member's pack(k) is visible, then REL.
// Full-copy staging after a single-launch pack: ONE XOR launch over the whole image once
// this rank's pack is done and every peer published every bucket (parity is not on the
// critical path: its D2H is queued after all the data).  Per-bucket events keep the
// parity D2H ordering uniform.
static int stage_xor_all(ckpt_ctx *c) {
    int rc;
    CUDA_TRY(cudaStreamWaitEvent(c->sX, c->ev_pack_all, 0));
    for (uint64_t k = 0; k < c->op_NB; ++k)
        if ((rc = wait_all(c, c->sX, kReady, bucket_seq(c, k), slot_of(c, k)))) return rc;
    if ((rc = do_encode_range(c, 0, 0, c->Lstar, c->sX))) return rc;
    for (uint64_t k = 0; k < c->op_NB; ++k) CUDA_TRY(cudaEventRecord(c->ev_xored[slot_of(c, k)], c->sX));
    // REL is a monotonic scalar: one signal covers every bucket
    return sig_signal(c, c->sX, kRel, bucket_seq(c, c->op_NB - 1), slot_of(c, c->op_NB - 1));
}

static bool xor_in_one_launch(const ckpt_ctx *c) {
    return c->m >= 2 && c->aec && single_launch(c) && !(c->opt.flags & CKPT_OPT_CE_GATHER);
}

static int stage_xor(ckpt_ctx *c, uint64_t k) {
    if (c->m < 2 || !c->aec) return CKPT_OK;
    if (xor_in_one_launch(c)) return k + 1 == c->op_NB ? stage_xor_all(c) : CKPT_OK;
    const uint32_t s = slot_of(c, k);
    int rc;
    if (c->opt.flags & CKPT_OPT_CE_GATHER) {
        if ((rc = wait_all(c, c->sG, kReady, bucket_seq(c, k), s))) return rc;
        if (ring_reuse(c, k)) CUDA_TRY(cudaStreamWaitEvent(c->sG, c->ev_xored[s], 0));
        if ((rc = do_gather_ce(c, k, c->sG))) return rc;
        CUDA_TRY(cudaEventRecord(c->ev_gathered[s], c->sG));
        if ((rc = sig_signal(c, c->sG, kRel, bucket_seq(c, k), s))) return rc;
        CUDA_TRY(cudaStreamWaitEvent(c->sX, c->ev_gathered[s], 0));
        if (ring_reuse(c, k)) CUDA_TRY(cudaStreamWaitEvent(c->sX, c->ev_d2h_par[s], 0));
        if ((rc = do_encode_gathered(c, k, c->sX))) return rc;
        CUDA_TRY(cudaEventRecord(c->ev_xored[s], c->sX));
        return CKPT_OK;
    }
    // Row me reads only the peers' units.  After a single-launch pack the XOR also waits
    // for this rank's own pack: the two would otherwise split HBM/NVLink bandwidth while
    // the parity is not on the critical path (its D2H is queued after all the data).
    if (single_launch(c) && k == 0) CUDA_TRY(cudaStreamWaitEvent(c->sX, c->ev_pack_all, 0));
    if ((rc = wait_all(c, c->sX, kReady, bucket_seq(c, k), s))) return rc;
    if (ring_reuse(c, k)) CUDA_TRY(cudaStreamWaitEvent(c->sX, c->ev_d2h_par[s], 0));
    if ((rc = do_encode(c, k, c->sX))) return rc;
    CUDA_TRY(cudaEventRecord(c->ev_xored[s], c->sX));
    return sig_signal(c, c->sX, kRel, bucket_seq(c, k), s);
}

// Stage 3: copy-engine D2H of data and parity into the ongoing host image.  With
// full-copy staging all data buckets are queued before any parity bucket (parity is
// ready long before the data stream reaches it); the ring interleaves them per slot.
static int stage_copy_parity(ckpt_ctx *c, uint64_t k);
static int stage_copy(ckpt_ctx *c, uint64_t k, bool with_parity = true) {
    const uint32_t s = slot_of(c, k);
    const uint64_t bb = bucket_begin(c, k), be = bucket_end(c, k);
    const uint64_t v = valid_in_bucket(c->L, bb, be);
    if (single_launch(c) && !(c->transport == CKPT_GROUP_LOCAL && c->m >= 2)) {
        if (v) {  // the single pack kernel publishes bucket k in this rank's READY row
            const uint32_t q = bucket_seq(c, k);
            CUresult r = p_wait32((CUstream)c->sC, (CUdeviceptr)(uintptr_t)(ready_row(c->flags, c->me) + q % kMaxB), q,
                                  CU_STREAM_WAIT_VALUE_GEQ);
            if (r != CUDA_SUCCESS) return fail(CKPT_ECUDA, "cuStreamWaitValue32 failed (%d)", (int)r);
        }
    } else if (v || !single_launch(c)) {
        CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_packed[s], 0));
    }
    if (device_only(c)) {  // the image stays in HBM: only order the completion events
        CUDA_TRY(cudaEventRecord(c->ev_d2h_data[s], c->sC));
        return with_parity ? stage_copy_parity(c, k) : CKPT_OK;
    }
    if (v && (c->opt.flags & CKPT_OPT_WINDOWED)) {  // HAS: only while the window is open
        CUresult r = p_wait32((CUstream)c->sC, (CUdeviceptr)(uintptr_t)c->window, 1u, CU_STREAM_WAIT_VALUE_AND);
        if (r != CUDA_SUCCESS) return fail(CKPT_ECUDA, "cuStreamWaitValue32(window) failed (%d)", (int)r);
    }
    if (v) {
        CUDA_TRY(cudaMemcpyAsync(c->hdata[c->ongoing].p + bb, slot_ptr(c, c->staging, k), v, cudaMemcpyDeviceToHost, c->sC));
        c->st.d2h_bytes += v;
        if (c->arc) {  // ARC: the same bucket again, into my holder's ARC-copy region
            uint8_t *dst = c->shm_hold[c->ongoing].p + c->Lstar + parity_bytes_of(c) + bb;
            CUDA_TRY(cudaMemcpyAsync(dst, slot_ptr(c, c->staging, k), v, cudaMemcpyDeviceToHost, c->sC));
            c->st.d2h_bytes += v;
            c->st.ce_copies++;
        }
    }
    CUDA_TRY(cudaEventRecord(c->ev_d2h_data[s], c->sC));
    return with_parity ? stage_copy_parity(c, k) : CKPT_OK;
}

static int stage_copy_parity(ckpt_ctx *c, uint64_t k) {
    if (c->m < 2 || !c->aec) return CKPT_OK;
    const uint32_t s = slot_of(c, k);
    const uint64_t bb = bucket_begin(c, k), be = bucket_end(c, k);
    const uint64_t pb = (be - bb) / (c->m - 1);
    CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_xored[s], 0));
    if (!device_only(c) && (c->opt.flags & CKPT_OPT_WINDOWED)) {
        CUresult r = p_wait32((CUstream)c->sC, (CUdeviceptr)(uintptr_t)c->window, 1u, CU_STREAM_WAIT_VALUE_AND);
        if (r != CUDA_SUCCESS) return fail(CKPT_ECUDA, "cuStreamWaitValue32(window) failed (%d)", (int)r);
    }
    if (!device_only(c)) {
        CUDA_TRY(cudaMemcpyAsync(c->hpar[c->ongoing].p + bb / (c->m - 1), parity_slot_ptr(c, k), pb,
                                 cudaMemcpyDeviceToHost, c->sC));
        c->st.d2h_bytes += pb;
        if (c->arc) {  // ARC_AEC: my parity row into my holder's ARC copy too (Q20)
            uint8_t *dst = c->shm_hold[c->ongoing].p + 2 * c->Lstar + parity_bytes_of(c) + bb / (c->m - 1);
            CUDA_TRY(cudaMemcpyAsync(dst, parity_slot_ptr(c, k), pb, cudaMemcpyDeviceToHost, c->sC));
            c->st.d2h_bytes += pb;
            c->st.ce_copies++;
        }
    }
    CUDA_TRY(cudaEventRecord(c->ev_d2h_par[s], c->sC));
    return CKPT_OK;
}

static int stage_finish(ckpt_ctx *c) {
    CUDA_TRY(cudaEventRecord(c->ev_pack_all, c->sP));
    CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_pack_all, 0));
    if (c->m >= 2 && c->aec) CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_xored[slot_of(c, c->op_NB ? c->op_NB - 1 : 0)], 0));
    CUDA_TRY(cudaEventRecord(c->ev_done, c->sC));
    if (c->opt.flags & CKPT_OPT_TIMING) CUDA_TRY(cudaEventRecord(c->ev_t1, c->sC));
    if (c->m >= 2) return sig_signal(c, c->sC, kDone, c->op_seq_base + (uint32_t)c->op_NB + 1, 0);
    return CKPT_OK;
}

static int begin_member(ckpt_ctx *c, cudaStream_t caller, uint64_t B) {
    int rc = prepare_op(c, B);
    if (rc) return rc;
    c->staging_id = 0;  // the pack overwrites the device copy
    if (c->nbuf == 1) {  // single buffer: overwritten in place
        c->completed = -1;
        meta_commit(c);
    }
    CUDA_TRY(cudaEventRecord(c->ev_capture, caller));
    if (c->opt.flags & CKPT_OPT_TIMING) CUDA_TRY(cudaEventRecord(c->ev_t0, caller));
    CUDA_TRY(cudaStreamWaitEvent(c->sP, c->ev_capture, 0));
    return CKPT_OK;
}

extern "C" int ckpt_snapshot(ckpt_ctx *c, uint64_t bucket_bytes, void *stream, uint64_t *id) {
    NvtxRange nvtx_("ckpt_snapshot");
    if (!c) return fail(CKPT_EINVAL, "snapshot: null context");
    if (!c->registered) return fail(CKPT_ESTATE, "snapshot: not registered");
    int rc = check_sticky(c);
    if (rc) return rc;
    if ((rc = host_sync(c))) return rc;  // the pack must not overwrite a staging still being copied
    if (c->pending_id || c->requested) return fail(CKPT_EBUSY, "snapshot: previous snapshot %llu not waited", (unsigned long long)c->pending_id);
    if ((rc = set_dev(c))) return rc;
    if (!c->grouped && (rc = setup_ungrouped(c))) return rc;
    if (c->arc && (rc = ensure_holder_mapped(c))) return rc;
    const uint64_t B = effective_bucket(c, bucket_bytes);
    if (!c->full_copy && B > c->slot_bytes)
        return fail(CKPT_EINVAL, "snapshot: bucket of %llu bytes exceeds slot capacity %llu", (unsigned long long)B,
                    (unsigned long long)c->slot_bytes);
    cudaStream_t caller = (cudaStream_t)stream;
    const uint64_t my_id = c->next_id++;
    if (c->m >= 2 && c->transport == CKPT_GROUP_LOCAL) {
        c->req_bucket = B;
        c->requested = true;
        c->pending_id = my_id;
        CUDA_TRY(cudaEventRecord(c->ev_capture, caller));  // capture point of this member
        bool all = true;
        for (uint32_t j = 0; j < c->m; ++j) all = all && c->members[j]->requested;
        if (all) {
            for (uint32_t j = 0; j < c->m; ++j)
                if (c->members[j]->req_bucket != B) return fail(CKPT_EINVAL, "snapshot: members passed different bucket sizes");
            // keep each member's capture event: begin_member must not re-record it
            for (uint32_t j = 0; j < c->m; ++j) {
                ckpt_ctx *o = c->members[j];
                if ((rc = set_dev(o)) || (rc = prepare_op(o, B))) return rc;
                o->staging_id = 0;
                if (o->nbuf == 1) {
                    o->completed = -1;
                    meta_commit(o);
                }
                CUDA_TRY(cudaStreamWaitEvent(o->sP, o->ev_capture, 0));
                if (o->opt.flags & CKPT_OPT_TIMING) CUDA_TRY(cudaEventRecord(o->ev_t0, o->sP));
            }
            const bool one = single_launch(c);
            if (one)
                for (uint32_t j = 0; j < c->m; ++j)
                    if ((rc = set_dev(c->members[j])) || (rc = issue_pack_all(c->members[j]))) goto bad;
            for (uint64_t k = 0; k < c->op_NB; ++k) {
                for (uint32_t j = 0; j < c->m && !one; ++j)
                    if ((rc = set_dev(c->members[j])) || (rc = stage_pack(c->members[j], k))) goto bad;
                for (uint32_t j = 0; j < c->m; ++j)
                    if ((rc = set_dev(c->members[j])) || (rc = stage_xor(c->members[j], k))) goto bad;
                for (uint32_t j = 0; j < c->m; ++j)
                    if ((rc = set_dev(c->members[j])) || (rc = stage_copy(c->members[j], k, !c->full_copy))) goto bad;
            }
            for (uint64_t k = 0; c->full_copy && k < c->op_NB; ++k)
                for (uint32_t j = 0; j < c->m; ++j)
                    if ((rc = set_dev(c->members[j])) || (rc = stage_copy_parity(c->members[j], k))) goto bad;
            for (uint32_t j = 0; j < c->m; ++j) {
                ckpt_ctx *o = c->members[j];
                if ((rc = set_dev(o)) || (rc = stage_finish(o))) goto bad;
                o->issued = true;
                o->requested = false;
                o->st.snapshots++;
            }
            set_dev(c);
        }
        if (id) *id = my_id;
        return CKPT_OK;
    bad:
        for (uint32_t j = 0; j < c->m; ++j) make_sticky(c->members[j], rc);
        return rc;
    }
    if ((rc = begin_member(c, caller, B))) return rc;
    const bool one = single_launch(c);
    if (one && (rc = issue_pack_all(c))) {
        make_sticky(c, rc);
        return rc;
    }
    for (uint64_t k = 0; k < c->op_NB; ++k) {
        if ((!one && (rc = stage_pack(c, k))) || (rc = stage_xor(c, k)) || (rc = stage_copy(c, k, !c->full_copy))) {
            make_sticky(c, rc);
            return rc;
        }
    }
    for (uint64_t k = 0; c->full_copy && k < c->op_NB; ++k) {
        if ((rc = stage_copy_parity(c, k))) {
            make_sticky(c, rc);
            return rc;
        }
    }
    if ((rc = stage_finish(c))) {
        make_sticky(c, rc);
        return rc;
    }
    c->pending_id = my_id;
    c->issued = true;
    c->st.snapshots++;
    if (id) *id = my_id;
    return CKPT_OK;
}

extern "C" int ckpt_fence(ckpt_ctx *c, uint64_t id, void *stream) {
    if (!c) return fail(CKPT_EINVAL, "fence: null");
    if (id == 0 || id >= c->next_id) return fail(CKPT_EINVAL, "fence: unknown snapshot id");
    if (id != c->pending_id) return CKPT_OK;  // already waited: nothing reads the tensors
    if (!c->issued) return fail(CKPT_ESTATE, "fence: LOCAL group snapshot not issued yet (members missing)");
    int rc = set_dev(c);
    if (rc) return rc;
    CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, c->ev_pack_all, 0));
    return CKPT_OK;
}

// Host-side wait on a stream with a timeout (peers that died never signal).
static int sync_stream_timeout(ckpt_ctx *c, cudaStream_t s, const char *what) {
    double limit = 600.0;
    if (const char *e = getenv("CKPT_TIMEOUT_S")) limit = atof(e);
    auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) return CKPT_OK;
        if (e != cudaErrorNotReady) return fail(CKPT_ECUDA, "%s: %s", what, cudaGetErrorString(e));
        double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > limit) {
            // snapshot of the flag page for the message, then release our own stream
            // waits so the context can be destroyed
            uint32_t f[kNumStages * kFlagStride] = {};
            cudaStream_t t = nullptr;
            if (c->flags && cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking) == cudaSuccess) {
                cudaMemcpyAsync(f, c->flags, sizeof f, cudaMemcpyDeviceToHost, t);
                cudaStreamSynchronize(t);
                cudaStreamDestroy(t);
            }
            char buf[512];
            int o = snprintf(buf, sizeof buf, "seq_base=%u NB=%llu", c->op_seq_base, (unsigned long long)c->op_NB);
            for (int st = 0; st < kNumStages && o < (int)sizeof buf; ++st) {
                o += snprintf(buf + o, sizeof buf - o, " %s=[", st == 0 ? "READY" : st == 1 ? "REL" : "DONE");
                for (uint32_t j = 0; j < c->m && o < (int)sizeof buf; ++j)
                    o += snprintf(buf + o, sizeof buf - o, "%u%s", f[st * kFlagStride + j], j + 1 < c->m ? "," : "]");
            }
            cudaMemset(c->flags, 0x7f, kFlagAlloc);
            cudaGetLastError();
            return fail(CKPT_EPEER, "%s: timed out after %.0f s waiting for peers (member %u: %s)", what, limit, c->me, buf);
        }
        std::this_thread::sleep_for(std::chrono::microseconds(el < 0.01 ? 20 : 200));
    }
}

static int wait_done_all(ckpt_ctx *c, uint32_t done_seq) {
    int rc;
    cudaStream_t ss[4] = {c->sP, c->sX, c->sC, c->sG};
    for (auto s : ss)
        if ((rc = sync_stream_timeout(c, s, "wait"))) return rc;
    if (c->m >= 2) {
        if (c->transport == CKPT_GROUP_IPC) {
            if ((rc = wait_all(c, c->sW, kDone, done_seq, 0))) return rc;
            if ((rc = sync_stream_timeout(c, c->sW, "wait(peers)"))) return rc;
        } else {
            for (uint32_t j = 0; j < c->m; ++j) {
                ckpt_ctx *o = c->members[j];
                if (o == c) continue;
                CUDA_TRY(cudaEventSynchronize(o->ev_done));
            }
        }
    }
    return CKPT_OK;
}

extern "C" int ckpt_wait(ckpt_ctx *c, uint64_t id) {
    NvtxRange nvtx_("ckpt_wait");
    if (!c) return fail(CKPT_EINVAL, "wait: null");
    if (id == 0 || id >= c->next_id) return fail(CKPT_ESTATE, "wait: unknown snapshot id %llu", (unsigned long long)id);
    if (id != c->pending_id) return c->completed_id >= id ? CKPT_OK : fail(CKPT_ESTATE, "wait: snapshot %llu was not committed", (unsigned long long)id);
    if (!c->issued) return fail(CKPT_ESTATE, "wait: LOCAL group snapshot not issued yet (members missing)");
    int rc = set_dev(c);
    if (rc) return rc;
    rc = wait_done_all(c, c->op_seq_base + (uint32_t)c->op_NB + 1);
    if (!rc) rc = check_sticky(c);
    if (!rc && (c->opt.flags & CKPT_OPT_TIMING)) {
        rc = harvest_timing(c);
        float ms = 0;
        if (!rc && cudaEventElapsedTime(&ms, c->ev_t0, c->ev_t1) == cudaSuccess) c->st.last_snapshot_ms = ms;
        cudaGetLastError();
    }
    c->pending_id = 0;
    c->issued = false;
    if (rc) {  // never commit a failed snapshot (S.431)
        make_sticky(c, rc);
        return rc;
    }
    clean_pad(c, c->ongoing);
    c->completed = c->ongoing;
    c->completed_id = id;
    if (c->nbuf == 2) c->ongoing ^= 1;
    if (c->full_copy) c->staging_id = id;
    c->staging_poisoned = false;
    meta_commit(c);
    return CKPT_OK;
}

// ------------------------------------------------------------------ load ------------
extern "C" int ckpt_load(ckpt_ctx *c, void *stream) {
    NvtxRange nvtx_("ckpt_load");
    if (!c) return fail(CKPT_EINVAL, "load: null");
    if (!c->registered) return fail(CKPT_ESTATE, "load: not registered");
    int rc = check_sticky(c);
    if (rc) return rc;
    if (c->pending_id || c->requested) return fail(CKPT_ESTATE, "load: a snapshot is in flight");
    if (c->rebuild_requested) return fail(CKPT_ESTATE, "load: a LOCAL group rebuild is not complete");
    if (!c->grouped || c->completed < 0) return fail(CKPT_ENOSNAP, "load: no completed snapshot");
    if (!device_image_valid(c) && (rc = host_sync(c))) return rc;
    if ((rc = set_dev(c))) return rc;
    cudaStream_t caller = (cudaStream_t)stream;
    // op geometry: bucket = ring slot (or the default bucket in full-copy mode)
    const uint32_t saved_seq = c->seq;
    if ((rc = prepare_op(c, effective_bucket(c, 0)))) return rc;
    c->seq = saved_seq;  // local op: no group sequence numbers consumed
    CUDA_TRY(cudaEventRecord(c->ev_capture, caller));
    const bool from_dev = device_image_valid(c);
    CUDA_TRY(cudaStreamWaitEvent(from_dev ? c->sP : c->sC, c->ev_capture, 0));
    const uint8_t *img = from_dev ? nullptr : c->hdata[c->completed].p;
    for (uint64_t k = 0; k < c->op_NB; ++k) {
        const uint32_t s = slot_of(c, k);
        const uint64_t bb = bucket_begin(c, k);
        const uint64_t v = valid_in_bucket(c->L, bb, bucket_end(c, k));
        if (!v) continue;
        if (ring_reuse(c, k)) CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_kdone[s], 0));
        if (!from_dev) {  // (from the device copy the unpack needs nothing from the copy stream,
                          // which may still hold a background host restore)
            CUDA_TRY(cudaMemcpyAsync(slot_ptr(c, c->staging, k), img + bb, v, cudaMemcpyHostToDevice, c->sC));
            c->st.h2d_bytes += v;
            CUDA_TRY(cudaEventRecord(c->ev_h2d[s], c->sC));
            CUDA_TRY(cudaStreamWaitEvent(c->sP, c->ev_h2d[s], 0));
        }
        if ((rc = do_pack(c, k, slot_ptr(c, c->staging, k), c->sP, true))) return rc;
        CUDA_TRY(cudaEventRecord(c->ev_kdone[s], c->sP));
    }
    CUDA_TRY(cudaStreamWaitEvent(c->sP, c->ev_capture, 0));
    CUDA_TRY(cudaEventRecord(c->ev_pack_all, c->sP));
    CUDA_TRY(cudaStreamWaitEvent(caller, c->ev_pack_all, 0));
    c->st.loads++;
    // a host-path load over full-copy staging leaves the data image there (its parity
    // buffer is not reloaded, so it is not a complete device image for a rebuild)
    if (c->opt.flags & CKPT_OPT_TIMING) {
        CUDA_TRY(cudaStreamSynchronize(c->sP));
        rc = harvest_timing(c);
    }
    return rc;
}

// ------------------------------------------------------------------ rebuild ---------
// Per bucket b (slot s), lost member kl:
//   survivor j: C: [reuse: own kernel(b-n) done, REL(b-n) from all] H2D data+parity -> READY(b)
//               X: own H2D, READY(b) from all -> rebuild row j into kl's slot -> REL(b)
//   lost kl   : X: [reuse: own D2H(b-n)] READY(b) ; READY(b) from all -> encode row kl -> REL(b)
//               C: REL(b) from all, own encode -> D2H data + parity into its image
static int rb_stage1(ckpt_ctx *c, uint64_t b, uint32_t kl) {
    const uint32_t s = slot_of(c, b);
    const uint64_t bb = bucket_begin(c, b), be = bucket_end(c, b);
    int rc;
    if (c->me != kl) {
        if (ring_reuse(c, b)) {
            CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_kdone[s], 0));
            if ((rc = wait_all(c, c->sC, kRel, bucket_seq(c, b - c->n_slots), s))) return rc;
        }
        const uint64_t v = valid_in_bucket(c->L, bb, be);
        const uint64_t pb = (be - bb) / (c->m - 1);
        if (!device_image_valid(c)) {  // else staging and parity already hold the image
            if (v) CUDA_TRY(cudaMemcpyAsync(slot_ptr(c, c->staging, b), c->hdata[c->completed].p + bb, v, cudaMemcpyHostToDevice, c->sC));
            CUDA_TRY(cudaMemcpyAsync(parity_slot_ptr(c, b), c->hpar[c->completed].p + bb / (c->m - 1), pb, cudaMemcpyHostToDevice, c->sC));
            c->st.h2d_bytes += v + pb;
        }
        CUDA_TRY(cudaEventRecord(c->ev_h2d[s], c->sC));
        return sig_signal(c, c->sC, kReady, bucket_seq(c, b), s);
    }
    if (ring_reuse(c, b)) {
        CUDA_TRY(cudaStreamWaitEvent(c->sX, c->ev_d2h_data[s], 0));
        CUDA_TRY(cudaStreamWaitEvent(c->sX, c->ev_d2h_par[s], 0));
    }
    return sig_signal(c, c->sX, kReady, bucket_seq(c, b), s);
}

static int rb_stage2(ckpt_ctx *c, uint64_t b, uint32_t kl) {
    const uint32_t s = slot_of(c, b);
    int rc;
    if (c->me != kl) CUDA_TRY(cudaStreamWaitEvent(c->sX, c->ev_h2d[s], 0));
    if ((rc = wait_all(c, c->sX, kReady, bucket_seq(c, b), s))) return rc;
    if (c->me != kl)
        rc = do_rebuild_row(c, b, kl, c->sX);
    else
        rc = do_encode(c, b, c->sX);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(c->ev_kdone[s], c->sX));
    return sig_signal(c, c->sX, kRel, bucket_seq(c, b), s);
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

static int rb_stage3(ckpt_ctx *c, uint64_t b, uint32_t kl) {
    if (c->me != kl) return CKPT_OK;
    const uint32_t s = slot_of(c, b);
    const uint64_t bb = bucket_begin(c, b), be = bucket_end(c, b);
    int rc;
    if (async_host_restore(c)) {
        if ((rc = wait_all(c, c->sX, kRel, bucket_seq(c, b), s))) return rc;
        CUDA_TRY(cudaEventRecord(c->ev_h2d[s], c->sX));  // bucket b of the device image complete
        CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_h2d[s], 0));
    } else {
        if ((rc = wait_all(c, c->sC, kRel, bucket_seq(c, b), s))) return rc;
    }
    CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_kdone[s], 0));
    const uint64_t v = valid_in_bucket(c->L, bb, be);
    const uint64_t pb = (be - bb) / (c->m - 1);
    if (!device_only(c) && v)
        CUDA_TRY(cudaMemcpyAsync(c->hdata[rb_target(c)].p + bb, slot_ptr(c, c->staging, b), v, cudaMemcpyDeviceToHost, c->sC));
    CUDA_TRY(cudaEventRecord(c->ev_d2h_data[s], c->sC));
    if (!device_only(c)) {
        CUDA_TRY(cudaMemcpyAsync(c->hpar[rb_target(c)].p + bb / (c->m - 1), parity_slot_ptr(c, b), pb, cudaMemcpyDeviceToHost, c->sC));
        c->st.d2h_bytes += v + pb;
    }
    CUDA_TRY(cudaEventRecord(c->ev_d2h_par[s], c->sC));
    return CKPT_OK;
}

static int rb_finish(ckpt_ctx *c, uint32_t kl) {
    CUDA_TRY(cudaEventRecord(c->ev_pack_all, c->sX));
    CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_pack_all, 0));
    CUDA_TRY(cudaEventRecord(c->ev_done, c->sC));
    if (c->me == kl && async_host_restore(c))  // DONE = device image complete, D2H continues
        return sig_signal(c, c->sX, kDone, c->op_seq_base + (uint32_t)c->op_NB + 1, 0);
    // DONE after every local stream finished
    return sig_signal(c, c->sC, kDone, c->op_seq_base + (uint32_t)c->op_NB + 1, 0);
}

// Wait for a background host restore (see async_host_restore) and publish it.
static int host_sync(ckpt_ctx *c) {
    if (!c->host_pending) return CKPT_OK;
    int rc = set_dev(c);
    if (rc) return rc;
    CUDA_TRY(cudaEventSynchronize(c->ev_done));
    c->host_pending = false;
    meta_commit(c);
    return CKPT_OK;
}

extern "C" int ckpt_sync(ckpt_ctx *c) {
    if (!c) return fail(CKPT_EINVAL, "sync: null");
    return host_sync(c);
}

static int rb_commit(ckpt_ctx *c, uint32_t kl, uint64_t version) {
    int rc;
    const bool bg = c->me == kl && async_host_restore(c);
    if (bg) {  // device image complete on sX; the copy stream is left running
        if (!(rc = sync_stream_timeout(c, c->sP, "rebuild")) && !(rc = sync_stream_timeout(c, c->sX, "rebuild")) &&
            c->transport == CKPT_GROUP_IPC && !(rc = wait_all(c, c->sW, kDone, c->op_seq_base + (uint32_t)c->op_NB + 1, 0)))
            rc = sync_stream_timeout(c, c->sW, "rebuild(peers)");
        if (!rc && c->transport == CKPT_GROUP_LOCAL)
            for (uint32_t j = 0; j < c->m && !rc; ++j)
                if (c->members[j] != c && cudaEventSynchronize(c->members[j]->ev_done) != cudaSuccess)
                    rc = fail(CKPT_ECUDA, "rebuild: peer event");
    } else {
        rc = wait_done_all(c, c->op_seq_base + (uint32_t)c->op_NB + 1);
    }
    if (!rc && (c->opt.flags & CKPT_OPT_TIMING)) rc = harvest_timing(c);
    if (rc) {
        make_sticky(c, rc);
        return rc;
    }
    if (c->me == kl) {
        clean_pad(c, rb_target(c));  // the pad is disjoint from the D2H'd [0, L)
        c->completed = rb_target(c);
        c->completed_id = version;
        if (bg)
            c->host_pending = true;  // meta is published by host_sync
        else
            meta_commit(c);
    }
    // full-copy staging now holds every member's completed image (survivors staged or
    // kept theirs, the lost member's was rebuilt and re-encoded in place)
    if (c->full_copy) c->staging_id = c->completed_id;
    c->st.rebuilds++;
    return CKPT_OK;
}

static int rebuild_aec(ckpt_ctx *c, int32_t lost, void *stream);
extern "C" int ckpt_recover(ckpt_ctx *c, uint32_t lost_mask, void *stream);

extern "C" int ckpt_rebuild(ckpt_ctx *c, int32_t lost, void *stream) {
    if (!c) return fail(CKPT_EINVAL, "rebuild: null");
    // ARC schemes also re-create the ARC copy the lost member held: the general path
    if (c->grouped && c->arc && lost >= 0 && (uint32_t)lost < c->m) return ckpt_recover(c, 1u << lost, stream);
    return rebuild_aec(c, lost, stream);
}

static int rebuild_aec(ckpt_ctx *c, int32_t lost, void *stream) {
    NvtxRange nvtx_("ckpt_rebuild");
    if (!c) return fail(CKPT_EINVAL, "rebuild: null");
    if (host_sync(c)) return CKPT_ECUDA;
    if (!c->registered || !c->grouped) return fail(CKPT_ESTATE, "rebuild: not protected");
    if (c->m < 2) return fail(CKPT_EUNRECOVERABLE, "rebuild: a group of one has no redundancy (P.460)");
    if (lost < 0 || (uint32_t)lost >= c->m) return fail(CKPT_EINVAL, "rebuild: lost rank %d out of range", lost);
    if (!c->aec) return fail(CKPT_EUNRECOVERABLE, "rebuild: the scheme has no parity");
    int rc = check_sticky(c);
    if (rc) return rc;
    if (c->pending_id || c->requested) return fail(CKPT_ESTATE, "rebuild: a snapshot is in flight");
    const uint32_t kl = (uint32_t)lost;
    if (c->me != kl && c->completed < 0)
        return fail(CKPT_EUNRECOVERABLE, "rebuild: survivor %u has no completed image (more than one loss)", c->me);
    if ((rc = set_dev(c))) return rc;
    cudaStream_t caller = (cudaStream_t)stream;
    const uint64_t B = effective_bucket(c, 0);
    if (c->transport == CKPT_GROUP_LOCAL) {
        c->rebuild_requested = true;
        c->rebuild_lost = lost;
        CUDA_TRY(cudaEventRecord(c->ev_capture, caller));
        for (uint32_t j = 0; j < c->m; ++j)
            if (!c->members[j]->rebuild_requested) return CKPT_OK;  // issued by the last member
        uint64_t version = 0;
        for (uint32_t j = 0; j < c->m; ++j) {
            ckpt_ctx *o = c->members[j];
            if (o->rebuild_lost != lost) return fail(CKPT_EINVAL, "rebuild: members disagree on the lost rank");
            if (j != kl) {
                if (o->completed < 0) return fail(CKPT_EUNRECOVERABLE, "rebuild: survivor %u has no completed image", j);
                version = std::max(version, o->completed_id);
            }
        }
        for (uint32_t j = 0; j < c->m; ++j) {
            ckpt_ctx *o = c->members[j];
            if ((rc = set_dev(o)) || (rc = prepare_op(o, B))) goto bad;
            CUDA_TRY(cudaStreamWaitEvent(o->sC, o->ev_capture, 0));
            CUDA_TRY(cudaStreamWaitEvent(o->sX, o->ev_capture, 0));
        }
        for (uint64_t b = 0; b < c->op_NB; ++b) {
            for (uint32_t j = 0; j < c->m; ++j)
                if ((rc = set_dev(c->members[j])) || (rc = rb_stage1(c->members[j], b, kl))) goto bad;
            for (uint32_t j = 0; j < c->m; ++j)
                if ((rc = set_dev(c->members[j])) || (rc = rb_stage2(c->members[j], b, kl))) goto bad;
            for (uint32_t j = 0; j < c->m; ++j)
                if ((rc = set_dev(c->members[j])) || (rc = rb_stage3(c->members[j], b, kl))) goto bad;
        }
        for (uint32_t j = 0; j < c->m; ++j)
            if ((rc = set_dev(c->members[j])) || (rc = rb_finish(c->members[j], kl))) goto bad;
        for (uint32_t j = 0; j < c->m; ++j) {
            ckpt_ctx *o = c->members[j];
            if ((rc = set_dev(o)) || (rc = rb_commit(o, kl, version))) goto bad;
            o->rebuild_requested = false;
        }
        return set_dev(c);
    bad:
        for (uint32_t j = 0; j < c->m; ++j) {
            make_sticky(c->members[j], rc);
            c->members[j]->rebuild_requested = false;
        }
        return rc;
    }
    // IPC: every member runs its own side; the version is the survivors' completed id
    if ((rc = prepare_op(c, B))) return rc;
    CUDA_TRY(cudaEventRecord(c->ev_capture, caller));
    CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_capture, 0));
    CUDA_TRY(cudaStreamWaitEvent(c->sX, c->ev_capture, 0));
    for (uint64_t b = 0; b < c->op_NB; ++b) {
        if ((rc = rb_stage1(c, b, kl)) || (rc = rb_stage2(c, b, kl)) || (rc = rb_stage3(c, b, kl))) {
            make_sticky(c, rc);
            return rc;
        }
    }
    if ((rc = rb_finish(c, kl))) {
        make_sticky(c, rc);
        return rc;
    }
    return rb_commit(c, kl, c->me == kl ? c->next_id - 1 : c->completed_id);
}

// ------------------------------------------------------------------ recover (1-2 losses)
// The oracle's oracle_recover, step by step: (1) ARC restore of every lost member whose
// holder survived (the member copies its image out of the holder's shared file), (2)
// AEC rebuild of one remaining loss (collective, rebuild_aec), (3) every lost member
// re-creates the ARC copy it holds from member me+1's completed image.
static inline uint32_t holder_of(const ckpt_ctx *c, uint32_t x) { return (x + c->m - 1) % c->m; }

static int recover_plan(const ckpt_ctx *c, uint32_t mask, int32_t *remaining) {
    *remaining = -1;
    const int nlost = __builtin_popcount(mask);
    if (nlost > 2) return fail(CKPT_EUNRECOVERABLE, "recover: %d losses (at most 2 are tolerated, P.507)", nlost);
    int left = 0;
    for (uint32_t x = 0; x < c->m; ++x) {
        if (!(mask & (1u << x))) continue;
        if (c->arc && !(mask & (1u << holder_of(c, x)))) continue;  // restored by ARC
        ++left;
        *remaining = (int32_t)x;
    }
    if (left > 1 || (left == 1 && !c->aec))
        return fail(CKPT_EUNRECOVERABLE, "recover: losses 0x%x exceed what scheme %u restores", mask, c->scheme);
    return CKPT_OK;
}

static int recover_step1(ckpt_ctx *c, uint32_t mask, uint64_t version) {
    if (!(mask & (1u << c->me)) || !c->arc || (mask & (1u << holder_of(c, c->me)))) return CKPT_OK;
    int rc = ensure_holder_mapped(c);
    if (rc) return rc;
    const int idx = rb_target(c);
    const uint64_t P = parity_bytes_of(c);
    // only [0, L) carries data; the zero pad is written here, never copied (a peer's pad
    // may still hold ckpt_forget poison while it is being cleaned)
    parallel_memcpy(c->hdata[idx].p, c->shm_hold[idx].p + c->Lstar + P, c->L);
    if (c->Lstar > c->L) memset(c->hdata[idx].p + c->L, 0, c->Lstar - c->L);
    if (c->aec) parallel_memcpy(c->hpar[idx].p, c->shm_hold[idx].p + 2 * c->Lstar + P, P);
    c->pad_dirty[idx] = false;
    c->completed = idx;
    c->completed_id = version;
    meta_commit(c);
    return CKPT_OK;
}

static int recover_step3(ckpt_ctx *c, uint32_t mask) {
    if (!(mask & (1u << c->me)) || !c->arc) return CKPT_OK;
    int rc = ensure_next_mapped(c);
    if (rc) return rc;
    const int idx = c->completed;
    if (idx < 0) return fail(CKPT_ESTATE, "recover: member %u has no completed image after restore", c->me);
    const uint64_t P = parity_bytes_of(c);
    const uint64_t Ln = c->peer_L[(c->me + 1) % c->m];
    parallel_memcpy(c->harc[idx], c->shm_next[idx].p, Ln);  // member me+1's data ...
    if (c->Lstar > Ln) memset(c->harc[idx] + Ln, 0, c->Lstar - Ln);  // ... and a clean pad
    if (c->aec) parallel_memcpy(c->harcp[idx], c->shm_next[idx].p + c->Lstar, P);
    c->arc_dirty[idx] = false;
    return CKPT_OK;
}

extern "C" int ckpt_recover(ckpt_ctx *c, uint32_t mask, void *stream) {
    NvtxRange nvtx_("ckpt_recover");
    if (!c) return fail(CKPT_EINVAL, "recover: null");
    if (!c->registered || !c->grouped) return fail(CKPT_ESTATE, "recover: not protected");
    if (c->m < 2) return fail(CKPT_EUNRECOVERABLE, "recover: a group of one has no redundancy (P.460)");
    if (mask >> c->m) return fail(CKPT_EINVAL, "recover: lost mask 0x%x names members >= m", mask);
    if (device_only(c) && c->arc) return fail(CKPT_EINVAL, "recover: ARC needs a host arena");
    int rc = check_sticky(c);
    if (rc) return rc;
    if (c->pending_id || c->requested) return fail(CKPT_ESTATE, "recover: a snapshot is in flight");
    int32_t rem;
    if ((rc = recover_plan(c, mask, &rem))) return rc;
    if (!mask) return CKPT_OK;
    if (!(mask & (1u << c->me)) && c->completed < 0)
        return fail(CKPT_ENOSNAP, "recover: survivor %u has no completed image", c->me);
    if (c->transport == CKPT_GROUP_LOCAL) {
        c->recover_requested = true;
        c->recover_mask = mask;
        c->recover_stream = stream;
        for (uint32_t j = 0; j < c->m; ++j)
            if (!c->members[j]->recover_requested) return CKPT_OK;  // run by the last member
        uint64_t version = 0;
        for (uint32_t j = 0; j < c->m; ++j) {
            ckpt_ctx *o = c->members[j];
            if (o->recover_mask != mask) return fail(CKPT_EINVAL, "recover: members disagree on the lost mask");
            if (!(mask & (1u << j))) version = std::max(version, o->completed_id);
        }
        for (uint32_t j = 0; j < c->m && !rc; ++j) rc = recover_step1(c->members[j], mask, version);
        for (uint32_t j = 0; j < c->m && !rc && rem >= 0; ++j)
            rc = rebuild_aec(c->members[j], rem, c->members[j]->recover_stream);
        for (uint32_t j = 0; j < c->m && !rc; ++j) rc = recover_step3(c->members[j], mask);
        for (uint32_t j = 0; j < c->m; ++j) c->members[j]->recover_requested = false;
        set_dev(c);
        return rc;
    }
    if ((rc = recover_step1(c, mask, c->next_id - 1))) return rc;
    if (rem >= 0 && (rc = rebuild_aec(c, rem, stream))) return rc;
    return recover_step3(c, mask);
}

// ------------------------------------------------------------------ HAS -------------
extern "C" int ckpt_window(ckpt_ctx *c, int open, void *stream) {
    if (!c) return fail(CKPT_EINVAL, "window: null");
    if (load_memops()) return fail(CKPT_ECUDA, "window: stream memory operations unavailable");
    int rc = set_dev(c);
    if (rc) return rc;
    CUresult r = p_write32((CUstream)stream, (CUdeviceptr)(uintptr_t)c->window, open ? 1u : 0u,
                           CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) return fail(CKPT_ECUDA, "cuStreamWriteValue32(window) failed (%d)", (int)r);
    return CKPT_OK;
}

extern "C" int ckpt_has_plan(uint32_t p, uint32_t P, double c, uint64_t bytes, double bio, ckpt_has_plan_t *out) {
    if (!out || P == 0 || p >= P || c < 0 || bio <= 0) return fail(CKPT_EINVAL, "has_plan: bad args");
    out->t_ss = (double)bytes / bio;                                          // EstimateSnapshotTime
    out->t_bubble = std::max(0.0, (0.8 * p + 2.0 * P - p - 2.0) * c);         // EstimateBubbleTime
    if (out->t_ss >= out->t_bubble && out->t_ss > 0) {                        // SplitParameter
        out->bubble_bytes = (uint64_t)std::floor((double)bytes * out->t_bubble / out->t_ss);
    } else {
        out->bubble_bytes = bytes;
    }
    out->compute_bytes = bytes - out->bubble_bytes;
    return CKPT_OK;
}

// ------------------------------------------------------------------ misc ------------
extern "C" int ckpt_forget(ckpt_ctx *c, uint8_t poison) {
    if (!c) return fail(CKPT_EINVAL, "forget: null");
    host_sync(c);
    if (c->pending_id || c->requested) return fail(CKPT_ESTATE, "forget: a snapshot is in flight");
    c->staging_id = 0;
    c->staging_poisoned = true;
    if (c->staging) {  // the device copy is lost with the member: poison staging + parity
        int rc = set_dev(c);
        if (rc) return rc;
        CUDA_TRY(cudaMemset(c->staging, poison, c->staging_bytes));
        if (c->parity) CUDA_TRY(cudaMemset(c->parity, poison, c->parity_bytes));
        CUDA_TRY(cudaDeviceSynchronize());
    }
    for (int i = 0; i < 2; ++i) {
        if (c->hdata[i].p) memset(c->hdata[i].p, poison, c->Lstar);
        if (c->hpar[i].p && c->m >= 2) memset(c->hpar[i].p, poison, c->Lstar / (c->m - 1));
        c->pad_dirty[i] = c->hdata[i].p != nullptr;
        if (c->harc[i]) {  // the ARC copy this member holds is lost with it
            memset(c->harc[i], poison, c->Lstar);
            if (c->harcp[i]) memset(c->harcp[i], poison, parity_bytes_of(c));
            c->arc_dirty[i] = true;
        }
    }
    c->completed = -1;
    c->completed_id = 0;
    meta_commit(c);
    return CKPT_OK;
}

extern "C" int ckpt_host_view(const ckpt_ctx *c, int which, const void **data, uint64_t *dlen, const void **par,
                              uint64_t *plen) {
    if (!c || which < 0 || which > 3) return fail(CKPT_EINVAL, "host_view: bad args");
    if (which >= 2) {
        if (!c->grouped || !c->arc) return fail(CKPT_EINVAL, "host_view: no ARC copy (scheme without ARC)");
        int idx = which == 2 ? c->completed : c->ongoing;
        if (idx < 0) return fail(CKPT_ENOSNAP, "host_view: no completed snapshot");
        if (data) *data = c->harc[idx];
        if (dlen) *dlen = c->Lstar;
        if (par) *par = c->harcp[idx];
        if (plen) *plen = c->harcp[idx] ? parity_bytes_of(c) : 0;
        return CKPT_OK;
    }
    if (!c->grouped) return fail(CKPT_ENOSNAP, "host_view: no host arena yet");
    if (host_sync(const_cast<ckpt_ctx *>(c))) return CKPT_ECUDA;
    if (device_only(c)) return fail(CKPT_EINVAL, "host_view: DEVICE_ONLY context has no host image");
    int idx = which == 0 ? c->completed : c->ongoing;
    if (idx < 0) return fail(CKPT_ENOSNAP, "host_view: no completed snapshot");
    if (data) *data = c->hdata[idx].p;
    if (dlen) *dlen = c->Lstar;
    if (par) *par = c->m >= 2 && c->aec ? c->hpar[idx].p : nullptr;
    if (plen) *plen = c->m >= 2 && c->aec ? c->Lstar / (c->m - 1) : 0;
    return CKPT_OK;
}

extern "C" int ckpt_get_stats(const ckpt_ctx *c, ckpt_stats *out) {
    if (!c || !out) return fail(CKPT_EINVAL, "get_stats: null");
    *out = c->st;
    return CKPT_OK;
}

extern "C" int ckpt_stats_reset(ckpt_ctx *c) {
    if (!c) return fail(CKPT_EINVAL, "stats_reset: null");
    c->st = ckpt_stats{};
    return CKPT_OK;
}
