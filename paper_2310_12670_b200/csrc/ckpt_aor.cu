// ckpt_aor.cu -- Asynchronous Optimizer Recomputing (PAPER.md P.494-505, Eq 4 P.502-504;
// include/ckpt_aor.h).
//
// Member i holds, in a POSIX shared-memory object, the fp32 replica of the ZeRO-1
// optimizer shard of member h = (i+1) mod m.  One ckpt_aor_step, all enqueued by the
// caller's thread at the call:
//   caller's stream : ... backward (gradient complete on every member, P.495) -> [ready]
//   copy stream     : wait [ready]; per chunk g (global index over all steps, slot g mod S):
//                       [g >= S: memop-wait CONSUMED >= g-S+1]  (the host freed the slot)
//                       D2H grad[bounds[h] + k*c : +c] -> staging slot
//                       memop-write LANDED = g+1                (host-mapped word)
//                     after the step's last chunk: memop-write the fence flag (device word;
//                     ckpt_aor_fence waits on it, zero SMs)
//   host worker     : per chunk: poll LANDED, apply Eq 4 to the replica with the thread
//                     pool, store CONSUMED = g+1
// The worker makes no CUDA call at all: a caller blocked inside the driver (a synchronous
// copy waiting on the fence, say) can never stall it, so the ring cannot deadlock.  No
// kernels: the update runs on "redundant host FLOPs" (P.505), the copies on copy engines.
#include "ckpt_internal.cuh"
#pragma GCC visibility push(default)
#include "../../include/ckpt_aor.h"
#pragma GCC visibility pop

#include <condition_variable>
#include <deque>
#include <functional>
#include <memory>

namespace reft {
void aor_sgd(float *w, const void *g, uint32_t dtype, uint64_t n, float eta, bool simd);
bool aor_simd();

constexpr uint32_t kAorMagic = 0x524F4152u;  // "RAOR"
constexpr uint32_t kAorVersion = 1;
constexpr uint64_t kAorHdr = 4096;           // header page; the replica starts page-aligned

struct AorHdr {  // offset 0 of every replica object
    uint32_t magic, version;
    uint64_t key;
    uint32_t owner, holder, m, reserved;
    uint64_t n;       // replica elements (fp32)
    uint64_t digest;  // of (m, bounds): every member must describe the same partition
    uint64_t state;   // (step << 8) | CKPT_AOR_*; atomic
};

inline uint64_t hdr_state(const AorHdr *h) { return __atomic_load_n(&h->state, __ATOMIC_ACQUIRE); }
inline void hdr_set(AorHdr *h, uint64_t step, uint32_t code) {
    __atomic_store_n(&h->state, (step << 8) | code, __ATOMIC_RELEASE);
}

std::string aor_name(uint64_t key, uint32_t j) {
    char s[64];
    snprintf(s, sizeof s, "/reft-aor-%016llx-%u", (unsigned long long)key, j);
    return s;
}

const char *aor_state_name(uint32_t code) {
    switch (code) {
        case CKPT_AOR_EMPTY: return "empty (never seeded)";
        case CKPT_AOR_CLEAN: return "clean";
        case CKPT_AOR_UPDATING: return "torn (an update was in flight)";
        case CKPT_AOR_POISONED: return "poisoned";
        case CKPT_AOR_SEEDING: return "torn (a seed was in flight)";
        default: return "corrupt";
    }
}

// A fixed set of host threads running one parallel-for at a time (the caller is thread 0).
class Pool {
  public:
    explicit Pool(unsigned nt) : nt_(std::max(1u, nt)) {
        for (unsigned i = 1; i < nt_; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> l(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto &t : th_) t.join();
    }
    unsigned size() const { return nt_; }
    void run(const std::function<void(unsigned)> &f) {
        if (nt_ == 1) return f(0);
        {
            std::lock_guard<std::mutex> l(mu_);
            fn_ = &f;
            pending_ = nt_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        f(0);
        std::unique_lock<std::mutex> l(mu_);
        done_.wait(l, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

  private:
    void loop(unsigned i) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(unsigned)> *f;
            {
                std::unique_lock<std::mutex> l(mu_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                f = fn_;
            }
            (*f)(i);
            std::lock_guard<std::mutex> l(mu_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    unsigned nt_;
    std::vector<std::thread> th_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    const std::function<void(unsigned)> *fn_ = nullptr;
    unsigned pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};
}  // namespace reft

struct ckpt_aor {
    int device = -1;
    ckpt_aor_options opt{};
    uint32_t m = 0, me = 0, owner = 0, holder = 0;  // owner: whose replica I hold; holder: who holds mine
    std::vector<uint64_t> bounds;
    uint64_t digest = 0;
    float *master = nullptr;
    const uint8_t *grad = nullptr;
    uint64_t n_me = 0, n_rep = 0;
    uint32_t esz = 4;
    uint64_t chunk_elems = 0, nchunks = 0, S = 0;

    HostBuf staging, own, peer;  // own: the object I hold; peer: my holder's (seed/restore)
    bool peer_alias = false;     // m = 1: my holder is me
    AorHdr *own_hdr = nullptr, *peer_hdr = nullptr;
    float *replica = nullptr, *peer_rep = nullptr;

    cudaStream_t sC = nullptr;
    uint32_t *dflag = nullptr;    // fence flag (device), written by a stream memop
    uint32_t *hflags = nullptr;   // host-mapped: [0] LANDED (device writes), [32] CONSUMED (host writes)
    CUdeviceptr d_landed = 0, d_consumed = 0;
    std::unique_ptr<Pool> pool;
    std::thread worker;

    struct Job {
        uint64_t step;
        float eta;
        uint32_t fence_seq;
        std::chrono::steady_clock::time_point t0;
    };
    mutable std::mutex mu;
    std::condition_variable cv_work, cv_done;
    std::deque<Job> jobs;
    uint64_t job_base = 0;   // global index of jobs.front()
    uint64_t enq_chunks = 0, processed = 0;
    uint64_t last_step = 0;  // the last id returned by ckpt_aor_step
    uint64_t done_step = 0;  // the replica's step once the queue drains
    uint32_t fence_seq = 0;
    int sticky = CKPT_OK;         // an enqueue failed: the stream state is unknown
    std::string sticky_msg;
    std::atomic<bool> stop{false};
    ckpt_aor_stats st{};
};

namespace {

double timeout_s() {
    const char *e = getenv("CKPT_TIMEOUT_S");
    return e ? atof(e) : 600.0;
}

uint64_t partition_digest(uint32_t m, const uint64_t *b) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](uint64_t v) {
        for (int i = 0; i < 8; ++i) {
            h ^= (v >> (8 * i)) & 0xff;
            h *= 1099511628211ull;
        }
    };
    mix(m);
    for (uint32_t j = 0; j <= m; ++j) mix(b[j]);
    return h;
}

int set_sticky_locked(ckpt_aor *a, int code, const std::string &msg) {
    if (a->sticky == CKPT_OK) {
        a->sticky = code;
        a->sticky_msg = msg;
    }
    a->cv_done.notify_all();
    return code;
}

int sticky_error(ckpt_aor *a) { return fail(a->sticky, "aor: %s", a->sticky_msg.c_str()); }

// Cyclic comparison of the 32-bit progress words: v has reached `want`.
inline bool reached(uint32_t v, uint64_t want) { return (int32_t)(v - (uint32_t)want) >= 0; }

// Enqueue the copy-stream work of one step's chunks (caller's thread, mu held).
int enqueue_chunks_locked(ckpt_aor *a, cudaEvent_t ready, uint32_t fence_seq) {
    cudaError_t e = cudaStreamWaitEvent(a->sC, ready, 0);
    if (e != cudaSuccess) return fail(CKPT_ECUDA, "aor_step: %s", cudaGetErrorString(e));
    for (uint64_t k = 0; k < a->nchunks; ++k) {
        const uint64_t g = a->enq_chunks + k, slot = g % a->S;
        if (g >= a->S && p_wait32((CUstream)a->sC, a->d_consumed, (uint32_t)(g - a->S + 1),
                                  CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
            return fail(CKPT_ECUDA, "aor_step: slot wait failed");
        const uint64_t e0 = k * a->chunk_elems, len = std::min(a->chunk_elems, a->n_rep - e0);
        e = cudaMemcpyAsync(a->staging.p + slot * a->opt.chunk_bytes, a->grad + (a->bounds[a->owner] + e0) * a->esz,
                            len * a->esz, cudaMemcpyDeviceToHost, a->sC);
        if (e != cudaSuccess) return fail(CKPT_ECUDA, "aor_step: D2H: %s", cudaGetErrorString(e));
        if (p_write32((CUstream)a->sC, a->d_landed, (uint32_t)(g + 1), CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
            return fail(CKPT_ECUDA, "aor_step: landed flag write failed");
        a->st.d2h_bytes += len * a->esz;
    }
    if (p_write32((CUstream)a->sC, (CUdeviceptr)(uintptr_t)a->dflag, fence_seq, CU_STREAM_WRITE_VALUE_DEFAULT) !=
        CUDA_SUCCESS)
        return fail(CKPT_ECUDA, "aor_step: fence flag write failed");
    a->enq_chunks += a->nchunks;
    return CKPT_OK;
}

// The host worker: no CUDA calls (see the file comment).
void worker_main(ckpt_aor *a) {
    volatile uint32_t *landed = a->hflags, *consumed = a->hflags + 32;
    for (;;) {
        uint64_t g;
        ckpt_aor::Job J;
        {
            std::unique_lock<std::mutex> l(a->mu);
            a->cv_work.wait(l, [&] { return a->stop.load() || a->processed < a->enq_chunks; });
            if (a->stop.load()) return;
            g = a->processed;
            J = a->jobs[g / a->nchunks - a->job_base];
        }
        const uint64_t k = g % a->nchunks, slot = g % a->S;
        if (k == 0) hdr_set(a->own_hdr, J.step, CKPT_AOR_UPDATING);
        auto t0 = std::chrono::steady_clock::now();
        for (unsigned spin = 0; !reached(__atomic_load_n(landed, __ATOMIC_ACQUIRE), g + 1); ++spin) {
            if (a->stop.load()) return;
            if (spin < 2048) {
                __builtin_ia32_pause();
            } else {
                std::this_thread::sleep_for(std::chrono::microseconds(20));
            }
        }
        auto t1 = std::chrono::steady_clock::now();
        const uint64_t e0 = k * a->chunk_elems, len = std::min(a->chunk_elems, a->n_rep - e0);
        const uint8_t *src = a->staging.p + slot * a->opt.chunk_bytes;
        float *dst = a->replica + e0;
        const unsigned nt = a->pool->size();
        const uint64_t per = align_up((len + nt - 1) / nt, 16);
        const uint32_t dt = a->opt.grad_dtype, esz = a->esz;
        const float eta = J.eta;
        a->pool->run([&](unsigned i) {
            const uint64_t lo = std::min(len, i * per), hi = std::min(len, lo + per);
            if (lo < hi) aor_sgd(dst + lo, src + lo * esz, dt, hi - lo, eta, true);
        });
        auto t2 = std::chrono::steady_clock::now();
        __atomic_store_n(consumed, (uint32_t)(g + 1), __ATOMIC_RELEASE);  // frees the slot
        std::lock_guard<std::mutex> l(a->mu);
        a->st.stall_s += std::chrono::duration<double>(t1 - t0).count();
        a->st.update_s += std::chrono::duration<double>(t2 - t1).count();
        a->st.chunks++;
        a->processed++;
        if (k == a->nchunks - 1) {
            hdr_set(a->own_hdr, J.step, CKPT_AOR_CLEAN);
            a->done_step = J.step;
            a->st.steps++;
            a->st.last_step_ms = std::chrono::duration<double, std::milli>(t2 - J.t0).count();
            a->jobs.pop_front();
            a->job_base++;
            a->cv_done.notify_all();
        }
    }
}

// Host-block until the queue is empty (mu not held).
int drain(ckpt_aor *a) {
    std::unique_lock<std::mutex> l(a->mu);
    const auto limit = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s());
    while (a->sticky == CKPT_OK && !a->jobs.empty())
        if (a->cv_done.wait_until(l, limit) == std::cv_status::timeout && !a->jobs.empty())
            return fail(CKPT_ESTATE, "aor: updates did not drain within %.0f s", timeout_s());
    return a->sticky == CKPT_OK ? CKPT_OK : sticky_error(a);
}

// Map my holder's replica object (it holds the replica of MY shard): wait for it (seed) or
// require it (restore), then check that it describes my shard.
int map_peer(ckpt_aor *a, bool wait) {
    if (a->peer_hdr) return CKPT_OK;
    if (a->holder == a->me) {
        a->peer_alias = true;
        a->peer_hdr = a->own_hdr;
        a->peer_rep = a->replica;
        return CKPT_OK;
    }
    const std::string name = aor_name(a->opt.key, a->holder);
    const uint64_t bytes = kAorHdr + a->n_me * 4;
    int rc = wait ? shm_map(a->peer, name, bytes, true) : shm_attach(a->peer, name, bytes, true);
    if (rc == CKPT_ENOSNAP)
        return fail(CKPT_EUNRECOVERABLE, "aor: the replica of member %u (held by member %u) does not exist",
                    a->me, a->holder);
    if (rc != CKPT_OK) return rc;
    AorHdr *h = (AorHdr *)a->peer.p;
    if (h->magic != kAorMagic || h->key != a->opt.key || h->owner != a->me || h->n != a->n_me ||
        h->digest != a->digest) {
        host_free(a->peer);
        return fail(CKPT_EMISMATCH, "aor: object %s does not hold member %u's shard of this partition",
                    name.c_str(), a->me);
    }
    a->peer_hdr = h;
    a->peer_rep = (float *)(a->peer.p + kAorHdr);
    return CKPT_OK;
}

}  // namespace

extern "C" {

void ckpt_aor_options_default(ckpt_aor_options *o) {
    if (!o) return;
    memset(o, 0, sizeof *o);
    o->struct_size = sizeof *o;
    o->grad_dtype = CKPT_DTYPE_FP32;
    o->chunk_bytes = 16ull << 20;
    o->n_slots = 0;
    o->threads = 0;
    o->priority = INT32_MIN;  // resolved to the device's least priority
    o->flags = 0;
    o->key = 0;
}

int ckpt_aor_create(int device, const ckpt_aor_options *o, const ckpt_aor_shard *s, ckpt_aor **out) {
    NvtxRange nv("ckpt_aor_create");
    if (!out || !s) return fail(CKPT_EINVAL, "aor_create: null argument");
    *out = nullptr;
    ckpt_aor_options opt;
    ckpt_aor_options_default(&opt);
    if (o) {
        if (o->struct_size != sizeof(ckpt_aor_options)) return fail(CKPT_EINVAL, "aor_create: struct_size mismatch");
        opt = *o;
    }
    if (opt.key == 0) return fail(CKPT_EINVAL, "aor_create: options.key must be non-zero");
    if (opt.grad_dtype != CKPT_DTYPE_FP32 && opt.grad_dtype != CKPT_DTYPE_BF16)
        return fail(CKPT_EINVAL, "aor_create: grad_dtype must be FP32 or BF16");
    if (opt.chunk_bytes < (64u << 10) || opt.chunk_bytes % 4096)
        return fail(CKPT_EINVAL, "aor_create: chunk_bytes must be a multiple of 4096 and >= 64 KiB");
    if (opt.n_slots == 1) return fail(CKPT_EINVAL, "aor_create: n_slots must be 0 or >= 2");
    if (opt.flags & ~CKPT_AOR_PERSIST) return fail(CKPT_EINVAL, "aor_create: unknown flags");
    if (s->m < 1 || s->m > CKPT_MAX_GROUP || s->my_index >= s->m || !s->bounds)
        return fail(CKPT_EINVAL, "aor_create: bad group (m=%u, my_index=%u)", s->m, s->my_index);
    if (s->bounds[0] != 0) return fail(CKPT_EINVAL, "aor_create: bounds[0] must be 0");
    for (uint32_t j = 0; j < s->m; ++j)
        if (s->bounds[j + 1] < s->bounds[j]) return fail(CKPT_EINVAL, "aor_create: bounds must be non-decreasing");

    auto a = std::make_unique<ckpt_aor>();
    a->device = device;
    a->opt = opt;
    a->m = s->m;
    a->me = s->my_index;
    a->owner = (a->me + 1) % a->m;
    a->holder = (a->me + a->m - 1) % a->m;
    a->bounds.assign(s->bounds, s->bounds + s->m + 1);
    a->digest = partition_digest(a->m, s->bounds);
    a->master = s->master;
    a->grad = (const uint8_t *)s->grad;
    a->n_me = a->bounds[a->me + 1] - a->bounds[a->me];
    a->n_rep = a->bounds[a->owner + 1] - a->bounds[a->owner];
    a->esz = opt.grad_dtype == CKPT_DTYPE_BF16 ? 2 : 4;
    a->chunk_elems = opt.chunk_bytes / a->esz;
    a->nchunks = (a->n_rep + a->chunk_elems - 1) / a->chunk_elems;
    a->S = opt.n_slots ? opt.n_slots : std::max<uint64_t>(1, a->nchunks);
    if (a->n_me && !a->master) return fail(CKPT_EINVAL, "aor_create: null master");
    if (a->n_rep && !a->grad) return fail(CKPT_EINVAL, "aor_create: null grad");

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
        cudaGetLastError();
        return fail(CKPT_ECUDA, "aor_create: no CUDA device %d", device);
    }
    CUDA_TRY(cudaSetDevice(device));
    if (load_memops() != CKPT_OK) return fail(CKPT_ECUDA, "aor_create: stream memory operations unavailable");
    auto on_device = [&](const void *p) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) && at.device == device;
    };
    if (a->n_me && !on_device(a->master)) return fail(CKPT_EINVAL, "aor_create: master is not memory of device %d", device);
    if (a->bounds[a->m] && !on_device(a->grad)) return fail(CKPT_EINVAL, "aor_create: grad is not memory of device %d", device);

    // The replica object this member holds: re-attach (same key: a restarted process) or create.
    const std::string name = aor_name(opt.key, a->me);
    const uint64_t obytes = kAorHdr + a->n_rep * 4;
    // pinned only when this member is its own holder (m = 1: seed and restore copy it over
    // PCIe); otherwise only host threads touch it
    const bool own_reg = a->holder == a->me;
    int rc = shm_attach(a->own, name, obytes, own_reg);
    if (rc == CKPT_OK) {
        AorHdr *h = (AorHdr *)a->own.p;
        if (h->magic != kAorMagic || h->version != kAorVersion || h->key != opt.key || h->owner != a->owner ||
            h->holder != a->me || h->m != a->m || h->n != a->n_rep || h->digest != a->digest) {
            host_free(a->own);
            return fail(CKPT_EMISMATCH, "aor_create: existing object %s describes another geometry", name.c_str());
        }
    } else if (rc == CKPT_ENOSNAP) {
        if ((rc = shm_create(a->own, name, obytes, own_reg)) != CKPT_OK) return rc;
        a->own.kind = kShmPeer;  // unlinked explicitly by destroy (unless persistent)
        AorHdr *h = (AorHdr *)a->own.p;
        h->magic = kAorMagic;
        h->version = kAorVersion;
        h->key = opt.key;
        h->owner = a->owner;
        h->holder = a->me;
        h->m = a->m;
        h->n = a->n_rep;
        h->digest = a->digest;
        hdr_set(h, 0, CKPT_AOR_EMPTY);
    } else {
        return rc;
    }
    a->own_hdr = (AorHdr *)a->own.p;
    a->replica = (float *)(a->own.p + kAorHdr);
    a->done_step = hdr_state(a->own_hdr) >> 8;

    auto cleanup_fail = [&](int code) {
        ckpt_aor_destroy(a.release());
        return code;
    };
    if (a->nchunks && (rc = host_alloc(a->staging, a->S * opt.chunk_bytes)) != CKPT_OK) return cleanup_fail(rc);
    int lo = 0, hi = 0;
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return cleanup_fail(fail(CKPT_ECUDA, "aor: priority range"));
    const int prio = opt.priority == INT32_MIN ? lo : std::max(hi, std::min(lo, opt.priority));
    if (cudaStreamCreateWithPriority(&a->sC, cudaStreamNonBlocking, prio) != cudaSuccess)
        return cleanup_fail(fail(CKPT_ECUDA, "aor: stream create failed"));
    if (cudaMalloc(&a->dflag, 128) != cudaSuccess || cudaMemset(a->dflag, 0, 128) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
        return cleanup_fail(fail(CKPT_ENOMEM, "aor: flag allocation failed"));
    void *dh = nullptr;
    if (cudaHostAlloc((void **)&a->hflags, 4096, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
        cudaHostGetDevicePointer(&dh, a->hflags, 0) != cudaSuccess) {
        cudaGetLastError();
        return cleanup_fail(fail(CKPT_ENOMEM, "aor: mapped host flags allocation failed"));
    }
    memset(a->hflags, 0, 4096);
    a->d_landed = (CUdeviceptr)(uintptr_t)dh;
    a->d_consumed = a->d_landed + 32 * sizeof(uint32_t);
    unsigned nt = opt.threads;
    if (nt == 0) nt = std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2));
    a->pool = std::make_unique<Pool>(nt);
    ckpt_aor *raw = a.get();
    a->worker = std::thread(worker_main, raw);
    *out = a.release();
    return CKPT_OK;
}

int ckpt_aor_destroy(ckpt_aor *a) {
    if (!a) return CKPT_OK;
    NvtxRange nv("ckpt_aor_destroy");
    int rc = (a->worker.joinable() && a->sticky == CKPT_OK) ? drain(a) : CKPT_OK;
    if (a->worker.joinable()) {
        {
            std::lock_guard<std::mutex> l(a->mu);
            a->stop = true;
        }
        a->cv_work.notify_all();
        a->worker.join();
    }
    a->pool.reset();
    if (a->device >= 0) cudaSetDevice(a->device);
    if (a->sC) {
        // after a failed drain, release every slot wait so the copy stream can finish
        if (a->hflags) __atomic_store_n(a->hflags + 32, (uint32_t)a->enq_chunks, __ATOMIC_RELEASE);
        cudaStreamSynchronize(a->sC);
        cudaStreamDestroy(a->sC);
    }
    if (a->dflag) cudaFree(a->dflag);
    if (a->hflags) cudaFreeHost(a->hflags);
    host_free(a->staging);
    if (!a->peer_alias) host_free(a->peer);
    const bool had_own = a->own.p != nullptr;
    host_free(a->own);
    if (had_own && !(a->opt.flags & CKPT_AOR_PERSIST)) shm_unlink(aor_name(a->opt.key, a->me).c_str());
    cudaGetLastError();
    delete a;
    return rc;
}

int ckpt_aor_seed(ckpt_aor *a, uint64_t step, void *stream) {
    NvtxRange nv("ckpt_aor_seed");
    if (!a) return fail(CKPT_EINVAL, "aor_seed: null context");
    if (a->sticky != CKPT_OK) return sticky_error(a);
    if (step >> 56) return fail(CKPT_EINVAL, "aor_seed: step out of range");
    CUDA_TRY(cudaSetDevice(a->device));
    int rc = map_peer(a, true);
    if (rc != CKPT_OK) return rc;
    if (a->peer_alias && (rc = drain(a)) != CKPT_OK) return rc;
    hdr_set(a->peer_hdr, step, CKPT_AOR_SEEDING);
    if (a->n_me) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        cudaError_t err = cudaEventRecord(e, (cudaStream_t)stream);
        if (err == cudaSuccess) err = cudaStreamWaitEvent(a->sC, e, 0);
        if (err == cudaSuccess)
            err = cudaMemcpyAsync(a->peer_rep, a->master, a->n_me * 4, cudaMemcpyDeviceToHost, a->sC);
        if (err == cudaSuccess) err = cudaStreamSynchronize(a->sC);
        cudaEventDestroy(e);
        if (err != cudaSuccess) return fail(CKPT_ECUDA, "aor_seed: %s", cudaGetErrorString(err));
        std::lock_guard<std::mutex> l(a->mu);
        a->st.d2h_bytes += a->n_me * 4;
    }
    hdr_set(a->peer_hdr, step, CKPT_AOR_CLEAN);
    if (a->peer_alias) {
        std::lock_guard<std::mutex> l(a->mu);
        a->done_step = step;
    }
    return CKPT_OK;
}

int ckpt_aor_step(ckpt_aor *a, float eta, void *stream, uint64_t *out) {
    NvtxRange nv("ckpt_aor_step");
    if (!a) return fail(CKPT_EINVAL, "aor_step: null context");
    CUDA_TRY(cudaSetDevice(a->device));
    std::lock_guard<std::mutex> l(a->mu);
    if (a->sticky != CKPT_OK) return sticky_error(a);
    uint64_t t;
    if (a->jobs.empty()) {
        const uint64_t s = hdr_state(a->own_hdr);
        if ((s & 0xff) != CKPT_AOR_CLEAN)
            return fail(CKPT_ESTATE, "aor_step: the held replica of member %u is %s", a->owner,
                        aor_state_name((uint32_t)(s & 0xff)));
        t = s >> 8;
        a->done_step = t;
    } else {
        t = a->last_step;
    }
    const uint64_t step = t + 1;
    const uint32_t seq = ++a->fence_seq;
    cudaEvent_t ready;
    CUDA_TRY(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    cudaError_t e = cudaEventRecord(ready, (cudaStream_t)stream);
    if (e != cudaSuccess) {
        cudaEventDestroy(ready);
        return fail(CKPT_ECUDA, "aor_step: %s", cudaGetErrorString(e));
    }
    a->last_step = step;
    if (a->nchunks == 0) {  // an empty replica: nothing to copy or apply
        e = cudaStreamWaitEvent(a->sC, ready, 0);
        cudaEventDestroy(ready);
        if (e != cudaSuccess) return fail(CKPT_ECUDA, "aor_step: %s", cudaGetErrorString(e));
        if (p_write32((CUstream)a->sC, (CUdeviceptr)(uintptr_t)a->dflag, seq, CU_STREAM_WRITE_VALUE_DEFAULT) !=
            CUDA_SUCCESS)
            return fail(CKPT_ECUDA, "aor_step: fence flag write failed");
        hdr_set(a->own_hdr, step, CKPT_AOR_CLEAN);
        a->done_step = step;
        a->st.steps++;
        a->st.last_step_ms = 0;
    } else {
        int rc = enqueue_chunks_locked(a, ready, seq);
        cudaEventDestroy(ready);  // released once the copy stream's wait on it has resolved
        if (rc != CKPT_OK) {
            set_sticky_locked(a, rc, ckpt_last_error());
            return rc;
        }
        a->jobs.push_back({step, eta, seq, std::chrono::steady_clock::now()});
        a->cv_work.notify_one();
    }
    if (out) *out = step;
    return CKPT_OK;
}

int ckpt_aor_fence(ckpt_aor *a, uint64_t step, void *stream) {
    if (!a) return fail(CKPT_EINVAL, "aor_fence: null context");
    CUDA_TRY(cudaSetDevice(a->device));
    uint32_t seq = 0;
    {
        std::lock_guard<std::mutex> l(a->mu);
        if (a->sticky != CKPT_OK) return sticky_error(a);
        if (step > a->last_step) return fail(CKPT_EINVAL, "aor_fence: step %llu was never issued",
                                             (unsigned long long)step);
        for (const auto &J : a->jobs)
            if (J.step == step) seq = J.fence_seq;
        if (seq == 0 && a->nchunks == 0 && step == a->last_step) seq = a->fence_seq;
    }
    if (seq == 0) return CKPT_OK;  // already applied: its gradient was copied long ago
    CUresult r = p_wait32((CUstream)stream, (CUdeviceptr)(uintptr_t)a->dflag, seq, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) return fail(CKPT_ECUDA, "aor_fence: stream wait failed (%d)", (int)r);
    return CKPT_OK;
}

int ckpt_aor_wait(ckpt_aor *a, uint64_t step) {
    NvtxRange nv("ckpt_aor_wait");
    if (!a) return fail(CKPT_EINVAL, "aor_wait: null context");
    std::unique_lock<std::mutex> l(a->mu);
    const auto limit = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s());
    for (;;) {
        if (a->sticky != CKPT_OK) return sticky_error(a);
        if (a->jobs.empty()) {
            const uint64_t s = hdr_state(a->own_hdr);
            if ((s & 0xff) == CKPT_AOR_CLEAN && (s >> 8) >= step) return CKPT_OK;
            return fail(CKPT_ESTATE, "aor_wait: the replica is %s at step %llu (< %llu)",
                        aor_state_name((uint32_t)(s & 0xff)), (unsigned long long)(s >> 8),
                        (unsigned long long)step);
        }
        if (a->done_step >= step && a->jobs.front().step > step) return CKPT_OK;
        if (a->cv_done.wait_until(l, limit) == std::cv_status::timeout)
            return fail(CKPT_ESTATE, "aor_wait: step %llu not applied within %.0f s", (unsigned long long)step,
                        timeout_s());
    }
}

int ckpt_aor_restore(ckpt_aor *a, void *stream, uint64_t *out) {
    NvtxRange nv("ckpt_aor_restore");
    if (!a) return fail(CKPT_EINVAL, "aor_restore: null context");
    if (a->sticky != CKPT_OK) return sticky_error(a);
    CUDA_TRY(cudaSetDevice(a->device));
    if (a->holder == a->me) {
        int rc = drain(a);
        if (rc != CKPT_OK) return rc;
    }
    int rc = map_peer(a, false);
    if (rc != CKPT_OK) return rc;
    const uint64_t s = hdr_state(a->peer_hdr);
    if ((s & 0xff) != CKPT_AOR_CLEAN)
        return fail(CKPT_EUNRECOVERABLE, "aor_restore: the replica of member %u held by member %u is %s", a->me,
                    a->holder, aor_state_name((uint32_t)(s & 0xff)));
    if (a->n_me) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        cudaError_t err = cudaMemcpyAsync(a->master, a->peer_rep, a->n_me * 4, cudaMemcpyHostToDevice, a->sC);
        if (err == cudaSuccess) err = cudaEventRecord(e, a->sC);
        if (err == cudaSuccess) err = cudaStreamWaitEvent((cudaStream_t)stream, e, 0);
        if (err == cudaSuccess) err = cudaStreamSynchronize(a->sC);
        cudaEventDestroy(e);
        if (err != cudaSuccess) return fail(CKPT_ECUDA, "aor_restore: %s", cudaGetErrorString(err));
        std::lock_guard<std::mutex> l(a->mu);
        a->st.h2d_bytes += a->n_me * 4;
    }
    if (hdr_state(a->peer_hdr) != s)
        return fail(CKPT_ESTATE, "aor_restore: the replica changed during the restore (holder not quiescent)");
    if (out) *out = s >> 8;
    return CKPT_OK;
}

int ckpt_aor_forget(ckpt_aor *a, uint8_t poison) {
    if (!a) return fail(CKPT_EINVAL, "aor_forget: null context");
    int rc = drain(a);
    if (rc != CKPT_OK) return rc;
    memset(a->replica, poison, a->n_rep * 4);
    hdr_set(a->own_hdr, 0, CKPT_AOR_POISONED);
    return CKPT_OK;
}

int ckpt_aor_view(ckpt_aor *a, const float **replica, uint64_t *n, uint64_t *step, uint32_t *state) {
    if (!a) return fail(CKPT_EINVAL, "aor_view: null context");
    int rc = drain(a);
    if (rc != CKPT_OK) return rc;
    const uint64_t s = hdr_state(a->own_hdr);
    if (replica) *replica = a->replica;
    if (n) *n = a->n_rep;
    if (step) *step = s >> 8;
    if (state) *state = (uint32_t)(s & 0xff);
    return CKPT_OK;
}

int ckpt_aor_get_stats(const ckpt_aor *a, ckpt_aor_stats *out) {
    if (!a || !out) return fail(CKPT_EINVAL, "aor_get_stats: null argument");
    std::lock_guard<std::mutex> l(a->mu);
    *out = a->st;
    return CKPT_OK;
}

int ckpt_aor_unlink(uint64_t key, uint32_t m) {
    if (key == 0 || m == 0 || m > CKPT_MAX_GROUP) return fail(CKPT_EINVAL, "aor_unlink: bad args");
    for (uint32_t j = 0; j < m; ++j) shm_unlink(aor_name(key, j).c_str());
    return CKPT_OK;
}

int ckpt_aor_apply(float *w, const void *grad, uint32_t grad_dtype, uint64_t n, float eta) {
    if (n && (!w || !grad)) return fail(CKPT_EINVAL, "aor_apply: null buffer");
    if (grad_dtype != CKPT_DTYPE_FP32 && grad_dtype != CKPT_DTYPE_BF16)
        return fail(CKPT_EINVAL, "aor_apply: grad_dtype must be FP32 or BF16");
    aor_sgd(w, grad, grad_dtype, n, eta, true);
    return CKPT_OK;
}

}  // extern "C"
