// ckpt_hostmem.cu -- small helpers and host memory: pinned/THP arenas, POSIX shared-memory files, timing events
#include "ckpt_internal.cuh"

using namespace reft;

// ------------------------------------------------------------------ small helpers ---
int set_dev(ckpt_ctx *c) {
    CUDA_TRY(cudaSetDevice(c->device));
    return CKPT_OK;
}

int ensure_events(std::vector<cudaEvent_t> &v, size_t n) {
    while (v.size() < n) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        v.push_back(e);
    }
    return CKPT_OK;
}

void destroy_events(std::vector<cudaEvent_t> &v) {
    for (auto e : v) cudaEventDestroy(e);
    v.clear();
}

// Timed launch bracket (CKPT_OPT_TIMING): events on the launching stream.
int timed_begin(ckpt_ctx *c, cudaStream_t s, int kind, TimedLaunch **out) {
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

int timed_end(TimedLaunch *t, cudaStream_t s) {
    if (t) CUDA_TRY(cudaEventRecord(t->b, s));
    return CKPT_OK;
}

int harvest_timing(ckpt_ctx *c) {
    for (size_t i = 0; i < c->timed_used; ++i) {
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, c->timed[i].a, c->timed[i].b));
        switch (c->timed[i].kind) {
            case 0: c->st.pack_ms += ms; break;
            case 1: c->st.xor_ms += ms; break;
            case 2: c->st.unpack_ms += ms; break;
            case 4: c->st.gather_ms += ms; break;
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
void prefault(uint8_t *p, uint64_t len) {
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
void parallel_memcpy(uint8_t *dst, const uint8_t *src, uint64_t n) {
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

int host_alloc(HostBuf &b, uint64_t bytes) {
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
std::string shm_name(uint64_t nonce, uint32_t member, int buf) {
    char s[64];
    snprintf(s, sizeof s, "/reft-%016llx-%u-%d", (unsigned long long)nonce, member, buf);
    return s;
}

int shm_create(HostBuf &b, const std::string &name, uint64_t bytes, bool reg) {
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
    if (reg && cudaHostRegister(p, len, cudaHostRegisterPortable) != cudaSuccess) {
        cudaGetLastError();
        munmap(p, len);
        shm_unlink(name.c_str());
        return fail(CKPT_ENOMEM, "cudaHostRegister of shm %s (%llu bytes) failed", name.c_str(), (unsigned long long)len);
    }
    b.p = (uint8_t *)p;
    b.bytes = len;
    b.kind = kShmOwn;
    b.registered = reg;
    b.name = name;
    return CKPT_OK;
}

int shm_map(HostBuf &b, const std::string &name, uint64_t bytes, bool reg) {
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
int shm_attach(HostBuf &b, const std::string &name, uint64_t bytes, bool reg) {
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

std::string meta_name(uint64_t key, uint32_t member) {
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

void host_free(HostBuf &b) {
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

