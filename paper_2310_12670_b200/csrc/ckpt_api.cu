// ckpt_api.cu -- host side of libreft_ckpt, part 1: the C ABI entry points (errors,
// driver memops, planner, lifecycle, register, group handshake / arena allocation,
// HAS planner, misc).  The other units: ckpt_hostmem.cu (host memory), ckpt_pipeline.cu
// (snapshot stages, load), ckpt_recovery.cu (rebuild / recover); shared state in
// ckpt_internal.cuh.
//
// Default snapshot (n_slots = 0, full-copy staging):
//   stream P (pack)  : one pack_all launch over every bucket; the kernel publishes
//                      READY(k) to the local row and every peer as bucket k lands
//   stream C (copy)  : per bucket: wait READY(k) (memop) -> D2H data(k)  (copy engine)
//   stream X (xor)   : own pack, every peer's READY -> one xor_encode over the image
//                      (peer reads over NVLink) -> D2H parity -> REL to every peer
//   end              : DONE to every peer; ckpt_wait waits DONE from all, commits.
// Slotted pipeline (n_slots > 0), per bucket k (slot s = k mod n_slots):
//   P: [slot reuse: own D2H(k-n), peers' XOR(k-n)] pack(k) -> READY(k) to every peer
//   X: own pack(k), peers' READY(k) -> xor_encode(k) -> REL(k) to every peer
//   C: D2H data slot(k) ; D2H parity slot(k)
// Cross-rank signals are 32-bit sequence numbers.  IPC groups write them into the
// peers' flag pages with stream memory operations (cuStreamWriteValue32 /
// cuStreamWaitValue32: zero SMs, no NCCL on the data path); LOCAL groups (all
// members in this process) use CUDA events instead.
#include "ckpt_internal.cuh"

using namespace reft;

// ------------------------------------------------------------------ errors ----------
thread_local std::string g_last_error;

int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}


// ------------------------------------------------------------------ driver memops ---
PFN_cuStreamWaitValue32_v8000 p_wait32 = nullptr;
PFN_cuStreamWriteValue32_v8000 p_write32 = nullptr;
static std::once_flag g_memop_once;
static int g_memop_status = CKPT_ECUDA;

int load_memops() {
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
    o->stripe_unit = 1024 * 1024;  // Q4; round 2: 1 MiB reads the m = 4 rows at the fabric's rate
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
    if (const char *x = getenv("CKPT_XOR_CTAS"); x && atoi(x) > 0) c->xor_ctas_push = atoi(x);
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
        const uint32_t all = CKPT_WINDOW_BUBBLE | CKPT_WINDOW_COMPUTE;  // windows start open
        e = cudaMemcpy(c->window, &all, sizeof all, cudaMemcpyHostToDevice);
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
    for (auto &t : c->host_bg)  // background host copies of an ARC restore
        if (t.joinable()) t.join();
    cudaSetDevice(c->device);
    if (c->window && (c->opt.flags & CKPT_OPT_WINDOWED)) {
        // a snapshot still waiting for a HAS window the caller will never open: open every
        // window so the copy stream drains (the gated copies not yet enqueued are dropped)
        cudaStream_t t = nullptr;
        if (cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking) == cudaSuccess) {
            cudaMemsetAsync(c->window, 0xff, sizeof(uint32_t), t);
            cudaStreamSynchronize(t);
            cudaStreamDestroy(t);
        }
        cudaGetLastError();
    }
    cudaStream_t ss[5] = {c->sP, c->sX, c->sC, c->sW, c->sG};
    for (auto s : ss)
        if (s) cudaStreamSynchronize(s);
    for (uint32_t j = 0; j < CKPT_MAX_GROUP; ++j) {
        if (c->peer_opened[j]) {
            if (c->peer_staging[j]) cudaIpcCloseMemHandle(c->peer_staging[j]);
            if (c->peer_flags[j]) cudaIpcCloseMemHandle(c->peer_flags[j]);
        }
        if (c->peer_parity_opened[j]) cudaIpcCloseMemHandle(c->peer_parity[j]);
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
    b.opt_flags = c->opt.flags;
    CUDA_TRY(cudaIpcGetMemHandle(&b.staging_h, c->staging));
    CUDA_TRY(cudaIpcGetMemHandle(&b.flags_h, c->flags));
    memset(buf, 0, CKPT_HANDLE_BYTES);
    memcpy(buf, &b, sizeof b);
    *len = CKPT_HANDLE_BYTES;
    return CKPT_OK;
}




int alloc_arena(ckpt_ctx *c) {
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
void meta_commit(ckpt_ctx *c) {
    if (!c->meta) return;
    const uint64_t st = c->completed < 0 ? 0 : (c->completed_id << 8) | (uint64_t)(c->completed + 1);
    __atomic_store_n(&c->meta->state, st, __ATOMIC_RELEASE);
}

// ARC push targets: the files of my holder (member me-1), pinned so that my copy engine
// can D2H straight into the holder's ARC-copy region.  Mapped at first use (the holder
// creates them in its own ckpt_protect).
int ensure_holder_mapped(ckpt_ctx *c) {
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
int ensure_next_mapped(ckpt_ctx *c) {
    const uint32_t nx = (c->me + 1) % c->m;
    for (int i = 0; i < c->nbuf; ++i) {
        if (c->shm_next[i].p) continue;
        int rc = shm_map(c->shm_next[i], shm_name(c->group_nonce, nx, i), shm_bytes(c), false);
        if (rc) return rc;
    }
    return CKPT_OK;
}

int setup_ungrouped(ckpt_ctx *c) {
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
            if ((hb[j]->opt_flags ^ c->opt.flags) & (CKPT_OPT_REBUILD_SHARES | CKPT_OPT_REBUILD_SELF | CKPT_OPT_XOR_PUSH))
                return fail(CKPT_EMISMATCH, "protect: members disagree on CKPT_OPT_REBUILD_SHARES / _SELF / CKPT_OPT_XOR_PUSH (member %u)", j);
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
            if ((g->members[j]->opt.flags ^ c->opt.flags) & (CKPT_OPT_REBUILD_SHARES | CKPT_OPT_REBUILD_SELF | CKPT_OPT_XOR_PUSH))
                return fail(CKPT_EMISMATCH, "protect: members disagree on CKPT_OPT_REBUILD_SHARES / _SELF / CKPT_OPT_XOR_PUSH (member %u)", j);
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
    if (c->aec && c->transport == CKPT_GROUP_IPC) {  // published for a rebuild of this member
        cudaIpcMemHandle_t h;
        CUDA_TRY(cudaIpcGetMemHandle(&h, c->parity));
        CUDA_TRY(cudaMemcpy((uint8_t *)c->flags + kParityHandleOff, &h, sizeof h, cudaMemcpyHostToDevice));
    }
    if (c->aec && (c->opt.flags & CKPT_OPT_CE_GATHER) && m > 2) {  // m = 2: pulled into the parity
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

// ------------------------------------------------------------------ HAS -------------
extern "C" int ckpt_window(ckpt_ctx *c, int open, void *stream) {
    if (!c) return fail(CKPT_EINVAL, "window: null");
    if (load_memops()) return fail(CKPT_ECUDA, "window: stream memory operations unavailable");
    int rc = set_dev(c);
    if (rc) return rc;
    if (open < 0 || (open & ~(int)(CKPT_WINDOW_BUBBLE | CKPT_WINDOW_COMPUTE | CKPT_WINDOW_COMM)))
        return fail(CKPT_EINVAL, "window: open must be a mask of CKPT_WINDOW_BUBBLE | CKPT_WINDOW_COMPUTE | CKPT_WINDOW_COMM");
    CUresult r = p_write32((CUstream)stream, (CUdeviceptr)(uintptr_t)c->window, (uint32_t)open,
                           CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) return fail(CKPT_ECUDA, "cuStreamWriteValue32(window) failed (%d)", (int)r);
    return issue_gated_more(c);  // a pending windowed snapshot: enqueue the next gated copies
}

extern "C" int ckpt_has_apply(ckpt_ctx *c, uint64_t bubble_bytes) {
    return ckpt_has_apply_layers(c, bubble_bytes, UINT64_MAX);
}

extern "C" int ckpt_has_apply_layers(ckpt_ctx *c, uint64_t bubble_bytes, uint64_t compute_bytes) {
    if (!c) return fail(CKPT_EINVAL, "has_apply: null");
    c->has_bubble_bytes = bubble_bytes;
    c->has_compute_bytes = compute_bytes;
    return CKPT_OK;
}

extern "C" int ckpt_has_plan3(uint32_t p, uint32_t P, double c, uint64_t bytes, double bio, double t_compute,
                              ckpt_has_plan3_t *out) {
    if (!out || t_compute < 0) return fail(CKPT_EINVAL, "has_plan3: bad args");
    ckpt_has_plan_t a;
    int rc = ckpt_has_plan(p, P, c, bytes, bio, &a);
    if (rc) return rc;
    out->t_ss = a.t_ss;
    out->t_bubble = a.t_bubble;
    out->t_compute = t_compute;
    out->bubble_bytes = a.bubble_bytes;
    const uint64_t rest = a.compute_bytes;
    const double cap = a.t_ss > 0 ? std::floor((double)bytes * t_compute / a.t_ss) : (double)rest;
    out->compute_bytes = cap >= (double)rest ? rest : (uint64_t)cap;
    out->comm_bytes = rest - out->compute_bytes;
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

