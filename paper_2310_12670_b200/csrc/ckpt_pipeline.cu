// ckpt_pipeline.cu -- the snapshot pipeline: cross-rank signals, kernel wrappers, bucket stages, snapshot/fence/wait, load
#include "ckpt_internal.cuh"

using namespace reft;


// ------------------------------------------------------------------ signals ---------
// IPC signals: cuStreamWriteValue32 into the peer's flag page (zero SMs).  Waits are
// cuStreamWaitValue32 on the local flag page.
// signal(stage, seq): tell every other member that this member reached `seq`.
int sig_signal(ckpt_ctx *c, cudaStream_t s, int stage, uint32_t seq, uint32_t slot) {
    if (c->m < 2) return CKPT_OK;
    if (c->transport == CKPT_GROUP_IPC) {
        auto addr = [&](uint32_t j) {
            return stage == kReady ? ready_row(c->peer_flags[j], c->me) + seq % kMaxB
                                   : c->peer_flags[j] + stage * kFlagStride + c->me;
        };
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
int sig_wait(ckpt_ctx *c, cudaStream_t s, uint32_t j, int stage, uint32_t seq, uint32_t slot) {
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

int wait_all(ckpt_ctx *c, cudaStream_t s, int stage, uint32_t seq, uint32_t slot, int32_t skip) {
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
int do_pack_ce(ckpt_ctx *c, uint64_t k, uint8_t *slot, cudaStream_t s, bool unpack) {
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

int do_pack(ckpt_ctx *c, uint64_t k, uint8_t *slot, cudaStream_t s, bool unpack) {
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
int do_encode(ckpt_ctx *c, uint64_t k, cudaStream_t s) {
    return do_encode_range(c, k, bucket_begin(c, k), bucket_end(c, k), s);
}
int do_encode_range(ckpt_ctx *c, uint64_t k, uint64_t bb, uint64_t be, cudaStream_t s) {
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
int do_rebuild_row(ckpt_ctx *c, uint64_t k, uint32_t kl, cudaStream_t s) {
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

// Re-encode lost rank kl's parity row (Eq 1 for row kl) on the survivors: every term of
// row kl is a survivor's data unit sigma(kl, j), so survivor i (i-th of the m-1) XORs
// stripes [s0, s1) of the bucket -- its own unit locally, m-2 over NVLink -- and stores
// the result into kl's parity slot.  The lost GPU then receives L* of data + L*/(m-1) of
// parity instead of pulling L* more to encode the row itself (reading Q27).
int do_encode_lost_share(ckpt_ctx *c, uint64_t k, uint32_t kl, cudaStream_t s) {
    const uint64_t bb = bucket_begin(c, k), be = bucket_end(c, k);
    const uint64_t stripe = (uint64_t)(c->m - 1) * c->unit;
    const uint64_t nst = (be - bb) / stripe;
    const uint32_t i = c->me - (c->me > kl ? 1u : 0u);
    const uint64_t s0 = nst * i / (c->m - 1), s1 = nst * (i + 1) / (c->m - 1);
    if (s1 <= s0) return CKPT_OK;
    if (!c->peer_parity[kl]) return fail(CKPT_ESTATE, "internal: parity of member %u not mapped", kl);
    XorArgs a;
    memset(&a, 0, sizeof a);
    for (uint32_t j = 0; j < c->m; ++j) {
        if (j == kl) continue;
        XorTerm &t = a.in[a.nin++];
        const uint64_t v = valid_in_bucket(c->peer_L[j], bb, be);
        t.base = slot_ptr(c, c->peer_staging[j], k) + s0 * stripe;
        t.valid = v > s0 * stripe ? v - s0 * stripe : 0;
        t.stride = stripe;
        t.off = (uint64_t)sigma(kl, j) * c->unit;
    }
    a.out = parity_slot_ptr_at(c, c->peer_parity[kl], k) + s0 * c->unit;
    a.out_valid = UINT64_MAX;
    a.out_stride = c->unit;
    a.out_off = 0;
    a.nstripes = s1 - s0;
    a.unit = c->unit;
    TimedLaunch *t;
    int rc = timed_begin(c, s, 3, &t);
    if (rc) return rc;
    CUDA_TRY(launch_xor(a, c->xor_ctas, s));
    rc = timed_end(t, s);
    if (rc) return rc;
    c->st.rebuild_launches++;
    c->st.rebuild_bytes_in += (uint64_t)a.nin * (s1 - s0) * c->unit;
    c->st.rebuild_bytes_out += (s1 - s0) * c->unit;
    return CKPT_OK;
}

// Map lost member kl's parity buffer (survivors only): LOCAL members share the process;
// IPC members read the handle kl published in its flag page at ckpt_protect.
int rebuild_map_parity(ckpt_ctx *c, uint32_t kl, bool wait) {
    if (c->me == kl || c->peer_parity[kl]) return CKPT_OK;
    if (c->transport == CKPT_GROUP_LOCAL) {
        c->peer_parity[kl] = c->members[kl]->parity;
        return c->peer_parity[kl] ? CKPT_OK : fail(CKPT_ESTATE, "rebuild: member %u has no parity buffer", kl);
    }
    cudaIpcMemHandle_t h;
    static const cudaIpcMemHandle_t zero = {};
    cudaStream_t t = nullptr;  // non-blocking: must not wait for the training streams
    CUDA_TRY(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
    // with `wait` (push encode: the peer may still be inside ckpt_protect) poll until the
    // handle appears, up to CKPT_TIMEOUT_S
    double limit = 600.0;
    if (const char *x = getenv("CKPT_TIMEOUT_S")) limit = atof(x);
    const auto t0 = std::chrono::steady_clock::now();
    cudaError_t e;
    for (;;) {
        memset(&h, 0, sizeof h);
        e = cudaMemcpyAsync(&h, (const uint8_t *)c->peer_flags[kl] + kParityHandleOff, sizeof h, cudaMemcpyDeviceToHost, t);
        if (e == cudaSuccess) e = cudaStreamSynchronize(t);
        if (e != cudaSuccess || !wait || memcmp(&h, &zero, sizeof h)) break;
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) break;
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
    }
    cudaStreamDestroy(t);
    if (e != cudaSuccess) return fail(CKPT_ECUDA, "rebuild: reading member %u's parity handle: %s", kl, cudaGetErrorString(e));
    if (!memcmp(&h, &zero, sizeof h)) return fail(CKPT_EPEER, "member %u published no parity handle", kl);
    void *p = nullptr;
    e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(CKPT_EPEER, "rebuild: cudaIpcOpenMemHandle of member %u's parity: %s", kl, cudaGetErrorString(e));
    }
    c->peer_parity[kl] = (uint8_t *)p;
    c->peer_parity_opened[kl] = true;
    return CKPT_OK;
}

// ------------------------------------------------------------------ snapshot --------
// The image's zero pad [L, L*) is structural (Q5) and never written by a D2H (which
// covers [0, L)); after ckpt_forget poisoned a buffer, re-zero it before it commits.
void clean_pad(ckpt_ctx *c, int buf) {
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

int check_sticky(ckpt_ctx *c) {
    if (c->sticky) return fail(c->sticky, "context has a sticky error: %s", c->sticky_msg.c_str());
    return CKPT_OK;
}

void make_sticky(ckpt_ctx *c, int rc) {
    if (!c->sticky) {
        c->sticky = rc;
        c->sticky_msg = g_last_error;
    }
    group_abort(c);  // peers waiting on this member's signals fail fast instead of timing out
}

// Write (my index + 1) into every peer's abort word (IPC groups; LOCAL members share the
// thread that failed).  Best effort: errors are ignored, the message of the failure stands.
void group_abort(ckpt_ctx *c) {
    if (c->abort_sent || c->transport != CKPT_GROUP_IPC || c->m < 2 || !c->grouped) return;
    c->abort_sent = true;
    const std::string keep = g_last_error;
    int dev = -1;
    cudaGetDevice(&dev);
    cudaSetDevice(c->device);
    cudaStream_t t = nullptr;
    if (cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking) == cudaSuccess) {
        static const uint32_t v[CKPT_MAX_GROUP] = {1, 2, 3, 4, 5, 6, 7, 8};
        for (uint32_t j = 0; j < c->m; ++j)
            if (j != c->me && c->peer_flags[j])
                cudaMemcpyAsync((uint8_t *)c->peer_flags[j] + kAbortOff, &v[c->me], 4, cudaMemcpyHostToDevice, t);
        cudaStreamSynchronize(t);
        cudaStreamDestroy(t);
    }
    cudaGetLastError();
    if (dev >= 0) cudaSetDevice(dev);
    g_last_error = keep;
}

// (index + 1) of a peer that aborted the group, or 0.
uint32_t peer_aborted(ckpt_ctx *c) {
    if (c->transport != CKPT_GROUP_IPC || c->m < 2 || !c->flags) return 0;
    uint32_t v = 0;
    cudaStream_t t = nullptr;
    if (cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    if (cudaMemcpyAsync(&v, (const uint8_t *)c->flags + kAbortOff, 4, cudaMemcpyDeviceToHost, t) == cudaSuccess)
        cudaStreamSynchronize(t);
    cudaStreamDestroy(t);
    cudaGetLastError();
    return v;
}

// Bucket = whole stripes ((m-1)u; A when unprotected).  With full-copy staging the
// single-launch pack also needs whole 64 KiB tile groups: B is rounded down to a
// multiple of lcm(stripe, kGroup).

uint64_t effective_bucket(const ckpt_ctx *c, uint64_t req) {
    uint64_t B = req ? req : c->opt.bucket_bytes;
    uint64_t q = c->m >= 2 ? (uint64_t)(c->m - 1) * c->unit : (uint64_t)c->opt.align;
    if (c->full_copy) q = q / std::gcd(q, kGroup) * kGroup;
    return std::max<uint64_t>(q, B / q * q);
}

bool single_launch(const ckpt_ctx *c) {
    return c->full_copy && !(c->opt.flags & CKPT_OPT_CE_PACK) &&
           (c->transport == CKPT_GROUP_LOCAL && c->m >= 2 ? true : load_memops() == CKPT_OK);
}

// The whole snapshot's pack as one launch (full-copy staging); the kernel publishes each
// bucket's READY flag itself (see PackAllArgs).  Buckets past this rank's L hold no data
// and are published up front.
int issue_pack_all(ckpt_ctx *c) {
    const uint64_t nb_data = (c->L + c->op_B - 1) / c->op_B;
    int rc;
    // push encode: the peers XOR-reduce into this parity stream; zero it before anything
    // this snapshot publishes (the peers' reductions wait for this member's READY)
    if (xor_push(c)) CUDA_TRY(cudaMemsetAsync(c->parity, 0, c->Lstar / (c->m - 1), c->sP));
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

int prepare_op(ckpt_ctx *c, uint64_t B) {
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
int stage_pack(ckpt_ctx *c, uint64_t k) {
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


// m = 2 is a mirror (Eq 1 with one term: P_r = D_{1-r}, zero-padded to L*, P.459): the
// copy engine pulls the peer's bucket straight into the parity slot and no XOR kernel runs.
bool ce_mirror(const ckpt_ctx *c) { return c->m == 2 && c->aec && (c->opt.flags & CKPT_OPT_CE_GATHER); }

int do_gather_ce(ckpt_ctx *c, uint64_t k, cudaStream_t s) {
    const uint64_t bb = bucket_begin(c, k), be = bucket_end(c, k);
    const uint64_t u = c->unit, pitch = (uint64_t)(c->m - 1) * u, nst = (be - bb) / pitch;
    const uint64_t gs = gather_stride(c, k);
    uint8_t *g = ce_mirror(c) ? parity_slot_ptr(c, k) : gather_slot_ptr(c, k);
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

int do_encode_gathered(ckpt_ctx *c, uint64_t k, cudaStream_t s) {
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
int stage_xor_all(ckpt_ctx *c) {
    int rc;
    CUDA_TRY(cudaStreamWaitEvent(c->sX, c->ev_pack_all, 0));
    for (uint64_t k = 0; k < c->op_NB; ++k)
        if ((rc = wait_all(c, c->sX, kReady, bucket_seq(c, k), slot_of(c, k)))) return rc;
    if ((rc = do_encode_range(c, 0, 0, c->Lstar, c->sX))) return rc;
    for (uint64_t k = 0; k < c->op_NB; ++k) CUDA_TRY(cudaEventRecord(c->ev_xored[slot_of(c, k)], c->sX));
    // REL is a monotonic scalar: one signal covers every bucket
    return sig_signal(c, c->sX, kRel, bucket_seq(c, c->op_NB - 1), slot_of(c, c->op_NB - 1));
}

// One encode launch over the whole image after this member's pack, also in DEVICE_ONLY
// mode where the parity is the critical path: round 2 tried per-bucket launches that start
// as soon as every member published bucket k (overlapping the packs), and the N=2
// device-only step got SLOWER (21.86 vs 21.30 ms): each 512 MiB launch ran at 575 GB/s
// against 675 for the single launch (pipeline fill and drain per launch, gaps at the
// READY waits), which ate the 3.5 ms of overlap (profiles/r02/r02p_n2_dev.jsonl).
bool xor_in_one_launch(const ckpt_ctx *c) {
    return c->m >= 2 && c->aec && single_launch(c) && !(c->opt.flags & CKPT_OPT_CE_GATHER);
}

bool xor_push(const ckpt_ctx *c) { return (c->opt.flags & CKPT_OPT_XOR_PUSH) && xor_in_one_launch(c); }

// Push-mode encode (CKPT_OPT_XOR_PUSH), part 1 on this member's XOR stream: once this
// member's pack is done (its own image is the only input) and every peer has zeroed its
// parity -- which precedes that peer's first READY in its stream order (issue_pack_all) --
// push every unit of the image into its row owner's parity as bulk XOR reductions, then
// tell every peer (REL) that its parity holds this member's terms.
int push_issue(ckpt_ctx *c) {
    int rc;
    if (!c->parity_peers_mapped) {  // once: every peer's parity stream, for the reductions
        for (uint32_t j = 0; j < c->m; ++j)
            if (j != c->me && (rc = rebuild_map_parity(c, j, true))) return rc;
        c->parity_peers_mapped = true;
    }
    CUDA_TRY(cudaStreamWaitEvent(c->sX, c->ev_pack_all, 0));
    if ((rc = wait_all(c, c->sX, kReady, bucket_seq(c, 0), slot_of(c, 0)))) return rc;
    XorPushArgs a;
    memset(&a, 0, sizeof a);
    a.src = c->staging;
    a.L = c->L;
    a.unit = c->unit;
    a.m = c->m;
    a.me = c->me;
    for (uint32_t r = 0; r < c->m; ++r) a.dst[r] = r == c->me ? nullptr : c->peer_parity[r];
    TimedLaunch *t;
    if ((rc = timed_begin(c, c->sX, 1, &t))) return rc;
    const int ctas = std::max(1, std::min(c->xor_ctas_push, c->max_ctas));
    CUDA_TRY(launch_xor_push(a, ctas, c->sX));
    if ((rc = timed_end(t, c->sX))) return rc;
    c->st.xor_launches++;
    c->st.xor_bytes_in += c->L;  // NVLink bytes of the encode: this member's image, out
    c->st.xor_bytes_out += c->Lstar / (c->m - 1);
    return sig_signal(c, c->sX, kRel, bucket_seq(c, c->op_NB - 1), slot_of(c, c->op_NB - 1));
}

// Part 2 (after every member's part 1 was issued -- LOCAL groups issue them in one
// thread): this member's parity row is complete once every peer's REL arrived.
int push_collect(ckpt_ctx *c) {
    int rc;
    if ((rc = wait_all(c, c->sX, kRel, bucket_seq(c, c->op_NB - 1), slot_of(c, c->op_NB - 1)))) return rc;
    for (uint64_t k = 0; k < c->op_NB; ++k) CUDA_TRY(cudaEventRecord(c->ev_xored[slot_of(c, k)], c->sX));
    return CKPT_OK;
}

int stage_xor(ckpt_ctx *c, uint64_t k) {
    if (c->m < 2 || !c->aec) return CKPT_OK;
    if (xor_in_one_launch(c)) return k + 1 == c->op_NB ? (xor_push(c) ? push_issue(c) : stage_xor_all(c)) : CKPT_OK;
    const uint32_t s = slot_of(c, k);
    int rc;
    if (c->opt.flags & CKPT_OPT_CE_GATHER) {
        if ((rc = wait_all(c, c->sG, kReady, bucket_seq(c, k), s))) return rc;
        if (ring_reuse(c, k)) CUDA_TRY(cudaStreamWaitEvent(c->sG, c->ev_xored[s], 0));
        if (ce_mirror(c)) {  // the gathered unit IS the parity: no XOR kernel
            if (ring_reuse(c, k)) CUDA_TRY(cudaStreamWaitEvent(c->sG, c->ev_d2h_par[s], 0));
            TimedLaunch *t;
            if ((rc = timed_begin(c, c->sG, 4, &t))) return rc;
            if ((rc = do_gather_ce(c, k, c->sG))) return rc;
            if ((rc = timed_end(t, c->sG))) return rc;
            c->st.gather_ops++;
            CUDA_TRY(cudaEventRecord(c->ev_xored[s], c->sG));
            return sig_signal(c, c->sG, kRel, bucket_seq(c, k), s);
        }
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
int stage_copy(ckpt_ctx *c, uint64_t k, bool with_parity) {
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
    if (v && (c->opt.flags & CKPT_OPT_WINDOWED)) {  // HAS: only while its window is open
        CUresult r = p_wait32((CUstream)c->sC, (CUdeviceptr)(uintptr_t)c->window, window_of(c, k),
                              CU_STREAM_WAIT_VALUE_AND);
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

int stage_copy_parity(ckpt_ctx *c, uint64_t k) {
    if (c->m < 2 || !c->aec) return CKPT_OK;
    const uint32_t s = slot_of(c, k);
    const uint64_t bb = bucket_begin(c, k), be = bucket_end(c, k);
    const uint64_t pb = (be - bb) / (c->m - 1);
    CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_xored[s], 0));
    if (!device_only(c) && (c->opt.flags & CKPT_OPT_WINDOWED)) {
        CUresult r = p_wait32((CUstream)c->sC, (CUdeviceptr)(uintptr_t)c->window, window_of(c, k),
                              CU_STREAM_WAIT_VALUE_AND);
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

int stage_finish(ckpt_ctx *c) {
    CUDA_TRY(cudaEventRecord(c->ev_pack_all, c->sP));
    CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_pack_all, 0));
    if (c->m >= 2 && c->aec) CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_xored[slot_of(c, c->op_NB ? c->op_NB - 1 : 0)], 0));
    CUDA_TRY(cudaEventRecord(c->ev_done, c->sC));
    if (c->opt.flags & CKPT_OPT_TIMING) CUDA_TRY(cudaEventRecord(c->ev_t1, c->sC));
    const uint32_t done_seq = c->op_seq_base + (uint32_t)c->op_NB + 1;
    int rc;
    if (c->m >= 2 && (rc = sig_signal(c, c->sC, kDone, done_seq, 0))) return rc;
    if (c->m < 2 || c->transport == CKPT_GROUP_IPC) {
        // completion = this member's last stream event and every peer's DONE, all queued on
        // sW now: ckpt_wait then polls ONE stream (small snapshots are latency-bound)
        CUDA_TRY(cudaStreamWaitEvent(c->sW, c->ev_done, 0));
        if (c->m >= 2 && (rc = wait_all(c, c->sW, kDone, done_seq, 0))) return rc;
        c->done_enqueued = true;
    }
    return CKPT_OK;
}

int begin_member(ckpt_ctx *c, cudaStream_t caller, uint64_t B) {
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

// HAS windows with one process per member: a gated copy waits on the device until the
// training stream opens its window, and the training stream is driven by the caller's
// thread -- so if ckpt_snapshot enqueued every bucket at once, a stream queue could fill
// and block that thread before it opens the first window (observed: a C3 snapshot of 700
// 32 MiB buckets hung in ckpt_snapshot).  The gated ops (data bucket g < NB; with full-copy
// staging, parity bucket g - NB after all data) are enqueued at most kGatedAhead beyond
// the last one whose copy completed; ckpt_window, ckpt_test and ckpt_wait top up.
constexpr uint64_t kGatedAhead = 32;

bool gated_progressive(const ckpt_ctx *c) {
    return (c->opt.flags & CKPT_OPT_WINDOWED) && !device_only(c) && !(c->transport == CKPT_GROUP_LOCAL && c->m >= 2);
}

int issue_gated(ckpt_ctx *c) {
    int rc;
    const bool one = single_launch(c);
    while (c->gate_next < c->gate_total) {
        if (c->gate_next >= kGatedAhead) {
            const uint64_t g = c->gate_next - kGatedAhead;
            cudaEvent_t e = g < c->op_NB ? c->ev_d2h_data[slot_of(c, g)] : c->ev_d2h_par[slot_of(c, g - c->op_NB)];
            const cudaError_t q = cudaEventQuery(e);
            if (q == cudaErrorNotReady) return CKPT_OK;
            if (q != cudaSuccess) return fail(CKPT_ECUDA, "snapshot: %s", cudaGetErrorString(q));
        }
        const uint64_t g = c->gate_next;
        if (g >= c->op_NB) {
            rc = stage_copy_parity(c, g - c->op_NB);
        } else if (c->full_copy) {
            rc = stage_copy(c, g, false);
        } else {  // ring staging: the whole bucket (its pack waits on an older bucket's copy)
            if (!one && (rc = stage_pack(c, g))) return rc;
            if ((rc = stage_xor(c, g)) == CKPT_OK) rc = stage_copy(c, g, true);
        }
        if (rc) return rc;
        ++c->gate_next;
    }
    if (c->gate_tail) {
        if ((rc = stage_finish(c))) return rc;
        c->gate_tail = false;
    }
    return CKPT_OK;
}

// top-up from the training thread's calls (no-op when nothing is pending)
int issue_gated_more(ckpt_ctx *c) {
    if (!c->issued || (c->gate_next >= c->gate_total && !c->gate_tail)) return CKPT_OK;
    int rc = issue_gated(c);
    if (rc) make_sticky(c, rc);
    return rc;
}

bool gated_pending(const ckpt_ctx *c) { return c->issued && (c->gate_next < c->gate_total || c->gate_tail); }

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
            if (xor_push(c))
                for (uint32_t j = 0; j < c->m; ++j)
                    if ((rc = set_dev(c->members[j])) || (rc = push_collect(c->members[j]))) goto bad;
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
    if (gated_progressive(c)) {
        // the un-gated device work first (pack, parity), then the window-gated copies a
        // few at a time: the rest is issued from ckpt_window / ckpt_test / ckpt_wait
        for (uint64_t k = 0; c->full_copy && k < c->op_NB; ++k)
            if ((!one && (rc = stage_pack(c, k))) || (rc = stage_xor(c, k))) {
                make_sticky(c, rc);
                return rc;
            }
        if (c->full_copy && !one) CUDA_TRY(cudaEventRecord(c->ev_pack_all, c->sP));  // every pack issued: ckpt_fence
        if (c->full_copy && xor_push(c) && (rc = push_collect(c))) {
            make_sticky(c, rc);
            return rc;
        }
        c->gate_next = 0;
        c->gate_total = c->op_NB + (c->full_copy && c->m >= 2 && c->aec ? c->op_NB : 0);
        c->gate_tail = true;
        c->pending_id = my_id;
        c->issued = true;
        c->st.snapshots++;
        if ((rc = issue_gated(c))) {
            make_sticky(c, rc);
            return rc;
        }
        if (id) *id = my_id;
        return CKPT_OK;
    }
    for (uint64_t k = 0; k < c->op_NB; ++k) {
        if ((!one && (rc = stage_pack(c, k))) || (rc = stage_xor(c, k)) || (rc = stage_copy(c, k, !c->full_copy))) {
            make_sticky(c, rc);
            return rc;
        }
    }
    if (xor_push(c) && (rc = push_collect(c))) {
        make_sticky(c, rc);
        return rc;
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
    if (!c->full_copy && gated_pending(c) && (rc = issue_gated_more(c))) return rc;
    if (!c->full_copy && gated_pending(c))
        return fail(CKPT_EBUSY, "fence: windowed ring snapshot %llu still issuing its packs (open the HAS windows, "
                                "then ckpt_test / ckpt_wait)", (unsigned long long)id);
    CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, c->ev_pack_all, 0));
    return CKPT_OK;
}

// Host-side wait on a stream with a timeout (peers that died never signal).
int sync_stream_timeout(ckpt_ctx *c, cudaStream_t s, const char *what) {
    double limit = 600.0;
    if (const char *e = getenv("CKPT_TIMEOUT_S")) limit = atof(e);
    auto t0 = std::chrono::steady_clock::now();
    double next_abort_check = 0.1;
    for (;;) {
        cudaError_t e = cudaStreamQuery(s);
        if (e == cudaSuccess) return CKPT_OK;
        if (e != cudaErrorNotReady) return fail(CKPT_ECUDA, "%s: %s", what, cudaGetErrorString(e));
        double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        uint32_t ab = 0;
        if (el > next_abort_check) {  // a peer's collective failed: it will never signal
            next_abort_check = el + 0.02;
            ab = peer_aborted(c);
        }
        if (ab || el > limit) {
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
            cudaMemset(c->flags, 0x7f, kAbortOff);  // release our waits: the REL/DONE lines
            cudaMemset((uint8_t *)c->flags + kFlagBytes, 0x7f, kFlagAlloc - kFlagBytes);  // and the READY rows
            cudaGetLastError();
            if (ab) {
                c->abort_sent = true;  // the group is gone: do not echo the abort
                return fail(CKPT_EPEER, "%s: member %u aborted the group (member %u: %s)", what, ab - 1, c->me, buf);
            }
            return fail(CKPT_EPEER, "%s: timed out after %.0f s waiting for peers (member %u: %s)", what, limit, c->me, buf);
        }
        if (el < 0.002) {  // the first 2 ms: poll without sleeping (small snapshots)
            std::this_thread::yield();
            continue;
        }
        std::this_thread::sleep_for(std::chrono::microseconds(el < 0.01 ? 20 : 200));
    }
}

int wait_done_all(ckpt_ctx *c, uint32_t done_seq) {
    int rc;
    if (c->done_enqueued) {  // see stage_finish
        c->done_enqueued = false;
        return sync_stream_timeout(c, c->sW, "wait");
    }
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

// Non-blocking completion test: *done = 1 once ckpt_wait(id) would return without waiting.
extern "C" int ckpt_test(ckpt_ctx *c, uint64_t id, int *done) {
    if (!c || !done) return fail(CKPT_EINVAL, "test: null");
    if (id == 0 || id >= c->next_id) return fail(CKPT_ESTATE, "test: unknown snapshot id %llu", (unsigned long long)id);
    *done = 0;
    if (id != c->pending_id) {
        *done = c->completed_id >= id ? 1 : 0;
        return CKPT_OK;
    }
    if (!c->issued) return CKPT_OK;
    int rc = set_dev(c);
    if (rc) return rc;
    if ((rc = issue_gated_more(c))) return rc;
    if (gated_pending(c)) return CKPT_OK;
    auto ready = [](cudaError_t e) { return e == cudaSuccess ? 1 : e == cudaErrorNotReady ? 0 : -1; };
    int r = 1;
    if (c->done_enqueued) {
        r = ready(cudaStreamQuery(c->sW));
    } else {
        cudaStream_t ss[4] = {c->sP, c->sX, c->sC, c->sG};
        for (auto x : ss)
            if (r == 1) r = ready(cudaStreamQuery(x));
        for (uint32_t j = 0; r == 1 && c->m >= 2 && c->transport == CKPT_GROUP_LOCAL && j < c->m; ++j)
            r = ready(cudaEventQuery(c->members[j]->ev_done));
    }
    if (r < 0) {
        cudaError_t e = cudaGetLastError();
        return fail(CKPT_ECUDA, "test: %s", cudaGetErrorString(e));
    }
    *done = r;
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
    if (gated_pending(c)) {  // HAS windows: keep topping up until every gated copy is enqueued
        double limit = 600.0;
        if (const char *e = getenv("CKPT_TIMEOUT_S")) limit = atof(e);
        const auto t0 = std::chrono::steady_clock::now();
        while (!rc && gated_pending(c)) {
            if ((rc = issue_gated_more(c))) break;
            if (!gated_pending(c)) break;
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
                rc = fail(CKPT_EPEER, "wait: window-gated copies made no progress in %.0f s (are the HAS windows "
                                      "ever opened?)", limit);
                break;
            }
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    }
    if (!rc) rc = wait_done_all(c, c->op_seq_base + (uint32_t)c->op_NB + 1);
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
    // every peer has protected (its DONE for this snapshot arrived), so every parity
    // handle is published: map them now, once, off the recovery path (a first
    // cudaIpcOpenMemHandle of a multi-GB buffer costs tens of ms).  A failure here is
    // left to the rebuild, which retries and reports it.
    if (c->transport == CKPT_GROUP_IPC && c->aec && c->m >= 2 && !c->parity_peers_mapped && !rebuild_self_encode(c)) {
        c->parity_peers_mapped = true;
        for (uint32_t j = 0; j < c->m; ++j)
            if (j != c->me && rebuild_map_parity(c, j, false)) cudaGetLastError();
    }
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
    if (from_dev && c->full_copy && !(c->opt.flags & CKPT_OPT_CE_PACK)) {
        // the whole completed image is in HBM: ONE unpack launch over [0, L) (no per-bucket
        // launches or tails; nothing waits on the copy stream)
        PackAllArgs a;
        memset(&a, 0, sizeof a);
        a.chunks = c->d_chunks;
        a.tile_first = c->d_tile_first;
        a.L = c->L;
        a.image = c->staging;
        a.bucket = align_up(std::max<uint64_t>(c->L, 1), kGroup);  // one "bucket": nothing to publish
        a.unpack = 1;
        TimedLaunch *t;
        if ((rc = timed_begin(c, c->sP, 2, &t))) return rc;
        CUDA_TRY(launch_pack_all(a, c->max_ctas, c->sP, !(c->opt.flags & CKPT_OPT_LSU_PACK)));
        if ((rc = timed_end(t, c->sP))) return rc;
        c->st.unpack_launches++;
    }
    for (uint64_t k = 0; k < c->op_NB && !(from_dev && c->full_copy && !(c->opt.flags & CKPT_OPT_CE_PACK)); ++k) {
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

