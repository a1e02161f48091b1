// ckpt_recovery.cu -- REFT-load step 3: AEC rebuild of a lost member, ARC restore, ckpt_recover, background host restore
#include "ckpt_internal.cuh"

using namespace reft;

// ------------------------------------------------------------------ rebuild ---------
// Per bucket b (slot s), lost member kl:
//   survivor j: C: [reuse: own kernel(b-n) done, REL(b-n) from all] H2D data+parity -> READY(b)
//               X: own H2D, READY(b) from all -> rebuild row j into kl's slot, then encode
//                  its share of kl's parity row into kl's parity slot -> REL(b)
//   lost kl   : X: [reuse: own D2H(b-n)] READY(b) ; READY(b) from all -> REL(b)
//               C: REL(b) from all, own encode -> D2H data + parity into its image
int rb_stage1(ckpt_ctx *c, uint64_t b, uint32_t kl) {
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

int rb_stage2(ckpt_ctx *c, uint64_t b, uint32_t kl) {
    const uint32_t s = slot_of(c, b);
    int rc;
    if (c->me != kl) CUDA_TRY(cudaStreamWaitEvent(c->sX, c->ev_h2d[s], 0));
    if ((rc = wait_all(c, c->sX, kReady, bucket_seq(c, b), s))) return rc;
    if (rebuild_self_encode(c))
        rc = c->me != kl ? do_rebuild_row(c, b, kl, c->sX) : do_encode(c, b, c->sX);
    else if (c->me != kl && !(rc = do_rebuild_row(c, b, kl, c->sX)))
        rc = do_encode_lost_share(c, b, kl, c->sX);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(c->ev_kdone[s], c->sX));
    return sig_signal(c, c->sX, kRel, bucket_seq(c, b), s);
}



int rb_stage3(ckpt_ctx *c, uint64_t b, uint32_t kl) {
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

int rb_finish(ckpt_ctx *c, uint32_t kl) {
    CUDA_TRY(cudaEventRecord(c->ev_pack_all, c->sX));
    CUDA_TRY(cudaStreamWaitEvent(c->sC, c->ev_pack_all, 0));
    CUDA_TRY(cudaEventRecord(c->ev_done, c->sC));
    if (c->me == kl && async_host_restore(c))  // DONE = device image complete, D2H continues
        return sig_signal(c, c->sX, kDone, c->op_seq_base + (uint32_t)c->op_NB + 1, 0);
    // DONE after every local stream finished
    return sig_signal(c, c->sC, kDone, c->op_seq_base + (uint32_t)c->op_NB + 1, 0);
}

// Wait for a background host restore (see async_host_restore) and publish it.
int host_sync(ckpt_ctx *c) {
    for (auto &t : c->host_bg)
        if (t.joinable()) t.join();
    c->host_bg.clear();
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

int rb_commit(ckpt_ctx *c, uint32_t kl, uint64_t version) {
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

extern "C" int ckpt_recover(ckpt_ctx *c, uint32_t lost_mask, void *stream);

extern "C" int ckpt_rebuild(ckpt_ctx *c, int32_t lost, void *stream) {
    if (!c) return fail(CKPT_EINVAL, "rebuild: null");
    // ARC schemes also re-create the ARC copy the lost member held: the general path
    if (c->grouped && c->arc && lost >= 0 && (uint32_t)lost < c->m) return ckpt_recover(c, 1u << lost, stream);
    return rebuild_aec(c, lost, stream);
}

int rebuild_aec(ckpt_ctx *c, int32_t lost, void *stream) {
    NvtxRange nvtx_("ckpt_rebuild");
    if (!c) return fail(CKPT_EINVAL, "rebuild: null");
    if (!c->registered || !c->grouped) return fail(CKPT_ESTATE, "rebuild: not protected");
    if (c->m < 2) return fail(CKPT_EUNRECOVERABLE, "rebuild: a group of one has no redundancy (P.460)");
    if (lost < 0 || (uint32_t)lost >= c->m) return fail(CKPT_EINVAL, "rebuild: lost rank %d out of range", lost);
    // a survivor that serves the rebuild from its device image touches no host buffer: a
    // background host restore (e.g. of an ARC restore just before, in ckpt_recover) may
    // keep running; the lost member and host-path survivors wait for it
    if ((c->me == (uint32_t)lost || !device_image_valid(c)) && host_sync(c)) return CKPT_ECUDA;
    if (!c->aec) return fail(CKPT_EUNRECOVERABLE, "rebuild: the scheme has no parity");
    int rc = check_sticky(c);
    if (rc) return rc;
    if (c->pending_id || c->requested) return fail(CKPT_ESTATE, "rebuild: a snapshot is in flight");
    const uint32_t kl = (uint32_t)lost;
    if (c->me != kl && c->completed < 0) {
        rc = fail(CKPT_EUNRECOVERABLE, "rebuild: survivor %u has no completed image (more than one loss)", c->me);
        group_abort(c);  // the other members would wait for this survivor's share forever
        return rc;
    }
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
            if ((rc = set_dev(o)) || (!rebuild_self_encode(o) && (rc = rebuild_map_parity(o, kl))) || (rc = prepare_op(o, B))) goto bad;
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
    if ((!rebuild_self_encode(c) && (rc = rebuild_map_parity(c, kl))) || (rc = prepare_op(c, B))) {
        make_sticky(c, rc);  // aborts the group: the peers fail fast instead of timing out
        return rc;
    }
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


int recover_plan(const ckpt_ctx *c, uint32_t mask, int32_t *remaining) {
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

// With full-copy staging and the device path allowed, the lost member's DEVICE image comes
// first: H2D of the holder's copy into the staging and parity buffer (PCIe-bound -- the
// floor for a member whose device memory is gone), after which ckpt_load unpacks from HBM;
// its own host image is re-written from the holder's file by host threads in the
// background (host_sync joins them before anything reads or overwrites the host image).
static bool arc_device_first(const ckpt_ctx *c) {
    return c->full_copy && !device_only(c) && !(c->opt.flags & CKPT_OPT_HOST_LOAD);
}

int recover_step1(ckpt_ctx *c, uint32_t mask, uint64_t version) {
    if (!(mask & (1u << c->me)) || !c->arc || (mask & (1u << holder_of(c, c->me)))) return CKPT_OK;
    int rc = ensure_holder_mapped(c);
    if (rc) return rc;
    if ((rc = host_sync(c))) return rc;
    const int idx = rb_target(c);
    const uint64_t P = parity_bytes_of(c);
    const uint8_t *src_d = c->shm_hold[idx].p + c->Lstar + P, *src_p = c->shm_hold[idx].p + 2 * c->Lstar + P;
    auto host_copy = [c, idx, src_d, src_p, P] {
        // only [0, L) carries data; the zero pad is written here, never copied (a peer's pad
        // may still hold ckpt_forget poison while it is being cleaned)
        parallel_memcpy(c->hdata[idx].p, src_d, c->L);
        if (c->Lstar > c->L) memset(c->hdata[idx].p + c->L, 0, c->Lstar - c->L);
        if (c->aec) parallel_memcpy(c->hpar[idx].p, src_p, P);
    };
    if (arc_device_first(c)) {
        if ((rc = set_dev(c))) return rc;
        // (full-copy staging holds [0, L) only: peers read the pad [L, L*) as zero, Q5)
        CUDA_TRY(cudaMemcpyAsync(c->staging, src_d, c->L, cudaMemcpyHostToDevice, c->sC));
        if (c->aec && P) CUDA_TRY(cudaMemcpyAsync(c->parity, src_p, P, cudaMemcpyHostToDevice, c->sC));
        if ((rc = sync_stream_timeout(c, c->sC, "arc restore"))) return rc;
        c->st.h2d_bytes += c->L + (c->aec ? P : 0);
        c->st.ce_copies += (c->aec && P) ? 2 : 1;
        c->staging_poisoned = false;
        c->host_bg.emplace_back(host_copy);
        c->pad_dirty[idx] = false;
        c->completed = idx;
        c->completed_id = version;
        c->staging_id = version;
        c->host_pending = true;  // meta is published by host_sync
        return CKPT_OK;
    }
    host_copy();
    c->pad_dirty[idx] = false;
    c->completed = idx;
    c->completed_id = version;
    meta_commit(c);
    return CKPT_OK;
}

int recover_step3(ckpt_ctx *c, uint32_t mask) {
    if (!(mask & (1u << c->me)) || !c->arc) return CKPT_OK;
    int rc = ensure_next_mapped(c);
    if (rc) return rc;
    const int idx = c->completed;
    if (idx < 0) return fail(CKPT_ESTATE, "recover: member %u has no completed image after restore", c->me);
    const uint64_t P = parity_bytes_of(c);
    const uint64_t Ln = c->peer_L[(c->me + 1) % c->m];
    auto host_copy = [c, idx, P, Ln] {
        parallel_memcpy(c->harc[idx], c->shm_next[idx].p, Ln);  // member me+1's data ...
        if (c->Lstar > Ln) memset(c->harc[idx] + Ln, 0, c->Lstar - Ln);  // ... and a clean pad
        if (c->aec) parallel_memcpy(c->harcp[idx], c->shm_next[idx].p + c->Lstar, P);
    };
    c->arc_dirty[idx] = false;
    if (arc_device_first(c)) {  // host-only work: in the background as well
        c->host_bg.emplace_back(host_copy);
        return CKPT_OK;
    }
    host_copy();
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

