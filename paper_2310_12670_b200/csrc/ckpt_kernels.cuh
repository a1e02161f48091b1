// ckpt_kernels.cuh -- device-side data structures and launchers of libreft_ckpt.
// Product code (the CUDA path); shares nothing with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace reft {

constexpr int kMaxTerms = 8;

// One contiguous piece of the packed image: bytes [dst, dst + nbytes) of the image
// come from device address src (src == 0: zero fill -- alignment gaps, reading Q6).
// Built once by the planner at ckpt_register; sorted by dst.
struct PackChunk {
    uint64_t src;
    uint64_t dst;
    uint64_t nbytes;
    uint64_t seg;
};

// Image tiles: the planner cuts every chunk (data and zero) at multiples of kTile
// bytes of image, so the chunks of tile i are exactly [tile_first[i], tile_first[i+1]).
// A launch splits the bucket's tiles evenly over its CTAs (balanced by bytes).
constexpr uint64_t kTile = 16 * 1024;

// Pack (tensors -> slot) or unpack (slot -> tensors) of the bucket's image range
// [bucket_begin, bucket_end) (clipped to the rank's L).  The slot holds image byte
// bucket_begin at address slot.
struct PackArgs {
    const PackChunk *chunks;
    const uint32_t *tile_first;
    uint64_t bucket_begin, bucket_end;
    uint8_t *slot;
    int unpack;
};

// One input stream of an XOR-gather: for stripe s and word i of a unit, the input
// byte address is base + s * stride + off + 16 * i; bytes at or beyond `valid`
// (relative to base) read as zero (zero pad of ranks shorter than L*, reading Q5).
struct XorTerm {
    const uint8_t *base;
    uint64_t valid;
    uint64_t stride;
    uint64_t off;
};


// out[s * out_stride + out_off + w] = XOR_t in_t[s * stride_t + off_t + w] for every
// stripe s < nstripes and byte w < unit (unit a multiple of 16).  Writes at or
// beyond out_valid are skipped.  Encode (Eq 1): terms = the m-1 peers' data slots,
// out = own parity slot.  Rebuild (Eq 2): terms = own parity + the m-2 other
// survivors, out = the lost rank's data slot (a P2P store over NVLink).
struct XorArgs {
    XorTerm in[kMaxTerms];
    int nin;
    uint8_t *out;
    uint64_t out_valid;
    uint64_t out_stride;
    uint64_t out_off;
    uint64_t nstripes;
    uint64_t unit;
};

// Whole-snapshot pack in ONE launch (full-copy staging): CTAs stride over 64 KiB
// groups of image tiles in order; the last CTA to finish a bucket publishes it: a
// release store of flag value seq_base+k+1 at index (value % maxb) of this rank's READY
// row, locally (the copy engine's D2H of bucket k waits on it with cuStreamWaitValue32)
// and in every peer's IPC-mapped flag page (their XOR of bucket k waits on it).  No
// kernel ever waits on another; only stream memory operations wait.
constexpr uint64_t kGroup = 4 * kTile;

struct PackAllArgs {
    const PackChunk *chunks;
    const uint32_t *tile_first;
    uint64_t L;            // image bytes to pack: [0, L)
    uint8_t *image;        // staging address of image byte 0
    uint64_t bucket;       // B, a multiple of kGroup
    uint32_t *counters;    // per bucket, zeroed before the launch
    uint32_t *ready_local; // this rank's READY row in its own flag page
    uint32_t *ready_peer[kMaxTerms];  // this rank's READY row in each peer's page
    int npeers;
    uint32_t seq_base;
    uint32_t maxb;
    int unpack;            // 1: the load direction (image -> tensors), nothing is published
};


// Push-mode XOR encode (CKPT_OPT_XOR_PUSH): member `me` sends every unit of its own image
// to the row it belongs to -- unit i of stripe s is term sigma(r, me) = i of row
// r = i + [i >= me] (Eq 1 P.474-477) -- as a bulk XOR reduction into row owner r's parity
// stream at P_r[s*u + w] (zeroed by its owner before its pack).  Only image bytes [0, L)
// are sent; the zero pad contributes nothing (Q5).  Reads are local HBM, writes are posted
// NVLink reductions (cp.reduce.async.bulk .xor.b64).
struct XorPushArgs {
    const uint8_t *src;
    uint64_t L;
    uint64_t unit;
    uint32_t m, me;
    uint8_t *dst[kMaxTerms + 1];  // parity stream of row owner r (unused for r = me)
};

// Fabric probe: bulk loads of n bytes from each of the npeers sources (peer staging over
// NVLink), interleaved over the peers in 16 KiB pieces, data discarded in SMEM.
struct ProbeArgs {
    const uint8_t *src[kMaxTerms];
    int npeers;
    uint64_t n;
};

// Launchers (return the cudaError_t of the launch).
cudaError_t launch_probe_pull(const ProbeArgs &a, int ctas, cudaStream_t s);
cudaError_t launch_xor_push(const XorPushArgs &a, int ctas, cudaStream_t s);
cudaError_t preload_kernels();
cudaError_t launch_pack_all(const PackAllArgs &a, int max_ctas, cudaStream_t s, bool tma);
cudaError_t launch_pack(const PackArgs &a, int max_ctas, cudaStream_t s, bool tma);
cudaError_t launch_xor(const XorArgs &a, int max_ctas, cudaStream_t s);

}  // namespace reft
