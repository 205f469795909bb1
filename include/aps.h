/*
 * aps.h -- C ABI of libaps, a B200-native (sm_100a) implementation of the
 * data-parallel hot path of Auto-Precision Scaling (APS, arXiv 1911.08907):
 * layer-wise low-precision gradient synchronisation.
 *
 * Paper citations ("P:n") are lines of the paper's LaTeX source with the
 * algorithm / equation / table they fall in.  Readings of ambiguous passages
 * ("A<k>") are listed in DESIGN.md.
 *
 * The method (Alg. 1 `alg:APS_grad`), per layer g of the gradient
 * list, with customised float (exp_bit, man_bit) and N ranks:
 *   upper_bound_exp <- 2^(exp_bit-1) - 1
 *   max_grad_exp    <- FindMaxExp(g * N)
 *   f~              <- upper_bound_exp - AllReduce(max_grad_exp, MAX)   (Eq. 4)
 *   g               <- g * 2^f~
 *   low_g           <- Cast(g, exp_bit, man_bit)  round-to-nearest-even
 *   low_g           <- AllReduce(low_g, SUM)  ring, re-quantised after
 *                      every add as CPD's low-precision accumulator
 *   g               <- Cast(low_g, 8, 23) / 2^f~, then / N
 *
 * Calls map to the method as:
 *   aps_layer_scales   -> FindMaxExp on every layer + AllReduce(E, MAX)
 *   aps_quantize_pack  -> f~, scale, Cast, pack into sub-32-bit codes
 *   aps_allreduce      -> the ring reduce-scatter (re-quantise after each add)
 *                         and all-gather of the packed codes
 *   aps_unscale        -> Cast back, unscale, average
 *   aps_sync           -> the four in order
 * Transports for the all-reduce (N > 1): an NCCL ring (nccl_comm) or peer
 * memory (aps_peer_export / aps_peer_import: owner-computes reduce over
 * NVLink load/store).  Variants: per-layer formats
 * (aps_init_mixed), reduction order and accumulator (aps_set_reduction),
 * stochastic rounding (aps_set_rounding); analysis: aps_census,
 * aps_round_off_error; CUDA-graph capture: aps_set_graph_safe.
 *
 * CONVENTIONS
 *  - Memory: every tensor pointer is a DEVICE pointer unless the name says
 *    host.  The library never allocates device memory: gradients, outputs and
 *    the workspace belong to the caller (e.g. torch).  NCCL communicators and
 *    CUDA streams are borrowed and must outlive the context.
 *  - Ordering: every call is enqueued on the context's stream and returns
 *    before the GPU work finishes, unless marked [sync].
 *  - Errors: every call returns an aps_status and never throws or aborts
 *    across the ABI; aps_last_error() gives a message.  CUDA and NCCL errors
 *    are captured as APS_ERR_CUDA / APS_ERR_NCCL.  Non-finite gradients are a
 *    deferred error: the device raises a flag, outputs are unspecified, and
 *    aps_status_sync() returns APS_ERR_NONFINITE (reading A4).
 *  - Formats: 2 <= exp_bits <= 8, 0 <= man_bits <= 23, 1+exp_bits+man_bits
 *    <= 32 (CPD: "number of exponent bits <= 8 and number of mantissa bits
 *    <= 23").  exp_bits = 1 (bias 0, no normal numbers) is rejected.
 *  - Layers: numels[l] >= 1 (int64; up to 2^31 tiles), layer buffers 16-byte
 *    aligned (APS_ERR_ALIGN otherwise).  Any numel is legal; tails are masked.
 *
 * PACKED LAYOUT (design rule, not in the paper):
 *  - b = 1 + exp_bits + man_bits bits per code; code = s | E | M, sign MSB,
 *    IEEE-style, all-ones exponent reserved for Inf/NaN (Table
 *    `precision_range`).
 *  - tile = 128 codes = 16*b bytes.  Layer l occupies ceil(n_l/128) tiles
 *    from tile offset sum_{k<l} ceil(n_k/128); padding codes are +0.  The
 *    tile count is padded to T' = p * ceil(T/p); chunk c (c = 0..p-1) is
 *    tiles [c T'/p, (c+1) T'/p).
 *  - code i of the buffer occupies bits [i*b, (i+1)*b), LSB-first, in a
 *    little-endian byte stream (b = 8: a plain uint8 array).
 *  - Ring order (reading A14): chunk c is accumulated in rank order
 *    c+1, c+2, ..., c (the owner adds last), every add re-quantised; after
 *    the all-gather every rank holds identical codes.
 */
#ifndef APS_H_
#define APS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct aps_ctx aps_ctx;

typedef enum {
    APS_OK = 0,
    APS_ERR_ARG = 1,        /* bad argument (NULL, size, rank, n_layers...) */
    APS_ERR_FORMAT = 2,     /* (exp_bits, man_bits) outside the valid set */
    APS_ERR_ALIGN = 3,      /* a layer / workspace pointer is misaligned */
    APS_ERR_CUDA = 4,       /* a CUDA runtime error (launch, copy) */
    APS_ERR_NCCL = 5,       /* an NCCL error */
    APS_ERR_NONFINITE = 6,  /* a gradient held Inf/NaN (deferred; see aps_status_sync) */
    APS_ERR_STATE = 7       /* call out of order, or no workspace set */
} aps_status;

/* Create a context.
 *   exp_bits, man_bits : the customised float (Alg. 1 inputs exp_bit, man_bit)
 *   world_size, rank   : N (Alg. 1 input) and this process's rank
 *   n_layers, numels   : host array [n_layers] of gradient element counts, in
 *                        the caller's layer order (the packed layout order)
 *   nccl_comm          : ncclComm_t (borrowed) of world_size ranks, or NULL.
 *                        NULL with world_size == 1: single GPU.  NULL with
 *                        world_size > 1: a SIMULATED rank (test mode): the
 *                        collectives must then go through aps_sim_*.
 *   cuda_stream        : cudaStream_t (borrowed); NULL = legacy default stream
 * Does not touch the device. */
aps_status aps_init(aps_ctx **out, int exp_bits, int man_bits, int world_size, int rank,
                    int n_layers, const int64_t *numels, void *nccl_comm, void *cuda_stream);

/* As aps_init with a format PER LAYER (hybrid precision):
 * layer l uses (exp_bits[l], man_bits[l]) -- the paper's per-layer precision
 * choice ("the last layer's gradients ... in higher precision",
 * Table last_layer_precision).  f~_l uses layer l's upper_bound_exp.
 * Packed layout: layer l's tiles are 16*b_l bytes each, in layer order; the
 * padding tiles up to T' continue the LAST layer's format (reading A22).  Ring
 * chunk c is still tiles [c T'/p, (c+1) T'/p); its byte size then differs per
 * chunk, its reduction runs per format run, and the all-gather forwards the
 * chunks around the ring (send/recv) instead of ncclAllGather.  Arrays are
 * host [n_layers]; everything else as aps_init.  Equal formats everywhere
 * behave exactly like aps_init. */
aps_status aps_init_mixed(aps_ctx **out, const int *exp_bits, const int *man_bits, int world_size, int rank,
                          int n_layers, const int64_t *numels, void *nccl_comm, void *cuda_stream);

/* Bytes of device workspace the context needs (packed buffer, one ring
 * receive chunk, layer and work tables, exponent vectors). */
size_t aps_workspace_bytes(const aps_ctx *ctx);

/* Attach caller-owned device workspace (>= aps_workspace_bytes, 256-byte
 * aligned).  Zero-fills it and uploads the layer tables (enqueued). */
aps_status aps_set_workspace(aps_ctx *ctx, void *dev, size_t bytes);

/* FindMaxExp(g * N) for every layer (Alg. 1 line 3): the local
 * exponent E_l = ceil(log2(N * max_i |g_l[i]|)) (exact, readings A2/A5;
 * INT32_MIN for an all-zero layer, A3; INT32_MAX if any element is non-finite,
 * A4), one fused multi-tensor kernel; then AllReduce(E, MAX) over the
 * communicator (int32 per layer, reading A6).
 *   grads : host array [n_layers] of device fp32 pointers (16-byte aligned). */
aps_status aps_layer_scales(aps_ctx *ctx, const float *const *grads);

/* f~_l = upper_bound_exp - E_l (0 for an all-zero layer), y = g * 2^f~ (one
 * binary32 rounding, reading A8), Cast(y, exp_bits, man_bits) with
 * round-to-nearest-even, gradual underflow (A10) and IEEE overflow
 * (A11), packed into the workspace's packed buffer (layout above).
 * Requires aps_layer_scales first. */
aps_status aps_quantize_pack(aps_ctx *ctx, const float *const *grads);

/* AllReduce(low_g, SUM) (Alg. 1 line 7) as a ring: p-1 reduce-scatter
 * steps over ncclSend/ncclRecv of packed bytes, each followed by the
 * unpack-add-requantise-repack kernel s <- Cast(fl32(dec(recv) + dec(own)))
 * (reading A13), then an all-gather of the packed chunks.  No-op
 * for world_size == 1.  Requires aps_quantize_pack first. */
aps_status aps_allreduce(aps_ctx *ctx);

/* out_l = fl32( fl32(dec(s) * 2^-f~_l) / N )  (Alg. 1 lines 8-9, P:254-256;
 * average = 0 skips the division, reading A16).
 *   out : host array [n_layers] of device fp32 pointers; may alias grads. */
aps_status aps_unscale(aps_ctx *ctx, float *const *out, int average);

/* aps_layer_scales, aps_quantize_pack, aps_allreduce, aps_unscale in order,
 * in place on grads.  With world_size == 1 (no NCCL communicator, nearest-even
 * rounding) the four run as ONE fused launch per format group -- two formats
 * share one launch -- (no collective separates FindMaxExp from Cast): a
 * warp-specialised wavefront over the work items that needs no co-residency
 * and no per-call host state (capture-safe). */
aps_status aps_sync(aps_ctx *ctx, float *const *grads, int average);

/* As aps_sync, reading grads and writing the result to out (out may alias
 * grads; out[l] 16-byte aligned, numels[l] fp32). */
aps_status aps_sync_out(aps_ctx *ctx, const float *const *grads, float *const *out, int average);

/* End-to-end entry with HOST buffers: copies host_in[l] (pinned host fp32)
 * into dev_grads[l], runs aps_sync in place, copies the result to host_out[l]
 * (pinned host fp32, may equal host_in).  All enqueued on the stream. */
aps_status aps_sync_host(aps_ctx *ctx, const float *const *host_in, float *const *dev_grads,
                         float *const *host_out, int average);

/* Select the hardware cvt.rn.satfinite.{e5m2,e4m3}x2 converters for (5,2) /
 * (4,3) (default on where available; bit-identical to the generic path on
 * the APS path, reading A12 -- the -m gpu tests check it) or the generic
 * bit-arithmetic codec (enable = 0).  Environment APS_HW_CVT=0 sets the
 * default off. */
aps_status aps_set_hw_convert(aps_ctx *ctx, int enable);

/* [sync] Wait for the stream; return APS_ERR_NONFINITE (and clear the flag)
 * if a non-finite gradient was seen since the last call, else APS_OK. */
aps_status aps_status_sync(aps_ctx *ctx);

/* [sync] Copy the scale exponents f~[n_layers] of the last quantize to host. */
aps_status aps_get_scales(aps_ctx *ctx, int32_t *host_out);

/* Device pointer and size of the packed buffer (valid after set_workspace). */
aps_status aps_get_packed(aps_ctx *ctx, const void **dev, size_t *bytes);

/* Layout queries (host only, no device): tiles T' and packed bytes 16*b*T'. */
aps_status aps_layout(int world_size, int exp_bits, int man_bits, int n_layers,
                      const int64_t *numels, int64_t *total_tiles, int64_t *packed_bytes);

/* aps_layout for per-layer formats (host only): T' and the packed bytes
 * sum_l 16 b_l T_l + (T' - T) 16 b_last (aps_init_mixed's layout). */
aps_status aps_layout_mixed(int world_size, int n_layers, const int64_t *numels, const int *exp_bits,
                            const int *man_bits, int64_t *total_tiles, int64_t *packed_bytes);

/* Ring schedule (host only): at reduce-scatter step `step` (0..p-2) rank
 * `rank` sends chunk (rank-1-step) mod p to rank+1 and receives chunk
 * (rank-2-step) mod p from rank-1, which it reduces into its own copy. */
aps_status aps_ring_step(int world_size, int rank, int step, int *send_chunk, int *recv_chunk);

/* ---- reduction order and accumulator ------
 * group_k: hierarchical all-reduce with groups of group_k consecutive ranks
 *   (intra-group reduce to a master, ring all-reduce across the
 *   masters, broadcast; the paper's round-off argument P:531-541).  Reading
 *   A23: tile t is accumulated over the members of each group in ring order
 *   c1+1, ..., c1 of its group chunk c1 = t / (T'/group_k), then over the
 *   p/group_k group sums in ring order c2+1, ..., c2 of its master chunk
 *   c2 = t / (T' group_k / p).  group_k = 1 or world_size: the flat ring (A14).
 *   Must divide world_size.
 * acc_exp_bits, acc_man_bits: accumulator format (CPD: "use a
 *   higher precision to store the accumulator"; reading A24): the running sum
 *   is re-quantised to it after every fp32 add and cast to the wire format
 *   once at the end.  Must hold every wire value (>= the wire's exp and man
 *   bits); equal to the wire format by default.
 * kahan: Kahan-compensated accumulation (reading A24): y = x - c,
 *   t = s + y, c = (t - s) - y, s = t, every result re-quantised.
 * Anything but the default (flat ring, wire accumulator, no compensation)
 * needs the peer transport (aps_peer_import / aps_sim_connect): the NCCL ring
 * moves partial sums in the wire format.  Accumulator variants need one
 * format for every layer (aps_init).  Errors: APS_ERR_ARG, APS_ERR_FORMAT. */
aps_status aps_set_reduction(aps_ctx *ctx, int group_k, int acc_exp_bits, int acc_man_bits, int kahan);

/* CUDA-graph capture.  Every path takes its per-call state from device memory
 * (self-resetting claim and completion counters, device-resident peer epochs and
 * stochastic-rounding call counter), so any aps_sync / aps_sync_out can be captured
 * and replayed as is.  Kept for source compatibility: records the flag, switches
 * nothing.  Errors: APS_ERR_STATE (no workspace). */
aps_status aps_set_graph_safe(aps_ctx *ctx, int enable);

/* Occupancy cap of the fused one-rank launch (aps_sync / aps_sync_out at
 * world_size 1): at most ctas_per_sm CTAs per SM (0 = as many as fit, the
 * default).  A cap leaves registers and warps of every SM to concurrent work on
 * other streams -- the backward kernels that the DDP hook's syncs overlap
 * (P:637-640); the sync itself then takes longer.  Errors: APS_ERR_ARG
 * (ctas_per_sm < 0). */
aps_status aps_set_occupancy(aps_ctx *ctx, int ctas_per_sm);

/* Rounding mode of every Cast ("some researchers
 * prefer stochastic rounding ... an unbiased estimate"; the paper's own runs use
 * round-to-nearest-even, the default).  mode 0: nearest even; mode 1: stochastic
 * (reading A26): x between its neighbours lo <= |x| < hi rounds up iff
 * r < (|x| - lo)/(hi - lo) * 2^32, r = SplitMix64(seed, phase << 40 | i) >> 32 with i the
 * element's code index in the packed layout and phase = the rank for the initial
 * Cast, p - 1 + a for the a-th add of the element's fold -- reproducible and
 * independent of thread order.  Stochastic mode needs one format, the wire-format
 * accumulator, and (world_size > 1) the peer transport; at world_size 1 aps_sync
 * runs the separate calls instead of the fused kernel.  Errors: APS_ERR_ARG. */
aps_status aps_set_rounding(aps_ctx *ctx, int mode, uint64_t seed);

/* ---- peer-memory transport (NVLink / NVSwitch load-store) ----------------
 * Alg. 1 line 7's all-reduce without NCCL: rank r loads the p ranks' packed
 * codes of ring chunk r straight from their workspaces (CUDA IPC mappings),
 * folds them in the reduction order above, and stores the reduced codes into
 * every rank's packed buffer (the all-gather, fused).  NVLink bytes per rank
 * equal the ring's.  The exponent MAX (Alg. 1 line 4) goes through peer
 * memory too.  Cross-rank ordering uses monotone epoch flags (system-scope
 * release/acquire); every cross-rank device wait gives up after
 * APS_PEER_TIMEOUT_S seconds (environment, default 120; APS_ERR_STATE from
 * aps_status_sync).  Bit-identical to the NCCL ring for the flat order.
 * Protocol: every rank calls aps_peer_export [sync] after aps_set_workspace,
 * the host gathers the world_size (handle, offset) pairs (e.g. over
 * torch.distributed), then every rank calls aps_peer_import.  All ranks must
 * then issue the same sequence of syncs.
 *   host_handle : APS_PEER_HANDLE_BYTES bytes (a cudaIpcMemHandle_t of the
 *                 allocation holding the workspace)
 *   host_offset : the workspace's byte offset in that allocation
 *   host_handles: [world_size * APS_PEER_HANDLE_BYTES], rank-major; host_offsets: [world_size]
 * A context created with nccl_comm = NULL and world_size > 1 becomes a real
 * rank of the peer transport here (no NCCL needed at all).
 * aps_destroy unmaps the peers (every rank must have finished its last sync). */
#define APS_PEER_HANDLE_BYTES 64
aps_status aps_peer_export(aps_ctx *ctx, void *host_handle, uint64_t *host_offset);
aps_status aps_peer_import(aps_ctx *ctx, const void *host_handles, const uint64_t *host_offsets);

/* [sync] Underflow / overflow census (the loss-scaling
 * comparison of section 3.1 P:173-179 and Fig. `aps_comparing` P:277-280:
 * "it will cause some small values to underflow, which will be cast to 0").
 * For every layer l, counts the nonzero finite elements g of grads[l] whose
 * Cast(g * 2^s_l) (this context's format, IEEE overflow) is +-0 (underflow,
 * host_counts[2 l]) or +-Inf (overflow, host_counts[2 l + 1]).
 *   host_scale_exp: [n_layers] s_l -- APS: aps_get_scales' f~; constant loss
 *   scaling: the same exponent for every layer; no scaling: 0.
 * Needs one format for every layer. */
aps_status aps_census(aps_ctx *ctx, const float *const *grads, const int32_t *host_scale_exp, uint64_t *host_counts);

/* Eq. (5) `equation:round_off_error`, reading A25: adds
 * sum over i with h[i] != 0 of |(h[i] - l[i]) / h[i]| (binary64) to *dev_sum and
 * the number of such i to *dev_count (device scalars the caller zeroes);
 * the average round-off error is sum / count.  h, l: device fp32 [n].
 * The binary64 sum is accumulated in a device-dependent order. */
aps_status aps_round_off_error(const float *h, const float *l, int64_t n, double *dev_sum,
                               unsigned long long *dev_count, void *cuda_stream);

const char *aps_last_error(const aps_ctx *ctx);
aps_status aps_destroy(aps_ctx *ctx);
const char *aps_version(void);

/* ---- NCCL plumbing (so callers need no NCCL binding) ---------------- */
/* Write a fresh ncclUniqueId (128 bytes) to host_uid. */
aps_status aps_nccl_unique_id(void *host_uid, size_t bytes);
/* ncclCommInitRank; *comm_out receives an ncclComm_t owned by the caller. */
aps_status aps_nccl_comm_init(void **comm_out, const void *host_uid, int world_size, int rank);
aps_status aps_nccl_comm_destroy(void *comm);

/* ---- test mode: p simulated ranks on one device --------------------- */
/* ctxs[p] created with nccl_comm == NULL and world_size == p, ranks 0..p-1,
 * sharing one stream.  grads: host array [p * n_layers], rank-major.
 * aps_sim_layer_scales = every rank's aps_layer_scales + the MAX exchange;
 * aps_sim_allreduce = the same ring schedule and reduce kernel as
 * aps_allreduce with device-to-device copies in place of send/recv. */
aps_status aps_sim_layer_scales(aps_ctx *const *ctxs, int p, const float *const *grads);
aps_status aps_sim_allreduce(aps_ctx *const *ctxs, int p);
/* Connect p simulated ranks through the peer transport (each context's
 * "peer" pointers are the other contexts' workspaces on the same device);
 * aps_sim_layer_scales / aps_sim_allreduce then run the peer kernels. */
aps_status aps_sim_connect(aps_ctx *const *ctxs, int p);

/* ---- test only: the device cast on arbitrary inputs ------------------ */
/* codes[i] = Cast(in[i]) (uint32 per code, unpacked); exercises Inf/NaN and
 * overflow, which APS never reaches.  hw = 1 selects the hardware
 * cvt.rn.satfinite.{e5m2,e4m3}x2 path used for (5,2)/(4,3) on the APS path
 * (exact only for |x| < (2 - 2^-(m+1)) * 2^bias, reading A12). */
aps_status aps_debug_cast(const float *in, uint32_t *codes, int64_t n, int exp_bits,
                          int man_bits, int hw, void *cuda_stream);
aps_status aps_debug_decode(const uint32_t *codes, float *out, int64_t n, int exp_bits,
                            int man_bits, int hw, void *cuda_stream);
/* codes[i] = stochastic-rounding Cast(in[i]) with r_i = SplitMix64(seed, phase << 40 | i) >> 32
 * (reading A26; aps_set_rounding). */
aps_status aps_debug_cast_sr(const float *in, uint32_t *codes, int64_t n, int exp_bits, int man_bits,
                             uint64_t seed, uint64_t phase, void *cuda_stream);
/* Reduce step on its own: own[i] <- Cast(fl32(dec(recv[i]) + dec(own[i]))),
 * over n_tiles tiles of packed codes. */
aps_status aps_debug_ring_reduce(uint8_t *own, const uint8_t *recv, int64_t n_tiles,
                                 int exp_bits, int man_bits, int hw, void *cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* APS_H_ */
