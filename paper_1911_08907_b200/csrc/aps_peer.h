// aps_peer.h -- peer-memory transport (aps_peer.cu): host-side launchers and the
// kernel argument block.  No device code.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace aps {

constexpr int kMaxPeers = 64;  // ranks reachable by load/store (8 on one NVSwitch box; 64 simulated)

// flag block of a rank's workspace: uint32 [kFlagWords], monotone epochs written by the peers
constexpr int kSlotE = 0;                   // [q]: rank q posted its E vector for epoch
constexpr int kSlotReady = kMaxPeers;       // [q]: rank q's packed codes of epoch are complete
constexpr int kSlotDone = 2 * kMaxPeers;    // [q]: rank q stored its reduced chunk into every rank
constexpr int kMineE = 3 * kMaxPeers;       // this rank's own E-exchange epoch (device-resident)
constexpr int kMineR = 3 * kMaxPeers + 1;   // this rank's own all-reduce epoch (device-resident)
constexpr int kFlagWords = 3 * kMaxPeers + 2;
// Epochs live on the device (incremented by post_E and by the ready signal), so a
// captured CUDA graph of a sync replays correctly.

struct PeerArgs {
    uint64_t timeout_ns;          // bound of a cross-rank wait (APS_PEER_TIMEOUT_S, default 120 s)
    uint8_t *packed[kMaxPeers];   // every rank's packed buffer (own included), mapped into this process
    uint32_t *flags[kMaxPeers];   // every rank's flag block
    int32_t *eslots[kMaxPeers];   // every rank's E slots: int32 [2][kMaxPeers][n_layers]
    int64_t tiles;                // T'
    int p, rank, group_k;         // world, this rank, hierarchical group size (1 = flat ring)
};

cudaError_t launch_peer_post_E(const PeerArgs &a, const int32_t *E_local, int n_layers, cudaStream_t s);
cudaError_t launch_peer_collect_E(const PeerArgs &a, int32_t *E_glob, int n_layers, uint32_t *err_flag,
                                  cudaStream_t s);
// raise flag `slot` at every rank with this rank's all-reduce epoch (incremented first if `next`)
cudaError_t launch_peer_signal(const PeerArgs &a, int slot, bool next, cudaStream_t s);
cudaError_t launch_peer_wait(const PeerArgs &a, int slot, uint32_t *err_flag, cudaStream_t s);
// real ranks (all running concurrently): signal + wait, and post + collect, as one launch each
cudaError_t launch_peer_signal_wait(const PeerArgs &a, int slot, bool next, uint32_t *err_flag, cudaStream_t s);
cudaError_t launch_peer_exchange_E(const PeerArgs &a, const int32_t *E_local, int32_t *E_glob, int n_layers,
                                   uint32_t *err_flag, cudaStream_t s);
// reduce n_tiles tiles of one format starting at tile0 / byte_off of the packed buffers
cudaError_t launch_peer_reduce(const PeerArgs &a, int64_t byte_off, int64_t tile0, int64_t n_tiles, int e, int m,
                               bool hw, int acc_e, int acc_m, bool kahan, cudaStream_t s);
struct DevTables;
// stochastic rounding (reading A26): quantise of rank `rank`, and the owner-computes reduce
cudaError_t launch_debug_cast_sr(const float *in, uint32_t *codes, int64_t n, int e, int m, uint64_t seed,
                                 uint64_t phase, cudaStream_t s);
cudaError_t launch_quant_pack_sr(const DevTables &t, int e, int m, uint64_t seed, int rank, cudaStream_t s);
// advance the stochastic-rounding call counter (one sync done; reading A27)
cudaError_t launch_sr_advance(uint32_t *call, cudaStream_t s);
cudaError_t launch_peer_reduce_sr(const PeerArgs &a, int64_t byte_off, int64_t tile0, int64_t n_tiles, int e, int m,
                                  uint64_t seed, const uint32_t *call, cudaStream_t s);
cudaError_t launch_census(const DevTables &t, const int32_t *sexp, unsigned long long *counts, int e, int m,
                          cudaStream_t s);
cudaError_t launch_round_off(const float *h, const float *l, int64_t n, double *sum, unsigned long long *cnt,
                             cudaStream_t s);

}  // namespace aps
