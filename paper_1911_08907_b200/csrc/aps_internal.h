// aps_internal.h -- declarations shared by aps_kernels.cu and aps_api.cpp
// (host-side launchers; no device code).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace aps {

constexpr int kTile = 128;        // codes per tile (layout rule, aps.h)
constexpr int kItemTiles = 64;    // tiles per work item (one CTA): 8192 elements
constexpr int kThreads = 256;

// One work item = a tile-aligned slice of one layer (<= kItemTiles tiles).
// Flat descriptor, precomputed on the host, so a kernel needs one load (no
// dependent item -> layer chain) to know everything but the per-call
// pointers.
struct Item {
    int32_t layer;
    int32_t tile_begin;   // within the layer
    int32_t n_tiles;
    int32_t cnt;          // valid elements: min(n_tiles * 128, numel - tile_begin * 128)
    int64_t tile_pos;     // first tile of the item in the packed buffer
    int32_t layer_items;  // work items of the layer
    int32_t fmt;          // format group of the layer (per-layer formats; 0 when uniform)
    int64_t byte_pos;     // byte offset of the item's first tile in the packed buffer
                          // (tiles are 16 * b bytes, b = the layer's code width)
};

struct LayerDev {
    int64_t numel;
    int64_t tile_off;    // first tile of the layer in the packed buffer
    int32_t n_items;
    int32_t pad0;
    int64_t pad1;
};

// Per-call gradient / output address of every work item (rebuilt on the
// device only when the caller's layer pointers change).
struct ItemPtr {
    const float *src;
    float *dst;
};

struct DevTables {
    const Item *items;
    const LayerDev *layers;
    const float *const *src;  // [n_layers] gradient pointers
    float *const *dst;        // [n_layers] output pointers
    uint32_t *amax;           // [n_layers] running abs-max bits (self-resetting)
    int32_t *E_local;         // [n_layers]
    int32_t *E_glob;          // [n_layers]
    int32_t *ftilde;          // [n_layers]
    uint32_t *flag;           // non-finite flag
    uint32_t *amax2;          // [2][n_layers] abs-max accumulators of the fused kernel (call parity)
    ItemPtr *iptr;            // [n_items] per-item addresses (fused LDG kernel)
    uint64_t *timeline;       // [kTimelineSlots] per-CTA phase stamps (flag 16)
    uint32_t *claim;          // [3 per format group] monotone work-claim counters (slot 2: the wavefront kernel)
    unsigned long long *claim64;  // wavefront claim counter (64-bit: the call index is derived on the device)
    uint32_t *ranges_done;    // self-resetting CTA-done counter of absmax_stream_kernel
    const int64_t *voff;      // [n_layers + 1] first vector (4 fp32) of each layer in a1's vector space
    const int32_t *cta_layer; // [absmax_grid()] layer holding the first vector of each a1 CTA's share
    uint32_t *layer_done;     // [n_layers] per-layer abs-max completion counters (fused kernel)
    uint32_t *bdone;          // [n_layers] per-layer quantise completion counters (fused kernel, self-resetting)
    uint32_t *sr_call;        // stochastic rounding: syncs since aps_set_rounding (per-call key, reading A27)
    uint8_t *packed;          // packed codes
    int n_items;
    int n_layers;
};

// a1: balanced abs-max stream over every layer (absmax_grid() CTAs; DevTables.voff /
// cta_layer describe the split), self-resetting done counter
constexpr int kAbsCtasPerSm = 4;
constexpr int kAbsMaxCtas = 1024;  // cta_layer table size (workspace)
int absmax_grid();
cudaError_t launch_absmax(const DevTables &t, int world, cudaStream_t s);
cudaError_t launch_quant_pack(const DevTables &t, int e, int m, bool hw, cudaStream_t s);
cudaError_t launch_unpack_unscale(const DevTables &t, int e, int m, bool hw, int world, int average,
                                  cudaStream_t s);
cudaError_t launch_ring_reduce(uint8_t *own, const uint8_t *recv, int64_t n_tiles, int e, int m,
                               bool hw, cudaStream_t s);
cudaError_t launch_sim_max(int32_t *const *E_glob, const int32_t *const *E_local, int p,
                           int n_layers, cudaStream_t s);
cudaError_t launch_debug_cast(const float *in, uint32_t *codes, int64_t n, int e, int m, bool hw,
                              cudaStream_t s);
cudaError_t launch_debug_decode(const uint32_t *codes, float *out, int64_t n, int e, int m,
                                bool hw, cudaStream_t s);

int sm_count();

constexpr int kFusedWarps = kThreads / 32;
#ifndef APS_FUSED_FLAGS
#define APS_FUSED_FLAGS 64  // 64: code / output stores with an L2 evict_first hint; +16: per-CTA timeline stamps
#endif
constexpr int kFusedDefaultFlags = APS_FUSED_FLAGS;  // fused kernel flags (compile time)
constexpr int kTimelineSlots = 4 * 2048;     // globaltimer stamps (4 per CTA) of the last fused launch
cudaError_t launch_build_item_ptrs(const DevTables &t, cudaStream_t s);
// wavefront variant (no grid barrier): claim_base advances by 2 * n_items + grid per call;
// call_no = wavefront calls before this one on these counters; lag = D positions.
#ifndef APS_WAVE_CTAS_PER_SM
#define APS_WAVE_CTAS_PER_SM 4
#endif
constexpr int kWaveCtasPerSm = APS_WAVE_CTAS_PER_SM;  // wavefront kernel occupancy (register budget)
int fused_p1_wave_grid(int e, int m, bool hw, int n_items);

#ifndef APS_WAVE_LAG_GRIDS
#define APS_WAVE_LAG_GRIDS 2
#endif
// lag D of the wavefront = (items of the largest layer) + kWaveLagGrids x grid positions
constexpr int kWaveLagGrids = APS_WAVE_LAG_GRIDS;
constexpr int kWaveOvershoot = 2;  // claims past the end per CTA and call (wavefront kernel claims 2 ahead)
// claim_base advances by 2 * n_items + kWaveOvershoot * grid per call.
// Per-call state of a wavefront launch.  graph = false: claim base (32-bit claim
// counter), call index and accumulator parity come from the host.  graph = true
// (capture-safe): all three are derived on the device from the 64-bit claim counter,
// which advances by exactly 2 * n_items + kWaveOvershoot * grid per call.
struct WaveCall {
    bool graph;
    uint32_t gen, claim_base, call_no;
};
cudaError_t launch_fused_p1_wave(const DevTables &t, int e, int m, bool hw, int average, const WaveCall &w, int lag,
                                 int grid, cudaStream_t s, bool cooperative = true);
// One wavefront launch over two format groups: items whose fmt == fmt2 use the
// binary32 codec (the hybrid FP32 classifier layer), the others (e, m, hw).
cudaError_t launch_fused_p1_wave_hybrid32(const DevTables &t, int e, int m, bool hw, int fmt2, int average,
                                          const WaveCall &w, int lag, int grid, cudaStream_t s);
// fused N = 1 sync, warp-specialised wavefront (aps_fused.cu): one cooperative launch per
// format group (hybrid FP32 classifier: one launch), self-resetting counters, no per-call host state
#ifndef APS_FUSED_CW
#define APS_FUSED_CW 1
#endif
#ifndef APS_CW_SLOTS
#define APS_CW_SLOTS 3
#endif
#ifndef APS_CW_CTAS_PER_SM
#define APS_CW_CTAS_PER_SM 3
#endif
constexpr int kCwCtasPerSm = APS_CW_CTAS_PER_SM;
cudaError_t launch_fused_cw(const DevTables &t, int e, int m, bool hw, int average, int max_layer_items, cudaStream_t s);
cudaError_t launch_fused_cw_hybrid32(const DevTables &t, int e, int m, bool hw, int fmt2, int average,
                                     int max_layer_items, cudaStream_t s);
// true when (e,m) has a hardware converter that is exact on the APS path
// formats with a hardware / exact fast codec: fp8 e5m2, e4m3 (APS regime only,
// reading A12), binary16, bfloat16, binary32 (every non-NaN input)
inline bool hw_available(int e, int m)
{
    return (e == 5 && m == 2) || (e == 4 && m == 3) || (e == 5 && m == 10) || (e == 8 && m == 7) ||
           (e == 8 && m == 23);
}

}  // namespace aps
