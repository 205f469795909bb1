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
    int32_t *E_local;         // [n_layers]
    int32_t *E_glob;          // [n_layers]
    int32_t *ftilde;          // [n_layers]
    uint32_t *flag;           // non-finite flag
    uint32_t *amax2;          // [2][n_layers] abs-max accumulators of the fused kernel (call parity)
    ItemPtr *iptr;            // [n_items] per-item addresses (fused LDG kernel)
    unsigned long long *claim64;  // claim counter of the control-warp kernel (per format group; self-resetting)
    uint32_t *ranges_done;    // self-resetting CTA-done counter of the a1-only launch
    uint32_t *layer_done;     // [n_layers] per-layer abs-max completion counters (fused kernel)
    uint32_t *bdone;          // [n_layers] per-layer quantise completion counters (fused kernel, self-resetting)
    uint32_t *sr_call;        // stochastic rounding: syncs since aps_set_rounding (per-call key, reading A27)
    uint8_t *packed;          // packed codes
    int n_items;
    int n_layers;
};

// a1 alone (aps_layer_scales): the control-warp kernel over the abs-max items
// (aps_fused.cu); DevTables.iptr must be current
cudaError_t launch_absmax_cw(const DevTables &t, int world, cudaStream_t s);

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

cudaError_t launch_build_item_ptrs(const DevTables &t, cudaStream_t s);
#ifndef APS_WAVE_LAG_GRIDS
#define APS_WAVE_LAG_GRIDS 2
#endif
// lag D of the wavefront = (items of the largest layer) + kWaveLagGrids x grid positions
constexpr int kWaveLagGrids = APS_WAVE_LAG_GRIDS;
// fused N = 1 sync, warp-specialised wavefront (aps_fused.cu): one launch per format group
// (hybrid FP32 classifier: one launch), self-resetting counters, no per-call host state
#ifndef APS_CW_SLOTS
#define APS_CW_SLOTS 3
#endif
#ifndef APS_CW_CTAS_PER_SM
#define APS_CW_CTAS_PER_SM 3
#endif
constexpr int kCwCtasPerSm = APS_CW_CTAS_PER_SM;
cudaError_t launch_fused_cw(const DevTables &t, int e, int m, bool hw, int average, int max_layer_items, cudaStream_t s,
                            int ctas_per_sm = 0);
// two format groups in one launch: items of group fmt2 use (e2, m2) (binary32 through the
// identity codec, any other format through the runtime codec)
cudaError_t launch_fused_cw_hybrid(const DevTables &t, int e, int m, bool hw, int e2, int m2, bool hw2, int fmt2,
                                   int average, int max_layer_items, cudaStream_t s, int ctas_per_sm = 0);
// true when (e,m) has a hardware converter that is exact on the APS path
// formats with a hardware / exact fast codec: fp8 e5m2, e4m3 (APS regime only,
// reading A12), binary16, bfloat16, binary32 (every non-NaN input)
inline bool hw_available(int e, int m)
{
    return (e == 5 && m == 2) || (e == 4 && m == 3) || (e == 5 && m == 10) || (e == 8 && m == 7) ||
           (e == 8 && m == 23);
}

}  // namespace aps
