// aps_api.cpp -- the C ABI of libaps (include/aps.h): context, workspace,
// phase checks, and the ring orchestration over NCCL send/recv (Alg. 1's
// AllReduce(low_g, SUM), as the ring all-reduce of P:410 / P:528).
#include "aps.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "aps_internal.h"
#include "aps_peer.h"

namespace aps {
constexpr uint32_t kFlagWaitTimeout = 2u;  // (mirrors aps_device.cuh)
}

namespace {

enum Phase { kNone = 0, kLocalScales = 1, kScales = 2, kPacked = 3, kReduced = 4 };

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

}  // namespace

struct aps_ctx {
    int e = 0, m = 0, b = 0, world = 1, rank = 0, n_layers = 0;
    bool sim = false;
    bool hw = true;
    ncclComm_t comm = nullptr;
    cudaStream_t stream = nullptr;
    std::vector<int64_t> numels;
    std::vector<aps::Item> items;
    std::vector<aps::LayerDev> layers;
    int ctas_per_sm = 0;                // aps_set_occupancy (0: as many as fit)
    int64_t tiles = 0;        // T' (padded to a multiple of world)
    int64_t packed_bytes = 0; // sum over tiles of 16 * b(tile)
    int64_t chunk_bytes = 0;  // packed_bytes / world (uniform formats)
    // per-layer formats (NEXT-2, hybrid precision): the layers' (e, m); items are
    // grouped by format (one launch per group); the ring reduces each chunk by
    // format segments and all-gathers unequal chunks with send/recv
    std::vector<int> le, lm;
    bool uniform = true, hw_enabled = true;
    struct Group {
        int e, m;
        bool hw;
        int item_begin, item_count, max_layer_items;
    };
    std::vector<Group> groups;
    struct Seg {
        int64_t byte_off, n_tiles;  // byte offset in the packed buffer, tiles
        int64_t tile0;              // first tile (global index: selects the reduction schedule)
        int e, m;
        bool hw;
    };
    std::vector<int64_t> chunk_byte;            // [world + 1]
    std::vector<std::vector<Seg>> chunk_segs;   // [world]
    int64_t max_chunk_bytes = 0;
    // workspace carve-up
    uint8_t *ws = nullptr;
    size_t ws_bytes = 0, need = 0;
    size_t off_packed = 0, off_recv = 0, off_items = 0, off_layers = 0, off_src = 0, off_dst = 0,
           off_eloc = 0, off_eglob = 0, off_ft = 0, off_flag = 0, off_amax2 = 0, off_iptr = 0, off_ldone = 0, off_claim64 = 0, off_bdone = 0, off_srcall = 0;
    int max_layer_items = 0;
    bool graph_safe = false;   // aps_set_graph_safe (every launch is capture-safe; recorded only)
    std::vector<const void *> host_key;            // aps_sync_host: pointer set of the cached copy runs
    std::vector<int> h2d_runs, d2h_runs;           // end layer of each coalesced copy
    bool iptr_valid = false;
    aps::DevTables t{};
    std::vector<const float *> src_cache;
    std::vector<float *> dst_cache;
    int phase = kNone;
    // format groups after the first run on side streams, concurrently with group 0
    // (disjoint layers, packed bytes and counters): fork/join through events
    std::vector<cudaStream_t> side;
    std::vector<cudaEvent_t> ev_join;
    cudaEvent_t ev_fork = nullptr;
    // reduction order and accumulator: hierarchical
    // group size (1 = flat ring), accumulator format, Kahan compensation
    int group_k = 1, acc_e = 0, acc_m = 0;
    bool kahan = false;
    // stochastic rounding (reading A26): counter-based draws keyed by (seed, phase, element)
    bool sr = false;
    uint64_t sr_seed = 0;
    // peer-memory transport (aps_peer.cu): every rank's workspace mapped here
    bool peer = false;
    aps::PeerArgs pa{};
    std::vector<void *> ipc_mapped;     // cudaIpcOpenMemHandle mappings (closed by aps_destroy)
    size_t off_pflags = 0, off_eslots = 0, off_census = 0;
    std::string err;
    bool stream_owned_ok() const { return ws != nullptr; }  // a workspace was attached: kernels may be queued
    ~aps_ctx()
    {
        for (void *p : ipc_mapped) cudaIpcCloseMemHandle(p);
        for (cudaStream_t s : side) cudaStreamDestroy(s);
        for (cudaEvent_t e : ev_join) cudaEventDestroy(e);
        if (ev_fork) cudaEventDestroy(ev_fork);
    }
};

namespace {

aps_status fail(aps_ctx *c, aps_status s, const std::string &msg)
{
    if (c) c->err = msg;
    return s;
}

#define APS_CUDA(ctx, expr)                                                                   \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail((ctx), APS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define APS_NCCL(ctx, expr)                                                                   \
    do {                                                                                      \
        ncclResult_t r_ = (expr);                                                             \
        if (r_ != ncclSuccess)                                                                \
            return fail((ctx), APS_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
    } while (0)

bool format_ok(int e, int m) { return e >= 2 && e <= 8 && m >= 0 && m <= 23 && 1 + e + m <= 32; }

int64_t layer_tiles(int64_t n) { return (n + aps::kTile - 1) / aps::kTile; }

// Upload the per-call pointer table if it changed (rarely: DDP buckets and
// optimizer-owned .grad buffers are stable).
template <class P>
aps_status upload_ptrs(aps_ctx *c, std::vector<P> &cache, P const *ptrs, size_t off)
{
    bool same = cache.size() == (size_t)c->n_layers;
    for (int l = 0; l < c->n_layers; ++l) {
        if (!ptrs[l]) return fail(c, APS_ERR_ARG, "NULL layer pointer");
        if (reinterpret_cast<uintptr_t>(ptrs[l]) % 16u)
            return fail(c, APS_ERR_ALIGN, "layer buffer not 16-byte aligned (layer " + std::to_string(l) + ")");
        if (same && cache[l] != ptrs[l]) same = false;
    }
    if (same) return APS_OK;
    c->iptr_valid = false;
    cache.assign(ptrs, ptrs + c->n_layers);
    APS_CUDA(c, cudaMemcpyAsync(c->ws + off, cache.data(), sizeof(P) * (size_t)c->n_layers,
                                cudaMemcpyHostToDevice, c->stream));
    return APS_OK;
}

aps_status need_ws(aps_ctx *c)
{
    if (!c) return APS_ERR_ARG;
    if (!c->ws) return fail(c, APS_ERR_STATE, "no workspace set (aps_set_workspace)");
    return APS_OK;
}

// Ring schedule (reading A14): chunk c accumulates in rank order c+1, ..., c.
inline int mod(int a, int p) { return ((a % p) + p) % p; }
inline int send_chunk(int p, int r, int s) { return mod(r - 1 - s, p); }
inline int recv_chunk(int p, int r, int s) { return mod(r - 2 - s, p); }

}  // namespace

extern "C" {

const char *aps_version(void) { return "libaps 0.1 (sm_100a)"; }

aps_status aps_layout(int world_size, int exp_bits, int man_bits, int n_layers, const int64_t *numels,
                      int64_t *total_tiles, int64_t *packed_bytes)
{
    if (!format_ok(exp_bits, man_bits)) return APS_ERR_FORMAT;
    if (world_size < 1 || n_layers < 1 || !numels) return APS_ERR_ARG;
    int64_t T = 0;
    for (int l = 0; l < n_layers; ++l) {
        if (numels[l] < 1) return APS_ERR_ARG;
        T += layer_tiles(numels[l]);
    }
    const int64_t Tp = (T + world_size - 1) / world_size * world_size;
    if (total_tiles) *total_tiles = Tp;
    if (packed_bytes) *packed_bytes = 16 * (int64_t)(1 + exp_bits + man_bits) * Tp;
    return APS_OK;
}

aps_status aps_ring_step(int world_size, int rank, int step, int *send_c, int *recv_c)
{
    if (world_size < 1 || rank < 0 || rank >= world_size || step < 0 || step > world_size - 2)
        return APS_ERR_ARG;
    if (send_c) *send_c = send_chunk(world_size, rank, step);
    if (recv_c) *recv_c = recv_chunk(world_size, rank, step);
    return APS_OK;
}

static aps_status init_common(aps_ctx **out, const int *e_arr, const int *m_arr, int world_size, int rank,
                              int n_layers, const int64_t *numels, void *nccl_comm, void *cuda_stream)
{
    if (!out) return APS_ERR_ARG;
    *out = nullptr;
    if (world_size < 1 || rank < 0 || rank >= world_size || n_layers < 1 || !numels || !e_arr || !m_arr)
        return APS_ERR_ARG;
    if (n_layers > (1 << 24)) return APS_ERR_ARG;
    for (int l = 0; l < n_layers; ++l)
        if (!format_ok(e_arr[l], m_arr[l])) return APS_ERR_FORMAT;
    aps_ctx *c = new (std::nothrow) aps_ctx();
    if (!c) return APS_ERR_ARG;
    c->le.assign(e_arr, e_arr + n_layers);
    c->lm.assign(m_arr, m_arr + n_layers);
    for (int l = 1; l < n_layers; ++l)
        if (c->le[l] != c->le[0] || c->lm[l] != c->lm[0]) c->uniform = false;
    c->e = e_arr[0];
    c->m = m_arr[0];
    c->b = 1 + c->e + c->m;
    c->world = world_size;
    c->rank = rank;
    c->n_layers = n_layers;
    c->comm = static_cast<ncclComm_t>(nccl_comm);
    c->sim = (world_size > 1 && !nccl_comm);
    c->stream = static_cast<cudaStream_t>(cuda_stream);
    c->hw = c->hw_enabled && aps::hw_available(c->e, c->m);
    if (c->comm) {
        int nr = 0;
        if (ncclCommCount(c->comm, &nr) != ncclSuccess || nr != world_size) {
            delete c;
            return APS_ERR_ARG;
        }
    }
    c->numels.assign(numels, numels + n_layers);
    std::vector<int64_t> layer_byte(n_layers);
    int64_t toff = 0, boff = 0;
    for (int l = 0; l < n_layers; ++l) {
        if (numels[l] < 1) {
            delete c;
            return APS_ERR_ARG;
        }
        const int64_t T = layer_tiles(numels[l]);
        if (T > INT32_MAX) {
            delete c;
            return APS_ERR_ARG;
        }
        const int64_t tb = 16 * (int64_t)(1 + c->le[l] + c->lm[l]);  // bytes per tile of this layer
        layer_byte[l] = boff;
        aps::LayerDev L{};
        L.numel = numels[l];
        L.tile_off = toff;
        L.n_items = 0;
        for (int64_t t0 = 0; t0 < T; t0 += aps::kItemTiles) {
            aps::Item it{};
            it.layer = l;
            it.tile_begin = (int32_t)t0;
            it.n_tiles = (int32_t)std::min<int64_t>(aps::kItemTiles, T - t0);
            it.cnt = (int32_t)std::min<int64_t>((int64_t)it.n_tiles * aps::kTile, numels[l] - t0 * aps::kTile);
            it.tile_pos = toff + t0;
            it.byte_pos = boff + t0 * tb;
            c->items.push_back(it);
            ++L.n_items;
        }
        for (size_t k = c->items.size() - (size_t)L.n_items; k < c->items.size(); ++k)
            c->items[k].layer_items = L.n_items;
        c->layers.push_back(L);
        toff += T;
        boff += T * tb;
    }
    if (c->items.size() > (size_t)INT32_MAX) {
        delete c;
        return APS_ERR_ARG;
    }
    const int64_t T = toff;
    c->tiles = (T + world_size - 1) / world_size * world_size;
    if (c->tiles > INT32_MAX) {  // tile indices are 32-bit on the device
        delete c;
        return APS_ERR_ARG;
    }
    const int64_t tb_last = 16 * (int64_t)(1 + c->le[n_layers - 1] + c->lm[n_layers - 1]);
    c->packed_bytes = boff + (c->tiles - T) * tb_last;  // padding tiles continue the last layer's format
    c->chunk_bytes = c->packed_bytes / world_size;     // (uniform formats)
    // format groups (first-appearance order; putting the smaller group first measured slower:
    // hybrid FP32 classifier 54.1 vs 49.1 us), items stably grouped by format
    std::vector<int> layer_group(n_layers);
    for (int l = 0; l < n_layers; ++l) {
        int g = 0;
        while (g < (int)c->groups.size() && (c->groups[g].e != c->le[l] || c->groups[g].m != c->lm[l])) ++g;
        if (g == (int)c->groups.size())
            c->groups.push_back({c->le[l], c->lm[l], c->hw_enabled && aps::hw_available(c->le[l], c->lm[l]), 0, 0, 0});
        layer_group[l] = g;
    }
    std::stable_sort(c->items.begin(), c->items.end(), [&](const aps::Item &a, const aps::Item &b) {
        return layer_group[a.layer] < layer_group[b.layer];
    });
    for (size_t k = 0; k < c->items.size(); ++k) {
        c->items[k].fmt = layer_group[c->items[k].layer];
        aps_ctx::Group &g = c->groups[layer_group[c->items[k].layer]];
        if (g.item_count == 0) g.item_begin = (int)k;
        ++g.item_count;
        g.max_layer_items = std::max(g.max_layer_items, c->items[k].layer_items);
    }
    // ring chunks: byte ranges and per-format segments
    auto tile_layer_byte = [&](int64_t t, int &layer) -> int64_t {  // byte offset of tile t
        if (t >= T) {
            layer = n_layers - 1;
            return boff + (t - T) * tb_last;
        }
        int lo = 0, hi = n_layers - 1;  // last layer with tile_off <= t
        while (lo < hi) {
            const int mid = (lo + hi + 1) / 2;
            if (c->layers[mid].tile_off <= t) lo = mid; else hi = mid - 1;
        }
        layer = lo;
        return layer_byte[lo] + (t - c->layers[lo].tile_off) * 16 * (int64_t)(1 + c->le[lo] + c->lm[lo]);
    };
    const int64_t ct = c->tiles / world_size;
    c->chunk_byte.resize(world_size + 1);
    c->chunk_segs.assign(world_size, {});
    for (int ch = 0; ch <= world_size; ++ch) {
        int lay;
        c->chunk_byte[ch] = ch == world_size ? c->packed_bytes : tile_layer_byte(ch * ct, lay);
    }
    for (int ch = 0; ch < world_size; ++ch) {
        int64_t t = ch * ct;
        const int64_t t_end = (ch + 1) * ct;
        while (t < t_end) {
            int lay;
            const int64_t byte = tile_layer_byte(t, lay);
            int64_t run_end = (t >= T) ? t_end : std::min<int64_t>(t_end, c->layers[lay].tile_off + layer_tiles(numels[lay]));
            if (run_end == T && lay == n_layers - 1) run_end = t_end;  // padding continues the last layer
            const int e = c->le[lay], m = c->lm[lay];
            std::vector<aps_ctx::Seg> &segs = c->chunk_segs[ch];
            if (!segs.empty() && segs.back().e == e && segs.back().m == m)
                segs.back().n_tiles += run_end - t;
            else
                segs.push_back({byte, run_end - t, t, e, m, c->hw_enabled && aps::hw_available(e, m)});
            t = run_end;
        }
        c->max_chunk_bytes = std::max(c->max_chunk_bytes, c->chunk_byte[ch + 1] - c->chunk_byte[ch]);
    }
    // workspace layout
    size_t o = 0;
    c->off_packed = o; o = align_up(o + (size_t)c->packed_bytes);
    c->off_recv = o;   o = align_up(o + (world_size > 1 ? (size_t)c->max_chunk_bytes : 0));
    c->off_items = o;  o = align_up(o + sizeof(aps::Item) * c->items.size());
    c->off_layers = o; o = align_up(o + sizeof(aps::LayerDev) * c->layers.size());
    c->off_src = o;    o = align_up(o + sizeof(void *) * (size_t)n_layers);
    c->off_dst = o;    o = align_up(o + sizeof(void *) * (size_t)n_layers);
    c->off_eloc = o;   o = align_up(o + 4 * (size_t)n_layers);
    c->off_eglob = o;  o = align_up(o + 4 * (size_t)n_layers);
    c->off_ft = o;     o = align_up(o + 4 * (size_t)n_layers);
    c->off_flag = o;   o = align_up(o + 4);
    c->off_amax2 = o;  o = align_up(o + 8 * (size_t)n_layers);
    c->off_iptr = o;   o = align_up(o + sizeof(aps::ItemPtr) * c->items.size());
    c->off_ldone = o;  o = align_up(o + 4 * (size_t)n_layers);
    c->off_bdone = o;  o = align_up(o + 4 * (size_t)n_layers);
    c->off_srcall = o; o = align_up(o + 4);
    // graph-safe counters: 64-bit wavefront claim counter per format group, absmax_ranges done counter
    c->off_claim64 = o; o = align_up(o + 8 * c->groups.size() + 4);
    // peer transport: flag block and E slots [2][world][n_layers] (world > 1 only)
    c->off_pflags = o; o = align_up(o + (world_size > 1 ? 4 * (size_t)aps::kFlagWords : 0));
    c->off_eslots = o; o = align_up(o + (world_size > 1 ? 2 * 4 * (size_t)world_size * (size_t)n_layers : 0));
    c->off_census = o; o = align_up(o + align_up(4 * (size_t)n_layers) + 16 * (size_t)n_layers);  // exps + [2] u64 counts
    c->acc_e = c->e;
    c->acc_m = c->m;

    for (const auto &L : c->layers) c->max_layer_items = std::max(c->max_layer_items, (int)L.n_items);
    c->need = o;
    *out = c;
    return APS_OK;
}

aps_status aps_init(aps_ctx **out, int exp_bits, int man_bits, int world_size, int rank, int n_layers,
                    const int64_t *numels, void *nccl_comm, void *cuda_stream)
{
    if (!out) return APS_ERR_ARG;
    *out = nullptr;
    if (!format_ok(exp_bits, man_bits)) return APS_ERR_FORMAT;
    if (n_layers < 1 || n_layers > (1 << 24)) return APS_ERR_ARG;
    std::vector<int> e(n_layers, exp_bits), m(n_layers, man_bits);
    return init_common(out, e.data(), m.data(), world_size, rank, n_layers, numels, nccl_comm, cuda_stream);
}

aps_status aps_init_mixed(aps_ctx **out, const int *exp_bits, const int *man_bits, int world_size, int rank,
                          int n_layers, const int64_t *numels, void *nccl_comm, void *cuda_stream)
{
    return init_common(out, exp_bits, man_bits, world_size, rank, n_layers, numels, nccl_comm, cuda_stream);
}

aps_status aps_layout_mixed(int world_size, int n_layers, const int64_t *numels, const int *exp_bits,
                            const int *man_bits, int64_t *total_tiles, int64_t *packed_bytes)
{
    if (world_size < 1 || n_layers < 1 || !numels || !exp_bits || !man_bits) return APS_ERR_ARG;
    int64_t T = 0, bytes = 0;
    for (int l = 0; l < n_layers; ++l) {
        if (!format_ok(exp_bits[l], man_bits[l])) return APS_ERR_FORMAT;
        if (numels[l] < 1) return APS_ERR_ARG;
        T += layer_tiles(numels[l]);
        bytes += 16 * (int64_t)(1 + exp_bits[l] + man_bits[l]) * layer_tiles(numels[l]);
    }
    const int64_t Tp = (T + world_size - 1) / world_size * world_size;
    if (total_tiles) *total_tiles = Tp;
    if (packed_bytes)
        *packed_bytes = bytes + (Tp - T) * 16 * (int64_t)(1 + exp_bits[n_layers - 1] + man_bits[n_layers - 1]);
    return APS_OK;
}

size_t aps_workspace_bytes(const aps_ctx *c) { return c ? c->need : 0; }

aps_status aps_set_workspace(aps_ctx *c, void *dev, size_t bytes)
{
    if (!c || !dev) return APS_ERR_ARG;
    if (reinterpret_cast<uintptr_t>(dev) % kAlign) return fail(c, APS_ERR_ALIGN, "workspace not 256-byte aligned");
    if (bytes < c->need) return fail(c, APS_ERR_ARG, "workspace too small");
    c->ws = static_cast<uint8_t *>(dev);
    c->ws_bytes = bytes;
    APS_CUDA(c, cudaMemsetAsync(c->ws, 0, c->need, c->stream));
    APS_CUDA(c, cudaMemcpyAsync(c->ws + c->off_items, c->items.data(), sizeof(aps::Item) * c->items.size(),
                                cudaMemcpyHostToDevice, c->stream));
    APS_CUDA(c, cudaMemcpyAsync(c->ws + c->off_layers, c->layers.data(),
                                sizeof(aps::LayerDev) * c->layers.size(), cudaMemcpyHostToDevice, c->stream));
    aps::DevTables &t = c->t;
    t.items = reinterpret_cast<const aps::Item *>(c->ws + c->off_items);
    t.layers = reinterpret_cast<const aps::LayerDev *>(c->ws + c->off_layers);
    t.src = reinterpret_cast<const float *const *>(c->ws + c->off_src);
    t.dst = reinterpret_cast<float *const *>(c->ws + c->off_dst);
    t.E_local = reinterpret_cast<int32_t *>(c->ws + c->off_eloc);
    // one rank: the global exponent vector IS the local one (no collective, no copy)
    t.E_glob = reinterpret_cast<int32_t *>(c->ws + (c->world == 1 ? c->off_eloc : c->off_eglob));
    t.ftilde = reinterpret_cast<int32_t *>(c->ws + c->off_ft);
    t.flag = reinterpret_cast<uint32_t *>(c->ws + c->off_flag);
    t.amax2 = reinterpret_cast<uint32_t *>(c->ws + c->off_amax2);
    t.iptr = reinterpret_cast<aps::ItemPtr *>(c->ws + c->off_iptr);
    t.claim64 = reinterpret_cast<unsigned long long *>(c->ws + c->off_claim64);
    t.ranges_done = reinterpret_cast<uint32_t *>(c->ws + c->off_claim64 + 8 * c->groups.size());
    t.layer_done = reinterpret_cast<uint32_t *>(c->ws + c->off_ldone);
    t.bdone = reinterpret_cast<uint32_t *>(c->ws + c->off_bdone);
    t.sr_call = reinterpret_cast<uint32_t *>(c->ws + c->off_srcall);

    if (c->groups.size() > 1 && c->side.empty()) {
        c->side.resize(c->groups.size() - 1);
        c->ev_join.resize(c->groups.size() - 1);
        for (size_t i = 0; i < c->side.size(); ++i) {
            APS_CUDA(c, cudaStreamCreateWithFlags(&c->side[i], cudaStreamNonBlocking));
            APS_CUDA(c, cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming));
        }
        APS_CUDA(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    }
    c->graph_safe = false;
    c->iptr_valid = false;
    t.packed = c->ws + c->off_packed;
    t.n_items = (int)c->items.size();
    t.n_layers = c->n_layers;
    c->src_cache.clear();
    c->dst_cache.clear();
    c->phase = kNone;
    return APS_OK;
}

// the tables of one format group: its items (contiguous after the grouping in init)
static aps::DevTables group_tables(const aps_ctx *c, const aps_ctx::Group &g)
{
    aps::DevTables t = c->t;
    t.items += g.item_begin;
    t.iptr += g.item_begin;
    t.n_items = g.item_count;
    t.claim64 += (&g - c->groups.data());
    return t;
}

// Launch `launch(group, tables, stream)` for every format group: group 0 on the
// context's stream, the others forked onto side streams and joined back (they
// touch disjoint layers, packed bytes and claim counters), so a small group (the
// FP32 classifier of the hybrid format) runs in the tail of the big one instead of
// after it.
extern "C++" {
template <class F>
static aps_status for_groups(aps_ctx *c, F launch)
{
    const bool concurrent = c->groups.size() > 1 && !c->side.empty();
    if (concurrent) {
        APS_CUDA(c, cudaEventRecord(c->ev_fork, c->stream));
        for (cudaStream_t s : c->side) APS_CUDA(c, cudaStreamWaitEvent(s, c->ev_fork, 0));
    }
    for (size_t g = 0; g < c->groups.size(); ++g) {
        cudaStream_t s = (concurrent && g > 0) ? c->side[g - 1] : c->stream;
        APS_CUDA(c, launch(c->groups[g], group_tables(c, c->groups[g]), s, !concurrent));
    }
    if (concurrent)
        for (size_t i = 0; i < c->side.size(); ++i) {
            APS_CUDA(c, cudaEventRecord(c->ev_join[i], c->side[i]));
            APS_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_join[i], 0));
        }
    return APS_OK;
}
}  // extern "C++"

// reduce the received copy of chunk ch into this rank's own copy, one launch per
// format segment of the chunk (a segment is a run of tiles of one format)
static aps_status reduce_chunk(aps_ctx *c, const aps_ctx *layout, int ch, const uint8_t *recv, cudaStream_t st)
{
    const int64_t base = layout->chunk_byte[ch];
    for (const auto &sg : layout->chunk_segs[ch])
        APS_CUDA(c, aps::launch_ring_reduce(c->t.packed + sg.byte_off, recv + (sg.byte_off - base), sg.n_tiles, sg.e,
                                            sg.m, sg.hw, st));
    return APS_OK;
}

static bool flat_reduction(const aps_ctx *c)
{
    return (c->group_k == 1 || c->group_k == c->world) && !c->kahan && c->acc_e == c->e && c->acc_m == c->m &&
           !c->sr;
}

// peer transport: announce this rank's packed codes, wait for every rank's
static aps_status peer_ready(aps_ctx *c)
{
    APS_CUDA(c, aps::launch_peer_signal_wait(c->pa, aps::kSlotReady, true, c->t.flag, c->stream));
    return APS_OK;
}

// peer transport: reduce this rank's chunk from every rank's codes, store it into every rank
static aps_status peer_reduce_own(aps_ctx *c)
{
    c->pa.group_k = c->group_k;
    if (c->sr) {
        for (const auto &sg : c->chunk_segs[c->rank])
            APS_CUDA(c, aps::launch_peer_reduce_sr(c->pa, sg.byte_off, sg.tile0, sg.n_tiles, sg.e, sg.m, c->sr_seed,
                                                   c->t.sr_call, c->stream));
        return APS_OK;
    }
    for (const auto &sg : c->chunk_segs[c->rank])
        APS_CUDA(c, aps::launch_peer_reduce(c->pa, sg.byte_off, sg.tile0, sg.n_tiles, sg.e, sg.m, sg.hw,
                                            c->uniform ? c->acc_e : sg.e, c->uniform ? c->acc_m : sg.m, c->kahan,
                                            c->stream));
    return APS_OK;
}

aps_status aps_set_hw_convert(aps_ctx *c, int enable)
{
    if (!c) return APS_ERR_ARG;
    c->hw_enabled = enable != 0;
    c->hw = c->hw_enabled && aps::hw_available(c->e, c->m);
    for (auto &g : c->groups) g.hw = c->hw_enabled && aps::hw_available(g.e, g.m);
    for (auto &segs : c->chunk_segs)
        for (auto &sg : segs) sg.hw = c->hw_enabled && aps::hw_available(sg.e, sg.m);
    return APS_OK;
}

aps_status aps_layer_scales(aps_ctx *c, const float *const *grads)
{
    if (aps_status s = need_ws(c)) return s;
    if (!grads) return fail(c, APS_ERR_ARG, "grads is NULL");
    if (aps_status s = upload_ptrs<const float *>(c, c->src_cache, grads, c->off_src)) return s;
    if (!c->iptr_valid) {  // per-item gradient addresses (output addresses: filled by the fused path)
        APS_CUDA(c, aps::launch_build_item_ptrs(c->t, c->stream));
        c->iptr_valid = true;
    }
    APS_CUDA(c, aps::launch_absmax_cw(c->t, c->world, c->stream));
    if (c->world == 1 && !c->comm) {
        c->phase = kScales;
    } else if (c->peer) {
        // AllReduce(max_grad_exp, MAX) over peer memory: post E to every rank, collect
        if (c->sim) {
            APS_CUDA(c, aps::launch_peer_post_E(c->pa, c->t.E_local, c->n_layers, c->stream));
            c->phase = kLocalScales;  // aps_sim_layer_scales collects after every rank posted
        } else {
            APS_CUDA(c, aps::launch_peer_exchange_E(c->pa, c->t.E_local, c->t.E_glob, c->n_layers, c->t.flag,
                                                    c->stream));
            c->phase = kScales;
        }
    } else if (c->sim) {
        c->phase = kLocalScales;  // aps_sim_layer_scales completes the exchange
    } else {
        // AllReduce(max_grad_exp, MAX) (Alg. 1 line 4): int32 per layer
        APS_NCCL(c, ncclAllReduce(c->t.E_local, c->t.E_glob, (size_t)c->n_layers, ncclInt32, ncclMax,
                                  c->comm, c->stream));
        c->phase = kScales;
    }
    return APS_OK;
}

aps_status aps_quantize_pack(aps_ctx *c, const float *const *grads)
{
    if (aps_status s = need_ws(c)) return s;
    if (c->phase < kScales) return fail(c, APS_ERR_STATE, "aps_quantize_pack before aps_layer_scales");
    if (!grads) return fail(c, APS_ERR_ARG, "grads is NULL");
    if (aps_status s = upload_ptrs<const float *>(c, c->src_cache, grads, c->off_src)) return s;
    if (c->sr) {  // stochastic rounding: one generic launch (uniform formats)
        APS_CUDA(c, aps::launch_quant_pack_sr(c->t, c->e, c->m, c->sr_seed, c->rank, c->stream));
        c->phase = kPacked;
        return APS_OK;
    }
    // one launch per format group (NEXT-2)
    if (aps_status s = for_groups(c, [&](const aps_ctx::Group &g, const aps::DevTables &t, cudaStream_t st, bool) {
            return aps::launch_quant_pack(t, g.e, g.m, g.hw, st);
        }))
        return s;
    c->phase = kPacked;
    return APS_OK;
}

aps_status aps_allreduce(aps_ctx *c)
{
    if (aps_status s = need_ws(c)) return s;
    if (c->phase != kPacked) return fail(c, APS_ERR_STATE, "aps_allreduce before aps_quantize_pack");
    if (c->world == 1 && !c->comm) {  // (a 1-rank communicator still goes through NCCL)
        c->phase = kReduced;
        return APS_OK;
    }
    if (c->sim) return fail(c, APS_ERR_STATE, "simulated rank: use aps_sim_allreduce");
    if (c->peer) {
        if (aps_status s = peer_ready(c)) return s;
        if (aps_status s = peer_reduce_own(c)) return s;
        APS_CUDA(c, aps::launch_peer_signal_wait(c->pa, aps::kSlotDone, false, c->t.flag, c->stream));
        c->phase = kReduced;
        return APS_OK;
    }
    if (!flat_reduction(c))
        return fail(c, APS_ERR_STATE, "hierarchical order / accumulator variants need the peer transport");
    const int p = c->world, r = c->rank;
    uint8_t *packed = c->t.packed;
    uint8_t *recv = c->ws + c->off_recv;
    // reduce-scatter: p-1 steps, each a send/recv of packed bytes then the
    // unpack-add-requantise-repack kernel per format segment (same stream: ordered)
    for (int s = 0; s < p - 1; ++s) {
        const int sc = send_chunk(p, r, s), rc = recv_chunk(p, r, s);
        APS_NCCL(c, ncclGroupStart());
        APS_NCCL(c, ncclSend(packed + c->chunk_byte[sc], (size_t)(c->chunk_byte[sc + 1] - c->chunk_byte[sc]),
                             ncclUint8, mod(r + 1, p), c->comm, c->stream));
        APS_NCCL(c, ncclRecv(recv, (size_t)(c->chunk_byte[rc + 1] - c->chunk_byte[rc]), ncclUint8, mod(r - 1, p),
                             c->comm, c->stream));
        APS_NCCL(c, ncclGroupEnd());
        if (aps_status st = reduce_chunk(c, c, rc, recv, c->stream)) return st;
    }
    // all-gather of the reduced chunks (pure data movement; rank r owns chunk r)
    if (c->uniform) {
        const size_t cb = (size_t)c->chunk_bytes;
        APS_NCCL(c, ncclAllGather(packed + (size_t)r * cb, packed, cb, ncclUint8, c->comm, c->stream));
    } else {
        // chunks of unequal byte size: p-1 ring forwarding steps (step s passes on chunk r-s)
        for (int s = 0; s < p - 1; ++s) {
            const int sc = mod(r - s, p), rc = mod(r - s - 1, p);
            APS_NCCL(c, ncclGroupStart());
            APS_NCCL(c, ncclSend(packed + c->chunk_byte[sc], (size_t)(c->chunk_byte[sc + 1] - c->chunk_byte[sc]),
                                 ncclUint8, mod(r + 1, p), c->comm, c->stream));
            APS_NCCL(c, ncclRecv(packed + c->chunk_byte[rc], (size_t)(c->chunk_byte[rc + 1] - c->chunk_byte[rc]),
                                 ncclUint8, mod(r - 1, p), c->comm, c->stream));
            APS_NCCL(c, ncclGroupEnd());
        }
    }
    c->phase = kReduced;
    return APS_OK;
}

aps_status aps_unscale(aps_ctx *c, float *const *out, int average)
{
    if (aps_status s = need_ws(c)) return s;
    if (c->phase < kPacked || (c->world > 1 && c->phase < kReduced))
        return fail(c, APS_ERR_STATE, "aps_unscale before aps_allreduce");
    if (!out) return fail(c, APS_ERR_ARG, "out is NULL");
    if (aps_status s = upload_ptrs<float *>(c, c->dst_cache, out, c->off_dst)) return s;
    if (aps_status s = for_groups(c, [&](const aps_ctx::Group &g, const aps::DevTables &t, cudaStream_t st, bool) {
            return aps::launch_unpack_unscale(t, g.e, g.m, g.hw, c->world, average, st);
        }))
        return s;
    // stochastic rounding: this sync is done, the next one draws with the next key (A27)
    if (c->sr) APS_CUDA(c, aps::launch_sr_advance(c->t.sr_call, c->stream));
    return APS_OK;
}

// two formats (the paper's hybrid precision: one low format + the FP32 classifier layer,
// P:545, or any second format) run as ONE launch whose second-format items switch codec
// inside the kernel (the second launch of a small group cost ~9 us of ramp and tail: a
// (5,6) last layer 54.9 vs 45.7 us).  Returns the group with fewer items (the kernel's
// second codec), or -1.
static int hybrid_second_group(const aps_ctx *c)
{
    if (c->groups.size() != 2) return -1;
    return c->groups[1].item_count <= c->groups[0].item_count ? 1 : 0;
}

aps_status aps_sync_out(aps_ctx *c, const float *const *grads, float *const *out, int average)
{
    if (aps_status s = need_ws(c)) return s;
    if (!grads || !out) return fail(c, APS_ERR_ARG, "NULL pointer array");
    if (c->world == 1 && !c->comm && !c->sr) {
        // one rank: FindMaxExp -> f~ -> Cast -> pack -> Cast back -> unscale in one
        // launch per format group (aps_fused.cu: quantise items trail their abs-max items
        // by D claim positions; a layer's items never straddle groups)
        if (aps_status s = upload_ptrs<const float *>(c, c->src_cache, grads, c->off_src)) return s;
        if (aps_status s = upload_ptrs<float *>(c, c->dst_cache, out, c->off_dst)) return s;
        if (!c->iptr_valid) {
            APS_CUDA(c, aps::launch_build_item_ptrs(c->t, c->stream));
            c->iptr_valid = true;
        }
        const int g2 = hybrid_second_group(c);
        if (g2 >= 0) {
            const aps_ctx::Group &lo = c->groups[1 - g2], &hi = c->groups[g2];
            APS_CUDA(c, aps::launch_fused_cw_hybrid(c->t, lo.e, lo.m, lo.hw, hi.e, hi.m, hi.hw, g2, average,
                                                    c->max_layer_items, c->stream, c->ctas_per_sm));
        } else {
            // one launch per format group, in order on the context's stream
            for (const auto &g : c->groups)
                APS_CUDA(c, aps::launch_fused_cw(group_tables(c, g), g.e, g.m, g.hw, average, g.max_layer_items,
                                                 c->stream, c->ctas_per_sm));
        }
        c->phase = kReduced;
        return APS_OK;
    }
    if (aps_status s = aps_layer_scales(c, grads)) return s;
    if (aps_status s = aps_quantize_pack(c, grads)) return s;
    if (aps_status s = aps_allreduce(c)) return s;
    return aps_unscale(c, out, average);
}

aps_status aps_sync(aps_ctx *c, float *const *grads, int average)
{
    return aps_sync_out(c, const_cast<const float *const *>(grads), grads, average);
}

static cudaError_t alloc_base(void *p, uint8_t **base);

aps_status aps_sync_host(aps_ctx *c, const float *const *host_in, float *const *dev_grads,
                         float *const *host_out, int average)
{
    if (aps_status s = need_ws(c)) return s;
    if (!host_in || !dev_grads || !host_out) return fail(c, APS_ERR_ARG, "NULL pointer array");
    // one copy per run of layers that are contiguous on both sides AND inside one
    // allocation on both sides (a flat gradient buffer with per-layer views -- DDP's
    // buckets -- moves in one transfer each way); runs are cached per pointer set
    std::vector<const void *> key;
    key.reserve(3 * (size_t)c->n_layers);
    for (int l = 0; l < c->n_layers; ++l) {
        key.push_back(host_in[l]);
        key.push_back(dev_grads[l]);
        key.push_back(host_out[l]);
    }
    if (key != c->host_key) {
        auto runs_of = [&](const void *const *a, const void *const *b, std::vector<int> &runs) -> aps_status {
            runs.clear();
            int l = 0;
            while (l < c->n_layers) {
                uint8_t *ba = nullptr, *bb = nullptr;  // allocation bases (unknown: never merge)
                const bool known = alloc_base(const_cast<void *>(a[l]), &ba) == cudaSuccess &&
                                   alloc_base(const_cast<void *>(b[l]), &bb) == cudaSuccess;
                (void)cudaGetLastError();
                size_t bytes = 4 * (size_t)c->numels[l];
                int k = l + 1;
                while (known && k < c->n_layers &&
                       static_cast<const char *>(a[k]) == static_cast<const char *>(a[l]) + bytes &&
                       static_cast<const char *>(b[k]) == static_cast<const char *>(b[l]) + bytes) {
                    uint8_t *ka = nullptr, *kb = nullptr;
                    if (alloc_base(const_cast<void *>(a[k]), &ka) != cudaSuccess || ka != ba ||
                        alloc_base(const_cast<void *>(b[k]), &kb) != cudaSuccess || kb != bb)
                        break;
                    bytes += 4 * (size_t)c->numels[k];
                    ++k;
                }
                runs.push_back(k);
                l = k;
            }
            return APS_OK;
        };
        if (aps_status s = runs_of(reinterpret_cast<const void *const *>(host_in),
                                   reinterpret_cast<const void *const *>(dev_grads), c->h2d_runs))
            return s;
        if (aps_status s = runs_of(reinterpret_cast<const void *const *>(dev_grads),
                                   reinterpret_cast<const void *const *>(host_out), c->d2h_runs))
            return s;
        c->host_key.swap(key);
    }
    auto copy_runs = [&](void *const *dst, const void *const *src, const std::vector<int> &runs,
                         cudaMemcpyKind kind) -> aps_status {
        int l = 0;
        for (int k : runs) {
            size_t bytes = 0;
            for (int q = l; q < k; ++q) bytes += 4 * (size_t)c->numels[q];
            APS_CUDA(c, cudaMemcpyAsync(dst[l], src[l], bytes, kind, c->stream));
            l = k;
        }
        return APS_OK;
    };
    if (aps_status s = copy_runs(reinterpret_cast<void *const *>(dev_grads),
                                 reinterpret_cast<const void *const *>(host_in), c->h2d_runs, cudaMemcpyHostToDevice))
        return s;
    if (aps_status s = aps_sync(c, dev_grads, average)) return s;
    return copy_runs(reinterpret_cast<void *const *>(host_out), reinterpret_cast<const void *const *>(dev_grads),
                     c->d2h_runs, cudaMemcpyDeviceToHost);
}

aps_status aps_status_sync(aps_ctx *c)
{
    if (aps_status s = need_ws(c)) return s;
    uint32_t flag = 0;
    APS_CUDA(c, cudaMemcpyAsync(&flag, c->t.flag, 4, cudaMemcpyDeviceToHost, c->stream));
    APS_CUDA(c, cudaStreamSynchronize(c->stream));
    if (flag) {
        APS_CUDA(c, cudaMemsetAsync(c->t.flag, 0, 4, c->stream));
        if (flag & aps::kFlagWaitTimeout)
            return fail(c, APS_ERR_STATE, "a device-side wait timed out (work counters out of step); outputs invalid");
        return fail(c, APS_ERR_NONFINITE, "non-finite gradient seen (outputs unspecified)");
    }
    return APS_OK;
}

aps_status aps_get_scales(aps_ctx *c, int32_t *host_out)
{
    if (aps_status s = need_ws(c)) return s;
    if (!host_out) return APS_ERR_ARG;
    APS_CUDA(c, cudaMemcpyAsync(host_out, c->t.ftilde, 4 * (size_t)c->n_layers, cudaMemcpyDeviceToHost, c->stream));
    APS_CUDA(c, cudaStreamSynchronize(c->stream));
    return APS_OK;
}

aps_status aps_get_packed(aps_ctx *c, const void **dev, size_t *bytes)
{
    if (aps_status s = need_ws(c)) return s;
    if (dev) *dev = c->t.packed;
    if (bytes) *bytes = (size_t)c->packed_bytes;
    return APS_OK;
}

const char *aps_last_error(const aps_ctx *c) { return c ? c->err.c_str() : "NULL context"; }

aps_status aps_set_reduction(aps_ctx *c, int group_k, int acc_exp_bits, int acc_man_bits, int kahan)
{
    if (!c) return APS_ERR_ARG;
    if (group_k < 1 || group_k > c->world || c->world % group_k)
        return fail(c, APS_ERR_ARG, "group_k must divide world_size");
    if (!format_ok(acc_exp_bits, acc_man_bits)) return fail(c, APS_ERR_FORMAT, "invalid accumulator format");
    const bool ext = kahan || acc_exp_bits != c->e || acc_man_bits != c->m;
    if (ext && !c->uniform) return fail(c, APS_ERR_ARG, "accumulator variants need one format for every layer");
    if (ext && c->sr) return fail(c, APS_ERR_ARG, "accumulator variants are not combined with stochastic rounding");
    if (acc_exp_bits < c->e || acc_man_bits < c->m)
        return fail(c, APS_ERR_FORMAT, "the accumulator must hold every wire value (exp and man bits >= the wire's)");
    c->group_k = group_k;
    c->acc_e = acc_exp_bits;
    c->acc_m = acc_man_bits;
    c->kahan = kahan != 0;
    return APS_OK;
}

aps_status aps_set_graph_safe(aps_ctx *c, int enable)
{
    if (aps_status s = need_ws(c)) return s;
    // every launch is capture-safe (self-resetting device counters, device-resident peer
    // epochs): nothing to switch; the flag is recorded for aps_debug_* introspection only
    c->graph_safe = enable != 0;
    return APS_OK;
}

aps_status aps_set_occupancy(aps_ctx *c, int ctas_per_sm)
{
    if (!c || ctas_per_sm < 0) return c ? fail(c, APS_ERR_ARG, "ctas_per_sm < 0") : APS_ERR_ARG;
    c->ctas_per_sm = ctas_per_sm;
    return APS_OK;
}

aps_status aps_set_rounding(aps_ctx *c, int mode, uint64_t seed)
{
    if (!c) return APS_ERR_ARG;
    if (mode != 0 && mode != 1) return fail(c, APS_ERR_ARG, "rounding mode must be 0 (nearest even) or 1 (stochastic)");
    if (mode == 1 && (!c->uniform || c->kahan || c->acc_e != c->e || c->acc_m != c->m))
        return fail(c, APS_ERR_ARG, "stochastic rounding needs one format and the wire-format accumulator");
    c->sr = mode == 1;
    c->sr_seed = seed;
    if (c->ws) APS_CUDA(c, cudaMemsetAsync(c->t.sr_call, 0, 4, c->stream));  // call k = 0 draws with SplitMix64(seed, 0)
    return APS_OK;
}

// base of the device allocation holding p (cuMemGetAddressRange through the runtime's
// driver entry point: libaps does not link libcuda)
static cudaError_t alloc_base(void *p, uint8_t **base)
{
    typedef int (*Fn)(unsigned long long *, size_t *, unsigned long long);
    static Fn fn = nullptr;
    if (!fn) {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q);
        if (e != cudaSuccess) return e;
        if (q != cudaDriverEntryPointSuccess || !f) return cudaErrorNotSupported;
        fn = reinterpret_cast<Fn>(f);
    }
    unsigned long long b = 0;
    size_t sz = 0;
    if (fn(&b, &sz, reinterpret_cast<unsigned long long>(p)) != 0) return cudaErrorInvalidValue;
    *base = reinterpret_cast<uint8_t *>(b);
    return cudaSuccess;
}

static void peer_set(aps_ctx *c, int q, uint8_t *ws)
{
    c->pa.packed[q] = ws + c->off_packed;
    c->pa.flags[q] = reinterpret_cast<uint32_t *>(ws + c->off_pflags);
    c->pa.eslots[q] = reinterpret_cast<int32_t *>(ws + c->off_eslots);
}

static void peer_common(aps_ctx *c)
{
    double tmo = 120.0;
    if (const char *v = std::getenv("APS_PEER_TIMEOUT_S")) tmo = std::atof(v);
    c->pa.timeout_ns = (uint64_t)(std::max(0.001, tmo) * 1e9);
    c->pa.p = c->world;
    c->pa.rank = c->rank;
    c->pa.tiles = c->tiles;
    c->pa.group_k = c->group_k;
    c->peer = true;
}

aps_status aps_peer_export(aps_ctx *c, void *host_handle, uint64_t *host_offset)
{
    if (aps_status s = need_ws(c)) return s;
    if (!host_handle || !host_offset) return APS_ERR_ARG;
    if (c->world < 2 || c->world > aps::kMaxPeers) return fail(c, APS_ERR_STATE, "peer transport needs 2..64 ranks");
    uint8_t *base = nullptr;
    APS_CUDA(c, alloc_base(c->ws, &base));
    cudaIpcMemHandle_t h;
    APS_CUDA(c, cudaIpcGetMemHandle(&h, base));
    static_assert(sizeof(h) <= APS_PEER_HANDLE_BYTES, "IPC handle size");
    std::memset(host_handle, 0, APS_PEER_HANDLE_BYTES);
    std::memcpy(host_handle, &h, sizeof(h));
    *host_offset = (uint64_t)(c->ws - base);
    APS_CUDA(c, cudaStreamSynchronize(c->stream));  // the workspace zero-fill is done before any peer writes
    return APS_OK;
}

aps_status aps_peer_import(aps_ctx *c, const void *host_handles, const uint64_t *host_offsets)
{
    if (aps_status s = need_ws(c)) return s;
    if (!host_handles || !host_offsets) return APS_ERR_ARG;
    if (c->world < 2 || c->world > aps::kMaxPeers) return fail(c, APS_ERR_STATE, "peer transport needs 2..64 ranks");
    if (c->peer) return fail(c, APS_ERR_STATE, "peers already imported");
    for (int q = 0; q < c->world; ++q) {
        if (q == c->rank) {
            peer_set(c, q, c->ws);
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const uint8_t *>(host_handles) + (size_t)q * APS_PEER_HANDLE_BYTES, sizeof(h));
        void *p = nullptr;
        APS_CUDA(c, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_mapped.push_back(p);
        peer_set(c, q, static_cast<uint8_t *>(p) + host_offsets[q]);
    }
    peer_common(c);
    c->sim = false;  // a rank created without a communicator is now a real rank of the peer transport
    return APS_OK;
}

aps_status aps_census(aps_ctx *c, const float *const *grads, const int32_t *host_scale_exp, uint64_t *host_counts)
{
    if (aps_status s = need_ws(c)) return s;
    if (!grads || !host_scale_exp || !host_counts) return fail(c, APS_ERR_ARG, "NULL argument");
    if (!c->uniform) return fail(c, APS_ERR_ARG, "aps_census needs one format for every layer");
    if (aps_status s = upload_ptrs<const float *>(c, c->src_cache, grads, c->off_src)) return s;
    int32_t *dexp = reinterpret_cast<int32_t *>(c->ws + c->off_census);
    unsigned long long *dcnt =
        reinterpret_cast<unsigned long long *>(c->ws + c->off_census + align_up(4 * (size_t)c->n_layers));
    APS_CUDA(c, cudaMemcpyAsync(dexp, host_scale_exp, 4 * (size_t)c->n_layers, cudaMemcpyHostToDevice, c->stream));
    APS_CUDA(c, cudaMemsetAsync(dcnt, 0, 16 * (size_t)c->n_layers, c->stream));
    APS_CUDA(c, aps::launch_census(c->t, dexp, dcnt, c->e, c->m, c->stream));
    APS_CUDA(c, cudaMemcpyAsync(host_counts, dcnt, 16 * (size_t)c->n_layers, cudaMemcpyDeviceToHost, c->stream));
    APS_CUDA(c, cudaStreamSynchronize(c->stream));
    return APS_OK;
}

aps_status aps_round_off_error(const float *h, const float *l, int64_t n, double *dev_sum,
                               unsigned long long *dev_count, void *stream)
{
    if (n < 0 || (n > 0 && (!h || !l)) || !dev_sum || !dev_count) return APS_ERR_ARG;
    return aps::launch_round_off(h, l, n, dev_sum, dev_count, static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? APS_OK : APS_ERR_CUDA;
}

aps_status aps_destroy(aps_ctx *c)
{
    // kernels still queued on the context's streams may read peer workspaces through the
    // IPC mappings ~aps_ctx closes: drain them first
    if (c && c->stream_owned_ok()) {
        cudaStreamSynchronize(c->stream);
        for (cudaStream_t s : c->side) cudaStreamSynchronize(s);
        (void)cudaGetLastError();
    }
    delete c;
    return APS_OK;
}

// ---------------------------------------------------------------- NCCL plumbing
aps_status aps_nccl_unique_id(void *host_uid, size_t bytes)
{
    if (!host_uid || bytes < sizeof(ncclUniqueId)) return APS_ERR_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return APS_ERR_NCCL;
    std::memcpy(host_uid, &id, sizeof(id));
    return APS_OK;
}

aps_status aps_nccl_comm_init(void **comm_out, const void *host_uid, int world_size, int rank)
{
    if (!comm_out || !host_uid || world_size < 1 || rank < 0 || rank >= world_size) return APS_ERR_ARG;
    ncclUniqueId id;
    std::memcpy(&id, host_uid, sizeof(id));
    ncclComm_t comm = nullptr;
    if (ncclCommInitRank(&comm, world_size, id, rank) != ncclSuccess) return APS_ERR_NCCL;
    *comm_out = comm;
    return APS_OK;
}

aps_status aps_nccl_comm_destroy(void *comm)
{
    if (!comm) return APS_ERR_ARG;
    return ncclCommDestroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? APS_OK : APS_ERR_NCCL;
}

// ---------------------------------------------------------------- simulated ranks (test mode)
static aps_status sim_check(aps_ctx *const *ctxs, int p)
{
    if (!ctxs || p < 2 || p > 64) return APS_ERR_ARG;
    for (int r = 0; r < p; ++r) {
        aps_ctx *c = ctxs[r];
        if (!c || !c->sim || c->world != p || c->rank != r) return APS_ERR_ARG;
        if (!c->ws) return fail(c, APS_ERR_STATE, "no workspace");
        if (c->stream != ctxs[0]->stream || c->le != ctxs[0]->le || c->lm != ctxs[0]->lm ||
            c->packed_bytes != ctxs[0]->packed_bytes || c->hw_enabled != ctxs[0]->hw_enabled)
            return fail(c, APS_ERR_ARG, "simulated ranks differ in stream/format/layout");
    }
    return APS_OK;
}

aps_status aps_sim_connect(aps_ctx *const *ctxs, int p)
{
    if (aps_status s = sim_check(ctxs, p)) return s;
    for (int r = 0; r < p; ++r) {
        for (int q = 0; q < p; ++q) peer_set(ctxs[r], q, ctxs[q]->ws);
        peer_common(ctxs[r]);
    }
    return APS_OK;
}

aps_status aps_sim_layer_scales(aps_ctx *const *ctxs, int p, const float *const *grads)
{
    if (aps_status s = sim_check(ctxs, p)) return s;
    if (!grads) return APS_ERR_ARG;
    for (int r = 0; r < p; ++r)
        if (aps_status s = aps_layer_scales(ctxs[r], grads + (size_t)r * ctxs[r]->n_layers)) return s;
    if (ctxs[0]->peer) {  // every rank posted its E; now every rank collects
        for (int r = 0; r < p; ++r) {
            aps_ctx *c = ctxs[r];
            APS_CUDA(c, aps::launch_peer_collect_E(c->pa, c->t.E_glob, c->n_layers, c->t.flag, c->stream));
            c->phase = kScales;
        }
        return APS_OK;
    }
    std::vector<int32_t *> dst(p);
    std::vector<const int32_t *> src(p);
    for (int r = 0; r < p; ++r) {
        dst[r] = ctxs[r]->t.E_glob;
        src[r] = ctxs[r]->t.E_local;
    }
    APS_CUDA(ctxs[0], aps::launch_sim_max(dst.data(), src.data(), p, ctxs[0]->n_layers, ctxs[0]->stream));
    for (int r = 0; r < p; ++r) ctxs[r]->phase = kScales;
    return APS_OK;
}

aps_status aps_sim_allreduce(aps_ctx *const *ctxs, int p)
{
    if (aps_status s = sim_check(ctxs, p)) return s;
    for (int r = 0; r < p; ++r)
        if (ctxs[r]->phase != kPacked) return fail(ctxs[r], APS_ERR_STATE, "sim allreduce before quantize");
    if (ctxs[0]->peer) {  // same kernels as aps_allreduce, phase by phase over the ranks
        for (int r = 0; r < p; ++r)
            APS_CUDA(ctxs[r], aps::launch_peer_signal(ctxs[r]->pa, aps::kSlotReady, true, ctxs[r]->stream));
        for (int r = 0; r < p; ++r) {
            aps_ctx *c = ctxs[r];
            APS_CUDA(c, aps::launch_peer_wait(c->pa, aps::kSlotReady, c->t.flag, c->stream));
            if (aps_status s = peer_reduce_own(c)) return s;
        }
        for (int r = 0; r < p; ++r)
            APS_CUDA(ctxs[r], aps::launch_peer_signal(ctxs[r]->pa, aps::kSlotDone, false, ctxs[r]->stream));
        for (int r = 0; r < p; ++r) {
            APS_CUDA(ctxs[r], aps::launch_peer_wait(ctxs[r]->pa, aps::kSlotDone, ctxs[r]->t.flag, ctxs[r]->stream));
            ctxs[r]->phase = kReduced;
        }
        return APS_OK;
    }
    for (int r = 0; r < p; ++r)
        if (!flat_reduction(ctxs[r]))
            return fail(ctxs[r], APS_ERR_STATE, "hierarchical order / accumulator variants need aps_sim_connect");
    aps_ctx *c0 = ctxs[0];
    const std::vector<int64_t> &cbyte = c0->chunk_byte;
    cudaStream_t st = c0->stream;
    for (int s = 0; s < p - 1; ++s) {
        // the "send/recv": rank r receives chunk recv_chunk(p, r, s) from rank r-1,
        // which sends exactly that chunk (send_chunk(p, r-1, s) == recv_chunk(p, r, s))
        for (int r = 0; r < p; ++r) {
            aps_ctx *me = ctxs[r], *prev = ctxs[mod(r - 1, p)];
            const int rc = recv_chunk(p, r, s);
            APS_CUDA(me, cudaMemcpyAsync(me->ws + me->off_recv, prev->t.packed + cbyte[rc],
                                         (size_t)(cbyte[rc + 1] - cbyte[rc]), cudaMemcpyDeviceToDevice, st));
        }
        for (int r = 0; r < p; ++r) {
            aps_ctx *me = ctxs[r];
            if (aps_status sr = reduce_chunk(me, me, recv_chunk(p, r, s), me->ws + me->off_recv, st)) return sr;
        }
    }
    for (int r = 0; r < p; ++r)
        for (int q = 0; q < p; ++q)
            if (q != r)
                APS_CUDA(ctxs[r], cudaMemcpyAsync(ctxs[r]->t.packed + cbyte[q], ctxs[q]->t.packed + cbyte[q],
                                                  (size_t)(cbyte[q + 1] - cbyte[q]), cudaMemcpyDeviceToDevice, st));
    for (int r = 0; r < p; ++r) ctxs[r]->phase = kReduced;
    return APS_OK;
}

// ---------------------------------------------------------------- debug
aps_status aps_debug_cast(const float *in, uint32_t *codes, int64_t n, int e, int m, int hw, void *stream)
{
    if (!format_ok(e, m)) return APS_ERR_FORMAT;
    if (n < 0 || (n > 0 && (!in || !codes))) return APS_ERR_ARG;
    if (hw && !aps::hw_available(e, m)) return APS_ERR_FORMAT;
    return aps::launch_debug_cast(in, codes, n, e, m, hw != 0, static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? APS_OK : APS_ERR_CUDA;
}

aps_status aps_debug_decode(const uint32_t *codes, float *out, int64_t n, int e, int m, int hw, void *stream)
{
    if (!format_ok(e, m)) return APS_ERR_FORMAT;
    if (n < 0 || (n > 0 && (!out || !codes))) return APS_ERR_ARG;
    if (hw && !aps::hw_available(e, m)) return APS_ERR_FORMAT;
    return aps::launch_debug_decode(codes, out, n, e, m, hw != 0, static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? APS_OK : APS_ERR_CUDA;
}

aps_status aps_debug_cast_sr(const float *in, uint32_t *codes, int64_t n, int e, int m, uint64_t seed, uint64_t phase,
                             void *stream)
{
    if (!format_ok(e, m)) return APS_ERR_FORMAT;
    if (n < 0 || (n > 0 && (!in || !codes))) return APS_ERR_ARG;
    return aps::launch_debug_cast_sr(in, codes, n, e, m, seed, phase, static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? APS_OK : APS_ERR_CUDA;
}


aps_status aps_debug_ring_reduce(uint8_t *own, const uint8_t *recv, int64_t n_tiles, int e, int m, int hw,
                                 void *stream)
{
    if (!format_ok(e, m)) return APS_ERR_FORMAT;
    if (n_tiles < 0 || (n_tiles > 0 && (!own || !recv))) return APS_ERR_ARG;
    if (hw && !aps::hw_available(e, m)) return APS_ERR_FORMAT;
    return aps::launch_ring_reduce(own, recv, n_tiles, e, m, hw != 0, static_cast<cudaStream_t>(stream)) == cudaSuccess
               ? APS_OK : APS_ERR_CUDA;
}

}  // extern "C"
