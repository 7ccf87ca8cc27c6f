// Domino handle shared by the domino translation units.
#pragma once

#include <vector>

#include "tsb_internal.cuh"

struct tsb_domino {
    int device = 0, side = 0, nchains = 0, W = 0, pitch = 0;
    size_t chain_stride = 0;  // uint2 elements per chain
    uint2 *buf[2] = {nullptr, nullptr};  // row r of chain c at buf + c * chain_stride + (r + 1) * pitch (global r)
    uint2 *buf_alloc[2] = {nullptr, nullptr};  // allocations (== buf unless windowed)
    // row windows (tsb_domino_create_window): only global rows [row_a, row_b)
    // are allocated (state, domain planes); buf / dom / fbits are offset so
    // that kernels index global rows
    bool windowed = false;
    int row_a = -1, row_b = 0;
    uint4 *dom_alloc = nullptr;
    uint32_t *fbits_alloc = nullptr;
    int cur = 0;
    uint4 *dom = nullptr;        // {crossable V, crossable H, existing V, existing H} per word
    uint32_t *fbits = nullptr;   // face (r, c) in the domain
    int2 *range = nullptr;
    int2 *tiles = nullptr;  // non-empty sweep tiles {word chunk, row band}
    int ntiles = 0;
    std::vector<int> band_start;  // first tile of every row band (tiles are band-major)
    int win_t0 = 0, win_tn = 0;   // swept tile range (row window; default all)
    int2 *mtiles = nullptr;       // tiles of the temporally blocked kernel (kMOut-row bands)
    int nmtiles = 0;
    int *m_order = nullptr;       // dispatch order of whole-domain multi-sweep launches (replay_tail_kernel)
    unsigned *m_cost = nullptr;   // last block duration per multi-sweep tile (cycles)
    int2 *m_perm = nullptr;       // mtiles in that order
    bool m_adapt = true;          // TSB_DOM_ADAPT=0: band-major order
    int m_order_every = 8;        // reorder on every n-th graph replay (TSB_DOM_ORDER_EVERY)
    std::vector<int> mband_start;
    int win_m0 = 0, win_mn = 0;
    int win_rows = 0;  // rows of the swept window (set with the tile lists; default: side)
    int m_pipe = -1;  // 2-word multi-sweep kernel: -1 auto, 0 one block per tile, 1 persistent pipelined (TSB_DOM_PIPE)
    int num_sms = 148;
    int m_wpl = 2;  // words per lane of the multi-sweep tiles (1: 30-word tiles for narrow lattices)
    bool coupled = false, g_coupled = false;  // chains 2j, 2j+1 share seeds (CFTP pairs): share the coins
    int collapse = 1, g_collapse = -1;  // skip sweeps followed by a sweep of the same colour (color_entry)
    int g_compact = -1;
    // run-collapsed walks (walk_compact): executed-sweep lists per chain
    std::vector<uint64_t> gkeys;  // host copies of the pushed chains' global keys
    uint32_t *xlist = nullptr;    // device [nchains][xpitch]
    int *xcnt = nullptr;          // device [nchains]
    size_t xpitch = 0;
    uint32_t *xpin[2] = {nullptr, nullptr};  // pinned staging: lists then counts
    cudaEvent_t xev[2] = {nullptr, nullptr};
    int xslot = 0;
    int tmode = 0;
    uint64_t t0 = 1ull << 52, t1 = 1ull << 52;
    uint64_t *tgrid = nullptr;
    uint64_t *seedinfo = nullptr;  // device [nchains][2]
    uint64_t *seed_pinned = nullptr;
    cudaEvent_t seed_ev = nullptr;
    uint8_t *bytes = nullptr;  // device staging for tilestate grids
    size_t bytes_cap = 0;
    int *bad = nullptr;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    // CUDA graph of kGraphSweeps sweeps, replayed by long walks
    uint64_t *step_dev = nullptr;
    uint8_t *colors = nullptr;  // [nchains][kGraphSweeps] colours of the current replay
    cudaStream_t cap_stream = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    int g_chain0 = -1, g_n = -1, g_cur = -1, g_tmode = -1;
    uint64_t g_t0 = 0, g_t1 = 0;
    int g_win0 = -1, g_winn = -1, g_winm = -1;
    // height export scratch (heights.cu), allocated on first use and owned by
    // the handle: no cudaMalloc / cudaFree per call
    int *hx_h = nullptr;        // side^2 int32: working heights / per-row prefix sums
    int *hx_flags = nullptr;    // 4 device flags
    int4 *hx_rows = nullptr;    // per row {first, last in-domain vertex, link column, ok}
    int *hx_off = nullptr;      // per row height offsets
    int hx_scan = -1;           // -1 not classified, 0 relaxation only, 1 row scan
    int hx_r0 = 0, hx_r1 = -1;  // non-empty vertex rows
    struct tsb_strip *strip = nullptr;  // device-driven strip exchange (strips.cu), if set up
    // work captured at the end of every graph replay (strip exchange), null: none
    int (*graph_tail)(tsb_domino *, cudaStream_t) = nullptr;
    int (*g_tail)(tsb_domino *, cudaStream_t) = nullptr;
};

constexpr int kGraphSweeps = 64;
constexpr int kStatePad = 2;  // == kPad in domino.cu: zero words left of every state row


// whole-grid operations are not available on row-window handles
#define TSB_FULL_ONLY(h)                                                                       \
    do {                                                                                       \
        if ((h) && (h)->windowed)                                                              \
            return tsb::fail(TSB_E_VALUE, "whole-grid operation on a row-window handle");      \
    } while (0)

namespace tsb {
int ensure_bytes(tsb_domino *h, size_t need);
int check_range(tsb_domino *h, int chain0, int n);
int push_seeds(tsb_domino *h, int n, const uint64_t *seeds);
int launch_sweep(tsb_domino *h, int chain0, int n, uint64_t step, int color_override, cudaStream_t stream,
                 const uint64_t *step_dev);
int settle(tsb_domino *h, int chain0, int n, int cur0);
int walk_steps(tsb_domino *h, int chain0, int n, uint64_t step0, uint64_t n_steps);
void strip_free(tsb_domino *h);
int strip_exchange(tsb_domino *h, cudaStream_t stream);
}  // namespace tsb
