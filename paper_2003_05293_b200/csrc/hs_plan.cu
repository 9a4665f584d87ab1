// hs_plan.cu -- host runtime + C ABI (include/holospots_b200.h).
//
// A plan owns one pupil's geometry on one device: the storage-order pixel
// list, the block-sorted dense list used by full-range passes, and a cache
// of block-sorted compressed-window lists (one per window offset of the
// CS-WGS schedule, solvers.py:212-222).  Solves are recorded once per
// (algorithm, iterations, subset, batch, spots, flags) into a CUDA graph
// and replayed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/holospots_b200.h"
#include "hs_kernels.cuh"
#include "hs_tile.cuh"
#include "hs_tilek.cuh"
#include "hs_xchg.cuh"
#include "hs_slab.cuh"
#include "hs_umma.cuh"
#include "hs_f64.cuh"

extern "C" void hs_widen_phases(const float *src, double *dst, int64_t n);  // hs_host.cu

using namespace hs;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CUDA_TRY(expr)                                                              \
    do {                                                                            \
        cudaError_t e_ = (expr);                                                    \
        if (e_ != cudaSuccess)                                                      \
            return fail(HS_ECUDA, "%s failed: %s", #expr, cudaGetErrorString(e_));  \
    } while (0)

constexpr int kColBlock = 64;  // dense layout: columns per CTA chunk
constexpr int kSplitBatch = 16;  // batches >= this record two graph branches (record_solve)
constexpr int kWidenChunksMax = 32; // pieces of a phase-code download widened as they land (HS_WIDEN_CHUNKS)
constexpr int kMaxSpots32 = 1024;   // largest n of the fp32 pixel kernels (G = 32 lanes x NL = 32)
constexpr int kMaxSpots = 4096;     // largest n overall (fp64 passes: the fold keeps 32 B per spot in smem)
// precision "auto": fp64 passes when the smallest pixel set a solve projects
// over holds fewer than this many pixels per spot
constexpr int64_t kAutoPixelsPerSpot = 512;
constexpr size_t kPass64SmemMax = 160 * 1024;

struct DevList {
    int32_t *rc = nullptr;
    float *amp = nullptr;
    int32_t *dst = nullptr;
    int64_t count = 0;
    int32_t chunk_len = 0;  // 0: choose from kTargetChunks
    int32_t sorted_rows = 0;
    // slab-ordered compressed window (hs_slab_kernel): entries (rc, amp bits)
    // chunk-major, padded per slab to kSlabL; first column of each chunk's slab
    int2 *ent = nullptr;
    int32_t *chunk_c0 = nullptr;
    int32_t sw = 0;
};

template <typename T>
int dalloc(T **p, size_t count)
{
    *p = nullptr;
    if (count == 0) return HS_OK;
    cudaError_t e = cudaMalloc((void **)p, count * sizeof(T));
    if (e != cudaSuccess)
        return fail(HS_ECUDA, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
    return HS_OK;
}

template <typename T>
void dfree(T *&p)
{
    if (p) cudaFree(p);
    p = nullptr;
}

// G lanes per pixel, NL spots per lane (a template value), np = G * NL.
// For n <= 128 the padded width is a multiple of 16 so the full-range passes
// can use the GEMM-tile kernel (ns = np / 16 spots per forward lane).
struct Config {
    int G, NL, np, spw, ns;
};

Config pick_config(int n)
{
    Config c{};
    const int choices[] = {4, 8, 10, 12, 14, 16, 32};
    if (n > kMaxSpots32) {  // fp64 passes only (NL = 0 marks "no fp32 kernel")
        c.G = 32;
        c.NL = 0;
        c.np = 32 * ((n + 31) / 32);
        c.ns = 0;
        c.spw = 1;
        return c;
    }
    if (n <= 128) {
        c.np = 16 * ((n + 15) / 16);
        c.ns = c.np / 16;
        c.G = 1;
        while (c.np / c.G > 16) c.G *= 2;
        c.NL = c.np / c.G;
    } else {
        c.ns = 0;
        c.G = 1;
        while (c.G < 32 && (n + c.G - 1) / c.G > 16) c.G *= 2;
        int nl = (n + c.G - 1) / c.G;
        nl += nl & 1;
        for (int v : choices)
            if (v >= nl) {
                c.NL = v;
                break;
            }
        c.np = c.G * c.NL;
    }
    c.spw = 32 / c.G;
    return c;
}

PassFn select_pass(const Config &c, int mode)
{
    switch (c.G) {
    case 1: return hs_select_g1(c.NL, mode);
    case 2: return hs_select_g2(c.NL, mode);
    case 4: return hs_select_g4(c.NL, mode);
    case 8: return hs_select_g8(c.NL, mode);
    case 16: return hs_select_g16(c.NL, mode);
    default: return hs_select_g32(c.NL, mode);
    }
}

size_t pass_smem(const Config &c) { return hs_pass_smem_bytes(c.G, c.NL); }

}  // namespace

struct hs_plan {
    int device = 0;
    cudaStream_t stream = nullptr;
    int side = 0;
    int64_t m = 0;
    double c1 = 0, c2 = 0, sum_amp = 0;
    std::vector<int32_t> h_rows, h_cols;
    std::vector<float> h_amp;
    std::vector<int32_t> h_index;  // grid -> storage index, -1 outside
    std::vector<int32_t> row_lo, row_hi;
    double *d_axis = nullptr;
    float *d_amp_img = nullptr;           // [side][side] amplitude, 0 outside
    int32_t *d_idx_img = nullptr;         // [side][side] storage index, -1 outside
    int32_t *d_tiles = nullptr;           // non-empty 64x64 tiles, packed (r0 << 16) | c0
    int32_t ntiles = 0;
    int32_t *d_utiles = nullptr;          // non-empty 128x64 tiles of the tcgen05 full pass
    int32_t nutiles = 0;
    bool umma_enabled = true;             // HS_UMMA=0: FFMA tiles (hs_tile) for every n
    int umma_max_n = kMaxSpots32;         // largest n on the tensor cores (HS_UMMA_MAXN, experiments)
    int num_sms = 148;
    bool pdl = false;                     // next pass launch: programmatic dependent launch
    int view0 = 0;                        // first pattern of the sub-batch being recorded
    cudaStream_t stream2 = nullptr;       // second branch of a split solve graph
    cudaStream_t stream3 = nullptr;       // tcgen05 operand-plane prep, beside the first passes
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr, prep_ev = nullptr;
    bool prep_pending = false;            // recording: full passes must wait for prep_ev
    bool pdl_enabled = true;              // HS_PDL=0 disables
    DevList storage;                      // storage order
    std::map<int, DevList> dense;         // full range, banded layout per slots-per-warp
    // compressed windows keyed (start, count, np): slab-ordered for np <= 128
    // (np > 0 in the key), else sorted (row, col) for the generic pass kernel
    std::map<std::tuple<int64_t, int64_t, int>, DevList> windows;

    // spot batch
    int batch = 0, n = 0, cap_batch = 0, cap_np = 0;
    int64_t cap_chunks = 0;
    Config cfg{};
    bool tables_valid = false;
    double *d_x = nullptr, *d_y = nullptr, *d_z = nullptr, *d_a0 = nullptr;
    double *d_theta = nullptr, *d_amp_in = nullptr;
    float2 *d_gx = nullptr, *d_gy = nullptr;
    float *d_gyp = nullptr;               // gy operand planes of the tcgen05 pass (umma_enabled)
    int64_t gyp_stride = 0;
    double *d_w = nullptr;
    float2 *d_coef = nullptr;
    float2 *d_part = nullptr;
    double2 *d_gpart = nullptr;
    int32_t *d_grp_cnt = nullptr, *d_pat_cnt = nullptr;
    int64_t part_stride = 0, gpart_stride = 0;
    int32_t cnt_stride = 0;
    int32_t *d_status = nullptr, *d_degen = nullptr, *d_qstatus = nullptr;
    double *d_fields = nullptr, *d_e = nullptr, *d_u = nullptr, *d_inten = nullptr, *d_rel = nullptr;
    double *d_phase = nullptr;   // [cap_batch][m] API scratch = d_out[0]
    double *d_out[2] = {nullptr, nullptr};  // solver phase outputs (double-buffered)
    // 4-byte phase codes (HS_WANT_PHASE32): device outputs, pinned host
    // staging, which slot holds codes, and the slot being recorded
    float *d_out32[2] = {nullptr, nullptr};
    float *h_stage32[2] = {nullptr, nullptr};
    bool slot32[2] = {false, false};
    float *rec_out32 = nullptr;
    struct WidenJob {
        const float *src;
        double *dst;
        int64_t n;
    } widen_job[2][kWidenChunksMax];      // [slot][chunk]
    int widen_chunks = 8;
    unsigned long long *d_trace = nullptr;  // HS_UMMA_TRACE probe buffer
    bool trace_next = false;
    unsigned char *d_raster = nullptr;      // [cap_batch][side][side] SLM gray rasters
    int out_slot = 0, next_slot = 0;
    cudaStream_t copy_stream = nullptr;     // D2H of phases, overlapped with solves
    cudaStream_t widen_stream[2] = {nullptr, nullptr};  // host widening of a slot's codes
    cudaEvent_t landed[2][kWidenChunksMax + 1] = {};     // a slot's code chunks (+ f64 part) reached the host
    double e2e_f64_frac = 0.375;          // hs_solve_host: share of patterns shipped as f64 (HS_E2E_F64_FRAC)
    cudaEvent_t solved[2] = {nullptr, nullptr}, copied[2] = {nullptr, nullptr};
    double *d_trace_w = nullptr, *d_trace_m = nullptr;
    int64_t trace_cap = 0;
    // fp64 passes (hs_f64.cuh): precision mode, buffers allocated on first use
    int precision_mode = HS_PREC_AUTO;    // hs_set_precision / HS_PRECISION
    bool use64 = false;                   // passes being recorded / launched run in fp64
    int last_precision = HS_PREC_FP32;    // precision of the last solve
    double *d_amp64 = nullptr;            // [m] storage-order amplitude
    double2 *d_gx64 = nullptr, *d_gy64 = nullptr;  // [B][side][np] (one allocation)
    double2 *d_coef64 = nullptr;          // [B][np]
    double2 *d_part64 = nullptr;          // [B][part_stride]
    bool tables64_valid = false;
    bool user_tables = false;             // pattern 0's tables came from hs_set_tables

    int last_alg = -1, last_iters = 0, last_flags = 0;
    // row-sharded solve state (hs_shard_*)
    struct {
        bool active = false;
        int rank = 0, world = 1, alg = 0, iters = 0, cs = 0, passes = 0;
        int64_t subset = 0, half = 1;
    } shard;
    // peer-memory exchange of the row-sharded solve (hs_shard_p2p_*)
    struct {
        char *local = nullptr;            // this rank's buffer: flags | xbuf
        size_t bytes = 0;
        int ngmax = 0;
        std::vector<char *> bases;        // [world] mapped buffer bases (own + peers)
        double2 **d_xbuf = nullptr;       // [world] device array of xbuf pointers
        unsigned long long **d_flags = nullptr;
        int32_t *d_cnt = nullptr;
        unsigned long long *d_epoch = nullptr;  // [2]: epoch counter, base of the current solve
        bool open = false;
        // captured p2p solves, keyed by (alg, iters, subset, batch, n, rank, world)
        std::map<std::tuple<int, int, int64_t, int, int, int, int>, cudaGraphExec_t> graphs;
    } xchg;
    int64_t last_launches = 0;
    std::map<std::tuple<int, int, int64_t, int, int, int>, cudaGraphExec_t> graphs;
};

namespace {

int upload_entries(const std::vector<int32_t> &rc, const std::vector<float> &amp,
                   const std::vector<int32_t> *dst, int32_t chunk_len, DevList *out)
{
    const int64_t cnt = (int64_t)rc.size();
    int r;
    if ((r = dalloc(&out->rc, cnt)) || (r = dalloc(&out->amp, cnt))) return r;
    if (dst && (r = dalloc(&out->dst, cnt))) return r;
    out->count = cnt;
    out->chunk_len = chunk_len;
    if (cnt) {
        CUDA_TRY(cudaMemcpy(out->rc, rc.data(), cnt * sizeof(int32_t), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(out->amp, amp.data(), cnt * sizeof(float), cudaMemcpyHostToDevice));
        if (dst) CUDA_TRY(cudaMemcpy(out->dst, dst->data(), cnt * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    return HS_OK;
}

void free_list(DevList &l)
{
    dfree(l.rc);
    dfree(l.amp);
    dfree(l.dst);
    dfree(l.ent);
    dfree(l.chunk_c0);
    l.count = 0;
}

inline int32_t pack_rc(int r, int c) { return (r << 16) | c; }

// Storage-order list: entry i is storage pixel i (API ranges slice it).
int build_storage(hs_plan *p)
{
    std::vector<int32_t> rc(p->m);
    for (int64_t i = 0; i < p->m; ++i) rc[i] = pack_rc(p->h_rows[i], p->h_cols[i]);
    return upload_entries(rc, p->h_amp, nullptr, 0, &p->storage);
}

// Full-range list for `spw` slots per warp: bands of 8*Rw rows split into
// blocks of kColBlock columns (one CTA chunk each); inside a block warp w owns
// rows band+w*Rw .. +Rw, and each warp step covers Rw rows x Cw columns, slot s
// at (row s % Rw, column s / Rw).  Off-aperture cells are zero-amplitude
// padding (dst = -1).
int get_dense(hs_plan *p, int spw, const DevList **out)
{
    auto it = p->dense.find(spw);
    if (it != p->dense.end()) {
        *out = &it->second;
        return HS_OK;
    }
    const int Rw = std::min(spw, 4), Cw = spw / Rw, TB = kWarps * Rw;
    std::vector<int32_t> rc, dst;
    std::vector<float> amp;
    const int side = p->side;
    for (int b0 = 0; b0 < side; b0 += TB) {
        int lo = side, hi = 0;
        for (int r = b0; r < std::min(b0 + TB, side); ++r) {
            lo = std::min(lo, p->row_lo[r]);
            hi = std::max(hi, p->row_hi[r]);
        }
        if (hi <= lo) continue;
        const int nblk = (hi - lo + kColBlock - 1) / kColBlock;
        for (int blk = 0; blk < nblk; ++blk) {
            const int c0 = lo + blk * kColBlock;
            for (int w = 0; w < kWarps; ++w)
                for (int t = 0; t < kColBlock / Cw; ++t)
                    for (int s = 0; s < spw; ++s) {
                        const int row = b0 + w * Rw + s % Rw;
                        const int col = c0 + t * Cw + s / Rw;
                        int32_t idx = -1;
                        if (row < side && col < side) idx = p->h_index[(int64_t)row * side + col];
                        rc.push_back(pack_rc(std::min(row, side - 1), std::min(col, side - 1)));
                        amp.push_back(idx >= 0 ? p->h_amp[idx] : 0.f);
                        dst.push_back(idx);
                    }
        }
    }
    DevList l;
    int r = upload_entries(rc, amp, &dst, TB * kColBlock, &l);
    if (r) return r;
    it = p->dense.emplace(spw, l).first;
    *out = &it->second;
    return HS_OK;
}

// Compressed window for the slab kernel: storage range [start, start+count)
// cut into column slabs of hs_slab_width(np) columns.  Inside a slab the
// row-runs (the window pixels of one grid row, by column) are sorted by
// length and taken two at a time: the two 16-lane pixel groups of a warp
// walk the two runs of a duo in lockstep, each run padded with
// zero-amplitude copies of its last entry to the duo's (even) length, so
// both groups change row on the same trip (no divergence on the V / flush
// path) and every pair-trip stays inside one run.  Duos are poured into
// (chunk, warp, trip) slots of kSlabP trips; a slab's last chunk is padded,
// so chunks never cross a slab.  Entry index of (chunk q, stream 2w + g,
// trip t) = q * kSlabL + (2w + g) * kSlabP + t.
int build_slab_window(hs_plan *p, int64_t start, int64_t count, int np, DevList *out)
{
    const int side = p->side;
    const int sw = hs_slab_width(np, side);
    std::vector<int64_t> keyed(count);
    for (int64_t i = 0; i < count; ++i) {
        const int64_t s = start + i;
        const int r = p->h_rows[s], c = p->h_cols[s];
        keyed[i] = ((int64_t)(c / sw) * side + r) * side + c;
    }
    std::sort(keyed.begin(), keyed.end());
    auto entry = [&](int64_t key, bool pad) {  // (row << 16 | slab-local column, amp bits)
        const int r = (int)((key / side) % side), c = (int)(key % side);
        int2 e;
        e.x = pack_rc(r, c % sw);
        e.y = 0;  // +0.0f
        if (!pad) {
            float a = p->h_amp[p->h_index[(int64_t)r * side + c]];
            memcpy(&e.y, &a, sizeof a);
        }
        return e;
    };
    std::vector<int2> ent;
    std::vector<int32_t> c0s;
    int64_t i = 0;
    while (i < count) {
        const int64_t slab = keyed[i] / ((int64_t)side * side);
        // row-runs of this slab: [begin, end) ranges of keyed
        std::vector<std::pair<int64_t, int64_t>> runs;
        while (i < count && keyed[i] / ((int64_t)side * side) == slab) {
            const int64_t b = i, row = (keyed[i] / side) % side;
            while (i < count && keyed[i] / ((int64_t)side * side) == slab && (keyed[i] / side) % side == row) ++i;
            runs.emplace_back(b, i);
        }
        std::stable_sort(runs.begin(), runs.end(), [](const std::pair<int64_t, int64_t> &x,
                                                      const std::pair<int64_t, int64_t> &y) {
            return x.second - x.first > y.second - y.first;
        });
        const size_t base = ent.size();
        int64_t slot = 0;  // trips poured so far: (chunk, warp, trip) = slot / (8P), ...
        constexpr int GR = kSlabStreams / kSlabWarps;  // pixel groups per warp
        auto place = [&](int g, const int2 &e) {
            const int64_t q = slot / ((int64_t)kSlabWarps * kSlabP);
            const int w = (int)((slot / kSlabP) % kSlabWarps), t = (int)(slot % kSlabP);
            const size_t idx = base + (size_t)q * kSlabL + (size_t)(GR * w + g) * kSlabP + t;
            if (ent.size() <= idx) ent.resize(base + (size_t)(q + 1) * kSlabL, make_int2(-1, 0));
            ent[idx] = e;
        };
        for (size_t k = 0; k < runs.size(); k += GR) {
            // even length: the kernel takes two pixels of a run per trip
            const int64_t len = (runs[k].second - runs[k].first + 1) & ~(int64_t)1;
            for (int64_t t = 0; t < len; ++t, ++slot)
                for (int g = 0; g < GR; ++g) {
                    // missing runs of the last group repeat run k (zero amplitude)
                    const auto &run = runs[k + g < runs.size() ? k + g : k];
                    const bool real = (k + g < runs.size()) && t < run.second - run.first;
                    const int64_t key = keyed[std::min(run.first + t, run.second - 1)];
                    place(g, entry(key, !real));
                }
        }
        // pad the slab's last chunk: each stream repeats its previous entry
        // (zero amplitude); streams with no entry in a warp segment repeat the
        // slab's first pixel
        const size_t total = ent.size() - base;
        for (size_t idx = 0; idx < total; ++idx) {
            if (ent[base + idx].x != -1) continue;
            const size_t t = idx % kSlabP;
            int2 e = (t > 0) ? ent[base + idx - 1] : entry(keyed[runs[0].first], true);
            e.y = 0;
            ent[base + idx] = e;
        }
        // row hint: the second entry of every pair carries (in its row bits,
        // which the kernel does not read for the column) the row of the
        // stream's next run in the chunk, so the kernel prefetches that gy
        // row a run ahead
        for (size_t sbase = base; sbase < ent.size(); sbase += kSlabP) {
            int hint = ent[sbase + kSlabP - 2].x >> 16;
            for (int t = kSlabP - 2; t >= 0; t -= 2) {
                const int row = ent[sbase + t].x >> 16;
                ent[sbase + t + 1].x = (hint << 16) | (ent[sbase + t + 1].x & 0xffff);
                if (t > 0 && (ent[sbase + t - 2].x >> 16) != row) hint = row;
            }
        }
        for (size_t q = base; q < ent.size(); q += kSlabL) c0s.push_back((int32_t)slab * sw);
    }
    int r;
    if ((r = dalloc(&out->ent, ent.size())) || (r = dalloc(&out->chunk_c0, c0s.size()))) return r;
    if (!ent.empty()) {
        CUDA_TRY(cudaMemcpy(out->ent, ent.data(), ent.size() * sizeof(int2), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(out->chunk_c0, c0s.data(), c0s.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    out->count = (int64_t)ent.size();
    out->chunk_len = kSlabL / 2;  // fold units are half-chunks (16 streams)
    out->sorted_rows = 1;
    out->sw = sw;
    return HS_OK;
}

// Compressed window: storage range [start, start+count).  np <= 128: the
// slab-ordered list of hs_slab_kernel; otherwise sorted by (row, col) for
// the generic pass kernel.
int get_window(hs_plan *p, int64_t start, int64_t count, const DevList **out)
{
    const int np = p->cfg.ns > 0 ? p->cfg.np : 0;
    auto key = std::make_tuple(start, count, np);
    auto it = p->windows.find(key);
    if (it == p->windows.end()) {
        DevList l;
        int r;
        if (np > 0) {
            r = build_slab_window(p, start, count, np, &l);
            if (r) {
                free_list(l);
                return r;
            }
        } else {
            std::vector<int64_t> keyed(count);
            for (int64_t i = 0; i < count; ++i) {
                const int64_t s = start + i;
                keyed[i] = ((int64_t)p->h_rows[s] * p->side + p->h_cols[s]) * p->m + s;
            }
            std::sort(keyed.begin(), keyed.end());
            std::vector<int32_t> rc(count);
            std::vector<float> amp(count);
            for (int64_t i = 0; i < count; ++i) {
                const int64_t s = keyed[i] % p->m;
                rc[i] = pack_rc(p->h_rows[s], p->h_cols[s]);
                amp[i] = p->h_amp[s];
            }
            r = upload_entries(rc, amp, nullptr, 0, &l);
            if (r) return r;
            l.sorted_rows = 1;
        }
        it = p->windows.emplace(key, l).first;
    }
    *out = &it->second;
    return HS_OK;
}

struct Geom {
    int32_t chunk_len, nchunks;
};

Geom geom_of(const DevList &l, int64_t count, int spw)
{
    Geom g;
    if (l.chunk_len) {
        g.chunk_len = l.chunk_len;
    } else {
        const int64_t unit = (int64_t)kWarps * spw;
        int64_t per = (count + kTargetChunks - 1) / kTargetChunks;
        per = ((per + unit - 1) / unit) * unit;
        g.chunk_len = (int32_t)std::min<int64_t>(std::max<int64_t>(per, unit), kMaxChunk);
    }
    g.nchunks = (int32_t)((count + g.chunk_len - 1) / g.chunk_len);
    return g;
}

void free_graphs(hs_plan *p)
{
    for (auto &kv : p->graphs) cudaGraphExecDestroy(kv.second);
    p->graphs.clear();
    // captured sharded solves hold the same buffers (tables, lists, partials)
    for (auto &kv : p->xchg.graphs) cudaGraphExecDestroy(kv.second);
    p->xchg.graphs.clear();
}

void free_fold(hs_plan *p)
{
    dfree(p->d_part);
    dfree(p->d_part64);
    dfree(p->d_gpart);
    dfree(p->d_grp_cnt);
    dfree(p->d_pat_cnt);
    p->cap_chunks = 0;
}

void free_batch(hs_plan *p)
{
    dfree(p->d_x); dfree(p->d_y); dfree(p->d_z); dfree(p->d_a0);
    dfree(p->d_theta); dfree(p->d_amp_in);
    dfree(p->d_gx); p->d_gy = nullptr; dfree(p->d_w); dfree(p->d_coef);
    dfree(p->d_gx64); p->d_gy64 = nullptr; dfree(p->d_coef64); p->tables64_valid = false;
    dfree(p->d_gyp); p->gyp_stride = 0;
    dfree(p->d_status); dfree(p->d_degen); dfree(p->d_qstatus);
    dfree(p->d_fields); dfree(p->d_e); dfree(p->d_u); dfree(p->d_inten); dfree(p->d_rel);
    dfree(p->d_out[1]);
    for (int k = 0; k < 2; ++k) {
        dfree(p->d_out32[k]);
        if (p->h_stage32[k]) cudaFreeHost(p->h_stage32[k]);
        p->h_stage32[k] = nullptr;
        p->slot32[k] = false;
    }
    dfree(p->d_raster);
    dfree(p->d_trace);
    dfree(p->d_phase);
    p->d_out[0] = nullptr;
    dfree(p->d_trace_w); dfree(p->d_trace_m);
    free_fold(p);
    p->cap_batch = p->cap_np = 0;
    p->trace_cap = 0;
    free_graphs(p);
}

int ensure_batch(hs_plan *p, int batch, int n)
{
    const Config cfg = pick_config(n);
    if (batch <= p->cap_batch && cfg.np <= p->cap_np) return HS_OK;
    free_batch(p);
    const int B = batch;
    const size_t bn = (size_t)B * cfg.np;
    int rc;
    if ((rc = dalloc(&p->d_x, bn)) || (rc = dalloc(&p->d_y, bn)) || (rc = dalloc(&p->d_z, bn)) ||
        (rc = dalloc(&p->d_a0, bn)) || (rc = dalloc(&p->d_theta, bn)) || (rc = dalloc(&p->d_amp_in, bn)) ||
        (rc = dalloc(&p->d_gx, (size_t)2 * B * p->side * cfg.np)) || (rc = dalloc(&p->d_w, bn)) ||
        (rc = dalloc(&p->d_coef, bn)) || (rc = dalloc(&p->d_status, B)) || (rc = dalloc(&p->d_degen, B)) ||
        (rc = dalloc(&p->d_qstatus, B)) || (rc = dalloc(&p->d_fields, bn * 2)) || (rc = dalloc(&p->d_e, B)) ||
        (rc = dalloc(&p->d_u, B)) || (rc = dalloc(&p->d_inten, bn)) || (rc = dalloc(&p->d_rel, bn)) ||
        (rc = dalloc(&p->d_phase, (size_t)B * p->m)) || (rc = dalloc(&p->d_out[1], (size_t)B * p->m)) ||
        (rc = dalloc(&p->d_raster, (size_t)B * p->side * p->side))) {
        free_batch(p);
        return rc;
    }
    if (p->umma_enabled && cfg.NL > 0) {
        p->gyp_stride = hs_umma_plane_floats(p->side, cfg.np);
        if ((rc = dalloc(&p->d_gyp, (size_t)B * p->gyp_stride))) {
            free_batch(p);
            return rc;
        }
    }
    CUDA_TRY(cudaMemset(p->d_status, 0, sizeof(int32_t) * B));
    p->d_gy = p->d_gx + (size_t)B * p->side * cfg.np;  // one allocation: gx | gy
    p->d_out[0] = p->d_phase;
    p->cap_batch = B;
    p->cap_np = cfg.np;
    return HS_OK;
}

// Fold buffers sized for `chunks` partials per pattern.
int ensure_fold(hs_plan *p, int64_t chunks)
{
    if (chunks <= p->cap_chunks && p->d_part) return HS_OK;
    free_fold(p);
    free_graphs(p);
    const int64_t groups = (chunks + kGroup - 1) / kGroup;
    const int B = p->cap_batch, np = p->cap_np;
    p->part_stride = chunks * np;
    p->gpart_stride = groups * np;
    p->cnt_stride = (int32_t)groups;
    int rc;
    if ((rc = dalloc(&p->d_part, (size_t)B * p->part_stride)) ||
        (rc = dalloc(&p->d_gpart, (size_t)B * p->gpart_stride)) ||
        (rc = dalloc(&p->d_grp_cnt, (size_t)B * groups)) || (rc = dalloc(&p->d_pat_cnt, (size_t)B)))
        return rc;
    CUDA_TRY(cudaMemset(p->d_grp_cnt, 0, sizeof(int32_t) * B * groups));
    CUDA_TRY(cudaMemset(p->d_pat_cnt, 0, sizeof(int32_t) * B));
    p->cap_chunks = chunks;
    return HS_OK;
}

int ensure_trace(hs_plan *p, int iters)
{
    const int64_t need = (int64_t)p->batch * std::max(iters, 1) * p->n;
    if (need <= p->trace_cap) return HS_OK;
    dfree(p->d_trace_w);
    dfree(p->d_trace_m);
    int rc;
    if ((rc = dalloc(&p->d_trace_w, need)) || (rc = dalloc(&p->d_trace_m, need))) return rc;
    p->trace_cap = need;
    free_graphs(p);
    return HS_OK;
}

// fp64 pass buffers (tables, coefficients, partials), allocated on first use.
int ensure64(hs_plan *p)
{
    int rc;
    if (!p->d_gx64) {
        const size_t tab = (size_t)p->cap_batch * p->side * p->cap_np;
        if ((rc = dalloc(&p->d_gx64, 2 * tab)) || (rc = dalloc(&p->d_coef64, (size_t)p->cap_batch * p->cap_np)))
            return rc;
        p->d_gy64 = p->d_gx64 + tab;
        p->tables64_valid = false;
    }
    if (!p->d_part64 && (rc = dalloc(&p->d_part64, (size_t)p->cap_batch * p->part_stride))) return rc;
    return HS_OK;
}

// 4-byte phase-code outputs and their pinned host staging (first use).
int ensure_out32(hs_plan *p)
{
    const size_t cnt = (size_t)p->cap_batch * p->m;
    for (int k = 0; k < 2; ++k) {
        int rc;
        if (!p->d_out32[k] && (rc = dalloc(&p->d_out32[k], cnt))) return rc;
        if (!p->h_stage32[k]) CUDA_TRY(cudaMallocHost(&p->h_stage32[k], cnt * sizeof(float)));
    }
    return HS_OK;
}

// Does a call projecting over at least `min_pixels` pixels per pattern run
// the fp64 passes?  (HS_PREC_AUTO rule: fewer than kAutoPixelsPerSpot pixels
// per spot, or more spots than the fp32 kernels carry.)
bool want64(const hs_plan *p, int64_t min_pixels)
{
    if (p->cfg.NL == 0) return true;
    if (p->precision_mode == HS_PREC_FP64) return true;
    if (p->precision_mode == HS_PREC_FP32) return false;
    return min_pixels < kAutoPixelsPerSpot * (int64_t)p->n;
}

UpdArgs upd_args(hs_plan *p, int act)
{
    UpdArgs u;
    memset(&u, 0, sizeof u);
    u.act = act;
    u.n = p->n;
    u.np = p->cfg.np;
    // a sub-batch view (p->view0) sees patterns view0 .. view0 + batch - 1
    const int64_t b0 = p->view0, n = p->n, np = p->cfg.np;
    u.a0 = p->d_a0 + b0 * n;
    u.w = p->d_w + b0 * np;
    if (p->use64) u.coef64 = p->d_coef64 + b0 * np;
    else u.coef = p->d_coef + b0 * np;
    u.trace_w = p->d_trace_w;
    u.trace_m = p->d_trace_m;
    u.iters = 1;
    u.status = p->d_status + b0;
    u.degen = p->d_degen + b0;
    u.qstatus = p->d_qstatus + b0;
    u.fields = p->d_fields + b0 * n * 2;
    u.inv_norm = 1.0 / (p->sum_amp * p->sum_amp);
    u.e = p->d_e + b0;
    u.u = p->d_u + b0;
    u.inten = p->d_inten + b0 * n;
    u.rel = p->d_rel + b0 * n;
    return u;
}

// Full-range tile list of the current configuration: the tcgen05 pass's
// 128 x 64 tiles (hs_umma) for 32 < n <= 1024 unless HS_UMMA=0, else the FFMA 64 x 64 tiles.
struct TileSet {
    const int32_t *d;
    int32_t n;
    bool umma;
};

TileSet tile_set(const hs_plan *p)
{
    // few spots: the per-tile fixed costs of the tensor-core pass outweigh its
    // MMA speed (config 1, N = 10: 0.181 vs 0.157 ms per solve).  Many spots:
    // the 3-term tf32 products (~2^-21 relative each, against 2^-24 for an
    // FFMA) leave the magnitudes ~5-10x further from the oracle than the
    // FFMA tiles'.  Where the fp32 passes run at all (>= 512 pixels per spot
    // under precision "auto"; fewer run the fp64 passes) that is <= 4e-6 at
    // 30 iterations (config 4: 4.1e-6 trace, 7.6e-6 intensities; tolerance
    // 1e-4; tools/accuracy_probe.py), so every n <= 1024 runs here.
    if (p->umma_enabled && p->n > 32 && p->n <= p->umma_max_n && p->d_gyp &&
        p->gyp_stride >= hs_umma_plane_floats(p->side, p->cfg.np))
        return {p->d_utiles, p->nutiles, true};
    return {p->d_tiles, p->ntiles, false};
}

int launch_tables(hs_plan *p, bool seed, bool with_prep = true)
{
    dim3 grid(p->side, p->batch);
    if (p->use64) {
        hs_tables64_kernel<<<grid, 128, 0, p->stream>>>(p->side, p->cfg.np, p->n, p->d_axis, p->c1, p->c2, p->d_x,
                                                        p->d_y, p->d_z, p->d_gx64, p->d_gy64, p->d_a0,
                                                        seed ? p->d_theta : nullptr, p->d_coef64, p->d_w);
        CUDA_TRY(cudaGetLastError());
        return HS_OK;
    }
    hs_tables_kernel<<<grid, 128, 0, p->stream>>>(p->side, p->cfg.np, p->n, p->d_axis, p->c1, p->c2, p->d_x,
                                                  p->d_y, p->d_z, p->d_gx, p->d_gy, p->d_a0,
                                                  seed ? p->d_theta : nullptr, p->d_coef, p->d_w);
    CUDA_TRY(cudaGetLastError());
    if (with_prep && p->d_gyp && tile_set(p).umma) {
        dim3 pg((unsigned)hs_umma_prep_blocks(p->side, p->cfg.np), p->batch);
        hs_umma_prep_kernel<<<pg, 256, 0, p->stream>>>(p->d_gx, p->d_gy, p->d_gyp, p->side, p->cfg.np,
                                                       (int64_t)p->side * p->cfg.np, p->gyp_stride);
        CUDA_TRY(cudaGetLastError());
    }
    return HS_OK;
}

FoldArgs fold_args(hs_plan *p, int32_t nchunks, const UpdArgs &u, int32_t lo = 0, int32_t hi = -1)
{
    FoldArgs f;
    memset(&f, 0, sizeof f);
    f.nchunks = nchunks;
    f.chunk_base = lo;
    f.chunk_end = hi < 0 ? nchunks : hi;
    f.np = p->cfg.np;
    const int64_t b0 = p->view0;
    if (p->use64) f.partials64 = p->d_part64 + b0 * p->part_stride;
    else f.partials = p->d_part + b0 * p->part_stride;
    f.part_stride = p->part_stride;
    f.gpart = p->d_gpart + b0 * p->gpart_stride;
    f.gpart_stride = p->gpart_stride;
    f.grp_cnt = p->d_grp_cnt + b0 * p->cnt_stride;
    f.pat_cnt = p->d_pat_cnt + b0;
    f.cnt_stride = p->cnt_stride;
    f.u = u;
    // trace rows are [B][iters][n]: offset by the view once the caller set iters
    return f;
}

// Launch a pass kernel on the plan stream; inside a solve graph every pass
// after the first is a programmatic dependent launch of the previous one
// (hs_pdl_launch_next / hs_pdl_wait_prev in the kernels): its CTAs launch
// and stage their static inputs while the previous pass folds.
template <typename Arg>
int launch_pass_kernel(hs_plan *p, void (*fn)(Arg), dim3 grid, dim3 block, size_t smem, const Arg &a)
{
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = p->stream;
    cudaLaunchAttribute attr[1];
    if (p->pdl && p->pdl_enabled) {
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    p->pdl = false;
    CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, a));
    return HS_OK;
}


// Full-range fused pass: tcgen05 tiles (np <= 112), FFMA GEMM tiles (hs_tile:
// n <= 128), spot-chunked FFMA tiles (hs_tilek: larger n).
int launch_tile(hs_plan *p, bool write, const UpdArgs &u, double *phase_out, int32_t lo = 0, int32_t hi = -1,
                unsigned char *raster = nullptr)
{
    const TileSet ts = tile_set(p);
    if (hi < 0) hi = ts.n;
    const Config &c = p->cfg;
    if (ts.n > p->cap_chunks) return fail(HS_ECUDA, "fold buffers too small (%d tiles)", ts.n);
    TileArgs a;
    memset(&a, 0, sizeof a);
    a.tiles = ts.d;
    a.gyp = p->d_gyp ? p->d_gyp + p->view0 * p->gyp_stride : nullptr;
    a.gyp_stride = p->gyp_stride;
    a.side = p->side;
    a.np = c.np;
    a.tab_stride = (int64_t)p->side * c.np;
    a.gx = p->d_gx + p->view0 * a.tab_stride;
    a.gy = p->d_gy + p->view0 * a.tab_stride;
    a.coef = p->d_coef + (int64_t)p->view0 * c.np;
    a.amp_img = p->d_amp_img;
    a.idx_img = p->d_idx_img;
    a.phase_out = phase_out ? phase_out + (int64_t)p->view0 * p->m : nullptr;
    a.phase_out32 = (phase_out && p->rec_out32) ? p->rec_out32 + (int64_t)p->view0 * p->m : nullptr;
    a.phase_stride = p->m;
    a.raster = raster ? raster + (int64_t)p->view0 * p->side * p->side : nullptr;
    a.f = fold_args(p, ts.n, u, lo, hi);
    a.n = p->n;
    if (p->trace_next) {
        a.trace = p->d_trace;
        p->trace_next = false;
    }
    if (hi <= lo) return HS_OK;
    dim3 grid(hi - lo, p->batch);
    if (ts.umma) {
        if (p->prep_pending) CUDA_TRY(cudaStreamWaitEvent(p->stream, p->prep_ev, 0));  // operand planes ready
        const int wmode = write ? (a.phase_out32 ? 2 : 1) : 0;
        return launch_pass_kernel(p, hs_select_umma(c.np, wmode), grid, dim3(kUThreads), hs_umma_smem_bytes(c.np),
                                  a);
    }
    const int spt = (p->n + 7) / 8;
    // n <= 128: all spots resident (hs_tile); larger n: spot-chunked (hs_tilek)
    const bool chunked = c.ns == 0;
    TileFn fn = chunked ? hs_select_tilek(write) : hs_select_tile(spt, write);
    const size_t smem = chunked ? hs_tilek_smem_bytes() : hs_tile_smem_bytes(spt, p->n);
    return launch_pass_kernel(p, fn, grid, dim3(kThreads), smem, a);
}

// Compressed-window pass over fold units [lo, hi) (half-chunks; lo, hi even)
// of a slab-ordered list.  A whole-chunk CTA streams cpc chunks (cpc | 16;
// unit ranges are fold-group-aligned), chosen to minimise waves x (cpc +
// staging cost); when even one chunk per CTA leaves SMs idle (small
// batches) each half-chunk gets its own CTA.  Every unit's partial is the
// same sum either way, so the choice never changes results.
int launch_slab(hs_plan *p, int mode, const DevList &l, int32_t nunits, const UpdArgs &u, int32_t lo, int32_t hi)
{
    const Config &c = p->cfg;
    if (mode != (PM_BWD | PM_FWD)) return fail(HS_ECUDA, "slab window lists support the fused pass only");
    if (nunits > p->cap_chunks) return fail(HS_ECUDA, "fold buffers too small (%d units)", nunits);
    if ((lo & 1) || (hi & 1)) return fail(HS_ECUDA, "slab unit range [%d, %d) splits a chunk", lo, hi);
    SlabArgs a;
    memset(&a, 0, sizeof a);
    a.ent = l.ent;
    a.chunk_c0 = l.chunk_c0;
    a.sw = l.sw;
    a.side = p->side;
    a.tab_stride = (int64_t)p->side * c.np;
    a.gx = p->d_gx + p->view0 * a.tab_stride;
    a.gy = p->d_gy + p->view0 * a.tab_stride;
    a.coef = p->d_coef + (int64_t)p->view0 * c.np;
    a.f = fold_args(p, nunits, u, lo, hi);
    if (p->trace_next) {
        a.trace = p->d_trace;
        p->trace_next = false;
    }
    const int64_t span = (hi - lo) / 2;  // chunks
    const bool half = span * p->batch * 4 < (int64_t)p->num_sms * 3;
    int best = 1;
    if (!half) {
        double best_cost = 1e300;
        for (int cpc = 1; cpc <= kGroup / 2; cpc *= 2) {
            const int64_t ctas = (span + cpc - 1) / cpc * p->batch;
            const int64_t waves = (ctas + p->num_sms - 1) / p->num_sms;
            const double cost = (double)waves * (std::min<int64_t>(cpc, span) + 0.5);
            if (cost < best_cost - 1e-9) {
                best_cost = cost;
                best = cpc;
            }
        }
    }
    static const int cpc_env = getenv("HS_SLAB_CPC") ? atoi(getenv("HS_SLAB_CPC")) : 0;
    if (!half && cpc_env > 0 && cpc_env <= kGroup / 2 && (kGroup / 2) % cpc_env == 0) best = cpc_env;
    a.cpc = best;
    const dim3 grid(half ? (unsigned)(2 * span) : (unsigned)((span + best - 1) / best), p->batch);
    return launch_pass_kernel(p, hs_select_slab(c.ns, half), grid, dim3(half ? kSlabThreads / 2 : kSlabThreads),
                              hs_slab_smem_bytes(c.np, l.sw), a);
}

// One pass over `count` entries of list `l` starting at entry `off`.
int launch_pass(hs_plan *p, int mode, const DevList &l, int64_t off, int64_t count, int64_t idx_base,
                const double *phase_in, double *phase_out, int64_t phase_stride, const UpdArgs &u,
                int32_t lo = 0, int32_t hi = -1, unsigned char *raster = nullptr)
{
    const Config &c = p->cfg;
    const Geom geo = geom_of(l, count, c.spw);
    if (count == 0) return HS_OK;
    if (geo.nchunks > p->cap_chunks) return fail(HS_ECUDA, "fold buffers too small (%d chunks)", geo.nchunks);
    PassArgs a;
    memset(&a, 0, sizeof a);
    a.rc = l.rc + off;
    a.amp = l.amp + off;
    a.dst = l.dst ? l.dst + off : nullptr;
    a.idx_base = idx_base;
    a.count = count;
    a.chunk_len = geo.chunk_len;
    a.np = c.np;
    a.nl = c.NL;
    a.sorted_rows = l.sorted_rows;
    a.raster = raster;
    a.side = p->side;
    a.tab_stride = (int64_t)p->side * c.np;
    a.gx = p->d_gx + p->view0 * a.tab_stride;
    a.gy = p->d_gy + p->view0 * a.tab_stride;
    a.coef = p->d_coef + (int64_t)p->view0 * c.np;
    a.phase_in = phase_in ? phase_in + p->view0 * phase_stride : nullptr;
    a.phase_out = phase_out ? phase_out + p->view0 * phase_stride : nullptr;
    a.phase_out32 = (phase_out && p->rec_out32) ? p->rec_out32 + p->view0 * phase_stride : nullptr;
    a.phase_stride = phase_stride;
    if (a.raster) a.raster += (int64_t)p->view0 * p->side * p->side;
    if (hi < 0) hi = geo.nchunks;
    if (hi <= lo) return HS_OK;
    if (l.sw > 0) return launch_slab(p, mode, l, geo.nchunks, u, lo, hi);
    a.f = fold_args(p, geo.nchunks, u, lo, hi);
    dim3 grid(hi - lo, p->batch);
    PassFn fn = select_pass(c, mode);
    fn<<<grid, kThreads, pass_smem(c), p->stream>>>(a);
    CUDA_TRY(cudaGetLastError());
    return HS_OK;
}

int reset_status(hs_plan *p)
{
    CUDA_TRY(cudaMemsetAsync(p->d_status, 0, sizeof(int32_t) * p->batch, p->stream));
    CUDA_TRY(cudaMemsetAsync(p->d_degen, 0, sizeof(int32_t) * p->batch, p->stream));
    CUDA_TRY(cudaMemsetAsync(p->d_qstatus, 0, sizeof(int32_t) * p->batch, p->stream));
    return HS_OK;
}

int ensure_tables(hs_plan *p)
{
    int rc;
    if (p->use64) {
        if ((rc = ensure64(p))) return rc;
        if (p->tables64_valid) return HS_OK;
        if ((rc = launch_tables(p, false))) return rc;
        p->tables64_valid = true;
        return HS_OK;
    }
    if (p->tables_valid) return HS_OK;
    if ((rc = launch_tables(p, false))) return rc;
    p->tables_valid = true;
    return HS_OK;
}

// fp64 pass over storage pixels [start, start + count) of every pattern of
// the current view (hs_pass64_kernel): chunk length ~count / kTargetChunks,
// a multiple of 8 pixels, at most kMaxChunk -- never more chunks than the
// fold buffers hold.
int launch_pass64(hs_plan *p, int mode, int64_t start, int64_t count, const double *phase_in, double *phase_out,
                  int64_t phase_stride, const UpdArgs &u, unsigned char *raster = nullptr)
{
    if (count == 0) return HS_OK;
    int64_t per = (count + kTargetChunks - 1) / kTargetChunks;
    per = std::min<int64_t>(std::max<int64_t>((per + 7) / 8 * 8, 8), kMaxChunk);
    const int32_t nchunks = (int32_t)((count + per - 1) / per);
    if (nchunks > p->cap_chunks) return fail(HS_ECUDA, "fold buffers too small (%d chunks)", nchunks);
    Pass64Args a;
    memset(&a, 0, sizeof a);
    a.rc = p->storage.rc;
    a.amp = p->d_amp64;
    a.start = start;
    a.count = count;
    a.chunk_len = (int32_t)per;
    a.n = p->n;
    a.np = p->cfg.np;
    a.tab_stride = (int64_t)p->side * p->cfg.np;
    a.gx = p->d_gx64 + p->view0 * a.tab_stride;
    a.gy = p->d_gy64 + p->view0 * a.tab_stride;
    a.coef = p->d_coef64 + (int64_t)p->view0 * p->cfg.np;
    a.phase_in = phase_in ? phase_in + p->view0 * phase_stride : nullptr;
    a.phase_out = phase_out ? phase_out + p->view0 * phase_stride : nullptr;
    a.phase_stride = phase_stride;
    a.raster = raster ? raster + (int64_t)p->view0 * p->side * p->side : nullptr;
    a.side = p->side;
    a.f = fold_args(p, nchunks, u);
    const size_t smem = hs_pass64_smem_bytes(p->cfg.np, (int)per);
    return launch_pass_kernel(p, hs_select_pass64(mode), dim3(nchunks, p->batch), dim3(kP64Threads), smem, a);
}

// The passes of one sub-batch (patterns view0 .. view0 + batch - 1) on the
// current p->stream.
int record_passes64(hs_plan *p, int alg, int iters, int64_t subset, int flags, double *out);

int record_passes(hs_plan *p, int alg, int iters, int64_t subset, int flags, double *out)
{
    if (p->use64) return record_passes64(p, alg, iters, subset, flags, out);
    int rc;
    const bool want_fields = (flags & HS_WANT_FIELDS) != 0;
    const int64_t m = p->m;
    const DevList *dense;
    if ((rc = get_dense(p, p->cfg.spw, &dense))) return rc;
    const int final_mode = want_fields ? (PM_BWD | PM_FWD | PM_WRITE) : (PM_BWD | PM_WRITE);
    const UpdArgs fin = upd_args(p, want_fields ? ACT_FINAL : ACT_NONE);
    const bool tiled = true;  // GEMM-tile full passes for every n (hs_tile / hs_tilek)
    unsigned char *raster = (flags & HS_WANT_RASTER) ? p->d_raster : nullptr;
    auto full_pass = [&](int mode, const UpdArgs &u) -> int {
        const bool wr = (mode & PM_WRITE) != 0;
        if (tiled && (mode & PM_FWD)) return launch_tile(p, wr, u, out, 0, -1, wr ? raster : nullptr);
        return launch_pass(p, mode, *dense, 0, dense->count, 0, nullptr, wr ? out : nullptr, m, u, 0, -1,
                           wr ? raster : nullptr);
    };
    if (alg == HS_ALG_RS) return full_pass(final_mode, fin);
    const int cs = (subset < m) ? std::max(0, iters - 2) : 0;
    const int64_t half = std::max<int64_t>(1, subset / 2);
    for (int j = 0; j <= iters; ++j) {
        // list of pass j: read_1 for j = 0, write_j otherwise
        const DevList *lst = nullptr;
        if (j == 0 ? cs > 0 : j <= cs) {
            const int64_t off = (j == 0) ? 0 : ((int64_t)(j - 1) * half) % (m - subset + 1);
            if ((rc = get_window(p, off, subset, &lst))) return rc;
        }
        UpdArgs u = fin;
        int mode = final_mode;
        if (j < iters) {
            u = upd_args(p, ACT_STEP);
            u.iter = j;
            u.iters = iters;
            u.trace_w += (int64_t)p->view0 * iters * p->n;  // trace rows [B][iters][n]
            u.trace_m += (int64_t)p->view0 * iters * p->n;
            mode = PM_BWD | PM_FWD;
        }
        p->pdl = (j > 0);  // pass 0 follows the tables kernel (normal dependency)
        if (lst)
            rc = launch_pass(p, mode, *lst, 0, lst->count, 0, nullptr, nullptr, 0, u);
        else
            rc = full_pass(mode, u);
        p->pdl = false;
        if (rc) return rc;
    }
    return HS_OK;
}

// The fp64 schedule: the same passes as record_passes over storage-order
// ranges (the windows of the schedule are contiguous storage ranges, so no
// lists are needed).
int record_passes64(hs_plan *p, int alg, int iters, int64_t subset, int flags, double *out)
{
    int rc;
    const bool want_fields = (flags & HS_WANT_FIELDS) != 0;
    const int64_t m = p->m;
    const int final_mode = want_fields ? (PM_BWD | PM_FWD | PM_WRITE) : (PM_BWD | PM_WRITE);
    const UpdArgs fin = upd_args(p, want_fields ? ACT_FINAL : ACT_NONE);
    unsigned char *raster = (flags & HS_WANT_RASTER) ? p->d_raster : nullptr;
    if (alg == HS_ALG_RS) return launch_pass64(p, final_mode, 0, m, nullptr, out, m, fin, raster);
    const int cs = (subset < m) ? std::max(0, iters - 2) : 0;
    const int64_t half = std::max<int64_t>(1, subset / 2);
    for (int j = 0; j <= iters; ++j) {
        int64_t off = 0, cnt = m;
        if (j == 0 ? cs > 0 : j <= cs) {
            off = (j == 0) ? 0 : ((int64_t)(j - 1) * half) % (m - subset + 1);
            cnt = subset;
        }
        UpdArgs u = fin;
        int mode = final_mode;
        if (j < iters) {
            u = upd_args(p, ACT_STEP);
            u.iter = j;
            u.iters = iters;
            u.trace_w += (int64_t)p->view0 * iters * p->n;
            u.trace_m += (int64_t)p->view0 * iters * p->n;
            mode = PM_BWD | PM_FWD;
        }
        p->pdl = (j > 0);
        rc = launch_pass64(p, mode, off, cnt, nullptr, j == iters ? out : nullptr, m, u,
                           j == iters ? raster : nullptr);
        p->pdl = false;
        if (rc) return rc;
    }
    return HS_OK;
}

// The solve schedule (solvers.py:192-235), fused: pass 0 superposes coef_0
// over read_1 and projects it; the fold of pass j applies iteration j+1's
// update (trace record j+1, coef_{j+1}); pass j >= 1 superposes coef_j over
// write_j (= read_{j+1}); the last pass writes the phase and yields the
// full-range fields of quality_report.  Batches of >= kSplitBatch patterns
// are recorded as two independent branches of the graph (halves of the
// batch on two streams): every pass ends in a partly filled wave and a
// serial fold tail, which the other branch's passes fill (+6% at B = 32).
// Patterns never interact, so the split cannot change any result.
int record_solve_passes(hs_plan *p, int alg, int iters, int64_t subset, int flags, double *out);

int record_solve(hs_plan *p, int alg, int iters, int64_t subset, int flags, double *out)
{
    int rc;
    if ((rc = reset_status(p))) return rc;
    if ((rc = launch_tables(p, true, false))) return rc;
    // the tcgen05 operand planes are first read by the full passes at the end
    // of the schedule: prepare them on a side stream beside the window passes
    if (!p->use64 && p->d_gyp && tile_set(p).umma) {
        CUDA_TRY(cudaEventRecord(p->fork_ev, p->stream));
        CUDA_TRY(cudaStreamWaitEvent(p->stream3, p->fork_ev, 0));
        dim3 pg((unsigned)hs_umma_prep_blocks(p->side, p->cfg.np), p->batch);
        hs_umma_prep_kernel<<<pg, 256, 0, p->stream3>>>(p->d_gx, p->d_gy, p->d_gyp, p->side, p->cfg.np,
                                                        (int64_t)p->side * p->cfg.np, p->gyp_stride);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaEventRecord(p->prep_ev, p->stream3));
        p->prep_pending = true;
    }
    const bool prep = p->prep_pending;
    rc = record_solve_passes(p, alg, iters, subset, flags, out);
    p->prep_pending = false;
    if (rc) return rc;
    // rejoin the side stream even when no tcgen05 pass waited on it (e.g. an
    // RS solve without fields runs its final pass on the row-run kernel)
    if (prep) CUDA_TRY(cudaStreamWaitEvent(p->stream, p->prep_ev, 0));
    return HS_OK;
}

int record_solve_passes(hs_plan *p, int alg, int iters, int64_t subset, int flags, double *out)
{
    int rc;
    if (flags & HS_WANT_RASTER)
        CUDA_TRY(cudaMemsetAsync(p->d_raster, 0, (size_t)p->batch * p->side * p->side, p->stream));
    static const bool no_split = getenv("HS_SPLIT") && atoi(getenv("HS_SPLIT")) == 0;
    if (p->batch < kSplitBatch || no_split) return record_passes(p, alg, iters, subset, flags, out);
    const int batch = p->batch, nb0 = batch / 2;
    cudaStream_t main = p->stream;
    CUDA_TRY(cudaEventRecord(p->fork_ev, main));
    CUDA_TRY(cudaStreamWaitEvent(p->stream2, p->fork_ev, 0));
    p->batch = nb0;
    rc = record_passes(p, alg, iters, subset, flags, out);
    if (!rc) {
        p->stream = p->stream2;
        p->view0 = nb0;
        p->batch = batch - nb0;
        rc = record_passes(p, alg, iters, subset, flags, out);
    }
    p->stream = main;
    p->view0 = 0;
    p->batch = batch;
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(p->join_ev, p->stream2));
    CUDA_TRY(cudaStreamWaitEvent(main, p->join_ev, 0));
    return HS_OK;
}

int check_device(hs_plan *p)
{
    CUDA_TRY(cudaSetDevice(p->device));
    return HS_OK;
}

// Compute entry points: forced fp32 cannot carry more than kMaxSpots32 spots.
int check_prec(hs_plan *p)
{
    if (p->cfg.NL == 0 && p->precision_mode == HS_PREC_FP32)
        return fail(HS_EINVAL, "precision fp32 carries at most %d spots (n = %d)", kMaxSpots32, p->n);
    return HS_OK;
}

int sync_and_check(hs_plan *p)
{
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    if (p->copy_stream) CUDA_TRY(cudaStreamSynchronize(p->copy_stream));
    for (int k = 0; k < 2; ++k)
        if (p->widen_stream[k]) CUDA_TRY(cudaStreamSynchronize(p->widen_stream[k]));
    CUDA_TRY(cudaGetLastError());
    return HS_OK;
}

}  // namespace

// ============================================================ C ABI ========
extern "C" {

const char *hs_last_error(void) { return g_err.c_str(); }

int hs_device_count(int *count)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    *count = n;
    return HS_OK;
}

int hs_max_spots(void) { return kMaxSpots; }

int hs_padded_spots(hs_plan *p) { return p->cfg.np; }

int hs_set_precision(hs_plan *p, int mode)
{
    if (mode != HS_PREC_AUTO && mode != HS_PREC_FP32 && mode != HS_PREC_FP64)
        return fail(HS_EINVAL, "precision mode %d invalid", mode);
    p->precision_mode = mode;
    return HS_OK;
}

int hs_get_precision(hs_plan *p, int *mode, int *last_solve)
{
    if (mode) *mode = p->precision_mode;
    if (last_solve) *last_solve = p->last_precision;
    return HS_OK;
}

int hs_plan_create(int device, int side, int64_t m, const int64_t *rows, const int64_t *cols,
                   const double *amplitude, const double *axis, double prism, double lens,
                   double sum_amplitude, hs_plan **out)
{
    *out = nullptr;
    if (side < 2 || side > 32767) return fail(HS_EINVAL, "side_px %d outside 2..32767", side);
    if (m < 1 || m > (int64_t)side * side) return fail(HS_EINVAL, "pixel count %lld invalid", (long long)m);
    std::unique_ptr<hs_plan> p(new hs_plan);
    p->device = device;
    CUDA_TRY(cudaSetDevice(device));
    CUDA_TRY(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        CUDA_TRY(cudaStreamCreateWithFlags(&p->widen_stream[k], cudaStreamNonBlocking));
        for (int q = 0; q <= kWidenChunksMax; ++q)
            CUDA_TRY(cudaEventCreateWithFlags(&p->landed[k][q], cudaEventDisableTiming));
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&p->stream2, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&p->stream3, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&p->prep_ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&p->fork_ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&p->join_ev, cudaEventDisableTiming));
    for (int k = 0; k < 2; ++k) {
        CUDA_TRY(cudaEventCreateWithFlags(&p->solved[k], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&p->copied[k], cudaEventDisableTiming));
    }
    p->side = side;
    p->m = m;
    p->c1 = prism;
    p->c2 = lens;
    p->sum_amp = sum_amplitude;
    p->h_rows.resize(m);
    p->h_cols.resize(m);
    p->h_amp.resize(m);
    p->h_index.assign((size_t)side * side, -1);
    p->row_lo.assign(side, side);
    p->row_hi.assign(side, 0);
    for (int64_t i = 0; i < m; ++i) {
        if (rows[i] < 0 || rows[i] >= side || cols[i] < 0 || cols[i] >= side)
            return fail(HS_EINVAL, "pixel %lld outside the grid", (long long)i);
        const int r = (int)rows[i], c = (int)cols[i];
        if (p->h_index[(size_t)r * side + c] >= 0) return fail(HS_EINVAL, "duplicate pixel (%d, %d)", r, c);
        p->h_rows[i] = r;
        p->h_cols[i] = c;
        p->h_amp[i] = (float)amplitude[i];
        p->h_index[(size_t)r * side + c] = (int32_t)i;
        p->row_lo[r] = std::min(p->row_lo[r], c);
        p->row_hi[r] = std::max(p->row_hi[r], c + 1);
    }
    int rc;
    if ((rc = dalloc(&p->d_axis, side)) || (rc = dalloc(&p->d_amp64, m))) return rc;
    CUDA_TRY(cudaMemcpy(p->d_axis, axis, sizeof(double) * side, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(p->d_amp64, amplitude, sizeof(double) * m, cudaMemcpyHostToDevice));
    if (const char *env = getenv("HS_E2E_F64_FRAC")) p->e2e_f64_frac = std::min(1.0, std::max(0.0, atof(env)));
    if (const char *env = getenv("HS_WIDEN_CHUNKS")) p->widen_chunks = std::min(kWidenChunksMax, std::max(1, atoi(env)));
    if (const char *env = getenv("HS_PRECISION")) {
        if (!strcmp(env, "fp32")) p->precision_mode = HS_PREC_FP32;
        else if (!strcmp(env, "fp64")) p->precision_mode = HS_PREC_FP64;
    }
    // exchange / host-fold update kernels: fields + scratch of up to kMaxSpots32 spots
    CUDA_TRY(cudaFuncSetAttribute((const void *)hs_gather_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double2) * 3 * kMaxSpots32)));
    CUDA_TRY(cudaFuncSetAttribute((const void *)hs_fold_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)(sizeof(double2) * 2 * kMaxSpots32)));
    for (int mode : std::initializer_list<int>{PM_BWD | PM_WRITE, PM_FWD, PM_BWD | PM_FWD, PM_BWD | PM_FWD | PM_WRITE})
        CUDA_TRY(cudaFuncSetAttribute((const void *)hs_select_pass64(mode),
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPass64SmemMax));
    if ((rc = build_storage(p.get()))) return rc;
    {
        const size_t cells = (size_t)side * side;
        std::vector<float> amp_img(cells, 0.f);
        for (int64_t i = 0; i < m; ++i) amp_img[(size_t)p->h_rows[i] * side + p->h_cols[i]] = p->h_amp[i];
        // 64-row bands; each band's tiles start at the band's first aperture
        // column (not a global 64-column grid): 276 instead of 284 tiles at 1152^2
        std::vector<int32_t> tiles;
        for (int r0 = 0; r0 < side; r0 += kTileR) {
            int lo = side, hi = 0;
            for (int r = r0; r < std::min(r0 + kTileR, side); ++r) {
                lo = std::min(lo, p->row_lo[r]);
                hi = std::max(hi, p->row_hi[r]);
            }
            for (int c0 = lo; c0 < hi; c0 += kTileC) tiles.push_back((r0 << 16) | c0);
        }
        p->ntiles = (int32_t)tiles.size();
        // the tcgen05 pass: 128-row bands, same column rule
        std::vector<int32_t> utiles;
        for (int r0 = 0; r0 < side; r0 += kUR) {
            int lo = side, hi = 0;
            for (int r = r0; r < std::min(r0 + kUR, side); ++r) {
                lo = std::min(lo, p->row_lo[r]);
                hi = std::max(hi, p->row_hi[r]);
            }
            for (int c0 = lo & ~(kUF - 1); c0 < hi; c0 += kUC) utiles.push_back((r0 << 16) | c0);  // X^T plane blocks of kUF
        }
        p->nutiles = (int32_t)utiles.size();
        if ((rc = dalloc(&p->d_amp_img, cells)) || (rc = dalloc(&p->d_idx_img, cells)) ||
            (rc = dalloc(&p->d_tiles, tiles.size())) || (rc = dalloc(&p->d_utiles, utiles.size())))
            return rc;
        CUDA_TRY(cudaMemcpy(p->d_amp_img, amp_img.data(), cells * sizeof(float), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(p->d_idx_img, p->h_index.data(), cells * sizeof(int32_t), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(p->d_tiles, tiles.data(), tiles.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(p->d_utiles, utiles.data(), utiles.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        if (const char *env = getenv("HS_UMMA")) p->umma_enabled = atoi(env) != 0;
        if (const char *env = getenv("HS_UMMA_MAXN")) p->umma_max_n = atoi(env);
        for (int np = 16; np <= kUNPC; np += 16)
            for (int w = 0; w < 3; ++w)
                CUDA_TRY(cudaFuncSetAttribute((const void *)hs_select_umma(np, w),
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)hs_umma_smem_bytes(np <= kUNPMax ? np : 1024)));
        CUDA_TRY(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, device));
        if (const char *env = getenv("HS_PDL")) p->pdl_enabled = atoi(env) != 0;
        for (int ns = 1; ns <= 8; ++ns)
            for (int h = 0; h < 4; ++h)
                CUDA_TRY(cudaFuncSetAttribute((const void *)hs_select_slab(ns, (h & 1) != 0, h >= 2),
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              kSlabSmemBudget));  // process-wide cap: never lower it per plan
        for (int w = 0; w < 2; ++w)
            CUDA_TRY(cudaFuncSetAttribute((const void *)hs_select_tilek(w != 0),
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hs_tilek_smem_bytes()));
        for (int spt = 1; spt <= 16; ++spt)
            for (int w = 0; w < 2; ++w)
                CUDA_TRY(cudaFuncSetAttribute((const void *)hs_select_tile(spt, w != 0),
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)hs_tile_smem_bytes(spt, 8 * spt)));
    }
    const int modes[4] = {PM_BWD | PM_WRITE, PM_FWD, PM_BWD | PM_FWD, PM_BWD | PM_FWD | PM_WRITE};
    const int gs[6] = {1, 2, 4, 8, 16, 32};
    const int nls[7] = {4, 8, 10, 12, 14, 16, 32};
    for (int G : gs)
        for (int NL : nls) {
            if (NL == 32 && G != 32) continue;
            Config c{G, NL, G * NL, 32 / G, 0};
            for (int mode : modes)
                CUDA_TRY(cudaFuncSetAttribute((const void *)select_pass(c, mode),
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pass_smem(c)));
        }
    *out = p.release();
    return HS_OK;
}

void hs_plan_destroy(hs_plan *p)
{
    if (!p) return;
    cudaSetDevice(p->device);
    hs_shard_p2p_close(p);
    cudaStreamSynchronize(p->stream);
    cudaStreamSynchronize(p->copy_stream);
    for (int k = 0; k < 2; ++k) cudaStreamSynchronize(p->widen_stream[k]);
    free_batch(p);
    free_list(p->storage);
    for (auto &kv : p->dense) free_list(kv.second);
    for (auto &kv : p->windows) free_list(kv.second);
    dfree(p->d_axis);
    dfree(p->d_amp64);
    dfree(p->d_amp_img);
    dfree(p->d_idx_img);
    dfree(p->d_tiles);
    dfree(p->d_utiles);
    cudaStreamDestroy(p->stream);
    cudaStreamDestroy(p->copy_stream);
    for (int k = 0; k < 2; ++k) {
        cudaStreamDestroy(p->widen_stream[k]);
        for (int q = 0; q <= kWidenChunksMax; ++q) cudaEventDestroy(p->landed[k][q]);
    }
    cudaStreamDestroy(p->stream2);
    cudaStreamDestroy(p->stream3);
    cudaEventDestroy(p->prep_ev);
    cudaEventDestroy(p->fork_ev);
    cudaEventDestroy(p->join_ev);
    for (int k = 0; k < 2; ++k) {
        cudaEventDestroy(p->solved[k]);
        cudaEventDestroy(p->copied[k]);
    }
    delete p;
}

int hs_set_spots(hs_plan *p, int batch, int n, const double *x, const double *y, const double *z,
                 const double *a0)
{
    if (batch < 1) return fail(HS_EINVAL, "batch must be >= 1");
    if (n < 1 || n > hs_max_spots()) return fail(HS_EINVAL, "spot count %d outside 1..%d", n, hs_max_spots());
    int rc;
    if ((rc = check_device(p))) return rc;
    if ((rc = ensure_batch(p, batch, n))) return rc;
    if (p->batch != batch || p->n != n) free_graphs(p);
    p->batch = batch;
    p->n = n;
    p->cfg = pick_config(n);
    const DevList *dense;
    if ((rc = get_dense(p, p->cfg.spw, &dense))) return rc;
    // slab windows: two fold units per kSlabL-entry chunk, plus one padded
    // tail chunk per slab
    const int64_t slab_chunks =
        p->cfg.ns > 0 ? 2 * (p->m / kSlabL + p->side / hs_slab_width(p->cfg.np, p->side) + 2) : 0;
    const int64_t chunks = std::max<int64_t>({(int64_t)geom_of(*dense, dense->count, p->cfg.spw).nchunks,
                                              (int64_t)kTargetChunks + 1, p->m / kMaxChunk + 2,
                                              (int64_t)p->ntiles, (int64_t)p->nutiles, slab_chunks});
    if ((rc = ensure_fold(p, chunks))) return rc;
    const size_t bytes = sizeof(double) * (size_t)batch * n;
    CUDA_TRY(cudaMemcpyAsync(p->d_x, x, bytes, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(p->d_y, y, bytes, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(p->d_z, z, bytes, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(p->d_a0, a0, bytes, cudaMemcpyHostToDevice, p->stream));
    p->tables_valid = false;
    p->tables64_valid = false;
    p->user_tables = false;
    return HS_OK;
}

// Test hook: one weight / theta update (hs_update, the device restatement of
// rebalance_weights, solvers.py:104-129) on caller fields -- the reference's
// floor-and-flag, all-zero and divergence cases run through the device code.
static __global__ void __launch_bounds__(kThreads) hs_update_probe_kernel(UpdArgs u, const double2 *E_in)
{
    __shared__ double dbuf[kThreads];
    __shared__ int ibuf[kThreads];
    extern __shared__ double2 Es[];     // [np] fields + [2 np] scratch
    for (int k = threadIdx.x; k < u.np; k += kThreads) Es[k] = k < u.n ? E_in[k] : make_double2(0.0, 0.0);
    __syncthreads();
    hs_update(u, 0, Es, reinterpret_cast<double *>(Es + u.np), dbuf, ibuf);
}

int hs_debug_update(int n, const double *w_in, const double *fields, double *w_out, double *mags_out,
                    int *status, int *degenerate)
{
    if (n < 1 || n > kMaxSpots) return fail(HS_EINVAL, "spot count %d outside 1..%d", n, kMaxSpots);
    const int np = 32 * ((n + 31) / 32);
    double *buf = nullptr;
    int32_t *ibuf = nullptr;
    // w [np] | a0 [n] | trace_w [n] | trace_m [n] | E [2 np] | coef64 [2 np]
    int rc;
    if ((rc = dalloc(&buf, (size_t)np + 3 * n + 4 * np)) || (rc = dalloc(&ibuf, 3))) {
        if (buf) cudaFree(buf);
        return rc;
    }
    double *w = buf, *a0 = w + np, *tw = a0 + n, *tm = tw + n, *E = tm + n, *coef = E + 2 * np;
    std::vector<double> ones(n, 1.0);
    CUDA_TRY(cudaMemset(buf, 0, sizeof(double) * ((size_t)np + 3 * n + 4 * np)));
    CUDA_TRY(cudaMemset(ibuf, 0, sizeof(int32_t) * 3));
    CUDA_TRY(cudaMemcpy(w, w_in, sizeof(double) * n, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(a0, ones.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(E, fields, sizeof(double) * 2 * n, cudaMemcpyHostToDevice));
    UpdArgs u;
    memset(&u, 0, sizeof u);
    u.act = ACT_STEP;
    u.n = n;
    u.np = np;
    u.a0 = a0;
    u.w = w;
    u.coef64 = reinterpret_cast<double2 *>(coef);
    u.trace_w = tw;
    u.trace_m = tm;
    u.iters = 1;
    u.status = ibuf;
    u.degen = ibuf + 1;
    u.qstatus = ibuf + 2;
    hs_update_probe_kernel<<<1, kThreads, 32 * np>>>(u, reinterpret_cast<const double2 *>(E));
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    int32_t st[3];
    CUDA_TRY(cudaMemcpy(st, ibuf, sizeof st, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(w_out, tw, sizeof(double) * n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(mags_out, tm, sizeof(double) * n, cudaMemcpyDeviceToHost));
    cudaFree(buf);
    cudaFree(ibuf);
    *status = st[0];
    *degenerate = st[1] != 0;
    return HS_OK;
}

int hs_set_tables(hs_plan *p, int n, const double *gx_re, const double *gx_im, const double *gy_re,
                  const double *gy_im)
{
    if (p->batch != 1) return fail(HS_EINVAL, "hs_set_tables needs a single-pattern spot set");
    if (n != p->n) return fail(HS_EINVAL, "table spot count %d != spot count %d", n, p->n);
    int rc;
    if ((rc = check_device(p)) || (rc = ensure64(p))) return rc;
    const size_t cnt = (size_t)p->side * n;
    double *tmp = nullptr;
    if ((rc = dalloc(&tmp, 4 * cnt))) return rc;
    const double *src[4] = {gx_re, gx_im, gy_re, gy_im};
    for (int q = 0; q < 4; ++q)
        CUDA_TRY(cudaMemcpyAsync(tmp + q * cnt, src[q], sizeof(double) * cnt, cudaMemcpyHostToDevice, p->stream));
    hs_pack_tables_kernel<<<p->side, 128, 0, p->stream>>>(p->side, n, p->cfg.np, tmp, tmp + cnt, p->d_gx64, p->d_gx);
    hs_pack_tables_kernel<<<p->side, 128, 0, p->stream>>>(p->side, n, p->cfg.np, tmp + 2 * cnt, tmp + 3 * cnt,
                                                          p->d_gy64, p->d_gy);
    CUDA_TRY(cudaGetLastError());
    rc = sync_and_check(p);
    cudaFree(tmp);
    if (rc) return rc;
    p->tables_valid = p->tables64_valid = true;
    p->user_tables = true;
    return HS_OK;
}

int hs_get_tables(hs_plan *p, double *gx_re, double *gx_im, double *gy_re, double *gy_im)
{
    if (p->batch < 1) return fail(HS_EINVAL, "no spots set");
    int rc;
    if ((rc = check_device(p))) return rc;
    p->use64 = true;
    rc = ensure_tables(p);
    p->use64 = false;
    if (rc) return rc;
    const size_t cnt = (size_t)p->side * p->n;
    double *tmp = nullptr;
    if ((rc = dalloc(&tmp, 4 * cnt))) return rc;
    hs_unpack_tables_kernel<<<p->side, 128, 0, p->stream>>>(p->side, p->n, p->cfg.np, p->d_gx64, tmp, tmp + cnt);
    hs_unpack_tables_kernel<<<p->side, 128, 0, p->stream>>>(p->side, p->n, p->cfg.np, p->d_gy64, tmp + 2 * cnt,
                                                            tmp + 3 * cnt);
    double *dst[4] = {gx_re, gx_im, gy_re, gy_im};
    for (int q = 0; q < 4; ++q)
        CUDA_TRY(cudaMemcpyAsync(dst[q], tmp + q * cnt, sizeof(double) * cnt, cudaMemcpyDeviceToHost, p->stream));
    rc = sync_and_check(p);
    cudaFree(tmp);
    return rc;
}

static int check_range(hs_plan *p, int64_t start, int64_t stop)
{
    if (p->batch < 1) return fail(HS_EINVAL, "no spots set");
    if (start < 0 || start > stop || stop > p->m)
        return fail(HS_EINVAL, "pixel range (%lld, %lld) outside 0..%lld", (long long)start, (long long)stop,
                    (long long)p->m);
    return HS_OK;
}

// API calls: precision of the passes of this call (want64 over the whole
// pupil), reset when the call returns.
struct Use64 {
    hs_plan *p;
    Use64(hs_plan *pl, int64_t pixels) : p(pl)
    {
        p->use64 = want64(p, pixels);
        if (p->use64 && ensure64(p)) p->use64 = false;  // allocation failure surfaces in ensure_tables
    }
    ~Use64() { p->use64 = false; }
};

// API passes act on pattern 0 only.
struct OnePattern {
    hs_plan *p;
    int saved;
    explicit OnePattern(hs_plan *pl) : p(pl), saved(pl->batch) { p->batch = 1; }
    ~OnePattern() { p->batch = saved; }
};

int hs_superpose(hs_plan *p, const double *amplitude, const double *theta, int64_t start, int64_t stop,
                 double *out)
{
    int rc;
    if ((rc = check_range(p, start, stop)) || (rc = check_device(p)) || (rc = check_prec(p))) return rc;
    Use64 prec(p, p->m);
    if ((rc = ensure_tables(p)) || (rc = reset_status(p))) return rc;
    if (stop == start) return HS_OK;
    const size_t bytes = sizeof(double) * p->n;
    CUDA_TRY(cudaMemcpyAsync(p->d_amp_in, amplitude, bytes, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(p->d_theta, theta, bytes, cudaMemcpyHostToDevice, p->stream));
    {
        OnePattern one(p);
        hs_seed_kernel<<<1, 256, 0, p->stream>>>(p->n, p->cfg.np, p->d_amp_in, p->d_theta, p->d_coef, nullptr,
                                                 p->use64 ? p->d_coef64 : nullptr);
        CUDA_TRY(cudaGetLastError());
        if (p->use64)
            rc = launch_pass64(p, PM_BWD | PM_WRITE, start, stop - start, nullptr, p->d_phase - start, 0,
                               upd_args(p, ACT_NONE));
        else
            rc = launch_pass(p, PM_BWD | PM_WRITE, p->storage, start, stop - start, 0, nullptr, p->d_phase, 0,
                             upd_args(p, ACT_NONE));
        if (rc) return rc;
    }
    CUDA_TRY(cudaMemcpyAsync(out, p->d_phase, sizeof(double) * (stop - start), cudaMemcpyDeviceToHost, p->stream));
    return sync_and_check(p);
}

int hs_forward(hs_plan *p, const double *phase, int64_t start, int64_t stop, double *fields)
{
    int rc;
    if ((rc = check_range(p, start, stop)) || (rc = check_device(p)) || (rc = check_prec(p))) return rc;
    Use64 prec(p, p->m);
    if ((rc = ensure_tables(p)) || (rc = reset_status(p))) return rc;
    if (stop == start) {  // kernels.py:234-235
        memset(fields, 0, sizeof(double) * 2 * p->n);
        return HS_OK;
    }
    CUDA_TRY(cudaMemcpyAsync(p->d_phase, phase, sizeof(double) * p->m, cudaMemcpyHostToDevice, p->stream));
    {
        OnePattern one(p);
        if (p->use64)
            rc = launch_pass64(p, PM_FWD, start, stop - start, p->d_phase, nullptr, 0, upd_args(p, ACT_FIELDS));
        else
            rc = launch_pass(p, PM_FWD, p->storage, start, stop - start, start, p->d_phase, nullptr, 0,
                             upd_args(p, ACT_FIELDS));
        if (rc) return rc;
    }
    CUDA_TRY(cudaMemcpyAsync(fields, p->d_fields, sizeof(double) * 2 * p->n, cudaMemcpyDeviceToHost, p->stream));
    return sync_and_check(p);
}

int hs_quality(hs_plan *p, const double *phase, double *e, double *u, double *intensities, double *relative,
               double *fields)
{
    if (!(p->sum_amp > 0.0)) return fail(HS_EZEROILLUM, "pupil carries no illumination");
    int rc;
    if ((rc = check_range(p, 0, p->m)) || (rc = check_device(p)) || (rc = check_prec(p))) return rc;
    Use64 prec(p, p->m);
    if ((rc = ensure_tables(p)) || (rc = reset_status(p))) return rc;
    const DevList *dense;
    if ((rc = get_dense(p, p->cfg.spw, &dense))) return rc;
    CUDA_TRY(cudaMemcpyAsync(p->d_phase, phase, sizeof(double) * p->m, cudaMemcpyHostToDevice, p->stream));
    {
        OnePattern one(p);
        if (p->use64)
            rc = launch_pass64(p, PM_FWD, 0, p->m, p->d_phase, nullptr, 0, upd_args(p, ACT_FINAL));
        else
            rc = launch_pass(p, PM_FWD, *dense, 0, dense->count, 0, p->d_phase, nullptr, 0, upd_args(p, ACT_FINAL));
        if (rc) return rc;
    }
    int32_t qs = 0;
    CUDA_TRY(cudaMemcpyAsync(e, p->d_e, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaMemcpyAsync(u, p->d_u, sizeof(double), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaMemcpyAsync(&qs, p->d_qstatus, sizeof(int32_t), cudaMemcpyDeviceToHost, p->stream));
    if (intensities)
        CUDA_TRY(cudaMemcpyAsync(intensities, p->d_inten, sizeof(double) * p->n, cudaMemcpyDeviceToHost, p->stream));
    if (relative)
        CUDA_TRY(cudaMemcpyAsync(relative, p->d_rel, sizeof(double) * p->n, cudaMemcpyDeviceToHost, p->stream));
    if (fields)
        CUDA_TRY(cudaMemcpyAsync(fields, p->d_fields, sizeof(double) * 2 * p->n, cudaMemcpyDeviceToHost, p->stream));
    if ((rc = sync_and_check(p))) return rc;
    if (qs) return fail(HS_EUNDEFINED, "all spot intensities are zero");
    return HS_OK;
}

int hs_probe(hs_plan *p, const double *phase, int64_t npts, const double *xyz, int batch, double *out)
{
    if (!(p->sum_amp > 0.0)) return fail(HS_EZEROILLUM, "pupil carries no illumination");
    if (batch < 1 || batch > hs_max_spots()) return fail(HS_EINVAL, "probe batch %d outside 1..%d", batch, hs_max_spots());
    if (npts < 0) return fail(HS_EINVAL, "negative probe count");
    int rc;
    if ((rc = check_device(p))) return rc;
    bool uploaded = false;
    std::vector<double> x, y, z, a;
    for (int64_t lo = 0; lo < npts; lo += batch) {
        const int n = (int)std::min<int64_t>(batch, npts - lo);
        x.resize(n); y.resize(n); z.resize(n); a.assign(n, 1.0);
        for (int k = 0; k < n; ++k) {
            x[k] = xyz[(lo + k) * 3 + 0];
            y[k] = xyz[(lo + k) * 3 + 1];
            z[k] = xyz[(lo + k) * 3 + 2];
        }
        if ((rc = hs_set_spots(p, 1, n, x.data(), y.data(), z.data(), a.data())) || (rc = check_prec(p))) return rc;
        Use64 prec(p, p->m);
        if ((rc = ensure_tables(p)) || (rc = reset_status(p))) return rc;
        if (!uploaded) {
            CUDA_TRY(cudaMemcpyAsync(p->d_phase, phase, sizeof(double) * p->m, cudaMemcpyHostToDevice, p->stream));
            uploaded = true;
        }
        if (p->use64) {
            rc = launch_pass64(p, PM_FWD, 0, p->m, p->d_phase, nullptr, 0, upd_args(p, ACT_FINAL));
        } else {
            const DevList *dense;
            if ((rc = get_dense(p, p->cfg.spw, &dense))) return rc;
            rc = launch_pass(p, PM_FWD, *dense, 0, dense->count, 0, p->d_phase, nullptr, 0, upd_args(p, ACT_FINAL));
        }
        if (rc) return rc;
        CUDA_TRY(cudaMemcpyAsync(out + lo, p->d_inten, sizeof(double) * n, cudaMemcpyDeviceToHost, p->stream));
    }
    return sync_and_check(p);
}

static int solve_into(hs_plan *p, int alg, int iters, int64_t subset, const double *theta0, int flags, int slot);

static void CUDART_CB widen_job_fn(void *arg)
{
    const auto *job = static_cast<const hs_plan::WidenJob *>(arg);
    hs_widen_phases(job->src, job->dst, job->n);
}

int hs_solve_async(hs_plan *p, int alg, int iters, int64_t subset, const double *theta0, int flags)
{
    return solve_into(p, alg, iters, subset, theta0, flags, 0);
}

static int solve_into(hs_plan *p, int alg, int iters, int64_t subset, const double *theta0, int flags, int slot)
{
    if (p->batch < 1) return fail(HS_EINVAL, "no spots set");
    if (alg != HS_ALG_RS && alg != HS_ALG_WGS && alg != HS_ALG_CSWGS)
        return fail(HS_EINVAL, "unknown algorithm %d", alg);
    if (alg == HS_ALG_RS) {
        iters = 0;
        subset = p->m;
    } else {
        if (iters < 1) return fail(HS_EINVAL, "iterations must be >= 1");
        if (alg == HS_ALG_CSWGS && iters < 2) return fail(HS_EINVAL, "cswgs needs iterations >= 2");
        if (alg == HS_ALG_WGS) subset = p->m;
        if (subset < 1 || subset > p->m) return fail(HS_EINVAL, "subset size %lld outside 1..M", (long long)subset);
    }
    if ((flags & HS_WANT_FIELDS) && !(p->sum_amp > 0.0)) return fail(HS_EZEROILLUM, "pupil carries no illumination");
    int rc;
    if ((rc = check_device(p)) || (rc = check_prec(p)) || (rc = ensure_trace(p, iters))) return rc;
    // precision of this solve: the smallest pixel set it projects over
    const bool windows = alg != HS_ALG_RS && subset < p->m && iters > 2;
    p->use64 = want64(p, windows ? subset : p->m);
    struct Reset64 {
        hs_plan *p;
        ~Reset64() { p->use64 = false; }
    } reset64{p};
    if (p->use64 && (rc = ensure64(p))) return rc;
    // fp32 solves may store 4-byte phase codes (the fp64 passes store f64)
    const bool codes = (flags & HS_WANT_PHASE32) && !p->use64;
    if (!codes) flags &= ~HS_WANT_PHASE32;
    if (codes && (rc = ensure_out32(p))) return rc;
    // host-side list building happens outside graph capture
    const DevList *l;
    if (!p->use64 && (rc = get_dense(p, p->cfg.spw, &l))) return rc;
    if (!p->use64 && windows) {
        const int64_t half = std::max<int64_t>(1, subset / 2);
        for (int j = 0; j <= iters - 2; ++j) {
            const int64_t off = j == 0 ? 0 : ((int64_t)(j - 1) * half) % (p->m - subset + 1);
            if ((rc = get_window(p, off, subset, &l))) return rc;
        }
    }
    const size_t bytes = sizeof(double) * (size_t)p->batch * p->n;
    CUDA_TRY(cudaMemcpyAsync(p->d_theta, theta0, bytes, cudaMemcpyHostToDevice, p->stream));
    auto key = std::make_tuple(alg, iters, subset, flags | (slot << 8) | ((int)p->use64 << 12), p->batch, p->n);
    auto it = p->graphs.find(key);
    if (it == p->graphs.end()) {
        cudaGraph_t graph;
        CUDA_TRY(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
        p->rec_out32 = codes ? p->d_out32[slot] : nullptr;
        rc = record_solve(p, alg, iters, subset, flags, p->d_out[slot]);
        p->rec_out32 = nullptr;
        cudaError_t ce = cudaStreamEndCapture(p->stream, &graph);
        if (rc) return rc;
        if (ce != cudaSuccess) return fail(HS_ECUDA, "graph capture failed: %s", cudaGetErrorString(ce));
        cudaGraphExec_t exec;
        ce = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) return fail(HS_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(ce));
        it = p->graphs.emplace(key, exec).first;
    }
    CUDA_TRY(cudaGraphLaunch(it->second, p->stream));
    p->out_slot = slot;
    p->slot32[slot] = codes;
    if (p->user_tables) {  // the solve rebuilt the tables from the spots
        p->tables_valid = p->tables64_valid = false;
        p->user_tables = false;
    }
    if (p->use64) p->tables64_valid = true;
    else p->tables_valid = true;
    p->last_precision = p->use64 ? HS_PREC_FP64 : HS_PREC_FP32;
    p->last_alg = alg;
    p->last_iters = iters;
    p->last_flags = flags;
    {   // tables(+seed) [+ tcgen05 operand planes] + passes, per graph branch
        static const bool no_split = getenv("HS_SPLIT") && atoi(getenv("HS_SPLIT")) == 0;
        const int branches = (p->batch >= kSplitBatch && !no_split) ? 2 : 1;
        const int prep = (!p->use64 && p->d_gyp && tile_set(p).umma) ? 1 : 0;
        p->last_launches = 1 + prep + (int64_t)branches * ((alg == HS_ALG_RS) ? 1 : iters + 1);
    }
    return HS_OK;
}

int hs_solve(hs_plan *p, int alg, int iters, int64_t subset, const double *theta0, int flags)
{
    int rc = hs_solve_async(p, alg, iters, subset, theta0, flags);
    if (rc) return rc;
    return sync_and_check(p);
}

int hs_sync(hs_plan *p)
{
    int rc;
    if ((rc = check_device(p))) return rc;
    return sync_and_check(p);
}

int hs_get_status(hs_plan *p, int32_t *status, int32_t *degenerate)
{
    int rc;
    if ((rc = check_device(p))) return rc;
    if (status)
        CUDA_TRY(cudaMemcpyAsync(status, p->d_status, sizeof(int32_t) * p->batch, cudaMemcpyDeviceToHost, p->stream));
    if (degenerate)
        CUDA_TRY(cudaMemcpyAsync(degenerate, p->d_degen, sizeof(int32_t) * p->batch, cudaMemcpyDeviceToHost,
                                 p->stream));
    return sync_and_check(p);
}

int hs_get_trace(hs_plan *p, double *weights, double *mags)
{
    int rc;
    if ((rc = check_device(p))) return rc;
    const size_t cnt = (size_t)p->batch * p->last_iters * p->n;
    if (cnt) {
        if (weights)
            CUDA_TRY(cudaMemcpyAsync(weights, p->d_trace_w, sizeof(double) * cnt, cudaMemcpyDeviceToHost, p->stream));
        if (mags)
            CUDA_TRY(cudaMemcpyAsync(mags, p->d_trace_m, sizeof(double) * cnt, cudaMemcpyDeviceToHost, p->stream));
    }
    return sync_and_check(p);
}

int hs_get_phase(hs_plan *p, int first, int count, double *phase)
{
    if (first < 0 || count < 0 || first + count > p->batch) return fail(HS_EINVAL, "pattern range invalid");
    int rc;
    if ((rc = check_device(p))) return rc;
    if (!count) return sync_and_check(p);
    const int slot = p->out_slot;
    if (p->slot32[slot]) {  // 4-byte codes: widened to the identical f64 phases on the device
        const size_t off = (size_t)first * p->m;
        hs_widen_codes_kernel<<<4 * p->num_sms, 256, 0, p->stream>>>(p->d_out32[slot] + off, p->d_out[slot] + off,
                                                                      (int64_t)count * p->m);
        CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaMemcpyAsync(phase, p->d_out[slot] + (size_t)first * p->m, sizeof(double) * count * p->m,
                             cudaMemcpyDeviceToHost, p->stream));
    return sync_and_check(p);
}

int hs_get_quality(hs_plan *p, double *e, double *u, double *intensities, double *relative, double *fields)
{
    if (!(p->last_flags & HS_WANT_FIELDS)) return fail(HS_EINVAL, "last solve did not compute fields");
    int rc;
    if ((rc = check_device(p))) return rc;
    const size_t B = p->batch, bn = (size_t)p->batch * p->n;
    if (e) CUDA_TRY(cudaMemcpyAsync(e, p->d_e, sizeof(double) * B, cudaMemcpyDeviceToHost, p->stream));
    if (u) CUDA_TRY(cudaMemcpyAsync(u, p->d_u, sizeof(double) * B, cudaMemcpyDeviceToHost, p->stream));
    if (intensities)
        CUDA_TRY(cudaMemcpyAsync(intensities, p->d_inten, sizeof(double) * bn, cudaMemcpyDeviceToHost, p->stream));
    if (relative)
        CUDA_TRY(cudaMemcpyAsync(relative, p->d_rel, sizeof(double) * bn, cudaMemcpyDeviceToHost, p->stream));
    if (fields)
        CUDA_TRY(cudaMemcpyAsync(fields, p->d_fields, sizeof(double) * 2 * bn, cudaMemcpyDeviceToHost, p->stream));
    return sync_and_check(p);
}

// Pipelined end-to-end call: spot/theta upload, solve into phase buffer
// `slot` (alternating), e/u download on the solve stream, and the phase
// download on the copy stream -- it overlaps the next call's solve.  The
// write-after-read on a phase buffer is ordered by events.
int hs_solve_host_async(hs_plan *p, int alg, int iters, int64_t subset, int batch, int n, const double *x,
                        const double *y, const double *z, const double *a0, const double *theta0, double *phase,
                        double *e, double *u)
{
    int rc;
    if ((rc = hs_set_spots(p, batch, n, x, y, z, a0))) return rc;
    const int slot = p->next_slot;
    CUDA_TRY(cudaStreamWaitEvent(p->stream, p->copied[slot], 0));
    static const bool no_codes = getenv("HS_E2E_CODES") && atoi(getenv("HS_E2E_CODES")) == 0;
    if ((rc = solve_into(p, alg, iters, subset, theta0, HS_WANT_FIELDS | (no_codes ? 0 : HS_WANT_PHASE32), slot)))
        return rc;
    if (e) CUDA_TRY(cudaMemcpyAsync(e, p->d_e, sizeof(double) * batch, cudaMemcpyDeviceToHost, p->stream));
    if (u) CUDA_TRY(cudaMemcpyAsync(u, p->d_u, sizeof(double) * batch, cudaMemcpyDeviceToHost, p->stream));
    if (!(phase && p->slot32[slot])) {
        CUDA_TRY(cudaEventRecord(p->solved[slot], p->stream));
        CUDA_TRY(cudaStreamWaitEvent(p->copy_stream, p->solved[slot], 0));
    }
    const size_t cnt = (size_t)batch * p->m;
    if (phase && p->slot32[slot]) {
        // The phases leave the device two ways at once, splitting the work
        // between the host link and the host cores (either alone is slower
        // than the solve; tools/e2e_probe.py):
        //  * patterns [0, nb64): widened to f64 on the device (hs_widen_codes,
        //    bit-identical) and copied as f64 into the caller's buffer;
        //  * patterns [nb64, batch): 4-byte codes copied to pinned staging in
        //    widen_chunks pieces, each widened on the host threads (a host
        //    function on the slot's widen stream) as soon as it lands.
        // Both overlap the next call's solve.
        const int nb64 = (int)std::lround(p->e2e_f64_frac * batch);
        const size_t c64 = (size_t)nb64 * p->m, c32 = cnt - c64;
        if (nb64 > 0) {
            hs_widen_codes_kernel<<<4 * p->num_sms, 256, 0, p->stream>>>(p->d_out32[slot], p->d_out[slot],
                                                                          (int64_t)c64);
            CUDA_TRY(cudaGetLastError());
        }
        CUDA_TRY(cudaEventRecord(p->solved[slot], p->stream));
        CUDA_TRY(cudaStreamWaitEvent(p->copy_stream, p->solved[slot], 0));
        const int nwc = p->widen_chunks;
        for (int q = 0; q < nwc && c32 > 0; ++q) {
            const size_t lo = c64 + c32 * q / nwc, hi = c64 + c32 * (q + 1) / nwc;
            CUDA_TRY(cudaMemcpyAsync(p->h_stage32[slot] + lo, p->d_out32[slot] + lo, sizeof(float) * (hi - lo),
                                     cudaMemcpyDeviceToHost, p->copy_stream));
            CUDA_TRY(cudaEventRecord(p->landed[slot][q], p->copy_stream));
            CUDA_TRY(cudaStreamWaitEvent(p->widen_stream[slot], p->landed[slot][q], 0));
            p->widen_job[slot][q] = {p->h_stage32[slot] + lo, phase + lo, (int64_t)(hi - lo)};
            CUDA_TRY(cudaLaunchHostFunc(p->widen_stream[slot], widen_job_fn, &p->widen_job[slot][q]));
        }
        if (c64 > 0)
            CUDA_TRY(cudaMemcpyAsync(phase, p->d_out[slot], sizeof(double) * c64, cudaMemcpyDeviceToHost,
                                     p->copy_stream));
        CUDA_TRY(cudaEventRecord(p->landed[slot][kWidenChunksMax], p->copy_stream));
        CUDA_TRY(cudaStreamWaitEvent(p->widen_stream[slot], p->landed[slot][kWidenChunksMax], 0));
        CUDA_TRY(cudaEventRecord(p->copied[slot], p->widen_stream[slot]));
    } else {
        if (phase)
            CUDA_TRY(cudaMemcpyAsync(phase, p->d_out[slot], sizeof(double) * cnt, cudaMemcpyDeviceToHost,
                                     p->copy_stream));
        CUDA_TRY(cudaEventRecord(p->copied[slot], p->copy_stream));
    }
    p->next_slot = slot ^ 1;
    return HS_OK;
}

int hs_host_copy_split(hs_plan *p, int batch, int *f64_patterns)
{
    *f64_patterns = (int)std::lround(p->e2e_f64_frac * batch);
    return HS_OK;
}

int hs_solve_host(hs_plan *p, int alg, int iters, int64_t subset, int batch, int n, const double *x,
                  const double *y, const double *z, const double *a0, const double *theta0, double *phase,
                  double *e, double *u)
{
    int rc = hs_solve_host_async(p, alg, iters, subset, batch, n, x, y, z, a0, theta0, phase, e, u);
    if (rc) return rc;
    return hs_sync(p);
}

// ------------------------------------------------------------------
// Row-sharded solve (one process per GPU).  Pass j of the schedule runs over
// the rank's fold-group-aligned chunk range; hs_shard_pass returns the
// rank's group partials, the caller all-gathers them (rank order = group
// order) and hs_shard_update folds all groups in order and applies the
// update -- identical on every rank and bitwise equal to hs_solve.
static void shard_range(int nchunks, int rank, int world, int *lo, int *hi)
{
    const int ng = (nchunks + kGroup - 1) / kGroup;
    const int g0 = (int)((int64_t)rank * ng / world), g1 = (int)((int64_t)(rank + 1) * ng / world);
    *lo = std::min(g0 * kGroup, nchunks);
    *hi = std::min(g1 * kGroup, nchunks);
}

// pass j: kind 0 = tile pass, 1 = list pass; list + chunk count
static int shard_pass_desc(hs_plan *p, int j, int *kind, const DevList **list, int *nchunks)
{
    auto &sh = p->shard;
    const int64_t m = p->m;
    const DevList *lst = nullptr;
    int rc;
    if (sh.alg != HS_ALG_RS && (j == 0 ? sh.cs > 0 : j <= sh.cs)) {
        const int64_t off = (j == 0) ? 0 : ((int64_t)(j - 1) * sh.half) % (m - sh.subset + 1);
        if ((rc = get_window(p, off, sh.subset, &lst))) return rc;
        *kind = 1;
    } else {
        *kind = 0;  // GEMM-tile full pass (every n)
        *list = nullptr;
        *nchunks = tile_set(p).n;
        return HS_OK;
    }
    *list = lst;
    *nchunks = geom_of(*lst, lst->count, p->cfg.spw).nchunks;
    return HS_OK;
}

int hs_shard_begin(hs_plan *p, int alg, int iters, int64_t subset, const double *theta0, int rank, int world)
{
    if (p->batch < 1) return fail(HS_EINVAL, "no spots set");
    if (world < 1 || rank < 0 || rank >= world) return fail(HS_EINVAL, "invalid rank %d / world %d", rank, world);
    if (alg != HS_ALG_RS && alg != HS_ALG_WGS && alg != HS_ALG_CSWGS) return fail(HS_EINVAL, "unknown algorithm");
    if (alg == HS_ALG_RS) {
        iters = 0;
        subset = p->m;
    } else {
        if (iters < 1) return fail(HS_EINVAL, "iterations must be >= 1");
        if (alg == HS_ALG_CSWGS && iters < 2) return fail(HS_EINVAL, "cswgs needs iterations >= 2");
        if (alg == HS_ALG_WGS) subset = p->m;
        if (subset < 1 || subset > p->m) return fail(HS_EINVAL, "subset size outside 1..M");
    }
    if (!(p->sum_amp > 0.0)) return fail(HS_EZEROILLUM, "pupil carries no illumination");
    if (p->cfg.NL == 0 || p->precision_mode == HS_PREC_FP64)
        return fail(HS_EINVAL, "the row-sharded solve runs the fp32 passes only (n <= %d)", kMaxSpots32);
    int rc;
    if ((rc = check_device(p)) || (rc = ensure_trace(p, iters))) return rc;
    auto &sh = p->shard;
    sh.active = true;
    sh.rank = rank;
    sh.world = world;
    sh.alg = alg;
    sh.iters = iters;
    sh.subset = subset;
    sh.cs = (alg != HS_ALG_RS && subset < p->m) ? std::max(0, iters - 2) : 0;
    sh.half = std::max<int64_t>(1, subset / 2);
    sh.passes = (alg == HS_ALG_RS) ? 1 : iters + 1;
    const size_t bytes = sizeof(double) * (size_t)p->batch * p->n;
    CUDA_TRY(cudaMemcpyAsync(p->d_theta, theta0, bytes, cudaMemcpyHostToDevice, p->stream));
    if ((rc = reset_status(p)) || (rc = launch_tables(p, true))) return rc;
    // phases this rank does not own stay NaN (0xff bytes) for the merge
    CUDA_TRY(cudaMemsetAsync(p->d_out[0], 0xff, sizeof(double) * (size_t)p->batch * p->m, p->stream));
    p->tables_valid = true;
    p->out_slot = 0;
    p->slot32[0] = false;   // the sharded passes write f64 phases into d_out[0]
    p->last_alg = alg;
    p->last_iters = iters;
    p->last_flags = HS_WANT_FIELDS;
    return HS_OK;
}

int hs_shard_pass(hs_plan *p, int j, double *groups, int *g_lo, int *g_hi, int *ngroups)
{
    auto &sh = p->shard;
    if (!sh.active || j < 0 || j >= sh.passes) return fail(HS_EINVAL, "shard pass %d out of range", j);
    int rc, kind, nch;
    const DevList *lst;
    if ((rc = check_device(p)) || (rc = shard_pass_desc(p, j, &kind, &lst, &nch))) return rc;
    int lo, hi;
    shard_range(nch, sh.rank, sh.world, &lo, &hi);
    const bool last = (j == sh.passes - 1);
    const int mode = last ? (PM_BWD | PM_FWD | PM_WRITE) : (PM_BWD | PM_FWD);
    const UpdArgs none = upd_args(p, ACT_NONE);
    if (kind == 0)
        rc = launch_tile(p, last, none, p->d_out[0], lo, hi);
    else
        rc = launch_pass(p, mode, *lst, 0, lst->count, 0, nullptr, last ? p->d_out[0] : nullptr, p->m, none, lo, hi);
    if (rc) return rc;
    const int ng = (nch + kGroup - 1) / kGroup;
    *g_lo = lo / kGroup;
    *g_hi = (hi + kGroup - 1) / kGroup;
    *ngroups = ng;
    if (*g_hi > *g_lo) {
        hs_group_fold_kernel<<<dim3(*g_hi - *g_lo, p->batch), 128, 0, p->stream>>>(fold_args(p, nch, none, lo, hi),
                                                                                *g_lo);
        CUDA_TRY(cudaGetLastError());
        const int np = p->cfg.np, cnt = *g_hi - *g_lo;
        if (groups)
            CUDA_TRY(cudaMemcpy2DAsync(groups, sizeof(double2) * cnt * np,
                                       p->d_gpart + (int64_t)*g_lo * np, sizeof(double2) * p->gpart_stride,
                                       sizeof(double2) * cnt * np, p->batch, cudaMemcpyDeviceToHost, p->stream));
    }
    return sync_and_check(p);
}

// ---- peer-memory exchange (hs_xchg.cuh): the sharded solve without host
// round trips.  Buffer = flags [world] (256-B padded) | xbuf [2][B][ngmax][np].
static const size_t kFlagBytes = 256;

int hs_shard_p2p_setup(hs_plan *p, unsigned char *handle_out)
{
    auto &sh = p->shard;
    auto &x = p->xchg;
    if (!sh.active) return fail(HS_EINVAL, "hs_shard_begin first");
    if ((size_t)sh.world * 8 > kFlagBytes) return fail(HS_EINVAL, "world %d too large", sh.world);
    int rc;
    if ((rc = check_device(p))) return rc;
    hs_shard_p2p_close(p);
    x.ngmax = (int)((p->cap_chunks + kGroup - 1) / kGroup);
    x.bytes = kFlagBytes + sizeof(double2) * (size_t)2 * p->batch * x.ngmax * p->cfg.np;
    CUDA_TRY(cudaMalloc((void **)&x.local, x.bytes));
    CUDA_TRY(cudaMemset(x.local, 0, kFlagBytes));
    CUDA_TRY(cudaDeviceSynchronize());
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, x.local));
    memcpy(handle_out, &h, sizeof h);
    if ((rc = dalloc(&x.d_cnt, 1))) return rc;
    CUDA_TRY(cudaMemset(x.d_cnt, 0, sizeof(int32_t)));
    if ((rc = dalloc(&x.d_epoch, 2))) return rc;
    CUDA_TRY(cudaMemset(x.d_epoch, 0, 2 * sizeof(unsigned long long)));
    return HS_OK;
}

int hs_shard_p2p_open(hs_plan *p, const unsigned char *handles)
{
    auto &sh = p->shard;
    auto &x = p->xchg;
    if (!x.local) return fail(HS_EINVAL, "hs_shard_p2p_setup first");
    int rc;
    if ((rc = check_device(p))) return rc;
    x.bases.assign(sh.world, nullptr);
    for (int r = 0; r < sh.world; ++r) {
        if (r == sh.rank) {
            x.bases[r] = x.local;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, handles + (size_t)r * sizeof h, sizeof h);
        void *ptr = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        x.bases[r] = (char *)ptr;
    }
    std::vector<double2 *> xb(sh.world);
    std::vector<unsigned long long *> fl(sh.world);
    for (int r = 0; r < sh.world; ++r) {
        fl[r] = (unsigned long long *)x.bases[r];
        xb[r] = (double2 *)(x.bases[r] + kFlagBytes);
    }
    if ((rc = dalloc(&x.d_xbuf, sh.world)) || (rc = dalloc(&x.d_flags, sh.world))) return rc;
    CUDA_TRY(cudaMemcpy(x.d_xbuf, xb.data(), sizeof(double2 *) * sh.world, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(x.d_flags, fl.data(), sizeof(void *) * sh.world, cudaMemcpyHostToDevice));
    x.open = true;
    return HS_OK;
}

// Enqueue pass j: the rank's chunk range, the peer publish of its groups and
// the gather + update.  Asynchronous: the device does the waiting.
int hs_shard_p2p_pass(hs_plan *p, int j)
{
    auto &sh = p->shard;
    auto &x = p->xchg;
    if (!sh.active || j < 0 || j >= sh.passes) return fail(HS_EINVAL, "shard pass %d out of range", j);
    if (!x.open) return fail(HS_EINVAL, "hs_shard_p2p_open first");
    int rc, kind, nch;
    const DevList *lst;
    if ((rc = check_device(p)) || (rc = shard_pass_desc(p, j, &kind, &lst, &nch))) return rc;
    int lo, hi;
    shard_range(nch, sh.rank, sh.world, &lo, &hi);
    const bool last = (j == sh.passes - 1);
    const int mode = last ? (PM_BWD | PM_FWD | PM_WRITE) : (PM_BWD | PM_FWD);
    const UpdArgs none = upd_args(p, ACT_NONE);
    if (j == 0) {  // epochs of this solve: base + 1 .. base + passes
        hs_epoch_advance_kernel<<<1, 32, 0, p->stream>>>(x.d_epoch, x.d_epoch + 1, sh.passes);
        CUDA_TRY(cudaGetLastError());
    }
    if (kind == 0)
        rc = launch_tile(p, last, none, p->d_out[0], lo, hi);
    else
        rc = launch_pass(p, mode, *lst, 0, lst->count, 0, nullptr, last ? p->d_out[0] : nullptr, p->m, none, lo, hi);
    if (rc) return rc;
    const int ng = (nch + kGroup - 1) / kGroup;
    if (ng > x.ngmax) return fail(HS_ECUDA, "exchange buffer too small (%d groups)", ng);
    UpdArgs u = upd_args(p, last ? ACT_FINAL : ACT_STEP);
    u.iter = j;
    u.iters = std::max(sh.iters, 1);
    XchgArgs a;
    memset(&a, 0, sizeof a);
    a.f = fold_args(p, nch, u, lo, hi);
    a.g_lo = lo / kGroup;
    a.g_hi = (hi + kGroup - 1) / kGroup;
    a.ngroups = ng;
    a.ngmax = x.ngmax;
    a.world = sh.world;
    a.rank = sh.rank;
    a.slot = j & 1;
    a.epoch0 = x.d_epoch + 1;
    a.pass = j;
    a.peer_xbuf = x.d_xbuf;
    a.peer_flags = x.d_flags;
    a.flags_local = (unsigned long long *)x.local;
    a.xbuf_local = (const double2 *)(x.local + kFlagBytes);
    a.pub_cnt = x.d_cnt;
    a.batch = p->batch;
    if (a.g_hi > a.g_lo) {
        hs_publish_kernel<<<dim3(a.g_hi - a.g_lo, p->batch), 128, 0, p->stream>>>(a);
        CUDA_TRY(cudaGetLastError());
    } else {  // a rank without groups still announces the epoch
        XchgArgs b = a;
        b.announce_only = 1;
        hs_publish_kernel<<<dim3(1, 1), 128, 0, p->stream>>>(b);
        CUDA_TRY(cudaGetLastError());
    }
    hs_gather_update_kernel<<<p->batch, kThreads, sizeof(double2) * 3 * p->cfg.np, p->stream>>>(a);
    CUDA_TRY(cudaGetLastError());
    if (last) sh.active = false;
    return HS_OK;
}

// All passes of the sharded solve begun by hs_shard_begin as one CUDA graph
// (captured on first use per (algorithm, iterations, subset, batch, n, rank,
// world), then replayed): the same kernels hs_shard_p2p_pass enqueues, with
// the epochs taken from device memory, so nothing is enqueued per pass.
int hs_shard_p2p_solve(hs_plan *p)
{
    auto &sh = p->shard;
    auto &x = p->xchg;
    if (!sh.active) return fail(HS_EINVAL, "hs_shard_begin first");
    if (!x.open) return fail(HS_EINVAL, "hs_shard_p2p_open first");
    int rc;
    if ((rc = check_device(p))) return rc;
    const auto key = std::make_tuple(sh.alg, sh.iters, sh.subset, p->batch, p->n, sh.rank, sh.world);
    auto it = x.graphs.find(key);
    if (it == x.graphs.end()) {
        // host-side list building happens outside graph capture
        const DevList *l;
        if ((rc = get_dense(p, p->cfg.spw, &l))) return rc;
        for (int j = 0; j < sh.passes; ++j) {
            int kind, nch;
            if ((rc = shard_pass_desc(p, j, &kind, &l, &nch))) return rc;
        }
        cudaGraph_t graph;
        CUDA_TRY(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
        for (int j = 0; j < sh.passes && !rc; ++j) rc = hs_shard_p2p_pass(p, j);
        cudaError_t ce = cudaStreamEndCapture(p->stream, &graph);
        if (rc) return rc;
        if (ce != cudaSuccess) return fail(HS_ECUDA, "graph capture failed: %s", cudaGetErrorString(ce));
        cudaGraphExec_t exec;
        ce = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ce != cudaSuccess) return fail(HS_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(ce));
        it = x.graphs.emplace(key, exec).first;
    }
    CUDA_TRY(cudaGraphLaunch(it->second, p->stream));
    sh.active = false;
    return HS_OK;
}

int hs_shard_p2p_close(hs_plan *p)
{
    auto &x = p->xchg;
    if (x.local) cudaStreamSynchronize(p->stream);
    for (auto &g : x.graphs) cudaGraphExecDestroy(g.second);
    x.graphs.clear();
    for (size_t r = 0; r < x.bases.size(); ++r)
        if (x.bases[r] && x.bases[r] != x.local) cudaIpcCloseMemHandle(x.bases[r]);
    x.bases.clear();
    if (x.local) cudaFree(x.local);
    x.local = nullptr;
    dfree(x.d_xbuf);
    dfree(x.d_flags);
    dfree(x.d_cnt);
    dfree(x.d_epoch);
    x.open = false;
    return HS_OK;
}

int hs_shard_groups(hs_plan *p, int j, int *g_lo, int *g_hi, int *ngroups)
{
    auto &sh = p->shard;
    if (!sh.active || j < 0 || j >= sh.passes) return fail(HS_EINVAL, "shard pass %d out of range", j);
    int rc, kind, nch, lo, hi;
    const DevList *lst;
    if ((rc = shard_pass_desc(p, j, &kind, &lst, &nch))) return rc;
    shard_range(nch, sh.rank, sh.world, &lo, &hi);
    *g_lo = lo / kGroup;
    *g_hi = (hi + kGroup - 1) / kGroup;
    *ngroups = (nch + kGroup - 1) / kGroup;
    return HS_OK;
}

int hs_shard_update(hs_plan *p, int j, const double *groups, int ngroups)
{
    auto &sh = p->shard;
    if (!sh.active || j < 0 || j >= sh.passes) return fail(HS_EINVAL, "shard pass %d out of range", j);
    int rc;
    if ((rc = check_device(p))) return rc;
    const int np = p->cfg.np;
    if ((int64_t)ngroups * np > p->gpart_stride) return fail(HS_EINVAL, "too many groups");
    CUDA_TRY(cudaMemcpy2DAsync(p->d_gpart, sizeof(double2) * p->gpart_stride, groups,
                               sizeof(double2) * ngroups * np, sizeof(double2) * ngroups * np, p->batch,
                               cudaMemcpyHostToDevice, p->stream));
    const bool last = (j == sh.passes - 1);
    UpdArgs u = upd_args(p, last ? ACT_FINAL : ACT_STEP);
    u.iter = j;
    u.iters = std::max(sh.iters, 1);
    hs_fold_update_kernel<<<p->batch, kThreads, sizeof(double2) * 2 * np, p->stream>>>(fold_args(p, 0, u), ngroups);
    CUDA_TRY(cudaGetLastError());
    if (last) sh.active = false;
    return sync_and_check(p);
}

// Standalone SLM raster of a storage-order phase (fileio.py:233-241 with
// PhaseLut.gray, fileio.py:202-213): linear table in closed form, custom
// table by first-minimum circular distance, both in fp64 in the reference's
// operation order.
static __device__ double hs_wrap_ref(double t)
{
    double w = fmod(t, kTwoPi);
    if (w >= kPi) w = __dadd_rn(w, -kTwoPi);
    if (w < -kPi) w = __dadd_rn(w, kTwoPi);
    return w;
}

static __global__ void hs_raster_kernel(int64_t m, const int32_t *rc, const double *phase, const double *lut,
                                        int side, unsigned char *out)
{
    __shared__ double tab[256];
    if (lut)
        for (int k = threadIdx.x; k < 256; k += blockDim.x) tab[k] = lut[k];
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const double p = hs_wrap_ref(phase[i]);
        unsigned char g;
        if (!lut) {
            g = hs_gray_linear(p);
        } else {
            double best = INFINITY;
            int bi = 0;
            for (int k = 0; k < 256; ++k) {
                const double d = fabs(hs_wrap_ref(__dadd_rn(p, -tab[k])));
                if (d < best) {
                    best = d;
                    bi = k;
                }
            }
            g = (unsigned char)bi;
        }
        const int v = rc[i];
        out[(int64_t)(v >> 16) * side + (v & 0xffff)] = g;
    }
}

int hs_raster(hs_plan *p, const double *phase, const double *lut, unsigned char *out)
{
    int rc;
    if ((rc = check_device(p))) return rc;
    const size_t cells = (size_t)p->side * p->side;
    double *d_lut = nullptr, *d_ph = nullptr;
    unsigned char *d_img = nullptr;
    if ((lut && (rc = dalloc(&d_lut, 256))) || (rc = dalloc(&d_ph, p->m)) || (rc = dalloc(&d_img, cells))) {
        dfree(d_lut);
        dfree(d_ph);
        return rc;
    }
    if (lut) CUDA_TRY(cudaMemcpyAsync(d_lut, lut, sizeof(double) * 256, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemcpyAsync(d_ph, phase, sizeof(double) * p->m, cudaMemcpyHostToDevice, p->stream));
    CUDA_TRY(cudaMemsetAsync(d_img, 0, cells, p->stream));
    hs_raster_kernel<<<4 * 148, 256, 0, p->stream>>>(p->m, p->storage.rc, d_ph, d_lut, p->side, d_img);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, d_img, cells, cudaMemcpyDeviceToHost, p->stream));
    rc = sync_and_check(p);
    dfree(d_lut);
    dfree(d_ph);
    dfree(d_img);
    return rc;
}

int hs_get_raster(hs_plan *p, int first, int count, unsigned char *out)
{
    if (!(p->last_flags & HS_WANT_RASTER)) return fail(HS_EINVAL, "last solve did not build rasters");
    if (first < 0 || count < 0 || first + count > p->batch) return fail(HS_EINVAL, "pattern range invalid");
    int rc;
    if ((rc = check_device(p))) return rc;
    const size_t cells = (size_t)p->side * p->side;
    if (count)
        CUDA_TRY(cudaMemcpyAsync(out, p->d_raster + first * cells, count * cells, cudaMemcpyDeviceToHost, p->stream));
    return sync_and_check(p);
}

void *hs_plan_stream(hs_plan *p) { return (void *)p->stream; }

int hs_last_launch_count(hs_plan *p, int64_t *launches)
{
    *launches = p->last_launches;
    return HS_OK;
}

// which: 0 = full-range fused pass (dense list), 1 = compressed-window fused
// pass over storage window [0, subset); both with the fold (ACT_FIELDS).
int hs_time_kernel(hs_plan *p, int which, int64_t subset, int reps, double *ms_per_launch,
                   double *pairs_per_launch)
{
    if (p->batch < 1) return fail(HS_EINVAL, "no spots set");
    if (reps < 1) return fail(HS_EINVAL, "reps must be >= 1");
    int rc;
    if ((rc = check_device(p)) || (rc = ensure_tables(p))) return rc;
    const DevList *l;
    if (which == 3 && (rc = ensure_out32(p))) return rc;
    if (which == 0 || which == 2 || which == 3) {
        rc = get_dense(p, p->cfg.spw, &l);
    } else {
        if (subset < 1 || subset > p->m) return fail(HS_EINVAL, "subset invalid");
        rc = get_window(p, 0, subset, &l);
    }
    if (rc) return rc;
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    const UpdArgs u = upd_args(p, ACT_FIELDS);
    if (which == 1 && getenv("HS_SLAB_TRACE")) {  // timing probe of one window-pass CTA
        if (!p->d_trace && (rc = dalloc(&p->d_trace, 128))) return rc;
        CUDA_TRY(cudaMemset(p->d_trace, 0, 128 * sizeof(unsigned long long)));
        p->trace_next = true;
        if ((rc = launch_pass(p, PM_BWD | PM_FWD, *l, 0, l->count, 0, nullptr, nullptr, 0, u))) return rc;
        CUDA_TRY(cudaStreamSynchronize(p->stream));
        unsigned long long t[128];
        CUDA_TRY(cudaMemcpy(t, p->d_trace, sizeof t, cudaMemcpyDeviceToHost));
        fprintf(stderr, "slab trace (cycles from CTA start%s):", HS_PROBES ? "" : "; empty: build with HS_PROBES=1");
        for (int i = 1; i < 128; ++i)
            if (t[i]) fprintf(stderr, " %d:%lld", i, (long long)(t[i] - t[0]));
        fprintf(stderr, "\n");
    }
    if (which == 0 && getenv("HS_UMMA_TRACE")) {  // timing probe of one tcgen05 CTA
        if (!p->d_trace && (rc = dalloc(&p->d_trace, 128))) return rc;
        CUDA_TRY(cudaMemset(p->d_trace, 0, 128 * sizeof(unsigned long long)));
        p->trace_next = true;
        if ((rc = launch_tile(p, false, u, nullptr))) return rc;
        CUDA_TRY(cudaStreamSynchronize(p->stream));
        unsigned long long t[128];
        CUDA_TRY(cudaMemcpy(t, p->d_trace, sizeof t, cudaMemcpyDeviceToHost));
        fprintf(stderr, "umma trace (cycles from CTA start%s):", HS_PROBES ? "" : "; empty: build with HS_PROBES=1");
        for (int i = 1; i < 128; ++i)
            if (t[i]) fprintf(stderr, " %d:%lld", i, (long long)(t[i] - t[0]));
        fprintf(stderr, "\n");
    }
    auto once = [&]() -> int {
        if (which == 0) return launch_tile(p, false, u, nullptr);
        if (which == 2) return launch_tile(p, true, u, p->d_out[0]);  // final pass: f64 phase write
        if (which == 3) {  // final pass: 4-byte phase codes (what solves store)
            p->rec_out32 = p->d_out32[0];
            const int r = launch_tile(p, true, u, p->d_out[0]);
            p->rec_out32 = nullptr;
            return r;
        }
        return launch_pass(p, PM_BWD | PM_FWD, *l, 0, l->count, 0, nullptr, nullptr, 0, u);
    };
    if ((rc = reset_status(p)) || (rc = once())) return rc;
    CUDA_TRY(cudaEventRecord(e0, p->stream));
    for (int r = 0; r < reps; ++r)
        if ((rc = once())) return rc;
    CUDA_TRY(cudaEventRecord(e1, p->stream));
    CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_per_launch = ms / reps;
    const int64_t pixels = (which != 1) ? p->m : subset;
    *pairs_per_launch = (double)pixels * p->n * p->batch;
    return HS_OK;
}

void *hs_host_alloc(int64_t bytes)
{
    void *ptr = nullptr;
    if (cudaHostAlloc(&ptr, (size_t)bytes, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return ptr;
}

void hs_host_free(void *ptr)
{
    if (ptr) cudaFreeHost(ptr);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// FP32 FMA-pipe peak microbenchmark (roofline denominator: MEASURED_PEAKS.json
// carries only HBM and bf16-tensor figures).  8 independent FFMA chains per
// thread, 148 x 8 CTAs of 256 threads.
// ---------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(256) hs_ffma_kernel(float *out, int iters, float a, float b)
{
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    float x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    const float s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
    if (s == 1.2345f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

extern "C" int hs_fma_peak(int device, double *tflops)
{
    CUDA_TRY(cudaSetDevice(device));
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    float *out = nullptr;
    CUDA_TRY(cudaMalloc(&out, sizeof(float) * blocks * threads));
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    hs_ffma_kernel<<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f);  // warm
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CUDA_TRY(cudaEventRecord(e0));
        hs_ffma_kernel<<<blocks, threads>>>(out, iters, 0.999999f, 1e-7f);
        CUDA_TRY(cudaEventRecord(e1));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 2.0 * blocks * threads * (double)iters * 16 * 8;
    *tflops = flops / (best * 1e-3) / 1e12;
    return HS_OK;
}
