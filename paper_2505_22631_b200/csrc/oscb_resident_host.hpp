// oscb_resident_host.hpp -- host side of the persistent shared-memory kernel: the graph
// "compiler" that turns the canonical CSR into the sliced-ELL neighbour stream the kernel
// walks (see oscb_resident.cuh), the tile-shape chooser and the launcher.
#pragma once
#include "oscb_host.hpp"
#include "oscb_resident.cuh"
#include "oscb_resident_fast.cuh"

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cmath>
#include <limits>
#include <numeric>
#include <type_traits>

namespace oscb {

struct ResidentPlan {
    int RT = 1, log2RT = 0, LPS = 1, C = 32, T = 1, W = 1;   // LPS: lanes per slot (RT / replicas per lane)
    int n_group_rows = 0;
    bool weighted = false;
    double fill = 1.0;          // real neighbours / stream entries
    double bank_conflicts = 0;  // stream positions whose slots collide on a bank class / all positions
    bool exact_f32_cut = false; // integer couplings small enough that float32 sums of them stay exact
    DevBuf<int> warp_start;
    DevBuf<uint16_t> rows, deg;
    DevBuf<float> rowsum;
    DevBuf<uint32_t> ginfo;
    DevBuf<uint2> stream;
    DevBuf<float> w32;
    DevBuf<double> w64;
};

// warps per CTA for a tile of RT replicas: as many slots as there are quads to hand out, in
// the fewest rounds the thread limit allows
static void tile_shape(int64_t n, int LPS, int max_threads, int *W, int *T)
{
    const int C = 32 / LPS;
    const int64_t Q = (n + 3) / 4;
    const int64_t s_max = (int64_t)(max_threads / 32) * C;
    const int64_t rounds = std::max<int64_t>(1, (Q + s_max - 1) / s_max);
    const int64_t slots = (Q + rounds - 1) / rounds;
    *W = (int)std::max<int64_t>(1, (slots + C - 1) / C);
    *T = (int)std::max<int64_t>(1, (Q + (int64_t)(*W) * C - 1) / ((int64_t)(*W) * C));
}

// pure host result of the graph compiler (also exported for CPU-side tests)
struct ResidentStreamHost {
    std::vector<int> warp_start;
    std::vector<uint16_t> rows;     // [W*T*4*C] own row * RT, n*RT when the slot has none
    std::vector<uint16_t> deg;      // [W*T*4*C] real degree of that row
    std::vector<float> rowsum;      // [W*T*4*C] sum of that row's couplings
    double max_abs_rowsum = 0.0;
    std::vector<uint32_t> ginfo;    // [W*T]
    std::vector<uint2> stream;      // [(n_group_rows + 1) * C] ids * RT; >= n*RT: zero padding rows
    std::vector<double> weights;    // [(n_group_rows + 1) * C * 4]
    int n_group_rows = 0;
    int64_t real = 0, positions = 0, conflicts = 0;
};

// A slot is LPS lanes wide (RT replicas / replicas per lane) and reads RT * pair_bytes contiguous
// bytes per neighbour.  `pair_bytes` (8: float2, 16: double2) fixes which slots share a 128-byte
// shared-memory wavefront: H = max(1, 128 / (RT * pair_bytes)) consecutive slots, and row j sits
// in bank class j mod H of that wavefront.  `keep_order` (parity mode) keeps every row in CSR order and
// only picks conflict-free padding rows; otherwise each row's neighbours are also reordered so
// that the H slots of a wavefront hit H different classes wherever the lists allow it.
static void compile_resident_stream(int n, const int *indptr, const int *indices, const double *wts, int RT, int LPS,
                                    int W, int T, int pair_bytes, bool keep_order, ResidentStreamHost *out)
{
    const int C = 32 / LPS, S = W * C;
    const int Q = (n + 3) / 4;
    const int H = std::max(1, std::min(C, (128 / pair_bytes) / RT));
    OSCB_REQUIRE((int64_t)(n + OSCB_PAD_ROWS) * RT <= 65535, "n * replicas_per_cta too large for 16-bit stream ids");
    OSCB_REQUIRE(H <= OSCB_PAD_ROWS, "internal: not enough padding rows");
    auto deg = [&](int i) { return i < n ? indptr[i + 1] - indptr[i] : 0; };

    // Quads ordered by the group-count profile of their rows (rows taken in descending degree, as
    // they are visited), heaviest first, then dealt to the slots boustrophedon: slot loads balance
    // and the C slots of a warp hold quads whose k-th rows need the same number of 4-neighbour
    // groups, which is what keeps the padding to a common G small (G22 shape: 0.92 fill at C = 4
    // against 0.86 for a plain total-degree sort; the rounding-to-4 bound is 0.93).
    std::vector<int> order(Q);
    std::iota(order.begin(), order.end(), 0);
    std::vector<std::array<int, 5>> qkey(Q);
    for (int q = 0; q < Q; ++q) {
        int d[4] = {deg(4 * q), deg(4 * q + 1), deg(4 * q + 2), deg(4 * q + 3)};
        std::sort(d, d + 4, [](int x, int y) { return x > y; });
        qkey[q] = {(d[0] + 3) / 4, (d[1] + 3) / 4, (d[2] + 3) / 4, (d[3] + 3) / 4, d[0] + d[1] + d[2] + d[3]};
    }
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return qkey[x] > qkey[y]; });
    // Consecutive runs of C quads in that order form the blocks that share a warp-round; a block
    // costs sum_k max_c G.  Blocks go to warps longest-first onto the least loaded warp (LPT), so
    // the per-warp stream lengths -- the CTA's step time is the longest one -- stay within a few %.
    std::vector<int> quad_of((size_t)W * T * C, -1);
    {
        const int n_blocks = (Q + C - 1) / C;
        OSCB_REQUIRE(n_blocks <= W * T, "internal: tile shape too small for the graph");
        (void)S;
        std::vector<int> bcost(n_blocks, 0), border(n_blocks);
        for (int b = 0; b < n_blocks; ++b) {
            int mx[4] = {0, 0, 0, 0};
            for (int c = 0; c < C && b * C + c < Q; ++c)
                for (int k = 0; k < 4; ++k) mx[k] = std::max(mx[k], qkey[order[b * C + c]][k]);
            bcost[b] = mx[0] + mx[1] + mx[2] + mx[3];
        }
        std::iota(border.begin(), border.end(), 0);
        std::stable_sort(border.begin(), border.end(), [&](int x, int y) { return bcost[x] > bcost[y]; });
        std::vector<int> wload(W, 0), wcount(W, 0);
        for (int b : border) {
            int best = -1;
            for (int w = 0; w < W; ++w)
                if (wcount[w] < T && (best < 0 || wload[w] < wload[best])) best = w;
            for (int c = 0; c < C && b * C + c < Q; ++c) quad_of[((size_t)best * T + wcount[best]) * C + c] = order[b * C + c];
            wload[best] += bcost[b];
            ++wcount[best];
        }
    }

    out->warp_start.assign(W, 0);
    out->rows.assign((size_t)W * T * 4 * C, (uint16_t)(n * RT));
    out->deg.assign((size_t)W * T * 4 * C, 0);
    out->rowsum.assign((size_t)W * T * 4 * C, 0.f);
    out->max_abs_rowsum = 0.0;
    out->ginfo.assign((size_t)W * T, 0);
    out->stream.clear();
    out->weights.clear();
    out->real = out->positions = out->conflicts = 0;
    int group_rows = 0;
    struct Item { int j; double w; };
    for (int w = 0; w < W; ++w) {
        out->warp_start[w] = group_rows;
        for (int t = 0; t < T; ++t) {
            int rows[32][4]; // [c][kk] row visited kk-th by slot c (or -1)
            int G[4] = {0, 0, 0, 0};
            for (int c = 0; c < C; ++c) {
                const int quad = quad_of[((size_t)w * T + t) * C + c];
                for (int kk = 0; kk < 4; ++kk) rows[c][kk] = -1;
                if (quad < 0) continue;
                int ks[4] = {0, 1, 2, 3};
                std::stable_sort(ks, ks + 4, [&](int x, int y) { return deg(4 * quad + x) > deg(4 * quad + y); });
                for (int kk = 0; kk < 4; ++kk) {
                    const int i = 4 * quad + ks[kk];
                    rows[c][kk] = i < n ? i : -1;
                    G[kk] = std::max(G[kk], (deg(i) + 3) / 4);
                }
            }
            for (int kk = 0; kk < 4; ++kk) {
                OSCB_REQUIRE(G[kk] <= 255, "row degree too large for the resident kernel");
                out->ginfo[(size_t)w * T + t] |= (uint32_t)G[kk] << (8 * kk);
                const int P = 4 * G[kk];
                // laid[c][p]: the entry slot c reads at position p (j = -1 - class for padding)
                std::vector<std::vector<Item>> laid(C, std::vector<Item>(P, Item{-1, 0.0}));
                for (int c = 0; c < C; ++c) {
                    const int i = rows[c][kk];
                    const size_t at = (((size_t)w * T + t) * 4 + kk) * C + c;
                    if (i >= 0) {
                        out->rows[at] = (uint16_t)(i * RT);
                        out->deg[at] = (uint16_t)deg(i);
                        double rs = 0.0, ra = 0.0;
                        for (int e = indptr[i]; e < indptr[i + 1]; ++e) { rs += wts ? wts[e] : 1.0; ra += std::fabs(wts ? wts[e] : 1.0); }
                        out->rowsum[at] = (float)rs;
                        out->max_abs_rowsum = std::max(out->max_abs_rowsum, ra);
                    }
                }
                for (int c0 = 0; c0 < C; c0 += H) {
                    // remaining items of each slot of this wavefront group, bucketed by bank class
                    std::vector<std::vector<std::vector<Item>>> bucket(H, std::vector<std::vector<Item>>(H));
                    std::vector<int> left(H, 0);
                    for (int hc = 0; hc < H; ++hc) {
                        const int i = rows[c0 + hc][kk];
                        if (i < 0) continue;
                        for (int e = indptr[i + 1] - 1; e >= indptr[i]; --e)        // reversed: pop_back() yields CSR order
                            bucket[hc][keep_order ? 0 : indices[e] % H].push_back(Item{indices[e], wts ? wts[e] : 1.0});
                        left[hc] = deg(i);
                    }
                    for (int p = 0; p < P; ++p) {
                        std::vector<char> used(H, 0);
                        std::vector<int> who(H);
                        std::iota(who.begin(), who.end(), 0);
                        // the slot with the least slack (fewest spare padding positions) chooses first
                        std::stable_sort(who.begin(), who.end(), [&](int x, int y) { return left[x] > left[y]; });
                        std::vector<int> pad_slots;
                        for (int hc : who) {
                            Item pick{-1, 0.0};
                            if (left[hc] > 0) {
                                if (keep_order) {
                                    pick = bucket[hc][0].back();
                                    bucket[hc][0].pop_back();
                                } else {
                                    int best = -1;
                                    for (int cls = 0; cls < H; ++cls)
                                        if (!used[cls] && !bucket[hc][cls].empty() &&
                                            (best < 0 || bucket[hc][cls].size() > bucket[hc][best].size()))
                                            best = cls;
                                    const bool spare = (P - p) > left[hc];
                                    if (best < 0 && spare) { pad_slots.push_back(hc); continue; }
                                    if (best < 0)   // forced conflict: take from the fullest bucket
                                        for (int cls = 0; cls < H; ++cls)
                                            if (!bucket[hc][cls].empty() && (best < 0 || bucket[hc][cls].size() > bucket[hc][best].size()))
                                                best = cls;
                                    pick = bucket[hc][best].back();
                                    bucket[hc][best].pop_back();
                                }
                                --left[hc];
                                const int cls = pick.j % H;
                                if (used[cls]) ++out->conflicts;
                                used[cls] = 1;
                                laid[c0 + hc][p] = pick;
                                ++out->real;
                            } else {
                                pad_slots.push_back(hc);
                            }
                        }
                        for (int hc : pad_slots) {         // padding takes a class nobody reads
                            int cls = 0;
                            while (cls < H - 1 && used[cls]) ++cls;
                            used[cls] = 1;
                            laid[c0 + hc][p] = Item{-1 - cls, 0.0};
                        }
                        ++out->positions;
                    }
                }
                for (int gidx = 0; gidx < G[kk]; ++gidx) {
                    for (int c = 0; c < C; ++c) {
                        uint32_t ids[4];
                        for (int u = 0; u < 4; ++u) {
                            const Item &it = laid[c][4 * gidx + u];
                            ids[u] = it.j >= 0 ? (uint32_t)(it.j * RT) : (uint32_t)((n + (-1 - it.j)) * RT);
                            out->weights.push_back(it.j >= 0 ? it.w : 0.0);
                        }
                        out->stream.push_back(make_uint2(ids[0] | (ids[1] << 16), ids[2] | (ids[3] << 16)));
                    }
                    ++group_rows;
                }
            }
        }
    }
    out->n_group_rows = group_rows;
    for (int c = 0; c < C; ++c) {          // the prefetch pad row
        const uint32_t pad = (uint32_t)(n * RT);
        out->stream.push_back(make_uint2(pad | (pad << 16), pad | (pad << 16)));
        for (int u = 0; u < 4; ++u) out->weights.push_back(0.0);
    }
}

static std::shared_ptr<ResidentPlan> build_resident_plan(oscb_graph *g, int RT, int LPS, int W, int T, int pair_bytes,
                                                         bool keep_order)
{
    auto plan = std::make_shared<ResidentPlan>();
    plan->RT = RT;
    plan->log2RT = 0;
    while ((1 << plan->log2RT) < RT) ++plan->log2RT;
    plan->LPS = LPS;
    plan->C = 32 / LPS;
    plan->W = W;
    plan->T = T;
    plan->weighted = !g->unit_weights;
    ResidentStreamHost h;
    compile_resident_stream((int)g->n, g->h_indptr.data(), g->h_indices.data(), g->h_w.data(), RT, LPS, W, T,
                            pair_bytes, keep_order, &h);
    OSCB_REQUIRE(h.real == g->nnz, "internal: resident plan lost neighbours (%lld of %lld)", (long long)h.real, (long long)g->nnz);
    plan->n_group_rows = h.n_group_rows;
    plan->fill = h.n_group_rows == 0 ? 1.0 : (double)h.real / (4.0 * (double)h.n_group_rows * plan->C);
    plan->bank_conflicts = h.positions ? (double)h.conflicts / (double)h.positions : 0.0;
    cudaStream_t s = g->stream;
    plan->warp_start.alloc(W);                plan->warp_start.upload(h.warp_start.data(), W, s);
    plan->rows.alloc(h.rows.size());          plan->rows.upload(h.rows.data(), h.rows.size(), s);
    plan->deg.alloc(h.deg.size());            plan->deg.upload(h.deg.data(), h.deg.size(), s);
    plan->rowsum.alloc(h.rowsum.size());      plan->rowsum.upload(h.rowsum.data(), h.rowsum.size(), s);
    plan->exact_f32_cut = g->int_weights && h.max_abs_rowsum * (double)g->n < 16777216.0;
    plan->ginfo.alloc(h.ginfo.size());        plan->ginfo.upload(h.ginfo.data(), h.ginfo.size(), s);
    plan->stream.alloc(h.stream.size());      plan->stream.upload(h.stream.data(), h.stream.size(), s);
    std::vector<float> wf(h.weights.begin(), h.weights.end());
    if (plan->weighted) {
        plan->w64.alloc(h.weights.size());    plan->w64.upload(h.weights.data(), h.weights.size(), s);
        plan->w32.alloc(wf.size());           plan->w32.upload(wf.data(), wf.size(), s);
    }
    OSCB_CUDA(cudaStreamSynchronize(s));
    return plan;
}

static std::shared_ptr<ResidentPlan> get_resident_plan(oscb_graph *g, int RT, int LPS, int W, int T, int pair_bytes,
                                                       bool keep_order)
{
    const uint64_t key = ((uint64_t)RT << 48) | ((uint64_t)LPS << 40) | ((uint64_t)W << 24) | ((uint64_t)T << 8) |
                         ((uint64_t)pair_bytes << 1) | (keep_order ? 1u : 0u);
    auto it = g->plans.find(key);
    if (it != g->plans.end()) return it->second;
    auto plan = build_resident_plan(g, RT, LPS, W, T, pair_bytes, keep_order);
    g->plans[key] = plan;
    return plan;
}

struct ResidentConfig {
    int RT = 0, LPS = 0, W = 0, T = 0, max_threads = 1024;
    size_t smem_min = 0; // without the stream staged in shared memory
};

static inline int max_threads_for(int precision) { return precision == OSCB_PREC_F64 ? 512 : 1024; }

// the specialised float32 kernel applies unless the float64 parity mode, injected noise or the
// generic variant was asked for
static inline bool wants_fast(const oscb_run_params *p)
{
    return p->precision == OSCB_PREC_F32 && p->noise_mode != OSCB_NOISE_HOST && p->variant != 1;
}
// replicas per lane of the float32 kernel: two whenever a tile has two (OSCB_FAST_RPL=1 disables)
static inline int fast_rpl(int RT)
{
    const char *e = getenv("OSCB_FAST_RPL");
    if (e && e[0] == '1') return 1;
    return RT >= 2 ? 2 : 1;
}

static size_t resident_smem_bytes(const oscb_graph *g, int precision, int n_states, int RT, int W, int T,
                                  int n_group_rows, bool idx_smem)
{
    const size_t pair = precision == OSCB_PREC_F64 ? 16 : 8;
    (void)n_states;
    return ResidentSmem::make((int)g->n, RT, 32 / RT, T, W, pair, pair / 2, n_group_rows, idx_smem, !g->unit_weights).total;
}

// tile width: the candidate with the lowest estimated time
static bool choose_resident_config(const oscb_graph *g, int precision, int n_states, int64_t R, int requested_rt,
                                   bool fast, ResidentConfig *out)
{
    if (g->n > 60000 || g->max_degree > 1020 || n_states > 254) return false;
    static const double eff[6] = {0.35, 0.5, 0.7, 0.85, 1.0, 1.0}; // gather efficiency by log2(RT)
    const int max_threads = max_threads_for(precision);
    double best_cost = std::numeric_limits<double>::infinity();
    bool found = false;
    for (int l = 5; l >= 0; --l) {
        const int RT = 1 << l;
        if (requested_rt > 0 && RT != requested_rt) continue;
        if (requested_rt <= 0 && RT > 1 && RT / 2 >= R) continue; // do not pad a tile more than 2x
        int W, T;
        const int LPS = fast ? RT / fast_rpl(RT) : RT;
        tile_shape(g->n, LPS, max_threads, &W, &T);
        if ((g->n + OSCB_PAD_ROWS) * RT > 65535) continue;
        const size_t need = fast ? FastSmem::make((int)g->n, RT, 32 / LPS, T, W, 0, n_states != 2, false, false, false,
                                                  !g->unit_weights).total
                                 : resident_smem_bytes(g, precision, n_states, RT, W, T, 0, false);
        if (need > (size_t)g->smem_optin) continue;
        const int64_t tiles = (R + RT - 1) / RT;
        const int by_smem = (int)std::max<size_t>(1, (size_t)(g->smem_optin + 1024) / (need + 1024));
        const int by_threads = std::max(1, 2048 / (W * 32));
        const int cps = std::min(by_smem, by_threads);
        const int64_t slots = (int64_t)g->sm_count * cps;
        const int64_t waves = (tiles + slots - 1) / slots;
        const int64_t per_sm = std::min<int64_t>(cps, (tiles + g->sm_count - 1) / g->sm_count);
        const double cost = (double)waves * (double)per_sm * RT / eff[l];
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            out->RT = RT;
            out->LPS = LPS;
            out->W = W;
            out->T = T;
            out->max_threads = max_threads;
            out->smem_min = need;
            found = true;
        }
    }
    return found;
}

static bool resident_fits(const oscb_graph *g, const oscb_run_params *p, int64_t R)
{
    ResidentConfig cfg;
    return choose_resident_config(g, p->precision, p->n_states, R, p->replicas_per_cta, wants_fast(p), &cfg);
}

template <typename T, int MAXT, bool STRICT>
static void launch_resident(oscb_graph *g, const ResidentArgs &args, int tiles, int threads, size_t smem, bool idx_smem,
                            bool weighted)
{
    auto go = [&](auto kernel) {
        OSCB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kernel<<<tiles, threads, smem, g->stream>>>(args);
    };
    if (idx_smem) {
        if (weighted) go(k_resident<T, MAXT, true, true, STRICT>);
        else go(k_resident<T, MAXT, true, false, STRICT>);
    } else {
        if (weighted) go(k_resident<T, MAXT, false, true, STRICT>);
        else go(k_resident<T, MAXT, false, false, STRICT>);
    }
}

// smem plan of the float32 production kernel: phases first, then the stream
struct FastFit {
    bool phi_smem = false, idx_smem = false, piggy = false, deg_smem = false, states = false;
    FastSmem lay;
    size_t smem = 0;
};
static FastFit fit_fast(const oscb_graph *g, int n_states, int objective, int RT, int C, int W, int T, int n_group_rows,
                        bool exact_f32_cut)
{
    const bool weighted = !g->unit_weights;
    FastFit f;
    f.states = n_states != 2;
    // scoring rides on the next step's gather: N = 2 max-cut (sign bits; weighted only while float32 sums of
    // the couplings stay exact) and N-state colouring (state bytes, a count)
    f.piggy = (n_states == 2 && objective == OSCB_OBJ_MAXCUT && (!weighted || exact_f32_cut)) ||
              (n_states != 2 && objective == OSCB_OBJ_COLORING);
    auto lay = [&](bool phi, bool idx) {
        return FastSmem::make((int)g->n, RT, C, T, W, n_group_rows, f.states, f.deg_smem, phi, idx, weighted);
    };
    const size_t cap = (size_t)g->smem_optin;
    // The neighbour stream is on the critical path of every gather (a phase is touched three
    // times per row and its load can be issued a whole row early), so the stream gets the
    // shared memory first, the phases second.  The degree table is read on scoring steps only
    // and goes to shared memory last.
    if (lay(false, true).total <= cap) f.idx_smem = true;
    if (f.idx_smem && lay(true, true).total <= cap) f.phi_smem = true;
    if (f.piggy && !weighted && n_states == 2) {
        f.deg_smem = true;
        if (lay(f.phi_smem, f.idx_smem).total > cap) f.deg_smem = false;
    }
    f.lay = lay(f.phi_smem, f.idx_smem);
    f.smem = f.lay.total;
    return f;
}

static void launch_resident_fast(oscb_graph *g, const ResidentArgs &ra, const ResidentPlan &plan, int n_states,
                                 const FastFit &f, int tiles, float2 *cs_next, const float *hks_table)
{
    FastArgs a;
    memset(&a, 0, sizeof(a));
    a.n = ra.n; a.RT = ra.RT; a.LRT = ra.log2RT; a.nRT = ra.n * ra.RT; a.C = ra.C; a.W = ra.W; a.n_rows = 4 * ra.T;
    a.LPS = plan.LPS; a.LLPS = 0;
    while ((1 << a.LLPS) < a.LPS) ++a.LLPS;
    const int rpl = ra.RT / plan.LPS;
    a.R_real = ra.R_real; a.n_group_rows = ra.n_group_rows; a.piggy = f.piggy ? 1 : 0; a.deg_smem = f.deg_smem ? 1 : 0;
    a.off_cs = (uint32_t)f.lay.cs; a.off_phi = (uint32_t)f.lay.phi; a.off_st = (uint32_t)f.lay.st;
    a.off_rows = (uint32_t)f.lay.rows; a.off_g = (uint32_t)f.lay.g; a.off_deg = (uint32_t)f.lay.deg;
    a.off_part = (uint32_t)f.lay.part; a.off_misc = (uint32_t)f.lay.misc; a.off_stream = (uint32_t)f.lay.stream;
    a.off_w = (uint32_t)f.lay.wstream; a.smem_total = (uint32_t)f.lay.total;
    a.hK = (float)(ra.h * ra.K); a.knsh = (float)ra.kn_sqrt_h;
    a.h = ra.h; a.ks_max = ra.ks_max; a.ks_period = ra.ks_period; a.ks_scale = ra.h * (n_states == 2 ? 2.0 : 1.0);
    a.tc = ra.tc;
    a.noise_on = ra.noise_mode == OSCB_NOISE_DEVICE; a.maximize = ra.maximize; a.use_target = ra.use_target;
    a.initial_sample = ra.initial_sample; a.n_sample_steps = ra.n_sample_steps; a.sample_offset = ra.sample_offset;
    a.step_begin = ra.step_begin; a.step_end = ra.step_end; a.cadence = ra.cadence; a.trace_stride = ra.trace_stride;
    a.target = ra.target;
    a.warp_start = ra.warp_start; a.rows = ra.rows; a.ginfo = ra.ginfo; a.deg = plan.deg.p; a.rowsum = plan.rowsum.p;
    a.stream = ra.stream;
    a.wstream = reinterpret_cast<const float *>(ra.wstream);
    a.phi = reinterpret_cast<float *>(ra.phi); a.seeds = ra.seeds; a.sample_steps = ra.sample_steps;
    a.cs_next = cs_next;
    a.hks_table = hks_table;
    a.n_bnd = 0;
    if (n_states != 2 && n_states <= 8) {
        a.n_bnd = n_states;
        fast_state_boundaries(n_states, a.bnd);
    }
    a.best_obj = ra.best_obj; a.energy = ra.energy; a.best_trace = ra.best_trace; a.best_states = ra.best_states;
    a.first_hit = ra.first_hit; a.nonfinite = ra.nonfinite;
    auto go = [&](auto kernel) {
        OSCB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)f.smem));
        kernel<<<tiles, plan.W * 32, f.smem, g->stream>>>(a);
    };
    auto by_mem = [&](auto nm, auto wt) {
        constexpr int NM = decltype(nm)::value;
        constexpr bool WT = decltype(wt)::value;
        if (rpl == 2) {
            if (f.idx_smem) { if (f.phi_smem) go(k_resident_fast<NM, WT, true, true, 2>); else go(k_resident_fast<NM, WT, true, false, 2>); }
            else go(k_resident_fast<NM, WT, false, false, 2>);
        } else {
            if (f.idx_smem) { if (f.phi_smem) go(k_resident_fast<NM, WT, true, true, 1>); else go(k_resident_fast<NM, WT, true, false, 1>); }
            else go(k_resident_fast<NM, WT, false, false, 1>);
        }
    };
    using two = std::integral_constant<int, 2>;
    using any = std::integral_constant<int, 0>;
    if (n_states == 2) { if (plan.weighted) by_mem(two{}, std::true_type{}); else by_mem(two{}, std::false_type{}); }
    else               { if (plan.weighted) by_mem(any{}, std::true_type{}); else by_mem(any{}, std::false_type{}); }
}

template <typename T, int MAXT, bool STRICT, bool FAST>
static void run_resident_impl(oscb_graph *g, const oscb_run_params *p, const ResidentConfig &cfg, int64_t steps,
                              int64_t cadence, const std::vector<long long> &sample_steps, const uint64_t *seeds,
                              int64_t R64, const double *phi0, const double *noise, oscb_run_outputs *out)
{
    cudaStream_t s = g->stream;
    const int n = (int)g->n, R = (int)R64;
    auto plan = get_resident_plan(g, cfg.RT, cfg.LPS, cfg.W, cfg.T, (int)(2 * sizeof(T)), STRICT);
    const int RT = plan->RT, tiles = (R + RT - 1) / RT, R_pad = tiles * RT;
    bool idx_smem = true;
    size_t smem = resident_smem_bytes(g, p->precision, p->n_states, RT, plan->W, plan->T, plan->n_group_rows, true);
    if (smem > (size_t)g->smem_optin) {
        idx_smem = false;
        smem = resident_smem_bytes(g, p->precision, p->n_states, RT, plan->W, plan->T, plan->n_group_rows, false);
    }
    FastFit fast;
    if (FAST) {
        fast = fit_fast(g, p->n_states, p->objective, RT, plan->C, plan->W, plan->T, plan->n_group_rows, plan->exact_f32_cut);
        smem = fast.smem;
    }
    OSCB_REQUIRE(smem <= (size_t)g->smem_optin, "resident kernel does not fit in shared memory (%zu bytes)", smem);
    const int maximize = p->objective == OSCB_OBJ_MAXCUT;
    const int64_t S = 1 + (int64_t)sample_steps.size();
    const size_t tot = (size_t)n * R, tot_pad = (size_t)n * R_pad;

    DevBuf<T> d_phi(tot_pad + 64);   // + one padding row: invalid rows load (never store) row n
    DevBuf<double> d_io(tot);
    std::vector<uint64_t> h_seeds(R_pad, 0);
    std::copy(seeds, seeds + R, h_seeds.begin());
    DevBuf<uint64_t> d_seeds(R_pad);
    d_seeds.upload(h_seeds.data(), R_pad, s);
    DevBuf<double> d_best(R_pad), d_energy((size_t)R_pad * S), d_btrace((size_t)R_pad * S), d_noise;
    DevBuf<uint8_t> d_best_states(tot_pad);
    DevBuf<long long> d_first(R_pad), d_samples(std::max<size_t>(1, sample_steps.size()));
    std::vector<double> h_best(R_pad, maximize ? -std::numeric_limits<double>::infinity()
                                               : std::numeric_limits<double>::infinity());
    std::vector<long long> h_first(R_pad, -1), h_samples(sample_steps);
    for (auto &v : h_samples) v += p->first_step;
    d_best.upload(h_best.data(), R_pad, s);
    d_first.upload(h_first.data(), R_pad, s);
    d_samples.upload(h_samples.data(), h_samples.size(), s);
    d_best_states.zero(s);
    const unsigned long long none = ~0ull;
    OSCB_CUDA(cudaMemcpyAsync(g->d_nonfinite.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));
    if (phi0) d_io.upload(phi0, tot, s);
    else k_initial_phases<<<(unsigned)(((long long)((n + 3) / 4) * R + 127) / 128), 128, 0, s>>>(d_seeds.p, d_io.p, n, R);
    k_to_tile_layout<T><<<(unsigned)((tot_pad + 255) / 256), 256, 0, s>>>(d_io.p, d_phi.p, n, R, RT, (long long)tot_pad);
    if (p->noise_mode == OSCB_NOISE_HOST) {
        d_noise.alloc((size_t)steps * tot);
        d_noise.upload(noise, (size_t)steps * tot, s);
    }

    ResidentArgs a;
    memset(&a, 0, sizeof(a));
    a.n = n; a.R_real = R; a.RT = RT; a.log2RT = plan->log2RT; a.C = plan->C; a.T = plan->T; a.W = plan->W;
    a.n_group_rows = plan->n_group_rows;
    a.warp_start = plan->warp_start.p; a.rows = plan->rows.p; a.ginfo = plan->ginfo.p; a.stream = plan->stream.p;
    a.wstream = plan->weighted ? (sizeof(T) == 8 ? (const void *)plan->w64.p : (const void *)plan->w32.p) : nullptr;
    a.phi = d_phi.p; a.seeds = d_seeds.p;
    a.step_begin = p->first_step; a.step_end = p->first_step + steps; a.noise_step0 = p->first_step;
    a.K = p->K; a.h = p->h; a.kn_sqrt_h = p->kn * std::sqrt(p->h); a.ks_max = p->ks_max; a.ks_period = p->ks_period;
    a.tc = make_trig_const(p->n_states);
    a.noise_mode = p->noise_mode;
    if (p->kn == 0.0 && p->noise_mode == OSCB_NOISE_DEVICE) a.noise_mode = OSCB_NOISE_NONE;
    a.noise_host = d_noise.p;
    a.cadence = cadence;
    a.sample_steps = d_samples.p; a.n_sample_steps = (int)sample_steps.size(); a.sample_offset = 1; a.initial_sample = 1;
    a.maximize = maximize;
    a.best_obj = d_best.p; a.best_states = d_best_states.p; a.energy = d_energy.p; a.best_trace = d_btrace.p;
    a.trace_stride = S; a.first_hit = d_first.p; a.use_target = p->use_target; a.target = p->target_objective;
    a.nonfinite = g->d_nonfinite.p;

    cudaEvent_t ev0, ev1;
    OSCB_CUDA(cudaEventCreate(&ev0));
    OSCB_CUDA(cudaEventCreate(&ev1));
    DevBuf<float2> d_stage;
    DevBuf<float> d_hks;
    if (FAST && p->n_states == 2) d_stage.alloc(tot_pad + 64);
    if (FAST) {
        // h * ks(step) (x2 for N = 2, where the SHIL term is 2 s c) for every step, in the reference's float64
        std::vector<float> hks((size_t)steps + 1);
        const double scale = p->h * (p->n_states == 2 ? 2.0 : 1.0);
        for (int64_t k = 0; k <= steps; ++k)
            hks[(size_t)k] = (float)(scale * ks_value(p->ks_max, p->ks_period, (double)(p->first_step + k) * p->h));
        d_hks.alloc(hks.size());
        d_hks.upload(hks.data(), hks.size(), s);
        OSCB_CUDA(cudaStreamSynchronize(s));        // the staging vector dies at the end of this block
    }
    OSCB_CUDA(cudaEventRecord(ev0, s));
    if (FAST) launch_resident_fast(g, a, *plan, p->n_states, fast, tiles, d_stage.p, d_hks.p);
    else launch_resident<T, MAXT, STRICT>(g, a, tiles, plan->W * 32, smem, idx_smem, plan->weighted);
    OSCB_CUDA(cudaEventRecord(ev1, s));
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            set_error("oscb_run(resident): kernel launch failed: %s (tiles %d, threads %d, smem %zu)", cudaGetErrorString(e),
                      tiles, plan->W * 32, smem);
            throw OscbFail{OSCB_ECUDA};
        }
    }
    k_from_tile_layout<T><<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(d_phi.p, d_io.p, n, R, RT);
    if (out->final_phases) d_io.download(out->final_phases, tot, s);
    if (out->best_states) d_best_states.download(out->best_states, tot, s);
    if (out->best_objective) d_best.download(out->best_objective, R, s);
    std::vector<double> h_energy, h_btrace;
    if (out->energy) { h_energy.resize((size_t)R * S); d_energy.download(h_energy.data(), h_energy.size(), s); }
    if (out->best_trace) { h_btrace.resize((size_t)R * S); d_btrace.download(h_btrace.data(), h_btrace.size(), s); }
    if (out->first_hit_step) d_first.download(h_first.data(), R, s);
    unsigned long long flag = none;
    OSCB_CUDA(cudaMemcpyAsync(&flag, g->d_nonfinite.p, sizeof(flag), cudaMemcpyDeviceToHost, s));
    OSCB_CUDA(cudaStreamSynchronize(s));
    float ms = 0.f;
    OSCB_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    for (int r = 0; r < R; ++r)
        for (int64_t k = 0; k < S; ++k) {
            if (out->energy) out->energy[(size_t)r * out->max_samples + k] = h_energy[(size_t)r * S + k];
            if (out->best_trace) out->best_trace[(size_t)r * out->max_samples + k] = h_btrace[(size_t)r * S + k];
        }
    if (out->first_hit_step)
        for (int r = 0; r < R; ++r) out->first_hit_step[r] = h_first[r];
    out->device_ms = ms;
    out->kernel_launches = 1;
    out->kernel_used = OSCB_KERNEL_RESIDENT;
    out->replicas_per_cta = RT;
    out->smem_bytes = (int64_t)smem;
    if (flag != none) {
        out->nonfinite[2] = (int64_t)(flag >> 36);
        out->nonfinite[0] = (int64_t)((flag >> 20) & 0xFFFFull);
        out->nonfinite[1] = (int64_t)(flag & 0xFFFFFull);
        set_error("non-finite phase for oscillator %lld (replica row %lld) after step %lld; parameters are numerically unstable",
                  (long long)out->nonfinite[1], (long long)out->nonfinite[0], (long long)out->nonfinite[2]);
        throw OscbFail{OSCB_ENONFINITE};
    }
}

static void run_resident(oscb_graph *g, const oscb_run_params *p, int64_t steps, int64_t cadence,
                         const std::vector<long long> &sample_steps, const uint64_t *seeds, int64_t R,
                         const double *phi0, const double *noise, oscb_run_outputs *out)
{
    ResidentConfig cfg;
    OSCB_REQUIRE(choose_resident_config(g, p->precision, p->n_states, R, p->replicas_per_cta, wants_fast(p), &cfg),
                 "the resident kernel cannot hold this problem (n = %lld, max degree %lld); use the streaming kernel",
                 (long long)g->n, (long long)g->max_degree);
    if (p->precision == OSCB_PREC_F64)
        run_resident_impl<double, 512, true, false>(g, p, cfg, steps, cadence, sample_steps, seeds, R, phi0, noise, out);
    else if (!wants_fast(p))   // injected noise / variant 1: the generic kernel
        run_resident_impl<float, 1024, false, false>(g, p, cfg, steps, cadence, sample_steps, seeds, R, phi0, noise, out);
    else
        run_resident_impl<float, 1024, false, true>(g, p, cfg, steps, cadence, sample_steps, seeds, R, phi0, noise, out);
}

} // namespace oscb
