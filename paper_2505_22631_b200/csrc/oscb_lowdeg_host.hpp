// oscb_lowdeg_host.hpp -- host side of k_lowdeg (oscb_lowdeg.cuh): which graphs it takes, the tile shape
// (replicas per CTA, warps, items per thread), the component-major slot map + ELL neighbour stream, and the
// launcher.  See the kernel header for the design.
#pragma once
#include "oscb_host.hpp"
#include "oscb_lowdeg.cuh"
#include "oscb_lowdeg.hpp"

#include <algorithm>
#include <map>
#include <array>
#include <cmath>
#include <limits>
#include <numeric>
#include <cstdlib>
#include <cstring>
#include <type_traits>

namespace oscb {

struct LowdegShape {
    int RT = 1, LRT = 0, C = 32, W = 1, QPT = 1, Q = 0, Qp = 0;
    int rpl = 1;                 // replicas per lane: 2 = k_lowdeg_pair (N = 2, looped stream)
    bool uniform = true;
    size_t smem = 0;
    double cost = 0.0;
};

// pure host result of the stream compiler (also exported to the CPU-side tests)
struct LowdegStreamHost {
    std::vector<uint32_t> quad_of;      // [Qp]
    std::vector<uint32_t> slot_of;      // [n] slot of oscillator i (component-major)
    std::vector<uint32_t> off;          // 4 per group entry: byte offset slot * RT * 8 (bit 31 of the 4th: last group of the row, looped form)
    std::vector<float> wt;              // 4 per group entry: couplings (0 for padding)
    std::vector<int> warp_start;        // looped form: first group row of each warp
    int group_rows = 0;                 // group rows (of C entries) without the prefetch pad
    int64_t real = 0;
    std::vector<int64_t> warp_groups;   // group rows per warp (work balance)
    std::vector<uint32_t> row_groups;   // looped form: [W][QPT] the group counts of an item's four rows, one byte each (saturating at 255)
};

struct LowdegPlan {
    LowdegShape sh;
    int nmode = 2;
    double w_total = 0.0;
    DevBuf<uint32_t> quad_of;
    DevBuf<uint4> soff;
    DevBuf<uint2> sidx;          // two-replica form: u16 slot numbers
    size_t n_ids = 0;            // entries of sidx
    DevBuf<float4> swt;
    DevBuf<int> warp_start;
    DevBuf<uint32_t> row_groups; // two-replica form: group counts of the rows (a byte each), [W][QPT]
};

static size_t lowdeg_smem_bytes(const LowdegShape &s, uint32_t *off_cnt, uint32_t *off_part, uint32_t *off_misc)
{
    size_t o = ((size_t)4 * s.Qp + OSCB_LD_PADS) * s.RT * 8;
    auto take = [&](size_t bytes) { size_t at = o; o += (bytes + 15) & ~(size_t)15; return at; };
    const size_t c = take((size_t)s.RT * 4), p = take((size_t)s.W * s.RT * 8), m = take((size_t)s.RT * 12 + 16);
    if (off_cnt) *off_cnt = (uint32_t)c;
    if (off_part) *off_part = (uint32_t)p;
    if (off_misc) *off_misc = (uint32_t)m;
    return o;
}

// Quads in the order their positions are dealt.  Uniform graphs keep the natural order (lattice-like graphs then
// gather from neighbouring slots); otherwise quads are sorted by the group counts of their four rows so that
// the C quads sharing a warp-instruction need the same number of groups, and the chunks of C are dealt to the
// warps round-robin (the per-warp stream lengths stay within a few groups of each other).
static void compile_lowdeg_stream(int n, const int *indptr, const int *indices, const double *wts, const LowdegShape &s,
                                  bool weighted_stream, LowdegStreamHost *out)
{
    const int Q = s.Q, Qp = s.Qp, C = s.C, W = s.W, QPT = s.QPT, RT = s.RT;
    auto deg = [&](int i) { return i < n ? indptr[i + 1] - indptr[i] : 0; };
    auto groups = [&](int i) { return std::max(1, (deg(i) + 3) / 4); };
    std::vector<int> order(Q);
    std::iota(order.begin(), order.end(), 0);
    // k_lowdeg_pair walks the four rows of a quad in descending degree (rowsel[q][k] = the component visited k-th), so the
    // rows that share a warp-row's k-th trip have similar lengths: a quad's long row no longer meets its neighbours' short
    // ones (G22 shape: 0.82 -> 0.90 of the stream entries are real neighbours).  The permutation travels in the top byte
    // of the quad table; slots, registers and stream are all in visiting order, only the noise component, the state
    // byte and the phase I/O look the component up.
    const bool sort_rows = s.rpl == 2 && !s.uniform;
    std::vector<std::array<uint8_t, 4>> rowsel(Q, std::array<uint8_t, 4>{0, 1, 2, 3});
    if (sort_rows)
        for (int q = 0; q < Q; ++q)
            std::stable_sort(rowsel[q].begin(), rowsel[q].end(), [&](uint8_t x, uint8_t y) { return deg(4 * q + x) > deg(4 * q + y); });
    if (!s.uniform) {
        std::vector<std::array<int, 4>> key(Q);
        for (int q = 0; q < Q; ++q)
            key[q] = {groups(4 * q + rowsel[q][0]), groups(4 * q + rowsel[q][1]), groups(4 * q + rowsel[q][2]), groups(4 * q + rowsel[q][3])};
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return key[x] > key[y]; });
    }
    // k_lowdeg_pair: the bank group of an oscillator's slot is its quad's place in the chunk mod Hq (see the row scheduling
    // below), and a row whose neighbours crowd into one bank group collides with its quarter-warp partners whatever their
    // order.  Swap quads of different bank groups inside a chunk (the chunk contents, hence the padding, stay as sorted)
    // while that evens out the rows' neighbour counts per bank group: sum over rows and groups of count^2, local search.
    const int Hq = std::max(1, std::min(C, 128 / (RT * 8)));
    if (sort_rows && Hq >= 2) {
        std::vector<int> cls(Q), cnt((size_t)n * Hq, 0);
        for (int idx = 0; idx < Q; ++idx) cls[order[idx]] = (idx % C) % Hq;
        for (int r = 0; r < n; ++r)
            for (int e = indptr[r]; e < indptr[r + 1]; ++e) ++cnt[(size_t)r * Hq + cls[indices[e] >> 2]];
        // move every oscillator of quad q from bank group a to b: returns the change of the objective (the CSR is symmetric:
        // the rows that see oscillator x are x's own neighbours)
        auto move = [&](int q, int a, int b) {
            long long d = 0;
            for (int x = 4 * q; x < std::min(n, 4 * q + 4); ++x)
                for (int e = indptr[x]; e < indptr[x + 1]; ++e) {
                    int *c = &cnt[(size_t)indices[e] * Hq];
                    d += 2 * (c[b] - c[a]) + 2;
                    --c[a];
                    ++c[b];
                }
            return d;
        };
        for (int pass = 0; pass < 6; ++pass) {
            bool any = false;
            for (int j0 = 0; j0 < Q; j0 += C) {
                const int m = std::min(C, Q - j0);
                for (int x = 0; x < m; ++x)
                    for (int y = x + 1; y < m; ++y) {
                        const int qa = order[j0 + x], qb = order[j0 + y], a = x % Hq, b = y % Hq;
                        if (a == b) continue;
                        const long long d = move(qa, a, b) + move(qb, b, a);
                        if (d < 0) { std::swap(order[j0 + x], order[j0 + y]); any = true; }
                        else { move(qb, a, b); move(qa, b, a); }
                    }
            }
            if (!any) break;
        }
    }
    // chunk j of C quads -> warp-row (t, w)
    out->quad_of.assign(Qp, 0xFFFFFFFFu);
    const int chunks = (Q + C - 1) / C;
    OSCB_REQUIRE(chunks <= W * QPT, "internal: lowdeg tile shape too small");
    for (int j = 0; j < chunks; ++j) {
        int t = j / W, w = j % W;
        if (!s.uniform && (t & 1)) w = W - 1 - w;                       // boustrophedon: balance the sorted chunks
        for (int c = 0; c < C && j * C + c < Q; ++c) out->quad_of[(size_t)(t * W + w) * C + c] = (uint32_t)order[j * C + c];
    }
    out->slot_of.assign(n, 0);
    for (int pos = 0; pos < Qp; ++pos) {
        const uint32_t q = out->quad_of[pos];
        if (q >= (uint32_t)Q) continue;
        for (int k = 0; k < 4; ++k)
            if (4 * (int)q + rowsel[q][k] < n) out->slot_of[4 * q + rowsel[q][k]] = (uint32_t)(k * Qp + pos);
    }
    out->off.clear();
    out->wt.clear();
    out->real = 0;
    out->warp_start.assign(W, 0);
    out->warp_groups.assign(W, 0);
    // Looped streams of k_lowdeg_pair: an LDS.128 is served a quarter-warp at a time, i.e. H = 128 / (RT * 8) consecutive
    // slots per 128-byte wavefront, and two of them collide when their targets fall in the same bank group (slot number mod
    // H) at different addresses.  The rows of such a group of H slots are therefore scheduled TOGETHER: at every position
    // each row takes a neighbour from a bank group nobody else in the quarter-warp uses; a row that has none left of a free
    // group spends one of its padding reads there instead (a row shorter than its warp-row's 4 G positions may pad
    // anywhere, and a pad slot exists for every bank group).  G22 shape, 8 replicas per tile: 1.40 wavefronts per ideal one
    // in CSR order, ~1.13 with each row ordered on its own, ~1.03 jointly.  Uniform streams keep the CSR order
    // (lattice-like graphs gather from neighbouring slots as they are), and so does the one-replica-per-lane kernel, whose
    // results then do not depend on the tile shape.  Float32 sums depend on the order, so k_lowdeg_pair's last bits depend
    // on the tile shape (like k_resident_fast's); the float64 parity mode always sums in CSR order.
    const int H = std::max(1, std::min(C, 128 / (RT * 8)));
    const bool joint = !s.uniform && H >= 2 && s.rpl == 2;
    // sched[c]: for every position of slot c's row in the current warp-row, a CSR entry, or -(1 + bank group) for padding
    std::vector<std::vector<int>> sched(C);
    auto schedule_rows = [&](const int *rows, int G) {
        const int P = 4 * G;
        for (int c = 0; c < C; ++c) sched[c].assign(P, -1);
        if (!joint) {
            for (int c = 0; c < C; ++c) {
                const int i = rows[c], d = i >= 0 ? deg(i) : 0;
                for (int u = 0; u < P; ++u) sched[c][u] = u < d ? indptr[i] + u : -(1 + c % OSCB_LD_PADS);
            }
            return;
        }
        for (int c0 = 0; c0 < C; c0 += H) {
            std::vector<std::vector<std::vector<int>>> bucket(H, std::vector<std::vector<int>>(H));   // [slot][bank group] -> CSR entries, reversed
            int left[32];
            for (int j = 0; j < H; ++j) {
                const int i = rows[c0 + j];
                left[j] = i >= 0 ? deg(i) : 0;
                if (i >= 0)
                    for (int e = indptr[i + 1] - 1; e >= indptr[i]; --e) bucket[j][out->slot_of[indices[e]] % H].push_back(e);
            }
            for (int pos = 0; pos < P; ++pos) {
                int order[32];
                for (int j = 0; j < H; ++j) order[j] = j;
                // rows with the least padding left choose first; position-dependent tie-break spreads the leftovers
                std::stable_sort(order, order + H, [&](int x, int y) { return (P - pos - left[x]) < (P - pos - left[y]); });
                uint32_t used = 0;
                int pads[32], n_pads = 0;
                for (int oi = 0; oi < H; ++oi) {
                    const int j = order[oi];
                    if (left[j] == 0) { pads[n_pads++] = j; continue; }
                    int cls = -1;
                    for (int k = 0; k < H; ++k) {
                        const int cand = (j + pos + k) % H;
                        if (!(used >> cand & 1u) && !bucket[j][cand].empty() && (cls < 0 || bucket[j][cand].size() > bucket[j][cls].size())) cls = cand;
                    }
                    if (cls < 0) {
                        if (P - pos - left[j] > 0) { pads[n_pads++] = j; continue; }       // pad here, keep the neighbours for later
                        for (int k = 0; k < H; ++k)
                            if (!bucket[j][k].empty() && (cls < 0 || bucket[j][k].size() > bucket[j][cls].size())) cls = k;
                    }
                    sched[c0 + j][pos] = bucket[j][cls].back();
                    bucket[j][cls].pop_back();
                    --left[j];
                    used |= 1u << cls;
                }
                for (int q = 0; q < n_pads; ++q) {
                    int cls = pads[q] % H;
                    for (int k = 0; k < H; ++k)
                        if (!(used >> ((pads[q] + k) % H) & 1u)) { cls = (pads[q] + k) % H; break; }
                    used |= 1u << cls;
                    sched[c0 + pads[q]][pos] = -(1 + cls);
                }
            }
        }
    };
    // one group entry of slot c: positions [4 g, 4 g + 4) of its scheduled row
    auto emit = [&](int g, int c, bool last) {
        for (int u = 0; u < 4; ++u) {
            const int e = sched[c][4 * g + u];
            const bool real = e >= 0;
            uint32_t o = real ? (uint32_t)(out->slot_of[indices[e]] * RT * 8) : (uint32_t)(((uint32_t)4 * Qp + (uint32_t)(-e - 1)) * RT * 8);
            if (u == 3 && last) o |= 0x80000000u;
            out->off.push_back(o);
            out->wt.push_back(real ? (wts ? (float)wts[e] : 1.0f) : 0.0f);
            if (real) ++out->real;
        }
    };
    auto row_of = [&](int t, int w, int c, int k) -> int {
        const uint32_t q = out->quad_of[(size_t)(t * W + w) * C + c];
        return q < (uint32_t)Q && 4 * (int)q + rowsel[q][k] < n ? 4 * (int)q + rowsel[q][k] : -1;
    };
    if (s.uniform) {
        // [t][w][k][c], one group per row
        std::vector<int> rows_now(C);
        for (int t = 0; t < QPT; ++t)
            for (int w = 0; w < W; ++w)
                for (int k = 0; k < 4; ++k) {
                    for (int c = 0; c < C; ++c) rows_now[c] = row_of(t, w, c, k);
                    schedule_rows(rows_now.data(), 1);
                    for (int c = 0; c < C; ++c) emit(0, c, false);
                }
        out->group_rows = QPT * W * 4;
        for (int w = 0; w < W; ++w) out->warp_groups[w] = (int64_t)QPT * 4;
    } else {
        // per warp: t, k, g in the order the kernel walks them
        int rows = 0, max_groups = 0;
        std::vector<int> rows_now(C);
        out->row_groups.assign((size_t)W * QPT, 0);
        for (int w = 0; w < W; ++w) {
            out->warp_start[w] = rows;
            for (int t = 0; t < QPT; ++t)
                for (int k = 0; k < 4; ++k) {
                    int G = 1;
                    for (int c = 0; c < C; ++c) {
                        const int i = rows_now[c] = row_of(t, w, c, k);
                        if (i >= 0) G = std::max(G, groups(i));
                    }
                    schedule_rows(rows_now.data(), G);
                    out->row_groups[(size_t)w * QPT + t] |= (uint32_t)std::min(G, 255) << (8 * k);
                    max_groups = std::max(max_groups, G);
                    for (int g = 0; g < G; ++g) {
                        for (int c = 0; c < C; ++c) emit(g, c, g == G - 1);
                        ++rows;
                    }
                }
            out->warp_groups[w] = rows - out->warp_start[w];
        }
        out->group_rows = rows;
        OSCB_REQUIRE(s.rpl != 2 || max_groups <= 255, "k_lowdeg_pair takes rows of up to 1020 neighbours");
        std::fill(rows_now.begin(), rows_now.end(), -1);
        schedule_rows(rows_now.data(), 1);
        for (int c = 0; c < C; ++c) emit(0, c, true);           // the prefetch pad row
    }
    if (sort_rows) {
        OSCB_REQUIRE(Q < 0xFFFFFF, "internal: quad numbers exceed 24 bits");
        for (uint32_t &qw : out->quad_of)
            if (qw < (uint32_t)Q) {
                const auto &r = rowsel[qw];
                qw |= (uint32_t)(r[0] | (r[1] << 2) | (r[2] << 4) | (r[3] << 6)) << 24;
            }
    }
    (void)weighted_stream;
}

// is this run one for k_lowdeg at all?
static bool lowdeg_kind(const oscb_graph *g, const oscb_run_params *p, int *nmode)
{
    if (g->is_dense || p->precision != OSCB_PREC_F32 || p->noise_mode == OSCB_NOISE_HOST || p->variant == 1) return false;
    if (g->n < 4 || g->nnz == 0) return false;
    if (p->n_states == 2 && p->objective == OSCB_OBJ_MAXCUT) {
        if (!g->unit_weights) {
            if (!g->int_weights) return false;
            double tot = 0.0, mx = 0.0;
            for (double w : g->h_w) { tot += std::fabs(w); mx = std::max(mx, std::fabs(w)); }
            if (mx > 65536.0 || tot >= 8388608.0) return false;       // float32 / int32 sums of couplings stay exact
        } else if ((double)g->nnz >= 8388608.0) return false;
        *nmode = 2;
        return true;
    }
    if (p->n_states == 3 && p->objective == OSCB_OBJ_COLORING && g->unit_weights) {
        *nmode = 3;
        return true;
    }
    return false;
}

static const int kLowdegQpt[] = {1, 2, 4, 5, 7, 10};

// the tile shape with the lowest estimated time; false when the kernel does not apply
static bool choose_lowdeg_shape(const oscb_graph *g, const oscb_run_params *p, int64_t R, bool forced, LowdegShape *out)
{
    int nmode;
    if (!lowdeg_kind(g, p, &nmode)) return false;
    // low degree: the instruction count per row is what matters; k_resident_fast wins from ~degree 10 on
    if (!forced && (g->max_degree > 16 || (double)g->nnz / (double)g->n > 8.0)) return false;
    const bool uniform = g->max_degree <= 4;
    const int Q = (int)((g->n + 3) / 4);
    double best = std::numeric_limits<double>::infinity();
    bool found = false;
    // OSCB_LOWDEG_RT / OSCB_LOWDEG_QPT pin the tile shape (tuning experiments)
    int want_rt = p->replicas_per_cta, want_qpt = 0;
    if (const char *e = getenv("OSCB_LOWDEG_RT")) { if (want_rt <= 0) want_rt = atoi(e); }
    if (const char *e = getenv("OSCB_LOWDEG_QPT")) want_qpt = atoi(e);
    int want_rpl = 0;
    if (const char *e = getenv("OSCB_LOWDEG_RPL")) want_rpl = atoi(e);
    for (int l = 5; l >= 0; --l) {
        const int RT = 1 << l;
        if (want_rt > 0 && RT != want_rt) continue;
        if (want_rt <= 0 && RT > 1 && RT / 2 >= R) continue;      // do not pad a tile more than 2x
      for (int rpl = 1; rpl <= 2; ++rpl) {
        // two replicas per lane (k_lowdeg_pair): N = 2 on a looped stream, tiles of an even number of replicas
        if (rpl == 2 && (nmode != 2 || uniform || RT < 2 || g->max_degree > 1020)) continue;
        if (want_rpl > 0 && rpl != want_rpl) continue;
        const int C = 32 * rpl / RT;
        const int rows = (Q + C - 1) / C;
        for (int QPT : kLowdegQpt) {
            if (want_qpt > 0 && QPT != want_qpt) continue;
            if (rpl == 2 && QPT > 5) continue;
            const int maxW = (rpl == 2 ? lowdeg_pair_max_threads(QPT) : lowdeg_max_threads(QPT)) / 32;
            const int W = (rows + QPT - 1) / QPT;
            if (W > maxW || W < 1) continue;
            LowdegShape s;
            s.RT = RT; s.LRT = l; s.C = C; s.W = W; s.QPT = QPT; s.Q = Q; s.Qp = W * QPT * C; s.uniform = uniform; s.rpl = rpl;
            s.smem = lowdeg_smem_bytes(s, nullptr, nullptr, nullptr);
            if (s.smem > (size_t)g->smem_optin) continue;
            // work of one CTA in warp-rows (idle lanes and ghost items included), CTAs resident per SM, and the
            // busiest SM's share of the tiles
            const int64_t tiles = (R + RT - 1) / RT;
            const int by_smem = (int)std::max<size_t>(1, ((size_t)g->smem_optin + 1024) / (s.smem + 1024));
            const int by_threads = std::max(1, 2048 / (W * 32));
            const int cps = std::min({by_smem, by_threads, 32});
            const int64_t slots = (int64_t)g->sm_count * cps;
            const int64_t waves = (tiles + slots - 1) / slots;
            const int64_t per_sm = std::min<int64_t>(cps, (tiles + g->sm_count - 1) / g->sm_count);
            double pad = 1.0;                                    // looped streams pad rows to the widest of C quads
            if (!uniform) pad = 1.0 + 0.04 * (C - 1);
            // few resident warps cannot hide the shared-memory and MUFU latencies
            const double warps_resident = (double)per_sm * W;
            const double occ = warps_resident >= 16 ? 1.0 : std::sqrt(16.0 / warps_resident);
            // (a warp-row of two-replica lanes does the gathers of twice the replicas for ~1.2-1.5x the instructions: measured ahead of one replica per lane on every looped N = 2 graph tried)
            s.cost = (double)waves * (double)per_sm * (double)W * QPT * pad * occ * (rpl == 2 ? 1.2 : 1.0);
            if (s.cost < best - 1e-9) { best = s.cost; *out = s; found = true; }
        }
      }
    }
    return found;
}

static std::shared_ptr<LowdegPlan> get_lowdeg_plan(oscb_graph *g, const LowdegShape &s, int nmode)
{
    const uint64_t key = (1ull << 63) | ((uint64_t)s.rpl << 48) | ((uint64_t)s.RT << 40) | ((uint64_t)s.W << 24) | ((uint64_t)s.QPT << 8) | (uint64_t)nmode;
    auto it = g->lowdeg_plans.find(key);
    if (it != g->lowdeg_plans.end()) return it->second;
    auto plan = std::make_shared<LowdegPlan>();
    plan->sh = s;
    plan->nmode = nmode;
    LowdegStreamHost h;
    compile_lowdeg_stream((int)g->n, g->h_indptr.data(), g->h_indices.data(), g->unit_weights ? nullptr : g->h_w.data(), s,
                          nmode == 2, &h);
    OSCB_REQUIRE(h.real == g->nnz, "internal: lowdeg plan lost neighbours (%lld of %lld)", (long long)h.real, (long long)g->nnz);
    double wt = 0.0;
    for (int64_t e = 0; e < g->nnz; ++e) wt += g->unit_weights ? 1.0 : g->h_w[e];
    plan->w_total = wt;
    cudaStream_t st = g->stream;
    plan->quad_of.alloc(h.quad_of.size());
    plan->quad_of.upload(h.quad_of.data(), h.quad_of.size(), st);
    const size_t entries = h.off.size() / 4;
    std::vector<uint2> idx16;
    if (s.rpl == 2) {
        OSCB_REQUIRE((size_t)4 * s.Qp + OSCB_LD_PADS <= 65536, "internal: k_lowdeg_pair slot numbers exceed 16 bits");
        idx16.resize(entries);
        const uint32_t sb = (uint32_t)s.RT * 8u;
        for (size_t e = 0; e < entries; ++e) {
            uint32_t id[4];
            for (int u = 0; u < 4; ++u) id[u] = (h.off[4 * e + u] & 0x7fffffffu) / sb;
            idx16[e] = make_uint2(id[0] | (id[1] << 16), id[2] | (id[3] << 16));
        }
        plan->sidx.alloc(entries);
        plan->sidx.upload(idx16.data(), entries, st);
        plan->n_ids = entries;
        plan->row_groups.alloc(h.row_groups.size());
        plan->row_groups.upload(h.row_groups.data(), h.row_groups.size(), st);
    }
    plan->soff.alloc(entries);
    plan->soff.upload(reinterpret_cast<const uint4 *>(h.off.data()), entries, st);
    if (nmode == 2) {
        plan->swt.alloc(entries);
        plan->swt.upload(reinterpret_cast<const float4 *>(h.wt.data()), entries, st);
    }
    plan->warp_start.alloc(h.warp_start.size());
    plan->warp_start.upload(h.warp_start.data(), h.warp_start.size(), st);
    OSCB_CUDA(cudaStreamSynchronize(st));
    g->lowdeg_plans[key] = plan;
    return plan;
}

// k_lowdeg_pair beyond the low degrees: a unit-coupling N = 2 max-cut graph of any degree whose slot stream fits in shared
// memory behind the pairs of an 8-replica tile (the G22 shape: 130 + 90 KB), when the batch fills the GPU with such tiles.
// There the pair kernel's leaner per-oscillator part beats k_resident_fast (2.18 vs 2.10 T updates/s on G22 x 1024).  Off
// that shape -- stream from L1 / L2, other tile sizes, weighted rows -- k_resident_fast measured ahead and keeps the run.
static bool lowdeg_pair_resident_shape(oscb_graph *g, const oscb_run_params *p, int64_t R, LowdegShape *out)
{
    int nmode;
    if (!lowdeg_kind(g, p, &nmode) || nmode != 2 || !g->unit_weights || g->max_degree <= 4 || g->max_degree > 1020) return false;
    if (getenv("OSCB_LOWDEG_RT") || getenv("OSCB_LOWDEG_QPT") || getenv("OSCB_LOWDEG_RPL")) return false;   // pinned shapes: the general chooser
    const int Q = (int)((g->n + 3) / 4);
    const int64_t sms = g->sm_count;
    // tiles of 8 replicas once tiles of 4 no longer fit one per SM (measured on the G22 shape: 2.45 T at 1024 replicas, 1.52 T
    // at 640 against 1.29 T for k_resident_fast); tiles of 4 below that while they still fill most of the GPU (2.02 T at 512
    // against 1.71 T, 2.34 T at 592 against 1.98 T); smaller batches stay with k_resident_fast's 1- and 2-replica tiles
    for (int RT : {8, 4}) {
        if (p->replicas_per_cta > 0 && p->replicas_per_cta != RT) continue;
        const int64_t tiles = (R + RT - 1) / RT;
        int64_t min_tiles = RT == 8 ? sms / 2 + 1 : sms * 3 / 5;
        if (const char *e = getenv("OSCB_LOWDEG_PAIR_MIN_TILES")) min_tiles = atoll(e);       // (tuning experiments)
        if (tiles < min_tiles || (RT == 4 && tiles > sms)) continue;
        const int C = 64 / RT, rows = (Q + C - 1) / C;
        for (int QPT : {RT == 8 ? 4 : 2, RT == 8 ? 5 : 4, RT == 8 ? 2 : 5}) {          // (16 warps of 128 registers measured best on both)
            const int W = (rows + QPT - 1) / QPT;
            if (W < (RT == 8 ? 8 : 4) || W > lowdeg_pair_max_threads(QPT) / 32) continue;
            LowdegShape s;
            s.RT = RT; s.LRT = RT == 8 ? 3 : 2; s.C = C; s.W = W; s.QPT = QPT; s.Q = Q; s.Qp = W * QPT * C; s.uniform = false; s.rpl = 2;
            s.smem = lowdeg_smem_bytes(s, nullptr, nullptr, nullptr);
            s.cost = 0.0;
            if (s.smem > (size_t)g->smem_optin || (size_t)4 * s.Qp + OSCB_LD_PADS > 65536) continue;
            if (s.smem + (size_t)g->nnz * 2 > (size_t)g->smem_optin) continue;        // even an unpadded stream would not fit
            auto plan = get_lowdeg_plan(g, s, nmode);
            if (s.smem + ((plan->n_ids * sizeof(uint2) + 15) & ~(size_t)15) > (size_t)g->smem_optin) continue;
            *out = s;
            return true;
        }
    }
    return false;
}

// The tile decomposition quantises the work of a batch: 1024 replicas are 128 tiles of 8, one per SM, and 20 SMs of a B200
// idle (a 7-replica tile costs what an 8-replica one costs).  A 4-replica tile advances a step in ~0.6 of the time of an
// 8-replica one, so a + b = all SMs tiles with 8a + 4b = R keep every SM busy if the replicas take turns in the fast lane:
// the run is cut into windows; in a window F = b / 2 "octets" (groups of 8 replicas) run as two 4-replica tiles for steps4
// steps while the other a run as 8-replica tiles for steps8 < steps4 steps, the fast set rotates, and after `windows`
// windows every octet has been fast `turns` times: (windows - turns) * steps8 + turns * steps4 = steps for all of them.
// Phases, best states and traces live in global memory between windows; the noise is a function of (seed, step, oscillator)
// and the schedule of the step number, so a replica's trajectory is the one of an unbroken run up to the float32 summation
// order of the tile shape it happens to be in (which differs between shapes anyway).
struct MixedTiles {
    LowdegShape s4;
    int tiles8 = 0, tiles4 = 0, fast_octets = 0, windows = 0, turns = 0;
    int64_t steps8 = 0, steps4 = 0;
};

// (k_lowdeg, one replica per lane, takes part too: flat200 x 4096 is 128 tiles of 32 replicas -> 108 tiles of 32 and 40 of 16.
// The field names keep the numbers of the two-replica case: "8" = the big tile, "4" = the half-size one, octet = a group of
// one big tile's replicas.)
static bool plan_mixed_tiles(oscb_graph *g, const oscb_run_params *p, const LowdegShape &s8, int nmode, int64_t R, int64_t steps, MixedTiles *m)
{
    if (const char *e = getenv("OSCB_LOWDEG_MIXED")) { if (atoi(e) == 0) return false; }
    if (p->replicas_per_cta > 0 || getenv("OSCB_LOWDEG_RT") || getenv("OSCB_LOWDEG_QPT")) return false;     // pinned shapes run as they are
    const int B = s8.RT;
    if (s8.rpl == 2 ? (B != 8 || !g->unit_weights) : (B < 4)) return false;
    if (R % B != 0) return false;
    const int64_t sms = g->sm_count, octets = R / B;
    if (octets >= sms || R < (B / 2) * sms) return false;           // one big tile per SM fills the GPU / half-size tiles alone do
    const int64_t F = sms - octets;                                 // a = octets - F big tiles, b = 2 F half-size ones: a + b = sms
    if (F < 1 || octets - F < 1) return false;
    int64_t gg = octets, x = F;
    while (x) { const int64_t t = gg % x; gg = x; x = t; }
    const int64_t windows = octets / gg, turns = F / gg;
    int64_t min_window = 256;
    if (const char *e = getenv("OSCB_LOWDEG_MIXED_MIN_WINDOW")) min_window = std::max<long long>(1, atoll(e));     // (tests)
    if (windows > 64 || steps < windows * min_window) return false;
    // the half-size tile: twice the quads per warp; two replicas per lane: 16 warps of two items, slot stream in shared memory
    LowdegShape s4;
    const int C = 2 * s8.C, rows = (s8.Q + C - 1) / C;
    bool found = false;
    const int qpt2[] = {2, 4, 5}, qpt1[] = {std::max(1, s8.QPT / 2), s8.QPT, 1, 2, 4, 5, 7, 10};
    const int *cand = s8.rpl == 2 ? qpt2 : qpt1;
    const int n_cand = s8.rpl == 2 ? 3 : 8;
    for (int ci = 0; ci < n_cand && !found; ++ci) {
        const int QPT = cand[ci];
        if (std::find(std::begin(kLowdegQpt), std::end(kLowdegQpt), QPT) == std::end(kLowdegQpt)) continue;
        const int W = (rows + QPT - 1) / QPT;
        const int maxW = (s8.rpl == 2 ? lowdeg_pair_max_threads(QPT) : lowdeg_max_threads(QPT)) / 32;
        if (W < (s8.rpl == 2 ? 4 : 1) || W > maxW) continue;
        s4 = s8;
        s4.RT = B / 2; s4.LRT = s8.LRT - 1; s4.C = C; s4.W = W; s4.QPT = QPT; s4.Qp = W * QPT * C;
        s4.smem = lowdeg_smem_bytes(s4, nullptr, nullptr, nullptr);
        if (s4.smem > (size_t)g->smem_optin) continue;
        if (s8.rpl == 2) {
            if ((size_t)4 * s4.Qp + OSCB_LD_PADS > 65536) continue;
            auto plan4 = get_lowdeg_plan(g, s4, nmode);
            if (s4.smem + ((plan4->n_ids * sizeof(uint2) + 15) & ~(size_t)15) > (size_t)g->smem_optin) continue;
        }
        found = true;
    }
    if (!found) return false;
    // steps of a window in the two lanes: steps4 / steps8 ~ the measured ratio of the step times (G22 shape, tiles of 8 and 4:
    // 16.7 / 9.2 us; flat200, tiles of 32 and 16: 4.29 / 2.54 us)
    double ratio = s8.rpl == 2 ? 1.8 : 1.7;
    if (const char *e = getenv("OSCB_LOWDEG_MIXED_RATIO")) ratio = std::max(1.0, atof(e));
    const int64_t slow = windows - turns;
    int64_t w0 = (int64_t)std::llround((double)steps / ((double)slow + (double)turns * ratio));
    int64_t steps8 = -1;
    for (int64_t d = 0; d <= turns && steps8 < 0; ++d)
        for (int64_t w : {w0 - d, w0 + d})
            if (w >= 1 && steps - slow * w >= turns && (steps - slow * w) % turns == 0 && (steps - slow * w) / turns >= w) { steps8 = w; break; }
    if (steps8 < 0) return false;
    m->s4 = s4; m->tiles8 = (int)(octets - F); m->tiles4 = (int)(2 * F); m->fast_octets = (int)F;
    m->windows = (int)windows; m->turns = (int)turns; m->steps8 = steps8; m->steps4 = (steps - slow * steps8) / turns;
    return true;
}

bool lowdeg_applies(oscb_graph *g, const oscb_run_params *p, int64_t R, bool forced)
{
    LowdegShape s;
    if (choose_lowdeg_shape(g, p, R, false, &s) || lowdeg_pair_resident_shape(g, p, R, &s)) return true;
    return forced && choose_lowdeg_shape(g, p, R, true, &s);
}

template <int NMODE, bool UNIFORM, bool RT1, bool WIN = false>
static void launch_lowdeg(oscb_graph *g, const LowdegArgs &a, const LowdegShape &s, int tiles, cudaStream_t stream = nullptr, size_t smem_request = 0)
{
    const size_t smem = std::max(s.smem, smem_request);
    auto go = [&](auto kernel) {
        OSCB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kernel<<<tiles, s.W * 32, smem, stream ? stream : g->stream>>>(a);
    };
    switch (s.QPT) {
    case 1: go(k_lowdeg<NMODE, 1, UNIFORM, RT1, WIN>); break;
    case 2: go(k_lowdeg<NMODE, 2, UNIFORM, RT1, WIN>); break;
    case 4: go(k_lowdeg<NMODE, 4, UNIFORM, RT1, WIN>); break;
    case 5: go(k_lowdeg<NMODE, 5, UNIFORM, RT1, WIN>); break;
    case 7: go(k_lowdeg<NMODE, 7, UNIFORM, RT1, WIN>); break;
    case 10: go(k_lowdeg<NMODE, 10, UNIFORM, RT1, WIN>); break;
    default: OSCB_REQUIRE(false, "internal: no lowdeg instantiation for %d items per thread", s.QPT);
    }
}

template <bool UNITW, bool IDS>
static void launch_lowdeg_pair(oscb_graph *g, const LowdegArgs &a, const LowdegShape &s, int tiles, size_t smem, cudaStream_t stream = nullptr)
{
    auto go = [&](auto kernel) {
        OSCB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kernel<<<tiles, s.W * 32, smem, stream ? stream : g->stream>>>(a);
    };
    switch (s.QPT) {
    case 1: go(k_lowdeg_pair<1, UNITW, IDS>); break;
    case 2: go(k_lowdeg_pair<2, UNITW, IDS>); break;
    case 4: go(k_lowdeg_pair<4, UNITW, IDS>); break;
    case 5: go(k_lowdeg_pair<5, UNITW, IDS>); break;
    default: OSCB_REQUIRE(false, "internal: no k_lowdeg_pair instantiation for %d items per thread", s.QPT);
    }
}

void run_lowdeg(oscb_graph *g, const oscb_run_params *p, int64_t steps, int64_t cadence,
                       const std::vector<long long> &sample_steps, const uint64_t *seeds, int64_t R64, const double *phi0,
                       oscb_run_outputs *out)
{
    cudaStream_t s = g->stream;
    const int n = (int)g->n, R = (int)R64;
    LowdegShape sh;
    int nmode = 2;
    OSCB_REQUIRE(lowdeg_kind(g, p, &nmode) && (choose_lowdeg_shape(g, p, R, false, &sh) || lowdeg_pair_resident_shape(g, p, R, &sh) ||
                                                 choose_lowdeg_shape(g, p, R, true, &sh)),
                 "the low-degree kernel takes float32, device noise, max degree <= 16 and N = 2 max-cut on integer couplings "
                 "or N = 3 colouring on unit couplings");
    auto plan = get_lowdeg_plan(g, sh, nmode);
    const int RT = sh.RT, tiles = (R + RT - 1) / RT, R_pad = tiles * RT, n4 = 4 * sh.Q;
    const int maximize = p->objective == OSCB_OBJ_MAXCUT;
    const int64_t S = 1 + (int64_t)sample_steps.size();
    const size_t tot = (size_t)n * R;

    DevBuf<double> d_io(tot);
    std::vector<uint64_t> h_seeds(R_pad, 0);
    std::copy(seeds, seeds + R, h_seeds.begin());
    DevBuf<uint64_t> d_seeds(R_pad);
    d_seeds.upload(h_seeds.data(), R_pad, s);
    DevBuf<double> d_best(R_pad), d_energy((size_t)R_pad * S), d_btrace((size_t)R_pad * S);
    DevBuf<uint8_t> d_best_states((size_t)R_pad * n4);
    DevBuf<long long> d_first(R_pad);
    DevBuf<int> d_samples(std::max<size_t>(1, sample_steps.size()));
    std::vector<double> h_best(R_pad, maximize ? -std::numeric_limits<double>::infinity() : std::numeric_limits<double>::infinity());
    std::vector<long long> h_first(R_pad, -1);
    std::vector<int> h_samples(sample_steps.begin(), sample_steps.end());
    for (auto &v : h_samples) v += (int)p->first_step;
    d_best.upload(h_best.data(), R_pad, s);
    d_first.upload(h_first.data(), R_pad, s);
    d_samples.upload(h_samples.data(), h_samples.size(), s);
    d_best_states.zero(s);
    const unsigned long long none = ~0ull;
    OSCB_CUDA(cudaMemcpyAsync(g->d_nonfinite.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));
    if (phi0) d_io.upload(phi0, tot, s);
    else launch_initial_phases(d_seeds.p, d_io.p, n, R, s);

    // h * ks(step) (x2 for N = 2, where the SHIL term is 2 s c) for every step, in the reference's float64
    std::vector<float> hks((size_t)steps + 1);
    const double scale = p->h * (p->n_states == 2 ? 2.0 : 1.0);
    for (int64_t k = 0; k <= steps; ++k)
        hks[(size_t)k] = (float)(scale * ks_value(p->ks_max, p->ks_period, (double)(p->first_step + k) * p->h));
    DevBuf<float> d_hks(hks.size());
    d_hks.upload(hks.data(), hks.size(), s);

    LowdegArgs a;
    memset(&a, 0, sizeof(a));
    a.n = n; a.Q = sh.Q; a.Qp = sh.Qp; a.RT = RT; a.LRT = sh.LRT; a.C = sh.C; a.W = sh.W; a.R_real = R; a.n4 = n4;
    lowdeg_smem_bytes(sh, &a.off_cnt, &a.off_part, &a.off_misc);
    a.hK = (float)(p->h * p->K);
    a.knsh = (float)(p->kn * std::sqrt(p->h));
    a.noise_on = (p->noise_mode == OSCB_NOISE_DEVICE && p->kn != 0.0) ? 1 : 0;
    a.maximize = maximize; a.use_target = p->use_target; a.n_sample_steps = (int)sample_steps.size();
    a.step_begin = (int)p->first_step; a.step_end = (int)(p->first_step + steps); a.cadence = (int)cadence; a.trace_stride = S;
    a.target = p->target_objective; a.w_total = plan->w_total;
    a.quad_of = plan->quad_of.p; a.soff = plan->soff.p; a.sidx = plan->sidx.p; a.swt = plan->swt.p; a.warp_start = plan->warp_start.p; a.row_groups = plan->row_groups.p;
    a.hks_table = d_hks.p; a.seeds = d_seeds.p; a.sample_steps = d_samples.p;
    if (nmode == 3) fast_state_boundaries(3, a.bnd);
    a.io = d_io.p; a.best_obj = d_best.p; a.energy = d_energy.p; a.best_trace = d_btrace.p; a.best_states = d_best_states.p;
    a.first_hit = d_first.p; a.nonfinite = g->d_nonfinite.p;

    size_t launched_smem = sh.smem;
    cudaEvent_t ev0, ev1;
    OSCB_CUDA(cudaEventCreate(&ev0));
    OSCB_CUDA(cudaEventCreate(&ev1));
    OSCB_CUDA(cudaStreamSynchronize(s));        // the host staging vectors above must outlive their copies
    OSCB_CUDA(cudaEventRecord(ev0, s));
    auto by_shape = [&](auto nm) {
        constexpr int NM = decltype(nm)::value;
        if (sh.uniform && RT == 1) launch_lowdeg<NM, true, true>(g, a, sh, tiles);       // (RT1 only with the straight-line stream)
        else if (sh.uniform) launch_lowdeg<NM, true, false>(g, a, sh, tiles);
        else launch_lowdeg<NM, false, false>(g, a, sh, tiles);
    };
    int launches = 1;
    MixedTiles mix;
    if (plan_mixed_tiles(g, p, sh, nmode, R, steps, &mix)) {
        // 8a + 4b = R replicas on a + b = all SMs (see plan_mixed_tiles): every window launches the a big tiles and the b
        // half-size tiles side by side on two streams; a window ends when both have.
        auto plan4 = get_lowdeg_plan(g, mix.s4, nmode);
        LowdegArgs a4 = a;
        a4.Qp = mix.s4.Qp; a4.RT = mix.s4.RT; a4.LRT = mix.s4.LRT; a4.C = mix.s4.C; a4.W = mix.s4.W;
        lowdeg_smem_bytes(mix.s4, &a4.off_cnt, &a4.off_part, &a4.off_misc);
        a4.quad_of = plan4->quad_of.p; a4.soff = plan4->soff.p; a4.sidx = plan4->sidx.p; a4.swt = plan4->swt.p;
        a4.warp_start = plan4->warp_start.p; a4.row_groups = plan4->row_groups.p;
        size_t smem8, smem4;
        if (sh.rpl == 2) {
            const size_t ids8 = (plan->n_ids * sizeof(uint2) + 15) & ~(size_t)15, ids4 = (plan4->n_ids * sizeof(uint2) + 15) & ~(size_t)15;
            a.off_ids = (uint32_t)sh.smem; a.n_ids = (uint32_t)plan->n_ids;
            a4.off_ids = (uint32_t)mix.s4.smem; a4.n_ids = (uint32_t)plan4->n_ids;
            smem8 = sh.smem + ids8; smem4 = mix.s4.smem + ids4;
        } else {
            // small tiles: ask for more than half an SM's shared memory so that the tiles land one per SM
            smem8 = std::max(sh.smem, (size_t)g->smem_optin / 2 + 2048);
            smem4 = std::max(mix.s4.smem, (size_t)g->smem_optin / 2 + 2048);
        }
        launched_smem = smem8;
        auto launch_tiles = [&](const LowdegArgs &aa, const LowdegShape &ss, int grid, size_t smem, cudaStream_t st) {
            if (ss.rpl == 2) launch_lowdeg_pair<true, true>(g, aa, ss, grid, smem, st);
            else if (nmode == 2 && ss.uniform) launch_lowdeg<2, true, false, true>(g, aa, ss, grid, st, smem);
            else if (nmode == 2) launch_lowdeg<2, false, false, true>(g, aa, ss, grid, st, smem);
            else if (ss.uniform) launch_lowdeg<3, true, false, true>(g, aa, ss, grid, st, smem);
            else launch_lowdeg<3, false, false, true>(g, aa, ss, grid, st, smem);
        };
        const int B = sh.RT;
        // per window: the tiles of the two lanes, grouped by the step they start from (the rotation leaves at most two
        // histories per lane) -- one launch per group, all of a window side by side on a pool of streams
        const int n8 = mix.tiles8, n4t = mix.tiles4;
        OSCB_REQUIRE(n8 <= OSCB_LD_TAB && n4t <= OSCB_LD_TAB, "internal: mixed-tile grids of %d / %d CTAs", n8, n4t);
        std::vector<int64_t> done(R / B, 0);
        std::vector<cudaStream_t> pool(1, s);
        std::vector<cudaEvent_t> pool_done;
        auto stream_at = [&](size_t i) {
            while (pool.size() <= i) {
                cudaStream_t st;
                OSCB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
                pool.push_back(st);
            }
            while (pool_done.size() <= i) {
                cudaEvent_t e;
                OSCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                pool_done.push_back(e);
            }
            return pool[i];
        };
        cudaEvent_t window_done;
        OSCB_CUDA(cudaEventCreateWithFlags(&window_done, cudaEventDisableTiming));
        OSCB_CUDA(cudaEventRecord(window_done, s));          // (the set-up above, on the run's stream)
        a.use_tab = a4.use_tab = 1;
        a.window_steps = (int)mix.steps8;
        a4.window_steps = (int)mix.steps4;
        std::vector<char> fast(R / B);
        launches = 0;
        for (int j = 0; j < mix.windows; ++j) {
            std::fill(fast.begin(), fast.end(), 0);
            for (int i = 0; i < mix.fast_octets; ++i) fast[((int64_t)j * mix.fast_octets + i) % (R / B)] = 1;
            std::map<int, std::vector<int>> big, small;          // first step -> tiles
            for (int o = 0; o < R / B; ++o) {
                const int at = (int)(p->first_step + done[o]);
                if (fast[o]) { small[at].push_back(2 * o); small[at].push_back(2 * o + 1); done[o] += mix.steps4; }
                else { big[at].push_back(o); done[o] += mix.steps8; }
            }
            size_t used = 0;
            auto launch_groups = [&](std::map<int, std::vector<int>> &groups, LowdegArgs &aa, const LowdegShape &ss, size_t smem) {
                for (auto &kv : groups) {
                    OSCB_REQUIRE(kv.second.size() <= OSCB_LD_TAB, "internal: mixed-tile group of %zu CTAs", kv.second.size());
                    aa.win_begin = kv.first;
                    std::copy(kv.second.begin(), kv.second.end(), aa.tab_tile);
                    cudaStream_t st = stream_at(used);
                    if (st != s) OSCB_CUDA(cudaStreamWaitEvent(st, window_done, 0));
                    launch_tiles(aa, ss, (int)kv.second.size(), smem, st);
                    OSCB_CUDA(cudaEventRecord(pool_done[used], st));
                    ++used;
                    ++launches;
                }
            };
            launch_groups(big, a, sh, smem8);
            launch_groups(small, a4, mix.s4, smem4);
            for (size_t i = 1; i < used; ++i) OSCB_CUDA(cudaStreamWaitEvent(s, pool_done[i], 0));
            OSCB_CUDA(cudaEventRecord(window_done, s));
        }
        for (int o = 0; o < R / B; ++o) OSCB_REQUIRE(done[o] == steps, "internal: mixed-tile schedule ends at step %lld", (long long)done[o]);
        OSCB_CUDA(cudaEventRecord(ev1, s));
        OSCB_CUDA(cudaStreamSynchronize(s));                // the events and the pool go out of scope here
        for (auto &e : pool_done) cudaEventDestroy(e);
        cudaEventDestroy(window_done);
        for (size_t i = 1; i < pool.size(); ++i) cudaStreamDestroy(pool[i]);
    }
    else if (sh.rpl == 2) {
        // the slot stream goes to shared memory when it fits behind the pairs (OSCB_LOWDEG_IDS=0: never)
        const size_t ids_bytes = (plan->n_ids * sizeof(uint2) + 15) & ~(size_t)15;
        const bool want_ids = !(getenv("OSCB_LOWDEG_IDS") && atoi(getenv("OSCB_LOWDEG_IDS")) == 0);
        const bool ids = want_ids && sh.smem + ids_bytes <= (size_t)g->smem_optin;
        size_t smem = sh.smem;
        if (ids) { a.off_ids = (uint32_t)sh.smem; a.n_ids = (uint32_t)plan->n_ids; smem += ids_bytes; }
        launched_smem = smem;
        if (ids) { if (g->unit_weights) launch_lowdeg_pair<true, true>(g, a, sh, tiles, smem); else launch_lowdeg_pair<false, true>(g, a, sh, tiles, smem); }
        else     { if (g->unit_weights) launch_lowdeg_pair<true, false>(g, a, sh, tiles, smem); else launch_lowdeg_pair<false, false>(g, a, sh, tiles, smem); }
    }
    else if (nmode == 2) by_shape(std::integral_constant<int, 2>{});
    else by_shape(std::integral_constant<int, 3>{});
    if (launches == 1) OSCB_CUDA(cudaEventRecord(ev1, s));
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            set_error("oscb_run(lowdeg): kernel launch failed: %s (tiles %d, threads %d, smem %zu)", cudaGetErrorString(e), tiles,
                      sh.W * 32, sh.smem);
            throw OscbFail{OSCB_ECUDA};
        }
    }
    if (out->final_phases) d_io.download(out->final_phases, tot, s);
    if (out->best_states)
        OSCB_CUDA(cudaMemcpy2DAsync(out->best_states, (size_t)n, d_best_states.p, (size_t)n4, (size_t)n, (size_t)R,
                                    cudaMemcpyDeviceToHost, s));
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
    out->kernel_launches = launches;
    out->kernel_used = OSCB_KERNEL_LOWDEG;
    out->replicas_per_cta = RT;
    out->smem_bytes = (int64_t)launched_smem;
    if (flag != none) {
        out->nonfinite[2] = (int64_t)(flag >> 36);
        out->nonfinite[0] = (int64_t)((flag >> 20) & 0xFFFFull);
        out->nonfinite[1] = (int64_t)(flag & 0xFFFFFull);
        set_error("non-finite phase for oscillator %lld (replica row %lld) after step %lld; parameters are numerically unstable",
                  (long long)out->nonfinite[1], (long long)out->nonfinite[0], (long long)out->nonfinite[2]);
        throw OscbFail{OSCB_ENONFINITE};
    }
}

} // namespace oscb
