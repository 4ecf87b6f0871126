// oscb_umma.cu -- host side of the tensor-core dense integrator (kernel: oscb_umma.cuh).
#include "oscb_umma.hpp"
#include "oscb_umma.cuh"
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <unistd.h>
#include <vector>

namespace oscb {

std::shared_ptr<UmmaPlan> umma_build_plan(const int8_t *J8_dev, int64_t n, int n_pad, int64_t row_begin, int64_t row_end,
                                          bool fp4_ok, cudaStream_t s)
{
    OSCB_REQUIRE(row_begin % UMMA_TILE == 0 && (row_end % UMMA_TILE == 0 || row_end == n),
                 "tensor-core dense path needs row shards aligned to %d rows", UMMA_TILE);
    auto plan = std::make_shared<UmmaPlan>();
    plan->n = (int)n;
    plan->tiles = (int)((n + UMMA_TILE - 1) / UMMA_TILE);
    plan->tile_begin = (int)(row_begin / UMMA_TILE);
    plan->tile_end = (int)((row_end + UMMA_TILE - 1) / UMMA_TILE);
    const int lt = plan->tile_end - plan->tile_begin;
    plan->A_img.alloc((size_t)lt * plan->tiles * UMMA_A_STAGE);
    plan->W.alloc((size_t)lt * UMMA_TILE);
    k_umma_build_a<<<dim3((unsigned)plan->tiles, (unsigned)lt), 256, 0, s>>>(J8_dev, (int)n, n_pad, (int)(row_end - row_begin),
                                                                            plan->tiles, plan->A_img.p, plan->W.p);
    OSCB_CUDA(cudaGetLastError());
    plan->fp4_ok = fp4_ok;
    if (fp4_ok) {
        // 4 bits per coupling: half the HBM bytes of the int8 image (tiles of 128 rows x 256 couplings)
        const int kt4 = (int)((n + UMMA_K4 - 1) / UMMA_K4);
        plan->A_fp4.alloc((size_t)lt * kt4 * UMMA_A_STAGE);
        k_umma_build_fp4<<<dim3((unsigned)kt4, (unsigned)lt), 256, 0, s>>>(J8_dev, (int)n, n_pad, (int)(row_end - row_begin), kt4,
                                                                          plan->A_fp4.p);
        OSCB_CUDA(cudaGetLastError());
    }
    OSCB_CUDA(cudaStreamSynchronize(s));
    return plan;
}

static inline size_t round256(size_t x) { return (x + 255) & ~(size_t)255; }

// The e2m1 stream halves the HBM bytes of J and is bit-identical to the int8 stream.  It runs on the block-scaled 4-bit
// tensor path (kind::mxf4, K = 64 per MMA, all scales 1.0), which also reads half the shared-memory bytes per coupling on the
// A side: 24.5 us per Euler step of SK 16384 at R = 1 against 41.8 us for the HBM-bound int8 stream.  It needs 21 B
// columns per replica instead of 9, so a launch takes at most 12 replicas; up to there it is ahead (R = 12: 44.6 vs 47.3 us).
// OSCB_UMMA_FP4 = 0 / 1 forces the choice.
bool umma_uses_fp4(const UmmaPlan &plan, int R, int n_states, int force_stream)
{
    // a row-sharded run agrees on ONE stream for all ranks (every rank writes digits into every peer's B image, so
    // the layouts must match): the caller passes the agreed choice and the process-local environment is not consulted
    if (force_stream == 8) return false;
    if (force_stream == 4) {
        OSCB_REQUIRE(plan.fp4_ok && R <= umma_max_replicas(n_states, true), "the packed e2m1 stream was requested but this shard / replica count cannot take it");
        return true;
    }
    if (!plan.fp4_ok) return false;
    if (const char *env = getenv("OSCB_UMMA_FP4")) return atoi(env) == 1;
    return R <= umma_max_replicas(n_states, true);      // the whole call fits one launch of the e2m1 stream (N = 2: 12)
}

struct UmmaSession::Impl {
    oscb_graph *g = nullptr;
    const UmmaPlan *plan = nullptr;
    UmmaSpec spec;
    std::vector<uint8_t> flags;
    int world = 1, rank = 0;
    UmmaArgs a{};
    // the exchange block (one cudaMalloc, so one IPC handle): [barrier counter | events | energy partials | B0 | B1]
    unsigned char *xbase = nullptr;
    size_t xbytes = 0, off_events = 0, off_en = 0, off_b[2] = {0, 0};
    void *peer_base[kUmmaMaxWorld] = {};
    bool peer_ipc[kUmmaMaxWorld] = {};
    bool connected = false;
    int32_t stream_sig() const { return (int32_t)((a.fp4 & 1) | ((a.NB & 0x1FF) << 1) | ((a.dcols & 0x3F) << 10) | ((a.ktiles & 0x7FFF) << 16)); }
    DevBuf<unsigned char> phi[2];
    DevBuf<uint64_t> d_seeds;
    DevBuf<uint8_t> d_flags, d_best;
    DevBuf<unsigned long long> d_timeout;
    DevBuf<int> d_acc;                      // split-K accumulator
    DevBuf<unsigned int> d_tile_cnt;
    int watchdog_ms = 20000;
    DevBuf<long long> d_trace;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    size_t tsize = 4;

    void point_rank(int w, unsigned char *base)
    {
        a.bar[w] = reinterpret_cast<unsigned int *>(base);
        a.events[w] = reinterpret_cast<long long *>(base + off_events);
        a.en_part[w] = reinterpret_cast<double *>(base + off_en);
        a.B_img[0][w] = base + off_b[0];
        a.B_img[1][w] = base + off_b[1];
    }
};

UmmaSession::UmmaSession(oscb_graph *g, const UmmaSpec &spec, int world, int rank) : m(new Impl())
{
    try {
        OSCB_REQUIRE(g && g->umma, "handle has no tensor-core plan (integer couplings |J| <= 127 on 128-row aligned shards)");
        OSCB_REQUIRE(spec.n_states >= 2 && spec.n_states <= 16, "tensor-core dense path takes N = 2..16 states");
        const bool want_fp4 = umma_uses_fp4(*g->umma, spec.R_total > 0 ? spec.R_total : spec.R, spec.n_states, spec.force_stream);
        OSCB_REQUIRE(spec.R >= 1 && spec.R <= umma_max_replicas(spec.n_states, want_fp4),
                     "tensor-core dense path takes 1..%d replicas per launch at N = %d", umma_max_replicas(spec.n_states, want_fp4), spec.n_states);
        OSCB_REQUIRE(world >= 1 && world <= kUmmaMaxWorld && rank >= 0 && rank < world, "bad world / rank %d / %d", world, rank);
        m->g = g;
        m->plan = g->umma.get();
        m->spec = spec;
        m->flags.assign(spec.flags, spec.flags + spec.steps + 1);
        m->spec.flags = m->flags.data();
        m->world = world;
        m->rank = rank;
        m->tsize = spec.precision == OSCB_PREC_F64 ? 8 : 4;
        const UmmaPlan &plan = *m->plan;
        UmmaArgs &a = m->a;
        a.n = plan.n;
        a.tiles = plan.tiles;
        a.tile_begin = plan.tile_begin;
        a.tile_end = plan.tile_end;
        a.R = spec.R;
        // couplings representable in e2m1 stream as packed 4-bit codes through the TMA unpack path when few replicas share the launch
        a.fp4 = umma_uses_fp4(plan, spec.R_total > 0 ? spec.R_total : spec.R, spec.n_states, spec.force_stream) ? 1 : 0;
        a.A_fp4 = plan.A_fp4.p;
        a.ktiles = a.fp4 ? (plan.n + UMMA_K4 - 1) / UMMA_K4 : plan.tiles;
        a.dcols = a.fp4 ? 2 * UMMA_D9 : 8;
        a.n_states = spec.n_states;
        a.maximize = spec.maximize;
        a.score_cols = spec.n_states == 2 ? 1 : spec.n_states;
        a.NB = ((a.dcols + a.score_cols) * spec.R + 15) / 16 * 16;
        OSCB_REQUIRE(a.NB <= 256, "too many replicas for one launch (%d B rows)", a.NB);
        const size_t b_stage = (size_t)a.NB * 128, stage = UMMA_A_STAGE + b_stage;
        const size_t ctl = 2560, slack = 1024;
        a.stages = (int)std::min<size_t>(12, ((size_t)g->smem_optin - ctl - slack) / stage);
        OSCB_REQUIRE(a.stages >= 2, "not enough shared memory for the tensor-core dense pipeline");
        smem = slack + (size_t)a.stages * stage + ctl;
        stages = a.stages;
        a.world = world;
        a.rank = rank;
        a.tmem_cols = 32;
        while (a.tmem_cols < a.NB + (a.fp4 ? UMMA_SF_COLS : 0)) a.tmem_cols *= 2;
        const int lt = plan.tile_end - plan.tile_begin;
        grid = std::min(lt, g->sm_count);
        if (const char *cap = getenv("OSCB_UMMA_MAX_GRID"))       // test knob: several row tiles per CTA on small graphs
            grid = std::max(1, std::min(grid, atoi(cap)));
        // split-K: a handle that owns few row tiles (a rank of a row-sharded run: 16 of the 128 tiles of SK 16384 at 8
        // GPUs) would keep one CTA per tile busy and leave the other SMs idle, each CTA still streaming a full-K row tile.
        // S CTAs then share a tile, S = SMs / tiles, when the per-CTA stream of a pass is long enough to pay for the
        // exchange of the partial sums (OSCB_UMMA_SPLITK = 1 disables, = S forces).
        a.splits = 1;
        if (grid == lt) {
            int S = std::min(g->sm_count / std::max(lt, 1), a.ktiles);
            const size_t stream = (size_t)a.ktiles * stage;       // bytes one CTA moves per pass for a whole-K row tile
            // (measured, one rank of SK 16384 alone on a B200, us per Euler step unsplit -> split: 2-GPU rank 20.4 -> 16.4
            // at S = 2, 4-GPU rank 20.3 -> 12.7 at S = 4, 8-GPU rank 20.1 -> 10.3 at S = 9; the whole graph on one GPU:
            // 25.1.  profiles/r02n_dense_rank_emulation.jsonl, tools/dense_rank_emulation.py)
            if (S < 2 || stream < (size_t)512 * 1024) S = 1;
            if (const char *e = getenv("OSCB_UMMA_SPLITK")) S = std::max(1, std::min({atoi(e), g->sm_count / std::max(lt, 1), a.ktiles}));
            a.splits = S;
            grid = lt * S;
        }
        splits = a.splits;
        m->d_acc.alloc((size_t)lt * UMMA_TILE * a.NB);
        m->d_tile_cnt.alloc((size_t)lt);
        a.acc_g = m->d_acc.p;
        a.tile_cnt = m->d_tile_cnt.p;
        a.ctas_total = (unsigned)grid;                            // world = 1; connect() fills in the real totals
        a.cta_offset = 0;
        a.passes = spec.steps + 1;
        a.first_step = spec.first_step;
        a.K = spec.K; a.h = spec.h; a.kn_sqrt_h = spec.kn_sqrt_h; a.ks_max = spec.ks_max; a.ks_period = spec.ks_period;
        a.tc = make_trig_const(spec.n_states);
        a.noise_on = spec.noise_on;
        a.ld_phi = (long long)lt * UMMA_TILE;

        const size_t E = (size_t)std::max<long long>(1, spec.n_events), S = (size_t)std::max<long long>(1, spec.n_samples);
        m->off_events = 256;
        m->off_en = m->off_events + round256(E * spec.R * sizeof(long long));
        // energy partials: one slot per CTA of ALL ranks (one CTA per row tile, or with split-K at most the SMs of every rank)
        m->off_b[0] = m->off_en + round256(S * (size_t)std::max(plan.tiles, world * g->sm_count) * spec.R * sizeof(double));
        m->off_b[1] = m->off_b[0] + round256((size_t)a.ktiles * b_stage);
        m->xbytes = m->off_b[1] + round256((size_t)a.ktiles * b_stage);
        OSCB_CUDA(cudaSetDevice(g->device));
        OSCB_CUDA(cudaMalloc(&m->xbase, m->xbytes));              // not pooled: the block is exported over CUDA IPC
        m->point_rank(rank, m->xbase);
        m->peer_base[rank] = m->xbase;
        m->connected = world == 1;

        for (int k = 0; k < 2; ++k) { m->phi[k].alloc((size_t)spec.R * a.ld_phi * m->tsize); a.phi[k] = m->phi[k].p; }
        m->d_seeds.alloc(spec.R);
        m->d_flags.alloc((size_t)a.passes);
        m->d_best.alloc((size_t)spec.R * a.ld_phi);
        a.A_img = plan.A_img.p;
        a.W = plan.W.p;
        a.seeds = m->d_seeds.p;
        a.flags = m->d_flags.p;
        a.best_states = m->d_best.p;
        a.nonfinite = g->d_nonfinite.p;
        a.trace = nullptr;
        m->d_timeout.alloc(1);
        a.timeout_flag = m->d_timeout.p;
        if (const char *e = getenv("OSCB_UMMA_WATCHDOG_MS")) m->watchdog_ms = std::max(1, atoi(e));
        a.watchdog_ns = (long long)m->watchdog_ms * 1000000ll;      // (%globaltimer: no clock-rate query -- that one costs tens of ms)
        OSCB_CUDA(cudaEventCreate(&m->ev0));
        OSCB_CUDA(cudaEventCreate(&m->ev1));
    } catch (...) {
        if (m->xbase) cudaFree(m->xbase);
        delete m;
        m = nullptr;
        throw;
    }
}

UmmaSession::~UmmaSession()
{
    if (!m) return;
    cudaSetDevice(m->g->device);
    cudaStreamSynchronize(m->g->stream);
    for (int w = 0; w < m->world; ++w)
        if (m->peer_ipc[w] && m->peer_base[w]) cudaIpcCloseMemHandle(m->peer_base[w]);
    if (m->xbase) cudaFree(m->xbase);
    if (m->ev0) cudaEventDestroy(m->ev0);
    if (m->ev1) cudaEventDestroy(m->ev1);
    delete m;
}

int UmmaSession::rows() const
{
    return std::min(m->a.n, m->a.tile_end * UMMA_TILE) - m->a.tile_begin * UMMA_TILE;
}

void UmmaSession::export_mem(UmmaExchange *out) const
{
    std::memset(out, 0, sizeof(*out));
    cudaIpcMemHandle_t h;
    OSCB_CUDA(cudaSetDevice(m->g->device));
    OSCB_CUDA(cudaIpcGetMemHandle(&h, m->xbase));
    static_assert(sizeof(h) <= sizeof(out->ipc), "IPC handle does not fit");
    std::memcpy(out->ipc, &h, sizeof(h));
    out->base = (uint64_t)(uintptr_t)m->xbase;
    out->bytes = m->xbytes;
    out->device = m->g->device;
    out->pid = (int32_t)getpid();
    out->grid = grid;
    out->stream_sig = m->stream_sig();
}

void UmmaSession::connect(const UmmaExchange *all)
{
    OSCB_CUDA(cudaSetDevice(m->g->device));
    unsigned total = 0;
    for (int w = 0; w < m->world; ++w) {
        const UmmaExchange &x = all[w];
        OSCB_REQUIRE(x.bytes == m->xbytes, "rank %d exchange block is %llu bytes, expected %zu (replicas / schedule differ?)", w,
                     (unsigned long long)x.bytes, m->xbytes);
        // at R = 1 the int8 and the e2m1 images have the SAME size, so the byte count alone would let a rank whose
        // shard holds a coupling outside {0, +-1, +-2, +-3, +-4, +-6} (int8 digits) corrupt its peers' e2m1 planes
        OSCB_REQUIRE(x.stream_sig == m->stream_sig(),
                     "rank %d streams J as %s (B image signature 0x%x) but rank %d as %s (0x%x): every rank of a row-sharded run "
                     "must use the same stream -- agree on it before create (dense_fused.run_dense_fused does; RunParams.variant 8 / 4)",
                     w, (x.stream_sig & 1) ? "packed e2m1" : "int8", (unsigned)x.stream_sig, m->rank, m->a.fp4 ? "packed e2m1" : "int8",
                     (unsigned)m->stream_sig());
        if (w == m->rank) m->a.cta_offset = (int)total;
        total += (unsigned)x.grid;
        if (w == m->rank) continue;
        if (x.pid == (int32_t)getpid()) {
            // same process (one process driving several GPUs, or virtual ranks on one GPU): the address is valid as is
            if (x.device != m->g->device) {
                int can = 0;
                OSCB_CUDA(cudaDeviceCanAccessPeer(&can, m->g->device, x.device));
                OSCB_REQUIRE(can, "device %d cannot access device %d", m->g->device, x.device);
                cudaError_t e = cudaDeviceEnablePeerAccess(x.device, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else OSCB_CUDA(e);
            }
            m->peer_base[w] = (void *)(uintptr_t)x.base;
        } else {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, x.ipc, sizeof(h));
            OSCB_CUDA(cudaIpcOpenMemHandle(&m->peer_base[w], h, cudaIpcMemLazyEnablePeerAccess));
            m->peer_ipc[w] = true;
        }
        m->point_rank(w, (unsigned char *)m->peer_base[w]);
    }
    // ranks that share this GPU (virtual ranks of the tests, OSCB_BENCH_BACKEND=gloo) must be co-resident: every
    // kernel spins on the others' arrivals
    unsigned here = 0;
    for (int w = 0; w < m->world; ++w)
        if (all[w].device == m->g->device) here += (unsigned)all[w].grid;
    OSCB_REQUIRE(here <= (unsigned)m->g->sm_count || here == (unsigned)grid,
                 "the ranks sharing device %d launch %u CTAs in all, more than its %d SMs: their persistent kernels cannot be "
                 "resident together (fewer ranks per GPU, or OSCB_UMMA_SPLITK=1 to keep one CTA per row tile)",
                 m->g->device, here, m->g->sm_count);
    m->a.ctas_total = total;
    m->connected = true;
}

void UmmaSession::prepare(const uint64_t *seeds, const double *d_phi0)
{
    OSCB_REQUIRE(m->connected, "connect() the ranks before prepare()");
    cudaStream_t s = m->g->stream;
    UmmaArgs &a = m->a;
    OSCB_CUDA(cudaSetDevice(m->g->device));
    OSCB_CUDA(cudaMemsetAsync(m->xbase, 0, m->xbytes, s));
    m->phi[0].zero(s); m->phi[1].zero(s); m->d_best.zero(s);
    m->d_seeds.upload(seeds, a.R, s);
    m->d_flags.upload(m->flags.data(), (size_t)a.passes, s);
    const unsigned long long none = ~0ull;
    OSCB_CUDA(cudaMemcpyAsync(m->g->d_nonfinite.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));
    OSCB_CUDA(cudaMemcpyAsync(m->d_timeout.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));
    m->d_acc.zero(s);
    m->d_tile_cnt.zero(s);
    if (const char *trace_path = getenv("OSCB_UMMA_TRACE")) {     // debug: per-CTA timeline of the first passes
        (void)trace_path;
        m->d_trace.alloc((size_t)grid * UMMA_TRACE_PASSES * UMMA_TRACE_SLOTS);
        m->d_trace.zero(s);
        a.trace = m->d_trace.p;
    }
    const long long tot = (long long)((a.n + 1) / 2) * a.R;      // one thread per pair of oscillators
    if (m->tsize == 8) k_umma_init<double><<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(a, d_phi0);
    else k_umma_init<float><<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(a, d_phi0);
    OSCB_CUDA(cudaGetLastError());
    OSCB_CUDA(cudaStreamSynchronize(s));      // the block is clean and initialised when prepare() returns
}

void UmmaSession::launch()
{
    cudaStream_t s = m->g->stream;
    OSCB_CUDA(cudaSetDevice(m->g->device));
    const void *fn = m->a.fp4 ? (m->tsize == 8 ? (const void *)k_dense_umma<double, true> : (const void *)k_dense_umma<float, true>)
                              : (m->tsize == 8 ? (const void *)k_dense_umma<double, false> : (const void *)k_dense_umma<float, false>);
    OSCB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    OSCB_CUDA(cudaEventRecord(m->ev0, s));
    void *kargs[] = {(void *)&m->a};
    OSCB_CUDA(cudaLaunchCooperativeKernel(fn, dim3((unsigned)grid), dim3(UMMA_THREADS), kargs, smem, s));
    OSCB_CUDA(cudaEventRecord(m->ev1, s));
}

void UmmaSession::export_final(double *d_final_full)
{
    cudaStream_t s = m->g->stream;
    const UmmaArgs &a = m->a;
    const unsigned blocks = (unsigned)(((long long)a.ld_phi * a.R + 255) / 256);
    const void *fin = a.phi[(a.passes - 1) & 1];
    if (m->tsize == 8) k_umma_export<double><<<blocks, 256, 0, s>>>(a, fin, d_final_full, a.n, (long long)a.tile_begin * UMMA_TILE);
    else k_umma_export<float><<<blocks, 256, 0, s>>>(a, fin, d_final_full, a.n, (long long)a.tile_begin * UMMA_TILE);
    OSCB_CUDA(cudaGetLastError());
}

void UmmaSession::finish(double *h_final_rows, uint8_t *h_best_rows, long long *h_events, double *h_energy)
{
    cudaStream_t s = m->g->stream;
    const UmmaArgs &a = m->a;
    const int R = a.R, nrows = rows();
    const long long E = m->spec.n_events, S = m->spec.n_samples;
    const unsigned ctas = a.ctas_total;
    OSCB_CUDA(cudaSetDevice(m->g->device));
    DevBuf<double> d_rows;
    if (h_final_rows) {
        d_rows.alloc((size_t)R * nrows);
        const unsigned blocks = (unsigned)(((long long)a.ld_phi * R + 255) / 256);
        const void *fin = a.phi[(a.passes - 1) & 1];
        if (m->tsize == 8) k_umma_export<double><<<blocks, 256, 0, s>>>(a, fin, d_rows.p, nrows, 0);
        else k_umma_export<float><<<blocks, 256, 0, s>>>(a, fin, d_rows.p, nrows, 0);
        OSCB_CUDA(cudaGetLastError());
        d_rows.download(h_final_rows, (size_t)R * nrows, s);
    }
    std::vector<double> h_en;
    if (h_events && E) OSCB_CUDA(cudaMemcpyAsync(h_events, m->xbase + m->off_events, (size_t)E * R * sizeof(long long), cudaMemcpyDeviceToHost, s));
    if (h_energy && S) {
        h_en.resize((size_t)S * ctas * R);
        OSCB_CUDA(cudaMemcpyAsync(h_en.data(), m->xbase + m->off_en, h_en.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    if (h_best_rows)
        OSCB_CUDA(cudaMemcpy2DAsync(h_best_rows, (size_t)nrows, m->d_best.p, (size_t)a.ld_phi, (size_t)nrows, (size_t)R,
                                    cudaMemcpyDeviceToHost, s));
    OSCB_CUDA(cudaMemcpyAsync(&nonfinite, m->g->d_nonfinite.p, sizeof(nonfinite), cudaMemcpyDeviceToHost, s));
    unsigned long long timed_out = ~0ull;
    OSCB_CUDA(cudaMemcpyAsync(&timed_out, m->d_timeout.p, sizeof(timed_out), cudaMemcpyDeviceToHost, s));
    OSCB_CUDA(cudaStreamSynchronize(s));
    OSCB_CUDA(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
    if (timed_out != ~0ull) {
        set_error("dense tensor-core run abandoned: rank %d waited more than %d ms at Euler step %llu for the other CTAs / ranks "
                  "of the step barrier (a peer rank never launched, died, or OSCB_UMMA_WATCHDOG_MS is too short); results are invalid",
                  m->rank, m->watchdog_ms, timed_out);
        throw OscbFail{OSCB_ECUDA};
    }
    if (h_energy)
        for (long long k = 0; k < S; ++k)
            for (int r = 0; r < R; ++r) {
                double e = 0.0;
                for (unsigned c = 0; c < ctas; ++c) e += h_en[((size_t)k * ctas + c) * R + r];   // CTA order: deterministic
                h_energy[k * R + r] = e;
            }
    if (const char *trace_path = getenv("OSCB_UMMA_TRACE")) {
        if (m->d_trace.p) {
            std::vector<long long> h((size_t)grid * UMMA_TRACE_PASSES * UMMA_TRACE_SLOTS);
            OSCB_CUDA(cudaMemcpy(h.data(), m->d_trace.p, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
            if (FILE *f = fopen(trace_path, "w")) {
                fprintf(f, "cta,pass,barrier_seen,tmem_full,arrived,barrier_wait_begin,tmem_loaded,updated,stored,cta_synced\n");
                for (int c = 0; c < grid; ++c)
                    for (int q = 0; q < UMMA_TRACE_PASSES && q < a.passes; ++q) {
                        const long long *t = &h[((size_t)c * UMMA_TRACE_PASSES + q) * UMMA_TRACE_SLOTS];
                        fprintf(f, "%d,%d,%lld,%lld,%lld,%lld,%lld,%lld,%lld,%lld\n", c, q, t[0], t[1], t[2], t[3], t[4], t[5], t[6], t[7]);
                    }
                fclose(f);
            }
        }
    }
}

} // namespace oscb
