// oscb_umma.cu -- host side of the tensor-core dense integrator (kernel: oscb_umma.cuh).
#include "oscb_umma.hpp"
#include "oscb_umma.cuh"
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <vector>

namespace oscb {

std::shared_ptr<UmmaPlan> umma_build_plan(const int8_t *J8_dev, int64_t n, int n_pad, int64_t row_begin, int64_t row_end,
                                          cudaStream_t s)
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
    OSCB_CUDA(cudaStreamSynchronize(s));
    return plan;
}

template <typename T>
static void umma_run_t(oscb_graph *g, const UmmaPlan &plan, UmmaSpec &spec)
{
    cudaStream_t s = g->stream;
    const int R = spec.R, n = plan.n;
    OSCB_REQUIRE(R >= 1 && R <= UMMA_MAXR, "tensor-core dense path takes 1..%d replicas per launch", UMMA_MAXR);
    UmmaArgs a{};
    a.n = n;
    a.tiles = plan.tiles;
    a.tile_begin = plan.tile_begin;
    a.tile_end = plan.tile_end;
    a.R = R;
    a.NB = (9 * R + 15) / 16 * 16;
    const size_t b_stage = (size_t)a.NB * 128, stage = UMMA_A_STAGE + b_stage;
    const size_t ctl = 2048, slack = 1024;
    a.stages = (int)std::min<size_t>(12, ((size_t)g->smem_optin - ctl - slack) / stage);
    OSCB_REQUIRE(a.stages >= 2, "not enough shared memory for the tensor-core dense pipeline");
    const size_t smem = slack + (size_t)a.stages * stage + ctl;
    a.world = 1;
    a.rank = 0;
    a.tmem_cols = 32;
    while (a.tmem_cols < a.NB) a.tmem_cols *= 2;
    const int lt = plan.tile_end - plan.tile_begin;
    int grid = std::min(lt, g->sm_count);
    if (const char *cap = getenv("OSCB_UMMA_MAX_GRID"))       // test knob: several row tiles per CTA on small graphs
        grid = std::max(1, std::min(grid, atoi(cap)));
    a.ctas_total = (unsigned)grid;
    a.cta_offset = 0;
    a.passes = spec.steps + 1;
    a.first_step = spec.first_step;
    a.K = spec.K; a.h = spec.h; a.kn_sqrt_h = spec.kn_sqrt_h; a.ks_max = spec.ks_max; a.ks_period = spec.ks_period;
    a.tc = make_trig_const(2);
    a.noise_on = spec.noise_on;
    a.ld_phi = (long long)lt * UMMA_TILE;

    DevBuf<uint8_t> B0((size_t)plan.tiles * b_stage), B1((size_t)plan.tiles * b_stage);
    DevBuf<T> phi0((size_t)R * a.ld_phi), phi1((size_t)R * a.ld_phi);
    DevBuf<uint64_t> d_seeds(R);
    DevBuf<uint8_t> d_flags((size_t)a.passes), d_best((size_t)R * a.ld_phi);
    DevBuf<unsigned int> d_bar(1);
    DevBuf<long long> d_events((size_t)std::max<long long>(1, spec.n_events) * R);
    DevBuf<double> d_en((size_t)std::max<long long>(1, spec.n_samples) * grid * R);
    B0.zero(s); B1.zero(s); phi0.zero(s); phi1.zero(s); d_best.zero(s); d_bar.zero(s); d_events.zero(s); d_en.zero(s);
    d_seeds.upload(spec.seeds, R, s);
    d_flags.upload(spec.flags, (size_t)a.passes, s);
    const unsigned long long none = ~0ull;
    OSCB_CUDA(cudaMemcpyAsync(g->d_nonfinite.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));

    a.A_img = plan.A_img.p;
    a.B_img[0][0] = B0.p; a.B_img[1][0] = B1.p;
    a.phi[0] = phi0.p; a.phi[1] = phi1.p;
    a.W = plan.W.p;
    a.seeds = d_seeds.p;
    a.flags = d_flags.p;
    a.bar[0] = d_bar.p;
    a.events[0] = d_events.p;
    a.en_part[0] = d_en.p;
    a.best_states = d_best.p;
    a.nonfinite = g->d_nonfinite.p;

    DevBuf<long long> d_trace;
    const char *trace_path = getenv("OSCB_UMMA_TRACE");           // debug: per-CTA timeline of the first passes
    if (trace_path) {
        d_trace.alloc((size_t)grid * UMMA_TRACE_PASSES * 4);
        d_trace.zero(s);
        a.trace = d_trace.p;
    }
    const long long tot = (long long)n * R;
    k_umma_init<T><<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(a, spec.d_phi0);
    OSCB_CUDA(cudaGetLastError());

    OSCB_CUDA(cudaFuncSetAttribute(k_dense_umma<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t ev0, ev1;
    OSCB_CUDA(cudaEventCreate(&ev0));
    OSCB_CUDA(cudaEventCreate(&ev1));
    OSCB_CUDA(cudaEventRecord(ev0, s));
    void *kargs[] = {(void *)&a};
    OSCB_CUDA(cudaLaunchCooperativeKernel((const void *)k_dense_umma<T>, dim3((unsigned)grid), dim3(UMMA_THREADS), kargs, smem, s));
    OSCB_CUDA(cudaEventRecord(ev1, s));

    if (spec.d_final)
        k_umma_export<T><<<(unsigned)(((long long)a.ld_phi * R + 255) / 256), 256, 0, s>>>(a, a.phi[(a.passes - 1) & 1], spec.d_final);
    std::vector<double> h_en((size_t)std::max<long long>(1, spec.n_samples) * grid * R);
    if (spec.h_events && spec.n_events) d_events.download(spec.h_events, (size_t)spec.n_events * R, s);
    if (spec.h_energy && spec.n_samples) d_en.download(h_en.data(), (size_t)spec.n_samples * grid * R, s);
    if (spec.h_best_states)
        OSCB_CUDA(cudaMemcpy2DAsync(spec.h_best_states, (size_t)n, d_best.p, (size_t)a.ld_phi, (size_t)n, (size_t)R,
                                    cudaMemcpyDeviceToHost, s));
    OSCB_CUDA(cudaMemcpyAsync(&spec.nonfinite, g->d_nonfinite.p, sizeof(none), cudaMemcpyDeviceToHost, s));
    OSCB_CUDA(cudaStreamSynchronize(s));
    OSCB_CUDA(cudaEventElapsedTime(&spec.ms, ev0, ev1));
    if (trace_path) {
        std::vector<long long> h((size_t)grid * UMMA_TRACE_PASSES * 4);
        OSCB_CUDA(cudaMemcpy(h.data(), d_trace.p, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
        if (FILE *f = fopen(trace_path, "w")) {
            fprintf(f, "cta,pass,barrier_seen,tmem_full,arrived,barrier_wait_begin\n");
            for (int c = 0; c < grid; ++c)
                for (int q = 0; q < UMMA_TRACE_PASSES && q < a.passes; ++q) {
                    const long long *t = &h[((size_t)c * UMMA_TRACE_PASSES + q) * 4];
                    fprintf(f, "%d,%d,%lld,%lld,%lld,%lld\n", c, q, t[0], t[1], t[2], t[3]);
                }
            fclose(f);
        }
    }
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    if (spec.h_energy)
        for (long long k = 0; k < spec.n_samples; ++k)
            for (int r = 0; r < R; ++r) {
                double e = 0.0;
                for (int c = 0; c < grid; ++c) e += h_en[((size_t)k * grid + c) * R + r];   // CTA order: deterministic
                spec.h_energy[k * R + r] = e;
            }
    spec.grid = grid;
    spec.stages = a.stages;
    spec.smem = smem;
}

void umma_run(oscb_graph *g, const UmmaPlan &plan, UmmaSpec &spec)
{
    if (spec.precision == OSCB_PREC_F64) umma_run_t<double>(g, plan, spec);
    else umma_run_t<float>(g, plan, spec);
}

} // namespace oscb
