// oscb_cluster_host.hpp -- host side of the cluster (latency-mode) integrator (kernel: oscb_cluster.cuh).
// Included by oscb.cu (the kernels it shares device code with live in that translation unit).
#pragma once
#include "oscb_host.hpp"
#include "oscb_cluster.cuh"
#include "oscb_stream.cuh"
#include <vector>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <limits>

namespace oscb {


struct ClusterShape {
    int rows_per_cta = 0, n_al = 0, nnz_cap = 0, threads = 0;
    bool weighted = false;
    ClusterSmem lay;
};

static bool cluster_shape(const oscb_graph *g, int CL_SIZE, ClusterShape *sh)
{
    if (g->is_dense || g->n < 64 || g->n > 65535) return false;
    const int n = (int)g->n;
    sh->rows_per_cta = ((n + CL_SIZE - 1) / CL_SIZE + 3) / 4 * 4;      // whole quads: a quad shares one Philox block
    sh->n_al = (n + 1 + 3) / 4 * 4;            // > n: pair n is the all-zero pair the padded gather slots read
    sh->weighted = !g->unit_weights;
    int cap = 0;
    for (int c = 0; c < CL_SIZE; ++c) {
        const int r0 = std::min(n, c * sh->rows_per_cta), r1 = std::min(n, (c + 1) * sh->rows_per_cta);
        cap = std::max(cap, g->h_indptr[r1] - g->h_indptr[r0]);
    }
    sh->nnz_cap = cap;
    sh->threads = std::max(64, std::min(1024, (sh->rows_per_cta * CL_LPR + 31) / 32 * 32));   // >= 2 warps: update + noise
    sh->lay = ClusterSmem::make(sh->n_al, sh->rows_per_cta, std::max(1, cap), sh->weighted);
    return sh->lay.total <= (size_t)g->smem_optin;
}

// one replica per 8-CTA cluster: float32, device noise, N = 2 max-cut, unit or exactly-summable integer
// couplings, few enough replicas that every cluster gets its own SMs (unless forced)
// Neighbour order of the cluster kernel.  A warp gathers 4 consecutive rows, 8 lanes each; its u-th load
// instruction touches list positions [8u, 8u + 8) of those rows, i.e. 32 random (cos, sin) pairs.  A pair
// spans two 4-byte banks, so the instruction needs at least 2 wavefronts and one more for every extra hit
// on a bank pair (column mod 16).  The order inside a row is free in float32 mode, so each instruction's 32
// columns are picked greedily from the rows' remaining neighbours to spread over the 16 bank pairs.
static void cluster_order_columns(const oscb_graph *g, int CL_SIZE, int rows_per_cta, std::vector<int> *cols, std::vector<float> *wts)
{
    const int n = (int)g->n;
    cols->assign(g->h_indices.begin(), g->h_indices.end());
    wts->resize(g->h_w.size());
    for (size_t e = 0; e < g->h_w.size(); ++e) (*wts)[e] = (float)g->h_w[e];
    std::vector<char> used;
    for (int c = 0; c < CL_SIZE; ++c) {
        const int r0 = std::min(n, c * rows_per_cta), r1 = std::min(n, (c + 1) * rows_per_cta);
        for (int w0 = r0; w0 < r1; w0 += 4) {
            const int w1 = std::min(r1, w0 + 4);
            int maxdeg = 0;
            for (int i = w0; i < w1; ++i) maxdeg = std::max(maxdeg, g->h_indptr[i + 1] - g->h_indptr[i]);
            std::vector<std::vector<int>> order(w1 - w0);
            std::vector<std::vector<char>> taken(w1 - w0);
            for (int i = w0; i < w1; ++i) taken[i - w0].assign(g->h_indptr[i + 1] - g->h_indptr[i], 0);
            for (int u = 0; u * CL_LPR < maxdeg; ++u) {
                int load[16] = {0};
                for (int i = w0; i < w1; ++i) {
                    const int beg = g->h_indptr[i], deg = g->h_indptr[i + 1] - beg;
                    auto &tk = taken[i - w0];
                    for (int pick = 0; pick < CL_LPR && (int)order[i - w0].size() < deg; ++pick) {
                        int best = -1, best_load = 1 << 30;
                        for (int q = 0; q < deg; ++q)
                            if (!tk[q] && load[g->h_indices[beg + q] & 15] < best_load) { best = q; best_load = load[g->h_indices[beg + q] & 15]; }
                        tk[best] = 1;
                        ++load[g->h_indices[beg + best] & 15];
                        order[i - w0].push_back(best);
                    }
                }
            }
            for (int i = w0; i < w1; ++i) {
                const int beg = g->h_indptr[i];
                for (size_t q = 0; q < order[i - w0].size(); ++q) {
                    (*cols)[beg + q] = g->h_indices[beg + order[i - w0][q]];
                    (*wts)[beg + q] = (float)g->h_w[beg + order[i - w0][q]];
                }
            }
        }
    }
}

static bool cluster_applies(const oscb_graph *g, const oscb_run_params *p, int64_t R, bool forced)
{
    if (p->precision != OSCB_PREC_F32 || p->noise_mode == OSCB_NOISE_HOST || p->variant == 1) return false;
    if (p->n_states != 2 || p->objective != OSCB_OBJ_MAXCUT) return false;
    ClusterShape sh;
    if (!cluster_shape(g, 8, &sh)) return false;
    if (sh.weighted) {
        // the piggybacked cut sums couplings in float32: exact only for small integers
        if (!g->int_weights) return false;
        double worst = 0.0;
        for (int64_t i = 0; i < g->n; ++i) {
            double t = 0.0;
            for (int e = g->h_indptr[i]; e < g->h_indptr[i + 1]; ++e) t += std::fabs(g->h_w[e]);
            worst = std::max(worst, t);
        }
        if (worst * (double)g->n >= 16777216.0) return false;
    }
    // latency mode pays off while every replica's cluster has SMs of its own
    return forced || R * 8 <= g->sm_count;
}

static void run_cluster(oscb_graph *g, const oscb_run_params *p, int64_t steps, int64_t cadence,
                 const std::vector<long long> &sample_steps, const uint64_t *seeds, int64_t R64, const double *phi0,
                 oscb_run_outputs *out)
{
    cudaStream_t s = g->stream;
    const int n = (int)g->n, R = (int)R64;
    // 16 CTAs per replica while at most half of the SMs are taken (R <= 4 on 148 SMs: 2.07 vs 2.26 us per step of G1; from
    // 8 replicas on, the 16-CTA clusters are slower, 50.6 vs 45.2 ms per 20 000 steps), else the portable 8.
    // OSCB_CLUSTER_SIZE = 8 / 16 forces.
    int CL_SIZE = R * 32 <= g->sm_count ? 16 : 8;
    if (const char *env = getenv("OSCB_CLUSTER_SIZE")) CL_SIZE = atoi(env) == 16 ? 16 : 8;
    ClusterShape sh;
    if (CL_SIZE == 16) {
        // a 16-CTA cluster has to fit one GPC: take it only if all R clusters can be resident at once
        int resident = 0;
        if (cluster_shape(g, 16, &sh)) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3((unsigned)(R * 16));
            cfg.blockDim = dim3((unsigned)sh.threads);
            cfg.dynamicSmemBytes = sh.lay.total;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            const void *f16 = (const void *)k_cluster_fast<16>;
            if (cudaFuncSetAttribute(f16, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.lay.total) != cudaSuccess ||
                cudaFuncSetAttribute(f16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
                cudaOccupancyMaxActiveClusters(&resident, f16, &cfg) != cudaSuccess)
                resident = 0;
            cudaGetLastError();
        }
        if (resident < R) CL_SIZE = 8;
    }
    OSCB_REQUIRE(cluster_shape(g, CL_SIZE, &sh), "the cluster kernel cannot hold this problem (n = %lld)", (long long)g->n);
    const int64_t S = 1 + (int64_t)sample_steps.size();
    const size_t tot = (size_t)n * R;

    DevBuf<double> d_io(tot);
    DevBuf<uint64_t> d_seeds(R);
    d_seeds.upload(seeds, R, s);
    DevBuf<double> d_best(R), d_energy((size_t)R * S), d_btrace((size_t)R * S);
    DevBuf<uint8_t> d_best_states(tot);
    DevBuf<long long> d_first(R), d_samples(std::max<size_t>(1, sample_steps.size()));
    std::vector<double> h_best(R, -std::numeric_limits<double>::infinity());
    std::vector<long long> h_first(R, -1), h_samples(sample_steps);
    for (auto &v : h_samples) v += p->first_step;
    std::vector<float> hks((size_t)steps + 1);
    for (int64_t k = 0; k <= steps; ++k)       // 2 h ks(step): the N = 2 SHIL term is 2 s c
        hks[(size_t)k] = (float)(2.0 * p->h * ks_value(p->ks_max, p->ks_period, (double)(p->first_step + k) * p->h));
    DevBuf<float> d_hks(hks.size());
    d_best.upload(h_best.data(), R, s);
    d_first.upload(h_first.data(), R, s);
    d_samples.upload(h_samples.data(), h_samples.size(), s);
    d_hks.upload(hks.data(), hks.size(), s);
    d_best_states.zero(s);
    const unsigned long long none = ~0ull;
    OSCB_CUDA(cudaMemcpyAsync(g->d_nonfinite.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));
    if (phi0) d_io.upload(phi0, tot, s);
    else k_initial_phases<<<(unsigned)(((long long)((n + 3) / 4) * R + 127) / 128), 128, 0, s>>>(d_seeds.p, d_io.p, n, R);

    ClusterArgs a;
    memset(&a, 0, sizeof(a));
    a.n = n; a.n_al = sh.n_al; a.rows_per_cta = sh.rows_per_cta; a.nnz_cap = sh.nnz_cap; a.weighted = sh.weighted ? 1 : 0;
    a.R_real = R;
    a.noise_on = (p->noise_mode == OSCB_NOISE_DEVICE && p->kn != 0.0) ? 1 : 0;
    a.use_target = p->use_target; a.initial_sample = 1; a.n_sample_steps = (int)sample_steps.size(); a.sample_offset = 1;
    a.hK = (float)(p->h * p->K); a.knsh = (float)(p->kn * std::sqrt(p->h));
    a.step_begin = p->first_step; a.step_end = p->first_step + steps; a.cadence = cadence; a.trace_stride = S;
    a.target = p->target_objective;
    a.off_cs = (uint32_t)sh.lay.cs; a.off_phi = (uint32_t)sh.lay.phi; a.off_st = (uint32_t)sh.lay.st;
    a.off_rowptr = (uint32_t)sh.lay.rowptr; a.off_rowsum = (uint32_t)sh.lay.rowsum; a.off_col = (uint32_t)sh.lay.col;
    a.off_sums = (uint32_t)sh.lay.sums; a.off_negw = (uint32_t)sh.lay.negw; a.off_kick = (uint32_t)sh.lay.kick;
    a.off_w = (uint32_t)sh.lay.w; a.off_xpart = (uint32_t)sh.lay.xpart; a.off_red = (uint32_t)sh.lay.red;
    a.off_misc = (uint32_t)sh.lay.misc; a.smem_total = (uint32_t)sh.lay.total;
    std::vector<int> h_cols;
    std::vector<float> h_wts;
    cluster_order_columns(g, CL_SIZE, sh.rows_per_cta, &h_cols, &h_wts);
    DevBuf<int> d_cols(std::max<size_t>(1, h_cols.size()));
    DevBuf<float> d_wts(std::max<size_t>(1, h_wts.size()));
    d_cols.upload(h_cols.data(), h_cols.size(), s);
    d_wts.upload(h_wts.data(), h_wts.size(), s);
    a.indptr = g->d_indptr.p; a.indices = d_cols.p; a.w32 = d_wts.p;
    a.hks_table = d_hks.p; a.phi_io = d_io.p; a.seeds = d_seeds.p; a.sample_steps = d_samples.p;
    a.best_obj = d_best.p; a.energy = d_energy.p; a.best_trace = d_btrace.p; a.best_states = d_best_states.p;
    a.first_hit = d_first.p; a.nonfinite = g->d_nonfinite.p;
    DevBuf<long long> d_dbg;
    if (getenv("OSCB_CLUSTER_TRACE")) { d_dbg.alloc(8); d_dbg.zero(s); a.dbg = d_dbg.p; }

    const void *fn = CL_SIZE == 16 ? (const void *)k_cluster_fast<16> : (const void *)k_cluster_fast<8>;
    OSCB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh.lay.total));
    if (CL_SIZE > 8) OSCB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    OSCB_CUDA(cudaStreamSynchronize(s));        // the host staging vectors die after this call
    cudaEvent_t ev0, ev1;
    OSCB_CUDA(cudaEventCreate(&ev0));
    OSCB_CUDA(cudaEventCreate(&ev1));
    OSCB_CUDA(cudaEventRecord(ev0, s));
    if (CL_SIZE == 16) k_cluster_fast<16><<<(unsigned)(R * 16), sh.threads, sh.lay.total, s>>>(a);
    else k_cluster_fast<8><<<(unsigned)(R * 8), sh.threads, sh.lay.total, s>>>(a);
    OSCB_CUDA(cudaEventRecord(ev1, s));
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            set_error("oscb_run(cluster): kernel launch failed: %s (clusters %d, threads %d, smem %zu)", cudaGetErrorString(e), R,
                      sh.threads, sh.lay.total);
            throw OscbFail{OSCB_ECUDA};
        }
    }
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
    if (a.dbg) {
        long long h[8];
        OSCB_CUDA(cudaMemcpy(h, d_dbg.p, sizeof(h), cudaMemcpyDeviceToHost));
        fprintf(stderr, "cluster trace (cycles per step, CTA 0): phase A %.0f, phase B %.0f, barrier %.0f, all %.0f\n", (double)h[0] / steps,
                (double)h[1] / steps, (double)h[2] / steps, (double)h[3] / steps);
    }
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
    out->kernel_used = OSCB_KERNEL_CLUSTER;
    out->replicas_per_cta = 1;
    out->smem_bytes = (int64_t)sh.lay.total;
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
