// oscb.cu -- the C ABI of liboscb.so (include/oscb.h): graph upload, single-step / score /
// energy entry points and the integrate loop, dispatching to the streaming kernels
// (oscb_stream.cuh), the persistent shared-memory kernel (oscb_resident.cuh) or the dense
// path (oscb_dense.cuh).  Everything numerical runs on the GPU; there is no CPU fallback.
//
// Reference behaviour restated by this file (paths relative to /root/reference/pkg/src/oscim/):
//   _simulate loop / sample scheduling / cadence     dynamics.py:333-431, :325-330
//   euler_step                                       dynamics.py:286-314
//   _score_kernel + score() best tracking            dynamics.py:193-223, :370-375
//   _check_finite                                    dynamics.py:276-283
#include "oscb_host.hpp"
#include "oscb_stream.cuh"
#include "oscb_resident_host.hpp"
#include "oscb_dense_host.hpp"
#include "oscb_umma.hpp"
#include "oscb_lowdeg.hpp"
#include "oscb_cluster_host.hpp"
#include <type_traits>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <utility>

namespace oscb {

static thread_local std::string g_last_error;

void set_error(const char *fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

// ---- device block pool -------------------------------------------------------------------
static std::mutex g_pool_mutex;
static std::map<std::pair<int, size_t>, std::vector<void *>> g_pool;
static size_t g_pool_bytes = 0;
static const size_t kPoolCap = (size_t)8 << 30;     // parked bytes above which frees go straight to cudaFree

void *pool_alloc(size_t bytes)
{
    int dev = 0;
    OSCB_CUDA(cudaGetDevice(&dev));
    bytes = (bytes + 255) & ~(size_t)255;
    {
        std::lock_guard<std::mutex> lock(g_pool_mutex);
        auto it = g_pool.find({dev, bytes});
        if (it != g_pool.end() && !it->second.empty()) {
            void *p = it->second.back();
            it->second.pop_back();
            g_pool_bytes -= bytes;
            return p;
        }
    }
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation) {            // give the parked blocks back and retry once
        cudaGetLastError();
        pool_trim();
        e = cudaMalloc(&p, bytes);
    }
    if (e != cudaSuccess) {
        set_error("cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
        throw OscbFail{e == cudaErrorMemoryAllocation ? OSCB_ENOMEM : OSCB_ECUDA};
    }
    return p;
}

void pool_free(void *p, size_t bytes)
{
    if (!p) return;
    bytes = (bytes + 255) & ~(size_t)255;
    cudaPointerAttributes attr;
    int dev = 0;
    if (cudaPointerGetAttributes(&attr, p) == cudaSuccess) dev = attr.device;
    else cudaGetLastError();
    std::lock_guard<std::mutex> lock(g_pool_mutex);
    if (g_pool_bytes + bytes > kPoolCap) {
        cudaFree(p);
        return;
    }
    g_pool[{dev, bytes}].push_back(p);
    g_pool_bytes += bytes;
}

void pool_trim()
{
    std::lock_guard<std::mutex> lock(g_pool_mutex);
    for (auto &kv : g_pool)
        for (void *p : kv.second) cudaFree(p);
    g_pool.clear();
    g_pool_bytes = 0;
}

template <typename F> static int guarded(F &&f)
{
    try {
        return f();
    } catch (const OscbFail &e) {
        return e.code;
    } catch (const std::bad_alloc &) {
        set_error("host allocation failed");
        return OSCB_ENOMEM;
    } catch (const std::exception &e) {
        set_error("internal error: %s", e.what());
        return OSCB_ECUDA;
    }
}

static inline unsigned blocks_for(long long total, int threads) { return (unsigned)((total + threads - 1) / threads); }

void launch_initial_phases(const uint64_t *d_seeds, double *d_phi, int n, int R, cudaStream_t s)
{
    k_initial_phases<<<blocks_for((long long)((n + 3) / 4) * R, 128), 128, 0, s>>>(d_seeds, d_phi, n, R);
}

// dynamics.py:325-330 (Python round() == round-half-even == nearbyint in the default mode)
static int64_t reference_cadence(int64_t n, int64_t pair_count)
{
    const double q = std::nearbyint((double)pair_count / (double)std::max<int64_t>(n, 1));
    return std::max<int64_t>(1, std::min<int64_t>(10, (int64_t)q));
}

// steps after which the reference takes a trace sample (dynamics.py:385, :404-408), computed
// with the same float arithmetic so the schedule is identical
static std::vector<long long> reference_sample_steps(int64_t steps, double h, double stride)
{
    std::vector<long long> out;
    double next_sample = stride;
    for (int64_t step = 0; step < steps; ++step) {
        const double t_next = (double)(step + 1) * h;
        if (t_next >= next_sample || step == steps - 1) {
            while (next_sample <= t_next) next_sample += stride;
            out.push_back(step);
        }
    }
    return out;
}

static void decode_nonfinite(unsigned long long key, int64_t out[3])
{
    out[2] = (int64_t)(key >> 36);
    out[0] = (int64_t)((key >> 20) & 0xFFFFull);
    out[1] = (int64_t)(key & 0xFFFFFull);
}

static void bind_device(const oscb_graph *g) { OSCB_CUDA(cudaSetDevice(g->device)); }

// ------------------------------------------------------------------------------------------
// graph construction
static oscb_graph *new_handle(int device)
{
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        set_error("no usable CUDA device (%s); liboscb has no CPU fallback", cudaGetErrorString(e));
        throw OscbFail{OSCB_ECUDA};
    }
    OSCB_REQUIRE(device >= 0 && device < count, "device %d out of range (have %d)", device, count);
    OSCB_CUDA(cudaSetDevice(device));
    std::unique_ptr<oscb_graph> g(new oscb_graph());
    g->device = device;
    OSCB_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    cudaDeviceProp prop;
    OSCB_CUDA(cudaGetDeviceProperties(&prop, device));
    g->sm_count = prop.multiProcessorCount;
    g->smem_optin = (int)prop.sharedMemPerBlockOptin;
    g->d_nonfinite.alloc(1);
    return g.release();
}

static void finish_csr(oscb_graph *g)
{
    const int64_t n = g->n, nnz = g->nnz;
    std::vector<int> iu, jv;
    std::vector<double> pw;
    std::vector<float> w32((size_t)nnz);
    bool unit = true, integral = true;
    int64_t maxdeg = 0;
    for (int64_t i = 0; i < n; ++i) {
        maxdeg = std::max<int64_t>(maxdeg, g->h_indptr[i + 1] - g->h_indptr[i]);
        for (int e = g->h_indptr[i]; e < g->h_indptr[i + 1]; ++e) {
            const double w = g->h_w[e];
            w32[e] = (float)w;
            if (w != 1.0) unit = false;
            if (w != std::nearbyint(w) || std::fabs(w) > 1e9) integral = false;
            if (i < g->h_indices[e]) {
                iu.push_back((int)i);
                jv.push_back(g->h_indices[e]);
                pw.push_back(w);
            }
        }
    }
    g->pairs = (int64_t)iu.size();
    g->unit_weights = unit;
    g->int_weights = integral;
    g->max_degree = maxdeg;
    cudaStream_t s = g->stream;
    g->d_indptr.alloc(n + 1);  g->d_indptr.upload(g->h_indptr.data(), n + 1, s);
    g->d_indices.alloc(nnz);   g->d_indices.upload(g->h_indices.data(), nnz, s);
    g->d_w64.alloc(nnz);       g->d_w64.upload(g->h_w.data(), nnz, s);
    g->d_w32.alloc(nnz);       g->d_w32.upload(w32.data(), nnz, s);
    g->d_iu.alloc(iu.size());  g->d_iu.upload(iu.data(), iu.size(), s);
    g->d_jv.alloc(jv.size());  g->d_jv.upload(jv.data(), jv.size(), s);
    g->d_pw.alloc(pw.size());  g->d_pw.upload(pw.data(), pw.size(), s);
    OSCB_CUDA(cudaStreamSynchronize(s));
}

static CsrDev csr_view(const oscb_graph *g)
{
    CsrDev c;
    c.n = (int)g->n;
    c.indptr = g->d_indptr.p;
    c.indices = g->d_indices.p;
    c.w64 = g->d_w64.p;
    c.w32 = g->d_w32.p;
    return c;
}

// ------------------------------------------------------------------------------------------
// streaming-path workspace for R replicas in precision T
template <typename T> struct StreamWork {
    using T2 = typename Vec2<T>::type;
    int n, R;
    DevBuf<T> phi[2];
    DevBuf<T2> cs[2];
    DevBuf<double> io;          // [R, n] float64 staging in the host layout
    DevBuf<uint8_t> states;     // [n, R]
    DevBuf<double> partial, obj, dense_partial;
    int P = 1, chunk = 1;
    int cur = 0;

    StreamWork(const oscb_graph *g, int R_) : n((int)g->n), R(R_)
    {
        const size_t tot = (size_t)n * R;
        for (int k = 0; k < 2; ++k) { phi[k].alloc(tot); cs[k].alloc(tot); }
        io.alloc(tot);
        states.alloc(tot);
        const int m = (int)g->pairs;
        P = std::max(1, std::min(64, (m + 255) / 256));
        chunk = (m + P - 1) / P;
        if (chunk < 1) chunk = 1;
        partial.alloc((size_t)P * R);
        obj.alloc(R);
        if (g->is_dense) dense_partial.alloc((size_t)n * R);
    }
    // host-layout float64 phases already in `io` -> device layout + trig
    void load_from_io(cudaStream_t s)
    {
        const long long tot = (long long)n * R;
        k_to_dev_layout<T><<<blocks_for(tot, 256), 256, 0, s>>>(io.p, phi[cur].p, n, R);
        k_trig<T><<<blocks_for(tot, 256), 256, 0, s>>>(phi[cur].p, cs[cur].p, tot);
    }
    void store_to_io(cudaStream_t s)
    {
        const long long tot = (long long)n * R;
        k_from_dev_layout<T><<<blocks_for(tot, 256), 256, 0, s>>>(phi[cur].p, io.p, n, R);
    }
};

template <typename T, bool STRICT>
static void launch_stream_step(const oscb_graph *g, StreamWork<T> &wk, const uint64_t *d_seeds,
                               const double *d_noise, const StepScalars &sc)
{
    const long long threads = (long long)((g->n + 3) / 4) * wk.R;
    const int nxt = wk.cur ^ 1;
    if (g->is_dense)
        launch_dense_step<T>(g, g->stream, wk.R, wk.phi[wk.cur].p, wk.cs[wk.cur].p, wk.phi[nxt].p, wk.cs[nxt].p, d_seeds,
                             d_noise, sc);
    else
        k_stream_step<T, STRICT><<<blocks_for(threads, 256), 256, 0, g->stream>>>(
            csr_view(g), wk.R, wk.phi[wk.cur].p, wk.cs[wk.cur].p, wk.phi[nxt].p, wk.cs[nxt].p, d_seeds,
            d_noise, sc, g->d_nonfinite.p);
    wk.cur = nxt;
}

// threshold + objective of the current phases -> wk.obj (and best bookkeeping when asked)
template <typename T>
static int launch_stream_score(const oscb_graph *g, StreamWork<T> &wk, int n_states, int maximize,
                               bool sequential, double *best_obj, uint8_t *improved,
                               uint8_t *best_states, long long *first_hit, int use_target,
                               double target, long long step)
{
    cudaStream_t s = g->stream;
    const long long tot = (long long)wk.n * wk.R;
    int launches = 0;
    k_threshold<T><<<blocks_for(tot, 256), 256, 0, s>>>(wk.phi[wk.cur].p, wk.states.p, tot, n_states);
    ++launches;
    int P = wk.P;
    if (g->is_dense) {
        launch_dense_pairs<T>(g, s, wk.R, maximize ? 0 : 1, wk.states.p, nullptr, wk.dense_partial.p, wk.partial.p, 1);
        P = 1;
        ++launches;
    } else if (sequential) {
        k_objective_seq<<<blocks_for(wk.R, 64), 64, 0, s>>>(wk.states.p, wk.R, g->d_iu.p, g->d_jv.p,
                                                            g->d_pw.p, (int)g->pairs, maximize, wk.partial.p);
        P = 1;
    } else {
        dim3 grid(blocks_for(wk.R, 32), (unsigned)wk.P);
        k_objective_partial<<<grid, 256, 0, s>>>(wk.states.p, wk.R, g->d_iu.p, g->d_jv.p, g->d_pw.p,
                                                 (int)g->pairs, wk.chunk, maximize, wk.partial.p);
    }
    ++launches;
    k_best_flag<<<blocks_for(wk.R, 128), 128, 0, s>>>(wk.partial.p, P, wk.obj.p, best_obj, improved,
                                                      first_hit, wk.R, maximize, use_target, target, step);
    ++launches;
    if (best_obj) {
        k_best_copy<<<blocks_for(tot, 256), 256, 0, s>>>(wk.states.p, improved, best_states, wk.n, wk.R);
        ++launches;
    }
    return launches;
}

static void check_launch(const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: kernel launch failed: %s", what, cudaGetErrorString(e));
        throw OscbFail{OSCB_ECUDA};
    }
}

// ------------------------------------------------------------------------------------------
// single step (euler_step parity entry point)
template <typename T, bool STRICT>
static void step_impl(oscb_graph *g, int64_t R, const double *phi_in, const double *noise, double K,
                      double ks, double h, double kn_sqrt_h, int n_states, double *phi_out,
                      int64_t *nonfinite)
{
    cudaStream_t s = g->stream;
    const size_t tot = (size_t)g->n * R;
    StreamWork<T> wk(g, (int)R);
    DevBuf<double> d_noise;
    wk.io.upload(phi_in, tot, s);
    if (noise) { d_noise.alloc(tot); d_noise.upload(noise, tot, s); }
    const unsigned long long none = ~0ull;
    OSCB_CUDA(cudaMemcpyAsync(g->d_nonfinite.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));
    wk.load_from_io(s);
    StepScalars sc;
    sc.K = K; sc.ks = ks; sc.h = h; sc.kn_sqrt_h = kn_sqrt_h;
    sc.tc = make_trig_const(n_states);
    sc.step = 0;
    sc.noise_mode = noise ? OSCB_NOISE_HOST : OSCB_NOISE_NONE;
    launch_stream_step<T, STRICT>(g, wk, nullptr, d_noise.p, sc);
    check_launch("oscb_step");
    wk.store_to_io(s);
    wk.io.download(phi_out, tot, s);
    unsigned long long flag = none;
    OSCB_CUDA(cudaMemcpyAsync(&flag, g->d_nonfinite.p, sizeof(flag), cudaMemcpyDeviceToHost, s));
    OSCB_CUDA(cudaStreamSynchronize(s));
    if (nonfinite) { nonfinite[0] = -1; nonfinite[1] = -1; }
    if (flag != none) {
        int64_t where[3];
        decode_nonfinite(flag, where);
        if (nonfinite) { nonfinite[0] = where[0]; nonfinite[1] = where[1]; }
        set_error("non-finite phase for oscillator %lld (replica row %lld)", (long long)where[1], (long long)where[0]);
        throw OscbFail{OSCB_ENONFINITE};
    }
}

// ------------------------------------------------------------------------------------------
// the integrate loop on the streaming kernels
struct RunPlan {
    int64_t steps, cadence;
    double stride;
    std::vector<long long> sample_steps; // a sample follows each of these steps
    int64_t n_samples;                   // 1 + sample_steps.size()
};

static RunPlan make_run_plan(const oscb_graph *g, const oscb_run_params *p)
{
    RunPlan rp;
    rp.steps = p->steps > 0 ? p->steps : (int64_t)std::ceil(p->t_stop / p->h);
    rp.cadence = p->cadence == 0 ? reference_cadence(g->n, g->pairs) : p->cadence;
    rp.stride = p->trace_stride > 0.0 ? p->trace_stride : p->ks_period / 2.0;
    rp.sample_steps = reference_sample_steps(rp.steps, p->h, rp.stride);
    rp.n_samples = 1 + (int64_t)rp.sample_steps.size();
    return rp;
}

template <typename T, bool STRICT>
static void run_stream(oscb_graph *g, const oscb_run_params *p, const RunPlan &rp, const uint64_t *seeds,
                       int64_t R64, const double *phi0, const double *noise, oscb_run_outputs *out)
{
    cudaStream_t s = g->stream;
    const int R = (int)R64, n = (int)g->n;
    const size_t tot = (size_t)n * R;
    const int maximize = p->objective == OSCB_OBJ_MAXCUT;
    const int64_t S = rp.n_samples;

    StreamWork<T> wk(g, R);
    DevBuf<uint64_t> d_seeds(R);
    d_seeds.upload(seeds, R, s);
    DevBuf<double> d_best(R), d_energy((size_t)R * S), d_btrace((size_t)R * S), d_noise;
    DevBuf<uint8_t> d_improved(R), d_best_states(tot);
    DevBuf<long long> d_first(R);
    {
        std::vector<double> init(R, maximize ? -std::numeric_limits<double>::infinity()
                                             : std::numeric_limits<double>::infinity());
        d_best.upload(init.data(), R, s);
        std::vector<long long> neg(R, -1);
        d_first.upload(neg.data(), R, s);
        OSCB_CUDA(cudaStreamSynchronize(s)); // the staging vectors die here
    }
    d_best_states.zero(s);
    const unsigned long long none = ~0ull;
    OSCB_CUDA(cudaMemcpyAsync(g->d_nonfinite.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));

    if (phi0) wk.io.upload(phi0, tot, s);
    else k_initial_phases<<<blocks_for((long long)((n + 3) / 4) * R, 128), 128, 0, s>>>(d_seeds.p, wk.io.p, n, R);
    wk.load_from_io(s);

    const long long noise_rows = p->noise_mode == OSCB_NOISE_HOST ? 256 : 0; // upload window (steps)
    if (noise_rows) d_noise.alloc((size_t)noise_rows * tot);

    cudaEvent_t ev0, ev1;
    OSCB_CUDA(cudaEventCreate(&ev0));
    OSCB_CUDA(cudaEventCreate(&ev1));
    int64_t launches = 0;
    OSCB_CUDA(cudaEventRecord(ev0, s));

    auto score = [&](long long step_label) {
        launches += launch_stream_score<T>(g, wk, p->n_states, maximize, false, d_best.p, d_improved.p,
                                           d_best_states.p, d_first.p, p->use_target, p->target_objective,
                                           step_label);
    };
    auto sample = [&](long long step_label, int64_t col) {
        score(step_label);
        if (g->is_dense)
            launch_dense_pairs<T>(g, s, R, 2, nullptr, wk.cs[wk.cur].p, wk.dense_partial.p, d_energy.p + col, S);
        else
            k_energy<T><<<R, 256, 0, s>>>(wk.phi[wk.cur].p, R, g->d_iu.p, g->d_jv.p, g->d_pw.p, (int)g->pairs,
                                          d_energy.p + col, S);
        k_record_best<<<blocks_for(R, 128), 128, 0, s>>>(d_best.p, d_btrace.p + col, S, R);
        launches += 2;
    };

    sample(-1, 0);
    size_t next_sample = 0;
    StepScalars sc;
    sc.K = p->K; sc.h = p->h; sc.kn_sqrt_h = p->kn * std::sqrt(p->h);
    sc.tc = make_trig_const(p->n_states);
    sc.noise_mode = p->noise_mode;
    if (p->kn == 0.0 && p->noise_mode == OSCB_NOISE_DEVICE) sc.noise_mode = OSCB_NOISE_NONE;
    for (int64_t step = 0; step < rp.steps; ++step) {
        const int64_t gstep = p->first_step + step;
        sc.ks = ks_value(p->ks_max, p->ks_period, (double)gstep * p->h);
        sc.step = (uint64_t)gstep;
        const double *noise_dev = nullptr;
        if (noise_rows) {
            if (step % noise_rows == 0) {
                const int64_t rows = std::min<int64_t>(noise_rows, rp.steps - step);
                OSCB_CUDA(cudaStreamSynchronize(s)); // previous window fully consumed
                d_noise.upload(noise + (size_t)step * tot, (size_t)rows * tot, s);
            }
            noise_dev = d_noise.p + (size_t)(step % noise_rows) * tot;
        }
        launch_stream_step<T, STRICT>(g, wk, d_seeds.p, noise_dev, sc);
        ++launches;
        if (next_sample < rp.sample_steps.size() && rp.sample_steps[next_sample] == step) {
            sample(gstep, 1 + (int64_t)next_sample);
            ++next_sample;
        } else if (rp.cadence > 0 && gstep % rp.cadence == 0) {
            score(gstep);
        }
    }
    OSCB_CUDA(cudaEventRecord(ev1, s));
    check_launch("oscb_run(stream)");

    wk.store_to_io(s);
    if (out->final_phases) wk.io.download(out->final_phases, tot, s);
    if (out->best_states) d_best_states.download(out->best_states, tot, s);
    if (out->best_objective) d_best.download(out->best_objective, R, s);
    std::vector<double> h_energy, h_btrace;
    if (out->energy) { h_energy.resize((size_t)R * S); d_energy.download(h_energy.data(), h_energy.size(), s); }
    if (out->best_trace) { h_btrace.resize((size_t)R * S); d_btrace.download(h_btrace.data(), h_btrace.size(), s); }
    std::vector<long long> h_first;
    if (out->first_hit_step) { h_first.resize(R); d_first.download(h_first.data(), R, s); }
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
    out->kernel_used = OSCB_KERNEL_STREAM;
    out->replicas_per_cta = 0;
    out->smem_bytes = 0;
    if (flag != none) {
        decode_nonfinite(flag, out->nonfinite);
        set_error("non-finite phase for oscillator %lld (replica row %lld) after step %lld; parameters are numerically unstable",
                  (long long)out->nonfinite[1], (long long)out->nonfinite[0], (long long)out->nonfinite[2]);
        throw OscbFail{OSCB_ENONFINITE};
    }
}

// ------------------------------------------------------------------------------------------
// the integrate loop of a dense integer-coupled max-cut graph on the tensor cores
// (oscb_umma.cuh): one persistent launch per chunk of <= 28 replicas
static bool umma_applies(const oscb_graph *g, const oscb_run_params *p)
{
    // OIM: N = 2 max-cut on any integer couplings; OPM: N-state colouring on unit couplings (the conflict
    // count ignores weights, dynamics.py:219-222, and sum_j J_ij [s_j == s_i] counts only when J is 0/1)
    const bool oim = p->n_states == 2 && p->objective == OSCB_OBJ_MAXCUT;
    const bool opm = p->n_states >= 3 && p->n_states <= 16 && p->objective == OSCB_OBJ_COLORING && g->unit_weights;
    return g->is_dense && g->umma && (oim || opm) && p->noise_mode != OSCB_NOISE_HOST && p->kernel != OSCB_KERNEL_STREAM;
}

// which passes score / sample: pass q integrates step q and first scores the phases it starts
// from (= the reference's score after step q - 1, dynamics.py:404-410)
struct UmmaSchedule {
    std::vector<uint8_t> flags;            // [steps + 1]
    std::vector<long long> event_step;     // step label of every scored pass (-1: initial sample)
    std::vector<long long> sample_event;   // event index of every sample
};

static UmmaSchedule umma_schedule(const oscb_run_params *p, const RunPlan &rp)
{
    UmmaSchedule sc;
    sc.flags.assign((size_t)rp.steps + 1, 0);
    sc.flags[0] = 3;
    sc.event_step.push_back(-1);
    sc.sample_event.push_back(0);
    size_t next_sample = 0;
    for (int64_t step = 0; step < rp.steps; ++step) {
        const int64_t gstep = p->first_step + step;
        if (next_sample < rp.sample_steps.size() && rp.sample_steps[next_sample] == step) {
            sc.flags[(size_t)step + 1] = 3;
            sc.sample_event.push_back((long long)sc.event_step.size());
            sc.event_step.push_back(gstep);
            ++next_sample;
        } else if (rp.cadence > 0 && gstep % rp.cadence == 0) {
            sc.flags[(size_t)step + 1] = 1;
            sc.event_step.push_back(gstep);
        }
    }
    return sc;
}

static UmmaSpec umma_spec(const oscb_run_params *p, const RunPlan &rp, const UmmaSchedule &sc, int R)
{
    UmmaSpec sp{};
    sp.R = R;
    sp.precision = p->precision;
    sp.noise_on = (p->noise_mode == OSCB_NOISE_DEVICE && p->kn != 0.0) ? 1 : 0;
    sp.n_states = p->n_states;
    sp.maximize = p->objective == OSCB_OBJ_MAXCUT ? 1 : 0;
    sp.K = p->K; sp.h = p->h; sp.kn_sqrt_h = p->kn * std::sqrt(p->h); sp.ks_max = p->ks_max; sp.ks_period = p->ks_period;
    sp.steps = rp.steps; sp.first_step = p->first_step;
    sp.flags = sc.flags.data();
    sp.n_events = (long long)sc.event_step.size();
    sp.n_samples = rp.n_samples;
    sp.force_stream = (p->variant == 8 || p->variant == 4) ? p->variant : 0;
    return sp;
}

// the score() / sample() bookkeeping of dynamics.py:370-384 replayed on the recorded cut sums
// (ev[e][r] = 2 * cut of scored pass e) for replicas [r0, r0 + Rc) of the outputs
static void umma_bookkeeping(const oscb_run_params *p, const UmmaSchedule &sc, const long long *ev, const double *en, int Rc,
                             int r0, oscb_run_outputs *out)
{
    const long long E = (long long)sc.event_step.size();
    for (int r = 0; r < Rc; ++r) {
        const bool maximize = p->objective == OSCB_OBJ_MAXCUT;
        double best = maximize ? -std::numeric_limits<double>::infinity() : std::numeric_limits<double>::infinity();
        long long first = -1;
        size_t k = 0;
        for (long long e = 0; e < E; ++e) {
            const double obj = 0.5 * (double)ev[(size_t)e * Rc + r];
            if (maximize ? obj > best : obj < best) {
                best = obj;
                if (p->use_target && first < 0 && (maximize ? obj >= p->target_objective : obj <= p->target_objective))
                    first = sc.event_step[(size_t)e];
            }
            if (k < sc.sample_event.size() && sc.sample_event[k] == e) {
                if (out->best_trace) out->best_trace[(size_t)(r0 + r) * out->max_samples + k] = best;
                if (out->energy) out->energy[(size_t)(r0 + r) * out->max_samples + k] = en[k * Rc + r];
                ++k;
            }
        }
        if (out->best_objective) out->best_objective[r0 + r] = best;
        if (out->first_hit_step) out->first_hit_step[r0 + r] = first;
    }
}

static void umma_raise_nonfinite(unsigned long long flag, oscb_run_outputs *out)
{
    if (flag == ~0ull) return;
    decode_nonfinite(flag, out->nonfinite);
    set_error("non-finite phase for oscillator %lld (replica row %lld) after step %lld; parameters are numerically unstable",
              (long long)out->nonfinite[1], (long long)out->nonfinite[0], (long long)out->nonfinite[2]);
    throw OscbFail{OSCB_ENONFINITE};
}

static void run_umma(oscb_graph *g, const oscb_run_params *p, const RunPlan &rp, const uint64_t *seeds, int64_t R64,
                     const double *phi0, oscb_run_outputs *out)
{
    cudaStream_t s = g->stream;
    const int R = (int)R64, n = (int)g->n;
    const size_t tot = (size_t)n * R;
    const int64_t S = rp.n_samples;
    const UmmaSchedule sc = umma_schedule(p, rp);
    const long long E = (long long)sc.event_step.size();
    DevBuf<double> io(tot);
    DevBuf<uint64_t> d_seeds(R);
    d_seeds.upload(seeds, R, s);
    if (phi0) io.upload(phi0, tot, s);
    else k_initial_phases<<<blocks_for((long long)((n + 3) / 4) * R, 128), 128, 0, s>>>(d_seeds.p, io.p, n, R);
    DevBuf<double> d_final(tot);
    double ms = 0.0;
    int64_t launches = 0, smem = 0;
    unsigned long long flag = ~0ull;
    const int chunk = umma_max_replicas(p->n_states, umma_uses_fp4(*g->umma, R, p->n_states));
    for (int r0 = 0; r0 < R; r0 += chunk) {
        const int Rc = std::min(chunk, R - r0);
        std::vector<long long> ev((size_t)E * Rc);
        std::vector<double> en((size_t)S * Rc);
        UmmaSpec spc = umma_spec(p, rp, sc, Rc);
        spc.R_total = R;
        const bool timing = getenv("OSCB_UMMA_TIMING") != nullptr;
        auto now = [] { return std::chrono::steady_clock::now(); };
        auto since = [&](std::chrono::steady_clock::time_point t0) { return std::chrono::duration<double, std::milli>(now() - t0).count(); };
        auto t0 = now();
        UmmaSession ses(g, spc, 1, 0);
        const double t_ctor = since(t0); t0 = now();
        ses.prepare(seeds + r0, io.p + (size_t)r0 * n);
        const double t_prep = since(t0); t0 = now();
        ses.launch();
        ses.export_final(d_final.p + (size_t)r0 * n);
        const double t_launch = since(t0); t0 = now();
        ses.finish(nullptr, out->best_states ? out->best_states + (size_t)r0 * n : nullptr, ev.data(), en.data());
        if (timing) fprintf(stderr, "[umma] ctor %.2f prepare %.2f launch %.2f finish %.2f (kernel %.2f) ms\n", t_ctor, t_prep, t_launch, since(t0), ses.ms);
        ms += ses.ms;
        launches += 1;
        smem = (int64_t)ses.smem;
        flag = std::min(flag, ses.nonfinite == ~0ull ? ~0ull : ses.nonfinite + ((unsigned long long)r0 << 20));
        umma_bookkeeping(p, sc, ev.data(), en.data(), Rc, r0, out);
    }
    if (out->final_phases) d_final.download(out->final_phases, tot, s);
    OSCB_CUDA(cudaStreamSynchronize(s));
    out->device_ms = ms;
    out->kernel_launches = launches;
    out->kernel_used = OSCB_KERNEL_DENSE_TC;
    out->replicas_per_cta = std::min(R, chunk);
    out->smem_bytes = smem;
    umma_raise_nonfinite(flag, out);
}

// workspace of the row-sharded dense driver: pairs and states of all n oscillators, row partials
struct ShardWork {
    int R = 0, precision = 0;
    DevBuf<unsigned char> cs;      // [n][R] pairs in the call's precision
    DevBuf<uint8_t> states;        // [n][R]
    DevBuf<double> partial;        // [rows][R]
    bool flag_armed = false;
};

static ShardWork &shard_work(oscb_graph *g, int R, int precision)
{
    if (!g->shard_work || g->shard_work->R != R || g->shard_work->precision != precision) {
        auto w = std::make_shared<ShardWork>();
        w->R = R;
        w->precision = precision;
        const size_t tot = (size_t)g->n * R;
        w->cs.alloc(tot * (precision == OSCB_PREC_F64 ? 16 : 8));
        w->states.alloc(tot);
        w->partial.alloc((size_t)(g->row_end - g->row_begin) * R);
        g->shard_work = w;
    }
    if (!g->shard_work->flag_armed) {
        const unsigned long long none = ~0ull;
        OSCB_CUDA(cudaMemcpy(g->d_nonfinite.p, &none, sizeof(none), cudaMemcpyHostToDevice));
        g->shard_work->flag_armed = true;
    }
    return *g->shard_work;
}

template <typename T>
static void shard_step_impl(oscb_graph *g, int R, const oscb_shard_step_params *p, const void *phi_full, void *phi_rows,
                            const uint64_t *seeds_dev, cudaStream_t s)
{
    using T2 = typename Vec2<T>::type;
    ShardWork &w = shard_work(g, R, p->precision);
    const long long tot = (long long)g->n * R;
    T2 *cs = reinterpret_cast<T2 *>(w.cs.p);
    k_trig<T><<<blocks_for(tot, 256), 256, 0, s>>>(reinterpret_cast<const T *>(phi_full), cs, tot);
    StepScalars sc;
    sc.K = p->K; sc.ks = p->ks; sc.h = p->h; sc.kn_sqrt_h = p->kn_sqrt_h;
    sc.tc = make_trig_const(p->n_states);
    sc.step = (uint64_t)p->step;
    sc.noise_mode = p->noise_on ? OSCB_NOISE_DEVICE : OSCB_NOISE_NONE;
    launch_dense_step<T>(g, s, R, reinterpret_cast<const T *>(phi_full), cs, reinterpret_cast<T *>(phi_rows),
                         (T2 *)nullptr, seeds_dev, nullptr, sc);
}

template <typename T>
static void shard_pairs_impl(oscb_graph *g, int R, int precision, const void *phi_full, int mode, int n_states,
                             double *partial_dev, cudaStream_t s)
{
    using T2 = typename Vec2<T>::type;
    ShardWork &w = shard_work(g, R, precision);
    const long long tot = (long long)g->n * R;
    if (mode == 2) {
        T2 *cs = reinterpret_cast<T2 *>(w.cs.p);
        k_trig<T><<<blocks_for(tot, 256), 256, 0, s>>>(reinterpret_cast<const T *>(phi_full), cs, tot);
        launch_dense_pairs<T>(g, s, R, 2, nullptr, cs, w.partial.p, partial_dev, 1);
    } else {
        k_threshold<T><<<blocks_for(tot, 256), 256, 0, s>>>(reinterpret_cast<const T *>(phi_full), w.states.p, tot, n_states);
        launch_dense_pairs<T>(g, s, R, mode, w.states.p, (const T2 *)nullptr, w.partial.p, partial_dev, 1);
    }
}

} // namespace oscb

// one rank of a fused row-sharded dense run (include/oscb.h: oscb_dense_fused_*)
struct oscb_fused {
    oscb_graph *g = nullptr;
    oscb_run_params params{};
    oscb::RunPlan rp;
    oscb::UmmaSchedule sched;
    std::unique_ptr<oscb::UmmaSession> session;
    oscb::DevBuf<double> io;
    int R = 0, world = 1, rank = 0;
};

using namespace oscb;

// ==========================================================================================
extern "C" {

const char *oscb_last_error(void) { return g_last_error.c_str(); }
int oscb_version(void) { return 100; }

int oscb_pool_trim(void)
{
    return guarded([&]() -> int {
        pool_trim();
        return OSCB_OK;
    });
}

int oscb_device_count(int *count)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(count != nullptr, "count is NULL");
        int c = 0;
        cudaError_t e = cudaGetDeviceCount(&c);
        if (e != cudaSuccess) {
            *count = 0;
            set_error("cudaGetDeviceCount: %s", cudaGetErrorString(e));
            return OSCB_ECUDA;
        }
        *count = c;
        return OSCB_OK;
    });
}

int oscb_graph_create_csr(int device, int64_t n, const int64_t *indptr, const int64_t *indices,
                          const double *data, oscb_graph **out)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(out != nullptr, "out is NULL");
        *out = nullptr;
        OSCB_REQUIRE(n >= 1, "problem must have at least one oscillator");
        OSCB_REQUIRE(n < (1ll << 20), "n = %lld exceeds the supported 2^20 oscillators", (long long)n);
        OSCB_REQUIRE(indptr != nullptr, "indptr is NULL");
        const int64_t nnz = indptr[n];
        OSCB_REQUIRE(indptr[0] == 0 && nnz >= 0 && nnz < (1ll << 31), "bad indptr (nnz = %lld)", (long long)nnz);
        OSCB_REQUIRE(nnz == 0 || (indices != nullptr && data != nullptr), "indices/data are NULL");
        std::unique_ptr<oscb_graph> g(new_handle(device));
        g->n = n;
        g->nnz = nnz;
        g->row_begin = 0;
        g->row_end = n;
        g->h_indptr.resize(n + 1);
        g->h_indices.resize(nnz);
        g->h_w.assign(data, data + nnz);
        for (int64_t i = 0; i <= n; ++i) {
            OSCB_REQUIRE(i == 0 || indptr[i] >= indptr[i - 1], "indptr must be non-decreasing");
            g->h_indptr[i] = (int)indptr[i];
        }
        for (int64_t i = 0; i < n; ++i)
            for (int64_t e = indptr[i]; e < indptr[i + 1]; ++e) {
                OSCB_REQUIRE(indices[e] >= 0 && indices[e] < n, "column index out of range in row %lld", (long long)i);
                OSCB_REQUIRE(std::isfinite(data[e]), "non-finite coupling in row %lld", (long long)i);
                g->h_indices[e] = (int)indices[e];
            }
        finish_csr(g.get());
        *out = g.release();
        return OSCB_OK;
    });
}

int oscb_graph_create_dense(int device, int64_t n, const double *J, int64_t row_begin, int64_t row_end,
                            oscb_graph **out)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(out != nullptr, "out is NULL");
        *out = nullptr;
        OSCB_REQUIRE(n >= 1 && J != nullptr, "dense J needs n >= 1 and a matrix");
        OSCB_REQUIRE(n < (1ll << 20), "n = %lld exceeds the supported 2^20 oscillators", (long long)n);
        OSCB_REQUIRE(0 <= row_begin && row_begin < row_end && row_end <= n, "bad row shard [%lld, %lld)",
                     (long long)row_begin, (long long)row_end);
        std::unique_ptr<oscb_graph> g(new_handle(device));
        g->n = n;
        g->is_dense = true;
        g->row_begin = row_begin;
        g->row_end = row_end;
        // J holds rows [row_begin, row_end) of the full matrix, row-major, n columns each
        build_dense(g.get(), J);
        // integer couplings on 128-row aligned shards also get the tile images of the tensor-core kernel
        if (g->dense->kind == DENSE_I8 && g->dense->tc_exact && row_begin % 128 == 0 && (row_end % 128 == 0 || row_end == n))
            g->umma = umma_build_plan(g->dense->J8.p, n, g->dense->n_pad, row_begin, row_end, g->dense->fp4_ok, g->stream);
        *out = g.release();
        return OSCB_OK;
    });
}

int oscb_graph_destroy(oscb_graph *g)
{
    if (!g) return OSCB_OK;
    cudaSetDevice(g->device);
    if (g->stream) {
        cudaStreamSynchronize(g->stream);
    }
    g->plans.clear();
    g->dense.reset();
    g->umma.reset();
    g->shard_work.reset();
    cudaStream_t s = g->stream;
    delete g;
    if (s) cudaStreamDestroy(s);
    return OSCB_OK;
}

int oscb_graph_get_info(const oscb_graph *g, oscb_graph_info *info)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(g && info, "NULL argument");
        info->n = g->n;
        info->nnz = g->nnz;
        info->pairs = g->pairs;
        info->device = g->device;
        info->is_dense = g->is_dense;
        info->unit_weights = g->unit_weights;
        info->int_weights = g->int_weights;
        info->row_begin = g->row_begin;
        info->row_end = g->row_end;
        info->max_degree = g->max_degree;
        return OSCB_OK;
    });
}

int oscb_initial_phases(oscb_graph *g, const uint64_t *seeds, int64_t R, double *phi_out)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(g && seeds && phi_out, "NULL argument");
        OSCB_REQUIRE(R >= 1 && R <= 65536, "replicas must be in [1, 65536]");
        bind_device(g);
        cudaStream_t s = g->stream;
        const int n = (int)g->n;
        DevBuf<uint64_t> d_seeds(R);
        d_seeds.upload(seeds, R, s);
        DevBuf<double> d_phi((size_t)n * R);
        k_initial_phases<<<blocks_for((long long)((n + 3) / 4) * R, 128), 128, 0, s>>>(d_seeds.p, d_phi.p, n, (int)R);
        check_launch("oscb_initial_phases");
        d_phi.download(phi_out, (size_t)n * R, s);
        OSCB_CUDA(cudaStreamSynchronize(s));
        return OSCB_OK;
    });
}

int oscb_device_normals(int device, uint64_t seed, int64_t step, int64_t n, int32_t precision, double *out)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(out != nullptr && n >= 1 && step >= 0, "bad argument");
        OSCB_REQUIRE(precision == OSCB_PREC_F32 || precision == OSCB_PREC_F64, "unknown precision %d", precision);
        int count = 0;
        cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0) {
            set_error("no usable CUDA device (%s); liboscb has no CPU fallback", cudaGetErrorString(e));
            return OSCB_ECUDA;
        }
        OSCB_REQUIRE(device >= 0 && device < count, "device %d out of range (have %d)", device, count);
        OSCB_CUDA(cudaSetDevice(device));
        DevBuf<double> d((size_t)n);
        const unsigned blocks = blocks_for((n + 3) / 4, 128);
        if (precision == OSCB_PREC_F64) k_device_normals<double><<<blocks, 128>>>(seed, (uint64_t)step, (int)n, d.p);
        else k_device_normals<float><<<blocks, 128>>>(seed, (uint64_t)step, (int)n, d.p);
        check_launch("oscb_device_normals");
        OSCB_CUDA(cudaMemcpy(out, d.p, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost));
        return OSCB_OK;
    });
}

int oscb_step(oscb_graph *g, int64_t R, const double *phi_in, const double *noise, double K, double ks,
              double h, double kn_sqrt_h, int32_t n_states, int32_t precision, double *phi_out,
              int64_t *nonfinite)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(g && phi_in && phi_out, "NULL argument");
        OSCB_REQUIRE(R >= 1 && R <= 65536, "replicas must be in [1, 65536]");
        OSCB_REQUIRE(n_states >= 2, "n_states must be >= 2");
        OSCB_REQUIRE(precision == OSCB_PREC_F32 || precision == OSCB_PREC_F64, "unknown precision %d", precision);
        OSCB_REQUIRE(g->row_begin == 0 && g->row_end == g->n, "oscb_step needs the whole graph, not a row shard");
        bind_device(g);
        if (precision == OSCB_PREC_F64)
            step_impl<double, true>(g, R, phi_in, noise, K, ks, h, kn_sqrt_h, n_states, phi_out, nonfinite);
        else
            step_impl<float, false>(g, R, phi_in, noise, K, ks, h, kn_sqrt_h, n_states, phi_out, nonfinite);
        return OSCB_OK;
    });
}

int oscb_score(oscb_graph *g, int64_t R, const double *phi, int32_t n_states, int32_t maximize,
               int64_t *states, double *objective)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(g && phi && objective, "NULL argument");
        OSCB_REQUIRE(R >= 1 && R <= 65536, "replicas must be in [1, 65536]");
        OSCB_REQUIRE(n_states >= 2 && n_states <= 255, "n_states must be in [2, 255]");
        OSCB_REQUIRE(g->row_begin == 0 && g->row_end == g->n, "oscb_score needs the whole graph, not a row shard");
        bind_device(g);
        cudaStream_t s = g->stream;
        const size_t tot = (size_t)g->n * R;
        StreamWork<double> wk(g, (int)R);
        wk.io.upload(phi, tot, s);
        k_to_dev_layout<double><<<blocks_for((long long)tot, 256), 256, 0, s>>>(wk.io.p, wk.phi[0].p, (int)g->n, (int)R);
        launch_stream_score<double>(g, wk, n_states, maximize, !g->int_weights, nullptr, nullptr, nullptr,
                                    nullptr, 0, 0.0, 0);
        check_launch("oscb_score");
        wk.obj.download(objective, R, s);
        if (states) {
            DevBuf<long long> d_states(tot);
            k_states_to_host_layout<<<blocks_for((long long)tot, 256), 256, 0, s>>>(wk.states.p, d_states.p, (int)g->n, (int)R);
            OSCB_CUDA(cudaMemcpyAsync(states, d_states.p, tot * sizeof(long long), cudaMemcpyDeviceToHost, s));
            OSCB_CUDA(cudaStreamSynchronize(s));
        }
        OSCB_CUDA(cudaStreamSynchronize(s));
        return OSCB_OK;
    });
}

int oscb_energy(oscb_graph *g, int64_t R, const double *phi, double *energy)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(g && phi && energy, "NULL argument");
        OSCB_REQUIRE(R >= 1 && R <= 65536, "replicas must be in [1, 65536]");
        OSCB_REQUIRE(g->row_begin == 0 && g->row_end == g->n, "oscb_energy needs the whole graph, not a row shard");
        bind_device(g);
        cudaStream_t s = g->stream;
        const size_t tot = (size_t)g->n * R;
        DevBuf<double> io(tot), dev(tot), en(R);
        io.upload(phi, tot, s);
        k_to_dev_layout<double><<<blocks_for((long long)tot, 256), 256, 0, s>>>(io.p, dev.p, (int)g->n, (int)R);
        if (g->is_dense) {
            DevBuf<double2> cs(tot);
            DevBuf<double> partial(tot);
            k_trig<double><<<blocks_for((long long)tot, 256), 256, 0, s>>>(dev.p, cs.p, (long long)tot);
            launch_dense_pairs<double>(g, s, (int)R, 2, nullptr, cs.p, partial.p, en.p, 1);
            check_launch("oscb_energy");
            en.download(energy, R, s);
            OSCB_CUDA(cudaStreamSynchronize(s));
            return OSCB_OK;
        }
        k_energy<double><<<(unsigned)R, 256, 0, s>>>(dev.p, (int)R, g->d_iu.p, g->d_jv.p, g->d_pw.p, (int)g->pairs, en.p, 1);
        check_launch("oscb_energy");
        en.download(energy, R, s);
        OSCB_CUDA(cudaStreamSynchronize(s));
        return OSCB_OK;
    });
}

int oscb_dense_shard_step(oscb_graph *g, int64_t R, const oscb_shard_step_params *p, const void *phi_full_dev,
                          void *phi_rows_out_dev, const uint64_t *seeds_dev, void *stream)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(g && p && phi_full_dev && phi_rows_out_dev, "NULL argument");
        OSCB_REQUIRE(g->is_dense && g->dense, "oscb_dense_shard_step needs a dense (row shard) handle");
        OSCB_REQUIRE(R >= 1 && R <= 65536, "replicas must be in [1, 65536]");
        OSCB_REQUIRE(p->precision == OSCB_PREC_F32 || p->precision == OSCB_PREC_F64, "unknown precision %d", p->precision);
        OSCB_REQUIRE(p->n_states >= 2 && p->n_states <= 255, "n_states must be in [2, 255]");
        OSCB_REQUIRE(!p->noise_on || seeds_dev != nullptr, "noise needs the seeds");
        bind_device(g);
        cudaStream_t s = stream ? (cudaStream_t)stream : g->stream;
        if (p->precision == OSCB_PREC_F64) shard_step_impl<double>(g, (int)R, p, phi_full_dev, phi_rows_out_dev, seeds_dev, s);
        else shard_step_impl<float>(g, (int)R, p, phi_full_dev, phi_rows_out_dev, seeds_dev, s);
        check_launch("oscb_dense_shard_step");
        return OSCB_OK;
    });
}

int oscb_dense_shard_objective(oscb_graph *g, int64_t R, int32_t precision, const void *phi_full_dev, int32_t n_states,
                               int32_t maximize, double *partial_dev, void *stream)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(g && phi_full_dev && partial_dev, "NULL argument");
        OSCB_REQUIRE(g->is_dense && g->dense, "oscb_dense_shard_objective needs a dense (row shard) handle");
        OSCB_REQUIRE(R >= 1 && R <= 65536, "replicas must be in [1, 65536]");
        OSCB_REQUIRE(precision == OSCB_PREC_F32 || precision == OSCB_PREC_F64, "unknown precision %d", precision);
        OSCB_REQUIRE(n_states >= 2 && n_states <= 255, "n_states must be in [2, 255]");
        bind_device(g);
        cudaStream_t s = stream ? (cudaStream_t)stream : g->stream;
        if (precision == OSCB_PREC_F64) shard_pairs_impl<double>(g, (int)R, precision, phi_full_dev, maximize ? 0 : 1, n_states, partial_dev, s);
        else shard_pairs_impl<float>(g, (int)R, precision, phi_full_dev, maximize ? 0 : 1, n_states, partial_dev, s);
        check_launch("oscb_dense_shard_objective");
        return OSCB_OK;
    });
}

int oscb_dense_shard_energy(oscb_graph *g, int64_t R, int32_t precision, const void *phi_full_dev, double *partial_dev,
                            void *stream)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(g && phi_full_dev && partial_dev, "NULL argument");
        OSCB_REQUIRE(g->is_dense && g->dense, "oscb_dense_shard_energy needs a dense (row shard) handle");
        OSCB_REQUIRE(R >= 1 && R <= 65536, "replicas must be in [1, 65536]");
        OSCB_REQUIRE(precision == OSCB_PREC_F32 || precision == OSCB_PREC_F64, "unknown precision %d", precision);
        bind_device(g);
        cudaStream_t s = stream ? (cudaStream_t)stream : g->stream;
        if (precision == OSCB_PREC_F64) shard_pairs_impl<double>(g, (int)R, precision, phi_full_dev, 2, 2, partial_dev, s);
        else shard_pairs_impl<float>(g, (int)R, precision, phi_full_dev, 2, 2, partial_dev, s);
        check_launch("oscb_dense_shard_energy");
        return OSCB_OK;
    });
}

int oscb_dense_fused_create(oscb_graph *shard, const oscb_run_params *p, int64_t R, int64_t pair_count, int32_t world,
                            int32_t rank, oscb_fused **out)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(shard && p && out, "NULL argument");
        *out = nullptr;
        OSCB_REQUIRE(shard->is_dense && shard->umma, "fused dense runs need integer couplings |J| <= 127 and 128-row aligned shards");
        OSCB_REQUIRE(p->kernel == OSCB_KERNEL_AUTO || p->kernel == OSCB_KERNEL_DENSE_TC, "fused dense runs use the tensor-core kernel");
        OSCB_REQUIRE(umma_applies(shard, p), "fused dense runs are N = 2 max-cut (integer couplings) or N-state colouring (unit couplings), device noise");
        OSCB_REQUIRE(p->precision == OSCB_PREC_F32 || p->precision == OSCB_PREC_F64, "unknown precision %d", p->precision);
        const int force = (p->variant == 8 || p->variant == 4) ? p->variant : 0;
        OSCB_REQUIRE(R >= 1 && R <= umma_max_replicas(p->n_states, umma_uses_fp4(*shard->umma, (int)R, p->n_states, force)), "fused dense runs take 1..%d replicas per session",
                     umma_max_replicas(p->n_states, umma_uses_fp4(*shard->umma, (int)R, p->n_states, force)));
        OSCB_REQUIRE(p->h > 0.0 && std::isfinite(p->h) && p->ks_period > 0.0, "bad h / ks_period");
        OSCB_REQUIRE(p->steps > 0 || (p->t_stop > 0.0 && std::isfinite(p->t_stop)), "t_stop must be finite and > 0");
        bind_device(shard);
        std::unique_ptr<oscb_fused> f(new oscb_fused());
        f->g = shard;
        f->params = *p;
        f->R = (int)R;
        f->world = world;
        f->rank = rank;
        f->rp = make_run_plan(shard, p);
        if (p->cadence == 0) f->rp.cadence = reference_cadence(shard->n, pair_count);
        OSCB_REQUIRE(f->rp.steps + p->first_step < (1ll << 28), "step index exceeds 2^28");
        f->sched = umma_schedule(p, f->rp);
        f->session.reset(new UmmaSession(shard, umma_spec(p, f->rp, f->sched, (int)R), world, rank));
        f->io.alloc((size_t)shard->n * R);
        *out = f.release();
        return OSCB_OK;
    });
}

int oscb_dense_fused_export(oscb_fused *f, void *mem)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(f && mem, "NULL argument");
        static_assert(sizeof(UmmaExchange) == OSCB_FUSED_MEM_BYTES, "oscb.h: OSCB_FUSED_MEM_BYTES out of date");
        f->session->export_mem(reinterpret_cast<UmmaExchange *>(mem));
        return OSCB_OK;
    });
}

int oscb_dense_fused_connect(oscb_fused *f, const void *all)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(f && all, "NULL argument");
        f->session->connect(reinterpret_cast<const UmmaExchange *>(all));
        return OSCB_OK;
    });
}

int oscb_dense_fused_prepare(oscb_fused *f, const uint64_t *seeds, const double *phi0)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(f && seeds, "NULL argument");
        bind_device(f->g);
        cudaStream_t s = f->g->stream;
        const int n = (int)f->g->n, R = f->R;
        if (phi0) f->io.upload(phi0, (size_t)n * R, s);
        else {
            DevBuf<uint64_t> d_seeds(R);
            d_seeds.upload(seeds, R, s);
            k_initial_phases<<<blocks_for((long long)((n + 3) / 4) * R, 128), 128, 0, s>>>(d_seeds.p, f->io.p, n, R);
            OSCB_CUDA(cudaStreamSynchronize(s));
        }
        f->session->prepare(seeds, f->io.p);
        return OSCB_OK;
    });
}

int oscb_dense_fused_launch(oscb_fused *f)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(f, "NULL argument");
        f->session->launch();
        check_launch("oscb_dense_fused_launch");
        return OSCB_OK;
    });
}

int oscb_dense_fused_finish(oscb_fused *f, oscb_run_outputs *out)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(f && out, "NULL argument");
        const RunPlan &rp = f->rp;
        const oscb_run_params *p = &f->params;
        OSCB_REQUIRE((!out->energy && !out->best_trace && !out->trace_t && !out->trace_ks) || out->max_samples >= rp.n_samples,
                     "trace buffers too small: need %lld samples, have %lld", (long long)rp.n_samples, (long long)out->max_samples);
        const int R = f->R;
        const long long E = (long long)f->sched.event_step.size(), S = rp.n_samples;
        std::vector<long long> ev((size_t)E * R);
        std::vector<double> en((size_t)S * R);
        f->session->finish(out->final_phases, out->best_states, ev.data(), en.data());
        out->n_samples = S;
        out->steps_executed = rp.steps;
        out->nonfinite[0] = out->nonfinite[1] = out->nonfinite[2] = -1;
        for (int64_t k = 0; k < S; ++k) {
            const double t = k == 0 ? (double)p->first_step * p->h : (double)(p->first_step + rp.sample_steps[k - 1] + 1) * p->h;
            if (out->trace_t) out->trace_t[k] = t;
            if (out->trace_ks) out->trace_ks[k] = ks_value(p->ks_max, p->ks_period, t);
        }
        umma_bookkeeping(p, f->sched, ev.data(), en.data(), R, 0, out);
        out->device_ms = f->session->ms;
        out->kernel_launches = 1;
        out->kernel_used = OSCB_KERNEL_DENSE_TC;
        out->replicas_per_cta = R;
        out->smem_bytes = (int64_t)f->session->smem;
        umma_raise_nonfinite(f->session->nonfinite, out);
        return OSCB_OK;
    });
}

int oscb_dense_fused_grid(const oscb_fused *f, int32_t *ctas, int32_t *splits)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(f && ctas && splits, "NULL argument");
        *ctas = f->session->grid;
        *splits = f->session->splits;
        return OSCB_OK;
    });
}

int oscb_dense_fused_rows(const oscb_fused *f, int64_t *rows)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(f && rows, "NULL argument");
        *rows = f->session->rows();
        return OSCB_OK;
    });
}

int oscb_dense_tc_stream(const oscb_graph *g, int32_t n_states, int64_t R, int32_t *coupling_bits, int32_t *replicas_per_launch)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(g && coupling_bits && replicas_per_launch, "NULL argument");
        OSCB_REQUIRE(g->umma != nullptr, "the handle has no tensor-core plan (dense integer couplings only)");
        OSCB_REQUIRE(n_states >= 2 && n_states <= 16 && R >= 1, "n_states in 2..16 and R >= 1");
        const bool fp4 = umma_uses_fp4(*g->umma, (int)std::min<int64_t>(R, 1 << 20), n_states);
        *coupling_bits = fp4 ? 4 : 8;
        *replicas_per_launch = umma_max_replicas(n_states, fp4);
        return OSCB_OK;
    });
}

int oscb_dense_fused_destroy(oscb_fused *f)
{
    if (!f) return OSCB_OK;
    return guarded([&]() -> int {
        bind_device(f->g);
        delete f;
        return OSCB_OK;
    });
}

int oscb_graph_nonfinite(oscb_graph *g, int64_t where[3], int32_t reset)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(g && where, "NULL argument");
        bind_device(g);
        OSCB_CUDA(cudaDeviceSynchronize());
        unsigned long long flag = ~0ull;
        OSCB_CUDA(cudaMemcpy(&flag, g->d_nonfinite.p, sizeof(flag), cudaMemcpyDeviceToHost));
        where[0] = where[1] = where[2] = -1;
        if (flag != ~0ull) decode_nonfinite(flag, where);
        if (reset) {
            const unsigned long long none = ~0ull;
            OSCB_CUDA(cudaMemcpy(g->d_nonfinite.p, &none, sizeof(none), cudaMemcpyHostToDevice));
        }
        return OSCB_OK;
    });
}

int oscb_selftest_sign_state(int device, uint64_t *mismatches)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(mismatches != nullptr, "NULL argument");
        int count = 0;
        cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0) {
            set_error("no usable CUDA device (%s); liboscb has no CPU fallback", cudaGetErrorString(e));
            return OSCB_ECUDA;
        }
        OSCB_REQUIRE(device >= 0 && device < count, "device %d out of range (have %d)", device, count);
        OSCB_CUDA(cudaSetDevice(device));
        DevBuf<unsigned long long> d(1);
        OSCB_CUDA(cudaMemset(d.p, 0, sizeof(unsigned long long)));
        k_selftest_sign_state<<<148 * 8, 256>>>(d.p);
        check_launch("oscb_selftest_sign_state");
        // and the float32 decision boundaries of the N-state threshold (N = 3..8) against the float64 rule
        for (int N = 3; N <= 8; ++N) {
            FastArgs fa;
            memset(&fa, 0, sizeof(fa));
            fa.n_bnd = N;
            fast_state_boundaries(N, fa.bnd);
            k_selftest_boundaries<<<148 * 8, 256>>>(N, fa, d.p);
            check_launch("oscb_selftest_sign_state(boundaries)");
        }
        unsigned long long h = 0;
        OSCB_CUDA(cudaMemcpy(&h, d.p, sizeof(h), cudaMemcpyDeviceToHost));
        *mismatches = h;
        return OSCB_OK;
    });
}

int oscb_resident_plan_host(int64_t n, const int64_t *indptr, const int64_t *indices, int32_t replicas_per_cta,
                            int32_t replicas_per_lane, int32_t max_threads, int32_t pair_bytes, int32_t keep_order, int32_t *warps,
                            int32_t *rounds, int64_t *group_rows, int64_t *bank_conflicts, int32_t *warp_start,
                            uint16_t *rows, uint32_t *ginfo, uint16_t *ids)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(n >= 1 && indptr && warps && rounds && group_rows, "bad argument");
        const int RT = replicas_per_cta;
        OSCB_REQUIRE(RT >= 1 && RT <= 32 && (RT & (RT - 1)) == 0, "replicas_per_cta must be a power of two <= 32");
        OSCB_REQUIRE(max_threads >= 32 && max_threads <= 1024 && max_threads % 32 == 0, "bad max_threads");
        OSCB_REQUIRE((replicas_per_lane == 1 || replicas_per_lane == 2) && replicas_per_lane <= RT, "replicas_per_lane must be 1 or 2 (<= replicas_per_cta)");
        const int LPS = RT / replicas_per_lane;
        OSCB_REQUIRE(pair_bytes == 8 || pair_bytes == 16, "pair_bytes must be 8 or 16");
        const int64_t nnz = indptr[n];
        std::vector<int> ip(n + 1), ix(nnz);
        for (int64_t i = 0; i <= n; ++i) ip[i] = (int)indptr[i];
        for (int64_t e = 0; e < nnz; ++e) ix[e] = (int)indices[e];
        int W, T;
        tile_shape(n, LPS, max_threads, &W, &T);
        ResidentStreamHost h;
        compile_resident_stream((int)n, ip.data(), ix.data(), nullptr, RT, LPS, W, T, pair_bytes, keep_order != 0, &h);
        *warps = W;
        *rounds = T;
        *group_rows = h.n_group_rows;
        if (bank_conflicts) *bank_conflicts = h.conflicts;
        if (ids) {
            OSCB_REQUIRE(warp_start && rows && ginfo, "NULL output");
            std::copy(h.warp_start.begin(), h.warp_start.end(), warp_start);
            std::copy(h.rows.begin(), h.rows.end(), rows);
            std::copy(h.ginfo.begin(), h.ginfo.end(), ginfo);
            for (size_t q = 0; q < h.stream.size(); ++q) {
                ids[4 * q + 0] = (uint16_t)(h.stream[q].x & 0xffffu);
                ids[4 * q + 1] = (uint16_t)(h.stream[q].x >> 16);
                ids[4 * q + 2] = (uint16_t)(h.stream[q].y & 0xffffu);
                ids[4 * q + 3] = (uint16_t)(h.stream[q].y >> 16);
            }
        }
        return OSCB_OK;
    });
}

int oscb_run(oscb_graph *g, const oscb_run_params *p, const uint64_t *seeds, int64_t R, const double *phi0,
             const double *noise, oscb_run_outputs *out)
{
    return guarded([&]() -> int {
        OSCB_REQUIRE(g && p && out, "NULL argument");
        OSCB_REQUIRE(R >= 1 && R <= 65536, "replicas must be in [1, 65536]");
        OSCB_REQUIRE(seeds != nullptr, "seeds is NULL");
        OSCB_REQUIRE(p->objective == OSCB_OBJ_MAXCUT || p->objective == OSCB_OBJ_COLORING, "unknown objective kind: %d", p->objective);
        OSCB_REQUIRE(p->n_states >= 2 && p->n_states <= 255, "n_states must be in [2, 255]");
        OSCB_REQUIRE(p->objective != OSCB_OBJ_MAXCUT || p->n_states == 2, "maxcut runs require n_states=2");
        OSCB_REQUIRE(p->precision == OSCB_PREC_F32 || p->precision == OSCB_PREC_F64, "unknown precision %d", p->precision);
        OSCB_REQUIRE(p->noise_mode >= OSCB_NOISE_DEVICE && p->noise_mode <= OSCB_NOISE_NONE, "unknown noise mode %d", p->noise_mode);
        OSCB_REQUIRE(p->noise_mode != OSCB_NOISE_HOST || noise != nullptr, "noise_mode HOST needs a noise array");
        OSCB_REQUIRE(std::isfinite(p->K) && std::isfinite(p->ks_max) && std::isfinite(p->kn), "non-finite parameter");
        OSCB_REQUIRE(p->h > 0.0 && std::isfinite(p->h), "h must be finite and > 0");
        OSCB_REQUIRE(p->ks_period > 0.0 && std::isfinite(p->ks_period), "ks_period must be finite and > 0");
        OSCB_REQUIRE(p->steps > 0 || (p->t_stop > 0.0 && std::isfinite(p->t_stop)), "t_stop must be finite and > 0");
        OSCB_REQUIRE(p->first_step >= 0, "first_step must be >= 0");
        OSCB_REQUIRE(g->row_begin == 0 && g->row_end == g->n, "oscb_run needs the whole graph; row shards use oscb_dense_*");
        bind_device(g);
        const RunPlan rp = make_run_plan(g, p);
        OSCB_REQUIRE(rp.steps + p->first_step < (1ll << 28), "step index exceeds 2^28");
        OSCB_REQUIRE((!out->energy && !out->best_trace && !out->trace_t && !out->trace_ks) || out->max_samples >= rp.n_samples,
                     "trace buffers too small: need %lld samples, have %lld", (long long)rp.n_samples, (long long)out->max_samples);
        out->n_samples = rp.n_samples;
        out->steps_executed = rp.steps;
        out->nonfinite[0] = out->nonfinite[1] = out->nonfinite[2] = -1;
        for (int64_t k = 0; k < rp.n_samples; ++k) {
            const double t = k == 0 ? (double)p->first_step * p->h
                                    : (double)(p->first_step + rp.sample_steps[k - 1] + 1) * p->h;
            if (out->trace_t) out->trace_t[k] = t;
            if (out->trace_ks) out->trace_ks[k] = ks_value(p->ks_max, p->ks_period, t);
        }

        int kernel = p->kernel;
        if (g->is_dense) {
            OSCB_REQUIRE(kernel != OSCB_KERNEL_RESIDENT, "dense couplings run on the streaming loop or the tensor-core kernel (no resident kernel)");
            OSCB_REQUIRE(kernel != OSCB_KERNEL_DENSE_TC || umma_applies(g, p),
                         "the tensor-core dense kernel needs integer couplings |J| <= 127, device noise, and N = 2 max-cut or N <= 16 colouring on unit couplings");
            if (umma_applies(g, p)) {
                run_umma(g, p, rp, seeds, R, phi0, out);
                return OSCB_OK;
            }
            kernel = OSCB_KERNEL_STREAM;
        }
        if (kernel == OSCB_KERNEL_CLUSTER)
            OSCB_REQUIRE(cluster_applies(g, p, R, true),
                         "the cluster kernel takes float32, device noise, N = 2 max-cut, 64 <= n <= 65535 and unit or small integer couplings");
        if ((kernel == OSCB_KERNEL_AUTO && cluster_applies(g, p, R, false)) || kernel == OSCB_KERNEL_CLUSTER) {
            run_cluster(g, p, rp.steps, rp.cadence, rp.sample_steps, seeds, R, phi0, out);
            return OSCB_OK;
        }
        if (kernel == OSCB_KERNEL_LOWDEG)
            OSCB_REQUIRE(lowdeg_applies(g, p, R, true),
                         "the low-degree kernel takes float32, device noise, max degree <= 16, n up to ~28000 and N = 2 max-cut on "
                         "integer couplings or N = 3 colouring on unit couplings");
        if ((kernel == OSCB_KERNEL_AUTO && lowdeg_applies(g, p, R, false)) || kernel == OSCB_KERNEL_LOWDEG) {
            run_lowdeg(g, p, rp.steps, rp.cadence, rp.sample_steps, seeds, R, phi0, out);
            return OSCB_OK;
        }
        if (kernel == OSCB_KERNEL_AUTO)
            kernel = resident_fits(g, p, R) ? OSCB_KERNEL_RESIDENT : OSCB_KERNEL_STREAM;
        if (kernel == OSCB_KERNEL_RESIDENT) {
            run_resident(g, p, rp.steps, rp.cadence, rp.sample_steps, seeds, R, phi0, noise, out);
            return OSCB_OK;
        }
        OSCB_REQUIRE(kernel == OSCB_KERNEL_STREAM, "unknown kernel selector %d", kernel);
        if (p->precision == OSCB_PREC_F64) run_stream<double, true>(g, p, rp, seeds, R, phi0, noise, out);
        else run_stream<float, false>(g, p, rp, seeds, R, phi0, noise, out);
        return OSCB_OK;
    });
}

} // extern "C"
