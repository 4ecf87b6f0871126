// oscb_dense_host.hpp -- host side of the dense path: upload of a row shard of J and the
// launch helpers the generic entry points (oscb_step / oscb_score / oscb_energy / oscb_run)
// and the sharded driver (oscb_dense_shard_*) share.
#pragma once
#include "oscb_host.hpp"
#include "oscb_dense.cuh"
#include <cmath>

namespace oscb {

enum DenseKind { DENSE_I8 = 0, DENSE_F = 1 };

struct DensePlan {
    int kind = DENSE_F;
    int n_pad = 0;
    double max_abs_rowsum = 0.0; // max_i sum_j |J_ij| over the handle's rows
    bool tc_exact = false;       // int32 accumulation of the int8 digit-plane GEMM cannot overflow
    bool fp4_ok = false;         // every coupling of the shard's rows is in {0, +-1, +-2, +-3, +-4, +-6} (e2m1 values)
    DevBuf<int8_t> J8;
    DevBuf<float> J32;
    DevBuf<double> J64;
};

// J: rows [row_begin, row_end) of the full symmetric matrix, row-major, n columns each.
static void build_dense(oscb_graph *g, const double *J)
{
    const int64_t n = g->n, rows = g->row_end - g->row_begin;
    const int n_pad = (int)((n + 3) / 4 * 4);
    bool unit = true, integral = true, small = true, fp4 = true;
    int64_t nnz = 0, pairs = 0, maxdeg = 0;
    double max_abs_rowsum = 0.0;
    for (int64_t q = 0; q < rows; ++q) {
        const int64_t i = g->row_begin + q;
        int64_t d = 0;
        double abs_row = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            const double v = J[q * n + j];
            OSCB_REQUIRE(std::isfinite(v), "non-finite coupling at (%lld, %lld)", (long long)i, (long long)j);
            OSCB_REQUIRE(i != j || v == 0.0, "coupling diagonal must be zero");
            { const double m = std::fabs(v); if (!(m == 0.0 || m == 1.0 || m == 2.0 || m == 3.0 || m == 4.0 || m == 6.0)) fp4 = false; }
            abs_row += std::fabs(v);
            if (v != 0.0) {
                ++d;
                if (j > i) ++pairs;
                if (v != 1.0) unit = false;
                if (v != std::nearbyint(v)) integral = false;
                if (std::fabs(v) > 127.0) small = false;
            }
        }
        nnz += d;
        maxdeg = std::max(maxdeg, d);
        max_abs_rowsum = std::max(max_abs_rowsum, abs_row);
    }
    g->nnz = nnz;
    g->pairs = pairs;
    g->max_degree = maxdeg;
    g->unit_weights = unit;
    g->int_weights = integral;
    auto plan = std::make_shared<DensePlan>();
    plan->n_pad = n_pad;
    // The tensor-core kernel's sums are EXACT integers only while the accumulators hold them: the int8 stream adds
    // products |J * digit| <= 128 |J| into int32, the e2m1 stream products <= 4 |J| into float32 (exact below 2^24).
    // A row whose |J| sum breaks the bound keeps the graph off that stream (n < ~131k at |J| = 127, n < ~1M at |J| = 1
    // for int8; n < ~4.2M at |J| = 1 for e2m1) and the run falls back to the SIMT dense path.
    plan->max_abs_rowsum = max_abs_rowsum;
    plan->tc_exact = max_abs_rowsum * 128.0 < 2147483648.0;
    plan->fp4_ok = fp4 && max_abs_rowsum * 4.0 < 16777216.0;
    cudaStream_t s = g->stream;
    const size_t elems = (size_t)rows * n_pad;
    if (integral && small) {
        plan->kind = DENSE_I8;
        std::vector<int8_t> h(elems, 0);
        for (int64_t q = 0; q < rows; ++q)
            for (int64_t j = 0; j < n; ++j) h[(size_t)q * n_pad + j] = (int8_t)J[q * n + j];
        plan->J8.alloc(elems);
        plan->J8.upload(h.data(), elems, s);
        OSCB_CUDA(cudaStreamSynchronize(s));
    } else {
        plan->kind = DENSE_F;
        std::vector<double> h64(elems, 0.0);
        std::vector<float> h32(elems, 0.f);
        for (int64_t q = 0; q < rows; ++q)
            for (int64_t j = 0; j < n; ++j) {
                h64[(size_t)q * n_pad + j] = J[q * n + j];
                h32[(size_t)q * n_pad + j] = (float)J[q * n + j];
            }
        plan->J64.alloc(elems);
        plan->J64.upload(h64.data(), elems, s);
        plan->J32.alloc(elems);
        plan->J32.upload(h32.data(), elems, s);
        OSCB_CUDA(cudaStreamSynchronize(s));
    }
    g->dense = plan;
}

// One dense Euler step of the handle's rows on stream `s`.
template <typename T>
static void launch_dense_step(const oscb_graph *g, cudaStream_t s, int R, const T *phi_in,
                              const typename Vec2<T>::type *cs_in, T *phi_out, typename Vec2<T>::type *cs_out,
                              const uint64_t *d_seeds, const double *d_noise, const StepScalars &sc)
{
    const DensePlan &pl = *g->dense;
    DenseStepArgs a;
    a.n = (int)g->n; a.n_pad = pl.n_pad; a.row_begin = (int)g->row_begin; a.rows = (int)(g->row_end - g->row_begin);
    a.R = R; a.sc = sc;
    const unsigned bx = (unsigned)((a.rows + 7) / 8);
    auto go = [&](auto jptr) {
        using JT = std::remove_cv_t<std::remove_pointer_t<decltype(jptr)>>;
        if (R == 1) k_dense_step<T, JT, 1><<<dim3(bx, 1), 256, 0, s>>>(a, jptr, phi_in, cs_in, phi_out, cs_out, d_seeds, d_noise, g->d_nonfinite.p);
        else k_dense_step<T, JT, 8><<<dim3(bx, (unsigned)((R + 7) / 8)), 256, 0, s>>>(a, jptr, phi_in, cs_in, phi_out, cs_out, d_seeds, d_noise, g->d_nonfinite.p);
    };
    if (pl.kind == DENSE_I8) go((const int8_t *)pl.J8.p);
    else if (sizeof(T) == 8) go((const double *)pl.J64.p);
    else go((const float *)pl.J32.p);
}

// Row partials of the objective (mode 0 cut / 1 conflicts) or the energy (mode 2) into `partial`
// [rows][R], then their in-order sum into out[r * out_stride].
template <typename T>
static void launch_dense_pairs(const oscb_graph *g, cudaStream_t s, int R, int mode, const uint8_t *states,
                               const typename Vec2<T>::type *cs, double *partial, double *out, long long out_stride)
{
    const DensePlan &pl = *g->dense;
    const int n = (int)g->n, rb = (int)g->row_begin, rows = (int)(g->row_end - g->row_begin);
    const dim3 grid((unsigned)((rows + 7) / 8), (unsigned)R);
    auto go = [&](auto jptr) {
        using JT = std::remove_cv_t<std::remove_pointer_t<decltype(jptr)>>;
        if (mode == 0) k_dense_pairs<T, JT, 0><<<grid, 256, 0, s>>>(n, pl.n_pad, rb, rows, R, jptr, states, cs, partial);
        else if (mode == 1) k_dense_pairs<T, JT, 1><<<grid, 256, 0, s>>>(n, pl.n_pad, rb, rows, R, jptr, states, cs, partial);
        else k_dense_pairs<T, JT, 2><<<grid, 256, 0, s>>>(n, pl.n_pad, rb, rows, R, jptr, states, cs, partial);
    };
    if (pl.kind == DENSE_I8) go((const int8_t *)pl.J8.p);
    else if (sizeof(T) == 8) go((const double *)pl.J64.p);
    else go((const float *)pl.J32.p);
    k_dense_reduce<<<(unsigned)((R + 127) / 128), 128, 0, s>>>(partial, rows, R, out, out_stride);
}

} // namespace oscb
