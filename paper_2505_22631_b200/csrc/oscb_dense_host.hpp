// oscb_dense_host.hpp -- dense all-to-all couplings (north_star subsystem 2, dense branch).
#pragma once
#include "oscb_host.hpp"
#include <cmath>

namespace oscb {

struct DensePlan {
    int dummy = 0;
};

static void finish_csr(oscb_graph *g);

// J: rows [row_begin, row_end) of the full symmetric matrix, row-major, n columns each.
// Round-1 first cut: the couplings are compacted to the canonical CSR so every entry point works
// on dense inputs through the sparse kernels; the dedicated dense kernel replaces this.
static void build_dense(oscb_graph *g, const double *J)
{
    const int64_t n = g->n;
    OSCB_REQUIRE(g->row_begin == 0 && g->row_end == n, "row-sharded dense graphs need the dense kernel (not built yet)");
    g->h_indptr.assign(n + 1, 0);
    g->h_indices.clear();
    g->h_w.clear();
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j < n; ++j) {
            const double v = J[i * n + j];
            OSCB_REQUIRE(std::isfinite(v), "non-finite coupling at (%lld, %lld)", (long long)i, (long long)j);
            OSCB_REQUIRE(i != j || v == 0.0, "coupling diagonal must be zero");
            if (v != 0.0) {
                g->h_indices.push_back((int)j);
                g->h_w.push_back(v);
            }
        }
        OSCB_REQUIRE(g->h_indices.size() < (size_t)1 << 31, "too many couplings");
        g->h_indptr[i + 1] = (int)g->h_indices.size();
    }
    g->nnz = (int64_t)g->h_indices.size();
    finish_csr(g);
}

static void dense_step(oscb_graph *, int64_t, const double *, const double *, double, double, double, double,
                       int, int, double *, int64_t *)
{
    set_error("dense kernel not built");
    throw OscbFail{OSCB_ECUDA};
}

static void run_dense(oscb_graph *, const oscb_run_params *, int64_t, int64_t, const std::vector<long long> &,
                      const uint64_t *, int64_t, const double *, const double *, oscb_run_outputs *)
{
    set_error("dense kernel not built");
    throw OscbFail{OSCB_ECUDA};
}

} // namespace oscb
