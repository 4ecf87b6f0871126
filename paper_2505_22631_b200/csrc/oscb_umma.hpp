// oscb_umma.hpp -- host interface of the tensor-core dense integrator (oscb_umma.cu), shared
// with the C ABI translation unit (oscb.cu).
#pragma once
#include "oscb_host.hpp"

namespace oscb {

// per dense int8 handle: the swizzled tile images of the handle's rows of J and their row sums
struct UmmaPlan {
    int n = 0, tiles = 0, tile_begin = 0, tile_end = 0;
    DevBuf<uint8_t> A_img;
    DevBuf<int> W;
};

// rows [row_begin, row_end) of J as int8 [rows][n_pad] on the device -> plan (row_begin % 128 == 0;
// row_end % 128 == 0 or row_end == n)
std::shared_ptr<UmmaPlan> umma_build_plan(const int8_t *J8_dev, int64_t n, int n_pad, int64_t row_begin, int64_t row_end,
                                          cudaStream_t s);

constexpr int kUmmaMaxReplicas = 28;

// One run of up to kUmmaMaxReplicas replicas on ONE GPU holding the whole graph.
struct UmmaSpec {
    int R = 1;
    int precision = OSCB_PREC_F32;
    int noise_on = 1;
    double K = 0, h = 0, kn_sqrt_h = 0, ks_max = 0, ks_period = 1;
    long long steps = 0, first_step = 0;
    const uint8_t *flags = nullptr;     // host [steps + 1]: bit 0 score the pass's input phases, bit 1 + energy sample
    long long n_events = 0, n_samples = 0;
    const uint64_t *seeds = nullptr;    // host [R]
    const double *d_phi0 = nullptr;     // device [R][n] float64, host layout
    double *d_final = nullptr;          // device [R][n] float64 (may be null)
    uint8_t *h_best_states = nullptr;   // host [R][n] (may be null)
    long long *h_events = nullptr;      // host [n_events][R]: 2 * cut of every scored pass
    double *h_energy = nullptr;         // host [n_samples][R]
    // filled by the run
    float ms = 0.f;
    int grid = 0, stages = 0;
    size_t smem = 0;
    unsigned long long nonfinite = ~0ull;
};

void umma_run(oscb_graph *g, const UmmaPlan &plan, UmmaSpec &spec);

} // namespace oscb
