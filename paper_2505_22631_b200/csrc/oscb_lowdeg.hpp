// oscb_lowdeg.hpp -- host interface of the low-degree persistent kernel (oscb_lowdeg.cu), shared with the
// C ABI translation unit (oscb.cu).
#pragma once
#include "oscb_host.hpp"
#include <vector>

namespace oscb {

// float32, device noise, max degree <= 16 (mean <= 8 unless `forced`), and N = 2 max-cut on integer couplings
// or N = 3 colouring on unit couplings
bool lowdeg_applies(oscb_graph *g, const oscb_run_params *p, int64_t R, bool forced);

// the whole run in one persistent launch (same contract as run_resident)
void run_lowdeg(oscb_graph *g, const oscb_run_params *p, int64_t steps, int64_t cadence,
                const std::vector<long long> &sample_steps, const uint64_t *seeds, int64_t R, const double *phi0,
                oscb_run_outputs *out);

} // namespace oscb
