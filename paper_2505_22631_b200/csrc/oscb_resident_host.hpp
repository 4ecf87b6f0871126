// oscb_resident_host.hpp -- host side of the persistent shared-memory kernel (stub until built).
#pragma once
#include "oscb_host.hpp"

namespace oscb {

struct ResidentPlan {
    int dummy = 0;
};

static bool resident_fits(const oscb_graph *, const oscb_run_params *, int64_t) { return false; }

static void run_resident(oscb_graph *, const oscb_run_params *, int64_t, int64_t, const std::vector<long long> &,
                         const uint64_t *, int64_t, const double *, const double *, oscb_run_outputs *)
{
    set_error("resident kernel not built");
    throw OscbFail{OSCB_ECUDA};
}

} // namespace oscb
