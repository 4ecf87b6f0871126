// oscb_lowdeg.cu -- translation unit of the low-degree persistent kernel: k_lowdeg (oscb_lowdeg.cuh) and its
// host side (oscb_lowdeg_host.hpp), plus the C-ABI test hook that exposes the stream compiler to CPU tests.
#include "oscb_lowdeg_host.hpp"

static int lowdeg_plan_host(const char *who, int rpl, int64_t n, const int64_t *indptr, const int64_t *indices, const double *weights,
                            int32_t replicas_per_cta, int32_t warps, int32_t items_per_thread, int32_t *uniform,
                            int64_t *group_rows, int64_t *entries, uint32_t *quad_of, uint32_t *slot_of,
                            uint32_t *offsets, float *couplings, int32_t *warp_start)
{
    using namespace oscb;
    try {
        OSCB_REQUIRE(n >= 4 && indptr && indices, "bad graph");
        std::vector<int> ip(n + 1), ix(indptr[n]);
        for (int64_t i = 0; i <= n; ++i) ip[i] = (int)indptr[i];
        for (int64_t e = 0; e < indptr[n]; ++e) ix[e] = (int)indices[e];
        int maxdeg = 0;
        for (int64_t i = 0; i < n; ++i) maxdeg = std::max(maxdeg, ip[i + 1] - ip[i]);
        LowdegShape s;
        s.RT = replicas_per_cta;
        s.LRT = 0;
        while ((1 << s.LRT) < s.RT) ++s.LRT;
        OSCB_REQUIRE((1 << s.LRT) == s.RT && s.RT <= 32 && s.RT >= rpl, "replicas_per_cta must be a power of two <= 32");
        s.rpl = rpl;
        s.C = 32 * rpl / s.RT; s.W = warps; s.QPT = items_per_thread; s.Q = (int)((n + 3) / 4); s.Qp = s.W * s.QPT * s.C;
        s.uniform = maxdeg <= 4;
        LowdegStreamHost h;
        compile_lowdeg_stream((int)n, ip.data(), ix.data(), weights, s, true, &h);
        if (uniform) *uniform = s.uniform ? 1 : 0;
        if (group_rows) *group_rows = h.group_rows;
        if (entries) *entries = (int64_t)(h.off.size() / 4);
        if (quad_of) std::copy(h.quad_of.begin(), h.quad_of.end(), quad_of);
        if (slot_of) std::copy(h.slot_of.begin(), h.slot_of.end(), slot_of);
        if (offsets) std::copy(h.off.begin(), h.off.end(), offsets);
        if (couplings) std::copy(h.wt.begin(), h.wt.end(), couplings);
        if (warp_start) std::copy(h.warp_start.begin(), h.warp_start.end(), warp_start);
        return OSCB_OK;
    } catch (const OscbFail &f) {
        return f.code;
    } catch (const std::exception &e) {
        set_error("%s: %s", who, e.what());
        return OSCB_ECUDA;
    }
}

extern "C" int oscb_lowdeg_plan_host(int64_t n, const int64_t *indptr, const int64_t *indices, const double *weights,
                                     int32_t replicas_per_cta, int32_t warps, int32_t items_per_thread, int32_t *uniform,
                                     int64_t *group_rows, int64_t *entries, uint32_t *quad_of, uint32_t *slot_of,
                                     uint32_t *offsets, float *couplings, int32_t *warp_start)
{
    return lowdeg_plan_host("oscb_lowdeg_plan_host", 1, n, indptr, indices, weights, replicas_per_cta, warps, items_per_thread, uniform,
                            group_rows, entries, quad_of, slot_of, offsets, couplings, warp_start);
}

extern "C" int oscb_lowdeg_pair_plan_host(int64_t n, const int64_t *indptr, const int64_t *indices, const double *weights,
                                          int32_t replicas_per_cta, int32_t warps, int32_t items_per_thread, int32_t *uniform,
                                          int64_t *group_rows, int64_t *entries, uint32_t *quad_of, uint32_t *slot_of,
                                          uint32_t *offsets, float *couplings, int32_t *warp_start)
{
    return lowdeg_plan_host("oscb_lowdeg_pair_plan_host", 2, n, indptr, indices, weights, replicas_per_cta, warps, items_per_thread, uniform,
                            group_rows, entries, quad_of, slot_of, offsets, couplings, warp_start);
}
