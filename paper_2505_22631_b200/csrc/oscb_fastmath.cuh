// oscb_fastmath.cuh -- float32 building blocks shared by the persistent throughput kernels (k_resident_fast,
// k_lowdeg, k_cluster_fast): MUFU Box-Muller, the MUFU trig with the N = 2 lattice state in the cosine's sign bit, and
// the reference threshold rule as a table of float32 decision boundaries.
#pragma once
#include "oscb_device.cuh"
#include <string.h>

namespace oscb {

// four standard normals from one Philox block, MUFU Box-Muller (same draw -> same normal as
// normals4(float) up to ~1e-6)
__device__ __forceinline__ void normals4_fast(uint4 x, float &z0, float &z1, float &z2, float &z3)
{
    const float inv32 = 2.3283064365386963e-10f;
    const float u0 = fminf(fmaf((float)x.x, inv32, 0.5f * inv32), 1.0f);
    const float u1 = fminf(fmaf((float)x.z, inv32, 0.5f * inv32), 1.0f);
    float r0, r1;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(-1.3862943611198906f * __log2f(u0)));
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(-1.3862943611198906f * __log2f(u1)));
    // angle 2 pi v, v in [-1/2, 1/2): the draw taken as a SIGNED 32-bit integer lands in [-pi, pi), where the MUFU
    // approximations are tightest, without a fold
    const float a0 = (float)(int)x.y * 1.4629180792671596e-9f, a1 = (float)(int)x.w * 1.4629180792671596e-9f;   // 2 pi 2^-32
    z0 = r0 * __cosf(a0); z1 = r0 * __sinf(a0);
    z2 = r1 * __cosf(a1); z3 = r1 * __sinf(a1);
}

// (sin, cos) of 2 pi y for a phase y in [0, 1), in ~11 instructions instead of sincospif's ~32: u = y - rint(y) is
// exact and lies in [-1/2, 1/2], so the angle 2 pi u is inside [-pi, pi], the interval on which the MUFU sine and
// cosine are specified (abs. error 2^-21.4 and 2^-21.2, ~4e-7: about the rounding of float32 near 1).  (Round 1 reduced
// to a quarter turn first and fixed the quadrant up afterwards: ~20 instructions for the same error bound.)
// The SIGN BIT of the cosine is then set from the exact comparison 0.25 < y < 0.75, written as |y - 1/2| < 1/4
// (y - 1/2 is exact on [1/4, 1) and can only round towards -1/4 below it), i.e. it IS the N = 2 lattice state of
// the reference (dynamics.py:203-213; ties at 0.25 / 0.75 -> state 0), also when the approximate magnitude
// underflows to zero: -0 carries state 1.  Consumers read the state from the bit, never from "c < 0".
// oscb_selftest_sign_state checks bit and values over every float32 in [0, 1).
__device__ __forceinline__ void trig_turns_direct(float y, float &s, float &c)
{
    const float a = 6.283185307179586f * (y - (y > 0.5f ? 1.0f : 0.0f));      // y - rint(y), on the ALU
    s = __sinf(a);
    const uint32_t state = fabsf(y - 0.5f) < 0.25f ? 0x80000000u : 0u;
    c = __uint_as_float((__float_as_uint(__cosf(a)) & 0x7FFFFFFFu) | state);
}

// Lattice state of a float32 phase for any N (dynamics.py:203-213): the reference rule is a step
// function of the phase, so it is evaluated as "how many decision boundaries lie at or below p";
// the boundaries are found on the host by bisection over float32 with the reference's own float64
// expression (fast_state_boundaries), and oscb_selftest_sign_state checks the table against the
// float64 rule for every float32 in [0, 1).
__device__ __forceinline__ uint32_t state_from_boundaries(float p, const float *bnd, int n)
{
    if (n == 3) {      // the 3-colouring case, without the loop
        const uint32_t st3 = (p >= bnd[0] ? 1u : 0u) + (p >= bnd[1] ? 1u : 0u) + (p >= bnd[2] ? 1u : 0u);
        return st3 == 3u ? 0u : st3;
    }
    uint32_t st = 0;
    for (int k = 0; k < n; ++k) st += (p >= bnd[k]) ? 1u : 0u;
    return st == (uint32_t)n ? 0u : st;
}

// Decision boundaries of the reference threshold rule on float32 phases: bnd[k] = the smallest
// float32 in [k/N, (k+1)/N] whose state is (k + 1) % N.  Inside that interval the state is k below
// the boundary and (k + 1) % N from it on (both distances are monotone in p), so a
// bisection over the float32 bit patterns with the float64 rule itself finds it exactly.
inline void fast_state_boundaries(int n_states, float *bnd)
{
    for (int k = 0; k < n_states; ++k) {
        uint32_t lo, hi;                 // state(lo) == k, state(hi) == (k + 1) % N
        float flo = (float)((double)k / n_states), fhi = k + 1 == n_states ? 0.99999994f : (float)((double)(k + 1) / n_states);
        memcpy(&lo, &flo, 4);
        memcpy(&hi, &fhi, 4);
        const int next = (k + 1) % n_states;
        // make sure the bracket ends are on the right sides (float rounding of k/N can land either way)
        auto st = [&](uint32_t bits) { float f; memcpy(&f, &bits, 4); return threshold_state((double)f, n_states); };
        while (st(lo) != k) --lo;
        while (st(hi) != next) hi = hi + 1 < 0x3F800000u ? hi + 1 : hi - 2;   // (the last interval ends below 1.0)
        while (hi - lo > 1) {
            const uint32_t mid = lo + (hi - lo) / 2;
            if (st(mid) == k) lo = mid; else hi = mid;
        }
        memcpy(&bnd[k], &hi, 4);
    }
}

} // namespace oscb
