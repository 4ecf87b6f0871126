// oscb_device.cuh -- device-side building blocks shared by every kernel of the OIM/OPM
// integrator: arithmetic traits for the two precisions, the Philox generators, the SHIL /
// trig helpers and the reference read-out (threshold) rule.
//
// Reference behaviour restated here (paths relative to /root/reference/pkg/src/oscim/):
//   trig precompute     dynamics.py:393-395   sin(2pi phi), cos(2pi phi), sin((2pi N) phi)
//   row update          dynamics.py:166-172   acc += w (s_i c_j - c_i s_j);  x = phi + h (K acc - ks shil) + kn sqrt(h) xi
//   wrap                dynamics.py:172       x - floor(x)
//   threshold           dynamics.py:203-213   nearest k/N, circular distance, ties -> smaller k
//   schedule            dynamics.py:83-88     triangular Ks(t)
//   initial phases      dynamics.py:127-129   numpy Philox4x64-10, counter 1<<192
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

namespace oscb {

#define OSCB_TWO_PI 6.283185307179586476925286766559

// ------------------------------------------------------------------------------------------
// precision traits
template <typename T> struct Vec2;
template <> struct Vec2<float> { using type = float2; };
template <> struct Vec2<double> { using type = double2; };

// ------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11): the device noise source.  The draw for
// (seed, step, oscillator i) is component (i & 3) of the block at counter
// (i >> 2, step_lo, step_hi, 'oscb'), key (seed_lo, seed_hi) -- a pure function of the triple,
// which is the contract the reference documents for its own stream (dynamics.py:97-105).
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k)
{
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ uint4 noise_block(uint64_t seed, uint64_t step, uint32_t quad)
{
    return philox4x32_10(make_uint4(quad, (uint32_t)step, (uint32_t)(step >> 32), 0x6F736362u),
                         make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

// four standard normals from one Philox block (Box-Muller on two uniform pairs)
__device__ __forceinline__ void normals4(uint4 x, float z[4])
{
    const float inv32 = 2.3283064365386963e-10f; // 2^-32
    // u in (0,1]: (x + 1) * 2^-32 would overflow to 0 for x = 2^32-1, use fma on the float
    float u0 = fmaf((float)x.x, inv32, 0.5f * inv32);
    float u1 = fmaf((float)x.z, inv32, 0.5f * inv32);
    u0 = fminf(u0, 1.0f);
    u1 = fminf(u1, 1.0f);
    const float r0 = sqrtf(-1.3862943611198906f * __log2f(u0)); // -2 ln u = -2 ln2 log2 u
    const float r1 = sqrtf(-1.3862943611198906f * __log2f(u1));
    float s0, c0, s1, c1;
    sincospif((float)x.y * (2.0f * inv32), &s0, &c0);
    sincospif((float)x.w * (2.0f * inv32), &s1, &c1);
    z[0] = r0 * c0; z[1] = r0 * s0; z[2] = r1 * c1; z[3] = r1 * s1;
}

__device__ __forceinline__ void normals4(uint4 x, double z[4])
{
    const double inv32 = 2.3283064365386962890625e-10;
    const double u0 = ((double)x.x + 0.5) * inv32, u1 = ((double)x.z + 0.5) * inv32;
    const double r0 = sqrt(-2.0 * log(u0)), r1 = sqrt(-2.0 * log(u1));
    double s0, c0, s1, c1;
    sincospi((double)x.y * (2.0 * inv32), &s0, &c0);
    sincospi((double)x.w * (2.0 * inv32), &s1, &c1);
    z[0] = r0 * c0; z[1] = r0 * s0; z[2] = r1 * c1; z[3] = r1 * s1;
}

// ------------------------------------------------------------------------------------------
// Philox4x64-10 with numpy's conventions, for the exact replay of initial phases:
// phi0[i] = word (i & 3) of block(counter = (1<<192) + 1 + (i >> 2), key = [seed, 0]),
// mapped to a double as (u64 >> 11) * 2^-53.
__device__ __forceinline__ void philox4x64_10(uint64_t c0, uint64_t c1, uint64_t c2, uint64_t c3,
                                              uint64_t k0, uint64_t k1, uint64_t out[4])
{
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const uint64_t hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0), lo0 = 0xD2E7470EE14C6C93ull * c0;
        const uint64_t hi1 = __umul64hi(0xCA5A826395121157ull, c2), lo1 = 0xCA5A826395121157ull * c2;
        const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B97F4A7C15ull;
        k1 += 0xBB67AE8584CAA73Bull;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// ------------------------------------------------------------------------------------------
// trig of one phase.  Parity (fp64) mode evaluates exactly the reference's expressions --
// the rounded product 2*pi*phi fed to sin/cos, (2*pi*N)*phi for the SHIL harmonic.  The fp32
// mode uses sincospi on the phase in turns (exact range reduction) and the multiple-angle
// identities for N = 2, 3.
struct TrigConst {
    double two_pi_n; // (2*pi) * N, rounded once like the reference's (TWO_PI * n_states)
    int n_states;
};
__host__ __device__ inline TrigConst make_trig_const(int n_states)
{
    TrigConst tc;
    tc.two_pi_n = OSCB_TWO_PI * (double)n_states;
    tc.n_states = n_states;
    return tc;
}

__device__ __forceinline__ void phase_trig(double phi, double &s, double &c)
{
    const double a = __dmul_rn(OSCB_TWO_PI, phi);
    sincos(a, &s, &c);
}
__device__ __forceinline__ void phase_trig(float phi, float &s, float &c)
{
    sincospif(2.0f * phi, &s, &c);
}
__device__ __forceinline__ double shil_term(double phi, double, double, const TrigConst &tc)
{
    return sin(__dmul_rn(tc.two_pi_n, phi));
}
__device__ __forceinline__ float shil_term(float phi, float s, float c, const TrigConst &tc)
{
    if (tc.n_states == 2) return 2.0f * s * c;
    if (tc.n_states == 3) return s * (3.0f - 4.0f * s * s);
    return sinpif((float)(2 * tc.n_states) * phi);
}

// x - floor(x) with the [0,1) guarantee: a tiny negative x makes x - floor(x) round to 1.0,
// which is the same point of the circle as 0.0 but violates PhaseState's contract
// (model.py:273-274), so it is folded to 0.
template <typename T> __device__ __forceinline__ T wrap_unit(T x)
{
    T y = x - floor(x);
    return (y >= T(1)) ? T(0) : y;
}

// dynamics.py:203-213 evaluated in fp64 on the value the phase holds, so the rounding is the
// reference's bit for bit for any phase representable in the kernel's precision.
__host__ __device__ __forceinline__ int threshold_state(double p, int n_states)
{
    // N = 2: d0 = min(p, 1-p), d1 = |p - 0.5|, both differences exact where the comparison is
    // close (Sterbenz), so "d1 < d0" is exactly 0.25 < p < 0.75 (ties at 0.25 / 0.75 -> state 0)
    if (n_states == 2) return (p > 0.25 && p < 0.75) ? 1 : 0;
    int best_k = 0;
    double best_d = 2.0;
    for (int k = 0; k < n_states; ++k) {
        double d = fabs(p - (double)k / (double)n_states);
        if (1.0 - d < d) d = 1.0 - d;
        if (d < best_d) { best_d = d; best_k = k; }
    }
    return best_k;
}

// dynamics.py:83-88 (Python float % on non-negative operands == fmod)
__host__ __device__ inline double ks_value(double ks_max, double period, double t)
{
    double tm = fmod(t, period);
    if (tm < 0.0) tm += period;
    const double half = 0.5 * period;
    return (tm <= half) ? ks_max * (tm / half) : ks_max * (2.0 - tm / half);
}

// first non-finite location, ordered like the reference's check (step, then row-major (r, i))
__device__ __forceinline__ void flag_nonfinite(unsigned long long *flag, uint64_t step, uint32_t r, uint32_t i)
{
    const unsigned long long key = (step << 36) | ((unsigned long long)(r & 0xFFFFu) << 20) | (i & 0xFFFFFu);
    atomicMin(flag, key);
}

} // namespace oscb
