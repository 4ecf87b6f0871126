// oscb_umma.cuh -- the dense (all-to-all, integer couplings) integrator on the 5th-generation
// tensor cores: ONE persistent kernel runs every Euler step of a run.
//
//   J * [cos Theta | sin Theta]  as an exact integer GEMM
//     A = J                    int8 [rows x n]        (SK couplings are +-1; any integer |J| <= 127)
//     B = digit planes of the (cos, sin) pairs:  c = 2^-30 * sum_k 2^(8k) d_k,  d_k signed bytes,
//         i.e. 4 int8 planes per component, plus the score planes: one plane of spins sigma = +-1
//         for the cut (OIM, N = 2) or N one-hot state planes for the colouring conflicts (OPM)
//     D = A * B^T              int32 in TMEM, tcgen05.mma kind::i8 (UTCIMMA), M = 128, K = 32
//   Integer accumulation is exact and order independent, so the coupling sums carry only the
//   2^-31 quantisation of each pair -- tighter than a float32 FMA chain over n = 16384 terms.
//
//   Second stream (template FP4), taken when every coupling is an e2m1 value {0, +-1, +-2, +-3, +-4, +-6} and the
//   replicas fit one launch: A = J as packed 4-bit e2m1 codes (tiles of 128 rows x 256 couplings, half the HBM and
//   shared-memory bytes), B = the same fixed-point pairs as 10 balanced base-9 digits per component (|d| <= 4, also
//   e2m1), D = float32 in TMEM holding exact integers (|sum| <= 24 n < 2^24), block-scaled tcgen05.mma kind::mxf4
//   (SASS UTCOMMA, K = 64 per instruction) with every ue8m0 block scale = 1.0.  Same integers, same results, bit for bit.
//
// Roles of the 576 threads of a CTA (one CTA per SM, one 128-row tile of J at a time):
//   warp 0   producer: cp.async.bulk (UBLKCP) of the 16 KB tile images of A (HBM stream) and
//            of B (L2 resident) into a ring of shared-memory stages, signalled on mbarriers;
//   warp 1   one elected lane issues the tcgen05.mma instructions and commits them;
//   warps 2-17 epilogue: tcgen05.ld of their 32 TMEM lanes, then per (row, replica) the fused
//            Euler update (SHIL, Philox noise, schedule, wrap; dynamics.py:166-172), the new
//            (cos, sin) digits written straight into the NEXT step's B image on every rank
//            (peer pointers: the push all-gather of the row-sharded multi-GPU run), the cut
//            contribution from the sigma plane (dynamics.py:214-223) and the sample energy
//            (dynamics.py:380).
// Steps are separated by one grid-wide (all ranks) arrive/wait on a monotonic counter; only the
// producer waits on it, and it prefetches the next step's A tiles first, so the HBM stream of J
// does not stop at a step boundary.
//
// Tile images: A and B live in global memory already in the 128-byte-swizzled K-major layout
// the UMMA shared-memory descriptor expects (byte (r, c) of a [rows x 128 B] tile at
// r*128 + ((c/16 ^ r%8)*16) + c%16), so a stage is filled by two plain bulk copies.
#pragma once
#include "oscb_device.cuh"
#include <cuda.h>      // CUtensorMap (type only; the encoder is fetched at run time, no libcuda link dependency)
#include <limits.h>

namespace oscb {

constexpr int UMMA_MAXW = 8;          // ranks a row-sharded run may span
constexpr int UMMA_TILE = 128;        // rows per tile = bytes of K per stage
constexpr int UMMA_A_STAGE = UMMA_TILE * UMMA_TILE;
constexpr int UMMA_K4 = 256;          // e2m1 stream: oscillators per k-block (128 bytes of packed 4-bit codes per row)
constexpr int UMMA_D9 = 10;           // e2m1 stream: balanced base-9 digits per component (9^10 / 2 > 2^30)
constexpr int UMMA_SF_COLS = 32;      // e2m1 stream: TMEM columns in front of the accumulator holding the (all 1.0) block scales
constexpr int UMMA_EPI_WARPS = 16;      // 4 groups x 4 TMEM lane quadrants
constexpr int UMMA_EPI_THREADS = UMMA_EPI_WARPS * 32;
constexpr int UMMA_THREADS = 64 + UMMA_EPI_THREADS;
constexpr int UMMA_MAXR = 28;         // 9 B rows per replica, N <= 256
constexpr int UMMA_RPG = UMMA_MAXR / 4; // replicas per epilogue group
constexpr int UMMA_TRACE_PASSES = 64;
constexpr int UMMA_TRACE_SLOTS = 8;

struct UmmaArgs {
    int n;                    // oscillators
    int tiles;                // ceil(n / 128): row tiles of the whole graph
    int ktiles;               // k-blocks of a row tile: tiles (int8 stream, 128 couplings per 128-byte row) or ceil(n / 256) (e2m1)
    int tile_begin, tile_end; // this rank's row tiles
    int R;                    // replicas (<= UMMA_MAXR)
    int NB;                   // rows of B: round_up(9 R, 16) -- the MMA N
    int stages;
    int world, rank;
    int tmem_cols;
    unsigned int ctas_total;  // CTAs of all ranks (grid barrier target per pass)
    int cta_offset;           // global index of this rank's CTA 0 (energy partials)
    long long passes;         // steps + 1 (the last pass only scores)
    long long first_step;
    double K, h, kn_sqrt_h, ks_max, ks_period;
    TrigConst tc;
    int noise_on;
    int n_states;             // N: 2 = OIM max-cut (one spin plane), >= 3 = OPM colouring (N one-hot state planes)
    int maximize;             // 1: max-cut (larger is better), 0: colouring conflicts (smaller is better)
    int score_cols;           // score planes per replica: 1 (N = 2) or N
    long long ld_phi;         // leading dimension of phi / best_states: local rows padded to tiles
    const uint8_t *A_img;     // [local tiles][tiles][16384]
    const uint8_t *A_fp4;     // [local tiles][ktiles][16384]: J as packed e2m1 codes (couplings in {0, +-1, +-2, +-3, +-4, +-6})
    int fp4;                  // 1: stream A_fp4 (half the HBM bytes), kind::mxf4 MMA against e2m1 base-9 digit planes
    int dcols;                // digit columns per replica: 8 (int8 stream: 4 base-256 digits per component) or 20 (e2m1: 10 base-9 digits)
    uint8_t *B_img[2][UMMA_MAXW];  // per buffer and rank: [ktiles][NB * 128]
    void *phi[2];             // [R][ld_phi] in T
    const int *W;             // [local rows] row sums of J
    const uint64_t *seeds;    // [R]
    const uint8_t *flags;     // [passes] bit 0: score the pass's input phases, bit 1: + energy sample
    unsigned int *bar[UMMA_MAXW];      // monotonic arrival counters, one per rank
    long long *events[UMMA_MAXW];      // [n_events][R]: sum_i sum_j J_ij [s_i != s_j] = 2 * cut (N = 2); sum_i sum_j J_ij [s_i == s_j] = 2 * conflicts (N >= 3)
    double *en_part[UMMA_MAXW];        // [n_samples][ctas_total][R]
    uint8_t *best_states;     // [R][ld_phi]
    unsigned long long *nonfinite;
    long long *trace;         // debug timeline [cta][UMMA_TRACE_PASSES][4] in SM clocks, or null
    int splits;               // split-K: CTAs sharing one row tile (1: a CTA owns whole row tiles).  > 1 only with one unit per CTA
    int *acc_g;               // split-K: [local tiles][NB][128] int32 partial-sum accumulator (zero between passes)
    unsigned int *tile_cnt;   // split-K: [local tiles] monotonic count of partials added
    unsigned long long *timeout_flag;  // first pass at which some CTA of this rank gave up waiting for the step barrier (0: none)
    long long watchdog_ns;             // nanoseconds (%globaltimer) a CTA waits for the other CTAs / ranks before it gives up
};

namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity)
{
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint32_t bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate)
{
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p; }"
                 ::"r"(tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
// block-scaled 4-bit MMA, K = 64 per instruction; one ue8m0 scale per 32 elements of a row, read from TMEM
__device__ __forceinline__ void mma_mxf4(uint32_t tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t sfa, uint32_t sfb,
                                         uint32_t accumulate)
{
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p; }"
                 ::"r"(tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(sfa), "r"(sfb) : "memory");
}
// 16 consecutive columns of the warp's 32 TMEM lanes <- one 32-bit value
__device__ __forceinline__ void tmem_fill16(uint32_t taddr, uint32_t v)
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, int *v)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int (&v)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_ld1(uint32_t taddr, int &v)
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(int id, int threads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

// K-major, 128-byte swizzle, rows of 128 bytes, 8-row groups 1024 bytes apart (SM100 descriptor
// version 1).  Advancing K by 32 bytes inside the swizzle atom adds 2 to the start-address field.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr)
{
    return (uint64_t)((addr >> 4) & 0x3FFFu) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// D = int32, A = B = signed 8-bit, both K-major, M = 128, N = nb
__host__ __device__ inline uint32_t instr_desc_i8(int nb)
{
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(nb >> 3) << 17) | ((uint32_t)(UMMA_TILE >> 4) << 24);
}

// kind::mxf4 (block scaled): D = float32, A = B = e2m1 packed two per byte, both K-major, ue8m0 scales (scale ids 0), K = 64
__host__ __device__ inline uint32_t instr_desc_mxf4(int nb)
{
    return (1u << 7) | (1u << 10) | ((uint32_t)(nb >> 3) << 17) | (1u << 23) | ((uint32_t)(UMMA_TILE >> 4) << 24);
}

// byte offset of (row r, k-byte c) inside a swizzled [rows x 128 B] tile image
__host__ __device__ inline uint32_t swz(uint32_t r, uint32_t c)
{
    return (r >> 3) * 1024u + (r & 7u) * 128u + ((((c >> 4) ^ (r & 7u)) << 4) | (c & 15u));
}

// c in [-1, 1] -> round(c 2^30) as four signed base-256 digits (d0 least significant)
template <typename T> __device__ __forceinline__ void pair_digits(T v, int (&d)[4])
{
    int q = (sizeof(T) == 8) ? __double2int_rn((double)v * 1073741824.0) : __float2int_rn((float)v * 1073741824.0f);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int lo = ((q & 0xFF) ^ 0x80) - 0x80;
        d[k] = lo;
        q = (q - lo) >> 8;
    }
    d[3] = q;
}
__device__ __forceinline__ long long digits_sum(const int *D)
{
    return (long long)D[0] + ((long long)D[1] << 8) + ((long long)D[2] << 16) + ((long long)D[3] << 24);
}

// e2m1 stream: round(c 2^30) as ten balanced base-9 digits (d0 least significant, |d| <= 4: every digit is an e2m1 value),
// returned as ten 4-bit e2m1 codes, digit k in bits [4k, 4k + 4)
template <typename T> __device__ __forceinline__ uint64_t pair_codes9(T v)
{
    const int q = (sizeof(T) == 8) ? __double2int_rn((double)v * 1073741824.0) : __float2int_rn((float)v * 1073741824.0f);
    // balanced digits d_k in [-4, 4]  <=>  plain base-9 digits e_k = d_k + 4 of u = q + sum_k 4 * 9^k = q + (9^10 - 1) / 2,
    // and u fits 32 bits (|q| <= 2^30 < (9^10 - 1) / 2 < 2^32 - 2^30): unsigned divisions by 9, no sign cases
    uint32_t u = (uint32_t)q + 1743392200u;
    // e2m1 codes of d = e - 4 for e = 0 .. 8:  -4 -> 0xE, -3 -> 0xD, -2 -> 0xC, -1 -> 0xA, 0 -> 0x0, 1 -> 0x2, 2 -> 0x4, 3 -> 0x5, 4 -> 0x6
    const uint64_t table = 0x65420ACDEull;
    uint64_t codes = 0;
#pragma unroll
    for (int k = 0; k < UMMA_D9; ++k) {
        const uint32_t t = __umulhi(u, 0x38E38E39u) >> 1;         // u / 9
        const uint32_t e = u - 9u * t;
        codes |= ((table >> (4u * e)) & 0xFull) << (4 * k);
        u = t;
    }
    return codes;
}
__device__ __forceinline__ long long digits_sum9(const int *D)
{
    long long s = 0;
#pragma unroll
    for (int k = UMMA_D9 - 1; k >= 0; --k) s = s * 9 + (long long)D[k];
    return s;
}
// the 4-bit codes of one oscillator and replica for the e2m1 B image: cos digits, sin digits, score planes
// (N = 2: one spin code; N >= 3: N one-hot codes, plane k in bits [4k, 4k + 4))
struct B4Codes {
    uint64_t c, s, sc;
};
template <typename T> __device__ __forceinline__ B4Codes make_b4(T cv, T sv, int state, int n_states)
{
    B4Codes o;
    o.c = pair_codes9<T>(cv);
    o.s = pair_codes9<T>(sv);
    o.sc = n_states == 2 ? (state ? 0xAull : 0x2ull) : (0x2ull << (4 * state));      // -1 / +1; one-hot +1
    return o;
}
// Two oscillators share every byte of the packed image (even index in the low nibble).  `which` selects what this
// caller stores for the pair (ev = codes of the even oscillator, od = of the odd one): bit 0 the cos planes, bit 1 the
// sin planes, bit 2 the score planes -- so two lanes can split the bytes of their pair.  kk = index of the EVEN
// oscillator inside its 256-wide k-block.
__device__ __forceinline__ void write_b4(uint8_t *Bimg, int NB, int R, int kb4, int kk, int r, const B4Codes &ev, const B4Codes &od,
                                         int n_states, int which)
{
    uint8_t *base = Bimg + (size_t)kb4 * NB * 128;
    const uint32_t c = (uint32_t)kk >> 1;
    const int row0 = 2 * UMMA_D9 * r;
    if (which & 1) {
#pragma unroll
        for (int k = 0; k < UMMA_D9; ++k)
            base[swz(row0 + k, c)] = (uint8_t)(((ev.c >> (4 * k)) & 0xF) | (((od.c >> (4 * k)) & 0xF) << 4));
    }
    if (which & 2) {
#pragma unroll
        for (int k = 0; k < UMMA_D9; ++k)
            base[swz(row0 + UMMA_D9 + k, c)] = (uint8_t)(((ev.s >> (4 * k)) & 0xF) | (((od.s >> (4 * k)) & 0xF) << 4));
    }
    if (which & 4) {
        const int srow = 2 * UMMA_D9 * R + (n_states == 2 ? r : r * n_states);
        const int planes = n_states == 2 ? 1 : n_states;
        for (int k = 0; k < planes; ++k)
            base[swz(srow + k, c)] = (uint8_t)(((ev.sc >> (4 * k)) & 0xF) | (((od.sc >> (4 * k)) & 0xF) << 4));
    }
}

// int8 stream: write the 8 digit bytes and the spin of oscillator (tile kb, column c) for replica r into one B image
template <typename T>
__device__ __forceinline__ void write_b(uint8_t *Bimg, int NB, int R, int kb, int c, int r, T cv, T sv, int state, int n_states)
{
    uint8_t *base = Bimg + (size_t)kb * NB * 128;
    int dc[4], ds[4];
    pair_digits<T>(cv, dc);
    pair_digits<T>(sv, ds);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        base[swz(8 * r + k, c)] = (uint8_t)dc[k];
        base[swz(8 * r + 4 + k, c)] = (uint8_t)ds[k];
    }
    if (n_states == 2) {
        base[swz(8 * R + r, c)] = state ? 0xFF : 0x01;                           // spin plane: sum_j J_ij sigma_j
    } else {
        for (int k = 0; k < n_states; ++k)                                       // one-hot planes: sum_j J_ij [s_j == k]
            base[swz(8 * R + r * n_states + k, c)] = k == state ? (uint8_t)1 : (uint8_t)0;
    }
}

__device__ __forceinline__ long long global_ns()
{
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned int ld_acquire(const unsigned int *p, bool sys)
{
    unsigned int v;
    if (sys) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release(unsigned int *p, bool sys)
{
    if (sys) asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
    else asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

} // namespace umma

// phases [R][n] float64 (host layout) -> this rank's rows in T, plus the B image of ALL n
// oscillators for pass 0 (every rank builds the full image locally).  One thread per PAIR of oscillators
// (the e2m1 image packs two per byte).
template <typename T>
__global__ void k_umma_init(UmmaArgs a, const double *__restrict__ phi0)
{
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int half = (a.n + 1) / 2;
    if (q >= (long long)half * a.R) return;
    const int r = (int)(q / half), j0 = 2 * (int)(q % half);
    const int row0 = a.tile_begin * UMMA_TILE, row1 = a.tile_end * UMMA_TILE;
    umma::B4Codes cd[2] = {{0, 0, 0}, {0, 0, 0}};
    for (int e = 0; e < 2; ++e) {
        const int j = j0 + e;
        if (j >= a.n) break;
        const T p = (T)phi0[(long long)r * a.n + j];
        T s, c;
        phase_trig(p, s, c);
        const int st = threshold_state((double)p, a.n_states);
        if (a.fp4) cd[e] = umma::make_b4<T>(c, s, st, a.n_states);
        else umma::write_b<T>(a.B_img[0][a.rank], a.NB, a.R, j / UMMA_TILE, j % UMMA_TILE, r, c, s, st, a.n_states);
        if (j >= row0 && j < row1) reinterpret_cast<T *>(a.phi[0])[(long long)r * a.ld_phi + (j - row0)] = p;
    }
    if (a.fp4) umma::write_b4(a.B_img[0][a.rank], a.NB, a.R, j0 / UMMA_K4, j0 % UMMA_K4, r, cd[0], cd[1], a.n_states, 7);
}

// this rank's rows as float64: out[r * ld_out + col0 + i] (col0 = first row and ld_out = n for
// the host layout [R][n]; col0 = 0 and ld_out = rows for the rank's own slice)
template <typename T>
__global__ void k_umma_export(UmmaArgs a, const void *phi, double *__restrict__ out, long long ld_out, long long col0)
{
    const int rows = min(a.n, a.tile_end * UMMA_TILE) - a.tile_begin * UMMA_TILE;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= (long long)rows * a.R) return;
    const int r = (int)(q / rows), i = (int)(q % rows);
    out[(long long)r * ld_out + col0 + i] = (double)reinterpret_cast<const T *>(phi)[(long long)r * a.ld_phi + i];
}

// int8 J rows [rows][n_pad] -> swizzled tile images + row sums
__global__ void k_umma_build_a(const int8_t *__restrict__ J, int n, int n_pad, int rows, int tiles, uint8_t *__restrict__ A_img,
                               int *__restrict__ W)
{
    // one CTA per (local tile, k-block); 256 threads move 16 KB
    const int lt = blockIdx.y, kb = blockIdx.x;
    uint8_t *img = A_img + ((size_t)lt * tiles + kb) * UMMA_A_STAGE;
    for (int q = threadIdx.x; q < UMMA_A_STAGE / 4; q += blockDim.x) {
        const int r = q / 32, c = (q % 32) * 4;
        const int row = lt * UMMA_TILE + r, col = kb * UMMA_TILE + c;
        uint32_t v = 0;
        if (row < rows && col < n_pad) v = *reinterpret_cast<const uint32_t *>(J + (size_t)row * n_pad + col); // n_pad % 4 == 0, zero padded
        *reinterpret_cast<uint32_t *>(img + umma::swz(r, c)) = v;
    }
    if (kb == 0) {
        for (int r = threadIdx.x; r < UMMA_TILE; r += blockDim.x) {
            const int row = lt * UMMA_TILE + r;
            int s = 0;
            if (row < rows)
                for (int j = 0; j < n; ++j) s += J[(size_t)row * n_pad + j];
            W[lt * UMMA_TILE + r] = s;
        }
    }
}

// int8 J rows with every coupling in {0, +-1, +-2, +-3, +-4, +-6} -> swizzled tile images of packed e2m1 codes: tile
// (lt, kb) covers 128 rows x 256 columns; byte c of a row holds column 2c in its low nibble and 2c + 1 in its high nibble.
__global__ void k_umma_build_fp4(const int8_t *__restrict__ J, int n, int n_pad, int rows, int ktiles, uint8_t *__restrict__ A_fp4)
{
    const int lt = blockIdx.y, kb = blockIdx.x;
    uint8_t *img = A_fp4 + ((size_t)lt * ktiles + kb) * UMMA_A_STAGE;
    for (int t = threadIdx.x; t < UMMA_A_STAGE; t += blockDim.x) {
        const int r = t >> 7, c = t & 127;
        const int row = lt * UMMA_TILE + r;
        uint32_t code[2] = {0, 0};
        for (int h = 0; h < 2; ++h) {
            const int col = kb * UMMA_K4 + 2 * c + h;
            int v = 0;
            if (row < rows && col < n) v = J[(size_t)row * n_pad + col];
            const int m = v < 0 ? -v : v;
            const uint32_t mag = m == 0 ? 0u : m == 1 ? 2u : m == 2 ? 4u : m == 3 ? 5u : m == 4 ? 6u : 7u;   // 6 -> 7
            code[h] = mag | (v < 0 ? 8u : 0u);
        }
        img[umma::swz((uint32_t)r, (uint32_t)c)] = (uint8_t)(code[0] | (code[1] << 4));
    }
}

template <typename T, bool FP4>
__global__ void __launch_bounds__(UMMA_THREADS, 1) k_dense_umma(const UmmaArgs a)
{
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = umma::smem_u32(smem_raw);
    const uint32_t base = (raw + 1023u) & ~1023u;
    uint8_t *smem = smem_raw + (base - raw);
    const int stages = a.stages;
    const uint32_t b_stage = (uint32_t)a.NB * 128u;
    const uint32_t sA = base, sB = base + (uint32_t)stages * UMMA_A_STAGE;
    uint8_t *ctl = smem + (size_t)stages * (UMMA_A_STAGE + b_stage);
    uint64_t *bars = reinterpret_cast<uint64_t *>(ctl);            // full[16], empty[16], tmem_full, tmem_empty
    const uint32_t bar_full = umma::smem_u32(bars), bar_empty = bar_full + 8u * 16;
    const uint32_t bar_tfull = bar_empty + 8u * 16, bar_tempty = bar_tfull + 8u;
    long long *best_s = reinterpret_cast<long long *>(ctl + 512);                // [32]
    double *en_acc = reinterpret_cast<double *>(best_s + 32);                    // [32]
    double *en_w = en_acc + 32;                                                  // [4][32]
    int *improved_s = reinterpret_cast<int *>(en_w + 128);                       // [32]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(improved_s + 32);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool sys = a.world > 1;
    // Work units.  splits == 1: CTA b owns row tiles b, b + grid, ... with their whole K range.  splits = S > 1 (a rank
    // of a row-sharded run owns few row tiles, or a small graph): the grid is exactly tiles x S, CTA b integrates
    // k-blocks [kb0, kb1) of row tile b / S; the S partial sums of a tile meet in a global int32 accumulator and the
    // split-0 CTA of the tile runs the update.  Integer sums: the result does not depend on S.
    const int S = a.splits;
    const int ksplit = S > 1 ? (int)blockIdx.x % S : 0;
    const int lt_first = S > 1 ? (int)blockIdx.x / S : (int)blockIdx.x;
    const int lt_stride = S > 1 ? 0 : (int)gridDim.x;
    const int kb0 = S > 1 ? (int)(((long long)ksplit * a.ktiles) / S) : 0;
    const int kb1 = S > 1 ? (int)(((long long)(ksplit + 1) * a.ktiles) / S) : a.ktiles;
    const bool lead = ksplit == 0;
    const int my_tiles = S > 1 ? 1 : (a.tile_end - a.tile_begin - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const long long per_pass = (long long)my_tiles * (kb1 - kb0);
    const uint32_t stage_tx = (uint32_t)UMMA_A_STAGE + b_stage;

    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            umma::mbar_init(bar_full + 8u * s, 1);
            umma::mbar_init(bar_empty + 8u * s, 1);
        }
        umma::mbar_init(bar_tfull, 1);
        umma::mbar_init(bar_tempty, UMMA_EPI_WARPS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(umma::smem_u32(tmem_slot)), "r"(a.tmem_cols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (threadIdx.x >= 64 && threadIdx.x - 64 < 32) {
        best_s[threadIdx.x - 64] = a.maximize ? LLONG_MIN : LLONG_MAX;
        en_acc[threadIdx.x - 64] = 0.0;
        improved_s[threadIdx.x - 64] = 0;
    }
    umma::tc_fence_before();
    __syncthreads();
    umma::tc_fence_after();
    const uint32_t tmem_sf = *tmem_slot;
    const uint32_t tmem = tmem_sf + (FP4 ? (uint32_t)UMMA_SF_COLS : 0u);          // the accumulator
    if (FP4) {
        // block scales of the mxf4 MMA: every ue8m0 byte = 127 (2^0), so their layout inside the columns does not matter
        if (warp >= 2 && warp < 6) {
            const uint32_t t = tmem_sf + ((uint32_t)((warp & 3) * 32) << 16);
            umma::tmem_fill16(t, 0x7F7F7F7Fu);
            umma::tmem_fill16(t + 16u, 0x7F7F7F7Fu);
            umma::tmem_st_wait();
        }
        umma::tc_fence_before();
        __syncthreads();
        umma::tc_fence_after();
    }

    if (warp == 0) {
        // ===== producer =====  (one thread; no divisions on this path: it paces the whole CTA)
        if (lane == 0) {
            struct Cursor {
                int s; uint32_t ph; int tk, kb;
            };
            Cursor ca{0, 0, 0, kb0}, cb{0, 0, 0, kb0};
            auto advance = [&](Cursor &c) {
                if (++c.s == stages) { c.s = 0; c.ph ^= 1u; }
                if (++c.kb == kb1) { c.kb = kb0; if (++c.tk == my_tiles) c.tk = 0; }
            };
            auto issue_a = [&](Cursor &c) {
                umma::mbar_wait(bar_empty + 8u * c.s, c.ph ^ 1u);
                umma::mbar_expect_tx(bar_full + 8u * c.s, stage_tx);
                const int lt = lt_first + c.tk * lt_stride;
                const uint8_t *img = FP4 ? a.A_fp4 : a.A_img;
                umma::bulk_g2s(sA + (uint32_t)c.s * UMMA_A_STAGE, img + ((size_t)lt * a.ktiles + c.kb) * UMMA_A_STAGE, UMMA_A_STAGE,
                               bar_full + 8u * c.s);
                advance(c);
            };
            auto issue_b = [&](Cursor &c, const uint8_t *Bsrc) {
                umma::bulk_g2s(sB + (uint32_t)c.s * b_stage, Bsrc + (size_t)c.kb * b_stage, b_stage, bar_full + 8u * c.s);
                advance(c);
            };
            const int per_pass_i = (int)per_pass;
            const int pre = per_pass_i < stages ? per_pass_i : stages;
            bool dead = false;
            for (long long pass = 0; pass < a.passes; ++pass) {
                const uint8_t *Bsrc = a.B_img[pass & 1][a.rank];
                int start = 0;
                if (pass > 0) {
                    for (int j = 0; j < pre; ++j) issue_a(ca);                  // J does not depend on the step: run ahead
                    const unsigned int target = a.ctas_total * (unsigned int)pass;
                    if (a.trace && pass < UMMA_TRACE_PASSES) a.trace[((long long)blockIdx.x * UMMA_TRACE_PASSES + pass) * UMMA_TRACE_SLOTS + 3] = clock64();
                    if (!dead) {
                        // watchdog: a peer rank that never launched (or died) must not hang this GPU.  After the
                        // deadline the run is abandoned -- the flag makes finish() fail -- and the kernel free-runs
                        // through its remaining passes without waiting, so it terminates.
                        const long long t_wait = umma::global_ns();
                        while ((int)(umma::ld_acquire(a.bar[a.rank], sys) - target) < 0) {
                            if (umma::global_ns() - t_wait > a.watchdog_ns) {
                                dead = true;
                                atomicMin(a.timeout_flag, (unsigned long long)pass);
                                break;
                            }
                        }
                    }
                    if (a.trace && pass < UMMA_TRACE_PASSES) a.trace[((long long)blockIdx.x * UMMA_TRACE_PASSES + pass) * UMMA_TRACE_SLOTS + 0] = clock64();
                    umma::fence_proxy_async();
                    for (int j = 0; j < pre; ++j) issue_b(cb, Bsrc);
                    start = pre;
                }
                for (int j = start; j < per_pass_i; ++j) {
                    issue_a(ca);
                    issue_b(cb, Bsrc);
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        if (lane == 0) {
            const uint32_t idesc = FP4 ? umma::instr_desc_mxf4(a.NB) : umma::instr_desc_i8(a.NB);
            const uint32_t sfa = tmem_sf, sfb = tmem_sf + (uint32_t)(UMMA_SF_COLS / 2);
            long long acc_it = 0;
            int s = 0;
            uint32_t ph = 0;
            for (long long pass = 0; pass < a.passes; ++pass) {
                for (int tk = 0; tk < my_tiles; ++tk) {
                    umma::mbar_wait(bar_tempty, (uint32_t)((acc_it & 1) ^ 1));
                    umma::tc_fence_after();
                    for (int kb = kb0; kb < kb1; ++kb) {
                        umma::mbar_wait(bar_full + 8u * s, ph);
                        umma::tc_fence_after();
                        const uint64_t ad = umma::smem_desc(sA + (uint32_t)s * UMMA_A_STAGE);
                        const uint64_t bd = umma::smem_desc(sB + (uint32_t)s * b_stage);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            if (FP4) umma::mma_mxf4(tmem, ad + 2u * k, bd + 2u * k, idesc, sfa, sfb, (uint32_t)(((kb - kb0) | k) != 0));
                            else umma::mma_i8(tmem, ad + 2u * k, bd + 2u * k, idesc, (uint32_t)(((kb - kb0) | k) != 0));
                        }
                        umma::tc_commit(bar_empty + 8u * s);
                        if (++s == stages) { s = 0; ph ^= 1u; }
                    }
                    umma::tc_commit(bar_tfull);
                    ++acc_it;
                }
            }
        }
    } else {
        // ===== epilogue: 16 warps.  Warp w reads TMEM lanes 32 (w % 4) .. +31 (a hardware rule), so the
        // four warps of "group" g = (w - 2) / 4 cover the 128 rows of the tile; group g owns the
        // replicas r = g, g + 4, ...  Everything that does not need the coupling sums (own trig,
        // SHIL, the Philox draw) is computed BEFORE the wait on the accumulator. =====
        const int et = (int)threadIdx.x - 64;
        const int quad = warp & 3;
        const int group = (warp - 2) >> 2;
        const int rowt = quad * 32 + lane;
        const uint32_t tlane = tmem + ((uint32_t)(quad * 32) << 16);
        const int R = a.R;
        const T hT = (T)a.h, KT = (T)a.K, knT = (T)a.kn_sqrt_h;
        long long e_idx = 0, s_idx = 0, acc_it = 0;
        const int row0 = a.tile_begin * UMMA_TILE;
        const int cta_global = a.cta_offset + (int)blockIdx.x;
        for (long long pass = 0; pass < a.passes; ++pass) {
            const int flags = a.flags[pass];
            const bool prev_scored = pass > 0 && (a.flags[pass - 1] & 1);
            const bool last = pass == a.passes - 1;
            const uint64_t gstep = (uint64_t)(a.first_step + pass);
            const T ksT = (T)ks_value(a.ks_max, a.ks_period, (double)gstep * a.h);
            const T *phi_in = reinterpret_cast<const T *>(a.phi[pass & 1]);
            T *phi_out = reinterpret_cast<T *>(a.phi[(pass + 1) & 1]);
            bool checked = false;
            for (int tk = 0; tk < my_tiles; ++tk) {
                const int lt = lt_first + tk * lt_stride;
                const int tile = a.tile_begin + lt;
                const int rowl = lt * UMMA_TILE + rowt;
                const int row = row0 + rowl;
                const bool valid = row < a.n && lead;          // (only the split-0 CTA of a tile updates its rows)
                // ---- before the sums exist ----
                T pre_p[UMMA_RPG], pre_s[UMMA_RPG], pre_c[UMMA_RPG], pre_d[UMMA_RPG];   // phase, sin, cos, h*(-ks shil) + kn xi
                const int Wi = valid ? a.W[rowl] : 0;
#pragma unroll
                for (int k = 0; k < UMMA_RPG; ++k) {
                    const int r = group + 4 * k;
                    pre_p[k] = pre_s[k] = pre_c[k] = pre_d[k] = T(0);
                    if (r < R && valid) {
                        const T p = phi_in[(long long)r * a.ld_phi + rowl];
                        T si, ci;
                        phase_trig(p, si, ci);
                        T kick = T(0);
                        if (a.noise_on && !last) {
                            T z[4];
                            normals4(noise_block(a.seeds[r], gstep, (uint32_t)(row >> 2)), z);
                            kick = z[row & 3];
                        }
                        pre_p[k] = p; pre_s[k] = si; pre_c[k] = ci;
                        pre_d[k] = kick;
                    }
                }
                umma::mbar_wait(bar_tfull, (uint32_t)(acc_it & 1));
                umma::tc_fence_after();
                if (a.trace && et == 0 && pass < UMMA_TRACE_PASSES) a.trace[((long long)blockIdx.x * UMMA_TRACE_PASSES + pass) * UMMA_TRACE_SLOTS + 1] = clock64();
                if (!checked) {
                    // the grid barrier of the previous pass is behind us: its cut totals are complete
                    if (prev_scored && et < R) {
                        const long long tot = *reinterpret_cast<volatile long long *>(a.events[a.rank] + (e_idx - 1) * R + et);
                        const int imp = a.maximize ? (tot > best_s[et]) : (tot < best_s[et]);
                        improved_s[et] = imp;
                        if (imp) best_s[et] = tot;
                    }
                    if (prev_scored) umma::named_bar_sync(1, UMMA_EPI_THREADS);
                    checked = true;
                }
                // column-major inside the tile ([col][row]): the 32 lanes of a warp add to 32 consecutive ints, one L2 line
                int *accrow = S > 1 ? a.acc_g + (size_t)lt * UMMA_TILE * a.NB + rowt : nullptr;
                auto acc_at = [&](int col) -> int * { return accrow + (size_t)col * UMMA_TILE; };
                if (S > 1) {
                    // ---- split-K: this CTA's partial sums of its K range -> the tile's global accumulator ----
                    for (int k = 0; k < UMMA_RPG; ++k) {
                        const int r = group + 4 * k;
                        if (r >= R) break;
                        const int dcols = a.dcols, sc = a.score_cols;
                        int P[2 * UMMA_D9];
                        if (FP4) {
#pragma unroll
                            for (int q4 = 0; q4 < 2 * UMMA_D9; q4 += 4) umma::tmem_ld4(tlane + (uint32_t)(2 * UMMA_D9 * r + q4), P + q4);
                        } else {
                            umma::tmem_ld8(tlane + (uint32_t)(8 * r), reinterpret_cast<int (&)[8]>(P));
                        }
                        umma::tmem_ld_wait();
                        for (int q = 0; q < dcols; ++q)
                            atomicAdd(acc_at(dcols * r + q), FP4 ? __float2int_rn(__int_as_float(P[q])) : P[q]);
                        for (int q = 0; q < sc; ++q) {
                            int v;
                            umma::tmem_ld1(tlane + (uint32_t)(dcols * R + r * sc + q), v);
                            umma::tmem_ld_wait();
                            atomicAdd(acc_at(dcols * R + r * sc + q), FP4 ? __float2int_rn(__int_as_float(v)) : v);
                        }
                    }
                    umma::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) umma::mbar_arrive(bar_tempty);          // the accumulator is free again
                    ++acc_it;
                    umma::named_bar_sync(1, UMMA_EPI_THREADS);
                    if (et == 0) umma::red_release(a.tile_cnt + lt, false); // (cumulative over the CTA barrier: all partials are in)
                    if (lead) {
                        if (et == 0) {
                            const unsigned int want = (unsigned int)S * (unsigned int)(pass + 1);
                            const long long t_wait = umma::global_ns();
                            while ((int)(umma::ld_acquire(a.tile_cnt + lt, false) - want) < 0) {
                                if (umma::global_ns() - t_wait > a.watchdog_ns) { atomicMin(a.timeout_flag, (unsigned long long)pass); break; }
                            }
                        }
                        umma::named_bar_sync(1, UMMA_EPI_THREADS);
                    }
                }
                if (S > 1 && !lead) {
                    if ((flags & 2) && lane == 0)
                        for (int r = group; r < R; r += 4) en_w[quad * 32 + r] = 0.0;
                } else {
#pragma unroll
                for (int k = 0; k < UMMA_RPG; ++k) {
                    const int r = group + 4 * k;
                    if (r >= R) break;                       // warp uniform
                    int D[2 * UMMA_D9], Dsig = 0;
                    const int dcols = a.dcols;
                    if (S > 1) {
                        // the tile's complete sums (already integers); zero them for the next pass -- the other splits add
                        // again only after this pass's grid barrier, which this CTA arrives at after these stores
                        for (int q = 0; q < dcols; ++q) D[q] = __ldcg(acc_at(dcols * r + q));
                        for (int q = 0; q < dcols; ++q) __stcg(acc_at(dcols * r + q), 0);
                        const int sc = a.score_cols;
                        for (int q = 0; q < sc; ++q) {
                            const int v = __ldcg(acc_at(dcols * R + r * sc + q));
                            __stcg(acc_at(dcols * R + r * sc + q), 0);
                            if (sc == 1 || q == ((flags & 1) ? threshold_state((double)pre_p[k], a.n_states) : 0)) Dsig = v;
                        }
                    } else if (FP4) {
#pragma unroll
                        for (int q4 = 0; q4 < 2 * UMMA_D9; q4 += 4) umma::tmem_ld4(tlane + (uint32_t)(2 * UMMA_D9 * r + q4), D + q4);
                    } else {
                        umma::tmem_ld8(tlane + (uint32_t)(8 * r), reinterpret_cast<int (&)[8]>(D));
                    }
                    const T p = pre_p[k], si = pre_s[k], ci = pre_c[k];
                    const int st = (flags & 1) ? threshold_state((double)p, a.n_states) : 0;
                    if ((flags & 1) && S == 1) {
                        if (a.n_states == 2) {
                            umma::tmem_ld1(tlane + (uint32_t)(dcols * R + r), Dsig);
                        } else {
                            // tcgen05.ld takes ONE column address for the whole warp: read the N state planes, keep the own state's
                            for (int q = 0; q < a.n_states; ++q) {
                                int v;
                                umma::tmem_ld1(tlane + (uint32_t)(dcols * R + r * a.n_states + q), v);
                                umma::tmem_ld_wait();
                                if (q == st) Dsig = v;
                            }
                        }
                    }
                    umma::tmem_ld_wait();
                    if (a.trace && et == 0 && k == 0 && pass < UMMA_TRACE_PASSES) a.trace[((long long)blockIdx.x * UMMA_TRACE_PASSES + pass) * UMMA_TRACE_SLOTS + 4] = clock64();

                    if (FP4 && S == 1) {
                        // the mxf4 accumulator is float32 holding exact integers (|sum| < 2^24): back to int
#pragma unroll
                        for (int q4 = 0; q4 < 2 * UMMA_D9; ++q4) D[q4] = __float2int_rn(__int_as_float(D[q4]));
                        Dsig = __float2int_rn(__int_as_float(Dsig));
                    }
                    const long long Sx = FP4 ? umma::digits_sum9(D) : umma::digits_sum(D);
                    const long long Sy = FP4 ? umma::digits_sum9(D + UMMA_D9) : umma::digits_sum(D + 4);
                    const long long at = (long long)r * a.ld_phi + rowl;
                    if (prev_scored && improved_s[r] && valid)
                        a.best_states[at] = (uint8_t)threshold_state((double)phi_out[at], a.n_states);   // phi_out still holds the scored phases
                    if (flags & 1) {
                        // N = 2: sum_j J_ij [s_i != s_j] = (W_i - sigma_i sum_j J_ij sigma_j) / 2;  N >= 3: sum_j J_ij [s_j == s_i]
                        long long contrib = 0;
                        if (valid) contrib = a.n_states == 2 ? ((long long)Wi - (st ? -(long long)Dsig : (long long)Dsig)) / 2 : (long long)Dsig;
                        for (int off = 16; off > 0; off >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, off);
                        if (lane == 0)
                            for (int w = 0; w < a.world; ++w) {
                                unsigned long long *dst = reinterpret_cast<unsigned long long *>(a.events[w] + e_idx * R + r);
                                if (sys) atomicAdd_system(dst, (unsigned long long)contrib);
                                else atomicAdd(dst, (unsigned long long)contrib);
                            }
                    }
                    if (flags & 2) {
                        const double sc = 9.313225746154785e-10; // 2^-30
                        double e = valid ? 0.5 * ((double)ci * ((double)Sx * sc) + (double)si * ((double)Sy * sc)) : 0.0;
                        for (int off = 16; off > 0; off >>= 1) e += __shfl_xor_sync(0xffffffffu, e, off);
                        if (lane == 0) en_w[quad * 32 + r] = e;
                    }
                    umma::B4Codes mine = {0, 0, 0};
                    if (!last && valid) {
                        const T scale = (T)9.313225746154785e-10;
                        const T accv = si * ((T)Sx * scale) - ci * ((T)Sy * scale);
                        const T shil = shil_term(p, si, ci, a.tc);
                        const T x = p + hT * (KT * accv - ksT * shil) + knT * pre_d[k];
                        if (!isfinite(x)) flag_nonfinite(a.nonfinite, gstep, (uint32_t)r, (uint32_t)row);
                        const T y = wrap_unit(x);
                        phi_out[at] = y;
                        T s2, c2;
                        phase_trig(y, s2, c2);
                        const int st2 = threshold_state((double)y, a.n_states);
                        if (FP4) {
                            mine = umma::make_b4<T>(c2, s2, st2, a.n_states);
                        } else {
                            for (int w = 0; w < a.world; ++w)
                                umma::write_b<T>(a.B_img[(pass + 1) & 1][w], a.NB, R, tile, rowt, r, c2, s2, st2, a.n_states);
                        }
                    }
                    if (a.trace && et == 0 && k == 0 && pass < UMMA_TRACE_PASSES) a.trace[((long long)blockIdx.x * UMMA_TRACE_PASSES + pass) * UMMA_TRACE_SLOTS + 5] = clock64();
                    if (FP4 && !last) {
                        // two oscillators per byte: lanes 2i and 2i + 1 swap codes, the even lane stores the pair's cos and
                        // score planes, the odd lane its sin planes (rows past n carry zero codes)
                        umma::B4Codes other;
                        other.c = __shfl_xor_sync(0xffffffffu, mine.c, 1);
                        other.s = __shfl_xor_sync(0xffffffffu, mine.s, 1);
                        other.sc = __shfl_xor_sync(0xffffffffu, mine.sc, 1);
                        const bool odd = lane & 1;
                        if (row - (int)odd < a.n) {
                            const int kk = (tile & 1) * UMMA_TILE + (rowt & ~1);
                            for (int w = 0; w < a.world; ++w)
                                umma::write_b4(a.B_img[(pass + 1) & 1][w], a.NB, R, tile >> 1, kk, r, odd ? other : mine, odd ? mine : other,
                                               a.n_states, odd ? 2 : 5);
                        }
                    }
                }
                }   // (leader / unsplit tile)
                if (a.trace && et == 0 && pass < UMMA_TRACE_PASSES) a.trace[((long long)blockIdx.x * UMMA_TRACE_PASSES + pass) * UMMA_TRACE_SLOTS + 6] = clock64();
                if (S == 1) {
                    umma::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) umma::mbar_arrive(bar_tempty);
                    ++acc_it;
                }
                if (flags & 2) {
                    umma::named_bar_sync(1, UMMA_EPI_THREADS);
                    if (et < R) en_acc[et] += ((en_w[et] + en_w[32 + et]) + en_w[64 + et]) + en_w[96 + et];
                    umma::named_bar_sync(1, UMMA_EPI_THREADS);
                }
            }
            if ((flags & 2) && et < R) {
                for (int w = 0; w < a.world; ++w)
                    a.en_part[w][((size_t)s_idx * a.ctas_total + cta_global) * R + et] = en_acc[et];
                en_acc[et] = 0.0;
            }
            // publish: every write of this pass (phases' digits on all ranks, cut atomics, energy
            // partials) before the arrival that lets the next pass start anywhere
            umma::fence_proxy_async();
            umma::named_bar_sync(1, UMMA_EPI_THREADS);
            if (et == 0) {
                if (a.trace && pass < UMMA_TRACE_PASSES) a.trace[((long long)blockIdx.x * UMMA_TRACE_PASSES + pass) * UMMA_TRACE_SLOTS + 7] = clock64();
                // red.release is the fence: it is cumulative over the CTA barrier above, so every epilogue thread's stores and
                // atomics of this pass are visible (gpu / system scope) to whoever acquires the counter
                for (int w = 0; w < a.world; ++w) umma::red_release(a.bar[w], sys);
                if (a.trace && pass < UMMA_TRACE_PASSES) a.trace[((long long)blockIdx.x * UMMA_TRACE_PASSES + pass) * UMMA_TRACE_SLOTS + 2] = clock64();
            }
            if (flags & 1) ++e_idx;
            if (flags & 2) ++s_idx;
        }
        // the last pass scored the final phases: wait for every rank's totals, then keep the states
        if (et == 0) {
            const unsigned int target = a.ctas_total * (unsigned int)a.passes;
            const long long t_wait = umma::global_ns();
            while ((int)(umma::ld_acquire(a.bar[a.rank], sys) - target) < 0) {
                if (umma::global_ns() - t_wait > a.watchdog_ns) {        // (same watchdog as the producer's)
                    atomicMin(a.timeout_flag, (unsigned long long)a.passes);
                    break;
                }
            }
        }
        umma::named_bar_sync(1, UMMA_EPI_THREADS);
        if ((a.flags[a.passes - 1] & 1) && et < R) {
            const long long tot = *reinterpret_cast<volatile long long *>(a.events[a.rank] + (e_idx - 1) * R + et);
            improved_s[et] = a.maximize ? (tot > best_s[et]) : (tot < best_s[et]);
        }
        umma::named_bar_sync(1, UMMA_EPI_THREADS);
        if (a.flags[a.passes - 1] & 1) {
            const T *phi_fin = reinterpret_cast<const T *>(a.phi[(a.passes - 1) & 1]);
            for (int tk = 0; tk < my_tiles; ++tk) {
                const int rowl = (lt_first + tk * lt_stride) * UMMA_TILE + rowt;
                if (row0 + rowl < a.n && lead)
                    for (int r = group; r < R; r += 4)
                        if (improved_s[r]) a.best_states[(long long)r * a.ld_phi + rowl] = (uint8_t)threshold_state((double)phi_fin[(long long)r * a.ld_phi + rowl], a.n_states);
            }
        }
    }
    umma::tc_fence_before();
    __syncthreads();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_sf), "r"(a.tmem_cols) : "memory");
}

} // namespace oscb
