// oscb_umma.hpp -- host interface of the tensor-core dense integrator (oscb_umma.cu), shared
// with the C ABI translation unit (oscb.cu).
#pragma once
#include "oscb_host.hpp"
#include <algorithm>

namespace oscb {

// per dense int8 handle: the swizzled tile images of the handle's rows of J and their row sums
struct UmmaPlan {
    int n = 0, tiles = 0, tile_begin = 0, tile_end = 0;
    DevBuf<uint8_t> A_img;
    DevBuf<uint8_t> A_fp4;    // packed e2m1 images, when every coupling is in {0, +-1, +-2, +-3, +-4, +-6}
    bool fp4_ok = false;
    DevBuf<int> W;
};

// rows [row_begin, row_end) of J as int8 [rows][n_pad] on the device -> plan (row_begin % 128 == 0;
// row_end % 128 == 0 or row_end == n)
std::shared_ptr<UmmaPlan> umma_build_plan(const int8_t *J8_dev, int64_t n, int n_pad, int64_t row_begin, int64_t row_end,
                                          bool fp4_ok, cudaStream_t s);

constexpr int kUmmaMaxReplicas = 28;      // N = 2: 9 B rows per replica; use umma_max_replicas(N) in general
inline int umma_max_replicas(int n_states, bool fp4 = false)
{
    return std::min(kUmmaMaxReplicas, 256 / ((fp4 ? 20 : 8) + (n_states == 2 ? 1 : n_states)));
}
bool umma_uses_fp4(const UmmaPlan &plan, int R, int n_states, int force_stream = 0);   // the packed e2m1 stream for a call of R replicas in all (see oscb_umma.cu)
constexpr int kUmmaMaxWorld = 8;

// what one rank of a row-sharded run publishes about its exchange block (the memory its peers
// push phase digits, cut sums, energy partials and barrier arrivals into)
struct UmmaExchange {
    unsigned char ipc[64];   // cudaIpcMemHandle_t of the block
    uint64_t base;           // device address in the owning process
    uint64_t bytes;
    int32_t device;
    int32_t pid;
    int32_t grid;            // CTAs this rank launches
    int32_t stream_sig;      // layout of the B image this rank reads and WRITES INTO ITS PEERS: (fp4, B rows, digit columns, K tiles)
};

// schedule and parameters of one run of <= kUmmaMaxReplicas replicas
struct UmmaSpec {
    int R = 1;
    int R_total = 0;                    // replicas of the whole call (several launches): picks the stream; 0 = R
    int force_stream = 0;               // 0: by plan / OSCB_UMMA_FP4; 8: the int8 stream; 4: the packed e2m1 stream (must be possible)
    int precision = OSCB_PREC_F32;
    int noise_on = 1;
    int n_states = 2, maximize = 1;     // N = 2 max-cut, or N-state colouring (unit couplings)
    double K = 0, h = 0, kn_sqrt_h = 0, ks_max = 0, ks_period = 1;
    long long steps = 0, first_step = 0;
    const uint8_t *flags = nullptr;     // host [steps + 1]: bit 0 score the pass's input phases, bit 1 + energy sample
    long long n_events = 0, n_samples = 0;
};

// One rank's side of a run: the whole graph on one GPU (world = 1) or a 128-row-aligned shard of
// it, with the per-step exchange pushed into the peers' blocks by the kernel itself.
class UmmaSession {
public:
    UmmaSession(oscb_graph *g, const UmmaSpec &spec, int world, int rank);
    ~UmmaSession();
    UmmaSession(const UmmaSession &) = delete;
    UmmaSession &operator=(const UmmaSession &) = delete;

    void export_mem(UmmaExchange *out) const;
    void connect(const UmmaExchange *all);                       // [world]; world = 1 needs no call
    // zero the exchange block, upload seeds, build this rank's phases and the pass-0 digit image
    // from d_phi0 (device, float64 [R][n]).  Every rank must have prepared before any rank launches.
    void prepare(const uint64_t *seeds, const double *d_phi0);
    void launch();                                               // asynchronous on the handle's stream
    // wait for the kernel; rows = this rank's rows.  Any pointer may be null.
    void finish(double *h_final_rows /* [R][rows] */, uint8_t *h_best_rows /* [R][rows] */, long long *h_events /* [E][R] */,
                double *h_energy /* [S][R] */);
    // same, but the final phases go to a device buffer in the host layout [R][n] (world = 1 path)
    void export_final(double *d_final_full);

    int rows() const;
    float ms = 0.f;
    int grid = 0, stages = 0, splits = 1;      // CTAs, ring depth, CTAs sharing one row tile (split-K)
    size_t smem = 0;
    unsigned long long nonfinite = ~0ull;

private:
    struct Impl;
    Impl *m;
};

} // namespace oscb
