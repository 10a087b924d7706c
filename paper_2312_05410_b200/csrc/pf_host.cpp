// pf_host.cpp -- host runtime of libpf: the C ABI of include/pf.h.
//
// Responsibilities:
//   * parameter presets and validation, including the stability bound (R-18);
//   * seeded initial conditions on the host (row a0; readings R-14..R-16), this library's own
//     implementation of the counter-based generator (the oracle has a separate one);
//   * device buffers in the padded layout of DESIGN.md 6, the stepping loop (two fused stage
//     kernels per explicit-midpoint step), CUDA-graph replay for launch-bound grids;
//   * halo exchange between y-slabs: NCCL p2p between ranks, or device copies in loopback mode;
//   * diagnostics / blow-up checks, get / set of fields, error reporting.
// Compiled with -ffp-contract=off so the initial fields are bitwise reproducible (R-16).
#include "pf.h"

#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <utility>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pf_internal.h"

namespace {
// NVTX range for profilers (nsys / ncu --nvtx): stage launches, halo exchanges, diagnostics and the
// small-grid launches show up named on the timeline.  Header-only NVTX v3; no-ops without a tool.
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};
}  // namespace

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

namespace {

thread_local std::string g_create_error;

std::string fmt(const char *f, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, f);
    vsnprintf(buf, sizeof buf, f, ap);
    va_end(ap);
    return buf;
}

// ---------------------------------------------------------------------------------------
// Counter-based generator (reading R-16): key = mix(seed ^ stream * C), draw(k) = mix(key + k).
class CounterRng {
public:
    CounterRng(uint64_t seed, uint64_t stream) : key_(mix(seed ^ (stream * 0xD1B54A32D192ED03ull))) {}
    uint64_t bits(uint64_t k) const { return mix(key_ + k); }
    double unif(uint64_t k) const { return (double)(bits(k) >> 11) * 0x1.0p-53; }
    double normal(uint64_t idx) const {   // Box-Muller, cosine branch
        const double u1 = unif(2 * idx), u2 = unif(2 * idx + 1);
        return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);
    }

private:
    static uint64_t mix(uint64_t z) {   // SplitMix64 output function of z + gamma
        z += 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    uint64_t key_;
};

enum Stream : uint64_t { kStreamC = 0, kStreamPhi = 1, kStreamCuts = 2, kStreamRate = 3, kStreamAngle = 4,
                         kStreamMobA = 5, kStreamMobB = 6, kStreamInflow = 7 };

// Velocity of global member gm (R-10, R-15, R-21).
void member_velocity(const pf_params &p, int64_t gm, double &vx, double &vy) {
    const CounterRng rng(p.seed, (uint64_t)gm * 8u + kStreamRate);
    const double mult = p.rate_lo + (p.rate_hi - p.rate_lo) * rng.unif(0);
    const double v0m = p.v0 * mult;
    double th_deg = p.theta_deg;   // per-member angle sweep (R-21)
    if (p.theta_span != 0.0) th_deg = p.theta_deg + p.theta_span * CounterRng(p.seed, (uint64_t)gm * 8u + kStreamAngle).unif(0);
    const double th = th_deg * (M_PI / 180.0);
    vx = v0m * std::cos(th);
    vy = -(v0m * std::sin(th));
}

// Composition mobilities of global member gm (R-6, R-23): species A scaled by
// a = mob_lo + (mob_hi - mob_lo) U(seed, 8gm+5, 0), species B by b (stream 8gm+6).
// out = {M_A^bulk, M_B^bulk, M_A^surf, M_B^surf}.
void member_mobility(const pf_params &p, int64_t gm, double out[4]) {
    const double a = p.mob_lo + (p.mob_hi - p.mob_lo) * CounterRng(p.seed, (uint64_t)gm * 8u + kStreamMobA).unif(0);
    const double b = p.mob_lo + (p.mob_hi - p.mob_lo) * CounterRng(p.seed, (uint64_t)gm * 8u + kStreamMobB).unif(0);
    out[0] = p.M_A_bulk * a;
    out[1] = p.M_B_bulk * b;
    out[2] = p.M_A_surf * a;
    out[3] = p.M_B_surf * b;
}

// Stochastic inflow value (R-27), this library's host implementation (the kernels have their own).
double inflow_host(const pf_params &p, int64_t gm, int64_t step, int i) {
    const CounterRng rng(p.seed, (uint64_t)gm * 8u + kStreamInflow);
    for (int a = 0; a < 8; ++a) {
        const uint64_t q = ((uint64_t)step * (uint64_t)p.nx + (uint64_t)i) * 8u + (uint64_t)a;
        const double u1 = rng.unif(2 * q), u2 = rng.unif(2 * q + 1);
        const double z = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);
        const double v = p.rho_in + p.noise_rho * z;
        if (v >= 0.0 && v <= 2.0 * p.rho_in) return v;
    }
    return p.rho_in;
}

// Column boundaries of the columnar recipe: ncols-1 distinct sorted cuts in [1, nx-1] (R-14).
std::vector<int64_t> column_cuts(const pf_params &p, int64_t gm) {
    const CounterRng rng(p.seed, (uint64_t)gm * 8u + kStreamCuts);
    std::vector<int64_t> cuts;
    const int want = p.ic_ncols - 1;
    for (uint64_t k = 0; (int)cuts.size() < want; ++k) {
        const int64_t cut = 1 + (int64_t)std::floor(rng.unif(k) * (double)(p.nx - 1));
        if (std::find(cuts.begin(), cuts.end(), cut) == cuts.end()) cuts.push_back(cut);
    }
    std::sort(cuts.begin(), cuts.end());
    return cuts;
}

// Initial fields of global member gm, global rows [y0, y0+rows), written row-major (row, i)
// into c/phi/rho (row a0 of SURVEY 8(a)).
void fill_initial(const pf_params &p, int64_t gm, int y0, int rows, double *c, double *phi,
                  double *rho) {
    const int nx = p.nx;
    const CounterRng rc(p.seed, (uint64_t)gm * 8u + kStreamC);
    const CounterRng rp(p.seed, (uint64_t)gm * 8u + kStreamPhi);
    const double delta = std::sqrt(2.0 * p.kappa_phi / p.W_phi);
    std::vector<int64_t> cuts;
    if (p.ic == PF_IC_COLUMNS) cuts = column_cuts(p, gm);
    std::vector<double> Hx(nx);
    for (int i = 0; i < nx; ++i) Hx[i] = p.ic_height + p.ic_amp * std::sin(2.0 * M_PI * (double)i / p.ic_wavelength);
    std::vector<double> ccol;
    if (p.ic == PF_IC_COLUMNS) {
        ccol.resize(nx);
        size_t q = 0;
        for (int i = 0; i < nx; ++i) {
            while (q < cuts.size() && (int64_t)i >= cuts[q]) ++q;
            ccol[i] = (q % 2 == 0) ? p.ic_c_lo : p.ic_c_hi;
        }
    }
    for (int r = 0; r < rows; ++r) {
        const int j = y0 + r;
        for (int i = 0; i < nx; ++i) {
            const uint64_t k = (uint64_t)j * (uint64_t)nx + (uint64_t)i;   // global cell index
            const size_t o = (size_t)r * nx + i;
            if (p.ic == PF_IC_NONE) {
                c[o] = phi[o] = rho[o] = 0.0;
                continue;
            }
            if (p.ic == PF_IC_FILM) {
                const double solid = (double)j < p.ic_height ? 1.0 : 0.0;
                phi[o] = solid + p.noise_phi * (2.0 * rp.unif(k) - 1.0);
                rho[o] = p.rho_in * (1.0 - solid);
            } else {
                const double ph = 0.5 * (1.0 - std::tanh(((double)j - Hx[i]) / delta));
                phi[o] = ph;
                rho[o] = p.rho_in * (1.0 - ph);
            }
            if (p.ic == PF_IC_COLUMNS)
                c[o] = ccol[i];
            else if (p.noise_c_gaussian)
                c[o] = p.ic_c0 + p.noise_c * rc.normal(k);
            else
                c[o] = p.ic_c0 + p.noise_c * (2.0 * rc.unif(k) - 1.0);
        }
    }
}

// Stability bound R-18.
double dt_limit(const pf_params &p) {
    const double Mc = std::max(std::max(std::fabs(p.M_A_bulk), std::fabs(p.M_B_bulk)),
                               std::max(std::fabs(p.M_A_surf), std::fabs(p.M_B_surf))) *
                      std::max(1.0, p.mob_hi);   // largest member multiplier (R-23)
    const double dx2 = p.dx * p.dx, dx4 = dx2 * dx2;
    // |f''| bound of the composition energy: 2 W_c (polynomial), 2|Omega| + T / (0.01 * 0.99) for
    // the regular solution on c in [0.05, 0.95] (R-28)
    const double fpp = p.fe_model == 1 ? 2.0 * std::fabs(p.omega) + p.temp_rs / (0.05 * 0.95) : 2.0 * p.W_c;
    const double a = Mc * (64.0 * p.kappa_c / dx4 + 8.0 * fpp / dx2);
    const double b = p.M_phi * (64.0 * p.kappa_phi / dx4 + 16.0 * p.W_phi / dx2);
    const double d = 8.0 * p.D_rho / dx2;
    return 1.6 / std::max(a, std::max(b, d));
}

pf::Coef make_coef(const pf_params &p) {
    pf::Coef K;
    const double dx2 = p.dx * p.dx;
    K.inv_dx2 = 1.0 / dx2;
    K.half_inv_dx2 = 0.5 / dx2;
    K.inv_2dx = 1.0 / (2.0 * p.dx);
    K.kc_dx2 = p.kappa_c / dx2;
    K.kp_dx2 = p.kappa_phi / dx2;
    K.W_c = p.W_c;
    K.W2c = 2.0 * p.W_c;
    K.W2p = 2.0 * p.W_phi;
    K.MBb = p.M_B_bulk;
    K.dMb = p.M_A_bulk - p.M_B_bulk;
    K.MBs = p.M_B_surf;
    K.dMs = p.M_A_surf - p.M_B_surf;
    K.mob = (p.mob_lo != 1.0 || p.mob_hi != 1.0) ? 2 : ((K.dMb != 0.0 || K.dMs != 0.0) ? 1 : 0);
    K.inv_sigma = 1.0 / p.sigma_surf;
    K.Mp_dx2 = p.M_phi / dx2;
    K.Dr_dx2 = p.D_rho / dx2;
    K.rho_in = p.rho_in;
    K.dx2 = dx2;
    K.half_kc = 0.5 * p.kappa_c;
    K.half_kp = 0.5 * p.kappa_phi;
    K.W_p = p.W_phi;
    K.fe = p.fe_model;
    K.omega = p.omega;
    K.temp = p.temp_rs;
    return K;
}

// Guard zones around every state buffer (checked builds, -DPF_GUARD_BYTES=N; 0 otherwise): filled
// with kGuardByte at creation and compared by pf_debug_guards, they catch any out-of-bounds global
// write of the stage kernels (compute-sanitizer is not available on the GPU pool).
#ifndef PF_GUARD_BYTES
#define PF_GUARD_BYTES 0
#endif
constexpr size_t kGuardBytes = PF_GUARD_BYTES;
constexpr unsigned char kGuardByte = 0x5A;

struct Slab {
    pf::Layout L{};
    void *U = nullptr;    // state u^n (also receives u^{n+1}: stage 2 updates in place)
    void *Us = nullptr;   // midpoint stage state u*
    void *alloc[2] = {nullptr, nullptr};   // the two allocations (guard zone + buffer + guard zone)
    size_t bytes = 0;                      // buffer bytes (without guards)
    double *partials = nullptr;
    double *diag = nullptr;   // members * kDiag
    pf::StreamPlan plan;      // streaming-kernel geometry and TMA tensor maps (plan.ok: in use)
    // halo_transport = 1 (B11, pf_halo.cu): the neighbours' buffers ([0] below, [1] above; IPC
    // mappings in the multi-process slab mode), their arrival counters this slab bumps, and this
    // slab's own counters ([0] arrivals from below, [1] from above)
    void *nbU[2] = {nullptr, nullptr}, *nbUs[2] = {nullptr, nullptr};
    unsigned *nbflag[2] = {nullptr, nullptr};
    unsigned *myflag = nullptr;
};

enum Mode { kSingle = 0, kLoopback = 1, kNccl = 2 };

// Grids up to this many cells (all members) use the persistent small-grid kernel by default.
constexpr int64_t kPersistentCells = 1 << 19;   // crossover ~2^20 (tools/small_grid_sweep.py)
// ... and up to this many the band kernel (one cluster per member) where its bands fit: it wins at
// 64^2 (1.00 vs 0.82 G), the one-barrier-per-step persistent kernel from 128^2 (3.15 vs 2.03 G;
// profiles/r2/small_grid_sweep_r2zf.jsonl)
constexpr int64_t kBandCells = 1 << 13;

}  // namespace

struct pf_ctx {
    pf_params p{};
    int mode = kSingle;
    int rank = 0, nranks = 1;
    size_t esz = 8;
    std::vector<Slab> slabs;
    int ny_host = 0;       // rows covered by the host buffers of get/set
    int y_host0 = 0;       // first global row of the host buffers
    cudaStream_t stream = nullptr;
    cudaStream_t comm_stream = nullptr;   // halo exchange, overlapped with interior compute
    cudaEvent_t ev_band = nullptr, ev_xchg = nullptr;
    bool overlap = false;                 // band / exchange / interior schedule in use
    bool fused = false;                   // one-pass step kernel in use (kernel_path 5)
    bool persistent = false;              // small-grid cooperative tile kernel (kernel_path 7)
    unsigned *pflags = nullptr;           // persistent step kernel: per-tile step flags (neighbour sync)
    uint32_t pepoch = 0;                  // ... steps its flags have counted so far
    bool band = false;                    // small-grid band kernel (kernel_path 6 / auto, pf_band.cu)
    pf::BandPlan bplan;
    ncclComm_t comm = nullptr;
    // halo_transport = 1 (B11): arrival counters (2 per slab), exchanges issued so far, blocks per
    // push (= counter increments per exchange and direction), IPC mappings to close
    bool peer = false;
    bool nccl_self = false;   // halo_transport = 2: loopback slabs exchanging through ncclSend / ncclRecv to self
    unsigned *xflags = nullptr;
    uint32_t xepoch = 0;
    int xblocks = 0;
    std::vector<void *> ipc_open;
    void *vel = nullptr;   // [members][2] in the storage precision
    double *h_diag = nullptr;
    double *staging = nullptr;
    size_t staging_n = 0;
    pf::Coef K{};
    int64_t steps = 0;
    double t = 0.0;
    bool blown = false;
    std::string err;
    int64_t launches = 0;
    // pf_run_host pipeline: copy streams and per-chunk events
    cudaStream_t h2d = nullptr, d2h = nullptr;
    std::vector<cudaEvent_t> ev_in, ev_done;
    // pf_trajectory: two device snapshot buffers, copy-done events
    double *snap[2] = {nullptr, nullptr};
    size_t snap_n = 0;
    cudaEvent_t ev_snap[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr};
    // CUDA graph of graph_steps steps
    cudaGraphExec_t gexec = nullptr;
    int gsteps = 0;
    // profiling
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_rec;
};

namespace {

pf_status set_err(pf_ctx *c, pf_status s, const std::string &m) {
    if (c) c->err = m;
    else g_create_error = m;
    return s;
}

#define CK(ctx, call)                                                                           \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            return set_err(ctx, PF_ERR_CUDA, fmt("%s failed: %s (%s:%d)", #call,                \
                                                 cudaGetErrorString(e_), __FILE__, __LINE__));  \
    } while (0)

#define NK(ctx, call)                                                                           \
    do {                                                                                        \
        ncclResult_t r_ = (call);                                                               \
        if (r_ != ncclSuccess)                                                                  \
            return set_err(ctx, PF_ERR_NCCL, fmt("%s failed: %s (%s:%d)", #call,                \
                                                 ncclGetErrorString(r_), __FILE__, __LINE__));  \
    } while (0)

pf_status validate(const pf_params *p, std::string &why) {
    if (!p) { why = "params is NULL"; return PF_ERR_ARG; }
    if (p->abi_version != PF_ABI_VERSION) {
        why = fmt("abi_version %u != %u", p->abi_version, PF_ABI_VERSION);
        return PF_ERR_ABI;
    }
    if (p->nx < 8 || p->ny < 8) { why = fmt("grid %dx%d: nx, ny must be >= 8 (S:152)", p->nx, p->ny); return PF_ERR_ARG; }
    if ((int64_t)p->nx * p->ny > (int64_t)1 << 31) { why = "grid larger than 2^31 cells"; return PF_ERR_ARG; }
    if (p->n_members < 1) { why = "n_members must be >= 1"; return PF_ERR_ARG; }
    if (p->member_offset < 0) { why = "member_offset must be >= 0"; return PF_ERR_ARG; }
    if (p->precision != PF_F64 && p->precision != PF_F32) { why = "precision must be PF_F64 or PF_F32"; return PF_ERR_ARG; }
    if (!(p->dx > 0) || !(p->dt > 0) || !std::isfinite(p->dx) || !std::isfinite(p->dt)) { why = "dx and dt must be finite and > 0"; return PF_ERR_ARG; }
    if (!(p->sigma_surf > 0)) { why = "sigma_surf must be > 0"; return PF_ERR_ARG; }
    if (p->kappa_c < 0 || p->kappa_phi < 0 || p->M_phi < 0 || p->D_rho < 0) { why = "kappa, M_phi, D_rho must be >= 0"; return PF_ERR_ARG; }
    if (p->M_A_bulk < 0 || p->M_B_bulk < 0 || p->M_A_surf < 0 || p->M_B_surf < 0) { why = "mobilities must be >= 0"; return PF_ERR_ARG; }
    if (p->check_every < 1) { why = "check_every must be >= 1"; return PF_ERR_ARG; }
    if (p->graph_steps < 0) { why = "graph_steps must be >= 0"; return PF_ERR_ARG; }
    if (p->fe_model != 0 && p->fe_model != 1) { why = "fe_model must be 0 or 1"; return PF_ERR_ARG; }
    if (p->fe_model == 1 && !(p->temp_rs >= 0)) { why = "temp_rs must be >= 0"; return PF_ERR_ARG; }
    if (!(p->noise_rho >= 0) || !std::isfinite(p->noise_rho)) { why = "noise_rho must be finite and >= 0"; return PF_ERR_ARG; }
    if (!(p->mob_lo > 0) || !(p->mob_hi >= p->mob_lo)) { why = "need 0 < mob_lo <= mob_hi"; return PF_ERR_ARG; }
    if (p->overlap_halo != 0 && p->overlap_halo != 1) { why = "overlap_halo must be 0 or 1"; return PF_ERR_ARG; }
    if (p->halo_transport < 0 || p->halo_transport > 2) { why = "halo_transport must be 0, 1 or 2"; return PF_ERR_ARG; }
    if (p->kernel_path < 0 || p->kernel_path > 7) { why = "kernel_path must be 0 .. 7"; return PF_ERR_ARG; }
    if (p->kernel_path == 2 || p->kernel_path == 4) { why = "kernel_path 2 and 4 (retired) are not available"; return PF_ERR_ARG; }
    if ((p->kernel_path == 3 || p->kernel_path == 5) && !(p->nx % 4 == 0 && p->nx >= 16)) { why = "streaming kernels need nx % 4 == 0 and nx >= 16"; return PF_ERR_ARG; }
    if (p->ic < PF_IC_FILM || p->ic > PF_IC_NONE) { why = "unknown ic"; return PF_ERR_ARG; }
    if ((p->ic == PF_IC_ROUGH_SUBSTRATE || p->ic == PF_IC_COLUMNS) && !(p->W_phi > 0)) { why = "tanh recipes need W_phi > 0"; return PF_ERR_ARG; }
    if (p->ic == PF_IC_ROUGH_SUBSTRATE && !(p->ic_wavelength != 0)) { why = "ic_wavelength must be != 0"; return PF_ERR_ARG; }
    if (p->ic == PF_IC_COLUMNS && (p->ic_ncols < 1 || p->ic_ncols > p->nx)) { why = "ic_ncols must be in [1, nx]"; return PF_ERR_ARG; }
    const double lim = dt_limit(*p);
    if (p->dt > lim) {
        why = fmt("dt = %g exceeds the stability bound %g (R-18)", p->dt, lim);
        return PF_ERR_UNSTABLE_DT;
    }
    return PF_OK;
}

void destroy(pf_ctx *c) {
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->gexec) cudaGraphExecDestroy(c->gexec);
    for (auto &s : c->slabs) {
        cudaFree(s.alloc[0]);
        cudaFree(s.alloc[1]);
        cudaFree(s.partials);
        cudaFree(s.diag);
    }
    cudaFree(c->vel);
    cudaFree(c->pflags);
    cudaFree(c->staging);
    if (c->h_diag) cudaFreeHost(c->h_diag);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (auto &r : c->ev_rec) {
        cudaEventDestroy(r.second.first);
        cudaEventDestroy(r.second.second);
    }
    for (void *q : c->ipc_open) cudaIpcCloseMemHandle(q);
    cudaFree(c->xflags);
    if (c->comm) ncclCommDestroy(c->comm);
    if (c->ev_band) cudaEventDestroy(c->ev_band);
    if (c->ev_xchg) cudaEventDestroy(c->ev_xchg);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    for (auto e : c->ev_in) cudaEventDestroy(e);
    for (auto e : c->ev_done) cudaEventDestroy(e);
    if (c->h2d) cudaStreamDestroy(c->h2d);
    for (int b = 0; b < 2; ++b) {
        cudaFree(c->snap[b]);
        if (c->ev_snap[b]) cudaEventDestroy(c->ev_snap[b]);
        if (c->ev_copied[b]) cudaEventDestroy(c->ev_copied[b]);
    }
    if (c->d2h) cudaStreamDestroy(c->d2h);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

// ---------------------------------------------------------------------------------------
// halo exchange of one state buffer (which = 0: U, 1: Us)

void *buf_of(Slab &s, int which) { return which == 0 ? s.U : s.Us; }

// y-slab decomposition; see pf_halo_plan in pf.h for the meaning of out[].
bool halo_plan(int ny, int nranks, int rank, int out[8]) {
    if (nranks < 1 || rank < 0 || rank >= nranks || ny % nranks != 0 || ny / nranks < 2) return false;
    const int rows = ny / nranks;
    out[0] = rank * rows;
    out[1] = rows;
    out[2] = rank > 0 ? rank - 1 : -1;
    out[3] = rank < nranks - 1 ? rank + 1 : -1;
    out[4] = 0;          // rows [0, 2) go down
    out[5] = rows - 2;   // rows [rows-2, rows) go up
    out[6] = -2;         // ghost rows [-2, 0) come from below
    out[7] = rows;       // ghost rows [rows, rows+2) come from above
    return true;
}

// One neighbour relation over NCCL (inside the caller's group): rows [srow, srow + 2) of every
// field of every member of `from` go to `peer`, rows [rrow, rrow + 2) of `to` come from it -- full
// padded rows (ghost columns too), one send / receive pair per (member, field) in that order.
pf_status nccl_rows(pf_ctx *c, Slab &from, int srow, Slab &to, int rrow, int peer, int which, cudaStream_t st) {
    const ncclDataType_t dt = c->p.precision == PF_F64 ? ncclFloat64 : ncclFloat32;
    const size_t rowb = (size_t)from.L.pitch * c->esz, cnt = 2 * (size_t)from.L.pitch;
    const char *sb = (const char *)buf_of(from, which);
    char *rb = (char *)buf_of(to, which);
    for (int m = 0; m < from.L.members; ++m)
        for (int f = 0; f < 3; ++f) {
            const size_t off = ((size_t)m * from.L.mstride + (size_t)f * from.L.fstride) * c->esz;
            NK(c, ncclSend(sb + off + (size_t)(srow + 2) * rowb, cnt, dt, peer, c->comm, st));
            NK(c, ncclRecv(rb + off + (size_t)(rrow + 2) * rowb, cnt, dt, peer, c->comm, st));
        }
    return PF_OK;
}

pf_status exchange(pf_ctx *c, int which, cudaStream_t st) {
    Nvtx nv("pf halo exchange");
    if (c->mode == kSingle) return PF_OK;
    const size_t rowb = (size_t)c->slabs[0].L.pitch * c->esz;   // full padded rows (ghost columns too)
    if (c->peer) {   // B11: one push kernel per slab (pf_halo.cu); finish_exchange awaits the arrivals
        for (auto &s : c->slabs) {
            pf::HaloPush h{};
            h.src = (const char *)buf_of(s, which);
            for (int d = 0; d < 2; ++d) {
                h.dst[d] = (char *)(which == 0 ? s.nbU[d] : s.nbUs[d]);
                h.flag[d] = s.nbflag[d];
            }
            h.rowb = (int64_t)rowb;
            h.fstride_b = s.L.fstride * (int64_t)c->esz;
            h.rows = s.L.ny_loc;
            h.nchunks = 3 * s.L.members;
            CK(c, pf::launch_halo_push(h, st));
            if (h.dst[0] || h.dst[1]) c->launches += 1;
        }
        ++c->xepoch;
        return PF_OK;
    }
    pf_status stx = PF_OK;
    if (c->mode == kLoopback && c->nccl_self) {
        // halo_transport = 2: the slabs of this one-GPU context exchange through a 1-rank NCCL
        // communicator, every transfer a ncclSend to self followed by its ncclRecv from self (NCCL
        // matches the k-th send to a peer with the k-th receive from it), in one group -- the issue
        // code (nccl_rows: counts, types, row addressing, stream) is the one the multi-rank
        // transport runs, so it is exercised on a one-GPU box.
        const int P = (int)c->slabs.size();
        NK(c, ncclGroupStart());
        for (int s = 0; s + 1 < P; ++s) {
            Slab &lo = c->slabs[s], &hi = c->slabs[s + 1];
            if ((stx = nccl_rows(c, lo, lo.L.ny_loc - 2, hi, -2, 0, which, st)) != PF_OK) return stx;
            if ((stx = nccl_rows(c, hi, 0, lo, lo.L.ny_loc, 0, which, st)) != PF_OK) return stx;
        }
        NK(c, ncclGroupEnd());
        return PF_OK;
    }
    if (c->mode == kLoopback) {
        const int P = (int)c->slabs.size();
        for (int s = 0; s < P; ++s) {
            Slab &me = c->slabs[s];
            int plan[8];
            halo_plan(c->p.ny, P, s, plan);
            const size_t pitch = (size_t)me.L.fstride * c->esz;
            char *mine = (char *)buf_of(me, which);
            if (plan[2] >= 0) {    // ghost rows [-2, 0)  <-  slab below, rows [rows-2, rows)
                Slab &lo = c->slabs[plan[2]];
                const char *src = (const char *)buf_of(lo, which) + (size_t)(plan[5] + 2) * rowb;
                CK(c, cudaMemcpy2DAsync(mine + (size_t)(plan[6] + 2) * rowb, pitch, src, pitch, 2 * rowb,
                                        (size_t)3 * me.L.members, cudaMemcpyDeviceToDevice, st));
            }
            if (plan[3] >= 0) {    // ghost rows [rows, rows+2)  <-  slab above, rows [0, 2)
                Slab &hi = c->slabs[plan[3]];
                const char *src = (const char *)buf_of(hi, which) + (size_t)(plan[4] + 2) * rowb;
                CK(c, cudaMemcpy2DAsync(mine + (size_t)(plan[7] + 2) * rowb, pitch, src, pitch, 2 * rowb,
                                        (size_t)3 * me.L.members, cudaMemcpyDeviceToDevice, st));
            }
        }
        return PF_OK;
    }
    // NCCL: 2 full padded rows of every field of every member to / from each neighbour.
    Slab &me = c->slabs[0];
    int plan[8];
    halo_plan(c->p.ny, c->nranks, c->rank, plan);
    NK(c, ncclGroupStart());
    if (plan[2] >= 0 && (stx = nccl_rows(c, me, plan[4], me, plan[6], plan[2], which, st)) != PF_OK) return stx;
    if (plan[3] >= 0 && (stx = nccl_rows(c, me, plan[5], me, plan[7], plan[3], which, st)) != PF_OK) return stx;
    NK(c, ncclGroupEnd());
    return PF_OK;
}

// B11: `st` waits until every neighbour's push of the latest exchange has arrived (the arrival
// counters reach xepoch * xblocks; cyclic GEQ compare, so the 32-bit counters may wrap).
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValueFn wait_value_fn() {
    static WaitValueFn fn = nullptr;
    if (!fn) {
        void *q = nullptr;
        cudaDriverEntryPointQueryResult r;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &q, cudaEnableDefault, &r) == cudaSuccess &&
            r == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<WaitValueFn>(q);
    }
    return fn;
}

pf_status finish_exchange(pf_ctx *c, cudaStream_t st) {
    if (!c->peer) return PF_OK;
    WaitValueFn wv = wait_value_fn();
    if (!wv) return set_err(c, PF_ERR_CUDA, "cuStreamWaitValue32 is not available");
    const uint32_t want = c->xepoch * (uint32_t)c->xblocks;
    for (auto &s : c->slabs)
        for (int d = 0; d < 2; ++d)
            if (s.nbU[d]) {
                CUresult r = wv((CUstream)st, (CUdeviceptr)(s.myflag + d), want, CU_STREAM_WAIT_VALUE_GEQ);
                if (r != CUDA_SUCCESS) return set_err(c, PF_ERR_CUDA, fmt("cuStreamWaitValue32 failed (%d)", (int)r));
            }
    return PF_OK;
}

cudaEvent_t take_event(pf_ctx *c) {
    if (!c->ev_pool.empty()) {
        cudaEvent_t e = c->ev_pool.back();
        c->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Rows [r0, r1) minus [g0, g1) (a gap only on the pair path, see Layout::g0).
pf_status launch_rows(pf_ctx *c, Slab &s, int stage, int r0, int r1, bool capture, int g0 = 0, int g1 = 0) {
    if (r1 <= r0) return PF_OK;
    Nvtx nv(stage == 1 ? "pf stage 1 (u* = u + dt/2 R(u))" : "pf stage 2 (u = u + dt R(u*))");
    pf::Layout L = s.L;
    L.r0 = r0;
    L.r1 = r1;
    L.g0 = g0;
    L.g1 = g1;
    const void *in = stage == 1 ? s.U : s.Us;
    void *out = stage == 1 ? s.Us : s.U;
    const double coef = stage == 1 ? 0.5 * c->p.dt : c->p.dt;
    CK(c, pf::launch_stage(c->p.precision, L, s.plan, c->K, stage, in, s.U, out, c->vel, coef, c->stream));
    if (!capture) c->launches += pf::kStageLaunches;
    return PF_OK;
}

// One explicit-midpoint step for every slab: stage 1, exchange, stage 2, exchange.
// Slab modes with the overlap schedule: each stage first updates the two boundary
// bands (rows [0, 2) and [ny_loc-2, ny_loc)), the halo exchange of those rows then runs on the
// comm stream while the interior rows [2, ny_loc-2) are updated -- the interior reads no ghost
// row, so it never waits for the exchange -- and the next stage waits for the exchange.
pf_status one_step(pf_ctx *c, bool capture, int64_t step) {
    const bool prof = c->prof && !capture;
    if (c->p.noise_rho > 0.0)   // stochastic inflow of this step (R-27); never inside a graph
        for (auto &s : c->slabs) {
            CK(c, pf::launch_inflow(c->p.precision, s.L, c->p.rho_in, c->p.noise_rho, c->p.seed, c->p.member_offset,
                                    step, s.U, s.Us, c->stream));
            if (!capture) c->launches += 1;
        }
    if (c->fused) {   // one fused pass per step (kernel_path 5, single domain): U -> Us, then swap
        Slab &S = c->slabs[0];
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (prof) {
            e0 = take_event(c);
            e1 = take_event(c);
            CK(c, cudaEventRecord(e0, c->stream));
        }
        CK(c, pf::launch_fused(c->p.precision, S.L, S.plan, c->K, S.Us, c->vel, c->p.dt, c->stream));
        if (!capture) c->launches += 1;
        std::swap(S.U, S.Us);
        pf::swap_plan_buffers(S.plan);
        if (prof) {
            CK(c, cudaEventRecord(e1, c->stream));
            c->ev_rec.push_back({1, {e0, e1}});
        }
        return PF_OK;
    }
    for (int stage = 1; stage <= 2; ++stage) {
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (prof) {
            e0 = take_event(c);
            e1 = take_event(c);
            CK(c, cudaEventRecord(e0, c->stream));
        }
        const int which = stage == 1 ? 1 : 0;   // buffer written by this stage
        pf_status st = PF_OK;
        if (!c->overlap) {
            for (auto &s : c->slabs)
                if ((st = launch_rows(c, s, stage, 0, s.L.ny_loc, capture)) != PF_OK) return st;
            if (prof) CK(c, cudaEventRecord(e1, c->stream));
            if ((st = exchange(c, which, c->stream)) != PF_OK) return st;
            if ((st = finish_exchange(c, c->stream)) != PF_OK) return st;
        } else {
            for (auto &s : c->slabs) {
                if (s.plan.ok) {   // pair kernel: both bands in one launch (rows [2, ny_loc-2) skipped)
                    if ((st = launch_rows(c, s, stage, 0, s.L.ny_loc, capture, 2, s.L.ny_loc - 2)) != PF_OK) return st;
                    continue;
                }
                if ((st = launch_rows(c, s, stage, 0, 2, capture)) != PF_OK) return st;
                if ((st = launch_rows(c, s, stage, s.L.ny_loc - 2, s.L.ny_loc, capture)) != PF_OK) return st;
            }
            CK(c, cudaEventRecord(c->ev_band, c->stream));
            CK(c, cudaStreamWaitEvent(c->comm_stream, c->ev_band, 0));
            if ((st = exchange(c, which, c->comm_stream)) != PF_OK) return st;
            CK(c, cudaEventRecord(c->ev_xchg, c->comm_stream));
            for (auto &s : c->slabs)
                if ((st = launch_rows(c, s, stage, 2, s.L.ny_loc - 2, capture)) != PF_OK) return st;
            if (prof) CK(c, cudaEventRecord(e1, c->stream));
            CK(c, cudaStreamWaitEvent(c->stream, c->ev_xchg, 0));
            if ((st = finish_exchange(c, c->stream)) != PF_OK) return st;
        }
        if (prof) c->ev_rec.push_back({stage, {e0, e1}});
    }
    return PF_OK;
}

// PF_NCCL_SELF_GRAPH=1: the send-to-self exchanges of transport 2 captured into the step graphs
// (experiment knob; off, a transport-2 ctx launches directly like the multi-rank NCCL mode).
bool nccl_self_graph() {
    static const bool on = [] { const char *v = getenv("PF_NCCL_SELF_GRAPH"); return v && atoi(v) != 0; }();
    return on;
}

pf_status ensure_graph(pf_ctx *c) {
    const bool self_graph = nccl_self_graph();
    if (c->gexec || c->p.graph_steps <= 0 || c->mode == kNccl || c->peer || (c->nccl_self && !self_graph)) return PF_OK;
    cudaGraph_t g = nullptr;
    CK(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    pf_status st = PF_OK;
    for (int i = 0; i < c->p.graph_steps && st == PF_OK; ++i) st = one_step(c, true, 0);
    cudaError_t e = cudaStreamEndCapture(c->stream, &g);
    if (st != PF_OK) {
        if (g) cudaGraphDestroy(g);
        return st;
    }
    if (e != cudaSuccess) return set_err(c, PF_ERR_CUDA, fmt("graph capture failed: %s", cudaGetErrorString(e)));
    e = cudaGraphInstantiate(&c->gexec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return set_err(c, PF_ERR_CUDA, fmt("graph instantiate failed: %s", cudaGetErrorString(e)));
    c->gsteps = c->p.graph_steps;
    return PF_OK;
}

// Launch the diagnostics of every slab (device results in slab.diag).
pf_status run_diag(pf_ctx *c) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->prof) {
        e0 = take_event(c);
        e1 = take_event(c);
        CK(c, cudaEventRecord(e0, c->stream));
    }
    for (auto &s : c->slabs) {
        CK(c, pf::launch_diag(c->p.precision, s.L, c->K, s.U, s.partials, s.diag, c->stream));
        c->launches += pf::kDiagLaunches;
    }
    if (c->prof) {
        CK(c, cudaEventRecord(e1, c->stream));
        c->ev_rec.push_back({3, {e0, e1}});
    }
    return PF_OK;
}

// Gather the kDiag record of every member summed over slabs (slab order) / ranks (rank order)
// into host array out[members * kDiag].
pf_status gather_diag(pf_ctx *c, std::vector<double> &out) {
    const int M = c->p.n_members;
    const size_t n = (size_t)M * pf::kDiag;
    out.assign(n, 0.0);
    pf_status st = run_diag(c);
    if (st != PF_OK) return st;
    if (c->mode == kNccl) {
        double *dall = nullptr;
        CK(c, cudaMallocAsync((void **)&dall, n * c->nranks * sizeof(double), c->stream));
        NK(c, ncclAllGather(c->slabs[0].diag, dall, n, ncclFloat64, c->comm, c->stream));
        std::vector<double> h(n * c->nranks);
        CK(c, cudaMemcpyAsync(h.data(), dall, h.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaFreeAsync(dall, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
        for (int r = 0; r < c->nranks; ++r)
            for (size_t k = 0; k < n; ++k) out[k] += h[r * n + k];
        return PF_OK;
    }
    if (c->nccl_self) {   // every slab's record through the 1-rank communicator's all-gather
        const size_t P = c->slabs.size();
        double *dall = nullptr;
        CK(c, cudaMallocAsync((void **)&dall, n * P * sizeof(double), c->stream));
        for (size_t s = 0; s < P; ++s)
            NK(c, ncclAllGather(c->slabs[s].diag, dall + s * n, n, ncclFloat64, c->comm, c->stream));
        CK(c, cudaMemcpyAsync(c->h_diag, dall, n * P * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CK(c, cudaFreeAsync(dall, c->stream));
        CK(c, cudaStreamSynchronize(c->stream));
        for (size_t s = 0; s < P; ++s)
            for (size_t k = 0; k < n; ++k) out[k] += c->h_diag[s * n + k];
        return PF_OK;
    }
    for (size_t s = 0; s < c->slabs.size(); ++s)
        CK(c, cudaMemcpyAsync(c->h_diag + s * n, c->slabs[s].diag, n * sizeof(double),
                              cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    for (size_t s = 0; s < c->slabs.size(); ++s)
        for (size_t k = 0; k < n; ++k) out[k] += c->h_diag[s * n + k];
    return PF_OK;
}

pf_status check_blowup(pf_ctx *c, int64_t from, int64_t to) {
    Nvtx nv("pf diagnostics / blow-up check");
    std::vector<double> d;
    pf_status st = gather_diag(c, d);
    if (st != PF_OK) return st;
    double nf[3] = {0, 0, 0};
    int worst = -1;
    for (int m = 0; m < c->p.n_members; ++m) {
        for (int f = 0; f < 3; ++f) nf[f] += d[(size_t)m * pf::kDiag + 5 + f];
        if (worst < 0 && d[(size_t)m * pf::kDiag + 4] > 0) worst = m;
    }
    if (nf[0] + nf[1] + nf[2] > 0) {
        c->blown = true;
        std::string fields;
        const char *names[3] = {"c", "phi", "rho"};
        for (int f = 0; f < 3; ++f)
            if (nf[f] > 0) fields += fmt("%s%s (%.0f cells)", fields.empty() ? "" : ", ", names[f], nf[f]);
        return set_err(c, PF_ERR_BLOWUP,
                       fmt("blow-up: non-finite %s in steps (%lld, %lld], first member %d", fields.c_str(),
                           (long long)from, (long long)to, worst + c->p.member_offset));
    }
    return PF_OK;
}

// B11 (halo_transport = 1): arrival counters, and the neighbours' buffers and counters -- device
// pointers of the other slabs in loopback, CUDA-IPC mappings of the neighbouring ranks' allocations
// (handles all-gathered over the NCCL communicator) in the multi-process slab mode.  Called after
// the initial fields and ghost frames are complete: the all-gather is also the barrier that keeps
// a neighbour's first push behind this rank's fill_ghosts.
pf_status setup_peer(pf_ctx *c) {
    const int nsl = (int)c->slabs.size();
    const size_t nflag = 2 * (size_t)nsl + 2;   // 2 per slab + the barrier word of peer_barrier
    CK(c, cudaMalloc((void **)&c->xflags, nflag * sizeof(unsigned)));
    CK(c, cudaMemsetAsync(c->xflags, 0, nflag * sizeof(unsigned), c->stream));
    c->xblocks = pf::halo_push_blocks(c->p.n_members, (int64_t)c->slabs[0].L.pitch * (int64_t)c->esz);
    for (int s = 0; s < nsl; ++s) c->slabs[s].myflag = c->xflags + 2 * s;
    if (c->mode == kLoopback) {
        for (int s = 0; s < nsl; ++s) {
            Slab &S = c->slabs[s];
            if (s > 0) {
                S.nbU[0] = c->slabs[s - 1].U;
                S.nbUs[0] = c->slabs[s - 1].Us;
                S.nbflag[0] = c->slabs[s - 1].myflag + 1;
            }
            if (s < nsl - 1) {
                S.nbU[1] = c->slabs[s + 1].U;
                S.nbUs[1] = c->slabs[s + 1].Us;
                S.nbflag[1] = c->slabs[s + 1].myflag + 0;
            }
        }
        return PF_OK;
    }
    // Every rank takes part in both collectives below even when one of its own steps failed, and
    // the all-reduce of the ok bits makes the ranks agree: a rank whose mapping failed must not
    // leave its neighbours waiting forever for pushes that never come.
    struct Rec {
        cudaIpcMemHandle_t h[3];   // U allocation, Us allocation, counters
        int32_t ok;
        int32_t pad[15];
    };
    Slab &S = c->slabs[0];
    Rec mine{};
    std::string why;
    mine.ok = cudaIpcGetMemHandle(&mine.h[0], S.alloc[0]) == cudaSuccess &&
              cudaIpcGetMemHandle(&mine.h[1], S.alloc[1]) == cudaSuccess &&
              cudaIpcGetMemHandle(&mine.h[2], c->xflags) == cudaSuccess;
    if (!mine.ok) why = fmt("cudaIpcGetMemHandle: %s", cudaGetErrorString(cudaGetLastError()));
    const int P = c->nranks;
    std::vector<Rec> all(P);
    Rec *d = nullptr;
    int32_t *okw = nullptr;
    CK(c, cudaMalloc((void **)&d, (size_t)(P + 1) * sizeof(Rec)));
    CK(c, cudaMalloc((void **)&okw, sizeof(int32_t)));
    auto collective = [&](ncclResult_t r) {
        if (r != ncclSuccess) why = fmt("NCCL (peer setup): %s", ncclGetErrorString(r));
        return r == ncclSuccess;
    };
    bool good = cudaMemcpyAsync(d + P, &mine, sizeof(Rec), cudaMemcpyHostToDevice, c->stream) == cudaSuccess &&
                collective(ncclAllGather(d + P, d, sizeof(Rec), ncclUint8, c->comm, c->stream)) &&
                cudaMemcpyAsync(all.data(), d, (size_t)P * sizeof(Rec), cudaMemcpyDeviceToHost, c->stream) ==
                    cudaSuccess &&
                cudaStreamSynchronize(c->stream) == cudaSuccess;
    for (int dd = 0; good && dd < 2; ++dd) {
        const int nb = dd == 0 ? c->rank - 1 : c->rank + 1;
        if (nb < 0 || nb >= P || !all[nb].ok) continue;
        void *q[3] = {nullptr, nullptr, nullptr};
        for (int k = 0; k < 3 && good; ++k) {
            cudaError_t e = cudaIpcOpenMemHandle(&q[k], all[nb].h[k], cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                why = fmt("cudaIpcOpenMemHandle (rank %d): %s", nb, cudaGetErrorString(e));
                good = false;
            } else {
                c->ipc_open.push_back(q[k]);
            }
        }
        if (!good) break;
        S.nbU[dd] = (char *)q[0] + kGuardBytes;
        S.nbUs[dd] = (char *)q[1] + kGuardBytes;
        S.nbflag[dd] = (unsigned *)q[2] + (dd == 0 ? 1 : 0);
    }
    int32_t ok = good && mine.ok ? 1 : 0, all_ok = 0;
    bool agreed = cudaMemcpyAsync(okw, &ok, sizeof ok, cudaMemcpyHostToDevice, c->stream) == cudaSuccess &&
                  collective(ncclAllReduce(okw, okw, 1, ncclInt32, ncclMin, c->comm, c->stream)) &&
                  cudaMemcpyAsync(&all_ok, okw, sizeof all_ok, cudaMemcpyDeviceToHost, c->stream) == cudaSuccess &&
                  cudaStreamSynchronize(c->stream) == cudaSuccess;
    cudaFree(d);
    cudaFree(okw);
    if (!agreed || !all_ok) {
        cudaGetLastError();
        return set_err(c, PF_ERR_CUDA, "peer halo transport setup failed" +
                                           (why.empty() ? std::string(" on another rank") : ": " + why));
    }
    return PF_OK;
}

// Multi-process peer transport: a device-side barrier on c->stream (a one-word all-reduce) that
// keeps the next push behind every rank's host writes and fill_ghosts (pf_set_fields).
pf_status peer_barrier(pf_ctx *c) {
    if (!c->peer || c->mode != kNccl) return PF_OK;
    unsigned *w = c->xflags + 2 * c->slabs.size();
    NK(c, ncclAllReduce(w, w, 1, ncclUint32, ncclSum, c->comm, c->stream));
    return PF_OK;
}

pf_status create_common(const pf_params *p, int mode, int rank, int nranks, const uint8_t *uid,
                        pf_ctx **out) {
    if (!out) return set_err(nullptr, PF_ERR_ARG, "out is NULL");
    *out = nullptr;
    std::string why;
    pf_status st = validate(p, why);
    if (st != PF_OK) return set_err(nullptr, st, why);
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_err(nullptr, PF_ERR_ARG, "bad rank / nranks");
    if (p->ny % nranks != 0 || p->ny / nranks < 2)
        return set_err(nullptr, PF_ERR_ARG, fmt("ny = %d must be a multiple of %d with >= 2 rows per slab", p->ny, nranks));
    pf_ctx *c = new pf_ctx();
    c->p = *p;
    c->mode = mode;
    c->rank = rank;
    c->nranks = nranks;
    c->esz = p->precision == PF_F64 ? 8 : 4;
    c->K = make_coef(*p);
    auto fail = [&](pf_status s) {
        g_create_error = c->err;
        destroy(c);
        return s;
    };
    cudaError_t e = cudaSetDevice(p->device);
    if (e != cudaSuccess) {
        c->err = fmt("cudaSetDevice(%d): %s", p->device, cudaGetErrorString(e));
        return fail(PF_ERR_CUDA);
    }
    e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess && mode != kSingle) e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess && mode != kSingle) e = cudaEventCreateWithFlags(&c->ev_band, cudaEventDisableTiming);
    if (e == cudaSuccess && mode != kSingle) e = cudaEventCreateWithFlags(&c->ev_xchg, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        c->err = fmt("cudaStreamCreate: %s", cudaGetErrorString(e));
        return fail(PF_ERR_CUDA);
    }
    // slabs
    const int nsl = mode == kLoopback ? nranks : 1;
    const int rows = p->ny / nranks;
    for (int s = 0; s < nsl; ++s) {
        Slab sl;
        sl.L.nx = p->nx;
        sl.L.ny = p->ny;
        sl.L.ny_loc = rows;
        sl.L.y0 = (mode == kLoopback ? s : rank) * rows;
        sl.L.members = p->n_members;
        sl.L.path = p->kernel_path;
        sl.L.gx = (int)(32 / c->esz);   // 32 B: 128-bit output pairs start on 32 B sectors
        sl.L.pitch = p->nx + 2 * sl.L.gx;
        sl.L.fstride = (int64_t)(rows + 4) * sl.L.pitch;
        sl.L.mstride = 3 * sl.L.fstride;
        sl.L.r0 = 0;
        sl.L.r1 = rows;
        sl.L.m0 = 0;
        const size_t bytes = (size_t)sl.L.mstride * p->n_members * c->esz;
        c->slabs.push_back(sl);
        Slab &S = c->slabs.back();
        S.bytes = bytes;
        if (cudaMalloc(&S.alloc[0], bytes + 2 * kGuardBytes) != cudaSuccess ||
            cudaMalloc(&S.alloc[1], bytes + 2 * kGuardBytes) != cudaSuccess) {
            cudaGetLastError();
            c->err = fmt("cudaMalloc of 2 x %zu bytes failed", bytes);
            return fail(PF_ERR_NOMEM);
        }
        S.U = (char *)S.alloc[0] + kGuardBytes;
        S.Us = (char *)S.alloc[1] + kGuardBytes;
        for (int b = 0; b < 2; ++b) {
            if (kGuardBytes) cudaMemsetAsync(S.alloc[b], kGuardByte, bytes + 2 * kGuardBytes, c->stream);
        }
        cudaMemsetAsync(S.U, 0, bytes, c->stream);
        cudaMemsetAsync(S.Us, 0, bytes, c->stream);
        e = pf::make_stream_plan(p->precision, S.L, S.U, S.Us, S.plan);
        if (e != cudaSuccess) {
            c->err = fmt("TMA tensor-map setup failed: %s", cudaGetErrorString(e));
            return fail(PF_ERR_CUDA);
        }
        const size_t pb = (size_t)p->n_members * pf::diag_blocks(S.L) * pf::kDiag * sizeof(double);
        if (cudaMalloc((void **)&S.partials, pb) != cudaSuccess ||
            cudaMalloc((void **)&S.diag, (size_t)p->n_members * pf::kDiag * sizeof(double)) != cudaSuccess) {
            cudaGetLastError();
            c->err = "cudaMalloc of diagnostics scratch failed";
            return fail(PF_ERR_NOMEM);
        }
    }
    // overlap schedule: slab modes, bands of 2 rows leave an interior of >= 4 rows
    c->overlap = mode != kSingle && rows >= 8 && p->overlap_halo != 0;
    c->fused = mode == kSingle && p->kernel_path == 5 && c->slabs[0].plan.fused;
    {   // small grids: one cooperative launch per check interval instead of two launches per step --
        // the band kernel (state in shared memory, neighbour flags) where its bands fit, else the
        // persistent tile kernel (grid barriers)
        const int64_t cells = (int64_t)p->n_members * p->nx * p->ny;
        const bool small = mode == kSingle && !(p->noise_rho > 0.0);
        if (small && (p->kernel_path == 6 || (p->kernel_path == 0 && cells <= kBandCells)))
            c->band = pf::make_band_plan(p->precision, c->slabs[0].L, c->bplan);
        if (p->kernel_path == 6 && !c->band) {
            c->err = "kernel_path 6: the band kernel needs a single-domain ctx without inflow noise, ny >= 2 and a band "
                     "(ny / min(16, ny / 2) rows) that fits one block's shared memory and 2048 cells";
            return fail(PF_ERR_ARG);
        }
        c->persistent = small && !c->band &&
                        (p->kernel_path == 7 || (p->kernel_path == 0 && cells <= kPersistentCells));
        if (c->persistent) {   // one flag per tile of the finest tiling (32 x 4)
            const size_t nflags = (size_t)((p->nx + 31) / 32) * ((p->ny + 3) / 4) * p->n_members;
            if (cudaMalloc((void **)&c->pflags, nflags * sizeof(unsigned)) != cudaSuccess ||
                cudaMemsetAsync(c->pflags, 0, nflags * sizeof(unsigned), c->stream) != cudaSuccess) {
                cudaGetLastError();
                c->err = "cudaMalloc of the persistent kernel's tile flags failed";
                return fail(PF_ERR_NOMEM);
            }
        }
    }
    c->ny_host = mode == kNccl ? rows : p->ny;
    c->y_host0 = mode == kNccl ? rank * rows : 0;
    if (cudaMallocHost((void **)&c->h_diag, nsl * (size_t)p->n_members * pf::kDiag * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        c->err = "cudaMallocHost failed";
        return fail(PF_ERR_NOMEM);
    }
    // per-member records: velocity (R-10, R-15, R-21) and mobilities (R-6, R-23), pf_cell.cuh
    {
        constexpr int W = pf::kMembStride;
        std::vector<double> v(W * (size_t)p->n_members);
        for (int m = 0; m < p->n_members; ++m) {
            const int64_t gm = (int64_t)p->member_offset + m;
            double *q = &v[W * (size_t)m];
            member_velocity(*p, gm, q[0], q[1]);
            double mob[4];
            member_mobility(*p, gm, mob);   // M_A^bulk, M_B^bulk, M_A^surf, M_B^surf
            q[2] = mob[1];
            q[3] = mob[0] - mob[1];
            q[4] = mob[3];
            q[5] = mob[2] - mob[3];
        }
        std::vector<float> vf(v.begin(), v.end());
        if (cudaMalloc(&c->vel, v.size() * c->esz) != cudaSuccess) {
            cudaGetLastError();
            c->err = "cudaMalloc failed";
            return fail(PF_ERR_NOMEM);
        }
        e = cudaMemcpy(c->vel, c->esz == 8 ? (const void *)v.data() : (const void *)vf.data(),
                       v.size() * c->esz, cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            c->err = fmt("cudaMemcpy: %s", cudaGetErrorString(e));
            return fail(PF_ERR_CUDA);
        }
    }
    if (mode == kNccl && p->halo_transport == 2) {
        c->err = "halo_transport 2 (NCCL send to self) is the one-GPU loopback stand-in: pf_create with n_slabs > 1";
        return fail(PF_ERR_ARG);
    }
    c->nccl_self = mode == kLoopback && p->halo_transport == 2;
    if (c->nccl_self) {   // a communicator of this one rank
        ncclUniqueId id;
        ncclResult_t r = ncclGetUniqueId(&id);
        if (r == ncclSuccess) r = ncclCommInitRank(&c->comm, 1, id, 0);
        if (r != ncclSuccess) {
            c->err = fmt("ncclCommInitRank (1 rank): %s", ncclGetErrorString(r));
            return fail(PF_ERR_NCCL);
        }
    }
    if (mode == kNccl) {
        ncclUniqueId id;
        std::memcpy(&id, uid, sizeof id);
        ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
        if (r != ncclSuccess) {
            c->err = fmt("ncclCommInitRank: %s", ncclGetErrorString(r));
            return fail(PF_ERR_NCCL);
        }
    }
    // The memsets above ran on the non-blocking ctx stream, the uploads below use synchronous
    // copies on the legacy stream (which does not order against non-blocking streams): fence both
    // sides explicitly.
    e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        c->err = fmt("create: %s", cudaGetErrorString(e));
        return fail(PF_ERR_CUDA);
    }
    // initial conditions, generated on the host per member and slab (row a0)
    for (auto &S : c->slabs) {
        const size_t n = (size_t)S.L.ny_loc * p->nx;
        std::vector<double> hc(n), hp(n), hr(n);
        for (int m = 0; m < p->n_members; ++m) {
            fill_initial(*p, (int64_t)p->member_offset + m, S.L.y0, S.L.ny_loc, hc.data(), hp.data(), hr.data());
            const double *src[3] = {hc.data(), hp.data(), hr.data()};
            for (int f = 0; f < 3; ++f) {
                char *dst = (char *)S.U + ((size_t)m * S.L.mstride + (size_t)f * S.L.fstride + (size_t)S.L.at(0, 0)) * c->esz;
                const size_t dp = (size_t)S.L.pitch * c->esz, w = (size_t)p->nx * c->esz;
                if (c->esz == 8) {
                    e = cudaMemcpy2D(dst, dp, src[f], w, w, S.L.ny_loc, cudaMemcpyHostToDevice);
                } else {
                    std::vector<float> tmp(src[f], src[f] + n);
                    e = cudaMemcpy2D(dst, dp, tmp.data(), w, w, S.L.ny_loc, cudaMemcpyHostToDevice);
                }
                if (e != cudaSuccess) {
                    c->err = fmt("cudaMemcpy: %s", cudaGetErrorString(e));
                    return fail(PF_ERR_CUDA);
                }
            }
        }
    }
    e = cudaDeviceSynchronize();   // every upload complete before the first kernel on c->stream
    if (e != cudaSuccess) {
        c->err = fmt("create: %s", cudaGetErrorString(e));
        return fail(PF_ERR_CUDA);
    }
    for (auto &S : c->slabs) {   // ghost frames of both buffers (rho reservoir rows in Us too)
        e = pf::launch_fill_ghosts(p->precision, S.L, p->rho_in, S.U, c->stream);
        if (e == cudaSuccess) e = pf::launch_fill_ghosts(p->precision, S.L, p->rho_in, S.Us, c->stream);
        if (e != cudaSuccess) {
            c->err = fmt("fill_ghosts: %s", cudaGetErrorString(e));
            return fail(PF_ERR_CUDA);
        }
        c->launches += 2 * pf::kFillLaunches;
    }
    c->peer = mode != kSingle && p->halo_transport == 1;
    if (c->peer && (st = setup_peer(c)) != PF_OK) return fail(st);
    st = exchange(c, 0, c->stream);
    if (st == PF_OK) st = finish_exchange(c, c->stream);
    if (st != PF_OK) return fail(st);
    e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        c->err = fmt("create: %s", cudaGetErrorString(e));
        return fail(PF_ERR_CUDA);
    }
    *out = c;
    return PF_OK;
}

pf_status check_member(pf_ctx *c, int32_t member, int &m0, int &nm) {
    if (member == -1) {
        m0 = 0;
        nm = c->p.n_members;
        return PF_OK;
    }
    if (member < 0 || member >= c->p.n_members) return set_err(c, PF_ERR_ARG, fmt("member %d out of range", member));
    m0 = member;
    nm = 1;
    return PF_OK;
}

pf_status ensure_staging(pf_ctx *c, size_t n) {
    if (c->staging_n >= n) return PF_OK;
    cudaFree(c->staging);
    c->staging = nullptr;
    c->staging_n = 0;
    if (cudaMalloc((void **)&c->staging, n * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        return set_err(c, PF_ERR_NOMEM, "cudaMalloc of staging buffer failed");
    }
    c->staging_n = n;
    return PF_OK;
}

}  // namespace

// =========================================================================================
extern "C" {

pf_status pf_default_params(int32_t cfg, pf_params *o) {
    if (!o) return set_err(nullptr, PF_ERR_ARG, "out is NULL");
    if (cfg < 1 || cfg > 5) return set_err(nullptr, PF_ERR_ARG, fmt("no preset %d (1..5)", cfg));
    pf_params p;
    std::memset(&p, 0, sizeof p);
    p.abi_version = PF_ABI_VERSION;
    p.n_members = 1;
    p.precision = PF_F64;
    p.dx = 1.0;
    p.dt = 1e-3;
    p.kappa_c = p.kappa_phi = 1.0;
    p.W_c = p.W_phi = 1.0;
    p.sigma_surf = 0.5;
    p.M_phi = 1.0;
    p.D_rho = 1.0;
    p.rho_in = 1.0;
    p.v0 = 0.5;
    p.theta_deg = 90.0;
    p.rate_lo = p.rate_hi = 1.0;
    p.mob_lo = p.mob_hi = 1.0;
    p.ic_wavelength = 32.0;
    p.ic_c0 = 0.5;
    p.ic_c_lo = 0.2;
    p.ic_c_hi = 0.8;
    p.check_every = 100;
    p.seed = (uint64_t)cfg;
    p.graph_steps = 0;
    p.overlap_halo = 1;
    if (cfg == 1) {             // configs[0]: 64^2 film, all mobilities 1
        p.nx = p.ny = 64;
        p.M_A_bulk = p.M_B_bulk = p.M_A_surf = p.M_B_surf = 1.0;
        p.ic = PF_IC_FILM;
        p.ic_height = 16.0;
        p.noise_c = 0.05;
        p.noise_phi = 0.01;
        p.graph_steps = 50;
    } else {                    // configs[1..4]: M_c / M_phi = 10
        p.M_A_bulk = p.M_B_bulk = p.M_A_surf = p.M_B_surf = 10.0;
        p.ic = PF_IC_ROUGH_SUBSTRATE;
        p.ic_height = 32.0;
        p.ic_amp = 2.0;
        p.noise_c = 0.05;
        p.noise_c_gaussian = 1;
        if (cfg == 2) {
            p.nx = p.ny = 256;
            p.graph_steps = 50;
        } else if (cfg == 3) {
            p.nx = p.ny = 512;
            p.n_members = 64;
            p.rate_lo = 0.5;
            p.rate_hi = 2.0;
        } else if (cfg == 4) {
            p.nx = p.ny = 4096;
            p.ic_height = 512.0;
        } else {
            p.nx = p.ny = 8192;
            p.precision = PF_F32;
            p.ic = PF_IC_COLUMNS;
            p.ic_height = 4096.0;
            p.ic_amp = 0.0;
            p.ic_ncols = 64;
            p.noise_c = 0.0;
            p.noise_c_gaussian = 0;
        }
    }
    *o = p;
    return PF_OK;
}

uint32_t pf_params_size(void) { return (uint32_t)sizeof(pf_params); }

pf_status pf_initial_fields(const pf_params *p, int64_t member, int32_t y0, int32_t rows,
                            double *fc, double *fp, double *fr) {
    if (!p || !fc || !fp || !fr) return set_err(nullptr, PF_ERR_ARG, "NULL argument");
    if (p->nx < 1 || y0 < 0 || rows < 0 || member < 0) return set_err(nullptr, PF_ERR_ARG, "bad extent");
    if (p->ic == PF_IC_COLUMNS && (p->ic_ncols < 1 || p->ic_ncols > p->nx))
        return set_err(nullptr, PF_ERR_ARG, "ic_ncols must be in [1, nx]");
    fill_initial(*p, member, y0, rows, fc, fp, fr);
    return PF_OK;
}

pf_status pf_member_velocity(const pf_params *p, int64_t member, double *vx, double *vy) {
    if (!p || !vx || !vy || member < 0) return set_err(nullptr, PF_ERR_ARG, "bad argument");
    member_velocity(*p, member, *vx, *vy);
    return PF_OK;
}

pf_status pf_member_mobility(const pf_params *p, int64_t member, double out[4]) {
    if (!p || !out || member < 0) return set_err(nullptr, PF_ERR_ARG, "bad argument");
    member_mobility(*p, member, out);
    return PF_OK;
}

pf_status pf_inflow_row(const pf_params *p, int64_t member, int64_t step, double *out) {
    if (!p || !out || member < 0 || step < 0 || p->nx < 1) return set_err(nullptr, PF_ERR_ARG, "bad argument");
    for (int i = 0; i < p->nx; ++i) out[i] = p->noise_rho > 0.0 ? inflow_host(*p, member, step, i) : p->rho_in;
    return PF_OK;
}

pf_status pf_dt_limit(const pf_params *p, double *dt_max) {
    if (!p || !dt_max) return set_err(nullptr, PF_ERR_ARG, "NULL argument");
    *dt_max = dt_limit(*p);
    return PF_OK;
}

pf_status pf_halo_plan(int32_t ny, int32_t nranks, int32_t rank, int32_t out[8]) {
    if (!out) return set_err(nullptr, PF_ERR_ARG, "out is NULL");
    int o[8];
    if (!halo_plan(ny, nranks, rank, o))
        return set_err(nullptr, PF_ERR_ARG, fmt("no slab plan for ny = %d, nranks = %d, rank = %d", ny, nranks, rank));
    for (int k = 0; k < 8; ++k) out[k] = o[k];
    return PF_OK;
}

pf_status pf_create(const pf_params *p, pf_ctx **out) { return create_common(p, kSingle, 0, 1, nullptr, out); }

pf_status pf_create_loopback(const pf_params *p, int32_t nslabs, pf_ctx **out) {
    if (nslabs < 1) return set_err(nullptr, PF_ERR_ARG, "nslabs must be >= 1");
    return create_common(p, nslabs == 1 ? kSingle : kLoopback, 0, nslabs, nullptr, out);
}

pf_status pf_nccl_unique_id(uint8_t out[128]) {
    if (!out) return set_err(nullptr, PF_ERR_ARG, "out is NULL");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return set_err(nullptr, PF_ERR_NCCL, fmt("ncclGetUniqueId: %s", ncclGetErrorString(r)));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
    return PF_OK;
}

pf_status pf_create_slab(const pf_params *p, int32_t rank, int32_t nranks, const uint8_t uid[128],
                         pf_ctx **out) {
    if (!uid) return set_err(nullptr, PF_ERR_ARG, "uid is NULL");
    return create_common(p, nranks == 1 ? kSingle : kNccl, rank, nranks, uid, out);
}

pf_status pf_step(pf_ctx *c, int64_t n) {
    Nvtx nv("pf_step");
    if (!c) return set_err(nullptr, PF_ERR_ARG, "ctx is NULL");
    if (n < 0) return set_err(c, PF_ERR_ARG, "n must be >= 0");
    if (c->blown) return set_err(c, PF_ERR_STATE, "state blew up; call pf_set_fields first");
    cudaSetDevice(c->p.device);
    const int64_t ce = c->p.check_every;
    int64_t left = n;
    while (left > 0) {
        int64_t chunk = ce - (c->steps % ce);
        if (chunk > left) chunk = left;
        int64_t done = 0;
        const bool use_graph = c->p.graph_steps > 0 && !c->prof && c->mode != kNccl && !(c->p.noise_rho > 0.0) &&
                               !c->fused && !c->persistent && !c->band &&
                               !c->peer && (!c->nccl_self || nccl_self_graph());   // fused swaps buffers on the host each step; peer waits on epochs
        if (c->band && !c->prof && chunk > 0) {
            Nvtx nv("pf band kernel (small grid)");
            Slab &S = c->slabs[0];
            CK(c, pf::launch_band(c->p.precision, S.L, c->bplan, c->K, S.U, c->vel, c->p.dt, chunk, c->stream));
            CK(c, pf::launch_fill_ghosts(c->p.precision, S.L, c->p.rho_in, S.U, c->stream));
            c->launches += 1 + pf::kFillLaunches;
            done = chunk;
        }
        if (c->persistent && !c->prof && chunk > 0) {
            Nvtx nv("pf persistent kernel (small grid)");
            Slab &S = c->slabs[0];
            CK(c, pf::launch_persistent(c->p.precision, S.L, c->K, S.U, S.Us, c->vel, c->p.dt, chunk, c->pflags,
                                        c->pepoch, c->stream));
            c->pepoch += (uint32_t)chunk;
            CK(c, pf::launch_fill_ghosts(c->p.precision, S.L, c->p.rho_in, S.U, c->stream));
            c->launches += 1 + pf::kFillLaunches;
            done = chunk;
        }
        if (use_graph && chunk >= c->p.graph_steps) {
            pf_status st = ensure_graph(c);
            if (st != PF_OK) return st;
            while (chunk - done >= c->gsteps) {
                CK(c, cudaGraphLaunch(c->gexec, c->stream));
                c->launches += (int64_t)c->gsteps * 2 * (int64_t)c->slabs.size() * pf::kStageLaunches;
                done += c->gsteps;
            }
        }
        for (; done < chunk; ++done) {
            pf_status st = one_step(c, false, c->steps + done);
            if (st != PF_OK) return st;
        }
        const int64_t from = c->steps;
        c->steps += chunk;
        c->t += (double)chunk * c->p.dt;
        left -= chunk;
        if (c->steps % ce == 0 || left == 0) {
            pf_status st = check_blowup(c, from, c->steps);
            if (st != PF_OK) return st;
        }
    }
    CK(c, cudaStreamSynchronize(c->stream));
    return PF_OK;
}

pf_status pf_run_host(pf_ctx *c, int64_t n, const double *ci, const double *pi, const double *ri, double *co,
                      double *po, double *ro, int32_t chunks) {
    if (!c) return set_err(nullptr, PF_ERR_ARG, "ctx is NULL");
    if (n < 0) return set_err(c, PF_ERR_ARG, "n must be >= 0");
    if (c->blown && !(ci && pi && ri)) return set_err(c, PF_ERR_STATE, "state blew up; pass all three input fields");
    cudaSetDevice(c->p.device);
    const int M = c->p.n_members;
    int K = chunks < 1 ? 1 : (chunks > M ? M : chunks);
    if (c->mode != kSingle || c->p.precision != PF_F64 || K < 2) {
        pf_status st = PF_OK;
        if (ci || pi || ri) st = pf_set_fields(c, -1, ci, pi, ri);
        if (st == PF_OK) st = pf_step(c, n);
        if (st == PF_OK && (co || po || ro)) st = pf_get_fields(c, -1, co, po, ro);
        return st;
    }
    Slab &S = c->slabs[0];
    if (!c->h2d) {
        CK(c, cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
        CK(c, cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    }
    while ((int)c->ev_in.size() < K) {
        cudaEvent_t a, b;
        CK(c, cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
        CK(c, cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
        c->ev_in.push_back(a);
        c->ev_done.push_back(b);
    }
    // chunk boundaries: 2 chunks split evenly; with >= 3 the first and last chunks are small
    // (~1/8 of the members each) so that the exposed upload of the first and download of the last
    // are short, and the middle chunks (most of the work) run at full size
    std::vector<int> bnd(K + 1, 0);
    if (K >= 3) {
        const int edge = std::max(1, std::min(M / 8, (M - (K - 2)) / 2));   // 1/8: best of 1/4 .. 1/32
        bnd[1] = edge;
        bnd[K - 1] = M - edge;
        for (int k = 2; k < K - 1; ++k) bnd[k] = edge + (int)((int64_t)(M - 2 * edge) * (k - 1) / (K - 2));
        bnd[K] = M;
    } else {
        for (int k = 0; k <= K; ++k) bnd[k] = (int)((int64_t)M * k / K);
    }
    const size_t hrow = (size_t)c->p.nx * sizeof(double), hmem = (size_t)S.L.ny_loc * hrow;
    const size_t dpitch = (size_t)S.L.pitch * sizeof(double);
    const double *src[3] = {ci, pi, ri};
    double *dst[3] = {co, po, ro};
    auto dev_field = [&](int m, int f) {
        return (char *)S.U + ((size_t)m * S.L.mstride + (size_t)f * S.L.fstride + (size_t)S.L.at(0, 0)) * 8;
    };
    // the compute stream must not overtake work already queued on it (previous calls)
    CK(c, cudaEventRecord(c->ev_done[0], c->stream));
    CK(c, cudaStreamWaitEvent(c->h2d, c->ev_done[0], 0));
    // 1. uploads, chunk by chunk, on the H2D stream
    for (int k = 0; k < K; ++k) {
        const int m0 = bnd[k], m1 = bnd[k + 1];
        for (int m = m0; m < m1; ++m)
            for (int f = 0; f < 3; ++f)
                if (src[f])
                    CK(c, cudaMemcpy2DAsync(dev_field(m, f), dpitch, (const char *)src[f] + (size_t)m * hmem, hrow,
                                            hrow, S.L.ny_loc, cudaMemcpyHostToDevice, c->h2d));
        CK(c, cudaEventRecord(c->ev_in[k], c->h2d));
    }
    // 2. per chunk on the compute stream: ghost frame, n steps, diagnostics; then its download
    for (int k = 0; k < K; ++k) {
        const int m0 = bnd[k], m1 = bnd[k + 1];
        pf::Layout L = S.L;
        L.m0 = m0;
        L.members = m1 - m0;
        CK(c, cudaStreamWaitEvent(c->stream, c->ev_in[k], 0));
        if (ci || pi || ri) {
            pf::Layout Lg = S.L;
            Lg.members = m1 - m0;
            CK(c, pf::launch_fill_ghosts(c->p.precision, Lg, c->p.rho_in, (char *)S.U + (size_t)m0 * S.L.mstride * 8,
                                         c->stream));
            c->launches += pf::kFillLaunches;
        }
        for (int64_t i = 0; i < n; ++i)
            for (int stage = 1; stage <= 2; ++stage) {
                if (stage == 1 && c->p.noise_rho > 0.0) {
                    CK(c, pf::launch_inflow(c->p.precision, L, c->p.rho_in, c->p.noise_rho, c->p.seed,
                                            c->p.member_offset, c->steps + i, S.U, S.Us, c->stream));
                    c->launches += 1;
                }
                const void *in = stage == 1 ? S.U : S.Us;
                void *out = stage == 1 ? S.Us : S.U;
                const double coef = stage == 1 ? 0.5 * c->p.dt : c->p.dt;
                CK(c, pf::launch_stage(c->p.precision, L, S.plan, c->K, stage, in, S.U, out, c->vel, coef, c->stream));
                c->launches += pf::kStageLaunches;
            }
        pf::Layout Ld = S.L;
        Ld.members = m1 - m0;
        const int nb = pf::diag_blocks(S.L);
        CK(c, pf::launch_diag(c->p.precision, Ld, c->K, (char *)S.U + (size_t)m0 * S.L.mstride * 8,
                              S.partials + (size_t)m0 * nb * pf::kDiag, S.diag + (size_t)m0 * pf::kDiag, c->stream));
        c->launches += pf::kDiagLaunches;
        CK(c, cudaEventRecord(c->ev_done[k], c->stream));
        CK(c, cudaStreamWaitEvent(c->d2h, c->ev_done[k], 0));
        for (int m = m0; m < m1; ++m)
            for (int f = 0; f < 3; ++f)
                if (dst[f])
                    CK(c, cudaMemcpy2DAsync((char *)dst[f] + (size_t)m * hmem, hrow, dev_field(m, f), dpitch, hrow,
                                            S.L.ny_loc, cudaMemcpyDeviceToHost, c->d2h));
    }
    CK(c, cudaMemcpyAsync(c->h_diag, S.diag, (size_t)M * pf::kDiag * sizeof(double), cudaMemcpyDeviceToHost, c->d2h));
    CK(c, cudaStreamSynchronize(c->d2h));
    CK(c, cudaStreamSynchronize(c->stream));
    const int64_t from = c->steps;
    c->steps += n;
    c->t += (double)n * c->p.dt;
    c->blown = false;
    double nf[3] = {0, 0, 0};
    int worst = -1;
    for (int m = 0; m < M; ++m) {
        for (int f = 0; f < 3; ++f) nf[f] += c->h_diag[(size_t)m * pf::kDiag + 5 + f];
        if (worst < 0 && c->h_diag[(size_t)m * pf::kDiag + 4] > 0) worst = m;
    }
    if (nf[0] + nf[1] + nf[2] > 0) {
        c->blown = true;
        std::string fields;
        const char *names[3] = {"c", "phi", "rho"};
        for (int f = 0; f < 3; ++f)
            if (nf[f] > 0) fields += fmt("%s%s (%.0f cells)", fields.empty() ? "" : ", ", names[f], nf[f]);
        return set_err(c, PF_ERR_BLOWUP, fmt("blow-up: non-finite %s in steps (%lld, %lld], first member %d",
                                             fields.c_str(), (long long)from, (long long)c->steps,
                                             worst + c->p.member_offset));
    }
    return PF_OK;
}

pf_status pf_trajectory(pf_ctx *c, int32_t n_snapshots, int64_t steps_between, double *out, double *times) {
    if (!c) return set_err(nullptr, PF_ERR_ARG, "ctx is NULL");
    if (n_snapshots < 1 || steps_between < 0 || !out) return set_err(c, PF_ERR_ARG, "bad trajectory arguments");
    if (c->blown) return set_err(c, PF_ERR_STATE, "state blew up; call pf_set_fields first");
    cudaSetDevice(c->p.device);
    const int M = c->p.n_members;
    const size_t per = (size_t)c->ny_host * c->p.nx;           // doubles per member snapshot
    const size_t n = per * M;
    if (c->snap_n < n) {
        for (int b = 0; b < 2; ++b) {
            cudaFree(c->snap[b]);
            c->snap[b] = nullptr;
        }
        c->snap_n = 0;
        for (int b = 0; b < 2; ++b)
            if (cudaMalloc((void **)&c->snap[b], n * sizeof(double)) != cudaSuccess) {
                cudaGetLastError();
                return set_err(c, PF_ERR_NOMEM, "cudaMalloc of snapshot buffers failed");
            }
        c->snap_n = n;
    }
    if (!c->d2h) {
        CK(c, cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
        CK(c, cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    }
    for (int b = 0; b < 2; ++b)
        if (!c->ev_snap[b]) {
            CK(c, cudaEventCreateWithFlags(&c->ev_snap[b], cudaEventDisableTiming));
            CK(c, cudaEventCreateWithFlags(&c->ev_copied[b], cudaEventDisableTiming));
        }
    for (int s = 0; s < n_snapshots; ++s) {
        if (s > 0) {
            pf_status st = pf_step(c, steps_between);
            if (st != PF_OK) {
                cudaStreamSynchronize(c->d2h);
                return st;
            }
        }
        const int b = s & 1;
        if (s >= 2) CK(c, cudaStreamWaitEvent(c->stream, c->ev_copied[b], 0));   // buffer b is free again
        for (auto &S : c->slabs) {
            CK(c, pf::launch_composite(c->p.precision, S.L, S.U, c->snap[b], (int64_t)per, S.L.y0 - c->y_host0,
                                       c->stream));
            c->launches += 1;
        }
        CK(c, cudaEventRecord(c->ev_snap[b], c->stream));
        CK(c, cudaStreamWaitEvent(c->d2h, c->ev_snap[b], 0));
        // out[m][s][row][x]: one strided copy for all members
        CK(c, cudaMemcpy2DAsync(out + (size_t)s * per, (size_t)n_snapshots * per * sizeof(double), c->snap[b],
                                per * sizeof(double), per * sizeof(double), (size_t)M, cudaMemcpyDeviceToHost, c->d2h));
        CK(c, cudaEventRecord(c->ev_copied[b], c->d2h));
        if (times) times[s] = c->t;
    }
    CK(c, cudaStreamSynchronize(c->d2h));
    return PF_OK;
}

// Trajectory file (NEXT-1 I/O; layout in include/pf.h): snapshot s of every member goes device ->
// pinned host buffer (d2h stream) while the next steps run; a writer thread appends it to the file
// while the GPU keeps stepping (pf_step blocks the calling thread).  Two host buffers.
pf_status pf_trajectory_file(pf_ctx *c, const char *path, int32_t n_snapshots, int64_t steps_between,
                             int32_t dtype) {
    if (!c) return set_err(nullptr, PF_ERR_ARG, "ctx is NULL");
    if (!path || n_snapshots < 1 || steps_between < 0 || (dtype != 0 && dtype != 1))
        return set_err(c, PF_ERR_ARG, "bad trajectory-file arguments");
    if (c->blown) return set_err(c, PF_ERR_STATE, "state blew up; call pf_set_fields first");
    Nvtx nv("pf trajectory file");
    cudaSetDevice(c->p.device);
    const int M = c->p.n_members;
    const size_t per = (size_t)c->ny_host * c->p.nx, n = per * M;
    FILE *f = std::fopen(path, "wb");
    if (!f) return set_err(c, PF_ERR_ARG, fmt("cannot open %s for writing", path));
    // header (little-endian, 96 bytes) + per-member records
    struct Header {
        char magic[8];
        uint32_t header_bytes, version;
        int32_t nx, ny_global, y0, ny_rows, members, member_offset, n_snapshots, dtype;
        int64_t steps_between, step0;
        double dt, t0, dx, rho_in;
    } h{};
    static_assert(sizeof(Header) == 96, "trajectory header layout");
    std::memcpy(h.magic, "PFTRAJ01", 8);
    h.header_bytes = (uint32_t)(sizeof(Header) + (size_t)M * 8 * sizeof(double));
    h.version = 1;
    h.nx = c->p.nx;
    h.ny_global = c->p.ny;
    h.y0 = c->y_host0;
    h.ny_rows = c->ny_host;
    h.members = M;
    h.member_offset = c->p.member_offset;
    h.n_snapshots = n_snapshots;
    h.dtype = dtype;
    h.steps_between = steps_between;
    h.step0 = c->steps;
    h.dt = c->p.dt;
    h.t0 = c->t;
    h.dx = c->p.dx;
    h.rho_in = c->p.rho_in;
    bool ok = std::fwrite(&h, sizeof h, 1, f) == 1;
    for (int m = 0; m < M && ok; ++m) {   // global id, v_x, v_y, M_A^b, M_B^b, M_A^s, M_B^s, 0
        double r[8] = {0};
        const int64_t gm = (int64_t)c->p.member_offset + m;
        r[0] = (double)gm;
        member_velocity(c->p, gm, r[1], r[2]);
        member_mobility(c->p, gm, r + 3);
        ok = std::fwrite(r, sizeof r, 1, f) == 1;
    }
    if (!ok) {
        std::fclose(f);
        return set_err(c, PF_ERR_ARG, fmt("write to %s failed", path));
    }
    // device snapshot buffers (shared with pf_trajectory), pinned host buffers, events
    if (c->snap_n < n) {
        for (int b = 0; b < 2; ++b) {
            cudaFree(c->snap[b]);
            c->snap[b] = nullptr;
        }
        c->snap_n = 0;
        for (int b = 0; b < 2; ++b)
            if (cudaMalloc((void **)&c->snap[b], n * sizeof(double)) != cudaSuccess) {
                cudaGetLastError();
                std::fclose(f);
                return set_err(c, PF_ERR_NOMEM, "cudaMalloc of snapshot buffers failed");
            }
        c->snap_n = n;
    }
    if (!c->d2h) {
        CK(c, cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
        CK(c, cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    }
    for (int b = 0; b < 2; ++b)
        if (!c->ev_snap[b]) {
            CK(c, cudaEventCreateWithFlags(&c->ev_snap[b], cudaEventDisableTiming));
            CK(c, cudaEventCreateWithFlags(&c->ev_copied[b], cudaEventDisableTiming));
        }
    double *hb[2] = {nullptr, nullptr};
    for (int b = 0; b < 2; ++b)
        if (cudaMallocHost((void **)&hb[b], n * sizeof(double)) != cudaSuccess) {
            cudaGetLastError();
            cudaFreeHost(hb[0]);
            std::fclose(f);
            return set_err(c, PF_ERR_NOMEM, "cudaMallocHost of the trajectory buffers failed");
        }
    // writer thread: snapshot s in host buffer s & 1, written once its copy event completed
    std::mutex mu;
    std::condition_variable cv;
    int queued = 0, written = 0;
    bool werr = false;
    std::vector<float> tmp(dtype == 1 ? n : 0);
    std::thread writer([&] {
        for (int s = 0; s < n_snapshots; ++s) {
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return queued > s || werr; });
                if (werr) return;
            }
            const int b = s & 1;
            bool good = cudaEventSynchronize(c->ev_copied[b]) == cudaSuccess;
            if (good && dtype == 0) {
                good = std::fwrite(hb[b], sizeof(double), n, f) == n;
            } else if (good) {
                for (size_t i = 0; i < n; ++i) tmp[i] = (float)hb[b][i];
                good = std::fwrite(tmp.data(), sizeof(float), n, f) == n;
            }
            std::lock_guard<std::mutex> lk(mu);
            if (!good) werr = true;
            written = s + 1;
            cv.notify_all();
            if (werr) return;
        }
    });
    std::vector<double> times((size_t)n_snapshots);
    pf_status st = PF_OK;
    for (int s = 0; s < n_snapshots && st == PF_OK; ++s) {
        if (s > 0 && (st = pf_step(c, steps_between)) != PF_OK) break;
        const int b = s & 1;
        {   // host buffer b is free once snapshot s - 2 is on disk
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return written >= s - 1 || werr; });
            if (werr) { st = set_err(c, PF_ERR_ARG, fmt("write to %s failed", path)); break; }
        }
        if (s >= 2) {
            cudaError_t e = cudaStreamWaitEvent(c->stream, c->ev_copied[b], 0);
            if (e != cudaSuccess) { st = set_err(c, PF_ERR_CUDA, cudaGetErrorString(e)); break; }
        }
        for (auto &S : c->slabs) {
            cudaError_t e = pf::launch_composite(c->p.precision, S.L, S.U, c->snap[b], (int64_t)per,
                                                 S.L.y0 - c->y_host0, c->stream);
            if (e != cudaSuccess) { st = set_err(c, PF_ERR_CUDA, cudaGetErrorString(e)); break; }
            c->launches += 1;
        }
        if (st != PF_OK) break;
        cudaEventRecord(c->ev_snap[b], c->stream);
        cudaStreamWaitEvent(c->d2h, c->ev_snap[b], 0);
        cudaMemcpyAsync(hb[b], c->snap[b], n * sizeof(double), cudaMemcpyDeviceToHost, c->d2h);
        cudaEventRecord(c->ev_copied[b], c->d2h);
        times[(size_t)s] = c->t;
        std::lock_guard<std::mutex> lk(mu);
        queued = s + 1;
        cv.notify_all();
    }
    {
        std::lock_guard<std::mutex> lk(mu);
        if (st != PF_OK) werr = true;
        cv.notify_all();
    }
    writer.join();
    if (st == PF_OK && werr) st = set_err(c, PF_ERR_ARG, fmt("write to %s failed", path));
    if (st == PF_OK && std::fwrite(times.data(), sizeof(double), times.size(), f) != times.size())
        st = set_err(c, PF_ERR_ARG, fmt("write to %s failed", path));
    cudaStreamSynchronize(c->d2h);
    cudaFreeHost(hb[0]);
    cudaFreeHost(hb[1]);
    if (std::fclose(f) != 0 && st == PF_OK) st = set_err(c, PF_ERR_ARG, fmt("closing %s failed", path));
    return st;
}

pf_status pf_get_fields(pf_ctx *c, int32_t member, double *fc, double *fp, double *fr) {
    if (!c) return set_err(nullptr, PF_ERR_ARG, "ctx is NULL");
    int m0, nm;
    pf_status st = check_member(c, member, m0, nm);
    if (st != PF_OK) return st;
    cudaSetDevice(c->p.device);
    double *dst[3] = {fc, fp, fr};
    const size_t hrow = (size_t)c->p.nx * sizeof(double);
    const size_t hmem = (size_t)c->ny_host * hrow;   // host bytes per member
    for (auto &S : c->slabs) {
        const size_t nloc = (size_t)S.L.ny_loc * c->p.nx;
        for (int f = 0; f < 3; ++f) {
            if (!dst[f]) continue;
            char *h = (char *)dst[f] + (size_t)(S.L.y0 - c->y_host0) * hrow;
            if (c->esz == 8) {
                for (int mm = 0; mm < nm; ++mm) {
                    const char *d = (const char *)S.U +
                                    ((size_t)(m0 + mm) * S.L.mstride + (size_t)f * S.L.fstride + S.L.at(0, 0)) * 8;
                    CK(c, cudaMemcpy2DAsync(h + mm * hmem, hrow, d, (size_t)S.L.pitch * 8, hrow, S.L.ny_loc,
                                            cudaMemcpyDeviceToHost, c->stream));
                }
            } else {
                st = ensure_staging(c, nloc * nm);
                if (st != PF_OK) return st;
                CK(c, pf::launch_pack_f64(c->p.precision, S.L, f, m0, nm, S.U, c->staging, c->stream));
                c->launches += 1;
                CK(c, cudaMemcpy2DAsync(h, hmem, c->staging, nloc * 8, nloc * 8, nm, cudaMemcpyDeviceToHost, c->stream));
            }
        }
    }
    CK(c, cudaStreamSynchronize(c->stream));
    return PF_OK;
}

pf_status pf_set_fields(pf_ctx *c, int32_t member, const double *fc, const double *fp, const double *fr) {
    if (!c) return set_err(nullptr, PF_ERR_ARG, "ctx is NULL");
    int m0, nm;
    pf_status st = check_member(c, member, m0, nm);
    if (st != PF_OK) return st;
    cudaSetDevice(c->p.device);
    const double *src[3] = {fc, fp, fr};
    const size_t hrow = (size_t)c->p.nx * sizeof(double);
    const size_t hmem = (size_t)c->ny_host * hrow;
    for (auto &S : c->slabs) {
        const size_t nloc = (size_t)S.L.ny_loc * c->p.nx;
        for (int f = 0; f < 3; ++f) {
            if (!src[f]) continue;
            const char *h = (const char *)src[f] + (size_t)(S.L.y0 - c->y_host0) * hrow;
            if (c->esz == 8) {
                for (int mm = 0; mm < nm; ++mm) {
                    char *d = (char *)S.U + ((size_t)(m0 + mm) * S.L.mstride + (size_t)f * S.L.fstride + S.L.at(0, 0)) * 8;
                    CK(c, cudaMemcpy2DAsync(d, (size_t)S.L.pitch * 8, h + mm * hmem, hrow, hrow, S.L.ny_loc,
                                            cudaMemcpyHostToDevice, c->stream));
                }
            } else {
                st = ensure_staging(c, nloc * nm);
                if (st != PF_OK) return st;
                CK(c, cudaMemcpy2DAsync(c->staging, nloc * 8, h, hmem, nloc * 8, nm, cudaMemcpyHostToDevice, c->stream));
                CK(c, pf::launch_unpack_f64(c->p.precision, S.L, f, m0, nm, c->staging, S.U, c->stream));
                c->launches += 1;
            }
        }
        CK(c, pf::launch_fill_ghosts(c->p.precision, S.L, c->p.rho_in, S.U, c->stream));
        c->launches += pf::kFillLaunches;
    }
    if ((st = peer_barrier(c)) != PF_OK) return st;
    st = exchange(c, 0, c->stream);
    if (st == PF_OK) st = finish_exchange(c, c->stream);
    if (st != PF_OK) return st;
    CK(c, cudaStreamSynchronize(c->stream));
    c->blown = false;
    return PF_OK;
}

pf_status pf_diagnostics(pf_ctx *c, int32_t member, double out[5]) {
    if (!c) return set_err(nullptr, PF_ERR_ARG, "ctx is NULL");
    if (!out) return set_err(c, PF_ERR_ARG, "out is NULL");
    if (member < 0 || member >= c->p.n_members) return set_err(c, PF_ERR_ARG, fmt("member %d out of range", member));
    cudaSetDevice(c->p.device);
    std::vector<double> d;
    pf_status st = gather_diag(c, d);
    if (st != PF_OK) return st;
    for (int k = 0; k < 5; ++k) out[k] = d[(size_t)member * pf::kDiag + k];
    return PF_OK;
}

pf_status pf_info(pf_ctx *c, int64_t *steps, double *t, int32_t *y0, int32_t *ny_local) {
    if (!c) return set_err(nullptr, PF_ERR_ARG, "ctx is NULL");
    if (steps) *steps = c->steps;
    if (t) *t = c->t;
    if (y0) *y0 = c->y_host0;
    if (ny_local) *ny_local = c->ny_host;
    return PF_OK;
}

pf_status pf_shape(pf_ctx *c, int32_t *nx, int32_t *ny, int32_t *members) {
    if (!c) return set_err(nullptr, PF_ERR_ARG, "ctx is NULL");
    if (nx) *nx = c->p.nx;
    if (ny) *ny = c->p.ny;
    if (members) *members = c->p.n_members;
    return PF_OK;
}

pf_status pf_set_time(pf_ctx *c, int64_t steps, double t) {
    if (!c) return set_err(nullptr, PF_ERR_ARG, "ctx is NULL");
    if (steps < 0) return set_err(c, PF_ERR_ARG, "steps must be >= 0");
    c->steps = steps;
    c->t = t;
    return PF_OK;
}

pf_status pf_launch_count(pf_ctx *c, int64_t *launches) {
    if (!c || !launches) return set_err(c, PF_ERR_ARG, "NULL argument");
    *launches = c->launches;
    return PF_OK;
}

pf_status pf_profile(pf_ctx *c, int32_t enable) {
    if (!c) return set_err(nullptr, PF_ERR_ARG, "ctx is NULL");
    CK(c, cudaStreamSynchronize(c->stream));
    for (auto &r : c->ev_rec) {
        c->ev_pool.push_back(r.second.first);
        c->ev_pool.push_back(r.second.second);
    }
    c->ev_rec.clear();
    c->prof = enable != 0;
    return PF_OK;
}

pf_status pf_profile_read(pf_ctx *c, double out[6]) {
    if (!c || !out) return set_err(c, PF_ERR_ARG, "NULL argument");
    CK(c, cudaStreamSynchronize(c->stream));
    for (int k = 0; k < 6; ++k) out[k] = 0.0;
    for (auto &r : c->ev_rec) {
        float ms = 0.f;
        CK(c, cudaEventElapsedTime(&ms, r.second.first, r.second.second));
        const int slot = 2 * (r.first - 1);
        out[slot] += ms;
        out[slot + 1] += 1.0;
    }
    return PF_OK;
}

pf_status pf_stream(pf_ctx *c, void **stream) {
    if (!c || !stream) return set_err(c, PF_ERR_ARG, "NULL argument");
    *stream = (void *)c->stream;
    return PF_OK;
}

const char *pf_last_error(const pf_ctx *c) { return c ? c->err.c_str() : g_create_error.c_str(); }

pf_status pf_debug_guards(pf_ctx *c, int64_t *guard_bytes, int64_t *corrupted) {
    if (!c || !guard_bytes || !corrupted) return set_err(c, PF_ERR_ARG, "NULL argument");
    cudaSetDevice(c->p.device);
    CK(c, cudaStreamSynchronize(c->stream));
    *guard_bytes = (int64_t)kGuardBytes;
    *corrupted = 0;
    if (kGuardBytes == 0) return PF_OK;
    std::vector<unsigned char> h(kGuardBytes);
    for (auto &S : c->slabs)
        for (int b = 0; b < 2; ++b)
            for (int side = 0; side < 2; ++side) {
                const char *g = (const char *)S.alloc[b] + (side ? kGuardBytes + S.bytes : 0);
                CK(c, cudaMemcpy(h.data(), g, kGuardBytes, cudaMemcpyDeviceToHost));
                for (unsigned char v : h) *corrupted += v != kGuardByte;
            }
    return PF_OK;
}

void pf_free(pf_ctx *c) { destroy(c); }

}  // extern "C"
