// pf_kernels.cu -- sm_100a kernels of the PVD phase-field midpoint step.
//
// pair_kernel (performance path): one fused pass per explicit-midpoint stage (section 4.2).
//   Persistent blocks walk x-strips of the grid in y.  A producer warp streams boxes of R rows x
//   3 fields (c, phi, rho) of a strip -- plus the stage-2 base rows -- into a shared-memory ring
//   with 3D TMA tensor copies (cp.async.bulk.tensor, mbarrier completion); compute warps (two
//   columns per lane) evaluate mu / M once per cell (row a2) and the flux divergence, source,
//   vapour and Euler-form update (rows a3-a5), exchanging x-neighbours by warp shuffles, and write
//   the result together with its ghost-frame copies (row a1).
// ws_kernel (experimental, kernel_path 5): one pass per midpoint step, stage-1 warps hand u* to
//   stage-2 warps through shared memory.
// stage_kernel (fallback path, any nx) and persistent_kernel (small grids): 2D shared-memory
//   tiles with a 2-cell halo, ghost rules applied by index.
// diag_kernel: fp64 sums, free energy E_h and non-finite counts with fixed-order reductions.
//
// Every cell's value comes from the same arithmetic (pf_cell.cuh) on every path, so results are
// bitwise independent of the kernel path, tiling, x-translation and slab decomposition.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cooperative_groups.h>
#include <cudaTypedefs.h>
#include <utility>

#include "pf_cell.cuh"
#include "pf_internal.h"

namespace cg = cooperative_groups;

// Compilation parts (build.py compiles this file once per part, in parallel): 0 = host plumbing,
// tile / persistent / diagnostics / ghost / pack kernels; 1-4 = pair kernel fp64 stage 1, fp64
// stage 2, fp32 stage 1, fp32 stage 2; 5 = warp-specialised step kernel.  Undefined = all.
#ifndef PF_PART
#define PF_PART -1
#endif
#define PF_IN(k) (PF_PART < 0 || PF_PART == (k))

#ifndef PF_PAIR_UNROLL
#define PF_PAIR_UNROLL 1   // unroll of the pair kernel's slot loop (experiment knob)
#endif
constexpr int kPairUnroll = PF_PAIR_UNROLL;
#ifndef PF_STEP_UNROLL
#define PF_STEP_UNROLL 0   // unroll of tile_step's per-phase cell loops (0: the compiler's choice)
#endif
#define PF_PRAGMA(x) _Pragma(#x)
#define PF_UNROLL_N(n) PF_PRAGMA(unroll n)
#if PF_STEP_UNROLL > 0
#define PF_STEP_LOOP_HINT PF_UNROLL_N(PF_STEP_UNROLL)
#else
#define PF_STEP_LOOP_HINT
#endif
#ifndef PF_STEP_TBY4_LOG2
#define PF_STEP_TBY4_LOG2 14   // step persistent kernel: 32 x 4 tiles up to 2^this cells, 32 x 8 above
#endif
#ifndef PF_TBY_LARGE
#define PF_TBY_LARGE 16    // persistent-kernel tile height above 2^17 cells (experiment knob)
#endif

namespace pf {

#if PF_IN(0)
int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v ? atoi(v) : dflt;
}
#else
int env_int(const char *name, int dflt);
#endif

namespace {

// ========================================================================================
// Tile kernel (fallback)
constexpr int BX = 32;   // tile width  (one warp across x)
constexpr int BY = 16;   // tile height (tile kernel; the persistent kernel picks 4 or 16)
constexpr int NT = 256;  // threads per block (32 x 8)

// Local row holding the c/phi value of local row ly after the global mirror rule (R-12),
// clamped so that rows no output depends on stay in bounds.
__device__ __forceinline__ int row_cphi(int ly, const Layout &L) {
    int g = L.y0 + ly;
    if (g < 0) g = -1 - g;
    if (g >= L.ny) g = 2 * L.ny - 1 - g;
    int r = g - L.y0;
    r = r < -2 ? -2 : r;
    r = r > L.ny_loc + 1 ? L.ny_loc + 1 : r;
    return r;
}

__device__ __forceinline__ int wrap_x(int gx, int nx) {
    gx += nx;               // gx >= -2 and nx >= 8
    return gx % nx;
}

template <typename real, int TBY = BY>
struct TileSmem {
    real sc[TBY + 4][BX + 4];
    real sp[TBY + 4][BX + 4];
    real sr[TBY + 2][BX + 2];
    real smc[TBY + 2][BX + 2];
    real smp[TBY + 2][BX + 2];
    real sM[TBY + 2][BX + 2];
};

// One stage on the tile (member m, columns [tx0, tx0 + 32), rows [ty0, ty0 + 16)): ghost rules
// applied by index, so the tile reads owned cells only (the ghost frame may be stale).
template <typename real, int MOB, int FE, int TBY = BY>
__device__ __forceinline__ void tile_stage(const Layout &L, const KC<real> &k, const real *__restrict__ in,
                                           const real *__restrict__ base, real *out, const real *__restrict__ vel,
                                           const double *etab, TileSmem<real, TBY> &ts, int m, int tx0, int ty0) {
    auto &sc = ts.sc;
    auto &sp = ts.sp;
    auto &sr = ts.sr;
    auto &smc = ts.smc;
    auto &smp = ts.smp;
    auto &sM = ts.sM;
    const int nx = L.nx;
    const real *ic = in + m * L.mstride;
    const real *ip = ic + L.fstride;
    const real *ir = ip + L.fstride;

    // ---- load c, phi with a 2-cell halo (ghost rules applied by index) ----
    for (int t = threadIdx.x; t < (TBY + 4) * (BX + 4); t += NT) {
        const int sy = t / (BX + 4), sx = t - sy * (BX + 4);
        const int64_t off = L.at(row_cphi(ty0 - 2 + sy, L), wrap_x(tx0 - 2 + sx, nx));
        sc[sy][sx] = ic[off];
        sp[sy][sx] = ip[off];
    }
    // ---- load rho with a 1-cell halo: bottom mirror, top reservoir (R-12) ----
    for (int t = threadIdx.x; t < (TBY + 2) * (BX + 2); t += NT) {
        const int sy = t / (BX + 2), sx = t - sy * (BX + 2);
        const int gx = wrap_x(tx0 - 1 + sx, nx);
        int g = L.y0 + ty0 - 1 + sy;
        real v;
        if (g >= L.ny) {
            v = k.rho_in;
        } else {
            if (g < 0) g = -1 - g;
            int r = g - L.y0;
            r = r < -2 ? -2 : r;
            r = r > L.ny_loc + 1 ? L.ny_loc + 1 : r;
            v = ir[L.at(r, gx)];
        }
        sr[sy][sx] = v;
    }
    __syncthreads();

    // ---- phase 1: mu_c, mu_phi, M on the tile + 1 ring ----
    const Mob<real> mo = MOB == 2 ? load_mob(vel, m) : Mob<real>{};
    for (int t = threadIdx.x; t < (TBY + 2) * (BX + 2); t += NT) {
        const int sy = t / (BX + 2), sx = t - sy * (BX + 2);
        const int ey = sy + 1, ex = sx + 1;
        real mc, mp, M;
        constitutive<real, MOB, FE>(k, mo, etab, sc[ey][ex], sp[ey][ex], sc[ey][ex - 1], sc[ey][ex + 1],
                                    sc[ey - 1][ex], sc[ey + 1][ex], sp[ey][ex - 1], sp[ey][ex + 1], sp[ey - 1][ex],
                                    sp[ey + 1][ex], mc, mp, M);
        smc[sy][sx] = mc;
        smp[sy][sx] = mp;
        sM[sy][sx] = M;
    }
    __syncthreads();

    // ---- phase 2: fluxes, source, vapour, update ----
    real vx, vy;
    scaled_velocity(k, vel, m, vx, vy);
    const int lx = threadIdx.x & (BX - 1);
    const int gx = tx0 + lx;
    for (int q = threadIdx.x / BX; q < TBY; q += NT / BX) {
        const int ly = ty0 + q;
        if (gx >= nx || ly >= L.r1) continue;
        const int y = q + 1, x = lx + 1;                    // ring coordinates
        const int cy = q + 2, cx = lx + 2;                   // c/phi tile coordinates
        const int64_t o = m * L.mstride + L.at(ly, gx);
        real oc, op, orr;
        const real fe = face_flux<real>(sM[y][x], sM[y][x + 1], smc[y][x], smc[y][x + 1]);
        const real fw = face_flux<real>(sM[y][x - 1], sM[y][x], smc[y][x - 1], smc[y][x]);
        const real fn = face_flux<real>(sM[y][x], sM[y + 1][x], smc[y][x], smc[y + 1][x]);
        const real fs = face_flux<real>(sM[y - 1][x], sM[y][x], smc[y - 1][x], smc[y][x]);
        cell_update<real>(k, vx, vy, fe, fw, fn, fs,
                          smp[y][x], smp[y][x - 1], smp[y][x + 1], smp[y - 1][x], smp[y + 1][x],
                          sp[cy][cx - 1], sp[cy][cx + 1], sp[cy - 1][cx], sp[cy + 1][cx],
                          sr[y][x], sr[y][x - 1], sr[y][x + 1], sr[y - 1][x], sr[y + 1][x],
                          base[o], base[o + L.fstride], base[o + 2 * L.fstride], oc, op, orr);
        PF_DCHECK(ly >= 0 && ly < L.ny_loc && gx >= 0 && gx < nx && m >= 0);
        out[o] = oc;
        out[o + L.fstride] = op;
        out[o + 2 * L.fstride] = orr;
    }
    __syncthreads();   // the tile's shared memory may be refilled next
}

// Both midpoint stages of one step on a tile, for the small-grid persistent kernel (one grid
// barrier per STEP instead of per stage): the tile loads u^n with a 4-cell halo (ghost rules by
// index), computes u* on the tile plus a 2-cell halo (the halo redundantly, bit for bit what the
// neighbouring tiles compute), fills u*'s out-of-domain halo rows with the ghost rules of u*'s own
// ghost frame (mirror rows; rho: bottom mirror, top reservoir -- computing them would flip the
// sign of the source, which is odd under the mirror), then stage 2 on the tile with base u^n.
// Same per-cell arithmetic and argument order as tile_stage: bitwise the two-launch result.
template <typename real, int TBY>
struct TileStepSmem {
    real c0[TBY + 8][BX + 8], p0[TBY + 8][BX + 8];                       // u^n c, phi: rows -4 .. TBY+3
    real r0[TBY + 6][BX + 6];                                            // u^n rho: rows -3 .. TBY+2
    real m1c[TBY + 6][BX + 6], m1p[TBY + 6][BX + 6], M1[TBY + 6][BX + 6]; // stage-1 mu / M: rows -3 .. TBY+2
    real cs[TBY + 4][BX + 4], ps[TBY + 4][BX + 4], rs[TBY + 4][BX + 4];   // u*: rows -2 .. TBY+1
    real m2c[TBY + 2][BX + 2], m2p[TBY + 2][BX + 2], M2[TBY + 2][BX + 2]; // stage-2 mu / M: rows -1 .. TBY
};

// Phase timeline of the step kernel (diagnostic build, -DPF_TRACE=1; read with
// pf_debug_step_trace): per block and step s < kStepTraceSteps, thread 0's global-timer stamps at
// [0] tile start, [1] u^n loaded, [2] stage-1 a2, [3] u*, [4] stage-2 a2, [5] tile done, [6] grid
// barrier passed -- each after the phase's CTA barrier.
#ifndef PF_TRACE
#define PF_TRACE 0
#endif
constexpr int kStepTraceBlocks = 160, kStepTraceSteps = 64;
static __device__ long long g_strace[kStepTraceBlocks][kStepTraceSteps][8];
__device__ __forceinline__ long long step_gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define PF_STEP_STAMP(trs, k)                                                                    \
    do {                                                                                          \
        if (PF_TRACE && (trs) >= 0 && threadIdx.x == 0) g_strace[blockIdx.x][(trs)][(k)] = step_gtimer(); \
    } while (0)

template <typename real, int MOB, int FE, int TBY, int NTH>
__device__ __forceinline__ void tile_step(const Layout &L, const KC<real> &k1, const KC<real> &k2,
                                          const real *__restrict__ in, real *out, const real *__restrict__ vel,
                                          const double *etab, TileStepSmem<real, TBY> &ts, int m, int tx0, int ty0,
                                          int trs = -1) {
    const int nx = L.nx;
    PF_STEP_STAMP(trs, 0);
    const real *ic = in + m * L.mstride;
    const real *ip = ic + L.fstride;
    const real *ir = ip + L.fstride;
    const Mob<real> mo = MOB == 2 ? load_mob(vel, m) : Mob<real>{};
    real vx, vy;
    scaled_velocity(k1, vel, m, vx, vy);
    // ---- u^n: c, phi with a 4-cell halo, rho with a 3-cell halo (ghost rules by index) ----
    PF_STEP_LOOP_HINT
    for (int t = threadIdx.x; t < (TBY + 8) * (BX + 8); t += NTH) {
        const int sy = t / (BX + 8), sx = t - sy * (BX + 8);
        const int64_t off = L.at(row_cphi(ty0 - 4 + sy, L), wrap_x(tx0 - 4 + sx, nx));
        ts.c0[sy][sx] = ic[off];
        ts.p0[sy][sx] = ip[off];
    }
    PF_STEP_LOOP_HINT
    for (int t = threadIdx.x; t < (TBY + 6) * (BX + 6); t += NTH) {
        const int sy = t / (BX + 6), sx = t - sy * (BX + 6);
        int g = L.y0 + ty0 - 3 + sy;
        real v;
        if (g >= L.ny) {
            v = k1.rho_in;
        } else {
            if (g < 0) g = -1 - g;
            int r = g - L.y0;
            r = r < -2 ? -2 : r;
            r = r > L.ny_loc + 1 ? L.ny_loc + 1 : r;
            v = ir[L.at(r, wrap_x(tx0 - 3 + sx, nx))];
        }
        ts.r0[sy][sx] = v;
    }
    __syncthreads();
    PF_STEP_STAMP(trs, 1);
    // ---- stage 1, a2: mu / M of u^n on rows -3 .. TBY+2, columns -3 .. 34 ----
    PF_STEP_LOOP_HINT
    for (int t = threadIdx.x; t < (TBY + 6) * (BX + 6); t += NTH) {
        const int sy = t / (BX + 6), sx = t - sy * (BX + 6);
        const int ey = sy + 1, ex = sx + 1;
        real mc, mp, M;
        constitutive<real, MOB, FE>(k1, mo, etab, ts.c0[ey][ex], ts.p0[ey][ex], ts.c0[ey][ex - 1], ts.c0[ey][ex + 1],
                                    ts.c0[ey - 1][ex], ts.c0[ey + 1][ex], ts.p0[ey][ex - 1], ts.p0[ey][ex + 1],
                                    ts.p0[ey - 1][ex], ts.p0[ey + 1][ex], mc, mp, M);
        ts.m1c[sy][sx] = mc;
        ts.m1p[sy][sx] = mp;
        ts.M1[sy][sx] = M;
    }
    __syncthreads();
    PF_STEP_STAMP(trs, 2);
    // ---- stage 1, a3-a5: u* on rows -2 .. TBY+1, columns -2 .. 33 (in-domain rows only) ----
    PF_STEP_LOOP_HINT
    for (int t = threadIdx.x; t < (TBY + 4) * (BX + 4); t += NTH) {
        const int sy = t / (BX + 4), sx = t - sy * (BX + 4);
        const int g = L.y0 + ty0 - 2 + sy;
        if (g < 0 || g >= L.ny) continue;
        const int y = sy + 1, x = sx + 1;          // mu / M and rho^n coordinates
        const int cy = sy + 2, cx = sx + 2;        // u^n c / phi coordinates
        real oc, op, orr;
        const real fe = face_flux<real>(ts.M1[y][x], ts.M1[y][x + 1], ts.m1c[y][x], ts.m1c[y][x + 1]);
        const real fw = face_flux<real>(ts.M1[y][x - 1], ts.M1[y][x], ts.m1c[y][x - 1], ts.m1c[y][x]);
        const real fn = face_flux<real>(ts.M1[y][x], ts.M1[y + 1][x], ts.m1c[y][x], ts.m1c[y + 1][x]);
        const real fs = face_flux<real>(ts.M1[y - 1][x], ts.M1[y][x], ts.m1c[y - 1][x], ts.m1c[y][x]);
        cell_update<real>(k1, vx, vy, fe, fw, fn, fs, ts.m1p[y][x], ts.m1p[y][x - 1], ts.m1p[y][x + 1],
                          ts.m1p[y - 1][x], ts.m1p[y + 1][x], ts.p0[cy][cx - 1], ts.p0[cy][cx + 1], ts.p0[cy - 1][cx],
                          ts.p0[cy + 1][cx], ts.r0[y][x], ts.r0[y][x - 1], ts.r0[y][x + 1], ts.r0[y - 1][x],
                          ts.r0[y + 1][x], ts.c0[cy][cx], ts.p0[cy][cx], ts.r0[y][x], oc, op, orr);
        ts.cs[sy][sx] = oc;
        ts.ps[sy][sx] = op;
        ts.rs[sy][sx] = orr;
    }
    __syncthreads();
    PF_STEP_STAMP(trs, 3);
    // ---- u*'s out-of-domain rows: its ghost rules (c, phi mirror; rho bottom mirror, top rho_in) ----
    if (L.y0 + ty0 - 2 < 0 || L.y0 + ty0 + TBY + 1 >= L.ny) {
        for (int t = threadIdx.x; t < (TBY + 4) * (BX + 4); t += NTH) {
            const int sy = t / (BX + 4), sx = t - sy * (BX + 4);
            const int g = L.y0 + ty0 - 2 + sy;
            if ((g >= 0 && g < L.ny) || g > L.ny + 1) continue;   // rows beyond ny+1 feed no output
            const int gm = g < 0 ? -1 - g : 2 * L.ny - 1 - g;   // mirrored in-domain row
            const int my = gm - (L.y0 + ty0 - 2);
            ts.cs[sy][sx] = ts.cs[my][sx];
            ts.ps[sy][sx] = ts.ps[my][sx];
            ts.rs[sy][sx] = g < 0 ? ts.rs[my][sx] : k1.rho_in;
        }
        __syncthreads();
    }
    // ---- stage 2, a2: mu / M of u* on rows -1 .. TBY, columns -1 .. 32 ----
    PF_STEP_LOOP_HINT
    for (int t = threadIdx.x; t < (TBY + 2) * (BX + 2); t += NTH) {
        const int sy = t / (BX + 2), sx = t - sy * (BX + 2);
        const int ey = sy + 1, ex = sx + 1;
        real mc, mp, M;
        constitutive<real, MOB, FE>(k2, mo, etab, ts.cs[ey][ex], ts.ps[ey][ex], ts.cs[ey][ex - 1], ts.cs[ey][ex + 1],
                                    ts.cs[ey - 1][ex], ts.cs[ey + 1][ex], ts.ps[ey][ex - 1], ts.ps[ey][ex + 1],
                                    ts.ps[ey - 1][ex], ts.ps[ey + 1][ex], mc, mp, M);
        ts.m2c[sy][sx] = mc;
        ts.m2p[sy][sx] = mp;
        ts.M2[sy][sx] = M;
    }
    __syncthreads();
    PF_STEP_STAMP(trs, 4);
    // ---- stage 2, a3-a5: u^{n+1} of the tile, base u^n ----
    const int lx = threadIdx.x & (BX - 1);
    const int gx = tx0 + lx;
    for (int q = threadIdx.x / BX; q < TBY; q += NTH / BX) {
        const int ly = ty0 + q;
        if (gx >= nx || ly >= L.ny_loc) continue;
        const int y = q + 1, x = lx + 1;          // stage-2 mu / M coordinates
        const int sy = q + 2, sx = lx + 2;        // u* coordinates
        const int64_t o = m * L.mstride + L.at(ly, gx);
        real oc, op, orr;
        const real fe = face_flux<real>(ts.M2[y][x], ts.M2[y][x + 1], ts.m2c[y][x], ts.m2c[y][x + 1]);
        const real fw = face_flux<real>(ts.M2[y][x - 1], ts.M2[y][x], ts.m2c[y][x - 1], ts.m2c[y][x]);
        const real fn = face_flux<real>(ts.M2[y][x], ts.M2[y + 1][x], ts.m2c[y][x], ts.m2c[y + 1][x]);
        const real fs = face_flux<real>(ts.M2[y - 1][x], ts.M2[y][x], ts.m2c[y - 1][x], ts.m2c[y][x]);
        cell_update<real>(k2, vx, vy, fe, fw, fn, fs, ts.m2p[y][x], ts.m2p[y][x - 1], ts.m2p[y][x + 1],
                          ts.m2p[y - 1][x], ts.m2p[y + 1][x], ts.ps[sy][sx - 1], ts.ps[sy][sx + 1], ts.ps[sy - 1][sx],
                          ts.ps[sy + 1][sx], ts.rs[sy][sx], ts.rs[sy][sx - 1], ts.rs[sy][sx + 1], ts.rs[sy - 1][sx],
                          ts.rs[sy + 1][sx], ts.c0[q + 4][lx + 4], ts.p0[q + 4][lx + 4], ts.r0[q + 3][lx + 3], oc, op,
                          orr);
        PF_DCHECK(ly >= 0 && ly < L.ny_loc && gx >= 0 && gx < nx);
        out[o] = oc;
        out[o + L.fstride] = op;
        out[o + 2 * L.fstride] = orr;
    }
    __syncthreads();   // the tile's shared memory may be refilled next
    PF_STEP_STAMP(trs, 5);
}

template <typename real, int MOB, int FE>
__global__ void __launch_bounds__(NT) stage_kernel(Layout L, KC<real> k, const real *__restrict__ in,
                                                   const real *__restrict__ base, real *out,
                                                   const real *__restrict__ vel) {
    __shared__ TileSmem<real> ts;
    __shared__ double etab[64];
    load_exp_table(etab);
    tile_stage<real, MOB, FE>(L, k, in, base, out, vel, etab, ts, L.m0 + (int)blockIdx.z, (int)blockIdx.x * BX,
                              L.r0 + (int)blockIdx.y * BY);
}

// Small-grid path ("B10"): a cooperative persistent kernel that advances every
// member by nsteps midpoint steps in ONE launch -- both stages of every step over all tiles, with
// a grid-wide barrier after each stage -- for grids too small to fill the GPU, where the two
// launches per step (not HBM) are the cost.  Same per-cell arithmetic and tiles as stage_kernel:
// bitwise identical results.  Writes owned cells only; the host rebuilds the ghost frame after.
// TBY: tile height -- 4 for the smallest grids (more, shorter tiles: lower latency per stage),
// 16 otherwise (tools/small_grid_sweep.py).
template <typename real, int MOB, int FE, int TBY>
__global__ void __launch_bounds__(NT) persistent_kernel(Layout L, KC<real> k1, KC<real> k2, real *U, real *Us,
                                                        const real *__restrict__ vel, int64_t nsteps) {
    __shared__ TileSmem<real, TBY> ts;
    __shared__ double etab[64];
    load_exp_table(etab);
    cg::grid_group grid = cg::this_grid();
    const int tx = (L.nx + BX - 1) / BX, ty = (L.ny_loc + TBY - 1) / TBY;
    const int ntiles = tx * ty * L.members;
    for (int64_t s = 0; s < nsteps; ++s) {
        for (int stage = 1; stage <= 2; ++stage) {
            const real *in = stage == 1 ? U : Us;
            real *out = stage == 1 ? Us : U;
            const KC<real> &kk = stage == 1 ? k1 : k2;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int m = t / (tx * ty), r = t - m * (tx * ty);
                const int by = r / tx, bxi = r - by * tx;
                tile_stage<real, MOB, FE, TBY>(L, kk, in, U, out, vel, etab, ts, L.m0 + m, bxi * BX, by * TBY);
            }
            grid.sync();
        }
    }
}

// Small-grid path, one grid barrier per STEP: tile_step (both stages on a tile with a 4-cell u^n
// halo) ping-pongs between U and Us; after an odd number of steps the result is copied back to U.
//
// Step ordering (flags != nullptr, PF_STEP_FLAGS): instead of a grid barrier per step, a tile of
// step s waits only for the (up to) 8 tiles its 4-cell u^n halo reaches to have finished step s-1
// -- flags[tile] counts the steps a tile has completed (release store after the tile's outputs;
// acquire polls, one thread per neighbour).  That also orders the buffer reuse: a tile writes into
// the buffer its neighbours read in step s-1 only after they finished that step.  (Grid barrier:
// ~1.2 us per step, 22% of the configs[1] kernel's stall samples.)
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename real, int MOB, int FE, int TBY, int kStepNT>
__global__ void __launch_bounds__(kStepNT) persistent_step_kernel(Layout L, KC<real> k1, KC<real> k2, real *U,
                                                                  real *Us, const real *__restrict__ vel,
                                                                  int64_t nsteps, unsigned *flags, uint32_t epoch) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileStepSmem<real, TBY> &ts = *reinterpret_cast<TileStepSmem<real, TBY> *>(smem_raw);
    __shared__ double etab[64];
    load_exp_table(etab);
    cg::grid_group grid = cg::this_grid();
    const int tx = (L.nx + BX - 1) / BX, ty = (L.ny_loc + TBY - 1) / TBY;
    const int ntiles = tx * ty * L.members;
    for (int64_t s = 0; s < nsteps; ++s) {
        const real *in = (s & 1) ? Us : U;
        real *out = (s & 1) ? U : Us;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            if (PF_TRACE && threadIdx.x == 0 && t == (int)blockIdx.x && blockIdx.x < kStepTraceBlocks && s < kStepTraceSteps)
                g_strace[blockIdx.x][s][7] = step_gtimer();
            const int m = t / (tx * ty), r = t - m * (tx * ty);
            const int by = r / tx, bxi = r - by * tx;
            if (flags && s > 0) {   // the neighbours' step s-1 (the previous launch: stream order)
                if (threadIdx.x < 9 && threadIdx.x != 4) {
                    const int dy = (int)threadIdx.x / 3 - 1, dx = (int)threadIdx.x % 3 - 1;
                    const int ny_ = by + dy, nx_ = (bxi + dx + tx) % tx;
                    if (ny_ >= 0 && ny_ < ty) {
                        const unsigned *f = flags + (m * ty + ny_) * tx + nx_;
                        const unsigned want = epoch + (unsigned)s;
                        while ((int)(ld_acquire_u32(f) - want) < 0) {
                        }
                    }
                }
                __syncthreads();
            }
            const int trs = PF_TRACE && t == (int)blockIdx.x && blockIdx.x < kStepTraceBlocks && s < kStepTraceSteps
                                ? (int)s : -1;
            tile_step<real, MOB, FE, TBY, kStepNT>(L, k1, k2, in, out, vel, etab, ts, L.m0 + m, bxi * BX, by * TBY,
                                                   trs);
            // tile_step ended with a CTA barrier, so the release (cumulative) covers the whole tile
            if (flags && threadIdx.x == 0) st_release_u32(flags + t, epoch + (unsigned)s + 1u);
        }
        if (!flags) grid.sync();
        if (PF_TRACE && threadIdx.x == 0 && blockIdx.x < kStepTraceBlocks && s < kStepTraceSteps)
            g_strace[blockIdx.x][s][6] = step_gtimer();
    }
    if (flags) grid.sync();   // the copy-back below reads every tile
    if (nsteps & 1) {   // the last step wrote Us: owned cells back to U
        const int64_t per = (int64_t)L.ny_loc * L.nx, total = per * L.members;
        for (int64_t q = (int64_t)blockIdx.x * kStepNT + threadIdx.x; q < total; q += (int64_t)gridDim.x * kStepNT) {
            const int64_t m = q / per, rem = q - m * per;
            const int r = (int)(rem / L.nx), x = (int)(rem - (int64_t)r * L.nx);
            const int64_t o = (L.m0 + m) * L.mstride + L.at(r, x);
            U[o] = Us[o];
            U[o + L.fstride] = Us[o + L.fstride];
            U[o + 2 * L.fstride] = Us[o + 2 * L.fstride];
        }
    }
}

#if PF_IN(0)
}  // namespace
}  // namespace pf
// Diagnostic: the step kernel's phase timeline of its last launch (PF_TRACE builds; zeros
// otherwise): out[160 blocks][64 steps][8] int64 global-timer ns, see PF_STEP_STAMP.
extern "C" int pf_debug_step_trace(long long *out) {
    return (int)cudaMemcpyFromSymbol(out, pf::g_strace, sizeof(pf::g_strace));
}
namespace pf {
namespace {
#endif

// ========================================================================================
// Ghost frame (row a1 in memory)
template <typename real>
__global__ void ghost_rows_kernel(Layout L, real rho_in, real *st) {
    // global y boundaries: c, phi mirror (r = -1 - g); rho: bottom mirror, top reservoir
    const int64_t per = (int64_t)4 * L.nx;   // 2 rows below + 2 rows above
    const int64_t total = per * 3 * L.members;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t mf = q / per;
        const int rem = (int)(q - mf * per);
        const int slot = rem / L.nx, x = rem - slot * L.nx;
        const int f = (int)(mf % 3);
        real *b = st + mf * L.fstride;
        if (slot < 2) {                           // ghost rows -1, -2 of the bottom slab
            if (L.y0 != 0) continue;
            const int r = -1 - slot;
            b[L.at(r, x)] = b[L.at(-1 - r, x)];
        } else {                                  // ghost rows ny_loc, ny_loc+1 of the top slab
            if (L.y0 + L.ny_loc != L.ny) continue;
            const int r = L.ny_loc + (slot - 2);
            b[L.at(r, x)] = (f == 2) ? rho_in : b[L.at(2 * L.ny_loc - 1 - r, x)];
        }
    }
}

template <typename real>
__global__ void ghost_cols_kernel(Layout L, real *st) {
    // periodic x ghost columns of every storage row (incl. ghost rows -> corners)
    const int gx = L.gx;
    const int64_t rows = (int64_t)(L.ny_loc + 4) * 3 * L.members;
    const int64_t total = rows * 2 * gx;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = q / (2 * gx);
        const int j = (int)(q - row * 2 * gx);
        const int64_t mf = row / (L.ny_loc + 4);
        const int r = (int)(row - mf * (L.ny_loc + 4)) - 2;
        real *b = st + mf * L.fstride;
        if (j < gx) {
            const int x = -gx + j;                // left ghost <- x + nx
            b[L.at(r, x)] = b[L.at(r, x + L.nx)];
        } else {
            const int x = L.nx + (j - gx);        // right ghost <- x - nx
            b[L.at(r, x)] = b[L.at(r, x - L.nx)];
        }
    }
}

// ========================================================================================
// diagnostics
constexpr int DT = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

template <typename real>
__global__ void __launch_bounds__(DT) diag_kernel(Layout L, Coef K, const real *__restrict__ st,
                                                  double *partials) {
    const int m = blockIdx.y;
    const int nx = L.nx;
    const real *c = st + m * L.mstride;
    const real *p = c + L.fstride;
    const real *r = p + L.fstride;
    double acc[kDiag];
#pragma unroll
    for (int q = 0; q < kDiag; ++q) acc[q] = 0.0;
    const int64_t ncell = (int64_t)L.ny_loc * nx;
    for (int64_t k = (int64_t)blockIdx.x * DT + threadIdx.x; k < ncell; k += (int64_t)gridDim.x * DT) {
        const int ly = (int)(k / nx), i = (int)(k - (int64_t)ly * nx);
        const int64_t o = L.at(ly, i);
        const double cc = (double)c[o], pp = (double)p[o], rr = (double)r[o];
        const bool fc = isfinite(cc), fp = isfinite(pp), fr = isfinite(rr);
        acc[0] += cc;
        acc[1] += pp;
        acc[2] += rr;
        const int64_t ox = L.at(ly, (i + 1 == nx) ? 0 : i + 1);
        const double dcx = (double)c[ox] - cc;
        const double dpx = (double)p[ox] - pp;
        const double omc = 1.0 - cc, omp = 1.0 - pp;
        double gc;
        if (K.fe == 1) {   // regular solution (R-28)
            const double t = cc < 1e-9 ? 1e-9 : (cc > 1.0 - 1e-9 ? 1.0 - 1e-9 : cc), u = 1.0 - t;
            gc = K.omega * t * u + K.temp * (t * log(t) + u * log(u));
        } else {
            gc = K.W_c * (cc * cc) * (omc * omc);
        }
        double e = K.dx2 * (gc * pp + K.W_p * (pp * pp) * (omp * omp));
        e += K.half_kc * (dcx * dcx) + K.half_kp * (dpx * dpx);
        if (L.y0 + ly < L.ny - 1) {      // y-face above (ghost row at the slab top)
            const int64_t oy = L.at(ly + 1, i);
            const double dcy = (double)c[oy] - cc, dpy = (double)p[oy] - pp;
            e += K.half_kc * (dcy * dcy) + K.half_kp * (dpy * dpy);
        }
        acc[3] += e;
        acc[4] += (fc && fp && fr) ? 0.0 : 1.0;
        acc[5] += fc ? 0.0 : 1.0;
        acc[6] += fp ? 0.0 : 1.0;
        acc[7] += fr ? 0.0 : 1.0;
    }
    __shared__ double red[DT / 32][kDiag];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < kDiag; ++q) {
        const double v = warp_sum(acc[q]);
        if (lane == 0) red[w][q] = v;
    }
    __syncthreads();
    if (threadIdx.x < kDiag) {
        double s = 0.0;
        for (int ww = 0; ww < DT / 32; ++ww) s += red[ww][threadIdx.x];
        partials[((int64_t)m * gridDim.x + blockIdx.x) * kDiag + threadIdx.x] = s;
    }
}

__global__ void __launch_bounds__(DT) diag_final(int nblk, const double *__restrict__ partials,
                                                 double dx2, double *out) {
    const int m = blockIdx.x;
    __shared__ double red[DT / 32][kDiag];
    double acc[kDiag];
#pragma unroll
    for (int q = 0; q < kDiag; ++q) acc[q] = 0.0;
    for (int b = threadIdx.x; b < nblk; b += DT)
#pragma unroll
        for (int q = 0; q < kDiag; ++q) acc[q] += partials[((int64_t)m * nblk + b) * kDiag + q];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < kDiag; ++q) {
        const double v = warp_sum(acc[q]);
        if (lane == 0) red[w][q] = v;
    }
    __syncthreads();
    if (threadIdx.x < kDiag) {
        double s = 0.0;
        for (int ww = 0; ww < DT / 32; ++ww) s += red[ww][threadIdx.x];
        if (threadIdx.x < 3) s *= dx2;
        out[(int64_t)m * kDiag + threadIdx.x] = s;
    }
}

template <typename real>
__global__ void pack_kernel(Layout L, int field, int member0, int nmem, const real *st, double *dst) {
    const int64_t per = (int64_t)L.ny_loc * L.nx;
    const int64_t total = per * nmem;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t mm = k / per, rem = k - mm * per;
        const int r = (int)(rem / L.nx), x = (int)(rem - (int64_t)r * L.nx);
        dst[k] = (double)st[(member0 + mm) * L.mstride + field * L.fstride + L.at(r, x)];
    }
}

template <typename real>
__global__ void unpack_kernel(Layout L, int field, int member0, int nmem, const double *src, real *st) {
    const int64_t per = (int64_t)L.ny_loc * L.nx;
    const int64_t total = per * nmem;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t mm = k / per, rem = k - mm * per;
        const int r = (int)(rem / L.nx), x = (int)(rem - (int64_t)r * L.nx);
        st[(member0 + mm) * L.mstride + field * L.fstride + L.at(r, x)] = (real)src[k];
    }
}

// Composite composition field of a snapshot (NEXT-1 of SURVEY 8(f)): the
// dataset stores c where the cell is solid (phi > 1/2) and 0 in the vapour.  fp64 output,
// dst[m * dst_mstride + (row0 + r) * nx + x] for local rows r of the slab.
template <typename real>
__global__ void composite_kernel(Layout L, const real *st, double *dst, int64_t dst_mstride, int row0) {
    const int64_t per = (int64_t)L.ny_loc * L.nx;
    const int64_t total = per * L.members;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = q / per, rem = q - m * per;
        const int r = (int)(rem / L.nx), x = (int)(rem - (int64_t)r * L.nx);
        const real *b = st + m * L.mstride;
        const double c = (double)b[L.at(r, x)], ph = (double)b[L.fstride + L.at(r, x)];
        dst[m * dst_mstride + (int64_t)(row0 + r) * L.nx + x] = ph > 0.5 ? c : 0.0;
    }
}

// Stochastic inflow (NEXT-3 of SURVEY 8(f); reading R-27): before each step the
// top slab's rho reservoir rows (ghost rows ny_loc, ny_loc+1 of U and Us, ghost columns included)
// get the step's truncated-Gaussian draw per column: attempt a = 0..7 takes z by Box-Muller
// (cosine branch) from counters 2q, 2q+1, q = (step nx + i) 8 + a, of stream 8m+7 of the
// counter generator (R-16); the first rho_in + sigma z inside [0, 2 rho_in] is used, else rho_in.
__device__ __forceinline__ uint64_t sm64_dev(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ double inflow_value(uint64_t seed, int64_t member, int64_t step, int nx, int i, double rho_in,
                               double sigma) {
    const uint64_t key = sm64_dev(seed ^ (((uint64_t)member * 8u + 7u) * 0xD1B54A32D192ED03ull));
    for (int a = 0; a < 8; ++a) {
        const uint64_t q = ((uint64_t)step * (uint64_t)nx + (uint64_t)i) * 8u + (uint64_t)a;
        const double u1 = (double)(sm64_dev(key + 2 * q) >> 11) * 0x1.0p-53;
        const double u2 = (double)(sm64_dev(key + 2 * q + 1) >> 11) * 0x1.0p-53;
        const double z = sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * 3.14159265358979323846 * u2);
        const double v = rho_in + sigma * z;
        if (v >= 0.0 && v <= 2.0 * rho_in) return v;
    }
    return rho_in;
}
template <typename real>
__global__ void inflow_kernel(Layout L, double rho_in, double sigma, uint64_t seed, int64_t gmember0, int64_t step,
                              real *U, real *Us) {
    const int64_t total = (int64_t)L.members * L.pitch;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int ml = (int)(q / L.pitch), xs = (int)(q - (int64_t)ml * L.pitch);
        const int m = L.m0 + ml;
        const int i = ((xs - L.gx) % L.nx + L.nx) % L.nx;
        const real v = (real)inflow_value(seed, gmember0 + m, step, L.nx, i, rho_in, sigma);
        const int64_t o = (int64_t)m * L.mstride + 2 * L.fstride + (int64_t)(L.ny_loc + 2) * L.pitch + xs;
        U[o] = v;
        U[o + L.pitch] = v;
        Us[o] = v;
        Us[o + L.pitch] = v;
    }
}

#include "pf_stream.cuh"

// Timeline trace of one block (diagnostic build, -DPF_TRACE=1; read with pf_debug_trace): per box
// g < kTraceBoxes the producer's wait start / issue time and each compute warp's full-barrier wait
// start / end, from the global nanosecond timer.
#ifndef PF_TRACE
#define PF_TRACE 0
#endif
constexpr int kTraceBoxes = 512, kTraceBlock = 37;
__device__ long long g_ptrace[5][kTraceBoxes][2];
__device__ long long g_bspan[1024][3];   // per block: griddep_wait return, SM id, compute warp 0's end
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// A dedicated producer warp issues the TMA boxes and waits on per-slot "empty" mbarriers.  (Measured
// alternative, round 2: no producer warp -- the last compute warp to release a slot refills it,
// elected by a shared-memory counter, with 15-16 compute warps per SM instead of 12-16: 5-8%
// slower on configs[2] stage 1 even with the schedule tabulated; the refill work sits on a compute
// warp's critical path.  DESIGN.md 7.)
// (Measured alternative, round 2: stage-1 rows staged in shared memory and written by cp.async.bulk
// per field -- 35% slower than the STG.128 stores below; the stores were not the bottleneck, the
// compute warps' dependency latency is.)
//
// Packed variant (V > 1, PF_PAIR_WG builds): V of these blocks share one CTA -- warpgroup 0 holds
// their V producer warps (setmaxnreg.dec to 24 registers), warpgroups 1.. their V * NCW = 12 or
// 16 compute warps (setmaxnreg.inc: the registers the producers gave up, 160 per thread for 12
// compute warps instead of the 128 the 4-blocks-per-SM layout allows).  Same rings, schedule and
// arithmetic per virtual block, so results are bitwise identical.
// Registers per compute thread of a packed block: the CTA's allocation (launch-bound cap x threads)
// minus the producer warpgroup's 24 per thread.  setmaxnreg.inc waits until the CTA's pool holds
// that many, so the launch checks the compiled register count against it (launch_pair_k).
__host__ __device__ constexpr int pair_packed_cap(int V, int NCW) {
    return (65536 / (128 + 32 * V * NCW)) / 8 * 8;
}
__host__ __device__ constexpr int pair_packed_regs(int V, int NCW) {
    return ((pair_packed_cap(V, NCW) * (128 + 32 * V * NCW) - 24 * 128) / (32 * V * NCW)) / 8 * 8 > 248
               ? 248
               : ((pair_packed_cap(V, NCW) * (128 + 32 * V * NCW) - 24 * 128) / (32 * V * NCW)) / 8 * 8;
}

template <typename real, int NCW, int R, int S, bool BASE, int MOB, int FE, int MINB, int V>
__global__ void __launch_bounds__(V == 1 ? 32 * NCW + 32 : 128 + 32 * V * NCW, V == 1 ? MINB : 1) pair_kernel(
    Layout L, KC<real> k, const __grid_constant__ CUtensorMap mapIn, const __grid_constant__ CUtensorMap mapBase,
    real *out, const real *__restrict__ vel, int Wo, int G, int NB) {
    static_assert(R >= 2, "rows k-1, k-2 must lie in the current or the previous box");
    static_assert(V == 1 || (V <= 4 && (V * NCW) % 4 == 0), "packed blocks fill whole warpgroups");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int bx = Wo + 2 * kPairHalo;
    const Ring<real> rg(bx, R, BASE);
    unsigned char *base_sm = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const bool producer = V == 1 ? warp == NCW : warp < 4;
    const int v = V == 1 ? 0 : (producer ? warp : (warp - 4) / NCW);   // virtual block of this warp
    const int cw = V == 1 ? warp : (warp - 4) - v * NCW;                // compute warp within it
    real *slots;
    uint64_t *full, *empty;
    double *etab;
    if (V == 1) {
        slots = reinterpret_cast<real *>(base_sm);
        full = reinterpret_cast<uint64_t *>(base_sm + (size_t)S * rg.slot_elems * sizeof(real));
        empty = full + S;
        etab = reinterpret_cast<double *>(empty + S);
    } else {
        const size_t vbytes = ((size_t)S * rg.slot_elems * sizeof(real) + (size_t)S * 16 + 127) / 128 * 128;
        etab = reinterpret_cast<double *>(base_sm);
        unsigned char *reg = base_sm + 64 * 8 + (size_t)(v < V ? v : 0) * vbytes;
        slots = reinterpret_cast<real *>(reg);
        full = reinterpret_cast<uint64_t *>(reg + (size_t)S * rg.slot_elems * sizeof(real));
        empty = full + S;
    }
    load_exp_table(etab);
    if (V == 1 ? t == 0 : (producer && warp < V && lane == 0)) {   // each virtual block's barriers
        for (int q = 0; q < S; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int vb = V == 1 ? (int)blockIdx.x : (int)blockIdx.x * V + v;
    const int nx = L.nx;
    // set-up above overlaps the previous launch's drain; no global access before griddep_wait.  No
    // explicit trigger: the dependent launch starts as this grid's blocks exit (triggering at block
    // start measured 20% slower on cfg3 -- waiting dependents crowd the SMs).  (Each role runs its
    // own copy of the prologue below: ptxas allocates registers per setmaxnreg region, so the two
    // regions must not merge again.)

    if (producer) {
        // ------------------------------- producer -------------------------------
        if (V > 1) asm volatile("setmaxnreg.dec.sync.aligned.u32 24;" ::: "memory");
        if (lane != 0 || v >= V) return;
        const Sched sch = make_sched(L, Wo, G, vb, NB);
        const uint32_t box_bytes = (uint32_t)(3 * R * bx * sizeof(real));
        griddep_wait();
        prefetch_tmap(&mapIn);
        if (BASE) prefetch_tmap(&mapBase);
        uint32_t g = 0;
        int64_t pos = sch.lo;
        Seg sg;
        while (next_seg(L, Wo, sch, pos, sg)) {
            const int n = sg.yb - sg.ya + 4, nsl = (n + R - 1) / R;
            const int bxs = sg.x0 - kPairHalo + L.gx;           // storage column of the box origin
            for (int j = 0; j < nsl; ++j, ++g) {
                const int slot = g % S;
                const long long tw = PF_TRACE ? gtimer() : 0;
                if (g >= (uint32_t)S) mbar_wait(&empty[slot], ((g / S) - 1) & 1u);
                real *sl = slots + slot * rg.slot_elems;
                const int k0 = sg.ya - 2 + j * R;                 // first row of the box
                mbar_expect_tx(&full[slot], BASE ? 2 * box_bytes : box_bytes);
                tma_load_3d(sl, &mapIn, bxs, k0 + 2, 3 * sg.m, &full[slot]);
                if (BASE) tma_load_3d(sl + rg.in_elems, &mapBase, bxs, k0, 3 * sg.m, &full[slot]);
                if (PF_TRACE && vb == kTraceBlock && g < (uint32_t)kTraceBoxes) {
                    g_ptrace[4][g][0] = tw;
                    g_ptrace[4][g][1] = gtimer();
                }
            }
        }
        return;
    }

    // --------------------------- compute warps ---------------------------------
    if (V > 1) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(pair_packed_regs(V, NCW)) : "memory");
    const Sched sch = make_sched(L, Wo, G, vb, NB);
    griddep_wait();
    if (PF_TRACE && cw == 0 && lane == 0 && vb < 1024) g_bspan[vb][0] = gtimer();
    // Lane l of warp w owns strip-relative columns cx, cx + 1 with cx = 60 w + 2 l - 2: lanes 1..30
    // write them, lane 0's right column and lane 31's left column are the flux halo.
    const int cx = kPairCols * cw + 2 * lane - 2;
    const int ci = kPairHalo + cx;          // its (even) column in a box row
    const int plane = R * bx;
    int sidx = 0;
    uint32_t par = 0;
    uint32_t gtr = 0;                       // PF_TRACE: box counter of this warp
    int64_t pos = sch.lo;
    Seg sg;
    while (next_seg(L, Wo, sch, pos, sg)) {
        const int n = sg.yb - sg.ya + 4, nsl = (n + R - 1) / R;
        const int x = sg.x0 + cx;
        const bool store = lane >= 1 && lane <= 30 && cx < sg.Wp;
        const bool xedge = (x < L.gx) | (x + 1 >= nx - L.gx);
        real *ob = out + sg.m * L.mstride;
        real vx, vy;
        scaled_velocity(k, vel, sg.m, vx, vy);
        const Mob<real> mo = MOB == 2 ? load_mob(vel, sg.m) : Mob<real>{};

        real A1x = 0, A1y = 0, A2x = 0, A2y = 0;          // mu_c rows k-1, k-2
        real M1x = 0, M1y = 0, M2x = 0, M2y = 0;          // M rows k-1, k-2
        real B1x = 0, B1y = 0, B2x = 0, B2y = 0, B3x = 0, B3y = 0;   // mu_phi rows k-1 .. k-3
        real P3x = 0, P3y = 0, R3x = 0, R3y = 0;          // phi, rho row k-3
        real Fsx = 0, Fsy = 0;                            // south face fluxes of row k-2
        const real *prev = slots + (sidx == 0 ? S - 1 : sidx - 1) * rg.slot_elems + ci;
#pragma unroll kPairUnroll
        for (int j = 0; j < nsl; ++j) {
            const real *cur = slots + sidx * rg.slot_elems + ci;
            PF_DCHECK(sidx >= 0 && sidx < S && ci >= 1 && (R - 1) * bx + 2 * plane + ci + 2 < rg.in_elems + 64);
            const long long tw0 = PF_TRACE ? gtimer() : 0;
            mbar_wait(&full[sidx], par);
            if (PF_TRACE && vb == kTraceBlock && lane == 0 && cw < 4 && gtr < (uint32_t)kTraceBoxes) {
                g_ptrace[cw][gtr][0] = tw0;
                g_ptrace[cw][gtr][1] = gtimer();
            }
            ++gtr;
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const int i = j * R + u;                  // row k = ya - 2 + i
                const real *rk = cur + u * bx;
                const real *rk1 = u >= 1 ? cur + (u - 1) * bx : prev + (R - 1) * bx;
                const real *rk2 = u >= 2 ? cur + (u - 2) * bx : prev + (R - 2 + u) * bx;
                const auto c0 = ld2(rk), c1 = ld2(rk1), c2 = ld2(rk2);
                const auto p0 = ld2(rk + plane), p1 = ld2(rk1 + plane), p2 = ld2(rk2 + plane);
                const auto r1 = ld2(rk1 + 2 * plane), r2 = ld2(rk2 + 2 * plane);
                // x-neighbours one column outside the lane's pair: the adjacent lanes' values
                // (lane 0's left and lane 31's right column only feed halo results)
                real cw1, ce1, pw1, pe1, pw2, pe2, rw2, re2;
                if (kSinglesShfl) {
                    cw1 = __shfl_up_sync(0xffffffffu, c1.y, 1);
                    ce1 = __shfl_down_sync(0xffffffffu, c1.x, 1);
                    pw1 = __shfl_up_sync(0xffffffffu, p1.y, 1);
                    pe1 = __shfl_down_sync(0xffffffffu, p1.x, 1);
                    pw2 = __shfl_up_sync(0xffffffffu, p2.y, 1);
                    pe2 = __shfl_down_sync(0xffffffffu, p2.x, 1);
                    rw2 = __shfl_up_sync(0xffffffffu, r2.y, 1);
                    re2 = __shfl_down_sync(0xffffffffu, r2.x, 1);
                } else {
                    cw1 = rk1[-1]; ce1 = rk1[2]; pw1 = rk1[plane - 1]; pe1 = rk1[plane + 2];
                    pw2 = rk2[plane - 1]; pe2 = rk2[plane + 2]; rw2 = rk2[2 * plane - 1]; re2 = rk2[2 * plane + 2];
                }
                // rotate the windows: row k-1 of the last iteration is row k-2 now
                A2x = A1x; A2y = A1y; M2x = M1x; M2y = M1y;
                B3x = B2x; B3y = B2y; B2x = B1x; B2y = B1y;
                // a2: mu_c, mu_phi, M of row k-1 at both columns
                constitutive<real, MOB, FE>(k, mo, etab, c1.x, p1.x, cw1, c1.y, c2.x, c0.x, pw1, p1.y, p2.x,
                                         p0.x, A1x, B1x, M1x);
                constitutive<real, MOB, FE>(k, mo, etab, c1.y, p1.y, c1.x, ce1, c2.y, c0.y, p1.x, pe1, p2.y,
                                         p0.y, A1y, B1y, M1y);
                // a3-a5: update of row k-2.  x faces: (a, a+1) in lane, (a+1, next a) by shuffle,
                // the west face of a is the previous lane's east face of its right column.
                const real An = __shfl_down_sync(0xffffffffu, A2x, 1);
                const real Mn = __shfl_down_sync(0xffffffffu, M2x, 1);
                const real Bn = __shfl_down_sync(0xffffffffu, B2x, 1);
                const real Bp = __shfl_up_sync(0xffffffffu, B2y, 1);
                const real fex = face_flux<real>(M2x, M2y, A2x, A2y);
                const real fey = face_flux<real>(M2y, Mn, A2y, An);
                const real fwx = __shfl_up_sync(0xffffffffu, fey, 1);
                const real fnx = face_flux<real>(M2x, M1x, A2x, A1x);
                const real fny = face_flux<real>(M2y, M1y, A2y, A1y);
                real bcx = c2.x, bcy = c2.y, bpx = p2.x, bpy = p2.y, brx = r2.x, bry = r2.y;
                if (BASE) {
                    const real *bs = cur + rg.in_elems + u * bx;
                    const auto b0 = ld2(bs), b1 = ld2(bs + plane), b2 = ld2(bs + 2 * plane);
                    bcx = b0.x; bcy = b0.y; bpx = b1.x; bpy = b1.y; brx = b2.x; bry = b2.y;
                }
                real ocx, opx, orx, ocy, opy, ory;
                cell_update<real>(k, vx, vy, fex, fwx, fnx, Fsx, B2x, Bp, B2y, B3x, B1x, pw2, p2.y, P3x,
                                  p1.x, r2.x, rw2, r2.y, R3x, r1.x, bcx, bpx, brx, ocx, opx, orx);
                cell_update<real>(k, vx, vy, fey, fex, fny, Fsy, B2y, B2x, Bn, B3y, B1y, p2.x, pe2, P3y,
                                  p1.y, r2.y, r2.x, re2, R3y, r1.y, bcy, bpy, bry, ocy, opy, ory);
                Fsx = fnx; Fsy = fny;
                P3x = p2.x; P3y = p2.y; R3x = r2.x; R3y = r2.y;
                if (store && i >= 4 && i < n) {
                    const int r = sg.ya - 4 + i;          // local row k-2
                    PF_DCHECK(sg.m >= L.m0 && sg.m < L.m0 + L.members && r >= L.r0 && r < L.r1 && x >= 0 && x + 1 < nx);
                    store_pair_ghosts<real>(L, ob, r, x, xedge, ocx, ocy, opx, opy, orx, ory);
                }
            }
            // the previous box is no longer read (its last row was row k-2 of iteration jR+1)
            __syncwarp();
            if (j >= 1 && lane == 0) mbar_arrive(&empty[sidx == 0 ? S - 1 : sidx - 1]);
            prev = cur;
            if (++sidx == S) { sidx = 0; par ^= 1u; }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[sidx == 0 ? S - 1 : sidx - 1]);   // the segment's last box
    }
    if (PF_TRACE && cw == 0 && lane == 0 && vb < 1024) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_bspan[vb][2] = gtimer();
        g_bspan[vb][1] = (long long)sm;
    }
}

// ----------------------------------------------------------------------------------------
// Warp-specialised step kernel (kernel_path 5): one pass per explicit-midpoint STEP through an
// on-chip pipeline, u^n read once and u^{n+1} written once (48 B per fp64 cell-step):
//   producer warp --TMA 1-row boxes of u^n--> input ring
//   NCW stage-1 warps (the pair kernel's arithmetic with coef dt/2): u*(k-2) from input rows
//       k .. k-2; they write u* and the base u^n of that row (6 planes) into a u* ring in shared
//       memory, each warp its 60 columns [60 w - 2, 60 w + 58) of the strip
//   NCW stage-2 warps (the pair kernel's arithmetic with coef dt): u^{n+1}(q-2) from u* rows
//       q .. q-2 of the u* ring, stored to HBM with the ghost frame.
// Both stages keep the pair kernel's register footprint (each warp runs one stage), so the SM
// holds as many compute warps as the two-pass path while HBM traffic drops from 120 to 48 B per
// cell-step.  At the global y boundaries stage 2 substitutes the identities the two-pass kernels
// get from u*'s mirrored ghost rows (zero boundary flux, mu_phi(-1) = mu_phi(0), phi*(-1) = phi*(0),
// rho*(-1) = rho*(0), rho* above the top = the reservoir row), so results are bitwise those of
// the stage kernels.  Single-domain contexts only.
__host__ __device__ constexpr int ws_packed_cap(int V, int NCW) { return (65536 / (128 + 64 * V * NCW)) / 8 * 8; }
__host__ __device__ constexpr int ws_packed_regs(int V, int NCW) {
    return ((ws_packed_cap(V, NCW) * (128 + 64 * V * NCW) - 24 * 128) / (64 * V * NCW)) / 8 * 8 > 248
               ? 248
               : ((ws_packed_cap(V, NCW) * (128 + 64 * V * NCW) - 24 * 128) / (64 * V * NCW)) / 8 * 8;
}

// Packed variant (V > 1): as pair_kernel's -- V blocks per CTA, their producers in warpgroup 0
// (setmaxnreg.dec), their 2 NCW compute warps each in the other warpgroups (setmaxnreg.inc).
template <typename real, int NCW, int SI, int SU, int MOB, int FE, int MINB, int V>
__global__ void __launch_bounds__(V == 1 ? 32 * (2 * NCW + 1) : 128 + 64 * V * NCW, V == 1 ? MINB : 1) ws_kernel(
    Layout L, KC<real> k, KC<real> k2, const __grid_constant__ CUtensorMap mapIn, real *out,
    const real *__restrict__ vel, int Wo, int G, int NB) {
    static_assert(V == 1 || (V <= 4 && (2 * V * NCW) % 4 == 0), "packed blocks fill whole warpgroups");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int bx = Wo + 2 * kPairHalo;
    const int in_el = ((3 * bx * (int)sizeof(real) + 127) / 128 * 128) / (int)sizeof(real);
    const int us_el = ((6 * bx * (int)sizeof(real) + 127) / 128 * 128) / (int)sizeof(real);
    unsigned char *base_sm = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    const bool producer = V == 1 ? warp == 2 * NCW : warp < 4;
    const int v = V == 1 ? 0 : (producer ? warp : (warp - 4) / (2 * NCW));
    const int cw = V == 1 ? warp : (warp - 4) - v * 2 * NCW;   // < NCW: stage-1 warp, else stage 2
    const size_t vbytes = ((size_t)SI * in_el * sizeof(real) + (size_t)SU * us_el * sizeof(real) + 64 * sizeof(real) +
                           (size_t)(2 * SI + 2 * SU) * 8 + 127) / 128 * 128;
    unsigned char *reg = V == 1 ? base_sm : base_sm + 64 * 8 + (size_t)(v < V ? v : 0) * vbytes;
    real *ring = reinterpret_cast<real *>(reg);
    real *usr = ring + (size_t)SI * in_el;
    uint64_t *full_in = reinterpret_cast<uint64_t *>(usr + (size_t)SU * us_el + 64);
    uint64_t *empty_in = full_in + SI;
    uint64_t *us_full = empty_in + SI;
    uint64_t *us_empty = us_full + SU;
    double *etab = V == 1 ? reinterpret_cast<double *>(us_empty + SU) : reinterpret_cast<double *>(base_sm);
    load_exp_table(etab);

    if (V == 1 ? t == 0 : (producer && warp < V && lane == 0)) {
        for (int q = 0; q < SI; ++q) {
            mbar_init(&full_in[q], 1);
            mbar_init(&empty_in[q], NCW);
        }
        for (int q = 0; q < SU; ++q) {
            mbar_init(&us_full[q], NCW);
            mbar_init(&us_empty[q], NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    const int nx = L.nx;
    const int vb = V == 1 ? (int)blockIdx.x : (int)blockIdx.x * V + v;
    const uint32_t box_bytes = (uint32_t)(3 * bx * sizeof(real));
    constexpr int LEAD = 4, TRAIL = 4;
    const unsigned FULL = 0xffffffffu;

    if (producer) {
        // ------------------------------- producer -------------------------------
        if (V > 1) asm volatile("setmaxnreg.dec.sync.aligned.u32 24;" ::: "memory");
        if (lane != 0 || v >= V) return;
        const Sched sch = make_sched(L, Wo, G, vb, NB);
        prefetch_tmap(&mapIn);
        uint32_t g = 0;
        int64_t pos = sch.lo;
        Seg sg;
        while (next_seg(L, Wo, sch, pos, sg)) {
            const int n = sg.yb - sg.ya + LEAD + TRAIL;
            const int bxs = sg.x0 - kPairHalo + L.gx;
            for (int j = 0; j < n; ++j, ++g) {
                const int slot = g % SI;
                if (g >= (uint32_t)SI) mbar_wait(&empty_in[slot], ((g / SI) - 1) & 1u);
                mbar_expect_tx(&full_in[slot], box_bytes);
                tma_load_3d(ring + slot * in_el, &mapIn, bxs, sg.ya - LEAD + j + 2, 3 * sg.m, &full_in[slot]);
            }
        }
        return;
    }

    if (V > 1) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(ws_packed_regs(V, NCW)) : "memory");
    const Sched sch = make_sched(L, Wo, G, vb, NB);
    if (cw < NCW) {
        // --------------------------- stage-1 warps ------------------------------
        const int cx = kPairCols * cw + 2 * lane - 4;         // strip column of the lane's left column
        const int ci = kPairHalo + cx;
        const bool wr = lane >= 1 && lane <= 30;               // writes u* columns [60 w - 2, 60 w + 58)
        int sidx = 0, uidx = 0;
        uint32_t par = 0, upar = 0;
        uint32_t ucount = 0;
        int64_t pos = sch.lo;
        Seg sg;
        while (next_seg(L, Wo, sch, pos, sg)) {
            const int n = sg.yb - sg.ya + LEAD + TRAIL;
            real vx, vy;
        scaled_velocity(k, vel, sg.m, vx, vy);
            const Mob<real> mo = MOB == 2 ? load_mob(vel, sg.m) : Mob<real>{};
            real A1x = 0, A1y = 0, A2x = 0, A2y = 0, M1x = 0, M1y = 0, M2x = 0, M2y = 0;
            real B1x = 0, B1y = 0, B2x = 0, B2y = 0, B3x = 0, B3y = 0, P3x = 0, P3y = 0, R3x = 0, R3y = 0;
            real Fsx = 0, Fsy = 0;
            const real *r1 = nullptr, *r2 = nullptr;
            for (int i = 0; i < n; ++i) {
                const real *r0 = ring + sidx * in_el + ci;
                mbar_wait(&full_in[sidx], par);
                if (i >= 2) {
                    const auto c0 = ld2(r0), c1 = ld2(r1), c2 = ld2(r2);
                    const auto p0 = ld2(r0 + bx), p1 = ld2(r1 + bx), p2 = ld2(r2 + bx);
                    const auto q1 = ld2(r1 + 2 * bx), q2 = ld2(r2 + 2 * bx);
                    const real cw1 = __shfl_up_sync(FULL, c1.y, 1), ce1 = __shfl_down_sync(FULL, c1.x, 1);
                    const real pw1 = __shfl_up_sync(FULL, p1.y, 1), pe1 = __shfl_down_sync(FULL, p1.x, 1);
                    const real pw2 = __shfl_up_sync(FULL, p2.y, 1), pe2 = __shfl_down_sync(FULL, p2.x, 1);
                    const real rw2 = __shfl_up_sync(FULL, q2.y, 1), re2 = __shfl_down_sync(FULL, q2.x, 1);
                    A2x = A1x; A2y = A1y; M2x = M1x; M2y = M1y;
                    B3x = B2x; B3y = B2y; B2x = B1x; B2y = B1y;
                    constitutive<real, MOB, FE>(k, mo, etab, c1.x, p1.x, cw1, c1.y, c2.x, c0.x, pw1, p1.y, p2.x,
                                                p0.x, A1x, B1x, M1x);
                    constitutive<real, MOB, FE>(k, mo, etab, c1.y, p1.y, c1.x, ce1, c2.y, c0.y, p1.x, pe1, p2.y,
                                                p0.y, A1y, B1y, M1y);
                    const real An = __shfl_down_sync(FULL, A2x, 1), Mn = __shfl_down_sync(FULL, M2x, 1);
                    const real Bn = __shfl_down_sync(FULL, B2x, 1), Bp = __shfl_up_sync(FULL, B2y, 1);
                    const real fex = face_flux<real>(M2x, M2y, A2x, A2y);
                    const real fey = face_flux<real>(M2y, Mn, A2y, An);
                    const real fwx = __shfl_up_sync(FULL, fey, 1);
                    const real fnx = face_flux<real>(M2x, M1x, A2x, A1x);
                    const real fny = face_flux<real>(M2y, M1y, A2y, A1y);
                    real csx, psx, rsx, csy, psy, rsy;
                    cell_update<real>(k, vx, vy, fex, fwx, fnx, Fsx, B2x, Bp, B2y, B3x, B1x, pw2, p2.y, P3x, p1.x,
                                      q2.x, rw2, q2.y, R3x, q1.x, c2.x, p2.x, q2.x, csx, psx, rsx);
                    cell_update<real>(k, vx, vy, fey, fex, fny, Fsy, B2y, B2x, Bn, B3y, B1y, p2.x, pe2, P3y, p1.y,
                                      q2.y, q2.x, re2, R3y, q1.y, c2.y, p2.y, q2.y, csy, psy, rsy);
                    Fsx = fnx; Fsy = fny;
                    P3x = p2.x; P3y = p2.y; R3x = q2.x; R3y = q2.y;
                    if (i >= LEAD) {          // u* row k-2 (and its base u^n row) into the u* ring
                        if (ucount >= (uint32_t)SU) mbar_wait(&us_empty[uidx], upar ^ 1u);
                        if (wr) {
                            real *u = usr + uidx * us_el + ci;
                            st2(u, csx, csy);
                            st2(u + bx, psx, psy);
                            st2(u + 2 * bx, rsx, rsy);
                            st2(u + 3 * bx, c2.x, c2.y);
                            st2(u + 4 * bx, p2.x, p2.y);
                            st2(u + 5 * bx, q2.x, q2.y);
                        }
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&us_full[uidx]);
                        ++ucount;
                        if (++uidx == SU) { uidx = 0; upar ^= 1u; }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty_in[sidx >= 2 ? sidx - 2 : sidx - 2 + SI]);   // row k-2 done
                }
                r2 = r1; r1 = r0;
                if (++sidx == SI) { sidx = 0; par ^= 1u; }
            }
            __syncwarp();
            if (lane == 0) {   // rows k-1, k of the segment's last iteration
                mbar_arrive(&empty_in[sidx >= 1 ? sidx - 1 : sidx - 1 + SI]);
                mbar_arrive(&empty_in[sidx >= 2 ? sidx - 2 : sidx - 2 + SI]);
            }
        }
        return;
    }

    // --------------------------- stage-2 warps ---------------------------------
    const int w2 = cw - NCW;
    const int cx = kPairCols * w2 + 2 * lane - 2;
    const int ci = kPairHalo + cx;
    int uidx = 0;
    uint32_t upar = 0;
    int64_t pos = sch.lo;
    Seg sg;
    while (next_seg(L, Wo, sch, pos, sg)) {
        const int n = sg.yb - sg.ya + 4;                 // u* rows ya-2 .. yb+1
        const int x = sg.x0 + cx;
        const bool store = lane >= 1 && lane <= 30 && cx < sg.Wp;
        const bool xedge = (x < L.gx) | (x + 1 >= nx - L.gx);
        real *ob = out + sg.m * L.mstride;
        real vx, vy;
        scaled_velocity(k, vel, sg.m, vx, vy);
        const Mob<real> mo = MOB == 2 ? load_mob(vel, sg.m) : Mob<real>{};
        real A1x = 0, A1y = 0, A2x = 0, A2y = 0, M1x = 0, M1y = 0, M2x = 0, M2y = 0;
        real B1x = 0, B1y = 0, B2x = 0, B2y = 0, B3x = 0, B3y = 0, P3x = 0, P3y = 0, R3x = 0, R3y = 0;
        real Fsx = 0, Fsy = 0;
        const real *r1 = nullptr, *r2 = nullptr;
        for (int i = 0; i < n; ++i) {
            const real *r0 = usr + uidx * us_el + ci;    // u* row q = ya - 2 + i
            mbar_wait(&us_full[uidx], upar);
            if (i >= 2) {
                const int q = sg.ya - 2 + i;
                const int gq = L.y0 + q - 1, gu = L.y0 + q - 2;   // global rows of mu2 and of the update
                const bool qbot = gq == 0, qtop = gq == L.ny - 1, ubot = gu == 0, utop = gu == L.ny - 1;
                const auto c0 = ld2(r0), c1 = ld2(r1), c2 = ld2(r2);
                const auto p0 = ld2(r0 + bx), p1 = ld2(r1 + bx), p2 = ld2(r2 + bx);
                const auto q1 = ld2(r1 + 2 * bx), q2 = ld2(r2 + 2 * bx);
                const real cw1 = __shfl_up_sync(FULL, c1.y, 1), ce1 = __shfl_down_sync(FULL, c1.x, 1);
                const real pw1 = __shfl_up_sync(FULL, p1.y, 1), pe1 = __shfl_down_sync(FULL, p1.x, 1);
                const real pw2 = __shfl_up_sync(FULL, p2.y, 1), pe2 = __shfl_down_sync(FULL, p2.x, 1);
                const real rw2 = __shfl_up_sync(FULL, q2.y, 1), re2 = __shfl_down_sync(FULL, q2.x, 1);
                // mu2 at row q-1: its down / up neighbour rows are mirrors at the global boundaries
                const real cdx = qbot ? c1.x : c2.x, cdy = qbot ? c1.y : c2.y, cux = qtop ? c1.x : c0.x,
                           cuy = qtop ? c1.y : c0.y;
                const real pdx = qbot ? p1.x : p2.x, pdy = qbot ? p1.y : p2.y, pux = qtop ? p1.x : p0.x,
                           puy = qtop ? p1.y : p0.y;
                A2x = A1x; A2y = A1y; M2x = M1x; M2y = M1y;
                B3x = B2x; B3y = B2y; B2x = B1x; B2y = B1y;
                constitutive<real, MOB, FE>(k, mo, etab, c1.x, p1.x, cw1, c1.y, cdx, cux, pw1, p1.y, pdx, pux, A1x,
                                            B1x, M1x);
                constitutive<real, MOB, FE>(k, mo, etab, c1.y, p1.y, c1.x, ce1, cdy, cuy, p1.x, pe1, pdy, puy, A1y,
                                            B1y, M1y);
                const real An = __shfl_down_sync(FULL, A2x, 1), Mn = __shfl_down_sync(FULL, M2x, 1);
                const real Bn = __shfl_down_sync(FULL, B2x, 1), Bp = __shfl_up_sync(FULL, B2y, 1);
                const real fex = face_flux<real>(M2x, M2y, A2x, A2y);
                const real fey = face_flux<real>(M2y, Mn, A2y, An);
                const real fwx = __shfl_up_sync(FULL, fey, 1);
                real fnx = face_flux<real>(M2x, M1x, A2x, A1x), fny = face_flux<real>(M2y, M1y, A2y, A1y);
                if (utop) { fnx = real(0); fny = real(0); }
                const real fsx = ubot ? real(0) : Fsx, fsy = ubot ? real(0) : Fsy;
                Fsx = fnx; Fsy = fny;
                const real qdx = ubot ? B2x : B3x, qdy = ubot ? B2y : B3y;
                const real qux = utop ? B2x : B1x, quy = utop ? B2y : B1y;
                const real phdx = ubot ? p2.x : P3x, phdy = ubot ? p2.y : P3y;
                const real phux = utop ? p2.x : p1.x, phuy = utop ? p2.y : p1.y;
                const auto rt = ld2(r1 + 5 * bx);            // base rho of row q-1: the reservoir if utop
                const real rdx = ubot ? q2.x : R3x, rdy = ubot ? q2.y : R3y;
                const real rux = utop ? rt.x : q1.x, ruy = utop ? rt.y : q1.y;
                const auto b0 = ld2(r2 + 3 * bx), b1 = ld2(r2 + 4 * bx), b2 = ld2(r2 + 5 * bx);   // u^n row q-2
                real ocx, opx, orx, ocy, opy, ory;
                cell_update<real>(k2, vx, vy, fex, fwx, fnx, fsx, B2x, Bp, B2y, qdx, qux, pw2, p2.y, phdx, phux,
                                  q2.x, rw2, q2.y, rdx, rux, b0.x, b1.x, b2.x, ocx, opx, orx);
                cell_update<real>(k2, vx, vy, fey, fex, fny, fsy, B2y, B2x, Bn, qdy, quy, p2.x, pe2, phdy, phuy,
                                  q2.y, q2.x, re2, rdy, ruy, b0.y, b1.y, b2.y, ocy, opy, ory);
                P3x = p2.x; P3y = p2.y; R3x = q2.x; R3y = q2.y;
                const int r = q - 2;
                if (store && r >= sg.ya && r < sg.yb) {
                    PF_DCHECK(sg.m >= L.m0 && sg.m < L.m0 + L.members && r >= L.r0 && r < L.r1 && x >= 0 && x + 1 < nx);
                    store_pair_ghosts<real>(L, ob, r, x, xedge, ocx, ocy, opx, opy, orx, ory);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&us_empty[uidx >= 2 ? uidx - 2 : uidx - 2 + SU]);   // row q-2 done
            }
            r2 = r1; r1 = r0;
            if (++uidx == SU) { uidx = 0; upar ^= 1u; }
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&us_empty[uidx >= 1 ? uidx - 1 : uidx - 1 + SU]);
            mbar_arrive(&us_empty[uidx >= 2 ? uidx - 2 : uidx - 2 + SU]);
        }
    }
}


// Pair kernel ring geometry per precision, stage and producer mode: about 128 registers per
// thread, so MINB = wslots / (warps per block) blocks fill the register file with 15-16 compute
// warps per SM (12-16 with the producer warp); rings of 2-row boxes as deep as the shared memory
// left to each of the MINB blocks allows (at most 8 boxes, at least 3: the box being read, the
// previous one, and one in flight).
#ifndef PF_F32_SLOTS
#define PF_F32_SLOTS 20
#endif
constexpr int kF32Slots = PF_F32_SLOTS;
#ifndef PF_F64_SLOTS
#define PF_F64_SLOTS 16
#endif
#ifndef PF_PAIR_R1
#define PF_PAIR_R1 2
#endif
#ifndef PF_PAIR_R2
#define PF_PAIR_R2 2
#endif
#ifndef PF_PAIR_WG
#define PF_PAIR_WG 2        // packed pair blocks (setmaxnreg): 0 off, 1 fp64, 2 fp64 + fp32 stage 1
#endif
#ifndef PF_S1_SMEM_KB
#define PF_S1_SMEM_KB 150   // fp64 stage-1 shared-memory budget per SM
#endif
template <typename real, int NCW, bool BASE>
struct PairCfg {
    static constexpr int R = BASE ? PF_PAIR_R2 : PF_PAIR_R1;   // rows per TMA box
    static constexpr int bx_max = kPairCols * NCW + 2 * kPairHalo;
    static constexpr int slot = (3 * R * bx_max * (int)sizeof(real) + 127) / 128 * 128 * (BASE ? 2 : 1);
    // fp64 stage 1 keeps its ring small (>= 3 boxes) to leave L1 to the output stores: measured
    // 4-5% faster than filling the shared memory (r1)
    static constexpr int smem_kb = (sizeof(real) == 8 && !BASE) ? PF_S1_SMEM_KB : 227;
    static constexpr int ring_raw(int b) { return ((smem_kb * 1024) / b - 2048) / slot; }
    static constexpr int ring(int b) { return (!BASE && sizeof(real) == 8 && ring_raw(b) < 3) ? 3 : ring_raw(b); }
    static constexpr int pick(int b) { return b <= 1 || ring(b) >= 3 ? b : pick(b - 1); }
    static constexpr int wslots = sizeof(real) == 8 ? PF_F64_SLOTS : kF32Slots;   // warp slots per SM budget
    static constexpr int wpb = NCW + 1;                                            // warps per block (+ producer)
    static constexpr int minb = pick(wslots / wpb > 8 ? 8 : wslots / wpb);
    static constexpr int S = ring(minb) > 8 ? 8 : ring(minb);
    static_assert(S >= 3, "ring too shallow");
    // packed blocks (pair_kernel V > 1): the minb blocks of an SM as one CTA when their compute
    // warps fill whole warpgroups.  Measured (one B200, tools/kbench.py, gpurun_out r2wg2): fp64
    // stage 1 -8% (cfg3) / -10.5% (cfg4), stage 2 -1%; fp32 (16 compute warps, 112 instead of 96
    // registers) stage 1 -6%, stage 2 +1% -- so fp32 packs stage 1 only.
    static constexpr bool pack = sizeof(real) == 8 ? PF_PAIR_WG >= 1 : (PF_PAIR_WG >= 2 && !BASE);
    static constexpr int V = (pack && minb > 1 && minb <= 4 && (minb * NCW) % 4 == 0) ? minb : 1;
};

template <typename real, int NCW, bool BASE, int MOB, int FE>
cudaError_t launch_pair_k(const Layout &L, const StreamPlan &P, const KC<real> &k, int stage, real *out,
                          const real *vel, cudaStream_t s) {
    using C = PairCfg<real, NCW, BASE>;
    constexpr int R = C::R, S = C::S, MINB = C::minb, V = C::V;
    const size_t smem = V == 1 ? stream_smem_bytes<real>(P.box_x, R, S, BASE)
                               : pair_packed_smem_bytes<real>(P.box_x, R, S, BASE, V);
    const int threads = V == 1 ? 32 * C::wpb : 128 + 32 * V * NCW;
    static int occ = -1, nsm = 0;
    static size_t smem_set = 0;
    auto kern = pair_kernel<real, NCW, R, S, BASE, MOB, FE, MINB, V>;
    if (smem > smem_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        smem_set = smem;
        occ = -1;
    }
    if (occ < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (V > 1) {   // the compute warps' setmaxnreg.inc must be satisfiable from the CTA's pool
            cudaFuncAttributes fa;
            cudaError_t e = cudaFuncGetAttributes(&fa, kern);
            if (e != cudaSuccess) return e;
            if (fa.numRegs * threads - 24 * 128 < pair_packed_regs(V, NCW) * 32 * V * NCW) return cudaErrorInvalidConfiguration;
        }
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
    }
    const int64_t R_ = (int64_t)L.members * P.strips * L.rows();
    const int64_t minrows = 16;
    int64_t B = (int64_t)occ * nsm * V;   // (virtual) blocks
    static const int nogroup = env_int("PF_STREAM_NOGROUP", 0);
    // grouped schedule when at least 4 groups of `strips` blocks fit in one resident wave
    int64_t G = B / P.strips;
    const int64_t T = (int64_t)L.members * L.rows();
    if (G > (T + minrows - 1) / minrows) G = (T + minrows - 1) / minrows;
    if (G >= 4 && !nogroup) {
        B = G * P.strips;
    } else {
        G = 0;
        // >= 16 rows per block, but never fewer blocks than (member, strip) windows: a 2-row
        // boundary band of the slab overlap schedule (4096 wide: 18 strips) otherwise ran on 3
        // blocks, 6 strips each back to back (~28 us per band launch, gpurun_out r2s3b)
        int64_t cap = (R_ + minrows - 1) / minrows;
        // (both bands in one launch, Layout::g0: a block per band and strip)
        const int64_t windows = (int64_t)L.members * P.strips * (L.g1 > L.g0 ? 2 : 1);
        if (cap < windows) cap = windows;
        if (B > cap) B = cap;
    }
    if (B < 1) B = 1;
    const int NB = (int)B;
    B = (B + V - 1) / V;                   // CTAs
    const int ri = R == 4 ? 1 : 0;
    const CUtensorMap &mIn = stage == 1 ? P.mapU[ri] : P.mapUs[ri];
    static const int pdl = env_int("PF_PDL", 1);
    if (pdl) {   // programmatic dependent launch (pair_kernel waits in-kernel)
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.gridDim = dim3((unsigned)B);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, L, k, mIn, P.mapU[ri], out, vel, P.Wo, (int)G, NB);
    }
    kern<<<(unsigned)B, threads, smem, s>>>(L, k, mIn, P.mapU[ri], out, vel, P.Wo, (int)G, NB);
    return cudaGetLastError();
}

template <typename real, int NCW, bool BASE>
cudaError_t launch_pair_h(const Layout &L, const StreamPlan &P, const KC<real> &k, int stage, real *out,
                          const real *vel, cudaStream_t s) {
    if (k.fe == 1) {
        switch (k.mob) {
            case 0: return launch_pair_k<real, NCW, BASE, 0, 1>(L, P, k, stage, out, vel, s);
            case 1: return launch_pair_k<real, NCW, BASE, 1, 1>(L, P, k, stage, out, vel, s);
            default: return launch_pair_k<real, NCW, BASE, 2, 1>(L, P, k, stage, out, vel, s);
        }
    }
    switch (k.mob) {
        case 0: return launch_pair_k<real, NCW, BASE, 0, 0>(L, P, k, stage, out, vel, s);
        case 1: return launch_pair_k<real, NCW, BASE, 1, 0>(L, P, k, stage, out, vel, s);
        default: return launch_pair_k<real, NCW, BASE, 2, 0>(L, P, k, stage, out, vel, s);
    }
}

// One stage of the pair kernel (both precisions, both stages: a separate compilation part each,
// see build.py).
template <typename real, bool BASE>
cudaError_t launch_pair(const Layout &L, const StreamPlan &P, const KC<real> &k, int stage, real *out,
                        const real *vel, cudaStream_t s) {
    switch (P.ncw) {
        case 1: return launch_pair_h<real, 1, BASE>(L, P, k, stage, out, vel, s);
        case 2: return launch_pair_h<real, 2, BASE>(L, P, k, stage, out, vel, s);
        case 3: return launch_pair_h<real, 3, BASE>(L, P, k, stage, out, vel, s);
        case 4: return launch_pair_h<real, 4, BASE>(L, P, k, stage, out, vel, s);
        default: return cudaErrorInvalidValue;
    }
}

// Warp-specialised step kernel: NCW stage-1 + NCW stage-2 warps + 1 producer per block.
#ifndef PF_WS_WG
#define PF_WS_WG 1          // packed ws blocks (setmaxnreg), fp64
#endif
template <typename real, int NCW>
struct WsCfg {
    static constexpr int minb = NCW <= 2 ? 3 : 2;
    static constexpr int SI = 8, SU = 6;
    static constexpr int V = (PF_WS_WG && sizeof(real) == 8 && (2 * minb * NCW) % 4 == 0) ? minb : 1;
};

template <typename real>
size_t ws_smem_bytes(int bx, int SI, int SU, int V) {
    const size_t in_b = (3 * bx * sizeof(real) + 127) / 128 * 128, us_b = (6 * bx * sizeof(real) + 127) / 128 * 128;
    if (V > 1)
        return 128 + 64 * 8 +
               (size_t)V * ((SI * in_b + SU * us_b + 64 * sizeof(real) + (size_t)(2 * SI + 2 * SU) * 8 + 127) / 128 * 128);
    return 128 + SI * in_b + SU * us_b + 64 * sizeof(real) + (size_t)(2 * SI + 2 * SU) * 8 + 64 * 8;
}

template <typename real, int NCW, int MOB, int FE>
cudaError_t launch_ws_k(const Layout &L, const StreamPlan &P, const KC<real> &k, const KC<real> &k2, real *out,
                        const real *vel, cudaStream_t s) {
    using C = WsCfg<real, NCW>;
    constexpr int V = C::V;
    const size_t smem = ws_smem_bytes<real>(P.fbox, C::SI, C::SU, V);
    static int occ = -1, nsm = 0;
    static size_t smem_set = 0;
    auto kern = ws_kernel<real, NCW, C::SI, C::SU, MOB, FE, C::minb, V>;
    const int threads = V == 1 ? 32 * (2 * NCW + 1) : 128 + 64 * V * NCW;
    if (smem > smem_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        smem_set = smem;
        occ = -1;
    }
    if (occ < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (V > 1) {   // the compute warps' setmaxnreg.inc must be satisfiable from the CTA's pool
            cudaFuncAttributes fa;
            cudaError_t e = cudaFuncGetAttributes(&fa, kern);
            if (e != cudaSuccess) return e;
            if (fa.numRegs * threads - 24 * 128 < ws_packed_regs(V, NCW) * 64 * V * NCW) return cudaErrorInvalidConfiguration;
        }
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
    }
    const int64_t T = (int64_t)L.members * (L.r1 - L.r0);
    const int64_t minrows = 24;
    int64_t B = (int64_t)occ * nsm * V;   // (virtual) blocks
    int64_t G = B / P.fstrips;
    if (G > (T + minrows - 1) / minrows) G = (T + minrows - 1) / minrows;
    if (G >= 4) {
        B = G * P.fstrips;
    } else {
        G = 0;
        const int64_t R_ = (int64_t)L.members * P.fstrips * (L.r1 - L.r0);
        if (B > (R_ + minrows - 1) / minrows) B = (R_ + minrows - 1) / minrows;
    }
    if (B < 1) B = 1;
    const int NB = (int)B;
    B = (B + V - 1) / V;
    kern<<<(unsigned)B, threads, smem, s>>>(L, k, k2, P.fmapU, out, vel, P.fWo, (int)G, NB);
    return cudaGetLastError();
}

template <typename real, int NCW>
cudaError_t launch_ws_n(const Layout &L, const StreamPlan &P, const KC<real> &k, const KC<real> &k2, real *out,
                        const real *vel, cudaStream_t s) {
    if (k.fe == 1) {
        switch (k.mob) {
            case 0: return launch_ws_k<real, NCW, 0, 1>(L, P, k, k2, out, vel, s);
            case 1: return launch_ws_k<real, NCW, 1, 1>(L, P, k, k2, out, vel, s);
            default: return launch_ws_k<real, NCW, 2, 1>(L, P, k, k2, out, vel, s);
        }
    }
    switch (k.mob) {
        case 0: return launch_ws_k<real, NCW, 0, 0>(L, P, k, k2, out, vel, s);
        case 1: return launch_ws_k<real, NCW, 1, 0>(L, P, k, k2, out, vel, s);
        default: return launch_ws_k<real, NCW, 2, 0>(L, P, k, k2, out, vel, s);
    }
}

cudaError_t upload_exp_table() {
    static bool done = false;
    if (done) return cudaSuccess;
    double t[64];
    for (int j = 0; j < 64; ++j) t[j] = exp2((double)j / 64.0);
    cudaError_t e = cudaMemcpyToSymbol(kExp2Tab, t, sizeof t);
    if (e == cudaSuccess) done = true;
    return e;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

bool encode_map(CUtensorMap *m, int precision, const Layout &L, void *buf, int box_x, int rows) {
    auto enc = get_encode();
    if (!enc) return false;
    const size_t esz = precision == 0 ? 8 : 4;
    cuuint64_t dims[3] = {(cuuint64_t)L.pitch, (cuuint64_t)(L.ny_loc + 4), (cuuint64_t)(3 * L.members)};
    cuuint64_t strides[2] = {(cuuint64_t)L.pitch * esz, (cuuint64_t)L.fstride * esz};
    cuuint32_t box[3] = {(cuuint32_t)box_x, (cuuint32_t)rows, 3};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, precision == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, buf,
                     dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace

#if PF_IN(0)
bool stream_eligible(const Layout &L) { return L.nx >= 16 && L.nx % 4 == 0 && L.ny_loc >= 2; }

cudaError_t make_stream_plan(int precision, const Layout &L, void *U, void *Us, StreamPlan &P) {
    P = StreamPlan();
    if (L.path == 1 || !stream_eligible(L)) return cudaSuccess;   // paths 0, 3, 5: the pair plan
    // pair kernel: strips of Wo <= 240 columns (box Wo + 8 <= 256 elements), Wo a multiple of 4
    // (16 B rows for fp32 too), split nx evenly; 60 output columns per compute warp
    int strips = (L.nx + 239) / 240;
    int Wo = (L.nx + strips - 1) / strips;
    Wo = (Wo + 3) / 4 * 4;
    strips = (L.nx + Wo - 1) / Wo;
    P.kind = 2;
    P.ncw = (Wo + kPairCols - 1) / kPairCols;
    P.Wo = Wo;
    P.strips = strips;
    P.box_x = Wo + 2 * kPairHalo;
    for (int ri = 0; ri < 2; ++ri)
        if (!encode_map(&P.mapU[ri], precision, L, U, P.box_x, ri ? 4 : 2) ||
            !encode_map(&P.mapUs[ri], precision, L, Us, P.box_x, ri ? 4 : 2))
            return cudaErrorInvalidValue;
    P.ok = true;
    if (L.path == 5) {
        // warp-specialised step kernel: strips of 60 NCW - 4 columns (stage-1 warps cover the strip
        // plus 2 columns of u* on each side), NCW in {2, 3} for the least idle columns
        static const int force = env_int("PF_WS_NCW", 0);
        int best = 3;
        if (force == 2 || force == 3) {
            best = force;
        } else {
            const int w3 = kPairCols * 3 - 4, w2 = kPairCols * 2 - 4;
            const int i3 = (L.nx + w3 - 1) / w3 * w3 - L.nx, i2 = (L.nx + w2 - 1) / w2 * w2 - L.nx;
            best = (i2 + L.nx / 40 < i3) ? 2 : 3;
        }
        P.fncw = best;
        P.fWo = kPairCols * best - 4;
        P.fstrips = (L.nx + P.fWo - 1) / P.fWo;
        P.fbox = P.fWo + 2 * kPairHalo;
        if (!encode_map(&P.fmapU, precision, L, U, P.fbox, 1) || !encode_map(&P.fmapUs, precision, L, Us, P.fbox, 1))
            return cudaErrorInvalidValue;
        P.fused = true;
        P.ws = true;
    }
    return cudaSuccess;
}
#endif

#if PF_IN(5)
cudaError_t launch_fused(int precision, const Layout &L, const StreamPlan &P, const Coef &K, void *out, const void *vel,
                         double dt, cudaStream_t s) {
    cudaError_t te = upload_exp_table();
    if (te != cudaSuccess) return te;
    if (!P.fused || !P.ws) return cudaErrorInvalidValue;
    if (precision == 0) {
        const KC<double> k1 = make_kc<double>(K, 0.5 * dt), k2 = make_kc<double>(K, dt);
        return P.fncw == 2 ? launch_ws_n<double, 2>(L, P, k1, k2, (double *)out, (const double *)vel, s)
                           : launch_ws_n<double, 3>(L, P, k1, k2, (double *)out, (const double *)vel, s);
    }
    const KC<float> k1 = make_kc<float>(K, 0.5 * dt), k2 = make_kc<float>(K, dt);
    return P.fncw == 2 ? launch_ws_n<float, 2>(L, P, k1, k2, (float *)out, (const float *)vel, s)
                       : launch_ws_n<float, 3>(L, P, k1, k2, (float *)out, (const float *)vel, s);
}
#endif

// The pair-kernel stage launch of one precision and stage (compilation parts 1-4).
#define PF_PAIR_ENTRY(NAME, REAL, BASE)                                                                          \
    cudaError_t NAME(const Layout &L, const StreamPlan &P, const Coef &K, int stage, void *out, const void *vel,   \
                     double coef, cudaStream_t s) {                                                              \
        cudaError_t te = upload_exp_table();                                                                     \
        if (te != cudaSuccess) return te;                                                                        \
        return launch_pair<REAL, BASE>(L, P, make_kc<REAL>(K, coef), stage, (REAL *)out, (const REAL *)vel, s);  \
    }
cudaError_t pair_stage1_f64(const Layout &, const StreamPlan &, const Coef &, int, void *, const void *, double, cudaStream_t);
cudaError_t pair_stage2_f64(const Layout &, const StreamPlan &, const Coef &, int, void *, const void *, double, cudaStream_t);
cudaError_t pair_stage1_f32(const Layout &, const StreamPlan &, const Coef &, int, void *, const void *, double, cudaStream_t);
cudaError_t pair_stage2_f32(const Layout &, const StreamPlan &, const Coef &, int, void *, const void *, double, cudaStream_t);
#if PF_IN(1)
PF_PAIR_ENTRY(pair_stage1_f64, double, false)
}  // namespace pf
// Diagnostic: the timeline trace of the fp64 stage-1 pair kernel's block kTraceBlock (PF_TRACE
// builds; zeros otherwise): [5 warps (4 compute, producer)][512 boxes][wait start, wait end / issue].
extern "C" int pf_debug_trace(long long *out) {
    return (int)cudaMemcpyFromSymbol(out, pf::g_ptrace, sizeof(pf::g_ptrace));
}
// [1024 blocks][griddep_wait return, SM id, compute warp 0's end] (PF_TRACE builds; zeros otherwise)
extern "C" int pf_debug_block_spans(long long *out) {
    return (int)cudaMemcpyFromSymbol(out, pf::g_bspan, sizeof(pf::g_bspan));
}
namespace pf {
#endif
#if PF_IN(2)
PF_PAIR_ENTRY(pair_stage2_f64, double, true)
#endif
#if PF_IN(3)
PF_PAIR_ENTRY(pair_stage1_f32, float, false)
#endif
#if PF_IN(4)
PF_PAIR_ENTRY(pair_stage2_f32, float, true)
#endif

#if PF_IN(0)
template <typename real, int MOB, int FE, int TBY, int kStepNT>
cudaError_t launch_persistent_step(const Layout &L, const KC<real> &k1, const KC<real> &k2, real *U, real *Us,
                                   const real *vel, int64_t nsteps, unsigned *flags, uint32_t epoch, cudaStream_t s) {
    static int occ = -1, nsm = 0;
    auto kern = persistent_step_kernel<real, MOB, FE, TBY, kStepNT>;
    const size_t smem = sizeof(TileStepSmem<real, TBY>);
    if (occ < 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kStepNT, smem);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
    }
    const int64_t ntiles = (int64_t)((L.nx + BX - 1) / BX) * ((L.ny_loc + TBY - 1) / TBY) * L.members;
    const int64_t maxb = (int64_t)occ * nsm;
    const int blocks = (int)(ntiles < maxb ? ntiles : maxb);
    Layout Lc = L;
    KC<real> a1 = k1, a2 = k2;
    static const int use_flags = env_int("PF_STEP_FLAGS", 0);   // measured: +0-6% at 256^2, -3% at 128^2 / 512^2
    unsigned *fl = use_flags ? flags : nullptr;
    void *args[] = {&Lc, &a1, &a2, &U, &Us, (void *)&vel, &nsteps, &fl, &epoch};
    return cudaLaunchCooperativeKernel((const void *)kern, blocks, kStepNT, args, smem, s);
}

template <typename real, int MOB, int FE, int TBY>
cudaError_t launch_persistent_b(const Layout &L, const KC<real> &k1, const KC<real> &k2, real *U, real *Us,
                                const real *vel, int64_t nsteps, cudaStream_t s) {
    static int occ = -1, nsm = 0;
    auto kern = persistent_kernel<real, MOB, FE, TBY>;
    if (occ < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, 0);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
    }
    const int64_t ntiles = (int64_t)((L.nx + BX - 1) / BX) * ((L.ny_loc + TBY - 1) / TBY) * L.members;
    const int64_t maxb = (int64_t)occ * nsm;
    const int blocks = (int)(ntiles < maxb ? ntiles : maxb);
    Layout Lc = L;
    KC<real> a1 = k1, a2 = k2;
    void *args[] = {&Lc, &a1, &a2, &U, &Us, (void *)&vel, &nsteps};
    return cudaLaunchCooperativeKernel((const void *)kern, blocks, NT, args, 0, s);
}

template <typename real, int MOB, int FE>
cudaError_t launch_persistent_t(const Layout &L, const KC<real> &k1, const KC<real> &k2, real *U, real *Us,
                                const real *vel, int64_t nsteps, unsigned *flags, uint32_t epoch, cudaStream_t s) {
    const int64_t cells = (int64_t)L.nx * L.ny_loc * L.members;
    static const int step = env_int("PF_PERSIST_STEP", 1);
    if (step) {   // one grid barrier per step (tile_step): 32 x 4 tiles / 512 threads up to 2^14 cells,
                  // 32 x 16 / 1024 up to 2^16, 32 x 8 / 256 above
#ifdef PF_STEP_TBY6
        static const int tby = env_int("PF_STEP_TBY", 0);   // experiment: force a tile shape
        if (tby == 4) return launch_persistent_step<real, MOB, FE, 4, 512>(L, k1, k2, U, Us, vel, nsteps, flags, epoch, s);
        if (tby == 6) return launch_persistent_step<real, MOB, FE, 6, 512>(L, k1, k2, U, Us, vel, nsteps, flags, epoch, s);
        if (tby == 8) return launch_persistent_step<real, MOB, FE, 8, 512>(L, k1, k2, U, Us, vel, nsteps, flags, epoch, s);
        if (tby == 9) return launch_persistent_step<real, MOB, FE, 8, 544>(L, k1, k2, U, Us, vel, nsteps, flags, epoch, s);
        if (tby == 16) return launch_persistent_step<real, MOB, FE, 16, 1024>(L, k1, k2, U, Us, vel, nsteps, flags, epoch, s);
        if (tby == 12) return launch_persistent_step<real, MOB, FE, 12, 704>(L, k1, k2, U, Us, vel, nsteps, flags, epoch, s);
        if (tby == 15) return launch_persistent_step<real, MOB, FE, 15, 1024>(L, k1, k2, U, Us, vel, nsteps, flags, epoch, s);
#endif
        if (cells <= (int64_t)1 << PF_STEP_TBY4_LOG2) return launch_persistent_step<real, MOB, FE, 4, 512>(L, k1, k2, U, Us, vel, nsteps, flags, epoch, s);
        // 2^14 .. 2^16 cells (configs[1]): 32 x 16 tiles with 1024 threads, so that every phase of
        // tile_step is one pass over its cells (32 x 8 / 512: 9.2 G on configs[1], 16 / 1024: 10.5 G)
        if (cells <= (int64_t)1 << 16) return launch_persistent_step<real, MOB, FE, 16, 1024>(L, k1, k2, U, Us, vel, nsteps, flags, epoch, s);
        return launch_persistent_step<real, MOB, FE, 8, 256>(L, k1, k2, U, Us, vel, nsteps, flags, epoch, s);
    }
    // one grid barrier per stage (round 1): 32 x 4 tiles up to 2^17 cells, 32 x 16 above
    if (cells <= (int64_t)1 << 17) return launch_persistent_b<real, MOB, FE, 4>(L, k1, k2, U, Us, vel, nsteps, s);
    return launch_persistent_b<real, MOB, FE, PF_TBY_LARGE>(L, k1, k2, U, Us, vel, nsteps, s);
}

cudaError_t launch_persistent(int precision, const Layout &L, const Coef &K, void *U, void *Us, const void *vel,
                              double dt, int64_t nsteps, unsigned *flags, uint32_t epoch, cudaStream_t s) {
    cudaError_t te = upload_exp_table();
    if (te != cudaSuccess) return te;
    if (precision == 0) {
        const KC<double> k1 = make_kc<double>(K, 0.5 * dt), k2 = make_kc<double>(K, dt);
        auto f = k1.fe == 1 ? (k1.mob == 0 ? launch_persistent_t<double, 0, 1> : k1.mob == 1 ? launch_persistent_t<double, 1, 1>
                                                                                        : launch_persistent_t<double, 2, 1>)
                            : (k1.mob == 0 ? launch_persistent_t<double, 0, 0> : k1.mob == 1 ? launch_persistent_t<double, 1, 0>
                                                                                        : launch_persistent_t<double, 2, 0>);
        return f(L, k1, k2, (double *)U, (double *)Us, (const double *)vel, nsteps, flags, epoch, s);
    }
    const KC<float> k1 = make_kc<float>(K, 0.5 * dt), k2 = make_kc<float>(K, dt);
    auto f = k1.fe == 1 ? (k1.mob == 0 ? launch_persistent_t<float, 0, 1> : k1.mob == 1 ? launch_persistent_t<float, 1, 1>
                                                                                   : launch_persistent_t<float, 2, 1>)
                        : (k1.mob == 0 ? launch_persistent_t<float, 0, 0> : k1.mob == 1 ? launch_persistent_t<float, 1, 0>
                                                                                   : launch_persistent_t<float, 2, 0>);
    return f(L, k1, k2, (float *)U, (float *)Us, (const float *)vel, nsteps, flags, epoch, s);
}

void swap_plan_buffers(StreamPlan &P) {
    for (int i = 0; i < 2; ++i) std::swap(P.mapU[i], P.mapUs[i]);
    std::swap(P.fmapU, P.fmapUs);
}

cudaError_t launch_stage(int precision, const Layout &L, const StreamPlan &P, const Coef &K, int stage,
                         const void *in, const void *base, void *out, const void *vel, double coef,
                         cudaStream_t s) {
    cudaError_t te = upload_exp_table();
    if (te != cudaSuccess) return te;
    if (P.ok) {
        if (precision == 0)
            return stage == 1 ? pair_stage1_f64(L, P, K, stage, out, vel, coef, s)
                              : pair_stage2_f64(L, P, K, stage, out, vel, coef, s);
        return stage == 1 ? pair_stage1_f32(L, P, K, stage, out, vel, coef, s)
                          : pair_stage2_f32(L, P, K, stage, out, vel, coef, s);
    }
    dim3 grid((L.nx + BX - 1) / BX, (L.r1 - L.r0 + BY - 1) / BY, L.members);
    if (precision == 0) {
        const KC<double> kd = make_kc<double>(K, coef);
        auto kern = kd.fe == 1 ? (kd.mob == 0 ? stage_kernel<double, 0, 1> : kd.mob == 1 ? stage_kernel<double, 1, 1> : stage_kernel<double, 2, 1>)
                               : (kd.mob == 0 ? stage_kernel<double, 0, 0> : kd.mob == 1 ? stage_kernel<double, 1, 0> : stage_kernel<double, 2, 0>);
        kern<<<grid, NT, 0, s>>>(L, kd, (const double *)in, (const double *)base, (double *)out, (const double *)vel);
    } else {
        const KC<float> kf = make_kc<float>(K, coef);
        auto kern = kf.fe == 1 ? (kf.mob == 0 ? stage_kernel<float, 0, 1> : kf.mob == 1 ? stage_kernel<float, 1, 1> : stage_kernel<float, 2, 1>)
                               : (kf.mob == 0 ? stage_kernel<float, 0, 0> : kf.mob == 1 ? stage_kernel<float, 1, 0> : stage_kernel<float, 2, 0>);
        kern<<<grid, NT, 0, s>>>(L, kf, (const float *)in, (const float *)base, (float *)out, (const float *)vel);
    }
    return cudaGetLastError();
}

cudaError_t launch_fill_ghosts(int precision, const Layout &L, double rho_in, void *state, cudaStream_t s) {
    const int64_t nr = (int64_t)4 * L.nx * 3 * L.members;
    const int64_t nc = (int64_t)(L.ny_loc + 4) * 3 * L.members * 2 * L.gx;
    const int b1 = (int)((nr + 255) / 256 > 4096 ? 4096 : (nr + 255) / 256);
    const int b2 = (int)((nc + 255) / 256 > 4096 ? 4096 : (nc + 255) / 256);
    if (precision == 0) {
        ghost_rows_kernel<double><<<b1, 256, 0, s>>>(L, rho_in, (double *)state);
        ghost_cols_kernel<double><<<b2, 256, 0, s>>>(L, (double *)state);
    } else {
        ghost_rows_kernel<float><<<b1, 256, 0, s>>>(L, (float)rho_in, (float *)state);
        ghost_cols_kernel<float><<<b2, 256, 0, s>>>(L, (float *)state);
    }
    return cudaGetLastError();
}

int diag_blocks(const Layout &L) {
    const int64_t ncell = (int64_t)L.ny_loc * L.nx;
    int64_t nb = (ncell + 8 * DT - 1) / (8 * DT);
    if (nb > 256) nb = 256;
    if (nb < 1) nb = 1;
    return (int)nb;
}

cudaError_t launch_diag(int precision, const Layout &L, const Coef &K, const void *state,
                        double *partials, double *out, cudaStream_t s) {
    const int nb = diag_blocks(L);
    dim3 grid(nb, L.members);
    if (precision == 0)
        diag_kernel<double><<<grid, DT, 0, s>>>(L, K, (const double *)state, partials);
    else
        diag_kernel<float><<<grid, DT, 0, s>>>(L, K, (const float *)state, partials);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    diag_final<<<L.members, DT, 0, s>>>(nb, partials, K.dx2, out);
    return cudaGetLastError();
}

cudaError_t launch_composite(int precision, const Layout &L, const void *state, double *dst, int64_t dst_mstride,
                             int row0, cudaStream_t s) {
    const int64_t total = (int64_t)L.ny_loc * L.nx * L.members;
    const int nb = (int)((total + 255) / 256 > 8192 ? 8192 : (total + 255) / 256);
    if (precision == 0)
        composite_kernel<double><<<nb, 256, 0, s>>>(L, (const double *)state, dst, dst_mstride, row0);
    else
        composite_kernel<float><<<nb, 256, 0, s>>>(L, (const float *)state, dst, dst_mstride, row0);
    return cudaGetLastError();
}

cudaError_t launch_inflow(int precision, const Layout &L, double rho_in, double sigma, uint64_t seed,
                          int64_t gmember0, int64_t step, void *U, void *Us, cudaStream_t s) {
    if (L.y0 + L.ny_loc != L.ny) return cudaSuccess;   // only the top slab has the reservoir
    const int64_t total = (int64_t)L.members * L.pitch;
    const int nb = (int)((total + 255) / 256 > 4096 ? 4096 : (total + 255) / 256);
    if (precision == 0)
        inflow_kernel<double><<<nb, 256, 0, s>>>(L, rho_in, sigma, seed, gmember0, step, (double *)U, (double *)Us);
    else
        inflow_kernel<float><<<nb, 256, 0, s>>>(L, rho_in, sigma, seed, gmember0, step, (float *)U, (float *)Us);
    return cudaGetLastError();
}

cudaError_t launch_pack_f64(int precision, const Layout &L, int field, int member0, int nmem,
                            const void *state, double *dst, cudaStream_t s) {
    const int64_t total = (int64_t)L.ny_loc * L.nx * nmem;
    const int nb = (int)((total + 255) / 256 > 4096 ? 4096 : (total + 255) / 256);
    if (precision == 0)
        pack_kernel<double><<<nb, 256, 0, s>>>(L, field, member0, nmem, (const double *)state, dst);
    else
        pack_kernel<float><<<nb, 256, 0, s>>>(L, field, member0, nmem, (const float *)state, dst);
    return cudaGetLastError();
}

cudaError_t launch_unpack_f64(int precision, const Layout &L, int field, int member0, int nmem,
                              const double *src, void *state, cudaStream_t s) {
    const int64_t total = (int64_t)L.ny_loc * L.nx * nmem;
    const int nb = (int)((total + 255) / 256 > 4096 ? 4096 : (total + 255) / 256);
    if (precision == 0)
        unpack_kernel<double><<<nb, 256, 0, s>>>(L, field, member0, nmem, src, (double *)state);
    else
        unpack_kernel<float><<<nb, 256, 0, s>>>(L, field, member0, nmem, src, (float *)state);
    return cudaGetLastError();
}

#endif  // PF_IN(0)

}  // namespace pf
