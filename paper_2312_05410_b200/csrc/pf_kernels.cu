// pf_kernels.cu -- sm_100a kernels of the PVD phase-field midpoint step.
//
// stage_kernel: one fused pass per explicit-midpoint stage (section 4.2):
//   load a tile of c, phi (+2 halo) and rho (+1 halo) into shared memory, applying the ghost
//   rules (x periodic, y mirror for c/phi, rho mirror below / reservoir above; R-12),
//   phase 1: h, p, e, M_c, mu_c, mu_phi on the tile + 1-ring (R-2..R-7),
//   phase 2: conservative flux divergence R_c, M_phi L(mu_phi), source S, vapour R_rho,
//            and the Euler-form update out = base + coef R (R-11).
// diag_kernel: fp64 sums, free energy E_h and non-finite counts, fixed-order reductions.
//
// Every cell's value comes from the same inlined code path (interior, tile ring, slab edge),
// so results are bitwise independent of tiling, x-translation and slab decomposition.
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "pf_cell.cuh"
#include "pf_internal.h"

namespace pf {
namespace {

constexpr int BX = 32;   // tile width  (one warp across x)
constexpr int BY = 16;   // tile height
constexpr int NT = 256;  // threads per block (32 x 8)

// Local storage row (relative to owned row 0) holding the c/phi value of local row ly,
// after the global mirror rule (R-12).  Clamped so that rows no output depends on stay
// in bounds.
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

template <typename real, bool HMIX>
__global__ void __launch_bounds__(NT) stage_kernel(Layout L, KC<real> k, const real *__restrict__ in,
                                                   const real *__restrict__ base, real *out,
                                                   const real *__restrict__ vel) {
    __shared__ real sc[BY + 4][BX + 4];
    __shared__ real sp[BY + 4][BX + 4];
    __shared__ real sr[BY + 2][BX + 2];
    __shared__ real smc[BY + 2][BX + 2];
    __shared__ real smp[BY + 2][BX + 2];
    __shared__ real sM[BY + 2][BX + 2];
    __shared__ double etab[64];
    load_exp_table(etab);

    const int m = blockIdx.z;
    const int tx0 = blockIdx.x * BX;
    const int ty0 = blockIdx.y * BY;
    const int nx = L.nx;
    const int64_t row0 = 2 * (int64_t)nx;                 // storage offset of owned row 0
    const real *ic = in + m * L.mstride + row0;
    const real *ip = ic + L.fstride;
    const real *ir = ip + L.fstride;

    // ---- load c, phi with a 2-cell halo (ghost rules applied by index) ----
    for (int t = threadIdx.x; t < (BY + 4) * (BX + 4); t += NT) {
        const int sy = t / (BX + 4), sx = t - sy * (BX + 4);
        const int gx = wrap_x(tx0 - 2 + sx, nx);
        const int r = row_cphi(ty0 - 2 + sy, L);
        const int64_t off = (int64_t)r * nx + gx;
        sc[sy][sx] = ic[off];
        sp[sy][sx] = ip[off];
    }
    // ---- load rho with a 1-cell halo: bottom mirror, top reservoir (R-12) ----
    for (int t = threadIdx.x; t < (BY + 2) * (BX + 2); t += NT) {
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
            v = ir[(int64_t)r * nx + gx];
        }
        sr[sy][sx] = v;
    }
    __syncthreads();

    // ---- phase 1: mu_c, mu_phi, M on the tile + 1 ring ----
    // A ring cell outside the global y range takes the values of its mirror cell (computed by
    // the same code from the same inputs), which makes the boundary face fluxes exactly zero.
    for (int t = threadIdx.x; t < (BY + 2) * (BX + 2); t += NT) {
        const int sy = t / (BX + 2), sx = t - sy * (BX + 2);
        int g = L.y0 + ty0 - 1 + sy;
        if (g < 0) g = -1 - g;
        if (g >= L.ny) g = 2 * L.ny - 1 - g;
        int ey = g - L.y0 - (ty0 - 2);                       // row in sc/sp
        ey = ey < 1 ? 1 : (ey > BY + 2 ? BY + 2 : ey);
        const int ex = sx + 1;
        real mc, mp, M;
        constitutive<real, HMIX>(k, etab, sc[ey][ex], sp[ey][ex], sc[ey][ex - 1], sc[ey][ex + 1], sc[ey - 1][ex],
                           sc[ey + 1][ex], sp[ey][ex - 1], sp[ey][ex + 1], sp[ey - 1][ex],
                           sp[ey + 1][ex], mc, mp, M);
        smc[sy][sx] = mc;
        smp[sy][sx] = mp;
        sM[sy][sx] = M;
    }
    __syncthreads();

    // ---- phase 2: fluxes, source, vapour, update ----
    const real vx = vel[2 * m], vy = vel[2 * m + 1];
    const int lx = threadIdx.x & (BX - 1);
    const int gx = tx0 + lx;
    for (int q = threadIdx.x / BX; q < BY; q += NT / BX) {
        const int ly = ty0 + q;
        if (gx >= nx || ly >= L.ny_loc) continue;
        const int y = q + 1, x = lx + 1;                    // ring coordinates
        const int cy = q + 2, cx = lx + 2;                   // c/phi tile coordinates
        const int64_t o = m * L.mstride + row0 + (int64_t)ly * nx + gx;
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
        out[o] = oc;
        out[o + L.fstride] = op;
        out[o + 2 * L.fstride] = orr;
    }
}

// ----------------------------------------------------------------------------------------
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
    const int64_t row0 = 2 * (int64_t)nx;
    const real *c = st + m * L.mstride + row0;
    const real *p = c + L.fstride;
    const real *r = p + L.fstride;
    double acc[kDiag];
#pragma unroll
    for (int q = 0; q < kDiag; ++q) acc[q] = 0.0;
    const int64_t ncell = (int64_t)L.ny_loc * nx;
    for (int64_t k = (int64_t)blockIdx.x * DT + threadIdx.x; k < ncell; k += (int64_t)gridDim.x * DT) {
        const int ly = (int)(k / nx), i = (int)(k - (int64_t)ly * nx);
        const double cc = (double)c[k], pp = (double)p[k], rr = (double)r[k];
        const bool fc = isfinite(cc), fp = isfinite(pp), fr = isfinite(rr);
        acc[0] += cc;
        acc[1] += pp;
        acc[2] += rr;
        const int ir = (i + 1 == nx) ? 0 : i + 1;
        const double dcx = (double)c[(int64_t)ly * nx + ir] - cc;
        const double dpx = (double)p[(int64_t)ly * nx + ir] - pp;
        const double omc = 1.0 - cc, omp = 1.0 - pp;
        double e = K.dx2 * (K.W_c * (cc * cc) * (omc * omc) * pp + K.W_p * (pp * pp) * (omp * omp));
        e += K.half_kc * (dcx * dcx) + K.half_kp * (dpx * dpx);
        if (L.y0 + ly < L.ny - 1) {      // y-face above (ghost row at the slab top)
            const double dcy = (double)c[k + nx] - cc, dpy = (double)p[k + nx] - pp;
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
        dst[k] = (double)st[(member0 + mm) * L.mstride + field * L.fstride + 2 * (int64_t)L.nx + rem];
    }
}

template <typename real>
__global__ void unpack_kernel(Layout L, int field, int member0, int nmem, const double *src, real *st) {
    const int64_t per = (int64_t)L.ny_loc * L.nx;
    const int64_t total = per * nmem;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t mm = k / per, rem = k - mm * per;
        st[(member0 + mm) * L.mstride + field * L.fstride + 2 * (int64_t)L.nx + rem] = (real)src[k];
    }
}


// ----------------------------------------------------------------------------------------
// Streaming stage kernel (the performance path).
//
// A persistent grid (one resident wave) walks the work in y.  The work is the concatenation of
// all (member, x-strip) columns of W cells, each ny_loc rows tall; block b owns the contiguous
// row range [R b / B, R (b+1) / B) of that concatenation, so every block gets the same number of
// rows (+-1) and only pays the halo prologue at its 1-2 segment starts.
//
// Rows arrive through a TMA bulk-copy ring (cp.async.bulk global -> shared, completion on an
// mbarrier per slot, S slots, issued S-3 rows ahead by thread 0).  Load k of a segment carries
// c/phi row k (+-HL halo columns, x wrap by separate copies), rho row k-1 and, for stage 2, the
// base row k-2.  Each thread owns one column: it keeps a sliding register window of its own
// column and takes x-neighbours from shared memory.  Per row: mu/M of row k-1 (own column plus
// two halo columns) -> smem, one __syncthreads, then the update of row k-2 and its coalesced
// store.  The arithmetic per cell is pf_cell.cuh's, the same as the tile kernel's.

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Streaming kernel configuration: NCW compute warps per block, each producing 30 output columns
// (it evaluates mu / M on 32 columns: its 30 plus one on each side), so a strip is at most
// 30 NCW columns wide; S ring slots.
template <typename real, int NCW, int S, bool BASE>
struct StreamCfg {
    static constexpr int HL = 16 / (int)sizeof(real);   // halo columns loaded (one 16 B chunk)
    static constexpr int WMAX = (30 * NCW + HL - 1) / HL * HL;   // widest strip (16 B multiple)
    static constexpr int RW = 32 * NCW + 2 * HL;        // smem row width (>= WMAX + 2 HL + 2)
    static constexpr int SLOT = 3 * RW + (BASE ? 3 * WMAX : 0);   // c, phi, rho (+ base) rows
    static constexpr size_t bytes = (size_t)S * SLOT * sizeof(real) + (size_t)S * 16 + 64 * 8;
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Work schedule shared by the producer and the compute warps.  Grouped mode (G > 0): blocks come in
// groups of `strips`; block b works on strip b % strips of the row range [T g/G, T (g+1)/G) of the
// concatenated (member, row) space (T = members * ny_loc rows, g = b / strips), so the blocks of a
// group stream the same rows at the same time and DRAM sees whole contiguous rows.  Ungrouped
// mode (G == 0): block b owns the row range [R b/B, R (b+1)/B) of the concatenated
// (member, strip, row) space, R = members * strips * ny_loc.
struct Seg {
    int m, x0, Wp, ya, yb;
};
struct Sched {
    int64_t lo, hi;
    int strip;        // grouped: fixed strip of this block; -1 ungrouped
};
__device__ __forceinline__ Sched make_sched(const Layout &L, int Wo, int G) {
    const int strips = (L.nx + Wo - 1) / Wo;
    Sched sc;
    if (G > 0) {
        const int g = blockIdx.x / strips;
        sc.strip = blockIdx.x - g * strips;
        const int64_t T = (int64_t)L.members * L.ny_loc;
        sc.lo = T * g / G;
        sc.hi = T * (g + 1) / G;
    } else {
        const int64_t R = (int64_t)L.members * strips * L.ny_loc;
        sc.strip = -1;
        sc.lo = R * blockIdx.x / gridDim.x;
        sc.hi = R * (blockIdx.x + 1) / gridDim.x;
    }
    return sc;
}
__device__ __forceinline__ bool next_seg(const Layout &L, int Wo, const Sched &sc, int64_t &pos, Seg &sg) {
    if (pos >= sc.hi) return false;
    const int nyl = L.ny_loc, strips = (L.nx + Wo - 1) / Wo;
    const int64_t col = pos / nyl;      // grouped: member; ungrouped: member * strips + strip
    sg.ya = (int)(pos - col * nyl);
    sg.yb = (int)min((int64_t)nyl, (int64_t)sg.ya + (sc.hi - pos));
    pos += sg.yb - sg.ya;
    int sidx;
    if (sc.strip >= 0) {
        sg.m = (int)col;
        sidx = sc.strip;
    } else {
        sg.m = (int)(col / strips);
        sidx = (int)(col - (int64_t)sg.m * strips);
    }
    sg.x0 = sidx * Wo;
    sg.Wp = min(Wo, L.nx - sg.x0);
    return true;
}

template <typename real, int NCW, int S, bool BASE, bool HMIX>
__global__ void __launch_bounds__(32 * NCW + 32, (NCW >= 8 ? 2 : 4)) stream_kernel(
    Layout L, KC<real> k, const real *__restrict__ in, const real *__restrict__ base, real *out,
    const real *__restrict__ vel, int Wo, int G, int dbg) {
    // dbg != 0 (PF_STREAM_DBG, experiments only): skip the arithmetic, keep every load and store.
    // BASE: stage 2 (the update base u^n is a separate buffer, streamed through the ring);
    // otherwise stage 1 (base = the stage input).
    // Warp roles.  Warps [0, NCW): compute.  Warp NCW: producer -- lane 0 issues the TMA bulk
    // copies of the row ring, gated per slot by an "empty" mbarrier that every compute warp
    // arrives on once it is done with the slot.  Compute warps never synchronise with each other:
    // warp w owns output columns x0 + 30w + [0, 30); lane l evaluates mu / M at column
    // x0 + 30w - 1 + l and passes them to lanes l -+ 1 by warp shuffles.  The row loop is unrolled
    // by 3 and computes unconditionally (only stores are predicated), so the per-lane sliding
    // windows rotate by register renaming.
    using Cfg = StreamCfg<real, NCW, S, BASE>;
    constexpr int HL = Cfg::HL, RW = Cfg::RW, SLOT = Cfg::SLOT, WMAX = Cfg::WMAX;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    real *slots = reinterpret_cast<real *>(smem_raw);
    uint64_t *full = reinterpret_cast<uint64_t *>(slots + S * SLOT);
    uint64_t *empty = full + S;
    double *etab = reinterpret_cast<double *>(empty + S);
    load_exp_table(etab);

    const int t = threadIdx.x;
    const int warp = t >> 5, lane = t & 31;
    if (t == 0) {
        for (int q = 0; q < S; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    const int nx = L.nx;
    const Sched sch = make_sched(L, Wo, G);

    if (warp == NCW) {
        // ------------------------------- producer -------------------------------
        if (lane != 0) return;
        uint32_t g = 0;
        int64_t pos = sch.lo;
        Seg sg;
        while (next_seg(L, Wo, sch, pos, sg)) {
            const int n = sg.yb - sg.ya + 4, npad = (n + 2) / 3 * 3;
            const real *fin = in + sg.m * L.mstride + 2 * (int64_t)nx;
            const real *fba = base + sg.m * L.mstride + 2 * (int64_t)nx;
            const bool wrapl = (sg.x0 == 0), wrapr = (sg.x0 + sg.Wp == nx);
            const uint32_t rowb = (uint32_t)((sg.Wp + 2 * HL) * sizeof(real));
            const uint32_t bb = (uint32_t)(sg.Wp * sizeof(real));
            for (int i = 0; i < npad; ++i, ++g) {
                const int slot = g % S;
                if (g >= (uint32_t)S) mbar_wait(&empty[slot], ((g / S) - 1) & 1u);
                if (i >= n) {
                    mbar_arrive(&full[slot]);          // padding: completes the phase, no data
                    continue;
                }
                const int kk = sg.ya - 2 + i;
                real *sl = slots + slot * SLOT;
                const int rc = row_cphi(kk, L);                   // c/phi source row (mirror rule)
                int grho = L.y0 + kk - 1;
                const bool rho_res = grho >= L.ny;                // reservoir row: rho_in, no copy
                if (grho < 0) grho = -1 - grho;
                const int rr = grho - L.y0;
                const bool wb = BASE && (kk - 2 >= sg.ya) && (kk - 2 < sg.yb);
                mbar_expect_tx(&full[slot], (rho_res ? 2u : 3u) * rowb + (wb ? 3u * bb : 0u));
                for (int f = 0; f < 3; ++f) {
                    if (f == 2 && rho_res) continue;
                    const real *row = fin + f * L.fstride + (int64_t)(f == 2 ? rr : rc) * nx;
                    real *d = sl + f * RW;
                    if (!wrapl && !wrapr) {
                        bulk_g2s(d, row + sg.x0 - HL, rowb, &full[slot]);
                    } else {
                        bulk_g2s(d, row + (wrapl ? nx - HL : sg.x0 - HL), HL * sizeof(real), &full[slot]);
                        bulk_g2s(d + HL, row + sg.x0, bb, &full[slot]);
                        bulk_g2s(d + HL + sg.Wp, row + (wrapr ? 0 : sg.x0 + sg.Wp), HL * sizeof(real), &full[slot]);
                    }
                }
                if (wb)
                    for (int f = 0; f < 3; ++f)
                        bulk_g2s(sl + 3 * RW + f * WMAX, fba + f * L.fstride + (int64_t)(kk - 2) * nx + sg.x0, bb,
                                 &full[slot]);
            }
        }
        return;
    }

    // --------------------------- compute warps ---------------------------------
    static_assert(S >= 4, "ring depth");
    const int cx = 30 * warp - 1 + lane;    // strip-relative column of this lane's mu / M
    const int ci = HL + cx;                 // its smem index
    const int bi = cx < 0 ? 0 : (cx >= WMAX ? WMAX - 1 : cx);   // base index (in range)
    int sidx = 0;                           // ring slot of the first load of the current group
    uint32_t par = 0;                       // its full-barrier phase parity
    int64_t pos = sch.lo;
    Seg sg;
    while (next_seg(L, Wo, sch, pos, sg)) {
        const int n = sg.yb - sg.ya + 4, npad = (n + 2) / 3 * 3;
        const bool store = lane >= 1 && lane <= 30 && cx < sg.Wp;
        const int64_t fs1 = L.fstride;
        real *op_ = out + sg.m * L.mstride + 2 * (int64_t)nx + (int64_t)(sg.ya - 4) * nx + sg.x0 + bi;
        const real vx = vel[2 * sg.m], vy = vel[2 * sg.m + 1];
        const int rho_res_i = L.ny - L.y0 - sg.ya + 3;   // first load whose rho row is the reservoir

        real c_m2 = 0, c_m1 = 0, c_0 = 0;                 // c rows k-2, k-1, k (own column)
        real p_m3 = 0, p_m2 = 0, p_m1 = 0, p_0 = 0;       // phi rows k-3 .. k
        real r_m3 = 0, r_m2 = 0, r_m1 = 0;                // rho rows k-3 .. k-1
        real a_m2 = 0, a_m1 = 0;                          // mu_c rows k-2, k-1
        real b_m3 = 0, b_m2 = 0, b_m1 = 0;                // mu_phi rows k-3 .. k-1
        real M_m2 = 0, M_m1 = 0;                          // M rows k-2, k-1
        real fn_m = 0;                                    // north face flux of row k-3
        for (int i0 = 0; i0 < npad; i0 += 3) {
            // ring slots of this group of 3 loads and of the 2 loads before it (wrapping mod S)
            const int q1 = sidx + 1 >= S ? sidx + 1 - S : sidx + 1;
            const int q2 = sidx + 2 >= S ? sidx + 2 - S : sidx + 2;
            const int qm1 = sidx >= 1 ? sidx - 1 : sidx - 1 + S;
            const int qm2 = sidx >= 2 ? sidx - 2 : sidx - 2 + S;
            const real *gq[5] = {slots + qm2 * SLOT + ci, slots + qm1 * SLOT + ci, slots + sidx * SLOT + ci,
                                 slots + q1 * SLOT + ci, slots + q2 * SLOT + ci};
            const int qs[5] = {qm2, qm1, sidx, q1, q2};
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int i = i0 + u;
                const real *s0 = gq[u + 2];                                          // load k
                const real *s1 = gq[u + 1];                                          // load k-1
                const real *s2 = gq[u];                                              // load k-2
                mbar_wait(&full[qs[u + 2]], par ^ (uint32_t)(sidx + u >= S));
                c_m2 = c_m1; c_m1 = c_0; c_0 = s0[0];
                p_m3 = p_m2; p_m2 = p_m1; p_m1 = p_0; p_0 = s0[RW];
                r_m3 = r_m2; r_m2 = r_m1;
                r_m1 = (i >= rho_res_i) ? k.rho_in : s0[2 * RW];
                a_m2 = a_m1;
                b_m3 = b_m2; b_m2 = b_m1;
                M_m2 = M_m1;
                if (dbg) {
                    if (dbg == 2 && warp < 8 && i >= 4 && i < n) {   // sector-aligned experiment
                        real *o2 = op_ - bi + 32 * warp + lane;
                        o2[0] = c_m2; o2[fs1] = p_m2; o2[2 * fs1] = r_m2;
                    } else if (dbg == 1 && store && i >= 4 && i < n) {
                        const real *bs = s0 - ci + 3 * RW + bi;
                        op_[0] = c_m2 + (BASE ? bs[0] : 0);
                        op_[fs1] = p_m2 + (BASE ? bs[WMAX] : 0);
                        op_[2 * fs1] = r_m2 + (BASE ? bs[2 * WMAX] : 0);
                    }
                    op_ += nx;
                    __syncwarp();
                    if (i >= 2 && lane == 0) mbar_arrive(&empty[qs[u]]);
                    continue;
                }
                // mu / M of row k-1 at this lane's column
                constitutive<real, HMIX>(k, etab, c_m1, p_m1, s1[-1], s1[1], c_m2, c_0, s1[RW - 1], s1[RW + 1], p_m2, p_0,
                                         a_m1, b_m1, M_m1);
                // update of row k-2.  East face flux from this lane's mu / M and lane+1's; the west
                // flux is lane-1's east flux; the south flux is last row's north flux.
                const real ar = __shfl_down_sync(0xffffffffu, a_m2, 1);
                const real Mr = __shfl_down_sync(0xffffffffu, M_m2, 1);
                const real bl = __shfl_up_sync(0xffffffffu, b_m2, 1), br_ = __shfl_down_sync(0xffffffffu, b_m2, 1);
                const real fe = face_flux<real>(M_m2, Mr, a_m2, ar);
                const real fw = __shfl_up_sync(0xffffffffu, fe, 1);
                const real fn = face_flux<real>(M_m2, M_m1, a_m2, a_m1);
                const real fs = fn_m;
                fn_m = fn;
                real bc = c_m2, bp = p_m2, bq = r_m2;   // stage 1: base = input
                if (BASE) {                               // stage 2: base row from the ring
                    const real *bs = s0 - ci + 3 * RW + bi;
                    bc = bs[0]; bp = bs[WMAX]; bq = bs[2 * WMAX];
                }
                real oc, op, orr;
                cell_update<real>(k, vx, vy, fe, fw, fn, fs, b_m2, bl, br_, b_m3, b_m1,
                                  s2[RW - 1], s2[RW + 1], p_m3, p_m1,
                                  r_m2, s1[2 * RW - 1], s1[2 * RW + 1], r_m3, r_m1,
                                  bc, bp, bq, oc, op, orr);
                if (store && i >= 4 && i < n) {
                    op_[0] = oc;
                    op_[fs1] = op;
                    op_[2 * fs1] = orr;
                }
                op_ += nx;
                __syncwarp();
                if (i >= 2 && lane == 0) mbar_arrive(&empty[qs[u]]);   // load i-2 is no longer read
            }
            sidx += 3;
            if (sidx >= S) { sidx -= S; par ^= 1u; }
        }
        // release the last two loads of the segment
        if (lane == 0) {
            mbar_arrive(&empty[sidx >= 2 ? sidx - 2 : sidx - 2 + S]);
            mbar_arrive(&empty[sidx >= 1 ? sidx - 1 : sidx - 1 + S]);
        }
        __syncwarp();
    }
}

template <typename real>
KC<real> make_kc(const Coef &K, double coef) {
    KC<real> k;
    k.half_inv_dx2 = (real)K.half_inv_dx2;
    k.inv_2dx = (real)K.inv_2dx;
    k.m_kc_dx2 = (real)(-K.kc_dx2);
    k.m_kp_dx2 = (real)(-K.kp_dx2);
    k.W_c = (real)K.W_c;
    k.W2c = (real)K.W2c;
    k.W2p = (real)K.W2p;
    k.MBb = (real)K.MBb;
    k.dMb = (real)K.dMb;
    k.MBs = (real)K.MBs;
    k.dMs = (real)K.dMs;
    k.two_inv_sigma = (real)(2.0 * K.inv_sigma);
    k.hmix = (K.dMb != 0.0 || K.dMs != 0.0) ? 1 : 0;
    k.Mp_dx2 = (real)K.Mp_dx2;
    k.Dr_dx2 = (real)K.Dr_dx2;
    k.rho_in = (real)K.rho_in;
    k.coef = (real)coef;
    return k;
}

}  // namespace

int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v ? atoi(v) : dflt;
}

template <typename real, int NCW, int S, bool BASE, bool HMIX>
cudaError_t launch_stream_b(const Layout &L, const KC<real> &k, const real *in, const real *base,
                            real *out, const real *vel, int Wo, cudaStream_t s) {
    using Cfg = StreamCfg<real, NCW, S, BASE>;
    static int occ = -1, nsm = 0;
    if (occ < 0) {
        cudaError_t e = cudaFuncSetAttribute(stream_kernel<real, NCW, S, BASE, HMIX>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::bytes);
        if (e != cudaSuccess) return e;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stream_kernel<real, NCW, S, BASE, HMIX>, 32 * NCW + 32,
                                                          Cfg::bytes);
        if (e != cudaSuccess) return e;
        if (occ < 1) occ = 1;
    }
    const int strips = (L.nx + Wo - 1) / Wo;
    const int64_t R = (int64_t)L.members * strips * L.ny_loc;
    const int64_t minrows = 16;
    int64_t B = (int64_t)occ * nsm;
    static const int dbg = env_int("PF_STREAM_DBG", 0), nogroup = env_int("PF_STREAM_NOGROUP", 0);
    // grouped schedule when at least 4 groups of `strips` blocks fit in one resident wave
    int64_t G = B / strips;
    const int64_t T = (int64_t)L.members * L.ny_loc;
    if (G > (T + minrows - 1) / minrows) G = (T + minrows - 1) / minrows;
    if (G >= 4 && !nogroup) {
        B = G * strips;
    } else {
        G = 0;
        if (B > (R + minrows - 1) / minrows) B = (R + minrows - 1) / minrows;
    }
    if (B < 1) B = 1;
    stream_kernel<real, NCW, S, BASE, HMIX><<<(unsigned)B, 32 * NCW + 32, Cfg::bytes, s>>>(L, k, in, base, out, vel, Wo, (int)G, dbg);
    return cudaGetLastError();
}

bool stream_eligible(const Layout &L) { return L.nx % 4 == 0 && L.nx >= 16; }

// Strip output width Wo (multiple of 4, <= 30 NCW) and warps per block NCW: 256 columns on 9
// compute warps for wide grids, narrower strips on fewer warps for small nx.  Ring depth: stage 1
// streams 3 rows per load, stage 2 six, so stage 1 affords a deeper ring in the same shared
// memory.  PF_STREAM_NCW / PF_STREAM_S1 / PF_STREAM_S2 / PF_STREAM_WO override (experiments).
template <typename real>
cudaError_t launch_stream(const Layout &L, const KC<real> &k, const real *in, const real *base, real *out,
                          const real *vel, int has_base, cudaStream_t s) {
    static const int envN = env_int("PF_STREAM_NCW", 0), envS1 = env_int("PF_STREAM_S1", 0),
                     envS2 = env_int("PF_STREAM_S2", 0), envWo = env_int("PF_STREAM_WO", 0);
    int ncw = L.nx >= 256 ? 9 : (L.nx >= 120 ? 5 : 3);
    if (envN) ncw = envN;
    int Wo = ncw == 9 ? 256 : (ncw == 5 ? 128 : 64);
    Wo = min(Wo, (30 * ncw) / 4 * 4);
    if (envWo) Wo = envWo;
    if (Wo > L.nx) Wo = L.nx;
    const int S = has_base ? (envS2 ? envS2 : 8) : (envS1 ? envS1 : 12);
#define PF_TRY(NN, SS, BB)                                                                      \
    if (ncw == NN && S == SS && has_base == BB)                                                \
        return k.hmix ? launch_stream_b<real, NN, SS, BB, true>(L, k, in, base, out, vel, Wo, s) \
                      : launch_stream_b<real, NN, SS, BB, false>(L, k, in, base, out, vel, Wo, s);
    PF_TRY(9, 8, 1) PF_TRY(9, 6, 1) PF_TRY(9, 7, 1) PF_TRY(9, 12, 0) PF_TRY(9, 6, 0) PF_TRY(9, 9, 0)
    PF_TRY(9, 15, 0) PF_TRY(5, 8, 1) PF_TRY(5, 12, 0) PF_TRY(3, 8, 1) PF_TRY(3, 12, 0)
#undef PF_TRY
    return cudaErrorInvalidValue;
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

cudaError_t launch_stage(int precision, const Layout &L, const Coef &K, const void *in,
                         const void *base, void *out, const void *vel, double coef, cudaStream_t s) {
    cudaError_t te = upload_exp_table();
    if (te != cudaSuccess) return te;
    const bool has_base = base != in;
    const bool stream = L.path != 1 && stream_eligible(L);
    if (stream) {
        if (precision == 0)
            return launch_stream<double>(L, make_kc<double>(K, coef), (const double *)in,
                                            (const double *)base, (double *)out, (const double *)vel,
                                            has_base, s);
        return launch_stream<float>(L, make_kc<float>(K, coef), (const float *)in, (const float *)base,
                                       (float *)out, (const float *)vel, has_base, s);
    }
    dim3 grid((L.nx + BX - 1) / BX, (L.ny_loc + BY - 1) / BY, L.members);
    if (precision == 0) {
        const KC<double> kd = make_kc<double>(K, coef);
        if (kd.hmix)
            stage_kernel<double, true><<<grid, NT, 0, s>>>(L, kd, (const double *)in, (const double *)base,
                                                           (double *)out, (const double *)vel);
        else
            stage_kernel<double, false><<<grid, NT, 0, s>>>(L, kd, (const double *)in, (const double *)base,
                                                            (double *)out, (const double *)vel);
    } else {
        const KC<float> kf = make_kc<float>(K, coef);
        if (kf.hmix)
            stage_kernel<float, true><<<grid, NT, 0, s>>>(L, kf, (const float *)in, (const float *)base,
                                                          (float *)out, (const float *)vel);
        else
            stage_kernel<float, false><<<grid, NT, 0, s>>>(L, kf, (const float *)in, (const float *)base,
                                                           (float *)out, (const float *)vel);
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

}  // namespace pf
