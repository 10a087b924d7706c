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

#include "pf_internal.h"

namespace pf {
namespace {

constexpr int BX = 32;   // tile width  (one warp across x)
constexpr int BY = 16;   // tile height
constexpr int NT = 256;  // threads per block (32 x 8)

template <typename real>
struct KC {                    // coefficients in the compute precision
    real half_inv_dx2, inv_2dx, kc_dx2, kp_dx2, W_c, W2c, W2p;
    real MBb, dMb, MBs, dMs, inv_sigma, Mp_dx2, Dr_dx2, rho_in, coef;
};

template <typename real>
__device__ __forceinline__ real dexp(real x);
template <>
__device__ __forceinline__ double dexp<double>(double x) { return exp(x); }
template <>
__device__ __forceinline__ float dexp<float>(float x) { return expf(x); }

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

// Cell-centre constitutive pass (a2): mu_c, mu_phi and M_c of one cell from its value and
// its 4 neighbours.  Sum orders are fixed (the same code for every cell).
template <typename real>
__device__ __forceinline__ void constitutive(const KC<real> &k, real c, real p, real cl, real cr,
                                             real cd, real cu, real pl, real pr, real pd, real pu,
                                             real &mu_c, real &mu_p, real &M) {
    const real lc = ((cl + cr) + (cd + cu)) - real(4) * c;   // dx^2 L(c)
    const real lp = ((pl + pr) + (pd + pu)) - real(4) * p;   // dx^2 L(phi)
    const real omc = real(1) - c;
    const real c1 = c * omc;                                 // c(1-c)
    // mu_c = 2 W_c c(1-c)(1-2c) phi - kappa_c L(c)                        (R-2, R-4)
    mu_c = k.W2c * c1 * (real(1) - real(2) * c) * p - k.kc_dx2 * lc;
    // mu_phi = W_c c^2(1-c)^2 + 2 W_phi phi(1-phi)(1-2phi) - kappa_phi L(phi)   (R-3)
    mu_p = k.W_c * (c1 * c1) + k.W2p * (p * (real(1) - p)) * (real(1) - real(2) * p) - k.kp_dx2 * lp;
    // mobility (R-5, R-6)
    real ch = c < real(0) ? real(0) : c;
    ch = ch > real(1) ? real(1) : ch;
    const real h = ch * ch * (real(3) - real(2) * ch);
    const real pp = p * p * (real(3) - real(2) * p);         // 1/4 (2-phit)(1+phit)^2
    const real q = (real(2) * p - real(1)) * k.inv_sigma;
    const real e = dexp<real>(-(q * q));
    const real mb = pp * (k.MBb + h * k.dMb);
    const real ms = k.MBs + h * k.dMs;
    M = mb + e * (ms - mb);
}

template <typename real>
__global__ void __launch_bounds__(NT) stage_kernel(Layout L, KC<real> k, const real *__restrict__ in,
                                                   const real *__restrict__ base, real *out,
                                                   const real *__restrict__ vel) {
    __shared__ real sc[BY + 4][BX + 4];
    __shared__ real sp[BY + 4][BX + 4];
    __shared__ real sr[BY + 2][BX + 2];
    __shared__ real smc[BY + 2][BX + 2];
    __shared__ real smp[BY + 2][BX + 2];
    __shared__ real sM[BY + 2][BX + 2];

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
        constitutive<real>(k, sc[ey][ex], sp[ey][ex], sc[ey][ex - 1], sc[ey][ex + 1], sc[ey - 1][ex],
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
        // R_c: conservative divergence of the face fluxes (M_a + M_b)/2 (mu_b - mu_a)/dx^2
        const real M0 = sM[y][x], m0 = smc[y][x];
        const real fe = (M0 + sM[y][x + 1]) * (smc[y][x + 1] - m0);
        const real fw = (sM[y][x - 1] + M0) * (m0 - smc[y][x - 1]);
        const real fn = (M0 + sM[y + 1][x]) * (smc[y + 1][x] - m0);
        const real fs = (sM[y - 1][x] + M0) * (m0 - smc[y - 1][x]);
        const real Rc = ((fe - fw) + (fn - fs)) * k.half_inv_dx2;
        // R_phi = M_phi L(mu_phi) + S
        const real lmp = ((smp[y][x - 1] + smp[y][x + 1]) + (smp[y - 1][x] + smp[y + 1][x])) -
                         real(4) * smp[y][x];
        const real r0 = sr[y][x];
        const int cy = q + 2, cx = lx + 2;                   // c/phi tile coordinates
        const real S = r0 * ((vx * (sp[cy][cx + 1] - sp[cy][cx - 1]) +
                              vy * (sp[cy + 1][cx] - sp[cy - 1][cx])) * k.inv_2dx);
        const real Rp = k.Mp_dx2 * lmp + S;
        // R_rho = D_rho L(rho) - v . G(rho) - S
        const real rl = sr[y][x - 1], rr = sr[y][x + 1], rd = sr[y - 1][x], ru = sr[y + 1][x];
        const real lr = ((rl + rr) + (rd + ru)) - real(4) * r0;
        const real adv = (vx * (rr - rl) + vy * (ru - rd)) * k.inv_2dx;
        const real Rr = (k.Dr_dx2 * lr - adv) - S;

        const int64_t o = m * L.mstride + row0 + (int64_t)ly * nx + gx;
        const real bc = base[o], bp = base[o + L.fstride], br = base[o + 2 * L.fstride];
        out[o] = bc + k.coef * Rc;
        out[o + L.fstride] = bp + k.coef * Rp;
        out[o + 2 * L.fstride] = br + k.coef * Rr;
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

template <typename real>
KC<real> make_kc(const Coef &K, double coef) {
    KC<real> k;
    k.half_inv_dx2 = (real)K.half_inv_dx2;
    k.inv_2dx = (real)K.inv_2dx;
    k.kc_dx2 = (real)K.kc_dx2;
    k.kp_dx2 = (real)K.kp_dx2;
    k.W_c = (real)K.W_c;
    k.W2c = (real)K.W2c;
    k.W2p = (real)K.W2p;
    k.MBb = (real)K.MBb;
    k.dMb = (real)K.dMb;
    k.MBs = (real)K.MBs;
    k.dMs = (real)K.dMs;
    k.inv_sigma = (real)K.inv_sigma;
    k.Mp_dx2 = (real)K.Mp_dx2;
    k.Dr_dx2 = (real)K.Dr_dx2;
    k.rho_in = (real)K.rho_in;
    k.coef = (real)coef;
    return k;
}

}  // namespace

cudaError_t launch_stage(int precision, const Layout &L, const Coef &K, const void *in,
                         const void *base, void *out, const void *vel, double coef, cudaStream_t s) {
    dim3 grid((L.nx + BX - 1) / BX, (L.ny_loc + BY - 1) / BY, L.members);
    if (precision == 0)
        stage_kernel<double><<<grid, NT, 0, s>>>(L, make_kc<double>(K, coef), (const double *)in,
                                                 (const double *)base, (double *)out,
                                                 (const double *)vel);
    else
        stage_kernel<float><<<grid, NT, 0, s>>>(L, make_kc<float>(K, coef), (const float *)in,
                                                (const float *)base, (float *)out,
                                                (const float *)vel);
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
