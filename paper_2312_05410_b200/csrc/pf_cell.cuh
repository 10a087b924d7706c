// pf_cell.cuh -- per-cell arithmetic of the discrete model, shared by every stage
// kernel (tile kernel and streaming kernel).  Every operation is an explicit round-to-nearest
// intrinsic (add / mul / fma), so no compiler contraction choice can differ between call sites:
// each cell's value is the same bit pattern on every code path, tiling, x-translation and slab
// decomposition (reading R-19).
#pragma once
#include <cstdint>

#include "pf_internal.h"

namespace pf {

template <typename real>
struct KC {                    // coefficients folded into the compute precision
    real half_inv_dx2, inv_2dx, m_kc_dx2, m_kp_dx2, W_c, W2c, W2p;   // m_ = negated
    real two_inv_sigma, Mp_dx2, Dr_dx2, rho_in, coef;
    real coefc;                // coef / (2 dx^2): the composition update's factor (R_c folded in)
    real MBb, dMb, MBs, dMs;   // mobilities shared by all members (MOB 0, 1)
    real omega, temp;          // regular-solution composition energy (FE 1, R-28)
    int fe;                    // 0 polynomial composition well (R-2), 1 regular solution (R-28)
    int mob;                   // 0: shared, M_A = M_B (h(c) drops out); 1: shared, M_A != M_B;
                               // 2: per member (record array, R-23)
    // exp_neg's constants as launch parameters rather than immediates: the compiler keeps them in
    // uniform registers (fp64 operands of DFMA / DADD) instead of re-materialising each 64-bit
    // immediate with two integer moves per use in the hot loop
    double ex_l2e64, ex_magic, ex_ln2hi, ex_ln2lo, ex_c6, ex_c24, ex_c120, ex_min;
};

// Per-member record (device array, storage precision, kMembStride values per member, pf_internal.h):
// velocity (R-10, R-15, R-21) and composition mobilities (R-6, R-23).
template <typename real>
struct Mob {
    real MBb, dMb, MBs, dMs;
};
template <typename real>
__device__ __forceinline__ Mob<real> load_mob(const real *memb, int m) {
    const real *q = memb + (int64_t)m * kMembStride + 2;
    return Mob<real>{q[0], q[1], q[2], q[3]};
}

__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// exp(x) for x <= 0 (the argument here is -(phit/sigma)^2), branch-free, table-driven:
// x = (64 n + j) ln2/64 + r with |r| <= ln2/128 (ln2 split as in fdlibm so the reduction is exact),
// exp(x) = 2^n * T[j] * P(r), T[j] = 2^(j/64) (host-computed, copied to shared memory by each
// block), P the Taylor polynomial of exp to degree 5 (truncation |r|^6/720 < 4e-17 relative),
// evaluated in Estrin form (dependency depth 3 instead of 5).  x is clamped to -708 (results below
// 1e-307 are irrelevant to M_c).  Max error ~2 ulp.
__constant__ double kExp2Tab[64];                        // 2^(j/64), filled by the host

// Constants (host side, set_exp_constants): kMagic = 1.5 * 2^52, 64 / ln 2, ln2 hi / 64 and lo / 64
// (negated), 1/6, 1/24, 1/120 and the clamp -708.
template <typename K>
__device__ __forceinline__ double exp_neg(double x, const double *tab, const K &k) {
    x = x > k.ex_min ? x : k.ex_min;
    const double kd = fma_(x, k.ex_l2e64, k.ex_magic);      // m = round(64 x / ln 2) in the low word
    const int m = __double2loint(kd);
    const double nd = sub_(kd, k.ex_magic);
    double r = fma_(nd, k.ex_ln2hi, x);
    r = fma_(nd, k.ex_ln2lo, r);
    // P(r) = (1 + r) + r^2 ((1/2 + r/6) + r^2 (1/24 + r/120))
    const double r2 = mul_(r, r);
    const double a = add_(r, 1.0);
    const double b = fma_(r, k.ex_c6, 0.5);
    const double c = fma_(r, k.ex_c120, k.ex_c24);
    double p = fma_(r2, fma_(r2, c, b), a);
    p = mul_(p, tab[m & 63]);
    return __hiloint2double(__double2hiint(p) + ((m >> 6) << 20), __double2loint(p));
}
template <typename K>
__device__ __forceinline__ float exp_neg(float x, const double *, const K &) { return expf(x); }

// The per-launch coefficient struct of a stage with factor coef (dt/2 or dt), from the ctx's
// coefficients (host side, shared by every kernel translation unit).
template <typename real>
inline KC<real> make_kc(const Coef &K, double coef) {
    KC<real> k;
    k.half_inv_dx2 = (real)K.half_inv_dx2;
    k.inv_2dx = (real)K.inv_2dx;
    k.m_kc_dx2 = (real)(-K.kc_dx2);
    k.m_kp_dx2 = (real)(-K.kp_dx2);
    k.W_c = (real)K.W_c;
    k.W2c = (real)K.W2c;
    k.W2p = (real)K.W2p;
    k.two_inv_sigma = (real)(2.0 * K.inv_sigma);
    k.MBb = (real)K.MBb;
    k.dMb = (real)K.dMb;
    k.MBs = (real)K.MBs;
    k.dMs = (real)K.dMs;
    k.mob = K.mob;
    k.fe = K.fe;
    k.omega = (real)K.omega;
    k.temp = (real)K.temp;
    k.Mp_dx2 = (real)K.Mp_dx2;
    k.Dr_dx2 = (real)K.Dr_dx2;
    k.rho_in = (real)K.rho_in;
    k.coef = (real)coef;
    k.coefc = (real)(coef * K.half_inv_dx2);
    k.ex_l2e64 = 92.332482616893656;                            // 64 / ln 2
    k.ex_magic = 6755399441055744.0;                            // 1.5 * 2^52
    k.ex_ln2hi = -(6.93147180369123816490e-01 / 64.0);          // ln 2 split as in fdlibm
    k.ex_ln2lo = -(1.90821492927058770002e-10 / 64.0);
    k.ex_c6 = 1.0 / 6.0;
    k.ex_c24 = 1.0 / 24.0;
    k.ex_c120 = 1.0 / 120.0;
    k.ex_min = -708.0;
    return k;
}

// Block-wide copy of the exp table into shared memory (call before the first exp_neg).
__device__ __forceinline__ void load_exp_table(double *tab) {
    for (int j = threadIdx.x; j < 64; j += blockDim.x) tab[j] = kExp2Tab[j];
}

template <typename real>
__device__ __forceinline__ real clamp01(real c) {
    const real a = c > real(0) ? c : real(0);
    return a < real(1) ? a : real(1);
}

// Row a2 (constitutive pass): mu_c, mu_phi and M_c of one cell from its value and its four
// neighbours (l = i-1, r = i+1, d = j-1, u = j+1).  P:310-331; readings R-1..R-7.
// The neighbour sums are ((l + r) + (d + u)): symmetric in (d, u), so a mirrored ghost row
// (u[-1] = u[0], u[-2] = u[1]) yields bit-identical mu / M to the cell it mirrors, and the
// boundary-face fluxes vanish exactly.
// Regular-solution composition energy (R-28): g(c) = Omega c~(1-c~) + T (c~ ln c~ + (1-c~) ln(1-c~)),
// c~ = min(max(c, 1e-9), 1 - 1e-9); returns g and g' = Omega (1 - 2c~) + T (ln c~ - ln(1-c~)).
template <typename real>
__device__ __forceinline__ void regular_solution(const KC<real> &k, real c, real &g, real &dg) {
    const real eps = real(1e-9), one = real(1);
    const real t = c < eps ? eps : (c > one - eps ? one - eps : c);
    const real u = sub_(one, t);
    const real lt = log(t), lu = log(u);
    g = fma_(k.omega, mul_(t, u), mul_(k.temp, fma_(t, lt, mul_(u, lu))));
    dg = fma_(k.omega, fma_(t, real(-2), one), mul_(k.temp, sub_(lt, lu)));
}

template <typename real, int MOB, int FE = 0>
__device__ __forceinline__ void constitutive(const KC<real> &k, const Mob<real> &mo, const double *etab, real c,
                                             real p, real cl, real cr, real cd, real cu, real pl, real pr, real pd,
                                             real pu, real &mu_c, real &mu_p, real &M) {
    const real one = real(1), m2 = real(-2), m4 = real(-4);
    const real lc = fma_(c, m4, add_(add_(cl, cr), add_(cd, cu)));   // dx^2 L(c)
    const real lp = fma_(p, m4, add_(add_(pl, pr), add_(pd, pu)));   // dx^2 L(phi)
    const real c1 = mul_(c, sub_(one, c));                            // c(1-c)
    const real t2c = fma_(c, m2, one);                                // 1-2c
    const real p1 = mul_(p, sub_(one, p));                            // phi(1-phi)
    const real t2p = fma_(p, m2, one);                                // 1-2phi
    if (FE == 1) {   // regular solution (R-28): mu_c = phi g'(c) - kappa_c L(c); mu_phi = g(c) + ...
        real g, dg;
        regular_solution(k, c, g, dg);
        mu_c = fma_(lc, k.m_kc_dx2, mul_(dg, p));
        mu_p = fma_(lp, k.m_kp_dx2, add_(g, mul_(mul_(p1, k.W2p), t2p)));
    } else {
        // mu_c = 2 W_c c(1-c)(1-2c) phi - kappa_c L(c)                          (R-2, R-4)
        mu_c = fma_(lc, k.m_kc_dx2, mul_(mul_(mul_(c1, k.W2c), t2c), p));
        // mu_phi = W_c c^2(1-c)^2 + 2 W_phi phi(1-phi)(1-2phi) - kappa_phi L(phi) (R-3)
        mu_p = fma_(lp, k.m_kp_dx2, fma_(mul_(c1, c1), k.W_c, mul_(mul_(p1, k.W2p), t2p)));
    }
    // M_c = M_bulk + e (M_surf_mix - M_bulk)                         (R-5, R-6)
    const real pp = mul_(mul_(p, p), fma_(p, m2, real(3)));           // 1/4 (2 - phit)(1 + phit)^2
    const real q = mul_(sub_(p, real(0.5)), k.two_inv_sigma);          // phit / sigma_surf
    const real e = exp_neg(mul_(-q, q), etab, k);
    real mb, ms;
    if (MOB != 0) {
        const real ch = clamp01(c);                                   // clamp(c, 0, 1)
        const real h = mul_(mul_(ch, ch), fma_(ch, m2, real(3)));     // smoothstep h(c)
        const real MBb = MOB == 2 ? mo.MBb : k.MBb, dMb = MOB == 2 ? mo.dMb : k.dMb;
        const real MBs = MOB == 2 ? mo.MBs : k.MBs, dMs = MOB == 2 ? mo.dMs : k.dMs;
        mb = mul_(pp, fma_(h, dMb, MBb));
        ms = fma_(h, dMs, MBs);
    } else {   // M_A = M_B: h (M_A - M_B) + M_B == M_B exactly
        mb = mul_(pp, k.MBb);
        ms = k.MBs;
    }
    M = fma_(e, sub_(ms, mb), mb);
}

// The member's velocity divided by 2 dx, the form cell_update takes (central differences G, R-8).
template <typename real>
__device__ __forceinline__ void scaled_velocity(const KC<real> &k, const real *vel, int m, real &vx, real &vy) {
    vx = mul_(vel[(int64_t)m * kMembStride], k.inv_2dx);
    vy = mul_(vel[(int64_t)m * kMembStride + 1], k.inv_2dx);
}

// Face flux (M_a + M_b) (mu_b - mu_a) of the face between cells a and b (times 2/dx^2 of the
// flux F = (M_a + M_b)/2 (mu_b - mu_a)/dx^2).  The same expression is used for a face
// seen from either of its cells, so the divergence telescopes (exact mass conservation).
template <typename real>
__device__ __forceinline__ real face_flux(real Ma, real Mb, real mua, real mub) {
    return mul_(add_(Ma, Mb), sub_(mub, mua));
}

// Rows a3-a5: right-hand sides and the Euler-form stage update of one cell, given the four face
// fluxes (east, west, north, south) of the composition equation.
//   R_c   = (fe - fw) + (fn - fs), times 1/(2 dx^2)                (conservative)
//   S     = rho (v_x G_x phi + v_y G_y phi)                        (R-10)
//   R_phi = M_phi L(mu_phi) + S                                    (R-7)
//   R_rho = D_rho L(rho) - v . G(rho) - 2 S                        (R-9: the paper's sink
//           grad(phit) . (rho v) with phit = 2 phi - 1 (R-1) is 2 S; S + S is exact)
//   out   = base + coef R                                          (R-11)
// vx, vy are the member's velocity divided by 2 dx (folded once per segment, see scaled_velocity).
template <typename real>
__device__ __forceinline__ void cell_update(const KC<real> &k, real vx, real vy,
                                            real fe, real fw, real fn, real fs,
                                            real q0, real ql, real qr, real qd, real qu,
                                            real pl, real pr, real pd, real pu,
                                            real r0, real rl, real rr, real rd, real ru,
                                            real bc, real bp, real br,
                                            real &oc, real &op, real &orr) {
    const real m4 = real(-4);
    const real Rc2 = add_(sub_(fe, fw), sub_(fn, fs));                      // 2 dx^2 R_c
    const real lq = fma_(q0, m4, add_(add_(ql, qr), add_(qd, qu)));          // dx^2 L(mu_phi)
    const real S = mul_(r0, fma_(vx, sub_(pr, pl), mul_(vy, sub_(pu, pd))));
    const real Rp = fma_(lq, k.Mp_dx2, S);
    const real lr = fma_(r0, m4, add_(add_(rl, rr), add_(rd, ru)));          // dx^2 L(rho)
    const real adv = fma_(vx, sub_(rr, rl), mul_(vy, sub_(ru, rd)));
    const real Rr = sub_(fma_(lr, k.Dr_dx2, -adv), add_(S, S));
    oc = fma_(Rc2, k.coefc, bc);
    op = fma_(Rp, k.coef, bp);
    orr = fma_(Rr, k.coef, br);
}

}  // namespace pf
