/*
 * pf_oracle.c -- the CPU ORACLE for the PVD phase-field DNS time step.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the slow, plain, single-threaded
 * reference the CUDA path is checked against.  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * leg may load it.  The product library (paper_2312_05410_b200/) never links,
 * loads or calls it, and it shares no code, header or constant generator with
 * that library: every formula below is written out again from the paper.
 *
 * Citations: "P:L" = /root/reference/PAPER.md line L, "S:L" = SPEC.md line L,
 * "R-n" = the reading of the paper recorded in DESIGN.md section 3 (copied from
 * SURVEY.md 8(c.2)).  The discrete model is DESIGN.md section 2.
 *
 * Structure: one whole-field pass per operator (Laplacian, gradient, chemical
 * potentials, mobility, fluxes, right-hand sides, update), exactly in the order
 * the equations are stated, fp64 throughout, no blocking or fusion.  Build with
 * -O2 -ffp-contract=off and without fast-math (R-16, R-19).
 *
 * Pinning status of every function is listed in DESIGN.md section 4; all of
 * them are pinned by tests in tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------------- */
/* Model parameters (the oracle's own struct; mirrors nothing in the library) */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t nx, ny;          /* grid: x periodic, y no-flux (R-12)              */
    double dx, dt;
    double kappa_c, kappa_phi, W_c, W_phi;          /* free energy (R-2..R-4)   */
    double MA_bulk, MB_bulk, MA_surf, MB_surf, sigma_surf; /* P:312-324, R-6    */
    double M_phi;            /* interface mobility (R-7)                        */
    double D_rho, rho_in;    /* vapour transport (R-9, R-12)         */
    double v_x, v_y;         /* vapour velocity of this member (R-10)           */
    int32_t fe;              /* composition free energy: 0 polynomial (R-2), 1 regular solution (R-28) */
    double omega, temp;      /* regular-solution interaction Omega and temperature T (R-28)          */
} orc_model;

/* Boundary rules for the ghost values (R-12). */
enum { ORC_MIRROR = 0, ORC_RESERVOIR = 1 };

/* Value of field u at (i, j) with the ghost rules of DESIGN.md 2 / SURVEY 8(c.1):
 * x wraps modulo nx; y mirrors about the boundary face (u[-1]=u[0],
 * u[-2]=u[1], u[ny]=u[ny-1], u[ny+1]=u[ny-2]); with ORC_RESERVOIR the top ghost
 * row holds the constant `top` (rho reservoir, R-12). */
static double nb_row(const double *u, int nx, int ny, int i, int j, int rule, double top, const double *toprow);
static double nb(const double *u, int nx, int ny, int i, int j, int rule, double top)
{
    return nb_row(u, nx, ny, i, j, rule, top, NULL);
}
/* As nb, with the reservoir row given per column (toprow[i], stochastic inflow R-27) when
 * toprow != NULL. */
static double nb_row(const double *u, int nx, int ny, int i, int j, int rule, double top, const double *toprow)
{
    while (i < 0) i += nx;       /* periodic wrap in x */
    while (i >= nx) i -= nx;
    if (j < 0) j = -1 - j;
    if (j >= ny) {
        if (rule == ORC_RESERVOIR) return toprow ? toprow[i] : top;
        j = 2 * ny - 1 - j;
    }
    return u[(size_t)j * nx + i];
}

/* ------------------------------------------------------------------------- */
/* Pointwise constitutive functions (R-1, R-5, R-6)               */
/* ------------------------------------------------------------------------- */

/* h(c): smooth switching function, smoothstep on c clamped to [0,1] (R-5). */
double orc_h(double c)
{
    double ch = c;
    if (ch < 0.0) ch = 0.0;
    if (ch > 1.0) ch = 1.0;
    return ch * ch * (3.0 - 2.0 * ch);
}

/* p(phi) = 1/4 (2 - phit)(1 + phit)^2 with phit = 2 phi - 1 (R-1).
 * Written literally in the paper's variable. */
double orc_p(double phi)
{
    double phit = 2.0 * phi - 1.0;
    return 0.25 * (2.0 - phit) * (1.0 + phit) * (1.0 + phit);
}

/* e(phi) = exp(-(phit / sigma_surf)^2) (R-1). */
double orc_e(double phi, double sigma_surf)
{
    double phit = 2.0 * phi - 1.0;
    double q = phit / sigma_surf;
    return exp(-(q * q));
}

/* M_c(phi, c) = M_bulk + M_surf with the garbled self-reference read as M_bulk
 * (R-6):
 *   M_bulk = p(phi) (h MA_bulk + (1-h) MB_bulk)
 *   M_surf = e(phi) (h MA_surf + (1-h) MB_surf - M_bulk)                     */
double orc_mobility_c(const orc_model *m, double c, double phi)
{
    double h = orc_h(c);
    double m_bulk = orc_p(phi) * (h * m->MA_bulk + (1.0 - h) * m->MB_bulk);
    double m_surf = orc_e(phi, m->sigma_surf) * (h * m->MA_surf + (1.0 - h) * m->MB_surf - m_bulk);
    return m_bulk + m_surf;
}

/* ------------------------------------------------------------------------- */
/* Difference operators ("second-order-central-difference", R-8)       */
/* ------------------------------------------------------------------------- */

/* L(u) = (u_{i+1,j} + u_{i-1,j} + u_{i,j+1} + u_{i,j-1} - 4 u_ij) / dx^2. */
static void laplacian_row(int nx, int ny, double dx, const double *u, int rule, double top, const double *toprow,
                          double *out);
void orc_laplacian(int nx, int ny, double dx, const double *u, int rule, double top, double *out)
{
    laplacian_row(nx, ny, dx, u, rule, top, NULL, out);
}
static void laplacian_row(int nx, int ny, double dx, const double *u, int rule, double top, const double *toprow,
                          double *out)
{
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            double s = nb_row(u, nx, ny, i + 1, j, rule, top, toprow) + nb_row(u, nx, ny, i - 1, j, rule, top, toprow)
                     + nb_row(u, nx, ny, i, j + 1, rule, top, toprow) + nb_row(u, nx, ny, i, j - 1, rule, top, toprow)
                     - 4.0 * u[(size_t)j * nx + i];
            out[(size_t)j * nx + i] = s / (dx * dx);
        }
}

/* G(u) = ((u_{i+1,j} - u_{i-1,j}) / (2dx), (u_{i,j+1} - u_{i,j-1}) / (2dx)). */
static void gradient_row(int nx, int ny, double dx, const double *u, int rule, double top, const double *toprow,
                         double *gx, double *gy)
{
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            gx[(size_t)j * nx + i] = (nb_row(u, nx, ny, i + 1, j, rule, top, toprow) - nb_row(u, nx, ny, i - 1, j, rule, top, toprow)) / (2.0 * dx);
            gy[(size_t)j * nx + i] = (nb_row(u, nx, ny, i, j + 1, rule, top, toprow) - nb_row(u, nx, ny, i, j - 1, rule, top, toprow)) / (2.0 * dx);
        }
}
void orc_gradient(int nx, int ny, double dx, const double *u, int rule, double top,
                  double *gx, double *gy)
{
    gradient_row(nx, ny, dx, u, rule, top, NULL, gx, gy);
}

/* ------------------------------------------------------------------------- */
/* Chemical potentials = variational derivatives of F (R-2..R-4) */
/*   f(c,phi) = W_c c^2 (1-c)^2 phi + W_phi phi^2 (1-phi)^2                    */
/*   mu_c   = df/dc   - kappa_c   L(c)                                         */
/*   mu_phi = df/dphi - kappa_phi L(phi)                                       */
/* ------------------------------------------------------------------------- */
/* Regular-solution variant (R-28; north_star "double-well and regular-solution derivatives"):
 *   g(c) = Omega c~(1-c~) + T (c~ ln c~ + (1-c~) ln(1-c~)),  c~ = min(max(c, eps), 1-eps),
 *   f = g(c~) phi + W_phi phi^2 (1-phi)^2,
 *   df/dc = phi (Omega (1 - 2c~) + T (ln c~ - ln(1-c~))),  df/dphi = g(c~) + ...        */
static const double ORC_FE_EPS = 1e-9;
static double clampe(double c) { return c < ORC_FE_EPS ? ORC_FE_EPS : (c > 1.0 - ORC_FE_EPS ? 1.0 - ORC_FE_EPS : c); }
static double g_rs(const orc_model *m, double c)
{
    double t = clampe(c);
    return m->omega * t * (1.0 - t) + m->temp * (t * log(t) + (1.0 - t) * log(1.0 - t));
}
static double dg_rs(const orc_model *m, double c)
{
    double t = clampe(c);
    return m->omega * (1.0 - 2.0 * t) + m->temp * (log(t) - log(1.0 - t));
}

void orc_mu(const orc_model *m, const double *c, const double *phi, double *mu_c, double *mu_phi)
{
    int nx = m->nx, ny = m->ny;
    size_t n = (size_t)nx * ny;
    double *lc = (double *)malloc(n * sizeof(double));
    double *lp = (double *)malloc(n * sizeof(double));
    orc_laplacian(nx, ny, m->dx, c, ORC_MIRROR, 0.0, lc);
    orc_laplacian(nx, ny, m->dx, phi, ORC_MIRROR, 0.0, lp);
    for (size_t k = 0; k < n; ++k) {
        double cc = c[k], pp = phi[k];
        double dfdc, dfdphi;
        if (m->fe == 1) {
            dfdc = pp * dg_rs(m, cc);
            dfdphi = g_rs(m, cc) + 2.0 * m->W_phi * pp * (1.0 - pp) * (1.0 - 2.0 * pp);
        } else {
            dfdc = 2.0 * m->W_c * cc * (1.0 - cc) * (1.0 - 2.0 * cc) * pp;
            dfdphi = m->W_c * cc * cc * (1.0 - cc) * (1.0 - cc)
                   + 2.0 * m->W_phi * pp * (1.0 - pp) * (1.0 - 2.0 * pp);
        }
        mu_c[k] = dfdc - m->kappa_c * lc[k];
        mu_phi[k] = dfdphi - m->kappa_phi * lp[k];
    }
    free(lc);
    free(lp);
}

/* Cell-centre mobility field M_c(phi, c). */
void orc_mobility_field(const orc_model *m, const double *c, const double *phi, double *M)
{
    size_t n = (size_t)m->nx * m->ny;
    for (size_t k = 0; k < n; ++k) M[k] = orc_mobility_c(m, c[k], phi[k]);
}

/* Deposition source S = grad(phi) . (rho v) (R-10); v constant. */
void orc_source(const orc_model *m, const double *phi, const double *rho, double *S)
{
    int nx = m->nx, ny = m->ny;
    size_t n = (size_t)nx * ny;
    double *gx = (double *)malloc(n * sizeof(double));
    double *gy = (double *)malloc(n * sizeof(double));
    orc_gradient(nx, ny, m->dx, phi, ORC_MIRROR, 0.0, gx, gy);
    for (size_t k = 0; k < n; ++k) S[k] = rho[k] * (m->v_x * gx[k] + m->v_y * gy[k]);
    free(gx);
    free(gy);
}

/* Right-hand sides (R-7..R-9):
 *   R_c   = sum over the 4 faces of the face flux  F = 1/2 (M_a + M_b)(mu_b - mu_a)/dx^2,
 *           zero flux through the two y-boundary faces;
 *   R_phi = M_phi L(mu_phi) + S,  S = grad(phi) . (rho v)  (phi in [0,1]: the paper's
 *           d(phit)/dt source grad(phit).(rho v) divided by d(phit)/d(phi) = 2, R-1);
 *   R_rho = D_rho L(rho) - v . G(rho) - grad(phit) . (rho v)   with phit = 2 phi - 1
 *           (P:340 written in the paper's variable phit in [-1,1]; R-9).
 * Any output pointer may be NULL.                                             */
static void rhs_row(const orc_model *m, const double *c, const double *phi, const double *rho, const double *toprow,
                    double *Rc, double *Rphi, double *Rrho, double *S_out);
void orc_rhs(const orc_model *m, const double *c, const double *phi, const double *rho,
             double *Rc, double *Rphi, double *Rrho, double *S_out)
{
    rhs_row(m, c, phi, rho, NULL, Rc, Rphi, Rrho, S_out);
}
/* The right-hand sides; toprow (or NULL: rho_in everywhere) is the rho reservoir row. */
static void rhs_row(const orc_model *m, const double *c, const double *phi, const double *rho, const double *toprow,
                    double *Rc, double *Rphi, double *Rrho, double *S_out)
{
    int nx = m->nx, ny = m->ny;
    size_t n = (size_t)nx * ny;
    double dx2 = m->dx * m->dx;
    double *mu_c = (double *)malloc(n * sizeof(double));
    double *mu_p = (double *)malloc(n * sizeof(double));
    double *M = (double *)malloc(n * sizeof(double));
    double *S = (double *)malloc(n * sizeof(double));
    double *Fx = (double *)malloc(n * sizeof(double));   /* Fx[j][i] : face i+1/2 */
    double *Fy = (double *)malloc(n * sizeof(double));   /* Fy[j][i] : face j+1/2 */
    double *lmu = (double *)malloc(n * sizeof(double));
    double *lrho = (double *)malloc(n * sizeof(double));
    double *grx = (double *)malloc(n * sizeof(double));
    double *gry = (double *)malloc(n * sizeof(double));
    double *phit = (double *)malloc(n * sizeof(double));
    double *gpx = (double *)malloc(n * sizeof(double));
    double *gpy = (double *)malloc(n * sizeof(double));

    orc_mu(m, c, phi, mu_c, mu_p);
    orc_mobility_field(m, c, phi, M);
    orc_source(m, phi, rho, S);

    /* face fluxes of the composition equation */
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            size_t k = (size_t)j * nx + i;
            size_t kx = (size_t)j * nx + (i + 1) % nx;
            Fx[k] = 0.5 * (M[k] + M[kx]) * (mu_c[kx] - mu_c[k]) / dx2;
            if (j < ny - 1) {
                size_t ky = (size_t)(j + 1) * nx + i;
                Fy[k] = 0.5 * (M[k] + M[ky]) * (mu_c[ky] - mu_c[k]) / dx2;
            } else {
                Fy[k] = 0.0;                     /* no-flux top face (R-12) */
            }
        }
    if (Rc)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                size_t k = (size_t)j * nx + i;
                double fxm = Fx[(size_t)j * nx + (i - 1 + nx) % nx];
                double fym = (j > 0) ? Fy[(size_t)(j - 1) * nx + i] : 0.0; /* no-flux bottom */
                Rc[k] = (Fx[k] - fxm) + (Fy[k] - fym);
            }

    orc_laplacian(nx, ny, m->dx, mu_p, ORC_MIRROR, 0.0, lmu);
    if (Rphi)
        for (size_t k = 0; k < n; ++k) Rphi[k] = m->M_phi * lmu[k] + S[k];

    laplacian_row(nx, ny, m->dx, rho, ORC_RESERVOIR, m->rho_in, toprow, lrho);
    gradient_row(nx, ny, m->dx, rho, ORC_RESERVOIR, m->rho_in, toprow, grx, gry);
    /* vapour sink of P:340 in the paper's order parameter phit = 2 phi - 1 (R-1, R-9) */
    for (size_t k = 0; k < n; ++k) phit[k] = 2.0 * phi[k] - 1.0;
    orc_gradient(nx, ny, m->dx, phit, ORC_MIRROR, 0.0, gpx, gpy);
    if (Rrho)
        for (size_t k = 0; k < n; ++k)
            Rrho[k] = m->D_rho * lrho[k] - (m->v_x * grx[k] + m->v_y * gry[k])
                    - rho[k] * (m->v_x * gpx[k] + m->v_y * gpy[k]);
    if (S_out) memcpy(S_out, S, n * sizeof(double));

    free(mu_c); free(mu_p); free(M); free(S); free(Fx); free(Fy);
    free(lmu); free(lrho); free(grx); free(gry); free(phit); free(gpx); free(gpy);
}

/* One explicit midpoint step (R-11):
 *   u*      = u^n + (dt/2) R(u^n)
 *   u^{n+1} = u^n + dt R(u*)                                                  */
static void step_row(const orc_model *m, double *c, double *phi, double *rho, const double *toprow);
void orc_step(const orc_model *m, double *c, double *phi, double *rho)
{
    step_row(m, c, phi, rho, NULL);
}
static void step_row(const orc_model *m, double *c, double *phi, double *rho, const double *toprow)
{
    size_t n = (size_t)m->nx * m->ny;
    double *Rc = (double *)malloc(n * sizeof(double));
    double *Rp = (double *)malloc(n * sizeof(double));
    double *Rr = (double *)malloc(n * sizeof(double));
    double *cs = (double *)malloc(n * sizeof(double));
    double *ps = (double *)malloc(n * sizeof(double));
    double *rs = (double *)malloc(n * sizeof(double));
    double hdt = 0.5 * m->dt;

    rhs_row(m, c, phi, rho, toprow, Rc, Rp, Rr, NULL);
    for (size_t k = 0; k < n; ++k) {
        cs[k] = c[k] + hdt * Rc[k];
        ps[k] = phi[k] + hdt * Rp[k];
        rs[k] = rho[k] + hdt * Rr[k];
    }
    rhs_row(m, cs, ps, rs, toprow, Rc, Rp, Rr, NULL);
    for (size_t k = 0; k < n; ++k) {
        c[k] = c[k] + m->dt * Rc[k];
        phi[k] = phi[k] + m->dt * Rp[k];
        rho[k] = rho[k] + m->dt * Rr[k];
    }
    free(Rc); free(Rp); free(Rr); free(cs); free(ps); free(rs);
}

/* n steps of orc_step. */
void orc_run(const orc_model *m, double *c, double *phi, double *rho, int64_t nsteps)
{
    for (int64_t s = 0; s < nsteps; ++s) orc_step(m, c, phi, rho);
}

/* Explicit forward Euler step u^{n+1} = u^n + dt R(u^n).  Not on the product
 * path; used only by the tests to show that the midpoint pin can tell the two
 * integrators apart. */
void orc_step_euler(const orc_model *m, double *c, double *phi, double *rho)
{
    size_t n = (size_t)m->nx * m->ny;
    double *Rc = (double *)malloc(n * sizeof(double));
    double *Rp = (double *)malloc(n * sizeof(double));
    double *Rr = (double *)malloc(n * sizeof(double));
    orc_rhs(m, c, phi, rho, Rc, Rp, Rr, NULL);
    for (size_t k = 0; k < n; ++k) {
        c[k] += m->dt * Rc[k];
        phi[k] += m->dt * Rp[k];
        rho[k] += m->dt * Rr[k];
    }
    free(Rc); free(Rp); free(Rr);
}

/* ------------------------------------------------------------------------- */
/* Diagnostics (north_star "Reductions")       */
/* ------------------------------------------------------------------------- */

/* Neumaier-compensated running sum. */
typedef struct { double s, comp; } nsum;
static void nadd(nsum *a, double x)
{
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->comp += (a->s - t) + x;
    else a->comp += (x - t) + a->s;
    a->s = t;
}
static double nval(const nsum *a) { return a->s + a->comp; }

/* Discrete free energy
 *   E_h = dx^2 sum_cells f(c, phi)
 *       + sum_{interior faces} [kappa_c/2 (dc)^2 + kappa_phi/2 (dphi)^2]
 * with f = W_c c^2 (1-c)^2 phi + W_phi phi^2 (1-phi)^2 (R-2); interior faces are
 * every x-face (periodic) and the y-faces between rows j and j+1 (the mirror
 * ghost makes the boundary faces contribute zero).  Summed in row-major cell
 * order, per cell: bulk term, x-face to the right, y-face above.             */
double orc_energy(const orc_model *m, const double *c, const double *phi)
{
    int nx = m->nx, ny = m->ny;
    double dx2 = m->dx * m->dx;
    nsum E = {0.0, 0.0};
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            size_t k = (size_t)j * nx + i;
            size_t kx = (size_t)j * nx + (i + 1) % nx;
            double cc = c[k], pp = phi[k];
            double fc = m->fe == 1 ? g_rs(m, cc) : m->W_c * cc * cc * (1.0 - cc) * (1.0 - cc);
            double f = fc * pp + m->W_phi * pp * pp * (1.0 - pp) * (1.0 - pp);
            nadd(&E, dx2 * f);
            double dcx = c[kx] - cc, dpx = phi[kx] - pp;
            nadd(&E, 0.5 * m->kappa_c * dcx * dcx + 0.5 * m->kappa_phi * dpx * dpx);
            if (j < ny - 1) {
                size_t ky = (size_t)(j + 1) * nx + i;
                double dcy = c[ky] - cc, dpy = phi[ky] - pp;
                nadd(&E, 0.5 * m->kappa_c * dcy * dcy + 0.5 * m->kappa_phi * dpy * dpy);
            }
        }
    return nval(&E);
}

/* out[0] = dx^2 sum c (mass of c), out[1] = dx^2 sum phi, out[2] = dx^2 sum rho,
 * out[3] = E_h, out[4] = number of cells where any field is not finite.      */
void orc_diagnostics(const orc_model *m, const double *c, const double *phi, const double *rho,
                     double out[5])
{
    size_t n = (size_t)m->nx * m->ny;
    double dx2 = m->dx * m->dx;
    nsum sc = {0, 0}, sp = {0, 0}, sr = {0, 0};
    double bad = 0.0;
    for (size_t k = 0; k < n; ++k) {
        nadd(&sc, c[k]);
        nadd(&sp, phi[k]);
        nadd(&sr, rho[k]);
        if (!isfinite(c[k]) || !isfinite(phi[k]) || !isfinite(rho[k])) bad += 1.0;
    }
    out[0] = dx2 * nval(&sc);
    out[1] = dx2 * nval(&sp);
    out[2] = dx2 * nval(&sr);
    out[3] = orc_energy(m, c, phi);
    out[4] = bad;
}

/* ------------------------------------------------------------------------- */
/* Seeded synthetic inputs (R-13..R-16).  This is the oracle's OWN copy of the */
/* counter-based generator; the library implements the same spec separately,  */
/* and tests/test_ic.py checks the two bit for bit.                            */
/* ------------------------------------------------------------------------- */

/* SplitMix64 finaliser of z + golden gamma (R-16). */
uint64_t orc_sm64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
/* key(seed, stream) = sm(seed ^ (stream * 0xD1B54A32D192ED03)); draw(k) = sm(key + k). */
uint64_t orc_draw(uint64_t seed, uint64_t stream, uint64_t k)
{
    uint64_t key = orc_sm64(seed ^ (stream * 0xD1B54A32D192ED03ull));
    return orc_sm64(key + k);
}
/* U = (draw >> 11) * 2^-53 in [0, 1). */
double orc_uniform(uint64_t seed, uint64_t stream, uint64_t k)
{
    return (double)(orc_draw(seed, stream, k) >> 11) * 0x1.0p-53;
}
/* Gaussian by Box-Muller, cos branch, draws k = 2 idx and 2 idx + 1 (R-16). */
double orc_gauss(uint64_t seed, uint64_t stream, uint64_t idx)
{
    double u1 = orc_uniform(seed, stream, 2 * idx);
    double u2 = orc_uniform(seed, stream, 2 * idx + 1);
    return sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * M_PI * u2);
}

/* Initial-condition recipe (R-14), the oracle's own description. */
typedef struct {
    int32_t kind;            /* 0 film, 1 rough tanh substrate, 2 columnar film   */
    double height, amp, wavelength;
    int32_t ncols;
    double c0, c_lo, c_hi, noise_c, noise_phi;
    int32_t noise_c_gaussian;
    double kappa_phi, W_phi, rho_in;
    double v0, theta_deg, rate_lo, rate_hi;
    double theta_span;       /* per-member angle sweep width in degrees (R-21) */
    double mob_lo, mob_hi;   /* per-member species-mobility multipliers (R-23) */
    uint64_t seed;
} orc_ic;

/* Velocity of global member m (R-10, R-15, R-21):
 *   v0_m = v0 (rate_lo + (rate_hi - rate_lo) U(seed, 8m+3, 0));
 *   theta_m = theta_deg + theta_span U(seed, 8m+4, 0)   (theta_span = 0: theta_deg; the paper
 *             sweeps the deposition angle over 50..90 degrees);
 *   v = v0_m (cos theta_m, -sin theta_m).                                   */
void orc_member_velocity(const orc_ic *ic, int64_t member, double *v_x, double *v_y)
{
    double u = orc_uniform(ic->seed, (uint64_t)member * 8u + 3u, 0);
    double mult = ic->rate_lo + (ic->rate_hi - ic->rate_lo) * u;
    double v0m = ic->v0 * mult;
    double th_deg = ic->theta_deg;
    if (ic->theta_span != 0.0)
        th_deg = ic->theta_deg + ic->theta_span * orc_uniform(ic->seed, (uint64_t)member * 8u + 4u, 0);
    double th = th_deg * (M_PI / 180.0);
    *v_x = v0m * cos(th);
    *v_y = -(v0m * sin(th));
}

/* Species-mobility multipliers of global member m (R-23; P:352 varies "species mobilites (M_A,
 * M_B)" between trajectories): a scales both mobilities of species A, b both of species B,
 *   a = mob_lo + (mob_hi - mob_lo) U(seed, 8m+5, 0),  b = mob_lo + (mob_hi - mob_lo) U(seed, 8m+6, 0). */
void orc_member_mobility(const orc_ic *ic, int64_t member, double *a, double *b)
{
    *a = ic->mob_lo + (ic->mob_hi - ic->mob_lo) * orc_uniform(ic->seed, (uint64_t)member * 8u + 5u, 0);
    *b = ic->mob_lo + (ic->mob_hi - ic->mob_lo) * orc_uniform(ic->seed, (uint64_t)member * 8u + 6u, 0);
}

/* Stochastic inflow (R-27; "top boundary rho = per-column draw from a Gaussian
 * N(rho_in, noise_sigma) truncated to [0, 2 rho_in], re-drawn each step"; "a random draw
 * from a truncated Gaussian distribution"): the reservoir value of column i for global step
 * `step` of global member m.  Attempt a = 0..7 draws z_a by Box-Muller (cosine branch) from the
 * uniforms at counters 2q, 2q+1, q = (step nx + i) 8 + a, of stream 8m+7; the first
 * v = rho_in + sigma z_a inside [0, 2 rho_in] is taken; after 8 rejections v = rho_in. */
double orc_inflow(uint64_t seed, int64_t member, int64_t step, int nx, int i, double rho_in, double sigma)
{
    const uint64_t stream = (uint64_t)member * 8u + 7u;
    for (int a = 0; a < 8; ++a) {
        uint64_t q = ((uint64_t)step * (uint64_t)nx + (uint64_t)i) * 8u + (uint64_t)a;
        double u1 = orc_uniform(seed, stream, 2 * q), u2 = orc_uniform(seed, stream, 2 * q + 1);
        double z = sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * M_PI * u2);
        double v = rho_in + sigma * z;
        if (v >= 0.0 && v <= 2.0 * rho_in) return v;
    }
    return rho_in;
}

/* n midpoint steps with the stochastic inflow row of each step (both stages of a step use the
 * same row); step0 = global index of the first step. */
void orc_run_inflow(const orc_model *m, double *c, double *phi, double *rho, int64_t nsteps, int64_t step0,
                    uint64_t seed, int64_t member, double sigma)
{
    double *row = (double *)malloc((size_t)m->nx * sizeof(double));
    for (int64_t s = 0; s < nsteps; ++s) {
        for (int i = 0; i < m->nx; ++i) row[i] = orc_inflow(seed, member, step0 + s, m->nx, i, m->rho_in, sigma);
        step_row(m, c, phi, rho, row);
    }
    free(row);
}

static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* Fill global rows [y0, y0+rows) of member m (row-major (j-y0)*nx+i, j = 0 bottom);
 * every value depends only on (i, j, nx, member), not on the window. */
int orc_initial_fields_rows(const orc_ic *ic, int nx, int64_t member, int y0, int rows,
                            double *c, double *phi, double *rho)
{
    uint64_t sc = (uint64_t)member * 8u + 0u, sp = (uint64_t)member * 8u + 1u;
    uint64_t scut = (uint64_t)member * 8u + 2u;
    double delta = sqrt(2.0 * ic->kappa_phi / ic->W_phi);
    int64_t *cuts = NULL;
    if (ic->kind == 2) {
        /* 63 distinct cut points in {1..nx-1}: cut = 1 + floor(U (nx-1)), skip
         * duplicates, then sort (R-14). */
        int ncut = ic->ncols - 1;
        if (ncut < 0 || ncut > nx - 1) return -1;
        cuts = (int64_t *)malloc((size_t)(ncut + 2) * sizeof(int64_t));
        int have = 0;
        for (uint64_t k = 0; have < ncut; ++k) {
            int64_t cut = 1 + (int64_t)floor(orc_uniform(ic->seed, scut, k) * (double)(nx - 1));
            int dup = 0;
            for (int q = 0; q < have; ++q) if (cuts[q] == cut) { dup = 1; break; }
            if (!dup) cuts[have++] = cut;
        }
        qsort(cuts, (size_t)ncut, sizeof(int64_t), cmp_i64);
    }
    for (int j = y0; j < y0 + rows; ++j)
        for (int i = 0; i < nx; ++i) {
            size_t k = (size_t)j * nx + i;         /* global counter index      */
            size_t o = (size_t)(j - y0) * nx + i;  /* position in the window    */
            double p, cc;
            if (ic->kind == 0) {
                double solid = (double)j < ic->height ? 1.0 : 0.0;
                double u = orc_uniform(ic->seed, sp, k);
                p = solid + ic->noise_phi * (2.0 * u - 1.0);
                rho[o] = ic->rho_in * (1.0 - solid);
            } else {
                double Hi = ic->height + ic->amp * sin(2.0 * M_PI * (double)i / ic->wavelength);
                p = 0.5 * (1.0 - tanh(((double)j - Hi) / delta));
                rho[o] = ic->rho_in * (1.0 - p);
            }
            if (ic->kind == 2) {
                int q = 0;
                while (q < ic->ncols - 1 && (int64_t)i >= cuts[q]) ++q;   /* column index */
                cc = (q % 2 == 0) ? ic->c_lo : ic->c_hi;
            } else if (ic->noise_c_gaussian) {
                cc = ic->c0 + ic->noise_c * orc_gauss(ic->seed, sc, k);
            } else {
                double u = orc_uniform(ic->seed, sc, k);
                cc = ic->c0 + ic->noise_c * (2.0 * u - 1.0);
            }
            phi[o] = p;
            c[o] = cc;
        }
    free(cuts);
    return 0;
}

/* Whole grid of member m. */
int orc_initial_fields(const orc_ic *ic, int nx, int ny, int64_t member,
                       double *c, double *phi, double *rho)
{
    return orc_initial_fields_rows(ic, nx, member, 0, ny, c, phi, rho);
}

/* Largest stable dt per R-18 (80% of the explicit-midpoint limit of the
 * 13-point biharmonic including the |f''| <= 2W term). */
double orc_dt_max(const orc_model *m, double M_c_max)
{
    double dx2 = m->dx * m->dx, dx4 = dx2 * dx2;
    double fpp = m->fe == 1 ? 2.0 * fabs(m->omega) + m->temp / (0.05 * 0.95) : 2.0 * m->W_c;   /* R-18, R-28 */
    double a = M_c_max * (64.0 * m->kappa_c / dx4 + 8.0 * fpp / dx2);
    double b = m->M_phi * (64.0 * m->kappa_phi / dx4 + 16.0 * m->W_phi / dx2);
    double d = 8.0 * m->D_rho / dx2;
    double mx = a;
    if (b > mx) mx = b;
    if (d > mx) mx = d;
    return 1.6 / mx;
}
