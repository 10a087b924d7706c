"""Name mapping from the library's pf_params to the oracle's Model / IC (test glue: renames
fields, computes nothing of the method)."""
from paper_2312_05410_b200 import pf


def model_kw(p):
    return dict(nx=p.nx, ny=p.ny, dx=p.dx, dt=p.dt, kappa_c=p.kappa_c, kappa_phi=p.kappa_phi,
                W_c=p.W_c, W_phi=p.W_phi, MA_bulk=p.M_A_bulk, MB_bulk=p.M_B_bulk,
                MA_surf=p.M_A_surf, MB_surf=p.M_B_surf, sigma_surf=p.sigma_surf, M_phi=p.M_phi,
                D_rho=p.D_rho, rho_in=p.rho_in, fe=p.fe_model, omega=p.omega, temp=p.temp_rs)


def ic_kw(p):
    kinds = {pf.PF_IC_FILM: "film", pf.PF_IC_ROUGH_SUBSTRATE: "rough", pf.PF_IC_COLUMNS: "columns"}
    return dict(kind=kinds[p.ic], height=p.ic_height, amp=p.ic_amp, wavelength=p.ic_wavelength,
                ncols=p.ic_ncols, c0=p.ic_c0, c_lo=p.ic_c_lo, c_hi=p.ic_c_hi, noise_c=p.noise_c,
                noise_phi=p.noise_phi, noise_c_gaussian=bool(p.noise_c_gaussian),
                kappa_phi=p.kappa_phi, W_phi=p.W_phi, rho_in=p.rho_in, v0=p.v0,
                theta_deg=p.theta_deg, rate_lo=p.rate_lo, rate_hi=p.rate_hi, theta_span=p.theta_span,
                mob_lo=p.mob_lo, mob_hi=p.mob_hi, seed=p.seed)


def oracle_member(ora, p, member_global):
    """(Model with the member's velocity and mobilities, IC) for the oracle."""
    ic = ora.IC(**ic_kw(p))
    m = ora.member_model_sweep(ora.Model(**model_kw(p)), ic, member_global)
    return m, ic


def normwise(gpu, ref):
    """R-17: max|F_gpu - F_ora| / max|F_ora| per field, max over fields."""
    err = 0.0
    for g, r in zip(gpu, ref):
        den = max(abs(r).max(), 1e-300)
        err = max(err, float(abs(g - r).max() / den))
    return err
