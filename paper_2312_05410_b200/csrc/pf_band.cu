// pf_band.cu -- small-grid path (SURVEY 7 item 6 / VERDICT r1 "B10"): every step of a check
// interval in ONE launch, the state resident in shared memory, halos moved through distributed
// shared memory inside a thread-block cluster.
//
// Grids too small to fill the GPU (configs[0] 64^2) are latency-bound: two stage launches per step
// (pair kernel) or two grid-wide barriers per step with an L2 reload of every tile (persistent tile
// kernel) dominate.  band_kernel gives every member one cluster of B <= 16 blocks (one SM each);
// block i of the cluster owns the band of rows [ny i / B, ny (i+1) / B) (>= 2 rows) over the full
// width.  The band's c, phi, rho plus a 2-row halo and 2 periodic ghost columns live in shared
// memory for the whole launch.  Per midpoint stage:
//   A  mu_c, mu_phi, M of rows -1 .. h (row a2) into shared memory;
//   B  face fluxes, source, vapour and the Euler-form update of the band's rows (rows a3-a5) into
//      registers (stage 1 also keeps u^n there as the stage-2 base);
//   C  the new values go to the block's own rows (with their periodic ghost columns and, at the
//      global y boundaries, the mirror rows, R-12), and the two bottom / two top rows are pushed
//      straight into the neighbouring blocks' halo rows with st.async stores that complete on the
//      receiving block's mbarrier of that halo parity;
//   -- a block waits for exactly its two neighbours' rows (no cluster-wide barrier per stage) --
// The halo rows are double-buffered by stage parity (a push of stage s+1 cannot overwrite rows a
// neighbour still reads in stage s), and no stage touches L2.  (Round 2: with the per-stage
// coefficient struct passed by reference -- selecting it at run time had copied it through local
// memory every stage, a third of the stage -- the st.async pushes beat one cluster barrier per
// stage, 1.34 vs 1.21 G cell-updates/s on configs[0]; build with -DPF_BAND_P2P=0 for the barrier.)  (Measured alternative: halo rows through a global buffer with per-band epoch
// flags, one block per SM over the whole GPU: 2-3x SLOWER than the persistent tile kernel -- every
// stage paid several L2 round trips.)
// The per-cell arithmetic is pf_cell.cuh with the argument order of the tile kernel, so results
// are bitwise those of every other stage kernel (tests/test_invariants_gpu.py).  The owned cells
// are written back to the state buffer at the end of the launch; the host rebuilds the ghost frame.
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdlib>

#include "pf_cell.cuh"
#include "pf_internal.h"

namespace cg = cooperative_groups;

namespace pf {
namespace {

constexpr int kBT = 512;         // threads per band block
constexpr int kMaxCells = 2048;  // owned cells per block (h * nx), MAXC = 1, 2 or 4 per thread
constexpr int kMaxCluster = 16;  // blocks per cluster (non-portable size)

// Shared-memory planes of one band.  U = c, phi, rho: storage rows [-2, -1] of stage parity 0, the
// same of parity 1, the h own rows, [h, h+1] of parity 0, of parity 1 (halo rows are double
// buffered by stage parity so that one cluster barrier per stage suffices); columns -2 .. nx+1.
// W = mu_c, mu_phi, M over rows -1 .. h, columns -1 .. nx.  hmax: the cluster's tallest band (every
// block uses the same plane sizes).
struct BandGeo {
    int hmax, nx, P, Q, uplane, wplane;
    __host__ __device__ BandGeo(int hmax_, int nx_) : hmax(hmax_), nx(nx_) {
        P = nx + 4;
        Q = nx + 2;
        uplane = (hmax + 8) * P;
        wplane = (hmax + 2) * Q;
    }
    // storage row of row r (-2 .. h+1) of a band of height h, halo parity par
    __host__ __device__ static int srow(int r, int h, int par) {
        return r < 0 ? r + 2 + 2 * par : (r < h ? r + 4 : r + 4 + 2 * par);
    }
    __host__ __device__ int u(int srw, int x) const { return srw * P + (x + 2); }
    __host__ __device__ int w(int r, int x) const { return (r + 1) * Q + (x + 1); }
    // + exp table + the two halo mbarriers (PF_BAND_P2P)
    __host__ __device__ size_t bytes(size_t esz) const { return (size_t)(3 * uplane + 3 * wplane) * esz + 64 * 8 + 16; }
};

// Phase timeline (diagnostic build, -DPF_TRACE=1; pf_debug_band_trace): per block of the first
// cluster and stage g < 128, thread 0's clock64 after phase A's CTA barrier, after phase B's, and
// after the stage's cluster barrier; [3] the stage start.
#ifndef PF_TRACE
#define PF_TRACE 0
#endif
__device__ long long g_btrace[16][128][4];
#define PF_BAND_STAMP(g, k)                                                                          \
    do {                                                                                             \
        if (PF_TRACE && threadIdx.x == 0 && blockIdx.x < 16 && (g) < 128) g_btrace[blockIdx.x][(g)][(k)] = clock64(); \
    } while (0)

#ifndef PF_BAND_P2P
#define PF_BAND_P2P 1   // halo rows by st.async + per-parity mbarriers (0: a cluster barrier per stage, 10% slower)
#endif
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// shared::cluster address of the same location in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_rank(uint32_t a, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
// asynchronous store into another CTA's shared memory, completing `bytes` on its mbarrier
__device__ __forceinline__ void st_async(uint32_t ra, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void st_async(uint32_t ra, float v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(ra),
                 "r"(__float_as_uint(v)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void hbar_init(uint64_t *b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void hbar_expect(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void hbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "HW_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra HW_%=;\n}" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}
// put() into the neighbour's plane (shared::cluster address rpl) with its periodic ghost copy
template <typename real>
__device__ __forceinline__ void push(uint32_t rpl, uint32_t rbar, const BandGeo &gg, int sr, int x, real v) {
    st_async(rpl + (uint32_t)gg.u(sr, x) * (uint32_t)sizeof(real), v, rbar);
    if (x < 2) st_async(rpl + (uint32_t)gg.u(sr, x + gg.nx) * (uint32_t)sizeof(real), v, rbar);
    if (x >= gg.nx - 2) st_async(rpl + (uint32_t)gg.u(sr, x - gg.nx) * (uint32_t)sizeof(real), v, rbar);
}

// Store value v of field plane `pl` at (storage row sr, column x) with its periodic ghost copy.
template <typename real>
__device__ __forceinline__ void put(real *pl, const BandGeo &gg, int sr, int x, real v) {
    PF_DCHECK(sr >= 0 && sr < gg.hmax + 8 && x >= 0 && x < gg.nx);
    pl[gg.u(sr, x)] = v;
    if (x < 2) pl[gg.u(sr, x + gg.nx)] = v;
    if (x >= gg.nx - 2) pl[gg.u(sr, x - gg.nx)] = v;
}

template <typename real, int MOB, int FE, int MAXC>
__global__ void __launch_bounds__(kBT, 1) band_kernel(Layout L, KC<real> k1, KC<real> k2, real *U,
                                                      const real *__restrict__ vel, int hmax, int64_t nsteps) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    const int nb = (int)cluster.num_blocks(), bi = (int)cluster.block_rank();
    const int m = L.m0 + (int)(blockIdx.x / nb);
    const int y0 = (int)((int64_t)L.ny_loc * bi / nb), y1 = (int)((int64_t)L.ny_loc * (bi + 1) / nb);
    const int h = y1 - y0, nx = L.nx;
    const bool bottom = bi == 0, top = bi == nb - 1;
    const BandGeo gg(hmax, nx);
    real *su = reinterpret_cast<real *>(smem_raw);
    real *sc = su, *sp = su + gg.uplane, *sr = su + 2 * gg.uplane;
    real *smc = su + 3 * gg.uplane, *smp = smc + gg.wplane, *sM = smp + gg.wplane;
    double *etab = reinterpret_cast<double *>(sM + gg.wplane);
    uint64_t *hbar = reinterpret_cast<uint64_t *>(etab + 64);   // halo rows of parity 0 / 1 arrived
    load_exp_table(etab);
    // the neighbours' shared memory (DSMEM): below = rank bi-1 (its rows h'-2, h'-1 are our rows
    // -2, -1), above = rank bi+1 (its rows 0, 1 are our rows h, h+1)
    real *su_dn = bottom ? su : cluster.map_shared_rank(su, bi - 1);
    real *su_up = top ? su : cluster.map_shared_rank(su, bi + 1);
    const int h_dn = bottom ? 0 : y0 - (int)((int64_t)L.ny_loc * (bi - 1) / nb);
    const int t = threadIdx.x;
    const real rho_in = k1.rho_in;
    const Mob<real> mo = MOB == 2 ? load_mob(vel, m) : Mob<real>{};
    real vx, vy;
    scaled_velocity(k1, vel, m, vx, vy);
    const real *gc = U + (int64_t)m * L.mstride;

    // ---- initial load: own rows and both parities of the halo rows from the state (ghost
    // rules by index, R-12) ----
    for (int q = t; q < (h + 8) * nx; q += kBT) {
        const int j = q / nx, x = q - j * nx;
        const int rr = j < 4 ? (j & 1) - 2 : (j < h + 4 ? j - 4 : h + ((j - h - 4) & 1));
        const int g = y0 + rr;
        const int gcp = g < 0 ? -1 - g : (g >= L.ny ? 2 * L.ny - 1 - g : g);
        put(sc, gg, j, x, gc[L.at(gcp, x)]);
        put(sp, gg, j, x, gc[L.fstride + L.at(gcp, x)]);
        put(sr, gg, j, x, g >= L.ny ? rho_in : gc[2 * L.fstride + L.at(gcp, x)]);
    }
    real base[3][MAXC];
    real outv[3][MAXC];
    const int nown = h * nx;
    // the cells of this thread, fixed for the whole launch (no index division in the step loop):
    // phase A cells q = t + i kBT (i < kAC) of the (h+2) x (nx+2) ring, phase B cells of the band
    constexpr int kAC = 4;
    const int nA = (h + 2) * (nx + 2);
    int arr[kAC], ax[kAC], by[MAXC], bx[MAXC];
#pragma unroll
    for (int i = 0; i < kAC; ++i) {
        const int q = t + i * kBT;
        arr[i] = q / (nx + 2) - 1;
        ax[i] = q - (arr[i] + 1) * (nx + 2) - 1;
    }
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
        const int q = t + i * kBT;
        by[i] = q / nx;
        bx[i] = q - by[i] * nx;
    }
    if (PF_BAND_P2P && t == 0) {
        hbar_init(&hbar[0]);
        hbar_init(&hbar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster.sync();   // every block has started (DSMEM targets exist) and loaded its band
    int par = 0;      // halo parity read by this stage
    // PF_BAND_P2P: the neighbours push their border rows with st.async, each completing its bytes
    // on this block's mbarrier of that halo parity: 2 rows x (nx + 4 ghost-column copies) x 3
    // fields per neighbour and stage.  A block waits for exactly the rows it reads, so no
    // cluster-wide barrier is needed per stage: the parity double-buffering makes a push of
    // stage g + 2 (same buffer as stage g) impossible before the neighbour finished reading it,
    // because that push needs the neighbour's stage-(g + 1) rows, sent after its reads.
    const uint32_t rx_bytes = (uint32_t)(((bottom ? 0 : 1) + (top ? 0 : 1)) * 2 * (nx + 4) * 3 * (int)sizeof(real));
    const uint32_t su_a = smem_addr(su), hb_a = smem_addr(hbar);
    const uint32_t rsu_dn = bottom ? 0u : mapa_rank(su_a, bi - 1), rhb_dn = bottom ? 0u : mapa_rank(hb_a, bi - 1);
    const uint32_t rsu_up = top ? 0u : mapa_rank(su_a, bi + 1), rhb_up = top ? 0u : mapa_rank(hb_a, bi + 1);
    const int64_t nstages = 2 * nsteps;

    // One midpoint stage; called with the stage's coefficient struct by reference (a struct selected
    // at run time, `KC k = stage == 1 ? k1 : k2`, was copied through local memory every stage:
    // ~1600 of ~4800 cycles per stage on configs[0], tools/trace_band.py)
    auto run_stage = [&](const KC<real> &k, const int stage, const int64_t s) {
            const int64_t g = 2 * s + stage - 1;   // stage index; reads halo parity par = g & 1
            if (PF_BAND_P2P && g > 0) {           // the neighbours' rows of stage g - 1
                if (t == 0) hbar_expect(&hbar[par], rx_bytes);
                hbar_wait(&hbar[par], (uint32_t)(((g - 1) >> 1) & 1));
            }
            PF_BAND_STAMP(g, 3);
            // A: mu_c, mu_phi, M on rows -1 .. h, columns -1 .. nx (row a2)
            auto cell_a = [&](int rr, int x) {
                const int o0 = gg.u(BandGeo::srow(rr, h, par), x);
                const int od = gg.u(BandGeo::srow(rr - 1, h, par), x), ou = gg.u(BandGeo::srow(rr + 1, h, par), x);
                real mc, mp, M;
                constitutive<real, MOB, FE>(k, mo, etab, sc[o0], sp[o0], sc[o0 - 1], sc[o0 + 1], sc[od], sc[ou],
                                            sp[o0 - 1], sp[o0 + 1], sp[od], sp[ou], mc, mp, M);
                smc[gg.w(rr, x)] = mc;
                smp[gg.w(rr, x)] = mp;
                sM[gg.w(rr, x)] = M;
            };
#pragma unroll
            for (int i = 0; i < kAC; ++i)
                if (t + i * kBT < nA) cell_a(arr[i], ax[i]);
            for (int q = t + kAC * kBT; q < nA; q += kBT) cell_a(q / (nx + 2) - 1, q - (q / (nx + 2)) * (nx + 2) - 1);
            __syncthreads();
            PF_BAND_STAMP(g, 0);
            // B: fluxes, source, vapour, update of the owned cells (rows a3-a5), into registers
#pragma unroll
            for (int i = 0; i < MAXC; ++i) {
                const int q = t + i * kBT;
                if (q < nown) {
                    const int y = by[i], x = bx[i];
                    const int c0 = gg.u(y + 4, x), w0 = gg.w(y, x), Q = gg.Q;
                    const int cd = gg.u(BandGeo::srow(y - 1, h, par), x), cu = gg.u(BandGeo::srow(y + 1, h, par), x);
                    if (stage == 1) {
                        base[0][i] = sc[c0];
                        base[1][i] = sp[c0];
                        base[2][i] = sr[c0];
                    }
                    const real fe = face_flux<real>(sM[w0], sM[w0 + 1], smc[w0], smc[w0 + 1]);
                    const real fw = face_flux<real>(sM[w0 - 1], sM[w0], smc[w0 - 1], smc[w0]);
                    const real fn = face_flux<real>(sM[w0], sM[w0 + Q], smc[w0], smc[w0 + Q]);
                    const real fs = face_flux<real>(sM[w0 - Q], sM[w0], smc[w0 - Q], smc[w0]);
                    cell_update<real>(k, vx, vy, fe, fw, fn, fs, smp[w0], smp[w0 - 1], smp[w0 + 1], smp[w0 - Q],
                                      smp[w0 + Q], sp[c0 - 1], sp[c0 + 1], sp[cd], sp[cu], sr[c0], sr[c0 - 1],
                                      sr[c0 + 1], sr[cd], sr[cu], base[0][i], base[1][i], base[2][i],
                                      outv[0][i], outv[1][i], outv[2][i]);
                }
            }
            __syncthreads();   // the block is done reading its own rows
            PF_BAND_STAMP(g, 1);
            // C: own rows (+ ghost columns, + mirror rows at the global boundaries) and the pushes
            // of the border rows into the neighbours' halos, all into halo parity np
            const int np = par ^ 1;
            const bool last = g == nstages - 1;   // P2P: no pushes nobody reads
#pragma unroll
            for (int i = 0; i < MAXC; ++i) {
                const int q = t + i * kBT;
                if (q < nown) {
                    const int y = by[i], x = bx[i];
#pragma unroll
                    for (int f = 0; f < 3; ++f) {
                        const real v = outv[f][i];
                        put(su + f * gg.uplane, gg, y + 4, x, v);
                        if (y < 2) {
                            if (!bottom) {
                                if (!PF_BAND_P2P) put(su_dn + f * gg.uplane, gg, BandGeo::srow(h_dn + y, h_dn, np), x, v);
                                else if (!last)
                                    push(rsu_dn + (uint32_t)(f * gg.uplane * (int)sizeof(real)), rhb_dn + 8u * np, gg,
                                         BandGeo::srow(h_dn + y, h_dn, np), x, v);
                            } else {
                                put(su + f * gg.uplane, gg, BandGeo::srow(-1 - y, h, np), x, v);   // mirror (rho too)
                            }
                        }
                        if (y >= h - 2) {
                            if (!top) {
                                if (!PF_BAND_P2P) put(su_up + f * gg.uplane, gg, BandGeo::srow(y - h, 2, np), x, v);
                                else if (!last)
                                    push(rsu_up + (uint32_t)(f * gg.uplane * (int)sizeof(real)), rhb_up + 8u * np, gg,
                                         BandGeo::srow(y - h, 2, np), x, v);
                            } else if (f != 2) {
                                put(su + f * gg.uplane, gg, BandGeo::srow(2 * h - 1 - y, h, np), x, v);
                            }
                        }
                    }
                }
            }
            if (PF_BAND_P2P) __syncthreads();   // own rows and mirror rows in place
            else cluster.sync();   // every halo row of parity np is in place; every block left phase B
            PF_BAND_STAMP(g, 2);
            par = np;
    };
    for (int64_t s = 0; s < nsteps; ++s) {
        run_stage(k1, 1, s);
        run_stage(k2, 2, s);
    }
    if (PF_BAND_P2P) cluster.sync();   // no block leaves while a neighbour may still address it
    // owned cells back to the state buffer (ghost frame rebuilt by the host)
    real *oc = U + (int64_t)m * L.mstride;
    for (int q = t; q < nown; q += kBT) {
        const int y = q / nx, x = q - y * nx;
        const int64_t o = L.at(y0 + y, x);
        PF_DCHECK(y0 + y >= 0 && y0 + y < L.ny_loc && x >= 0 && x < nx && m < L.m0 + L.members);
        oc[o] = sc[gg.u(y + 4, x)];
        oc[L.fstride + o] = sp[gg.u(y + 4, x)];
        oc[2 * L.fstride + o] = sr[gg.u(y + 4, x)];
    }
}

cudaError_t upload_exp_table_band() {
    static bool done = false;
    if (done) return cudaSuccess;
    double t[64];
    for (int j = 0; j < 64; ++j) t[j] = exp2((double)j / 64.0);
    cudaError_t e = cudaMemcpyToSymbol(kExp2Tab, t, sizeof t);
    if (e == cudaSuccess) done = true;
    return e;
}


template <typename real, int MOB, int FE, int MAXC>
cudaError_t launch_band_c(const Layout &L, const BandPlan &B, const KC<real> &k1, const KC<real> &k2, void *U,
                          const void *vel, int64_t nsteps, cudaStream_t s) {
    auto kern = band_kernel<real, MOB, FE, MAXC>;
    static size_t smem_set = 0;
    if (B.smem > smem_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)B.smem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        smem_set = B.smem;
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)B.bands_per_member;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)B.blocks);
    cfg.blockDim = dim3(kBT);
    cfg.dynamicSmemBytes = B.smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, L, k1, k2, (real *)U, (const real *)vel, B.hmax, nsteps);
}

template <typename real, int MOB, int FE>
cudaError_t launch_band_t(const Layout &L, const BandPlan &B, const Coef &K, void *U, const void *vel, double dt,
                          int64_t nsteps, cudaStream_t s) {
    const KC<real> k1 = make_kc<real>(K, 0.5 * dt), k2 = make_kc<real>(K, dt);
    const int64_t cells = (int64_t)B.hmax * L.nx;
    if (cells <= kBT) return launch_band_c<real, MOB, FE, 1>(L, B, k1, k2, U, vel, nsteps, s);
    if (cells <= 2 * kBT) return launch_band_c<real, MOB, FE, 2>(L, B, k1, k2, U, vel, nsteps, s);
    return launch_band_c<real, MOB, FE, 4>(L, B, k1, k2, U, vel, nsteps, s);
}

}  // namespace

}  // namespace pf
// Diagnostic: the band kernel's phase timeline of its last launch (PF_TRACE builds; zeros
// otherwise): out[16 blocks][128 stages][4] clock64 cycles (see PF_BAND_STAMP).
extern "C" int pf_debug_band_trace(long long *out) {
    return (int)cudaMemcpyFromSymbol(out, pf::g_btrace, sizeof(pf::g_btrace));
}
namespace pf {

bool make_band_plan(int precision, const Layout &L, BandPlan &B) {
    B = BandPlan();
    const size_t esz = precision == 0 ? 8 : 4;
    int dev = 0, maxsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    // one cluster per member, bands of >= 2 rows, at most 16 blocks (non-portable cluster size)
    static const int maxc = getenv("PF_BAND_CLUSTER") ? atoi(getenv("PF_BAND_CLUSTER")) : kMaxCluster;   // A/B knob
    const int cmax = maxc >= 1 && maxc <= kMaxCluster ? maxc : kMaxCluster;
    const int bpm = L.ny_loc / 2 < cmax ? L.ny_loc / 2 : cmax;
    if (bpm < 1) return false;
    const int hmax = (L.ny_loc + bpm - 1) / bpm;
    if ((int64_t)hmax * L.nx > kMaxCells) return false;
    const size_t smem = BandGeo(hmax, L.nx).bytes(esz);
    if ((int)smem > maxsm) return false;
    B.ok = true;
    B.bands_per_member = bpm;
    B.blocks = bpm * L.members;
    B.hmax = hmax;
    B.smem = smem;
    return true;
}

cudaError_t launch_band(int precision, const Layout &L, const BandPlan &B, const Coef &K, void *U, const void *vel,
                        double dt, int64_t nsteps, cudaStream_t s) {
    cudaError_t te = upload_exp_table_band();
    if (te != cudaSuccess) return te;
    if (!B.ok || nsteps < 1) return cudaErrorInvalidValue;
    if (precision == 0) {
        auto f = K.fe == 1 ? (K.mob == 0 ? launch_band_t<double, 0, 1> : K.mob == 1 ? launch_band_t<double, 1, 1>
                                                                                 : launch_band_t<double, 2, 1>)
                           : (K.mob == 0 ? launch_band_t<double, 0, 0> : K.mob == 1 ? launch_band_t<double, 1, 0>
                                                                                 : launch_band_t<double, 2, 0>);
        return f(L, B, K, U, vel, dt, nsteps, s);
    }
    auto f = K.fe == 1 ? (K.mob == 0 ? launch_band_t<float, 0, 1> : K.mob == 1 ? launch_band_t<float, 1, 1>
                                                                           : launch_band_t<float, 2, 1>)
                       : (K.mob == 0 ? launch_band_t<float, 0, 0> : K.mob == 1 ? launch_band_t<float, 1, 0>
                                                                           : launch_band_t<float, 2, 0>);
    return f(L, B, K, U, vel, dt, nsteps, s);
}

}  // namespace pf
