// pf_stream.cuh -- device plumbing shared by the streaming stage kernels (pf_kernels.cu pair / ws
// kernels, pf_split.cu split kernel): mbarriers, 3D TMA tile loads, the strip / row schedule of the
// persistent blocks, the ring geometry, the ghost-frame stores and 128-bit pair loads / stores.
// Internal; included inside namespace pf { namespace { ... } } of each translation unit.
#pragma once
#include <climits>
#ifndef PF_STORE_HINT
#define PF_STORE_HINT 0   // output pair stores: 0 default, 1 streaming (.cs), 2 write-through (.wt)
#endif

// ========================================================================================
// Streaming kernel
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
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp is suspended until the phase completes (or the
// hint elapses) instead of re-issuing the try_wait / branch loop, which took ~40% of the stage
// kernels' issue slots.
#ifndef PF_SUSPEND_NS
#define PF_SUSPEND_NS 1000000
#endif
constexpr uint32_t kSuspendNs = PF_SUSPEND_NS;
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    if (kSuspendNs == 0) {   // plain try_wait loop (A/B knob)
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
            "r"(parity)
            : "memory");
        return;
    }
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(kSuspendNs)
        : "memory");
}
// 3D TMA tile load: box at (x, y, z) of the tensor map -> shared memory, completion on bar.
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
// Programmatic dependent launch: a stage launch may be scheduled while the previous launch on the
// stream drains; griddep_wait() returns once that launch has completed and its writes are visible.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// Work schedule shared by the producer and the compute warps.  Grouped mode (G > 0): blocks come
// in groups of `strips`; block b works on strip b % strips of the row range [T g/G, T (g+1)/G) of
// the concatenated (member, row) space (T = members * ny_loc rows, g = b / strips), so the blocks
// of a group stream the same rows at the same time.  Ungrouped mode (G == 0): block b owns the
// row range [R b/B, R (b+1)/B) of the concatenated (member, strip, row) space.
struct Seg {
    int m, x0, Wp, ya, yb;
};
struct Sched {
    int64_t lo, hi;
    int strip;        // grouped: fixed strip of this block; -1 ungrouped
};
// b / nb: the (virtual) block index and count; blocks b >= nb get an empty range.
__device__ __forceinline__ Sched make_sched(const Layout &L, int Wo, int G, int b, int nb) {
    const int strips = (L.nx + Wo - 1) / Wo;
    const int nyl = L.rows();           // rows of this launch's row window (minus its gap)
    Sched sc;
    if (b >= nb) {
        sc.strip = 0;
        sc.lo = sc.hi = 0;
    } else if (G > 0) {
        const int g = b / strips;
        sc.strip = b - g * strips;
        const int64_t T = (int64_t)L.members * nyl;
        sc.lo = T * g / G;
        sc.hi = T * (g + 1) / G;
    } else {
        const int64_t R = (int64_t)L.members * strips * nyl;
        sc.strip = -1;
        sc.lo = R * b / nb;
        sc.hi = R * (b + 1) / nb;
    }
    return sc;
}
__device__ __forceinline__ Sched make_sched(const Layout &L, int Wo, int G) {
    return make_sched(L, Wo, G, (int)blockIdx.x, (int)gridDim.x);
}
__device__ __forceinline__ bool next_seg(const Layout &L, int Wo, const Sched &sc, int64_t &pos, Seg &sg) {
    if (pos >= sc.hi) return false;
    const int nyl = L.rows(), strips = (L.nx + Wo - 1) / Wo;
    const int64_t col = pos / nyl;      // grouped: member; ungrouped: member * strips + strip
    const int la = (int)(pos - col * nyl);
    int lb = (int)min((int64_t)nyl, (int64_t)la + (sc.hi - pos));
    const int gv = L.g0 - L.r0;         // window rows before the gap: a segment never spans it
    if (la < gv && lb > gv) lb = gv;
    pos += lb - la;
    const int sh = la < gv ? 0 : L.g1 - L.g0;
    sg.ya = L.r0 + la + sh;
    sg.yb = L.r0 + lb + sh;
    int sidx;
    if (sc.strip >= 0) {
        sg.m = (int)col;
        sidx = sc.strip;
    } else {
        sg.m = (int)(col / strips);
        sidx = (int)(col - (int64_t)sg.m * strips);
    }
    sg.m += L.m0;                       // buffer index of the member
    sg.x0 = sidx * Wo;
    sg.Wp = min(Wo, L.nx - sg.x0);
    return true;
}

// Shared-memory geometry of the ring (runtime box width bx).
template <typename real>
struct Ring {
    int bx;            // box width in elements (Wo + 2 HL)
    int in_elems;      // one input box: 3 fields x R rows x bx (rounded to 128 B)
    int slot_elems;    // input box (+ base box for stage 2)
    __host__ __device__ static int round128(int elems) {
        const int b = elems * (int)sizeof(real);
        return ((b + 127) / 128 * 128) / (int)sizeof(real);
    }
    __host__ __device__ Ring(int bx_, int R, bool base) : bx(bx_) {
        in_elems = round128(3 * R * bx);
        slot_elems = in_elems * (base ? 2 : 1);
    }
};

// Warpgroup-packed pair blocks (V > 1): V virtual blocks per CTA, each with its own ring and
// barriers; the exp table once.
template <typename real>
size_t pair_region_bytes(int bx, int R, int S, bool base) {
    Ring<real> rg(bx, R, base);
    return ((size_t)S * rg.slot_elems * sizeof(real) + (size_t)S * 16 + 127) / 128 * 128;
}
template <typename real>
size_t pair_packed_smem_bytes(int bx, int R, int S, bool base, int V) {
    return 128 + 64 * 8 + (size_t)V * pair_region_bytes<real>(bx, R, S, base) + 64 * sizeof(real);
}

template <typename real>
size_t stream_smem_bytes(int bx, int R, int S, bool base) {
    Ring<real> rg(bx, R, base);
    return 128 + (size_t)S * rg.slot_elems * sizeof(real) + 64 * sizeof(real) /* read slack */ +
           (size_t)S * 16 + 64 * 8;   // full, empty barriers; exp table
}

// Store one output value (field f, local row r, column x) and its ghost-frame copies: periodic
// x ghost columns and, at the global y boundaries, the mirror ghost rows (c, phi; rho at the
// bottom; rho's top ghost rows hold the reservoir value and are never overwritten).
template <typename real>
__device__ __forceinline__ void store_row_ghosts(const Layout &L, real *b, int r, int x, real v) {
    PF_DCHECK(r >= -2 && r < L.ny_loc + 2 && x >= 0 && x < L.nx);
    b[L.at(r, x)] = v;
    if (x < L.gx) b[L.at(r, x + L.nx)] = v;
    if (x >= L.nx - L.gx) b[L.at(r, x - L.nx)] = v;
}
template <typename real>
__device__ __forceinline__ void store_with_ghosts(const Layout &L, real *b, int f, int r, int x, real v) {
    const int g = L.y0 + r;
    store_row_ghosts(L, b, r, x, v);
    if (g <= 1) store_row_ghosts(L, b, -1 - r, x, v);                                // y0 == 0 here
    else if (g >= L.ny - 2 && f != 2) store_row_ghosts(L, b, 2 * L.ny_loc - 1 - r, x, v);   // top slab
}

// ----------------------------------------------------------------------------------------
// Pair kernel (default performance path).  Same producer / ring / schedule as stream_kernel, but
// every compute lane owns TWO adjacent columns, so a warp covers 64 columns (60 outputs plus one
// halo column on each side).  Per row and pair of cells a lane issues 128-bit shared loads, 10
// shuffles and 128-bit global stores -- half the per-cell shuffle, load, barrier, loop and store
// instructions of the one-column layout -- and the two columns give the scheduler independent
// fp64 chains.  The per-cell arithmetic is the same pf_cell.cuh code, so results are bitwise
// identical to the tile and stream kernels.
template <typename real> struct Vec2;
template <> struct Vec2<double> { using T = double2; };
template <> struct Vec2<float> { using T = float2; };

template <typename real>
__device__ __forceinline__ typename Vec2<real>::T ld2(const real *p) {
    return *reinterpret_cast<const typename Vec2<real>::T *>(p);
}
template <typename real>
__device__ __forceinline__ void st2(real *p, real x, real y) {
    typename Vec2<real>::T v;
    v.x = x;
    v.y = y;
#if PF_STORE_HINT == 1
    __stcs(reinterpret_cast<typename Vec2<real>::T *>(p), v);   // streaming (evict-first) store
#elif PF_STORE_HINT == 2
    __stwt(reinterpret_cast<typename Vec2<real>::T *>(p), v);   // write-through
#else
    *reinterpret_cast<typename Vec2<real>::T *>(p) = v;
#endif
}

// A lane's two adjacent outputs (columns x, x + 1 of local row r; fields c, phi, rho) and their
// ghost-frame copies (row a1), without divergent scalar paths: the main pairs are stored by every
// lane; the mirror rows at the global y boundaries are a whole-row (warp-uniform) extra store; only
// the lanes whose pair lies in the periodic ghost band (x < gx or x >= nx - gx: both columns,
// gx even) add their ghost-column pair.  Round 1 sent such lanes through per-value scalar
// store_with_ghosts calls, a divergent path every warp of the first and last strip executed on
// every row: those blocks ran ~40% longer than the middle strips (block timeline trace, DESIGN 7).
template <typename real>
__device__ __forceinline__ void store_pair_ghosts(const Layout &L, real *ob, int r, int x, bool xedge, real ocx,
                                                  real ocy, real opx, real opy, real orx, real ory) {
    auto put = [&](int rr, int xc, bool rho) {
        real *q = ob + L.at(rr, xc);
        st2(q, ocx, ocy);
        st2(q + L.fstride, opx, opy);
        if (rho) st2(q + 2 * L.fstride, orx, ory);
    };
    const int g = L.y0 + r;
    const int rm = g <= 1 ? -1 - r : (g >= L.ny - 2 ? 2 * L.ny_loc - 1 - r : INT_MIN);   // mirror row
    put(r, x, true);
    if (rm != INT_MIN) put(rm, x, g <= 1);       // rho: bottom mirror; its top ghost rows keep rho_in
    if (xedge) {
        const int xg = x < L.gx ? x + L.nx : x - L.nx;
        put(r, xg, true);
        if (rm != INT_MIN) put(rm, xg, g <= 1);
    }
}

constexpr int kPairCols = 60;   // output columns per compute warp
constexpr int kPairHalo = 4;    // box columns left of the strip (and right of it)
#ifndef PF_SINGLES_SHFL
#define PF_SINGLES_SHFL 1
#endif
constexpr bool kSinglesShfl = PF_SINGLES_SHFL;
