// pf_stats.cu -- NEXT-2 of SURVEY 8(f): microstructure statistics of the paper's evaluation
// (section 2.3, section 4.5; readings R-24..R-26 of
// DESIGN.md 11), on the GPU:
//   indicator I = [composite c >= threshold]                                  (R-24)
//   S2(r) = (1/N) sum_x I(x) I(x + r) = IFFT(|FFT(I)|^2) / N^2  (cuFFT, unnormalised inverse)
//   centred map out[ny/2 + dy][nx/2 + dx], radial average over bins round(|r|) (R-25)
//   Rel. L2 of two maps ||a - b|| / ||a||
// The FFTs are cuFFT (a library primitive); indicator, spectrum, shift, binning and the norms are
// this file's kernels.  Binning and norms use fixed-order block reductions (deterministic).
#include <cufft.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "pf.h"

namespace {

__global__ void indicator_kernel(const double *comp, double *ind, int64_t n, double thr) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x)
        ind[q] = comp[q] >= thr ? 1.0 : 0.0;
}

// |Z|^2 in place (imaginary part 0): the spectrum of the autocorrelation.
__global__ void power_kernel(cufftDoubleComplex *z, int64_t n) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const cufftDoubleComplex v = z[q];
        z[q].x = v.x * v.x + v.y * v.y;
        z[q].y = 0.0;
    }
}

// Unnormalised inverse -> S2 (divide by N^2) and fftshift into the centred map.
__global__ void shift_kernel(const double *corr, double *out, int nx, int ny, int batch) {
    const int64_t per = (int64_t)nx * ny, total = per * batch;
    const double inv = 1.0 / ((double)per * (double)per);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = q / per, rem = q - b * per;
        const int y = (int)(rem / nx), x = (int)(rem - (int64_t)y * nx);
        const int sy = (y + ny / 2) % ny, sx = (x + nx / 2) % nx;     // r = (y, x) -> centred slot
        out[b * per + (int64_t)sy * nx + sx] = corr[q] * inv;
    }
}

int bin_of(int y, int x, int nx, int ny) {   // round(|r|) of a centred-map entry (R-25)
    const int dy = y - ny / 2, dx = x - nx / 2;
    return (int)std::floor(std::sqrt((double)(dx * dx + dy * dy)) + 0.5);
}

// One block per (map, bin): fixed-order sum over the bin's entries (cells listed bin by bin in
// `perm`, bin k = perm[off[k] .. off[k+1])), then the mean.
__global__ void radial_kernel(const double *maps, const int *perm, const int *off, double *prof, int64_t per,
                              int nbins) {
    const int bin = blockIdx.x, b = blockIdx.y;
    const double *m = maps + b * per;
    const int lo = off[bin], hi = off[bin + 1];
    double s = 0.0;
    for (int q = lo + (int)threadIdx.x; q < hi; q += blockDim.x) s += m[perm[q]];
    __shared__ double ss[256];
    ss[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) ss[threadIdx.x] += ss[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) prof[(int64_t)b * nbins + bin] = hi > lo ? ss[0] / (double)(hi - lo) : 0.0;
}

// Per map pair: out[b] = ||a - p|| / ||a|| (fixed-order block reduction).
__global__ void rel_l2_kernel(const double *a, const double *p, int64_t per, double *out) {
    const int b = blockIdx.x;
    double d = 0.0, t = 0.0;
    for (int64_t q = threadIdx.x; q < per; q += blockDim.x) {
        const double av = a[b * per + q], dv = av - p[b * per + q];
        d += dv * dv;
        t += av * av;
    }
    __shared__ double sd[256], st[256];
    sd[threadIdx.x] = d;
    st[threadIdx.x] = t;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            sd[threadIdx.x] += sd[threadIdx.x + w];
            st[threadIdx.x] += st[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[b] = sqrt(sd[0]) / sqrt(st[0]);
}

int nblocks(int64_t n) { return (int)((n + 255) / 256 > 8192 ? 8192 : (n + 255) / 256); }

struct Scratch {
    double *comp = nullptr, *ind = nullptr, *corr = nullptr, *maps = nullptr, *prof = nullptr;
    int *perm = nullptr, *off = nullptr;
    cufftDoubleComplex *spec = nullptr;
    cufftHandle fwd = 0, inv = 0;
    bool fwd_ok = false, inv_ok = false;
    ~Scratch() {
        cudaFree(comp); cudaFree(ind); cudaFree(corr); cudaFree(maps); cudaFree(prof); cudaFree(spec);
        cudaFree(perm); cudaFree(off);
        if (fwd_ok) cufftDestroy(fwd);
        if (inv_ok) cufftDestroy(inv);
    }
};

// S2 maps (centred, device) of `batch` composite fields already on the device.
pf_status s2_device(Scratch &w, const double *dcomp, int nx, int ny, int batch, double thr) {
    const int64_t per = (int64_t)nx * ny, n = per * batch, nc = (int64_t)ny * (nx / 2 + 1) * batch;
    if (cudaMalloc(&w.ind, n * 8) != cudaSuccess || cudaMalloc(&w.corr, n * 8) != cudaSuccess ||
        cudaMalloc(&w.maps, n * 8) != cudaSuccess || cudaMalloc(&w.spec, nc * sizeof(cufftDoubleComplex)) != cudaSuccess)
        return PF_ERR_NOMEM;
    int dims[2] = {ny, nx};
    if (cufftPlanMany(&w.fwd, 2, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, batch) != CUFFT_SUCCESS) return PF_ERR_CUDA;
    w.fwd_ok = true;
    if (cufftPlanMany(&w.inv, 2, dims, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, batch) != CUFFT_SUCCESS) return PF_ERR_CUDA;
    w.inv_ok = true;
    indicator_kernel<<<nblocks(n), 256>>>(dcomp, w.ind, n, thr);
    if (cufftExecD2Z(w.fwd, w.ind, w.spec) != CUFFT_SUCCESS) return PF_ERR_CUDA;
    power_kernel<<<nblocks(nc), 256>>>(w.spec, nc);
    if (cufftExecZ2D(w.inv, w.spec, w.corr) != CUFFT_SUCCESS) return PF_ERR_CUDA;
    shift_kernel<<<nblocks(n), 256>>>(w.corr, w.maps, nx, ny, batch);
    return cudaGetLastError() == cudaSuccess ? PF_OK : PF_ERR_CUDA;
}

}  // namespace

extern "C" {

int32_t pf_s2_nbins(int32_t nx, int32_t ny) {
    const double r = std::sqrt((double)(nx / 2) * (nx / 2) + (double)(ny / 2) * (ny / 2));
    return (int32_t)std::floor(r + 0.5) + 1;
}

pf_status pf_s2(const double *comp, int32_t nx, int32_t ny, int32_t batch, double threshold, double *s2,
                double *radial, int32_t nbins) {
    if (!comp || nx < 2 || ny < 2 || batch < 1) return PF_ERR_ARG;
    if (radial && nbins != pf_s2_nbins(nx, ny)) return PF_ERR_ARG;
    const int64_t per = (int64_t)nx * ny, n = per * batch;
    Scratch w;
    if (cudaMalloc(&w.comp, n * 8) != cudaSuccess) return PF_ERR_NOMEM;
    if (cudaMemcpy(w.comp, comp, n * 8, cudaMemcpyHostToDevice) != cudaSuccess) return PF_ERR_CUDA;
    pf_status st = s2_device(w, w.comp, nx, ny, batch, threshold);
    if (st != PF_OK) return st;
    if (radial) {
        // cells grouped by bin (counting sort on the host, row-major order within a bin)
        std::vector<int> cnt(nbins + 1, 0), perm(per);
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) ++cnt[bin_of(y, x, nx, ny) + 1];
        for (int k = 0; k < nbins; ++k) cnt[k + 1] += cnt[k];
        std::vector<int> pos(cnt.begin(), cnt.end() - 1);
        for (int y = 0; y < ny; ++y)
            for (int x = 0; x < nx; ++x) perm[pos[bin_of(y, x, nx, ny)]++] = y * nx + x;
        if (cudaMalloc(&w.prof, (size_t)batch * nbins * 8) != cudaSuccess || cudaMalloc(&w.perm, per * sizeof(int)) != cudaSuccess ||
            cudaMalloc(&w.off, (nbins + 1) * sizeof(int)) != cudaSuccess)
            return PF_ERR_NOMEM;
        if (cudaMemcpy(w.perm, perm.data(), per * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMemcpy(w.off, cnt.data(), (nbins + 1) * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess)
            return PF_ERR_CUDA;
        radial_kernel<<<dim3(nbins, batch), 256>>>(w.maps, w.perm, w.off, w.prof, per, nbins);
        if (cudaMemcpy(radial, w.prof, (size_t)batch * nbins * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return PF_ERR_CUDA;
    }
    if (s2 && cudaMemcpy(s2, w.maps, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return PF_ERR_CUDA;
    return cudaDeviceSynchronize() == cudaSuccess ? PF_OK : PF_ERR_CUDA;
}

pf_status pf_s2_rel_l2(const double *comp_true, const double *comp_pred, int32_t nx, int32_t ny, int32_t batch,
                       double threshold, double *out) {
    if (!comp_true || !comp_pred || !out || nx < 2 || ny < 2 || batch < 1) return PF_ERR_ARG;
    const int64_t per = (int64_t)nx * ny, n = per * batch;
    Scratch a, b;
    if (cudaMalloc(&a.comp, n * 8) != cudaSuccess || cudaMalloc(&b.comp, n * 8) != cudaSuccess) return PF_ERR_NOMEM;
    if (cudaMemcpy(a.comp, comp_true, n * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(b.comp, comp_pred, n * 8, cudaMemcpyHostToDevice) != cudaSuccess)
        return PF_ERR_CUDA;
    pf_status st = s2_device(a, a.comp, nx, ny, batch, threshold);
    if (st == PF_OK) st = s2_device(b, b.comp, nx, ny, batch, threshold);
    if (st != PF_OK) return st;
    if (cudaMalloc(&a.prof, (size_t)batch * 8) != cudaSuccess) return PF_ERR_NOMEM;
    rel_l2_kernel<<<batch, 256>>>(a.maps, b.maps, per, a.prof);
    if (cudaMemcpy(out, a.prof, (size_t)batch * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return PF_ERR_CUDA;
    return cudaDeviceSynchronize() == cudaSuccess ? PF_OK : PF_ERR_CUDA;
}

}  // extern "C"
