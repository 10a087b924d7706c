// pf_halo.cu -- B11: the slab halo exchange as peer stores (halo_transport = 1, include/pf.h).
//
// After a midpoint stage every y-slab owes its neighbours its two boundary rows of c, phi
// and rho (BASELINE configs[3] "2-cell halo exchanged per stage").  Instead of
// NCCL send/recv pairs (ncclGroupStart, 2 x 3 x members sends + receives, each one NCCL kernel and
// its proxy round trip), ONE kernel per slab and stage stores the rows straight into the
// neighbours' ghost rows -- through CUDA-IPC mappings of the neighbours' state buffers over
// NVLink / NVSwitch in the multi-process slab mode, through plain device pointers in the
// single-process loopback mode -- and then bumps an arrival counter that lives in the receiver's
// memory.  The receiver's stream waits for the counter with a stream memory operation
// (cuStreamWaitValue32, GEQ): no kernel spins on a flag, so a persistent stage kernel that holds
// every SM can never starve the push it waits for.
//
// Layout: [member][field][storage row = row + 2][pitch]; the two rows of one
// (member, field) are 2 * rowb contiguous bytes, and member m field f starts at (3m + f) * fstride.
//   down (dir 0): my rows [0, 2)           -> the slab below's ghost rows [rows, rows + 2)
//   up   (dir 1): my rows [rows - 2, rows) -> the slab above's ghost rows [-2, 0)
// Every slab has the same `rows` (ny % nranks == 0), so both sides agree on every offset.
//
// Ordering (why the counter is enough):
//   * data before counter: each thread fences at system scope after its stores, the block
//     barrier orders all of them before thread 0's system-scope atomic add;
//   * no write-after-read on the ghost rows: a slab reads the ghost rows of buffer B only in the
//     boundary-band launches of the stage that reads B, and its neighbour pushes into B's ghost
//     rows again only after it has waited for this slab's NEXT push, which this slab issues after
//     those band launches (pf_host.cpp one_step).
#include <cuda_runtime.h>

#include "pf_internal.h"

namespace pf {

namespace {

template <typename V>
__global__ void __launch_bounds__(256) halo_push_kernel(HaloPush h) {
    const int dir = blockIdx.y;
    char *dst = h.dst[dir];
    if (dst == nullptr) return;
    const int64_t per = 2 * h.rowb / (int64_t)sizeof(V);   // vectors per (member, field) chunk
    const int64_t total = per * h.nchunks;
    const int64_t src_row = dir == 0 ? 2 : h.rows;           // storage row of the first sent row
    const int64_t dst_row = dir == 0 ? h.rows + 2 : 0;       // storage row of the first ghost row
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i / per, j = i - k * per;
        const int64_t off = k * h.fstride_b;
        const V v = reinterpret_cast<const V *>(h.src + off + src_row * h.rowb)[j];
        reinterpret_cast<V *>(dst + off + dst_row * h.rowb)[j] = v;
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd_system(h.flag[dir], 1u);
}

}  // namespace

int halo_push_blocks(int members, int64_t rowb) {
    const int64_t bytes = 2 * rowb * 3 * (int64_t)members;   // per direction
    const int64_t b = (bytes + 256 * 16 * 4 - 1) / (256 * 16 * 4);   // ~4 16-byte vectors per thread
    return (int)(b < 1 ? 1 : b > 148 ? 148 : b);
}

cudaError_t launch_halo_push(const HaloPush &h, cudaStream_t s) {
    if (h.dst[0] == nullptr && h.dst[1] == nullptr) return cudaSuccess;
    const dim3 grid(halo_push_blocks(h.nchunks / 3, h.rowb), 2);
    if (h.rowb % 16 == 0)
        halo_push_kernel<uint4><<<grid, 256, 0, s>>>(h);
    else if (h.rowb % 8 == 0)
        halo_push_kernel<uint2><<<grid, 256, 0, s>>>(h);
    else
        halo_push_kernel<unsigned><<<grid, 256, 0, s>>>(h);
    return cudaGetLastError();
}

}  // namespace pf
