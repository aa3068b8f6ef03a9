// Halo box pack / unpack (general Cartesian topologies).
//
// The reference exchanges every message as a NumPy slice copy of a strided
// box (exchange_multilayer_halos, sp/halo.py:239-271; boxes from
// build_halo_plan, sp/halo.py:194-229).  z-slab messages are whole storage
// planes and move without packing; x and y messages (and z messages of
// topologies with px or py > 1) are strided sub-boxes.  One launch packs all
// send boxes of an axis phase into their contiguous buffers, one launch
// unpacks all receive buffers into their boxes: both sides of a phase, no
// per-message launches, no torch copies.
#include "sp200_device.cuh"
#include "sp200_internal.h"

namespace sp200 {

struct BoxSet {
    sp_box_t b[SP_MAX_BOXES];
    int64_t start[SP_MAX_BOXES + 1];  // element prefix sums over the boxes
    int n;
    int64_t ex, ey;
};

// flat element index over the concatenated boxes -> (box, z, y, x); the x run
// of a row is contiguous in both the grid and the buffer
template <bool PACK>
__global__ void k_boxes(double *grid, BoxSet s) {
    const int64_t total = s.start[s.n];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        int k = 0;
        while (k + 1 < s.n && e >= s.start[k + 1]) ++k;
        const sp_box_t &b = s.b[k];
        const int64_t w = b.x1 - b.x0, hgt = b.y1 - b.y0;
        const int64_t l = e - s.start[k];
        const int64_t row = l / w, x = l - row * w;
        const int64_t z = row / hgt, y = row - z * hgt;
        const int64_t g = ((b.z0 + z) * s.ey + (b.y0 + y)) * s.ex + (b.x0 + x);
        if (PACK) b.buf[l] = grid[g];
        else grid[g] = b.buf[l];
    }
}

static int run_boxes(bool pack, double *grid, int64_t ex, int64_t ey, int64_t ez, int nbox,
                     const sp_box_t *boxes, void *stream) {
    if (!grid || (nbox > 0 && !boxes)) return set_error(SP_EINVAL, "null argument");
    if (nbox < 0 || nbox > SP_MAX_BOXES)
        return set_error(SP_EINVAL, "%d boxes outside [0, %d]", nbox, SP_MAX_BOXES);
    BoxSet s;
    s.n = nbox;
    s.ex = ex;
    s.ey = ey;
    s.start[0] = 0;
    for (int k = 0; k < nbox; ++k) {
        const sp_box_t &b = boxes[k];
        if (!b.buf) return set_error(SP_EINVAL, "box %d: null buffer", k);
        if (b.x0 < 0 || b.y0 < 0 || b.z0 < 0 || b.x1 > ex || b.y1 > ey || b.z1 > ez ||
            b.x0 > b.x1 || b.y0 > b.y1 || b.z0 > b.z1)
            return set_error(SP_EINVAL, "box %d [%lld,%lld)x[%lld,%lld)x[%lld,%lld) outside storage", k,
                             (long long)b.x0, (long long)b.x1, (long long)b.y0, (long long)b.y1,
                             (long long)b.z0, (long long)b.z1);
        s.b[k] = b;
        s.start[k + 1] = s.start[k] + (b.x1 - b.x0) * (b.y1 - b.y0) * (b.z1 - b.z0);
    }
    // empty boxes contribute no elements; skip them in the search by keeping
    // their prefix equal (the while loop steps over them)
    const int64_t total = s.start[nbox];
    if (total == 0) return SP_OK;
    int64_t blocks = (total + 255) / 256;
    const int64_t cap = (int64_t)sm_count() * 16;
    if (blocks > cap) blocks = cap;
    if (pack) k_boxes<true><<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(grid, s);
    else k_boxes<false><<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(grid, s);
    count_launch();
    return check_launch(pack ? "sp_pack_boxes" : "sp_unpack_boxes");
}

}  // namespace sp200

using namespace sp200;

extern "C" {

int sp_pack_boxes(const double *grid, int64_t ex, int64_t ey, int64_t ez, int nbox,
                  const sp_box_t *boxes, void *stream) {
    return run_boxes(true, const_cast<double *>(grid), ex, ey, ez, nbox, boxes, stream);
}

int sp_unpack_boxes(double *grid, int64_t ex, int64_t ey, int64_t ez, int nbox,
                    const sp_box_t *boxes, void *stream) {
    return run_boxes(false, grid, ex, ey, ez, nbox, boxes, stream);
}

}  // extern "C"
