// Host-side internals shared by the sp200 translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sp200.h"

// A/B-only kernel variants (the first K1 k_sweep1, alternative K2 tile
// configurations behind tuning key 2): compiled only with -DSP200_AB=1
#ifndef SP200_AB
#define SP200_AB 0
#endif

namespace sp200 {

// Per-thread error message + status helpers.
int set_error(int code, const char *fmt, ...);
int check_launch(const char *what);
void count_launch(int n = 1);

// Tuning table (sp_set_tuning).
struct Tuning {
    int64_t zchunk = 0;     // 0 = automatic
    int64_t force_cpasync = 0;
    int64_t cfg_index[SP_MAX_FUSED + 1] = {0, 0, 0, 0, 0};
    int64_t debug = 0;
    int64_t signal_kernels = 0;  // sp_signal / sp_wait through kernels, not stream memory ops
    int64_t two_launch = 0;      // K2 split pass as two launches instead of one split grid
    int64_t balanced_split = 0;  // K2 split pass: full column + equal piece per CTA (A/B)
    int64_t zchunk2 = 0;         // K2 split pass: z-chunk length of the remaining tiles (0 = model)
    int64_t k3_stash = 0;          // 1: K3 at T=4 keeps the band stash + unstash kernels instead of storing in place (A/B)
    int64_t k2_layout = 0;       // K2 two-grid kernel: 0 lane pairs, 1 columns, 2 columns + level-1 shuffles
};
Tuning &tuning();

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// Launchers implemented in sp200_temporal.cu.
int launch_temporal(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
                    int64_t nx, int64_t ny, int64_t nz, int64_t off, int levels, int64_t zlo,
                    int64_t zhi, bool copy_ring, cudaStream_t stream);
int launch_temporal_mirror(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
                           int64_t nx, int64_t ny, int64_t nz, int64_t off, int levels,
                           int64_t zlo, int64_t zhi, double *mirror, int64_t mirror_zshift,
                           cudaStream_t stream);
bool tma_eligible(const void *ptr, int64_t ex, int64_t ey);
int64_t compressed_workspace(int64_t nx, int64_t ny, int64_t depth, int levels);
int64_t compressed_workspace_for(const double *data, int64_t ex, int64_t ey, int64_t nx, int64_t ny,
                                 int64_t depth, int levels);
int launch_compressed(double *data, int64_t ex, int64_t ey, int64_t ez, int64_t nx, int64_t ny,
                      int64_t nz, int64_t src_off, int direction, int levels, int64_t zlo,
                      int64_t zhi, void *ws, int64_t ws_bytes, cudaStream_t stream);
int launch_sweep1(const double *src, double *dst, int64_t ex, int64_t ey, int64_t ez,
                  int64_t nx, int64_t ny, int64_t nz, int64_t off, int64_t zlo, int64_t zhi,
                  bool copy_ring, cudaStream_t stream);

}  // namespace sp200
