// step.cu -- one forward-Euler time step of the vortex particle method (section 2):
//   dx_i/dt = u_i                   convection, Eq. (7)
//   dgamma_i/dt = (Eq. 8)           stretching
//   d sigma^2/dt = 2 nu             diffusion by core spreading, Eq. (9)
// "the updates happen simultaneously" with forward Euler, here on
// the device: one fused elementwise kernel after the evaluation; the core size is uniform
// (reading R4), so sigma^2 += 2 nu dt is a host-side parameter update for the next step.
#include <cuda_runtime.h>

#include "vfmm_internal.h"

namespace vfmm {

namespace {

// x += u dt wrapped into [lo, lo + len) (periodic box; a value that rounds onto the upper face
// is mapped to lo, keeping the half-open box), gamma += dgamma dt
__global__ void euler_update_kernel(float* __restrict__ pos, float* __restrict__ gam,
                                    const float* __restrict__ vel,
                                    const float* __restrict__ dgam, int64_t n, float dt, float lo,
                                    float len, int periodic) {
    const float hi = lo + len;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < 3 * n;
         i += (int64_t)gridDim.x * blockDim.x) {
        float x = fmaf(vel[i], dt, pos[i]);
        if (periodic) {
            if (x >= hi || x < lo) x -= len * floorf((x - lo) / len);
            if (x >= hi) x = lo;
            if (x < lo) x = lo;
        }
        pos[i] = x;
        gam[i] = fmaf(dgam[i], dt, gam[i]);
    }
}

}  // namespace

void launch_euler_update(float* pos, float* gamma, const float* vel, const float* dgamma,
                         int64_t n, float dt, float lo, float len, int periodic, cudaStream_t st) {
    int64_t g = (3 * n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    if (g < 1) g = 1;
    euler_update_kernel<<<(unsigned)g, 256, 0, st>>>(pos, gamma, vel, dgamma, n, dt, lo, len,
                                                     periodic);
}

}  // namespace vfmm
