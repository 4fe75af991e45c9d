// Opt-in velocity post-pass of Position Based Fluids (Macklin & Mueller
// 2013, eqs. 15-17): vorticity confinement and XSPH viscosity, run after each
// substep's finalize.  The reference has neither, so
// they are OFF by default (xsph_c = vorticity_eps = 0 leaves every frame
// bit-identical to the reference) and sit outside the parity contract; the
// tests check them against an independent float64 implementation of the
// paper's equations and against analytic fields (rigid rotation: omega =
// +2 Omega z).
//
// gradW(x_i - x_j) below is the spiky gradient with respect to x_i
// (spiky_grad).  Eq. 15 differentiates with respect to p_j, which is its
// negative, so the SPH curl estimate reads
//   omega_i = sum_j (v_i - v_j) x gradW(x_i - x_j)                 (eq. 15)
//   eta_i   = sum_j (|omega_j| - |omega_i|) gradW(x_i - x_j)      (grad |omega|)
//   N_i     = eta_i / |eta_i|  (0 when eta_i = 0)
//   v_i    += dt * eps * (N_i x omega_i)                          (eq. 16)
//   v_i    += c * sum_j (v_j - v_i) W(x_i - x_j)                  (eq. 17, XSPH)
//
// over the substep's frozen lists at the finalized positions, Jacobi-style
// (every sum reads the velocities finalize produced), then the speed cap.
#pragma once

#include "apbf_kernels.cuh"

namespace apbf_gpu {

// Pass 1: omega_i (float4: xyz, |omega| in .w) and the XSPH-corrected
// velocity into Vx, for every order position.
__global__ void k_post_omega(int n, const Ctl* ctl, const int* __restrict__ order,
                             const float4* __restrict__ X, const float4* __restrict__ V,
                             const int* __restrict__ nbr, const int* __restrict__ nbrCount,
                             const long long* __restrict__ groupBase, KernelConsts kc, float xsph_c,
                             float4* __restrict__ Om, float4* __restrict__ Vx) {
    if (ctl->abort) return;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int i = order[k];
    const float4 xi = X[i], vi = V[i];
    const int cnt = nbrCount[k];
    const int* lst = list_lane(nbr, groupBase[k >> 5], k & 31);
    float ox = 0.f, oy = 0.f, oz = 0.f, sx = 0.f, sy = 0.f, sz = 0.f;
    for (int e = 0; e < cnt; ++e) {
        const int j = list_at(lst, e);
        if (j == i) continue;
        const float4 xj = X[j], vj = V[j];
        const float rx = xi.x - xj.x, ry = xi.y - xj.y, rz = xi.z - xj.z;
        const float r2 = sqn3(rx, ry, rz);
        float gx, gy, gz;
        spiky_grad(kc, r2, rx, ry, rz, gx, gy, gz);
        const float ux = vj.x - vi.x, uy = vj.y - vi.y, uz = vj.z - vi.z;
        // (v_i - v_j) x g = -(u x g) = g x u
        ox += gy * uz - gz * uy;
        oy += gz * ux - gx * uz;
        oz += gx * uy - gy * ux;
        const float w = poly6_r2(kc, r2);
        sx += ux * w;
        sy += uy * w;
        sz += uz * w;
    }
    Om[i] = make_float4(ox, oy, oz, sqrtf(sqn3(ox, oy, oz)));
    Vx[i] = make_float4(vi.x + xsph_c * sx, vi.y + xsph_c * sy, vi.z + xsph_c * sz, 0.f);
}

// Pass 2: eta_i, N_i and the confinement impulse; v = Vx + dt eps (N x omega),
// then the speed cap (solver.hpp:350-353) so the reference's invariant holds.
__global__ void k_post_apply(int n, Ctl* ctl, const int* __restrict__ order, const float4* __restrict__ X,
                             const float4* __restrict__ Om, const float4* __restrict__ Vx,
                             const int* __restrict__ nbr, const int* __restrict__ nbrCount,
                             const long long* __restrict__ groupBase, KernelConsts kc, float dt, float eps,
                             float cap, float4* __restrict__ V) {
    if (ctl->abort) return;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int i = order[k];
    const float4 xi = X[i], oi = Om[i];
    const int cnt = nbrCount[k];
    const int* lst = list_lane(nbr, groupBase[k >> 5], k & 31);
    float ex = 0.f, ey = 0.f, ez = 0.f;
    if (eps != 0.0f) {
        for (int e = 0; e < cnt; ++e) {
            const int j = list_at(lst, e);
            if (j == i) continue;
            const float4 xj = X[j];
            const float rx = xi.x - xj.x, ry = xi.y - xj.y, rz = xi.z - xj.z;
            float gx, gy, gz;
            spiky_grad(kc, sqn3(rx, ry, rz), rx, ry, rz, gx, gy, gz);
            const float d = Om[j].w - oi.w;
            ex += d * gx;
            ey += d * gy;
            ez += d * gz;
        }
    }
    float4 v = Vx[i];
    const float en = sqrtf(sqn3(ex, ey, ez));
    if (en > 0.0f) {
        const float nx = ex / en, ny = ey / en, nz = ez / en;
        v.x += dt * eps * (ny * oi.z - nz * oi.y);
        v.y += dt * eps * (nz * oi.x - nx * oi.z);
        v.z += dt * eps * (nx * oi.y - ny * oi.x);
    }
    const float s = sqrtf(sqn3(v.x, v.y, v.z));
    if (s > cap) {
        const float f = cap / s;
        v.x *= f;
        v.y *= f;
        v.z *= f;
    }
    V[i] = make_float4(v.x, v.y, v.z, 0.f);
}

}  // namespace apbf_gpu
