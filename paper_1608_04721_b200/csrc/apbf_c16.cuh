// Solver passes over the compact 16-bit frozen lists (c16_decode, built by
// k_build_lists<true>).  Per pair they stream 2 bytes of list instead of 4
// bytes of list plus 4 bytes of cached coefficient, so lists (~60 MB at 1M
// particles) and the gathered particle arrays stay resident in the 126 MB L2
// across the iterations of a substep; delta-p recomputes the spiky
// coefficient with the same exact fast sqrt/division as the lambda pass.
//
// Bit-identical to k_lambda / k_deltap_apply (and so to computeLambda /
// computeDeltaP, solver.hpp:98-141): same per-pair arithmetic, same list
// order, same exact-IEEE redo whenever a pair leaves the fast-path range.
#pragma once

#include "apbf_kernels.cuh"

namespace apbf_gpu {

// computeLambda over compact lists; also publishes PL (see k_lambda).
// kCoef: also cache each pair's coefficient for delta-p (as k_lambda).
template <int kBT, int kK, bool kZero, bool kCoef>
__global__ void __launch_bounds__(kBT) k_lambda_c16(
    int n, int iter, Ctl* ctl, const int* __restrict__ activeCount, const int* __restrict__ order,
    const float4* __restrict__ P, const float* __restrict__ W, float* __restrict__ L,
    const unsigned short* __restrict__ nbr16, const int4* __restrict__ lbase,
    const long long* __restrict__ groupBase, SolverConsts sc, int substep, int ownB, int ownE,
    float4* __restrict__ PL, float* __restrict__ coef) {
    if (ctl->abort) return;
    const int active = activeCount[iter];
    const int upto = activeCount[iter - 1];
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if ((k & ~31) >= upto) return;  // whole warp idle
    bool bad = false;
    int i = 0;
    if (k >= active && k < upto) {  // finished after the previous iteration
        const int f = order[k];
        const float4 q = P[f];
        PL[f] = make_float4(q.x, q.y, q.z, kZero ? 0.0f : L[f]);
    }
    if (k < active) {
        const int4 lb = lbase[k];
        const int cnt = lb.w;
        const long long lbo = groupBase[k >> 5] + (k & 31);
        const unsigned short* lst = nbr16 + lbo;
        float* cf = coef + lbo;
        i = order[k];
        const float4 xi = P[i];
        float rho = 0.f, gxs = 0.f, gys = 0.f, gzs = 0.f, denomJ = 0.f;
        bool slow = !sc.fastDiv;
        auto pair = [&](int j, const float4& pj, float wj, int e) {
            const float rx = xi.x - pj.x, ry = xi.y - pj.y, rz = xi.z - pj.z;
            const float r2 = sqn3(rx, ry, rz);
            rho += pj.w * poly6_r2(sc.kc, r2);
            const float c = spiky_coef_fast(sc.kc, r2, slow);
            if (kCoef) __stcg(cf + e * 32, c);
            const float gx = c * rx;  // may be -0 for a zero-gradient pair:
            const float gy = c * ry;  // the sums below start at +0 and are
            const float gz = c * rz;  // never -0, so adding it is exact
            gxs += gx;
            gys += gy;
            gzs += gz;
            const float dj = wj * sqn3(gx, gy, gz);
            denomJ += (j == i) ? 0.0f : dj;
        };
        int e0 = 0;
        for (; e0 + kK <= cnt; e0 += kK) {
            int jj[kK];
            float4 pp[kK];
            float ww[kK];
#pragma unroll
            for (int q = 0; q < kK; ++q) jj[q] = c16_decode(lst[(e0 + q) * 32], lb);
#pragma unroll
            for (int q = 0; q < kK; ++q) {
                pp[q] = __ldg(P + jj[q]);
                ww[q] = __ldg(W + jj[q]);
            }
#pragma unroll
            for (int q = 0; q < kK; ++q) pair(jj[q], pp[q], ww[q], e0 + q);
        }
        if (e0 < cnt) {
            int jj[kK];
            float4 pp[kK];
            float ww[kK];
#pragma unroll
            for (int q = 0; q < kK; ++q) jj[q] = (e0 + q < cnt) ? c16_decode(lst[(e0 + q) * 32], lb) : i;
#pragma unroll
            for (int q = 0; q < kK; ++q) {
                pp[q] = __ldg(P + jj[q]);
                ww[q] = __ldg(W + jj[q]);
            }
#pragma unroll
            for (int q = 0; q < kK; ++q)
                if (e0 + q < cnt) pair(jj[q], pp[q], ww[q], e0 + q);
        }
        if (slow) {  // exact IEEE redo of the whole sweep (practically never)
            rho = gxs = gys = gzs = denomJ = 0.f;
            for (int e = 0; e < cnt; ++e) {
                const int j = c16_decode(lst[e * 32], lb);
                const float4 pj = P[j];
                const float rx = xi.x - pj.x, ry = xi.y - pj.y, rz = xi.z - pj.z;
                const float r2 = sqn3(rx, ry, rz);
                rho += pj.w * poly6_r2(sc.kc, r2);
                if (kCoef) {
                    const float rn = sqrtf(r2);
                    const float a = sc.kc.h - rn;
                    const float cc = sc.kc.spiky * a * a / rn;
                    cf[e * 32] = (rn >= sc.kc.h || rn == 0.0f) ? 0.0f : cc;
                }
                if (j != i) {
                    float gx, gy, gz;
                    spiky_grad(sc.kc, r2, rx, ry, rz, gx, gy, gz);
                    gxs += gx;
                    gys += gy;
                    gzs += gz;
                    denomJ += W[j] * sqn3(gx, gy, gz);
                }
            }
        }
        const float c = rho * sc.invRho0 - 1.0f;
        const float sx = sc.invRho0 * gxs, sy = sc.invRho0 * gys, sz = sc.invRho0 * gzs;
        const float denom = W[i] * sqn3(sx, sy, sz) + sc.invRho0sq * denomJ + sc.eps;
        const float lam = -c / denom;
        L[i] = lam;
        PL[i] = make_float4(xi.x, xi.y, xi.z, lam);
        bad = !isfinite(lam) && i >= ownB && i < ownE;
    }
    report_bad(ctl, kPassLambda, bad, i - ownB);
    if (bad) {
        ctl->bad_substep[kPassLambda] = substep;
        ctl->bad_iter[kPassLambda] = iter;
    }
}

// computeDeltaP + apply with SDF projection over compact lists (see
// k_deltap_apply); neighbours gathered from PL = (x*, lambda).
// kCoef: gradients from the lambda pass's cached coefficients.
template <int kBT, int kK, bool kCoef>
__global__ void __launch_bounds__(kBT) k_deltap_c16(
    int n, int iter, Ctl* ctl, const int* __restrict__ activeCount, const int* __restrict__ order,
    const float4* __restrict__ Pc, float4* __restrict__ Pn, const float* __restrict__ W,
    const float* __restrict__ L, const unsigned short* __restrict__ nbr16,
    const int4* __restrict__ lbase, const long long* __restrict__ groupBase,
    const Scene* __restrict__ scene, SolverConsts sc, int substep, int ownB, int ownE,
    const float4* __restrict__ PL, const float* __restrict__ coef) {
    if (ctl->abort) return;
    const int active = activeCount[iter];
    const int upto = activeCount[iter - 1];
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if ((k & ~31) >= upto) return;  // whole warp idle
    bool bad = false;
    int i = 0;
    if (k < active && order[k] >= ownB && order[k] < ownE) {
        const int4 lb = lbase[k];
        const int cnt = lb.w;
        const long long lbo = groupBase[k >> 5] + (k & 31);
        const unsigned short* lst = nbr16 + lbo;
        const float* cf = coef + lbo;
        i = order[k];
        const float4 xi = Pc[i];
        const float lamI = L[i];
        float sx = 0.f, sy = 0.f, sz = 0.f;
        bool slow = !kCoef && !sc.fastDiv;
        // one term of computeDeltaP (solver.hpp:131-139), in list order
        auto term = [&](int j, const float4& pj, float cc) {
            const float rx = xi.x - pj.x, ry = xi.y - pj.y, rz = xi.z - pj.z;
            const float c = kCoef ? cc : spiky_coef_fast(sc.kc, sqn3(rx, ry, rz), slow);
            const float s = (j == i) ? 0.0f : lamI + pj.w;  // self: 0 * (+0) adds +0
            sx += s * (c * rx);
            sy += s * (c * ry);
            sz += s * (c * rz);
        };
        int e0 = 0;
        for (; e0 + kK <= cnt; e0 += kK) {
            int jj[kK];
            float4 pp[kK];
#pragma unroll
            for (int q = 0; q < kK; ++q) jj[q] = c16_decode(lst[(e0 + q) * 32], lb);
            float cc[kK];
#pragma unroll
            for (int q = 0; q < kK; ++q) {
                pp[q] = __ldg(PL + jj[q]);
                cc[q] = kCoef ? __ldcg(cf + (e0 + q) * 32) : 0.0f;
            }
#pragma unroll
            for (int q = 0; q < kK; ++q) term(jj[q], pp[q], cc[q]);
        }
        if (e0 < cnt) {
            int jj[kK];
            float4 pp[kK];
#pragma unroll
            for (int q = 0; q < kK; ++q) jj[q] = (e0 + q < cnt) ? c16_decode(lst[(e0 + q) * 32], lb) : i;
            float cc[kK];
#pragma unroll
            for (int q = 0; q < kK; ++q) {
                pp[q] = __ldg(PL + jj[q]);
                cc[q] = (kCoef && e0 + q < cnt) ? __ldcg(cf + (e0 + q) * 32) : 0.0f;
            }
#pragma unroll
            for (int q = 0; q < kK; ++q)
                if (e0 + q < cnt) term(jj[q], pp[q], cc[q]);
        }
        if (slow) {  // exact IEEE redo (practically never)
            sx = sy = sz = 0.f;
            for (int e = 0; e < cnt; ++e) {
                const int j = c16_decode(lst[e * 32], lb);
                if (j == i) continue;
                const float4 pj = PL[j];
                const float rx = xi.x - pj.x, ry = xi.y - pj.y, rz = xi.z - pj.z;
                float gx, gy, gz;
                spiky_grad(sc.kc, sqn3(rx, ry, rz), rx, ry, rz, gx, gy, gz);
                const float s = lamI + pj.w;
                sx += s * gx;
                sy += s * gy;
                sz += s * gz;
            }
        }
        const float kk = W[i] / sc.rho0;
        float px = xi.x + kk * sx;
        float py = xi.y + kk * sy;
        float pz = xi.z + kk * sz;
        if (scene->n > 0) {
            float gx, gy, gz;
            const float phi = scene_distance(*scene, px, py, pz, gx, gy, gz);
            if (phi < sc.radius) {
                const float d = sc.radius - phi;
                px += d * gx;
                py += d * gy;
                pz += d * gz;
            }
        }
        Pn[i] = make_float4(px, py, pz, xi.w);
        bad = !finite3(px, py, pz);
    } else if (k >= active && k < upto) {  // finished: carry x* into Pn
        const int f = order[k];
        if (f >= ownB && f < ownE) Pn[f] = Pc[f];
    }
    report_bad(ctl, kPassApply, bad, i - ownB);
    if (bad) {
        ctl->bad_substep[kPassApply] = substep;
        ctl->bad_iter[kPassApply] = iter;
    }
}

}  // namespace apbf_gpu
