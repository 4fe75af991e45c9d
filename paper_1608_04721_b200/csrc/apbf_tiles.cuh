// apbf_tiles.cuh -- cell-tile solver passes.
//
// A tile is kTileP consecutive cell-sorted slots and runs as one CTA.  Its
// candidate set is the union of its particles' 9 x-row runs
// (uniform_grid.hpp:147-157): a short list of disjoint, ascending slot
// intervals fixed at list-build time.  Every frozen list (uniform_grid.hpp:
// 179-213) is stored as u16 indices into that candidate array -- ascending
// candidate index == ascending slot, so every per-particle sum keeps the
// reference's order.  Each solver pass stages the candidates' x*, mass and
// invMass (lambda pass) or x* and lambda (delta-p pass) in shared memory
// once per tile and all neighbour gathers are shared-memory loads.
//
// Tiles whose candidate set exceeds kCandMax or kMaxRuns (pathological
// clumping) keep int32 slot lists and gather from global memory.
#pragma once

#include "apbf_kernels.cuh"

namespace apbf_gpu {

constexpr int kTileP = 128;    // particles per tile = threads per CTA
constexpr int kMaxRuns = 32;   // merged candidate intervals per tile
constexpr int kCandMax = 2048; // staged candidates per tile
constexpr int kMaxHome = 12;   // distinct home rows per tile

struct TileInfo {
    int nRuns;          // merged candidate runs
    int C;              // candidates, -1 = fallback tile (int32 slot lists)
    unsigned listBase;  // first list element (u16 units, or int32 units for fallback)
    int cap;            // padded per-particle list stride (multiple of 8)
};

// Candidate index of slot s inside the tile's merged runs (s must be inside).
__device__ __forceinline__ int cand_of(const int2* runs, int nRuns, int s) {
    int lo = 0, hi = nRuns - 1;
    while (lo < hi) {  // last run with start <= s
        const int mid = (lo + hi + 1) >> 1;
        if (runs[mid].x <= s) lo = mid;
        else hi = mid - 1;
    }
    return runs[lo].y + (s - runs[lo].x);
}

// Slot of candidate c (c < C).  runOff holds the candidate offsets.
__device__ __forceinline__ int slot_of(const int2* runs, int nRuns, int c) {
    int lo = 0, hi = nRuns - 1;
    while (lo < hi) {  // last run with off <= c
        const int mid = (lo + hi + 1) >> 1;
        if (runs[mid].y <= c) lo = mid;
        else hi = mid - 1;
    }
    return runs[lo].x + (c - runs[lo].y);
}

// ---------------------------------------------------------- list build

// One CTA per tile: candidate runs, per-particle frozen lists (u16 candidate
// indices, padded [particle][entry] slab), tile max level.
__global__ void __launch_bounds__(kTileP) k_tile_build(
    int n, Ctl* ctl, const float4* __restrict__ P, const int* __restrict__ cellStart,
    const int* __restrict__ LV, float h, float h2, TileInfo* __restrict__ info,
    int2* __restrict__ runsOut, int* __restrict__ tileMax, unsigned short* __restrict__ lists,
    long long listCap, int* __restrict__ fbLists, long long fbCap, int* __restrict__ nbrCount) {
    if (ctl->abort) return;
    __shared__ int s_row[kTileP], s_cx[kTileP];
    __shared__ int2 s_runs[kMaxRuns];
    __shared__ int s_nRuns, s_C, s_fallback, s_cap;
    __shared__ unsigned s_base;
    __shared__ int s_max[kTileP / 32], s_cmax[kTileP / 32];
    const int t = blockIdx.x, p = threadIdx.x;
    const int i = t * kTileP + p;
    const bool valid = i < n;
    const GridDev& G = ctl->grid[0];
    const int dx = G.dims[0], dy = G.dims[1], dz = G.dims[2];
    float qx = 0.f, qy = 0.f, qz = 0.f;
    int c[3] = {0, 0, 0};
    bool degenerate = false;
    if (valid) {
        const float4 q = P[i];
        qx = q.x;
        qy = q.y;
        qz = q.z;
        const float pp[3] = {qx, qy, qz};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int v = f2i_trunc(floorf((pp[a] - G.origin[a]) / h));
            c[a] = v;
            // query coordinates equal the binning ones for every finite cloud
            // (origin = min - h, dims from max + h); anything else takes the
            // generic path below
            if (v < 0 || v > G.dims[a] - 1) degenerate = true;
        }
        s_row[p] = c[2] * dy + c[1];
        s_cx[p] = c[0];
    } else {
        s_row[p] = -1;
        s_cx[p] = 0;
    }
    const int anyDegenerate = __syncthreads_or(degenerate);
    // tile max level (for skipping inactive tiles per iteration)
    int lv = valid ? LV[i] : 0;
    lv = warp_max_i(lv);
    if ((p & 31) == 0) s_max[p >> 5] = lv;
    if (p == 0) {
        s_fallback = anyDegenerate;
        // home rows in slot order: particles are sorted by (row, cx)
        int hRow[kMaxHome], hX0[kMaxHome], hX1[kMaxHome], H = 0;
        for (int q = 0; q < kTileP && !s_fallback; ++q) {
            const int r = s_row[q];
            if (r < 0) break;
            if (H == 0 || hRow[H - 1] != r) {
                if (H == kMaxHome) {
                    s_fallback = 1;
                    break;
                }
                hRow[H] = r;
                hX0[H] = s_cx[q];
                hX1[H] = s_cx[q];
                ++H;
            } else {
                hX1[H - 1] = s_cx[q];
            }
        }
        // candidate rows with merged x-ranges, sorted by (row, x0)
        int eRow[kMaxHome * 9], eX0[kMaxHome * 9], eX1[kMaxHome * 9], E = 0;
        for (int h = 0; h < H && !s_fallback; ++h) {
            const int cz = hRow[h] / dy, cy = hRow[h] - cz * dy;
            const int x0 = imax_std(hX0[h] - 1, 0), x1 = imin_std(hX1[h] + 1, dx - 1);
            for (int z = imax_std(cz - 1, 0); z <= imin_std(cz + 1, dz - 1); ++z)
                for (int y = imax_std(cy - 1, 0); y <= imin_std(cy + 1, dy - 1); ++y) {
                    const int r = z * dy + y;
                    // insertion keeping (row, x0) order, merging overlaps/adjacency
                    int pos = E;
                    while (pos > 0 && (eRow[pos - 1] > r || (eRow[pos - 1] == r && eX0[pos - 1] > x0))) --pos;
                    for (int m = E; m > pos; --m) {
                        eRow[m] = eRow[m - 1];
                        eX0[m] = eX0[m - 1];
                        eX1[m] = eX1[m - 1];
                    }
                    eRow[pos] = r;
                    eX0[pos] = x0;
                    eX1[pos] = x1;
                    ++E;
                }
        }
        // merge pass
        int M = 0;
        for (int e = 0; e < E; ++e) {
            if (M > 0 && eRow[M - 1] == eRow[e] && eX0[e] <= eX1[M - 1] + 1) {
                eX1[M - 1] = imax_std(eX1[M - 1], eX1[e]);
            } else {
                eRow[M] = eRow[e];
                eX0[M] = eX0[e];
                eX1[M] = eX1[e];
                ++M;
            }
        }
        int nR = 0, C = 0;
        for (int e = 0; e < M && !s_fallback; ++e) {
            const long long rb = (long long)eRow[e] * dx;
            const int b = cellStart[rb + eX0[e]], en = cellStart[rb + eX1[e] + 1];
            if (en <= b) continue;
            if (nR == kMaxRuns) {
                s_fallback = 1;
                break;
            }
            s_runs[nR] = make_int2(b, C);
            ++nR;
            C += en - b;
        }
        if (C > kCandMax) s_fallback = 1;
        s_nRuns = s_fallback ? 0 : nR;
        s_C = s_fallback ? -1 : C;
    }
    __syncthreads();
    if (p == 0) {
        int m = s_max[0];
        for (int w = 1; w < kTileP / 32; ++w) m = imax_std(m, s_max[w]);
        tileMax[t] = m;
    }
    const bool fb = s_fallback != 0;
    const int nRuns = s_nRuns;
    // the particle's own 9 runs (uniform_grid.hpp:135-158)
    int lo[3] = {0, 0, 0}, hi[3] = {-1, -1, -1};
    bool any = false;
    if (valid) {
        any = true;
        const float pp[3] = {qx, qy, qz};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int cc = f2i_trunc(floorf((pp[a] - G.origin[a]) / h));
            lo[a] = imax_std(cc - 1, 0);
            hi[a] = imin_std(cc + 1, G.dims[a] - 1);
            if (lo[a] > hi[a]) any = false;
        }
    }
    int cnt = 0;
    if (any) {
        for (int z = lo[2]; z <= hi[2]; ++z)
            for (int y = lo[1]; y <= hi[1]; ++y) {
                const long long rb = ((long long)z * dy + y) * dx;
                const int b = cellStart[rb + lo[0]], e = cellStart[rb + hi[0] + 1];
                for (int j = b; j < e; ++j) {
                    const float4 pj = P[j];
                    cnt += sqn3(qx - pj.x, qy - pj.y, qz - pj.z) < h2;
                }
            }
    }
    if (valid) nbrCount[i] = cnt;
    int cmax = warp_max_i(cnt);
    if ((p & 31) == 0) s_cmax[p >> 5] = cmax;
    __syncthreads();
    if (p == 0) {
        int m = s_cmax[0];
        for (int w = 1; w < kTileP / 32; ++w) m = imax_std(m, s_cmax[w]);
        const int cap = (m + 7) & ~7;
        s_cap = cap;
        const unsigned long long need = (unsigned long long)cap * kTileP;
        unsigned long long base;
        bool over;
        if (fb) {
            base = atomicAdd(&ctl->list_alloc_fb, need);
            over = base + need > (unsigned long long)fbCap;
        } else {
            base = atomicAdd(&ctl->list_alloc, need);
            over = base + need > (unsigned long long)listCap;
        }
        if (over) {
            atomicOr(&ctl->list_overflow, 1);
            ctl->abort = 1;
        }
        s_base = (unsigned)base;
        TileInfo ti;
        ti.nRuns = nRuns;
        ti.C = s_C;
        ti.listBase = (unsigned)base;
        ti.cap = cap;
        info[t] = ti;
        for (int r = 0; r < nRuns; ++r) runsOut[(long long)t * kMaxRuns + r] = s_runs[r];
    }
    __syncthreads();
    if (ctl->list_overflow) return;
    {
        const int wsum = warp_sum_i(cnt);
        if ((p & 31) == 0) atomicAdd(&ctl->list_entries, (unsigned long long)wsum);
    }
    if (!any || cnt == 0) return;
    const unsigned base = s_base + (unsigned)(p * s_cap);
    int w = 0;
    for (int z = lo[2]; z <= hi[2]; ++z)
        for (int y = lo[1]; y <= hi[1]; ++y) {
            const long long rb = ((long long)z * dy + y) * dx;
            const int b = cellStart[rb + lo[0]], e = cellStart[rb + hi[0] + 1];
            if (e <= b) continue;
            const int cb = fb ? 0 : cand_of(s_runs, nRuns, b);
            for (int j = b; j < e; ++j) {
                const float4 pj = P[j];
                if (sqn3(qx - pj.x, qy - pj.y, qz - pj.z) < h2) {
                    if (fb) fbLists[base + w] = j;
                    else lists[base + w] = (unsigned short)(cb + (j - b));
                    ++w;
                }
            }
        }
}

// Stage the tile's candidates into shared memory (coalesced per run).
template <bool kLambdaPass>
__device__ __forceinline__ void stage_candidates(const int2* s_runs, int nRuns, int C,
                                                 const float4* __restrict__ P,
                                                 const float* __restrict__ aux, float4* s_p,
                                                 float* s_aux) {
    for (int c = threadIdx.x; c < C; c += kTileP) {
        const int s = slot_of(s_runs, nRuns, c);
        s_p[c] = P[s];
        s_aux[c] = aux[s];
    }
}

// Load up to 8 u16 list entries of this particle starting at e (16-B load).
__device__ __forceinline__ uint4 load8(const unsigned short* __restrict__ lists, unsigned off) {
    return __ldg(reinterpret_cast<const uint4*>(lists + off));
}
__device__ __forceinline__ int pick16(const uint4& v, int q) {
    const unsigned w = q < 4 ? (q < 2 ? v.x : v.y) : (q < 6 ? v.z : v.w);
    return (q & 1) ? (int)(w >> 16) : (int)(w & 0xffffu);
}

// ------------------------------------------------------- lambda (tiles)

// computeLambda (solver.hpp:98-120) for every particle of the tile with
// level >= iter; neighbours gathered from shared memory.
template <bool kCoef>
__global__ void __launch_bounds__(kTileP) k_lambda_tile(
    int n, int iter, Ctl* ctl, const TileInfo* __restrict__ info, const int2* __restrict__ runs,
    const int* __restrict__ tileMax, const float4* __restrict__ P, const float* __restrict__ W,
    float* __restrict__ L, const int* __restrict__ LV, const unsigned short* __restrict__ lists,
    const int* __restrict__ fbLists, const int* __restrict__ nbrCount, float* __restrict__ coef,
    SolverConsts sc, int substep) {
    if (ctl->abort) return;
    const int t = blockIdx.x;
    if (tileMax[t] < iter) return;
    extern __shared__ __align__(128) unsigned char s_raw[];
    float4* s_p = reinterpret_cast<float4*>(s_raw);
    float* s_w = reinterpret_cast<float*>(s_raw + sizeof(float4) * kCandMax);
    __shared__ int2 s_runs[kMaxRuns];
    const TileInfo ti = info[t];
    const bool fb = ti.C < 0;
    if (threadIdx.x < ti.nRuns) s_runs[threadIdx.x] = runs[(long long)t * kMaxRuns + threadIdx.x];
    __syncthreads();
    if (!fb) stage_candidates<true>(s_runs, ti.nRuns, ti.C, P, W, s_p, s_w);
    __syncthreads();
    const int i = t * kTileP + threadIdx.x;
    bool bad = false;
    if (i < n && LV[i] >= iter) {
        const float4 xi = P[i];
        const int cnt = nbrCount[i];
        const unsigned off = ti.listBase + threadIdx.x * ti.cap;
        float rho = 0.f, gxs = 0.f, gys = 0.f, gzs = 0.f, denomJ = 0.f;
        if (!fb) {
            const int selfC = cand_of(s_runs, ti.nRuns, i);
            for (int e0 = 0; e0 < cnt; e0 += 8) {
                const uint4 v = load8(lists, off + e0);
                const int m = imin_std(8, cnt - e0);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (q >= m) break;
                    const int cj = pick16(v, q);
                    const float4 pj = s_p[cj];
                    const float wj = s_w[cj];
                    const float rx = xi.x - pj.x, ry = xi.y - pj.y, rz = xi.z - pj.z;
                    const float r2 = sqn3(rx, ry, rz);
                    rho += pj.w * poly6_r2(sc.kc, r2);
                    const float rn = sqrtf(r2);
                    const float a = sc.kc.h - rn;
                    const float c = sc.kc.spiky * a * a / rn;
                    const bool zero = (rn >= sc.kc.h || rn == 0.0f);
                    const float gx = zero ? 0.0f : c * rx;
                    const float gy = zero ? 0.0f : c * ry;
                    const float gz = zero ? 0.0f : c * rz;
                    if (kCoef) coef[off + e0 + q] = zero ? 0.0f : c;
                    gxs += gx;
                    gys += gy;
                    gzs += gz;
                    const float dj = wj * sqn3(gx, gy, gz);
                    denomJ += (cj == selfC) ? 0.0f : dj;
                }
            }
        } else {
            for (int e = 0; e < cnt; ++e) {
                const int j = fbLists[off + e];
                const float4 pj = P[j];
                const float wj = W[j];
                const float rx = xi.x - pj.x, ry = xi.y - pj.y, rz = xi.z - pj.z;
                const float r2 = sqn3(rx, ry, rz);
                rho += pj.w * poly6_r2(sc.kc, r2);
                float gx, gy, gz;
                spiky_grad(sc.kc, r2, rx, ry, rz, gx, gy, gz);
                gxs += gx;
                gys += gy;
                gzs += gz;
                const float dj = wj * sqn3(gx, gy, gz);
                denomJ += (j == i) ? 0.0f : dj;
            }
        }
        const float cc = rho * sc.invRho0 - 1.0f;
        const float sx = sc.invRho0 * gxs, sy = sc.invRho0 * gys, sz = sc.invRho0 * gzs;
        const float denom = W[i] * sqn3(sx, sy, sz) + sc.invRho0sq * denomJ + sc.eps;
        const float lam = -cc / denom;
        L[i] = lam;
        bad = !isfinite(lam);
    }
    report_bad(ctl, kPassLambda, bad, i);
    if (bad) {
        ctl->bad_substep[kPassLambda] = substep;
        ctl->bad_iter[kPassLambda] = iter;
    }
}

// -------------------------------------------------- delta-p + apply (tiles)

// computeDeltaP + apply + SDF projection (solver.hpp:125-141, 328-338) for
// level >= iter; particles with level == iter-1 finished after the previous
// iteration and copy their final x* Pc -> Pn (nobody reads Pn here).
template <bool kZeroFinished, bool kCoef>
__global__ void __launch_bounds__(kTileP) k_deltap_tile(
    int n, int iter, Ctl* ctl, const TileInfo* __restrict__ info, const int2* __restrict__ runs,
    const int* __restrict__ tileMax, const float4* __restrict__ Pc, float4* __restrict__ Pn,
    const float* __restrict__ W, const float* __restrict__ L, const int* __restrict__ LV,
    const unsigned short* __restrict__ lists, const int* __restrict__ fbLists,
    const int* __restrict__ nbrCount, const float* __restrict__ coef,
    const Scene* __restrict__ scene, SolverConsts sc, int substep) {
    if (ctl->abort) return;
    const int t = blockIdx.x;
    const int tmax = tileMax[t];
    if (tmax < iter - 1) return;
    const int i = t * kTileP + threadIdx.x;
    if (tmax < iter) {  // copy-forward only
        if (i < n && LV[i] == iter - 1) Pn[i] = Pc[i];
        return;
    }
    extern __shared__ __align__(128) unsigned char s_raw[];
    float4* s_p = reinterpret_cast<float4*>(s_raw);  // (x*, lambda) per candidate
    __shared__ int2 s_runs[kMaxRuns];
    const TileInfo ti = info[t];
    const bool fb = ti.C < 0;
    if (threadIdx.x < ti.nRuns) s_runs[threadIdx.x] = runs[(long long)t * kMaxRuns + threadIdx.x];
    __syncthreads();
    if (!fb) {
        for (int c = threadIdx.x; c < ti.C; c += kTileP) {
            const int s = slot_of(s_runs, ti.nRuns, c);
            const float4 q = Pc[s];
            float lam = L[s];
            if (kZeroFinished && !(LV[s] >= iter)) lam = 0.0f;
            s_p[c] = make_float4(q.x, q.y, q.z, lam);
        }
    }
    __syncthreads();
    bool bad = false;
    const int lv = i < n ? LV[i] : -1;
    if (lv >= iter) {
        const float4 xi = Pc[i];
        const float lamI = L[i];
        const int cnt = nbrCount[i];
        const unsigned off = ti.listBase + threadIdx.x * ti.cap;
        float sx = 0.f, sy = 0.f, sz = 0.f;
        if (!fb) {
            const int selfC = cand_of(s_runs, ti.nRuns, i);
            for (int e0 = 0; e0 < cnt; e0 += 8) {
                const uint4 v = load8(lists, off + e0);
                const int m = imin_std(8, cnt - e0);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (q >= m) break;
                    const int cj = pick16(v, q);
                    const float4 pj = s_p[cj];
                    const float rx = xi.x - pj.x, ry = xi.y - pj.y, rz = xi.z - pj.z;
                    float gx, gy, gz;
                    if (kCoef) {
                        const float c = coef[off + e0 + q];
                        gx = c * rx;
                        gy = c * ry;
                        gz = c * rz;
                    } else {
                        spiky_grad(sc.kc, sqn3(rx, ry, rz), rx, ry, rz, gx, gy, gz);
                    }
                    const float s = lamI + pj.w;
                    const bool self = (cj == selfC);
                    sx += self ? 0.0f : s * gx;
                    sy += self ? 0.0f : s * gy;
                    sz += self ? 0.0f : s * gz;
                }
            }
        } else {
            for (int e = 0; e < cnt; ++e) {
                const int j = fbLists[off + e];
                if (j == i) continue;
                float lamJ = L[j];
                if (kZeroFinished && !(LV[j] >= iter)) lamJ = 0.0f;
                const float4 pj = Pc[j];
                const float rx = xi.x - pj.x, ry = xi.y - pj.y, rz = xi.z - pj.z;
                float gx, gy, gz;
                spiky_grad(sc.kc, sqn3(rx, ry, rz), rx, ry, rz, gx, gy, gz);
                const float s = lamI + lamJ;
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
    } else if (lv == iter - 1) {
        Pn[i] = Pc[i];
    }
    report_bad(ctl, kPassApply, bad, i);
    if (bad) {
        ctl->bad_substep[kPassApply] = substep;
        ctl->bad_iter[kPassApply] = iter;
    }
}

// meanAbsConstraint (solver.hpp:166-180) over all particles with the tile
// lists (debug path: global gathers).
__global__ void __launch_bounds__(kTileP) k_residual_tile(
    int n, int iter, const Ctl* ctl, const int* __restrict__ activeCount,
    const TileInfo* __restrict__ info, const int2* __restrict__ runs, const float4* __restrict__ P,
    const unsigned short* __restrict__ lists, const int* __restrict__ fbLists,
    const int* __restrict__ nbrCount, SolverConsts sc, double* __restrict__ out) {
    if (ctl->abort) return;
    if (activeCount[iter] == 0) return;
    __shared__ int2 s_runs[kMaxRuns];
    const int t = blockIdx.x;
    const TileInfo ti = info[t];
    if (threadIdx.x < ti.nRuns) s_runs[threadIdx.x] = runs[(long long)t * kMaxRuns + threadIdx.x];
    __syncthreads();
    const int i = t * kTileP + threadIdx.x;
    double c = 0.0;
    if (i < n) {
        const float4 xi = P[i];
        const int cnt = nbrCount[i];
        const unsigned off = ti.listBase + threadIdx.x * ti.cap;
        float rho = 0.f;
        for (int e = 0; e < cnt; ++e) {
            const int j = ti.C < 0 ? fbLists[off + e] : slot_of(s_runs, ti.nRuns, lists[off + e]);
            const float4 pj = P[j];
            rho += pj.w * poly6_r2(sc.kc, sqn3(xi.x - pj.x, xi.y - pj.y, xi.z - pj.z));
        }
        c = (double)fabsf(rho / sc.rho0 - 1.0f);
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, c);
}

// Slot-based pre-stabilization (level < S), sdf.hpp:261-278.
__global__ void k_prestabilize_slots(int n, Ctl* ctl, int S, const int* __restrict__ LV,
                                     float4* __restrict__ XS, float4* __restrict__ X,
                                     const Scene* __restrict__ scene, float r, int iters,
                                     int substep, int ownB = 0, int ownE = 0x7fffffff) {
    if (ctl->abort) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool bad = false;
    if (i < n && LV[i] < S) {
        float4 s = XS[i];
        float4 x = X[i];
        if (scene->n > 0) {
            for (int it = 0; it < iters; ++it) {
                float gx, gy, gz;
                const float phi = scene_distance(*scene, s.x, s.y, s.z, gx, gy, gz);
                if (phi < r) {
                    const float kk = r - phi;
                    const float dx = kk * gx, dy = kk * gy, dz = kk * gz;
                    s.x += dx;
                    s.y += dy;
                    s.z += dz;
                    x.x += dx;
                    x.y += dy;
                    x.z += dz;
                }
            }
            XS[i] = s;
            X[i] = x;
        }
        bad = !finite3(s.x, s.y, s.z) && i >= ownB && i < ownE;
    }
    report_bad(ctl, kPassPrestab, bad, i - ownB);
    if (bad) ctl->bad_substep[kPassPrestab] = substep;
}

}  // namespace apbf_gpu
