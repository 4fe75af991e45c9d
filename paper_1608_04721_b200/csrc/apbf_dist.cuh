// apbf_dist.cuh -- kernels of the z-slab domain decomposition.
//
// Rank g owns the particles whose cell layer cz (of the substep's GLOBAL
// grid) lies in [zlo_g, zhi_g).  Every substep each rank sends every other
// rank q -- in its current (previous global) storage order -- the particles
// whose cz falls in q's slab extended by the 2-layer halo; q concatenates
// what it receives in source-rank order (its own particles in place g) and
// stable-sorts by cell, which reproduces the single-GPU global order
// restricted to its extended range.  Owned particles are then contiguous,
// lower ghosts precede them and upper ghosts follow, so every neighbour list
// and every per-particle sum is the single-GPU one, bit for bit.
#pragma once

#include "apbf_kernels.cuh"
#include "apbf_transport.h"

namespace apbf_gpu {

constexpr int kMaxRanks = 32;

__device__ __forceinline__ int layer_of(const GridDev& G, float h, float z) {
    const int v = f2i_trunc(floorf((z - G.origin[2]) / h));
    return imin_std(imax_std(v, 0), G.dims[2] - 1);
}

// Work per cz layer (global grid g) -> hist[dims.z]: each particle counts
// with its level (its particle-iterations this substep), so equal-sum slabs
// balance the solver work of APBF rather than the particle count.  The
// histogram holds `cap` layers (a device-sized grid): a deeper grid flags
// need_layers and aborts the frame (identically on every rank: the grid is
// global), and the host grows the histogram and runs the frame again.
//
// Each CTA takes one contiguous range of the storage order (cell order, so
// the range spans few layers) and aggregates in shared memory over a window
// of kHistWin layers from the range's first one; global atomics then go one
// per (CTA, layer) -- per warp they serialise at L2 on the few bins (about
// 600 per bin at 1M particles and 50 layers: 25 us).
constexpr int kHistItems = 4;
constexpr int kHistWin = 64;
__global__ void __launch_bounds__(256) k_layer_hist(int n, const float4* __restrict__ P, const int* __restrict__ LV,
                                                    Ctl* ctl, int g, float h, int* __restrict__ hist, int cap) {
    __shared__ int s_h[kHistWin];
    __shared__ int s_key0;
    if (ctl->abort) return;
    const GridDev G = ctl->grid[g];
    if (G.dims[2] > cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            ctl->need_layers = G.dims[2];
            ctl->abort = 1;
        }
        return;
    }
    const int per = (n + gridDim.x - 1) / gridDim.x;
    const int b0 = blockIdx.x * per, b1 = imin_std(n, b0 + per);
    for (int t = threadIdx.x; t < kHistWin; t += blockDim.x) s_h[t] = 0;
    if (threadIdx.x == 0) s_key0 = b0 < n ? layer_of(G, h, P[b0].z) : 0;
    __syncthreads();
    const int key0 = s_key0;
    for (int base = b0; base < b1; base += kHistItems * blockDim.x) {
        float z[kHistItems];
        int lv[kHistItems];
#pragma unroll
        for (int j = 0; j < kHistItems; ++j) {  // the chunk's loads issued together
            const int i = base + j * blockDim.x + threadIdx.x;
            z[j] = i < b1 ? P[i].z : 0.f;
            lv[j] = i < b1 ? LV[i] : 0;
        }
#pragma unroll
        for (int j = 0; j < kHistItems; ++j) {
            const int i = base + j * blockDim.x + threadIdx.x;
            // one shared atomic per distinct layer of the warp (a warp inside
            // one layer -- nearly all of them -- skips the match)
            const int key = i < b1 ? layer_of(G, h, z[j]) : -1;
            const int val = i < b1 ? 1 + lv[j] : 0;
            const unsigned same = __all_sync(0xffffffffu, key == __shfl_sync(0xffffffffu, key, 0))
                                      ? 0xffffffffu
                                      : __match_any_sync(0xffffffffu, key);
            const int sum = __reduce_add_sync(same, val);
            if (key >= 0 && (threadIdx.x & 31) == __ffs(same) - 1) {
                const int d = key - key0;
                if (d >= 0 && d < kHistWin) atomicAdd(&s_h[d], sum);
                else atomicAdd(&hist[key], sum);
            }
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < kHistWin; t += blockDim.x)
        if (s_h[t]) atomicAdd(&hist[key0 + t], s_h[t]);
}

// The slab partition on the device (identical on every rank: same global
// histogram in, same slabs out), so no host round trip sits between the
// histogram all-reduce and the exchange.  Too few layers: slab_error + abort.
// (Up to kPartSmem layers the histogram is staged in shared memory by the
// whole CTA and one thread then walks it; deeper grids walk it in global
// memory.  Launch with 4 * min(cap, kPartSmem) bytes of dynamic shared memory.)
constexpr int kPartSmem = 12000;
__global__ void k_slab_partition(const int* __restrict__ hist, Ctl* ctl, int G, int minLayers,
                                 int* __restrict__ zr, int cap) {
    extern __shared__ int s_hist[];
    if (ctl->abort) return;
    const int dz = imin_std(ctl->grid[0].dims[2], cap);  // (dims.z <= cap: k_layer_hist aborts otherwise)
    const bool staged = dz <= kPartSmem;
    if (staged)
        for (int z = threadIdx.x; z < dz; z += blockDim.x) s_hist[z] = hist[z];
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (!slab_partition(staged ? s_hist : hist, dz, G, minLayers, zr, zr + G)) {
        ctl->slab_error = 1;
        ctl->abort = 1;
    }
}

// Per-destination record classes of a substep's exchange, sent ahead of the
// records so that the receiver knows every size of its substep after ONE
// host synchronisation: [0] total, [1..4] records in layers lo-2 .. lo+1,
// [5..8] records in layers hi-2 .. hi+1 of the destination's slab [lo, hi).
// (The receiver's stable cell sort puts them in z-major order, so its slab
// bounds are prefix sums of these.)
constexpr int kCls = 9;

// Destination bit mask: bit q set when cz in [lo[q] - halo, hi[q] + halo);
// with cls != nullptr also the kCls class counts per destination (per-CTA
// shared-memory counters, one global atomic per non-zero counter and CTA).
__global__ void k_dest_mask(int n, const float4* __restrict__ P, const Ctl* ctl, int g, float h,
                            const int* __restrict__ lo, const int* __restrict__ hi, int G, int halo,
                            unsigned* __restrict__ mask, int* __restrict__ cls = nullptr) {
    __shared__ int s_cls[kMaxRanks * kCls];
    if (cls) {
        for (int t = threadIdx.x; t < G * kCls; t += blockDim.x) s_cls[t] = 0;
        __syncthreads();
    }
    // (grid-stride: the per-CTA counters flush from a few hundred CTAs, not
    // one per 256 particles -- their global atomics serialise on few words)
    const bool run = !ctl->abort;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; run && i < n; i += gridDim.x * blockDim.x) {
        const int cz = layer_of(ctl->grid[g], h, P[i].z);
        unsigned m = 0;
        for (int q = 0; q < G; ++q) {
            const int l = lo[q], u = hi[q];
            if (cz >= l - halo && cz < u + halo) {
                m |= 1u << q;
                if (cls) {
                    atomicAdd(&s_cls[q * kCls], 1);
                    if (cz >= l - 2 && cz < l + 2) atomicAdd(&s_cls[q * kCls + 1 + (cz - (l - 2))], 1);
                    if (cz >= u - 2 && cz < u + 2) atomicAdd(&s_cls[q * kCls + 5 + (cz - (u - 2))], 1);
                }
            }
        }
        mask[i] = m;
    }
    if (cls) {
        __syncthreads();
        for (int t = threadIdx.x; t < G * kCls; t += blockDim.x)
            if (s_cls[t]) atomicAdd(&cls[t], s_cls[t]);
    }
}

// Exclusive scan of the G per-destination totals (G <= 32).
__global__ void k_dest_starts(const int* __restrict__ destCount, int G, int* __restrict__ destStart) {
    const int q = threadIdx.x;
    const int v = q < G ? destCount[q] : 0;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (q >= o) incl += x;
    }
    if (q < G) destStart[q] = incl - v;
}

// Metrics exchange ranges from the all-reduced per-rank metrics-grid layer
// spans (lo = min, hi = max over each rank's owned particles): every other
// rank's [lo, hi + 1) plus the k_dest_mask halo, everything for rank g.
__global__ void k_metrics_ranges(int G, int g, int* __restrict__ lo, int* __restrict__ hi) {
    const int q = threadIdx.x;
    if (q >= G) return;
    if (q == g) {
        lo[q] = -(1 << 29);
        hi[q] = 1 << 29;
    } else if (lo[q] > hi[q]) {  // empty rank
        lo[q] = 1 << 29;
        hi[q] = -(1 << 29);
    } else {
        hi[q] = hi[q] + 1;  // exclusive
    }
}

// Stable expansion by destination: per tile (kTileSize elements) counts of
// every destination bit, column-major tileCount[q * numTiles + tile].
__global__ void __launch_bounds__(kTileThreads) k_mask_tile_counts(int n, const unsigned* __restrict__ mask,
                                                                   int G, int numTiles,
                                                                   int* __restrict__ tileCount) {
    __shared__ int s_c[kMaxRanks];
    for (int q = threadIdx.x; q < G; q += blockDim.x) s_c[q] = 0;
    __syncthreads();
    const int tile = blockIdx.x;
    for (int r = 0; r < kTileRounds; ++r) {
        const int k = tile * kTileSize + r * kTileThreads + threadIdx.x;
        const unsigned m = k < n ? mask[k] : 0u;
        for (int q = 0; q < G; ++q) {
            const unsigned b = __ballot_sync(0xffffffffu, (m >> q) & 1u);
            if ((threadIdx.x & 31) == 0 && b) atomicAdd(&s_c[q], __popc(b));
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < G; q += blockDim.x) tileCount[(long long)q * numTiles + tile] = s_c[q];
}

// outIdx[destStart[q] + tileOffset[q][tile] + rank] = k, rank = number of
// earlier elements of the tile with bit q (order preserving).
__global__ void __launch_bounds__(kTileThreads) k_mask_scatter(int n, const unsigned* __restrict__ mask,
                                                               int G, int numTiles,
                                                               const int* __restrict__ tileOffset,
                                                               const int* __restrict__ destStart,
                                                               int* __restrict__ outIdx) {
    __shared__ int s_run[kMaxRanks];
    __shared__ int s_wc[kTileThreads / 32][kMaxRanks];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = blockIdx.x;
    for (int q = threadIdx.x; q < G; q += blockDim.x) s_run[q] = 0;
    __syncthreads();
    for (int r = 0; r < kTileRounds; ++r) {
        const int k = tile * kTileSize + r * kTileThreads + threadIdx.x;
        const unsigned m = k < n ? mask[k] : 0u;
        for (int q = 0; q < G; ++q) {
            const unsigned b = __ballot_sync(0xffffffffu, (m >> q) & 1u);
            if (lane == 0) s_wc[warp][q] = __popc(b);
        }
        __syncthreads();
        for (int q = 0; q < G; ++q) {
            const unsigned b = __ballot_sync(0xffffffffu, (m >> q) & 1u);
            if ((m >> q) & 1u) {
                int before = s_run[q] + __popc(b & ((1u << lane) - 1u));
                for (int w = 0; w < warp; ++w) before += s_wc[w][q];
                outIdx[destStart[q] + tileOffset[(long long)q * numTiles + tile] + before] = k;
            }
        }
        __syncthreads();
        for (int q = threadIdx.x; q < G; q += blockDim.x) {
            int s = 0;
            for (int w = 0; w < kTileThreads / 32; ++w) s += s_wc[w][q];
            s_run[q] += s;
        }
        __syncthreads();
    }
}

// Exclusive scan of tileCount[q][*] per destination q (one block each).
__global__ void __launch_bounds__(1024) k_mask_scan(int numTiles, int* __restrict__ tileCount,
                                                    int* __restrict__ destCount) {
    const int q = blockIdx.x;
    int* row = tileCount + (long long)q * numTiles;
    __shared__ int s_w[32];
    __shared__ int s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int t0 = 0; t0 < numTiles; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        const int v = t < numTiles ? row[t] : 0;
        int incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int x = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += x;
        }
        if (lane == 31) s_w[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int w = s_w[lane];
            int wi = w;
            for (int o = 1; o < 32; o <<= 1) {
                const int x = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += x;
            }
            s_w[lane] = wi - w;
        }
        __syncthreads();
        const int excl = s_carry + s_w[warp] + incl - v;
        if (t < numTiles) row[t] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) destCount[q] = s_carry;
}

// 16-word particle record for the all-to-all: x(3) v(3) x*(3) mass invMass
// lambda level pad(3).
struct alignas(64) Rec {
    float x[3], v[3], xs[3], m, w, lam;
    int lv;
    int pad[3];
};

// Records for the other ranks, sized on the device (enqueued ahead of the
// substep's host synchronisation): destination q's segment starts at
// destStart[q] and holds destCount[q] records; the rank's own segment g is
// skipped: the local sort reads it in place (SelfMap).  Grid-stride over the
// records that leave.
__global__ void k_pack_recs(const int* __restrict__ idx, StateSet s, Rec* __restrict__ out,
                            const int* __restrict__ destCount, const int* __restrict__ destStart, int G, int g) {
    const int total = destStart[G - 1] + destCount[G - 1];
    const int selfB = destStart[g], selfN = destCount[g];
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total - selfN; t += gridDim.x * blockDim.x) {
        const int k = t < selfB ? t : t + selfN;
        const int i = idx[k];
        const float4 x = s.X[i], v = s.V[i], xs = s.XS[i];
        Rec r;
        r.x[0] = x.x;
        r.x[1] = x.y;
        r.x[2] = x.z;
        r.v[0] = v.x;
        r.v[1] = v.y;
        r.v[2] = v.z;
        r.xs[0] = xs.x;
        r.xs[1] = xs.y;
        r.xs[2] = xs.z;
        r.m = xs.w;
        r.w = s.W[i];
        r.lam = s.L[i];
        r.lv = s.LV[i];
        r.pad[0] = r.pad[1] = r.pad[2] = 0;
        out[k] = r;
    }
}

__global__ void k_unpack_recs(int cnt, const Rec* __restrict__ in, StateSet d, int skipB = 0, int skipE = 0) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= cnt || (k >= skipB && k < skipE)) return;
    const Rec r = in[k];
    d.X[k] = make_float4(r.x[0], r.x[1], r.x[2], 0.f);
    d.V[k] = make_float4(r.v[0], r.v[1], r.v[2], 0.f);
    d.XS[k] = make_float4(r.xs[0], r.xs[1], r.xs[2], r.m);
    d.W[k] = r.w;
    d.L[k] = r.lam;
    d.LV[k] = r.lv;
}

// One all-reduce instead of three for the substep's grid: [~abort, lo(3),
// ~hi(3)] all-reduced with MIN (bitwise not reverses the order of ordered
// ints without overflow), then written back (k_grid_unpack_params).
__global__ void k_grid_reduce_pack(const Ctl* ctl, int g, int* __restrict__ buf) {
    const GridDev& G = ctl->grid[g];
    buf[0] = ~ctl->abort;
    for (int a = 0; a < 3; ++a) {
        buf[1 + a] = G.lo_ord[a];
        buf[4 + a] = ~G.hi_ord[a];
    }
}
// The substep's grid after its all-reduce, in one launch: unpack, the grid
// parameters (thread 0, k_grid_params), and the two per-substep counters the
// next passes accumulate into cleared by the whole CTA (instead of two
// memset nodes and two single-thread kernels).
__global__ void k_grid_unpack_params(Ctl* ctl, int g, const int* __restrict__ buf, float h, float pad,
                                     int* __restrict__ zeroA, int nA, int* __restrict__ zeroB, int nB) {
    for (int t = threadIdx.x; t < nA; t += blockDim.x) zeroA[t] = 0;
    for (int t = threadIdx.x; t < nB; t += blockDim.x) zeroB[t] = 0;
    if (threadIdx.x != 0) return;
    GridDev& G = ctl->grid[g];
    ctl->abort = ~buf[0];
    for (int a = 0; a < 3; ++a) {
        G.lo_ord[a] = buf[1 + a];
        G.hi_ord[a] = ~buf[4 + a];
    }
    grid_params(ctl, g, h, pad);
}

// K16 for the owned slice [b, b + m) of the sorted set, written to the front
// of the other set (this rank's state for the next substep) together with
// the fields finalize does not change: the slab path's finalize and
// compaction in one pass.  Arithmetic and error reports as k_finalize.
__global__ void k_finalize_owned(int m, int b, Ctl* ctl, const float4* __restrict__ Pf, StateSet from,
                                 StateSet to, float dt, float cap, int substep) {
    if (ctl->abort) return;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    bool badV = false, badX = false;
    if (i < m) {
        const float4 s = Pf[b + i];
        float4 v, xo;
        finalize_particle(s, from.X[b + i], dt, cap, v, xo, badV, badX);
        to.X[i] = xo;
        to.V[i] = v;
        to.XS[i] = s;
        to.W[i] = from.W[b + i];
        to.L[i] = from.L[b + i];
        to.LV[i] = from.LV[b + i];
    }
    finalize_report(ctl, badV, badX, i, substep);
}

// The iteration order's levels (0, never active, outside [b, e) or inside
// the excluded [xb, xe)) and their per-tile histogram, in one pass.
// With ob < oe also the level sum of the owned slots [ob, oe) (the rank's
// particle-iterations, solver.hpp:311-313) into ctl->total_iterations.
__global__ void __launch_bounds__(kTileThreads) k_mask_level_tiles(int n, Ctl* ctl,
                                                                   const int* __restrict__ LV, int b, int e,
                                                                   int xb, int xe, int* __restrict__ LVo,
                                                                   int nMax, int numTiles,
                                                                   int* __restrict__ tileCount, int ob = 0,
                                                                   int oe = 0) {
    if (ctl->abort) return;
    extern __shared__ int s_cnt[];
    __shared__ int s_tot;
    for (int l = threadIdx.x; l <= nMax; l += blockDim.x) s_cnt[l] = 0;
    if (threadIdx.x == 0) s_tot = 0;
    __syncthreads();
    int tot = 0;
    for (int r = 0; r < kTileRounds; ++r) {
        const int k = blockIdx.x * kTileSize + r * kTileThreads + threadIdx.x;
        if (k < n) {
            const int raw = LV[k];
            const int lv = (k >= b && k < e && !(k >= xb && k < xe)) ? raw : 0;
            LVo[k] = lv;
            atomicAdd(&s_cnt[imin_std(imax_std(lv, 0), nMax)], 1);
            if (k >= ob && k < oe) tot += raw;
        }
    }
    tot = warp_sum_i(tot);
    if ((threadIdx.x & 31) == 0 && tot) atomicAdd(&s_tot, tot);
    __syncthreads();
    for (int l = threadIdx.x; l <= nMax; l += blockDim.x)
        tileCount[(long long)l * numTiles + blockIdx.x] = s_cnt[l];
    if (threadIdx.x == 0 && s_tot) atomicAdd(&ctl->total_iterations, (unsigned long long)s_tot);
}

// Metrics ghost records: (x, y, z, mass) + owned flag in the w of a second
// float? -- packed as float4 xyzm and an int flag array.
// Sized on the device (ahead of the host synchronisation, as k_pack_recs):
// every destination's (x, y, z, mass) records; the rank's own segment goes
// straight to its place in the received array (after the records of ranks
// q < g) together with its owned flag, the others' flags are cleared.
__global__ void k_pack_pm(const int* __restrict__ idx, const float4* __restrict__ X,
                          const float4* __restrict__ XS, float4* __restrict__ out,
                          const int* __restrict__ destCount, const int* __restrict__ destStart,
                          const int* __restrict__ recvCls, int G, int g, float4* __restrict__ recv,
                          int* __restrict__ ownedFlag) {
    const int total = destStart[G - 1] + destCount[G - 1];
    const int selfB = destStart[g], selfE = selfB + destCount[g];
    int off = 0, nRecv = 0;
    for (int q = 0; q < G; ++q) {
        if (q < g) off += recvCls[q * kCls];
        nRecv += recvCls[q * kCls];
    }
    const int stride = gridDim.x * blockDim.x;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < total; k += stride) {
        const int i = idx[k];
        const float4 x = X[i];
        const float4 r = make_float4(x.x, x.y, x.z, XS[i].w);
        if (k >= selfB && k < selfE) recv[off + k - selfB] = r;
        else out[k] = r;
    }
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nRecv; k += stride)
        ownedFlag[k] = (k >= off && k < off + selfE - selfB) ? 1 : 0;
}

// Densities of the owned particles of a sorted (position, mass) array whose
// owned flags travelled through the same permutation.
__global__ void k_density_stats_owned(int n, Ctl* ctl, const float4* __restrict__ S,
                                      const int* __restrict__ owned, const int* __restrict__ cellStart,
                                      KernelConsts kc) {
    if (ctl->abort) return;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const GridDev& G = ctl->grid[1];
    float rho = 0.f;
    const bool valid = k < n && owned[k];
    if (valid) {
        const float4 q = S[k];
        const float p[3] = {q.x, q.y, q.z};
        int lo[3], hi[3];
        bool any = true;
        for (int a = 0; a < 3; ++a) {
            const int c = f2i_trunc(floorf((p[a] - G.origin[a]) / kc.h));
            lo[a] = imax_std(c - 1, 0);
            hi[a] = imin_std(c + 1, G.dims[a] - 1);
            if (lo[a] > hi[a]) any = false;
        }
        if (any)
            scan_candidates_all(G, cellStart, S, lo, hi, q.x, q.y, q.z, kc.h2,
                                [&](int, const float4& pj, float r2, bool m) {
                                    const float t = pj.w * poly6_r2_in(kc, r2);
                                    rho += m ? t : 0.0f;
                                });
    }
    double s = valid ? (double)rho : 0.0;
    int mn = valid ? f2ord(rho) : 0x7fffffff;
    int mx = valid ? f2ord(rho) : (int)0x80000000;
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&ctl->rho_sum, s);
        atomicMin(&ctl->rho_min_ord, mn);
        atomicMax(&ctl->rho_max_ord, mx);
    }
}

// gather of an int array through a permutation (owned flags of the metrics sort)
__global__ void k_gather_int(int n, const int* __restrict__ perm, const int* __restrict__ in,
                             int* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) out[k] = in[perm[k]];
}

// lo[q] = INT_MAX, hi[q] = INT_MIN: the identity of the span all-reduce
__global__ void k_span_init(int G, int* __restrict__ lo, int* __restrict__ hi) {
    const int q = threadIdx.x;
    if (q < G) {
        lo[q] = 0x7fffffff;
        hi[q] = (int)0x80000000;
    }
}

// metrics-grid cz range of the owned particles (positions X) -> *lo_out, *hi_out
__global__ void k_layer_minmax(int n, const float4* __restrict__ X, const Ctl* ctl, int g, float h,
                               int* __restrict__ lo_out, int* __restrict__ hi_out) {
    __shared__ int s_lo[32], s_hi[32];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int lo = 0x7fffffff, hi = (int)0x80000000;
    if (i < n) lo = hi = layer_of(ctl->grid[g], h, X[i].z);
    lo = warp_min_i(lo);
    hi = warp_max_i(hi);
    if ((threadIdx.x & 31) == 0) {
        s_lo[threadIdx.x >> 5] = lo;
        s_hi[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // one atomic pair per block
        const bool in = threadIdx.x < (blockDim.x >> 5);
        lo = warp_min_i(in ? s_lo[threadIdx.x] : 0x7fffffff);
        hi = warp_max_i(in ? s_hi[threadIdx.x] : (int)0x80000000);
        if (threadIdx.x == 0) {
            atomicMin(lo_out, lo);
            atomicMax(hi_out, hi);
        }
    }
}

}  // namespace apbf_gpu
