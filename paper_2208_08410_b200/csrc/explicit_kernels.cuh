// explicit_kernels.cuh — NEXT#1: the explicit-Gram path of Alg. 2 (lines 6-9) with the
// distributed Gram of Alg. 3, deflated exactly.
//
// Alg. 2 forms B = X'^T X' and iterates v1 = B v.  Re-forming B for every component (P:116 with the
// residual X' of Alg. 1 line 8) would cost a Gram per component; Eq. 1 updates it but
// assumes U^T U = I (reading R7).  Exact instead: with B0 = A^T A, P = A^T U (n x l) and Q = U^T U,
//     X'^T X' = B0 - P S V^T - V S P^T + V S Q S V^T,
// so  y = B0 v - P c - V g,   c = S (V^T v),   g = S (P^T v - Q c).
// B0 is built once (the paper's Alg. 3 Gram: the tcgen05 3xTF32 CTA-pair kernel of gram_tc.cuh,
// fp32-level products; TSVD_GRAM_CUBLAS=1 keeps round 1's three cuBLAS TF32 GEMMs of a hi/lo split
// of A), P and Q grow by one column per component from the extraction pass
// (u = A v / sigma, P[:, l] = A^T u, Q[l, :] = U^T u: one pass of the fused kernel with c = 0).
// Per iteration the n x n B0 is streamed once (n^2 * 4 bytes instead of 4 m n): gb_persist runs all
// iterations of a component in one cooperative kernel, each CTA owning whole rows of B0, so y_r is
// complete in the CTA that streams row r and one grid barrier per iteration suffices.
#pragma once
#include "persist_kernels.cuh"

namespace tsvd {

// (round-1 cuBLAS path, TSVD_GRAM_CUBLAS=1) hi/lo split of fp32 A into two TF32-exact fp32 arrays:
// hi = rna_tf32(a), lo = rna_tf32(a - hi);
// hi hi^T + hi lo^T + lo hi^T recovers a a^T to ~2^-21 relative (the three-term TF32 product)
__global__ void split_tf32(const float *__restrict__ A, int64_t rows, int64_t cols, int64_t lda,
                           float *__restrict__ hi, float *__restrict__ lo) {
    const int64_t total = rows * cols;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols, c = i - r * cols;
        const float a = A[r * lda + c];
        uint32_t h;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(a));
        const float hf = __uint_as_float(h);
        uint32_t l2;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l2) : "f"(a - hf));
        hi[i] = hf;
        lo[i] = __uint_as_float(l2);
    }
}

// Symmetric task schedule of the Gram (n_b(n_b+1)/2 block tasks instead of n_b^2): only the
// blocks (I <= J) are multiplied; this kernel fills the strictly-lower blocks by transposition.
// M[c][r] = B[r + c*ldb] (column-major as cuBLAS wrote it): blocks with blk(c) < blk(r) were not
// computed; they take M[r][c].  32x32 tiles through shared memory (both sides coalesced).
__global__ void gram_mirror(float *__restrict__ B, int64_t n, int64_t ldb, int64_t bs) {
    __shared__ float tile[32][33];
    const int64_t c0 = (int64_t)blockIdx.y * 32, r0 = (int64_t)blockIdx.x * 32;
    if (c0 / bs >= r0 / bs) return;  // (bs is a multiple of 32: one block row and column per tile)
    const int tx = threadIdx.x, ty = threadIdx.y;                   // 32 x 8
    for (int k = ty; k < 32; k += 8) {                              // read M[r][c] (contiguous in c)
        const int64_t r = r0 + k, c = c0 + tx;
        if (r < n && c < n) tile[k][tx] = B[c + r * ldb];
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {  // write M[c][r] (contiguous in r) where blk(c) < blk(r)
        const int64_t c = c0 + k, r = r0 + tx;
        if (r < n && c < n && c / bs < r / bs) B[r + c * ldb] = tile[tx][k];
    }
}

struct GbParams {
    const float *B;          // n x ldb fp32 (B0 = A^T A)
    int64_t ldb;
    int64_t rows;            // n
    int32_t n, n4;
    const float *P;          // n x ldp fp32 (A^T U)
    int32_t ldp;
    const double *V;         // n x ldv fp64
    int32_t ldv;
    const double *S;
    const double *Q;         // k x ldq fp64 (U^T U)
    int32_t ldq;
    int32_t l;
    int32_t stages, stage_bytes, row_bytes;
    double *ybuf;
    int64_t ystride;
    LoopState *st;
    double *c;               // out: last c (for the report / resume)
    double *part;            // [2][G][part_ld]: yy, vy, V^T y (l), P^T y (l); the two halves
                             // alternate, so a CTA writing the next totals never races a CTA
                             // still reading the previous ones (a barrier separates reuse)
    int32_t part_ld;
    unsigned *gbar;
    double eps;
    int32_t fixed_T, max_iter;
    int32_t serpentine;
    // world > 1: this rank iterates on rows [row0, row0 + rows) of B0 only; every iteration's y rows
    // and per-CTA sums go to every rank as stamped words (value halves + exchange stamp, as N7):
    // yx[r] = rank r's y area [2 parity][n], sx[r] = its sums area [2][world][G][2 + 2 l]
    int64_t row0;
    int32_t world, rank;
    ulonglong2 *yx[kMaxRanks];
    ulonglong2 *sx[kMaxRanks];
};

// world > 1: sums of the per-CTA quantities over [rank][CTA] in that fixed order, from the stamped
// sums area (half-warp per quantity); a stale first read leaves warp 0 polling with a back-off
__device__ __forceinline__ void gx_totals(const ulonglong2 *area, int E, int nqx, unsigned stamp, double *tot_c,
                                          LoopState *st) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
    const int hl = lane & 15;
    const unsigned long long t0 = globaltimer_ns();
    for (;;) {
        bool ok = true;
        for (int q0 = 2 * warp; q0 < nqx; q0 += 2 * NW) {
            const int q = q0 + (lane >> 4);
            double v = q < nqx ? ll_try_sum<10>(area + q, nqx, hl, 16, E, stamp, ok) : 0.0;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (hl == 0 && q < nqx) tot_c[q] = v;
        }
        if (__syncthreads_and(ok)) return;
        if (warp == 0)
            for (int e = lane; e < E; e += 32)
                for (unsigned spin = 0;; ++spin) {
                    const ulonglong2 w = ld_volatile_u2(area + (int64_t)e * nqx + nqx - 1);
                    if ((unsigned)(w.x >> 32) == stamp && (unsigned)(w.y >> 32) == stamp) break;
                    if ((spin & 255) == 255 && globaltimer_ns() - t0 > 30000000000ull) {
                        st->status = -6;
                        st->stop = 1;
                        break;
                    }
                    __nanosleep(64);
                }
        __syncthreads();
        __shared__ int tout_s;  // give-up decision taken once and shared: the whole block returns
        if (threadIdx.x == 0) tout_s = globaltimer_ns() - t0 > 30000000000ull;
        __syncthreads();
        if (tout_s) return;
    }
}

template <int T, int NV>
__global__ void __launch_bounds__(T) gb_persist(const GbParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int NW = T / 32;
    griddep_launch();
    griddep_wait();
    LoopState *st = p.st;
    if (st->stop || st->done) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, b = blockIdx.x;
    const int S = p.stages, l = p.l;
    const int kp = (p.part_ld - 2) / 2;  // room per vector in part / tot
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)S * p.stage_bytes);
    double *red = reinterpret_cast<double *>(bars + kMaxStages);  // [2][NW]
    double *cvec = red + 2 * NW;                                   // [kp]
    double *gvec = cvec + kp;                                      // [kp]
    double *tot = gvec + kp;                                       // [2 + 2 kp]
    __shared__ int64_t slot_row[kMaxStages];
    __shared__ double ny_s;
    __shared__ int done_s;
    __shared__ int64_t plo, pnr, pk;
    __shared__ int pp, pslot, pit0;
    const int64_t lo = p.row0 + p.rows * b / G;  // global rows of B0 (row0 = 0 on one GPU)
    const int nr = (int)(p.row0 + p.rows * (b + 1) / G - lo);
    int it = st->it;
    const bool mx = p.world > 1;
    unsigned xe = st->xepoch;  // world > 1: exchanges so far (monotone: a stale stamp never matches)
    const int nqx = 2 + 2 * l;  // exchanged sums: yy, vy, V^T y (l), P^T y (l)
    __shared__ double totc[2 + 2 * 128];

    auto feed = [&]() {
        const int64_t k = pk;
        const int64_t row = (p.serpentine && ((pit0 + pp) & 1)) ? plo + pnr - 1 - k : plo + k;
        if (k + 1 == pnr) {
            pk = 0;
            pp = pp + 1;
        } else {
            pk = k + 1;
        }
        const int slot = pslot;
        pslot = slot + 1 == S ? 0 : slot + 1;
        slot_row[slot] = row;
        mbar_arrive_expect_tx(&bars[slot], (uint32_t)(p.n4 * 16));
        tma_load_1d(smem + (size_t)slot * p.stage_bytes, p.B + row * p.ldb, (uint32_t)(p.n4 * 16), &bars[slot]);
    };
    if (tid == 0) {
        plo = lo;
        pnr = nr;
        pk = 0;
        pp = 0;
        pslot = 0;
        pit0 = it;
        for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
        fence_barrier_init();
        if (nr > 0)
            for (int s = 0; s < S; ++s) feed();
        ny_s = st->ny;
    }
    __syncthreads();

    int pb = 0;  // half of part[] written next
    auto my_part = [&]() { return p.part + ((int64_t)pb * G + b) * p.part_ld; };
    // sums over the CTAs of part[.][q], q < nq, in a fixed order (half-warp per quantity)
    auto grid_totals = [&](int nq) {
        const int hl = lane & 15;
        const double *half = p.part + (int64_t)pb * G * p.part_ld;
        for (int q0 = 2 * warp; q0 < nq; q0 += 2 * NW) {
            const int q = q0 + (lane >> 4);
            double s = q < nq ? strided_sum<10>(half + q, p.part_ld, hl, 16, G) : 0.0;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (hl == 0 && q < nq) tot[q] = s;
        }
        __syncthreads();
        pb ^= 1;
    };
    // c = S (V^T v), g = S (P^T v - Q c) from tot[2 ..] = (V^T y, P^T y) and ||y|| (v = y / ny)
    auto make_cg = [&](double ny) {
        for (int i = tid; i < l; i += T) cvec[i] = p.S[i] * (tot[2 + i] / ny);
        __syncthreads();
        for (int i = tid; i < l; i += T) {
            double qc = 0.0;
            for (int j = 0; j < l; ++j) qc += p.Q[(int64_t)i * p.ldq + j] * cvec[j];
            gvec[i] = p.S[i] * (tot[2 + kp + i] / ny - qc);
            if (b == 0) p.c[i] = cvec[i];
        }
        __syncthreads();
    };

    // ---- c, g of the first iterate (v = y_cur / ||y_cur||): V^T v and P^T v over this CTA's rows
    {
        const double *ycur = p.ybuf + (int64_t)(it & 1) * p.ystride;
        double vt = 0.0, pt = 0.0;
        if (tid < l)
            for (int64_t r = lo; r < lo + nr; ++r) {
                const double yr = __ldcg(ycur + r);
                vt += p.V[r * p.ldv + tid] * yr;
                pt += (double)p.P[r * p.ldp + tid] * yr;
            }
        if (mx) {
            const unsigned sx = ++xe;
            for (int r = 0; r < p.world; ++r) {
                ulonglong2 *dst = p.sx[r] + (((int64_t)(sx & 1u) * p.world + p.rank) * G + b) * nqx;
                if (tid == 0) {
                    ll_send(dst + 0, sx, 0.0);
                    ll_send(dst + 1, sx, 0.0);
                }
                if (tid < l) {
                    ll_send(dst + 2 + tid, sx, vt);
                    ll_send(dst + 2 + l + tid, sx, pt);
                }
            }
            gx_totals(p.sx[p.rank] + (int64_t)(sx & 1u) * p.world * G * nqx, p.world * G, nqx, sx, totc, st);
            for (int i = tid; i < l; i += T) {
                tot[2 + i] = totc[2 + i];
                tot[2 + kp + i] = totc[2 + l + i];
            }
            __syncthreads();
        } else {
            double *pr = my_part();
            if (tid == 0) pr[0] = pr[1] = 0.0;
            if (tid < l) {
                pr[2 + tid] = vt;
                pr[2 + kp + tid] = pt;
            }
            __threadfence();
            grid_sync(p.gbar);
            grid_totals(2 + kp + l);
        }
        make_cg(ny_s);
    }

    const int tail = p.n & 3;
    int cs = 0, rb = 0;
    uint32_t cph = 0;
    for (;;) {
        const double inv = 1.0 / ny_s;
        const double *ycur = p.ybuf + (int64_t)(it & 1) * p.ystride;
        double *ynew = p.ybuf + (int64_t)((it + 1) & 1) * p.ystride;
        float4 vr[NV];
        if (mx && it != pit0) {  // the previous iteration's y rows of every rank, stamped
            const ulonglong2 *ya = p.yx[p.rank] + (int64_t)(xe & 1u) * p.n;
            const unsigned long long t0 = globaltimer_ns();
            for (unsigned spin = 0;; ++spin) {
                bool ok = true;
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    const int idx = k * T + tid;
                    double y4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (idx < p.n4 && 4 * idx + c < p.n) {
                            const ulonglong2 w = ld_volatile_u2(ya + 4 * (int64_t)idx + c);
                            ok &= (unsigned)(w.x >> 32) == xe && (unsigned)(w.y >> 32) == xe;
                            y4[c] = __hiloint2double((int)(unsigned)w.y, (int)(unsigned)w.x);
                        }
                    vr[k] = make_float4((float)(y4[0] * inv), (float)(y4[1] * inv), (float)(y4[2] * inv),
                                        (float)(y4[3] * inv));
                }
                if (ok) break;
                if ((spin & 255) == 255 && globaltimer_ns() - t0 > 30000000000ull) {
                    st->status = -6;
                    st->stop = 1;
                    break;
                }
                __nanosleep(64);
            }
        } else {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int idx = k * T + tid;
            double2 lo2 = make_double2(0.0, 0.0), hi2 = lo2;
            if (idx < p.n4) {
                lo2 = __ldcg(reinterpret_cast<const double2 *>(ycur + 4 * idx));
                hi2 = __ldcg(reinterpret_cast<const double2 *>(ycur + 4 * idx + 2));
            }
            vr[k] = make_float4((float)(lo2.x * inv), (float)(lo2.y * inv), (float)(hi2.x * inv), (float)(hi2.y * inv));
        }
        }
        const unsigned sxn = xe + 1u;  // world > 1: this iteration's exchange stamp
        const double cv = tid < l ? cvec[tid] : 0.0, gv = tid < l ? gvec[tid] : 0.0;
        double a_yy = 0.0, a_vy = 0.0, a_vt = 0.0, a_pt = 0.0;
        // the row-dependent loads besides the TMA row (V_r, P_r deflation entries, y_cur[r] of the
        // stop test) are issued one row ahead: slot_row of the next slot was written by the producer
        // at least one block barrier ago when S >= 3 (it feeds a slot right after the barrier of the
        // row that freed it), so their global-memory latency no longer sits between the row landing
        // and its dot product (per row 1.75 us against 1.5 us of HBM time before)
        double vri_n = 0.0, pri_n = 0.0, ycr_n = 0.0;
        auto row_loads = [&](int slot) {
            const int64_t rr = slot_row[slot];
            if (tid < l) {
                vri_n = p.V[rr * p.ldv + tid];
                pri_n = (double)p.P[rr * p.ldp + tid];
            }
            if (tid == 0) ycr_n = __ldcg(ycur + rr);
        };
        if (nr > 0) row_loads(cs);
        for (int k = 0; k < nr; ++k) {
            const int64_t r = slot_row[cs];
            if (S < 3 && k > 0) row_loads(cs);  // (a 2-stage ring: the next row's slot may be unwritten)
            const double vri = vri_n, pri = pri_n, ycr = ycr_n;
            if (S >= 3 && k + 1 < nr) row_loads(cs + 1 == S ? 0 : cs + 1);
            mbar_wait(&bars[cs], cph);
            const float4 *row = reinterpret_cast<const float4 *>(smem + (size_t)cs * p.stage_bytes);
            float q0 = 0.f, q1 = 0.f, q2 = 0.f, q3 = 0.f;
#pragma unroll
            for (int kk = 0; kk < NV; ++kk) {
                const int idx = kk * T + tid;
                float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
                if (idx < p.n4) {
                    a = row[idx];
                    if (tail && idx == p.n4 - 1) {
                        if (tail < 2) a.y = 0.f;
                        if (tail < 3) a.z = 0.f;
                        a.w = 0.f;
                    }
                }
                q0 = fmaf(a.x, vr[kk].x, q0);
                q1 = fmaf(a.y, vr[kk].y, q1);
                q2 = fmaf(a.z, vr[kk].z, q2);
                q3 = fmaf(a.w, vr[kk].w, q3);
            }
            double part = (double)((q0 + q1) + (q2 + q3));
            if (tid < l) part -= pri * cv + vri * gv;  // - P_r c - V_r g (exact deflation)
            part = warp_sum(part);
            if (lane == 0) red[rb * NW + warp] = part;
            __syncthreads();
            if (tid == 0) {
                fence_proxy_async_smem();
                feed();
            }
            double y = 0.0;
            y = sum_warps<NW>(red + rb * NW, lane);
            rb ^= 1;
            if (++cs == S) {
                cs = 0;
                cph ^= 1u;
            }
            if (tid == 0) {
                __stcg(ynew + r, y);
                a_yy += y * y;
                a_vy += (ycr * inv) * y;
            }
            if (mx && tid < p.world)  // y_r to every rank (one thread per destination rank)
                ll_send(p.yx[tid] + (int64_t)(sxn & 1u) * p.n + r, sxn, y);
            if (tid < l) {
                a_vt += vri * y;
                a_pt += pri * y;
            }
        }
        if (mx) {
            xe = sxn;
            for (int r = 0; r < p.world; ++r) {
                ulonglong2 *dst = p.sx[r] + (((int64_t)(sxn & 1u) * p.world + p.rank) * G + b) * nqx;
                if (tid == 0) {
                    ll_send(dst + 0, sxn, a_yy);
                    ll_send(dst + 1, sxn, a_vy);
                }
                if (tid < l) {
                    ll_send(dst + 2 + tid, sxn, a_vt);
                    ll_send(dst + 2 + l + tid, sxn, a_pt);
                }
            }
            gx_totals(p.sx[p.rank] + (int64_t)(sxn & 1u) * p.world * G * nqx, p.world * G, nqx, sxn, totc, st);
            if (tid < 2) tot[tid] = totc[tid];
            for (int i = tid; i < l; i += T) {
                tot[2 + i] = totc[2 + i];
                tot[2 + kp + i] = totc[2 + l + i];
            }
            __syncthreads();
        } else {
            double *pr = my_part();
            if (tid == 0) {
                pr[0] = a_yy;
                pr[1] = a_vy;
            }
            if (tid < l) {
                pr[2 + tid] = a_vt;
                pr[2 + kp + tid] = a_pt;
            }
            __threadfence();
            grid_sync(p.gbar);
            grid_totals(2 + kp + l);
        }
        const int itn = it + 1;
        if (tid == 0) {
            const double nyn = sqrt(tot[0]);
            int done = 0, status = 0;
            double d = 0.0;
            if (!isfinite(nyn)) {
                status = -7;
                done = 2;
            } else if (nyn == 0.0) {  // rank exhausted (reading R14)
                status = 2;
                done = 2;
            } else {
                d = fabs(tot[1]) / nyn;  // |v0 . v1|
                if (p.fixed_T > 0) {
                    if (itn >= p.fixed_T) done = 1;
                } else if (d >= 1.0 - p.eps) {
                    done = 1;
                } else if (itn >= p.max_iter) {
                    done = 1;
                    status = 1;
                }
            }
            ny_s = (nyn > 0.0 && isfinite(nyn)) ? nyn : 1.0;
            done_s = done;
            if (b == 0) {
                st->it = itn;
                if (mx) st->xepoch = xe;
                if (done < 2) {
                    st->ny = nyn;
                    st->d = d;
                }
                if (done) {
                    st->status = status;
                    st->done = 1;
                    if (done == 2) st->stop = 1;
                }
            }
        }
        __syncthreads();
        it = itn;
        const int done = done_s;
        if (done) {
            if (mx) {  // the full final y (every rank's rows) into this rank's ybuf for the extraction
                const ulonglong2 *ya = p.yx[p.rank] + (int64_t)(xe & 1u) * p.n;
                double *yfin = p.ybuf + (int64_t)(it & 1) * p.ystride;
                const unsigned long long t0 = globaltimer_ns();
                for (int64_t j = (int64_t)b * T + tid; j < p.n; j += (int64_t)G * T)
                    yfin[j] = ll_recv(ya + j, xe, t0, st);
            }
            break;
        }
        make_cg(ny_s);
    }
    if (tid == 0 && nr > 0)  // drain the rows fed ahead
        for (int j = 0; j < S; ++j) {
            mbar_wait(&bars[cs], cph);
            if (++cs == S) {
                cs = 0;
                cph ^= 1u;
            }
        }
}

// Extraction of component l on the explicit path after one fused pass with c = 0 that
// stored t_r = (A v)_r (u_out), per-CTA partials of A^T t (ypart) and U^T t (wpart), and sum t^2:
// sigma = ||A v||, U[:, l] = t / sigma, P[:, l] = A^T t / sigma, Q[l, i] = Q[i, l] = (U^T t)_i /
// sigma (Q[l, l] = sum t^2 / sigma^2), S[l] = sigma, V[:, l] = v, stat[l].  Fixed-order sums.
struct GxParams {
    int64_t rows, n;
    int l, parts, ldu, ldp, ldv, ldq;
    const double *u_out, *ypart, *wpart, *sq_part;
    int64_t ypart_ld;
    int wpart_ld;
    const double *ybuf;
    int64_t ystride;
    float *U, *P;
    double *V, *S, *Q;
    CompStat *stat;
    LoopState *st;
};

// World > 1: the extraction pass's per-CTA partials reduced in CTA order into one rank vector
// out = [A_g^T u_g (n) | U_g^T u_g (l) | ||u_g||^2] for the cross-rank all-reduce; gram_ext_finish
// then runs on it with parts = 1.
__global__ void gx_reduce(const GxParams p, double *__restrict__ out, int64_t wofs) {
    griddep_launch();
    griddep_wait();
    const int64_t total = p.n + p.l + 1;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < total; j += (int64_t)gridDim.x * blockDim.x) {
        double a = 0.0;
        if (j < p.n) {
            for (int b = 0; b < p.parts; ++b) a += p.ypart[(int64_t)b * p.ypart_ld + j];
            out[j] = a;
        } else if (j < p.n + p.l) {
            const int i = (int)(j - p.n);
            for (int b = 0; b < p.parts; ++b) a += p.wpart[(int64_t)b * p.wpart_ld + i];
            out[wofs + i] = a;
        } else {
            for (int b = 0; b < p.parts; ++b) a += p.sq_part[b];
            out[wofs + p.l] = a;
        }
    }
}

__global__ void gram_ext_finish(const GxParams p) {
    __shared__ double sig_s;
    LoopState *st = p.st;
    griddep_launch();
    griddep_wait();
    if (st->stop) {
        if (blockIdx.x == 0 && threadIdx.x == 0 && !p.stat[p.l].valid) {
            p.stat[p.l].status = st->status;
            p.stat[p.l].it = st->it;
        }
        return;
    }
    if (threadIdx.x == 0) {
        double s2 = 0.0;
        for (int b = 0; b < p.parts; ++b) s2 += p.sq_part[b];
        sig_s = sqrt(s2);
    }
    __syncthreads();
    const double sg = sig_s;
    const bool ok = sg > 0.0 && isfinite(sg);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    const double *y = p.ybuf + (int64_t)(st->it & 1) * p.ystride;
    const double inv_ny = 1.0 / st->ny;
    if (ok) {
        for (int64_t r = tid; r < p.rows; r += nt) p.U[r * p.ldu + p.l] = (float)(p.u_out[r] / sg);
        for (int64_t j = tid; j < p.n; j += nt) {
            double a = 0.0;
            for (int b = 0; b < p.parts; ++b) a += p.ypart[(int64_t)b * p.ypart_ld + j];
            p.P[j * p.ldp + p.l] = (float)(a / sg);
            p.V[j * p.ldv + p.l] = y[j] * inv_ny;
        }
    }
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < p.l; i += blockDim.x) {
            double w = 0.0;
            for (int b = 0; b < p.parts; ++b) w += p.wpart[(int64_t)b * p.wpart_ld + i];
            const double q = ok ? w / sg : 0.0;
            p.Q[(int64_t)p.l * p.ldq + i] = q;
            p.Q[(int64_t)i * p.ldq + p.l] = q;
        }
        if (threadIdx.x == 0) {
            double s2 = 0.0;
            for (int b = 0; b < p.parts; ++b) s2 += p.sq_part[b];
            p.Q[(int64_t)p.l * p.ldq + p.l] = ok ? s2 / (sg * sg) : 0.0;
            CompStat cs = p.stat[p.l];
            cs.it = st->it;
            cs.d = st->d;
            cs.status = ok ? st->status : (isfinite(sg) ? 2 : -7);
            cs.sigma = sg;
            cs.valid = ok ? 1 : 0;
            p.stat[p.l] = cs;
            if (ok) p.S[p.l] = sg;
            else {  // no energy left (R14) or non-finite: later kernels are no-ops
                st->status = cs.status;
                st->stop = 1;
            }
        }
    }
}

}  // namespace tsvd
