// km_walk_body.cuh — the body of the walk kernel (km_walk.cu), compiled twice:
//   KM_WALK_NAME k_walk,       KM_SKIP1 0: every row of a batch is staged
//   KM_WALK_NAME k_walk_skip1, KM_SKIP1 1: the a/u of a batch are staged one batch ahead of its
//                               rows and only the rows that fail clause 1 are read (SURVEY §8(f)
//                               NEXT-2)
// A preprocessor switch (not a template parameter) keeps the KM_SKIP1 0 kernel's source, and so
// its register allocation, exactly the measured k_walk's.
template <int DP, bool CSMEM, int R, int NH, bool HSMEM>
__global__ void __launch_bounds__(walk_threads_dr(DP, R), 1)
KM_WALK_NAME(AssignParams p)
{
    extern __shared__ __align__(16) float smem[];
    const int k = p.k;
    float *sC = smem;                               // k*DP (CSMEM)
    const int k4 = (k + 3) & ~3;                   // sections stay 16-B aligned
    float *sF = smem + (CSMEM ? k * DP : 0);        // k
    float *sS = sF + k4;                            // k
    float *sH = sS + k4;                            // k x NH H rows (HSMEM)
    // per-warp staging of the next batch (cp.async): x rows, then a, then u
    constexpr int kRowsB = 32 * R;
    constexpr int kTab = walk_tab_cap(DP, HSMEM, KM_SKIP1);   // candidates of A's list kept in shared memory
    float *stg = sH + (HSMEM ? k * NH : 0) +
                 (threadIdx.x >> 5) * (walk_warp_floats(DP, R, KM_SKIP1) + walk_tab_floats(DP, HSMEM, KM_SKIP1));
    float *tabB = stg + walk_warp_floats(DP, R, KM_SKIP1);   // kTab / 2 pair blocks (2 DP floats each)
    float *tabC = tabB + kTab * DP;                           // |c'|^2 of the kTab candidates
    int tabA = -1;                                            // cluster whose table head is in tabB / tabC
#if KM_SKIP1
    // a second [a | u] slot: the a/u of the batch after the one whose rows are staged
    float *sAU2 = stg + kRowsB * (DP + 2) + 3 * kQueue;
#endif
    int *sQ = reinterpret_cast<int *>(stg + kRowsB * DP + 2 * kRowsB);   // mover queue: row, from, to
    if (CSMEM) {
        const float4 *src = reinterpret_cast<const float4 *>(p.Cneg);
        float4 *dst = reinterpret_cast<float4 *>(sC);
        for (int i = threadIdx.x; i < k * DP / 4; i += blockDim.x) dst[i] = src[i];
    }
    for (int i = threadIdx.x; i < k; i += blockDim.x) { sF[i] = p.f[i]; sS[i] = p.s[i]; }
    if (HSMEM)
        for (int i = threadIdx.x; i < k * NH; i += blockDim.x) sH[i] = p.WH[i];
    __syncthreads();
    CRow<CSMEM> Cn;
    if constexpr (CSMEM) {
        uint32_t b = (uint32_t)__cvta_generic_to_shared(sC);
        asm volatile("mov.u32 %0, %0;" : "+r"(b));
        Cn.base = b;
    } else {
        Cn.base = p.Cneg;
    }
    double *acc = p.acc + (int64_t)(blockIdx.x % p.nslab) * k * (DP + 1);
    const float eps = *p.eps;
    const int lane = threadIdx.x & 31;
    const int n = (int)p.n;                        // < 2^31 (kmeans_create enforces it)
    const int kp = p.wpad;                          // candidate rows per cluster block
    const int kcols = k - 1;
    constexpr int kChunk = kWalkChunk >= 2 * 32 * R ? kWalkChunk : 2 * 32 * R;   // rows per work claim (a multiple of 32 R)
    const int ib = p.wbits;                         // key index bits
    const uint32_t kmask = ~((1u << ib) - 1u);
    const float qtrunc = 1.f + __uint_as_float((uint32_t)(127 - 23 + ib) << 23) * 1.0001f;   // 1 + 2^(ib-23)
    // expansion-form error: |q~ - |x'-c'|^2| <= kappa (xx + cmax)
    const float kappa = 2.f * (2.f * DP + 20.f) * 5.9604645e-8f;
    constexpr int kRows = 32 * R;                   // rows per warp batch

    // per-lane counters: 32 bits (a lane's rows and walk steps stay far below 2^32; registers
    // are what bounds the resident warps), widened for the warp reduction at the end
    unsigned long long c_dists = 0;
    unsigned c_changed32 = 0, c_clause132 = 0, c_refined32 = 0, c_fb32 = 0, steps32 = 0;

    auto claim = [&]() -> int {
        int c = 0;
        if (lane == 0) c = atomicAdd(p.work, 1);
        c = __shfl_sync(kFull, c, 0);
        return c < (n + kChunk - 1) / kChunk ? c * kChunk : n;   // n: no more work
    };
#if KM_SKIP1
    // batch starts b0 (processed), b1 (rows staged), b2 (a/u staged); slot: the a/u slot of b0
    int sk_end = 0, sk_next = 0, b0 = n, b1 = n, b2 = n, slot = 0;
    auto next_batch = [&]() -> int {
        if (sk_next >= sk_end) {
            const int c = claim();
            if (c >= n) { sk_next = sk_end = n; return n; }
            sk_next = c;
            sk_end = min(c + kChunk, n);
        }
        const int b = sk_next;
        sk_next += kRows;
        return b;
    };
    auto au_slot = [&](int sl) -> float * { return sl ? sAU2 : stg + kRowsB * DP; };
    auto stage_au = [&](int r0, int sl) {          // a, u of rows [r0, r0 + 32 R) -> slot sl
        if (r0 < n) {
            float *ad = au_slot(sl);
#pragma unroll
            for (int c = lane; c < kRowsB / 2; c += 32) {
                if (c < kRowsB / 4) cp_async16(ad + 4 * c, p.a + r0 + 4 * c);
                else cp_async16(ad + kRowsB + 4 * (c - kRowsB / 4), p.u + r0 + 4 * (c - kRowsB / 4));
            }
        }
    };
    // x of the rows of batch r0 that fail clause 1 (their a/u are in slot sl): clause-1 rows are
    // never read ("no I/O requests are made")
    auto stage_x_live = [&](int r0, int sl) {
        if (r0 >= n) return;
        const float *ad = au_slot(sl);
        unsigned live[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int r = 32 * i + lane;
            const int av = __float_as_int(ad[r]);
            const bool v = r0 + r < n;
            const bool l = v && !(__fadd_ru(ad[kRowsB + r], sF[v ? av : 0]) <= sS[v ? av : 0]);
            live[i] = __ballot_sync(kFull, l);
        }
        const float4 *xs = reinterpret_cast<const float4 *>(p.X + (size_t)r0 * DP);
        float4 *xd = reinterpret_cast<float4 *>(stg);
#pragma unroll
        for (int c = lane; c < kRowsB * DP / 4; c += 32) {
            const int r = c / (DP / 4);
            unsigned w = live[0];
#pragma unroll
            for (int i = 1; i < R; ++i) w = (r >> 5) == i ? live[i] : w;
            if ((w >> (r & 31)) & 1u) cp_async16(xd + stg_swz<DP>(c), xs + c);
        }
    };
    int chunk_row = n;
#else
    // the work counter is fetched one chunk ahead by lane 0 and broadcast only when that chunk
    // starts, so the atomic's round trip overlaps a whole chunk of work
    constexpr int kBatches = kChunk / kRows;
    const int nchunks = (n + kChunk - 1) / kChunk;
    int chunk_row = claim();
    int ahead_c = 0;                                // lane 0: the claimed chunk after chunk_row
    if (lane == 0) ahead_c = atomicAdd(p.work, 1);
    int bt = 0;
#endif
    // stage rows [r0, r0 + 32 R) of X, a, u into this warp's buffer (16-B cp.async per lane)
    auto stage = [&](int r0) {
        const float4 *xs = reinterpret_cast<const float4 *>(p.X + (size_t)r0 * DP);
        float4 *xd = reinterpret_cast<float4 *>(stg);
#pragma unroll
        for (int c = lane; c < kRowsB * DP / 4; c += 32) cp_async16(xd + stg_swz<DP>(c), xs + c);
        float *ad = stg + kRowsB * DP;
#pragma unroll
        for (int c = lane; c < kRowsB / 2; c += 32) {
            if (c < kRowsB / 4) cp_async16(ad + 4 * c, p.a + r0 + 4 * c);
            else cp_async16(ad + kRowsB + 4 * (c - kRowsB / 4), p.u + r0 + 4 * (c - kRowsB / 4));
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
#if KM_SKIP1
    b0 = next_batch();
    b1 = b0 < n ? next_batch() : n;
    stage_au(b0, 0);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    stage_x_live(b0, 0);
    stage_au(b1, 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    chunk_row = b0;
#else
    if (chunk_row < n) stage(chunk_row);
#endif
    // mover queue (shared memory, kQueue entries per warp; mq warp-uniform)
    int mq = 0;
    auto flush_moves = [&]() {
        __syncwarp();
        // coordinate-parallel deltas: lanes = (mover, coordinate), 32 / DP movers per step, so
        // each fp64 RED instruction writes whole row segments of two slab rows; all the movers'
        // coordinates are loaded before the first RED (one L2 round trip per flush, not per step)
        {
            constexpr int G = DP >= 32 ? 1 : 32 / DP;           // movers per step
            constexpr int CL = DP >= 32 ? 32 : DP;              // lanes per mover
            constexpr int NS = 32 / G;                          // steps for 32 movers
            constexpr int NJ = DP >= 32 ? DP / 32 : 1;          // coordinates per lane per step
            const int nm = min(mq, 32);
            const int sub = lane / CL, co = lane % CL;
            float xv[NS][NJ];
#pragma unroll
            for (int st = 0; st < NS; ++st) {
                const int m = st * G + sub;
                const int mrow = m < nm ? sQ[m] : -1;
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj) {
                    const int j = jj * CL + co;
                    xv[st][jj] = (mrow >= 0 && j < p.d) ? __ldg(p.X + (size_t)mrow * DP + j) : 0.f;
                }
            }
#pragma unroll
            for (int st = 0; st < NS; ++st) {
                const int m = st * G + sub;
                if (st * G >= nm) break;
                const bool on = m < nm;
                const int mfrom = on ? sQ[kQueue + m] : 0, mto = on ? sQ[2 * kQueue + m] : 0;
                double *ra = acc + (int64_t)mfrom * (DP + 1), *rb = acc + (int64_t)mto * (DP + 1);
#pragma unroll
                for (int jj = 0; jj < NJ; ++jj) {
                    const int j = jj * CL + co;
                    if (on && j < p.d) {
                        atomicAdd(rb + j, (double)xv[st][jj]);
                        atomicAdd(ra + j, -(double)xv[st][jj]);
                    }
                }
                if (on && co == 0) {
                    atomicAdd(rb + DP, 1.0);
                    atomicAdd(ra + DP, -1.0);
                }
            }
        }
        __syncwarp();
        if (mq > 32) {   // keep the overflow (< 32 entries) at the front
            int e0 = 0, e1 = 0, e2 = 0;
            const bool mv = lane < mq - 32;
            if (mv) { e0 = sQ[32 + lane]; e1 = sQ[kQueue + 32 + lane]; e2 = sQ[2 * kQueue + 32 + lane]; }
            __syncwarp();
            if (mv) { sQ[lane] = e0; sQ[kQueue + lane] = e1; sQ[2 * kQueue + lane] = e2; }
            __syncwarp();
            mq -= 32;
        } else {
            mq = 0;
        }
    };

    while (chunk_row < n) {
#if KM_SKIP1
        const int row0 = b0;
#else
        const int row0 = chunk_row + bt * kRows;
#endif
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        float x[R][DP];
        int aold[R];
        float uu[R];
        bool valid[R], active[R];
        unsigned amask = 0;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int r = 32 * i + lane;
#pragma unroll
            for (int j = 0; j < DP; j += 4) {
                const float4 t = reinterpret_cast<const float4 *>(stg)[stg_swz<DP>(r * (DP / 4) + j / 4)];
                x[i][j] = t.x; x[i][j + 1] = t.y; x[i][j + 2] = t.z; x[i][j + 3] = t.w;
            }
#if KM_SKIP1
            const float *aus = au_slot(slot);
            aold[i] = __float_as_int(aus[r]);
            const float uold = aus[kRowsB + r];
#else
            aold[i] = __float_as_int(stg[kRowsB * DP + r]);
            const float uold = stg[kRowsB * DP + kRowsB + r];
#endif
            const int row = row0 + r;
            valid[i] = row < n;
            if (!valid[i]) aold[i] = 0;
            uu[i] = valid[i] ? __fadd_ru(uold, sF[aold[i]]) : 0.f;          // u += f(a)
            const bool c1 = valid[i] && uu[i] <= sS[aold[i]];                  // clause 1
            active[i] = valid[i] && !c1;
            c_clause132 += c1;
            amask |= __ballot_sync(kFull, active[i]) ? (1u << i) : 0u;
        }
        __syncwarp();
        // warp cluster A: the middle row's if active, else the first active row's
        auto pickA = [&]() -> int {
            int A;
            if constexpr (R <= 2) {
                const int mid = R == 1 ? 16 : 0;            // R = 2: lane 0 of the second half
                const unsigned m_mid = __ballot_sync(kFull, active[R - 1]);
                if ((m_mid >> mid) & 1u) A = __shfl_sync(kFull, aold[R - 1], mid);
                else {
                    const unsigned m0 = __ballot_sync(kFull, active[0]);
                    A = m0 ? __shfl_sync(kFull, aold[0], __ffs(m0) - 1) : __shfl_sync(kFull, aold[R - 1], __ffs(m_mid) - 1);
                }
            } else {                                       // row 32 (R / 2), else the first active row
                const unsigned m_mid = __ballot_sync(kFull, active[R / 2]);
                if (m_mid & 1u) A = __shfl_sync(kFull, aold[R / 2], 0);
                else {
                    int fi = 0, fl = 0;
#pragma unroll
                    for (int i = R - 1; i >= 0; --i) {
                        const unsigned m = __ballot_sync(kFull, active[i]);
                        if (m) { fi = i; fl = __ffs(m) - 1; }
                    }
                    int av = aold[0];
#pragma unroll
                    for (int i = 1; i < R; ++i) av = fi == i ? aold[i] : av;
                    A = __shfl_sync(kFull, av, fl);
                }
            }
            return A;
        };
#if KM_WALK_TAB
        // chosen before the next batch is staged, so that the table copy's group precedes the rows'
        int A = 0;
        if (amask) A = pickA();
#endif
        [[maybe_unused]] bool staged_next = false;
#if KM_WALK_TAB
        if constexpr (kTab > 0) {
            // head of A's candidate table -> this warp's shared-memory copy (its own cp.async group,
            // committed before the next batch's rows so that the walk waits for it alone)
            if (amask && A != tabA) {
                tabA = A;
                const int capn = min(kTab, kp);
                const float4 *src = p.Wblk + (int64_t)A * (kp / 2) * walk_pair_f4(DP);
                float4 *dst = reinterpret_cast<float4 *>(tabB);
                for (int c = lane; c < (capn / 2) * (DP / 2); c += 32) cp_async16(dst + c, src + c);
                if (lane < capn / 2) cp_async8(tabC + 2 * lane, p.Wcc + (int64_t)A * kp + 2 * lane);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
#endif
#if KM_SKIP1
        // rows of b1 that fail clause 1 (their a/u are here), a/u of b2 into b0's slot
        b2 = b1 < n ? next_batch() : n;
        stage_x_live(b1, slot ^ 1);
        stage_au(b2, slot);
        asm volatile("cp.async.commit_group;" ::: "memory");
        b0 = b1;
        b1 = b2;
        slot ^= 1;
        chunk_row = b0;                             // loop condition
#else
        if (++bt == kBatches || chunk_row + bt * kRows >= n) {
            bt = 0;
            const int c = __shfl_sync(kFull, ahead_c, 0);
            chunk_row = c < nchunks ? c * kChunk : n;
            if (lane == 0 && chunk_row < n) ahead_c = atomicAdd(p.work, 1);
        }
        if (chunk_row < n) { stage(chunk_row + bt * kRows); staged_next = true; }
#endif

        int anew[R];
        float unew[R], ut[R];
        bool defer[R];
#pragma unroll
        for (int i = 0; i < R; ++i) { anew[i] = aold[i]; unew[i] = uu[i]; ut[i] = 0.f; defer[i] = false; }
        if (amask) {
#if !KM_WALK_TAB
            const int A = pickA();
#endif
            float4 cA[DP / 4];
#pragma unroll
            for (int j = 0; j < DP / 4; ++j) cA[j] = Cn.ld(A, DP, 4 * j);
            float xc[R][DP], xx[R], lo[R], T[R];
            int pl[R];
            bool misfit[R];
            int pm = 0;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                // x' = x - C^[A] (direct form's arithmetic), xx = |x'|^2
                float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
                for (int j = 0; j < DP; j += 4) {
                    const float4 c = cA[j / 4];
                    const float2 t0 = add2(make_float2(x[i][j], x[i][j + 1]), make_float2(c.x, c.y));
                    const float2 t1 = add2(make_float2(x[i][j + 2], x[i][j + 3]), make_float2(c.z, c.w));
                    xc[i][j] = t0.x; xc[i][j + 1] = t0.y; xc[i][j + 2] = t1.x; xc[i][j + 3] = t1.y;
                    a0 = fma2(t0, t0, a0);
                    a1 = fma2(t1, t1, a1);
                }
                const float2 s2 = add2(a0, a1);
                xx[i] = s2.x + s2.y;
                misfit[i] = active[i] && aold[i] != A;
                lo[i] = 0.f; T[i] = 0.f; pl[i] = 0;
                if (active[i]) {
                    if (!misfit[i]) {
                        ut[i] = upper_d(xx[i], p.g_up, eps);
                        lo[i] = lower_d(xx[i], p.g_dn, eps);
                        T[i] = ut[i];
                    } else {
                        const float qo = dist2<DP, CSMEM>(x[i], Cn, aold[i]);
                        ut[i] = upper_d(qo, p.g_up, eps);
                        lo[i] = lower_d(qo, p.g_dn, eps);
                        T[i] = __fmul_ru(__fadd_ru(ut[i], upper_d(xx[i], p.g_up, eps)), 0.5f);
                    }
                    if constexpr (HSMEM) pl[i] = count_below_s<NH>(sH + A * NH, T[i]);
                    else pl[i] = count_below_u<NH>(p.WH + (int64_t)A * NH, T[i]);
                }
                pm = max(pm, pl[i]);
            }
            pm = __reduce_max_sync(kFull, pm);
            // the walk: candidates j < pm of A's list, two per step, keys (q & kmask) | j
            const float4 *blk = p.Wblk + (int64_t)A * (kp / 2) * walk_pair_f4(DP);
            const float2 *ccA = reinterpret_cast<const float2 *>(p.Wcc + (int64_t)A * kp);
            // prefix max of |c'|^2 over the rows the walk evaluates (bounds the error of every
            // key); loaded before the walk so its latency overlaps it
            const float cmax = pm > 0 ? __ldg(p.Wmeta + (int64_t)A * kp + ((pm + 1) & ~1) - 1).x : 0.f;
            int m1[R], m2[R];
#pragma unroll
            for (int i = 0; i < R; ++i) { m1[i] = 0x7fffffff; m2[i] = 0x7fffffff; }
            // one step: candidates (j, j + 1); TB: from this warp's shared-memory table head
            auto step = [&](const int j, auto TBt) {
                constexpr bool TB = decltype(TBt)::value;
                const float4 *tb4 = reinterpret_cast<const float4 *>(tabB) + (j >> 1) * (DP / 2);
                const float4 *gb4 = blk + (int64_t)(j >> 1) * walk_pair_f4(DP);
                float2 cc;
                if constexpr (TB) cc = reinterpret_cast<const float2 *>(tabC)[j >> 1];
                else cc = __ldg(ccA + (j >> 1));
                float2 q[R];
                if constexpr (DP >= 32 && KM_WALK_HALVES && HSMEM) {   // (measured: +2 % on C4, -3.5 % on C5)
                    // wide rows: the pair block is consumed in two halves of DP/2 coordinates, so
                    // only DP/4 float4 of it are live at once (registers bound the resident warps)
#pragma unroll
                    for (int i = 0; i < R; ++i) q[i] = add2s(xx[i], cc);
#if KM_WALK_CHAINS2
                    float2 qb[R];
#pragma unroll
                    for (int i = 0; i < R; ++i) qb[i] = make_float2(0.f, 0.f);
#endif
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float4 v[DP / 4];
#pragma unroll
                        for (int e = 0; e < DP / 4; e += 2) {
                            if constexpr (TB) { v[e] = tb4[h * (DP / 4) + e]; v[e + 1] = tb4[h * (DP / 4) + e + 1]; }
                            else ldg256(gb4 + h * (DP / 4) + e, v[e], v[e + 1]);
                        }
#if KM_WALK_CHAINS2
                        // two accumulation chains per row (even / odd coordinates): with 3 warps per
                        // sub-partition the FFMA2 dependency latency is the top stall once the
                        // candidate loads come from shared memory; the error bound kappa holds for
                        // any summation order
#pragma unroll
                        for (int i = 0; i < R; ++i)
#pragma unroll
                            for (int e = 0; e < DP / 4; ++e) {
                                q[i] = fma2s(xc[i][h * (DP / 2) + 2 * e], make_float2(v[e].x, v[e].y), q[i]);
                                qb[i] = fma2s(xc[i][h * (DP / 2) + 2 * e + 1], make_float2(v[e].z, v[e].w), qb[i]);
                            }
#else
#pragma unroll
                        for (int i = 0; i < R; ++i)
#pragma unroll
                            for (int e = 0; e < DP / 4; ++e) {
                                q[i] = fma2s(xc[i][h * (DP / 2) + 2 * e], make_float2(v[e].x, v[e].y), q[i]);
                                q[i] = fma2s(xc[i][h * (DP / 2) + 2 * e + 1], make_float2(v[e].z, v[e].w), q[i]);
                            }
#endif
                    }
#if KM_WALK_CHAINS2
#pragma unroll
                    for (int i = 0; i < R; ++i) q[i] = add2(q[i], qb[i]);
#endif
                } else {
                    float4 v[DP / 2];
#pragma unroll
                    for (int e = 0; e < DP / 2; e += 2) {    // 32-byte loads: half the L1 requests
                        if constexpr (TB) { v[e] = tb4[e]; v[e + 1] = tb4[e + 1]; }
                        else ldg256(gb4 + e, v[e], v[e + 1]);
                    }
#pragma unroll
                    for (int i = 0; i < R; ++i) q[i] = q_pair<DP>(xc[i], xx[i], cc, v);
                }
#pragma unroll
                for (int i = 0; i < R; ++i) {
                    int k0, k1;
                    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(k0) : "r"(__float_as_uint(q[i].x)), "r"(kmask), "r"(j));
                    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(k1) : "r"(__float_as_uint(q[i].y)), "r"(kmask), "r"(j + 1));
                    const int lo2 = min(k0, k1), hi2 = max(k0, k1);
                    m2[i] = min(min(max(m1[i], lo2), m2[i]), hi2);
                    m1[i] = min(m1[i], lo2);
                }
            };
            {
                int j = 0;
                if constexpr (kTab > 0) {
                    // the table head of A landed (its group precedes the next batch's rows)
                    if (staged_next) asm volatile("cp.async.wait_group 1;" ::: "memory");
                    else asm volatile("cp.async.wait_group 0;" ::: "memory");
                    __syncwarp();
                    const int je = min(pm, min(kTab, kp));
                    for (; j < je; j += 2) step(j, km_true{});
                }
                for (; j < pm; j += 2) step(j, km_false{});
            }
            steps32 += (unsigned)pm;
            const float2 *mA = p.Wmeta + (int64_t)A * kp;
#pragma unroll
            for (int i = 0; i < R; ++i) {
                if (!active[i]) continue;
                // rigorous decision (same procedure as the tensor-core epilogue).  Fast paths in
                // the squared domain: a key value v with v > thr = (u_t + epsr)^2 + E has a lower
                // distance bound above u_t, the upper bound of the own cluster's distance.
                const float E = __fmul_ru(kappa, __fadd_ru(xx[i], cmax));
                const float epsr = __fadd_ru(eps, __fmul_ru(1.2e-7f, __fadd_ru(sqrt_up(xx[i]), sqrt_up(cmax))));
                const float ue = __fadd_ru(ut[i], epsr);
                const float thr = __fadd_ru(__fmul_ru(ue, ue), E);
                const float v1 = m1[i] == 0x7fffffff ? INFINITY : __int_as_float(m1[i] & kmask);
                const float v2 = m2[i] == 0x7fffffff ? INFINITY : __int_as_float(m2[i] & kmask);
                bool fallback = false, stay;
                if (!misfit[i]) {
                    stay = v1 > thr;
                } else {
                    // misfit: stays if A is farther than u_t and every candidate but the own
                    // cluster's column is: either all keys exceed thr, or only the best does not
                    // and the best is the own cluster (then any other key is >= m2 > thr)
                    const bool a_far = __fmul_rd(sqrt_dn(xx[i]), p.g_dn) > __fadd_ru(ut[i], eps);
                    stay = a_far && (v1 > thr ||
                                     (v2 > thr && __float_as_int(__ldg(&mA[m1[i] & ~kmask].y)) == aold[i]));
                }
                if (stay) {
                    unew[i] = ut[i];
                } else if (!misfit[i]) {
                    // moves to the best candidate if its interval is clear of the own cluster's
                    // and of every other candidate's (>= m2)
                    const float U1 = __fadd_ru(sqrt_up(__fadd_ru(__fmul_ru(fmaxf(v1, 0.f), qtrunc), E)), epsr);
                    const float L2 = v2 == INFINITY ? INFINITY
                                                    : fmaxf(0.f, __fsub_rd(sqrt_dn(fmaxf(__fsub_rd(v2, E), 0.f)), epsr));
                    if (U1 < fminf(lo[i], L2)) {
                        anew[i] = __float_as_int(__ldg(&mA[m1[i] & ~kmask].y));
                        unew[i] = U1;
                    } else {
                        fallback = true;
                    }
                } else {
                    auto U_of = [&](int key) {
                        const float v = fmaxf(__int_as_float(key & kmask), 0.f);
                        return __fadd_ru(sqrt_up(__fadd_ru(__fmul_ru(v, qtrunc), E)), epsr);
                    };
                    auto L_of = [&](int key) {
                        if (key == 0x7fffffff) return INFINITY;
                        const float v = __int_as_float(key & kmask);
                        return fmaxf(0.f, __fsub_rd(sqrt_dn(fmaxf(__fsub_rd(v, E), 0.f)), epsr));
                    };
                    const int cc1 = m1[i] != 0x7fffffff ? __float_as_int(__ldg(&mA[m1[i] & ~kmask].y)) : -1;
                    const int cc2 = m2[i] != 0x7fffffff ? __float_as_int(__ldg(&mA[m2[i] & ~kmask].y)) : -1;
                    float Uo = ut[i], Lo = lo[i], Ui = INFINITY, Li = INFINITY, Lother = INFINITY;
                    int ci = -1;
                    if (cc1 == aold[i]) {      // own cluster is the best candidate: merge
                        Uo = fminf(Uo, U_of(m1[i])); Lo = fmaxf(Lo, L_of(m1[i]));
                        ci = cc2;
                        if (ci >= 0) { Ui = U_of(m2[i]); Li = L_of(m2[i]); Lother = -1.f; }   // third unknown
                    } else {
                        ci = cc1;
                        if (ci >= 0) { Ui = U_of(m1[i]); Li = L_of(m1[i]); }
                        Lother = L_of(m2[i]);
                    }
                    const float UA = upper_d(xx[i], p.g_up, eps), LA = lower_d(xx[i], p.g_dn, eps);
                    if (Uo < fminf(Li, LA)) {
                        unew[i] = Uo;
                    } else if (UA < fminf(Lo, Li)) {
                        anew[i] = A; unew[i] = UA;
                    } else if (ci >= 0 && Ui < fminf(fminf(Lo, LA), Lother)) {
                        anew[i] = ci; unew[i] = Ui;
                    } else {
                        fallback = true;
                    }
                }
                if (fallback) {
                    ++c_fb32;
                    const uint64_t *nl = p.NL + (int64_t)aold[i] * p.ks;
                    float xr[DP];
                    {
                        const float4 *src = reinterpret_cast<const float4 *>(p.X + (size_t)(row0 + 32 * i + lane) * DP);
#pragma unroll
                        for (int j = 0; j < DP / 4; ++j) {
                            const float4 t = __ldg(src + j);
                            xr[4 * j] = t.x; xr[4 * j + 1] = t.y; xr[4 * j + 2] = t.z; xr[4 * j + 3] = t.w;
                        }
                    }
                    float bq = dist2<DP, CSMEM>(xr, Cn, aold[i]), q2 = INFINITY;
                    int bc = aold[i];
                    for (int j = 0; j < kcols; ++j) {
                        const uint64_t key = __ldg(nl + j);
                        if (!(key_h(key) < ut[i])) break;
                        const int c = key_c(key);
                        const float q = dist2<DP, CSMEM>(xr, Cn, c);
                        q2 = fminf(q2, fmaxf(q, bq));
                        bc = q < bq ? c : bc;
                        bq = fminf(q, bq);
                    }
                    const float ub = upper_d(bq, p.g_up, eps);
                    if (q2 < INFINITY && lower_d(q2, p.g_dn, eps) <= ub) {
                        anew[i] = refine64(p.X + (size_t)(row0 + 32 * i + lane) * DP, p.d, p.C64, k, aold[i], nl, ut[i], &unew[i]);
                        ++c_refined32;
                    } else {
                        anew[i] = bc;
                        unew[i] = ub;
                    }
                }
                // MTI distance count 1 + #{c : H[a][c] < u_t}; misfit rows: deferred
                if (!misfit[i]) {
                    c_dists += (unsigned long long)(1 + pl[i]);
                } else if constexpr (HSMEM) {      // own list's H row is in shared memory
                    c_dists += (unsigned long long)(1 + count_below_s<NH>(sH + aold[i] * NH, ut[i]));
                } else {
                    defer[i] = true;                 // counted by k_mti_count
                }
            }
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int rb = row0 + 32 * i;
            if constexpr (!HSMEM) {   // deferred counts: per 32-row group: defer[rb + i], dcount[rb / 32]
                const unsigned dm = __ballot_sync(kFull, defer[i]);
                if (defer[i])
                    p.defer[rb + __popc(dm & ((1u << lane) - 1u))] =
                        ((unsigned long long)(uint32_t)aold[i] << 32) | __float_as_uint(ut[i]);
                if (lane == 0 && rb < n) p.dcount[rb / 32] = __popc(dm);
            }
            if (valid[i]) {
                if (anew[i] != aold[i]) p.a[rb + lane] = anew[i];
                p.u[rb + lane] = unew[i];
            }
            // S3 as a delta (B5): movers are queued in shared memory and their fp64
            // deltas applied 32 at a time, so the REDs run with full warps
            {
                const bool mv = valid[i] && anew[i] != aold[i];
                const unsigned mm = __ballot_sync(kFull, mv);
                if (mm) {
                    c_changed32 += mv;
                    if (mv) {
                        const int slot = mq + __popc(mm & ((1u << lane) - 1u));
                        sQ[slot] = rb + lane; sQ[kQueue + slot] = aold[i]; sQ[2 * kQueue + slot] = anew[i];
                    }
                    mq += __popc(mm);
                    if (mq >= 32) flush_moves();
                }
            }
        }
    }
    flush_moves();
    unsigned long long c_changed = c_changed32, c_clause1 = c_clause132, c_refined = c_refined32,
                       c_fb = c_fb32, steps = steps32;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        c_changed += __shfl_xor_sync(kFull, c_changed, o);
        c_dists += __shfl_xor_sync(kFull, c_dists, o);
        c_clause1 += __shfl_xor_sync(kFull, c_clause1, o);
        c_refined += __shfl_xor_sync(kFull, c_refined, o);
        c_fb += __shfl_xor_sync(kFull, c_fb, o);
    }
    if (lane == 0) {
        if (c_changed) atomicAdd(p.counters + 0, c_changed);
        if (c_dists) atomicAdd(p.counters + 1, c_dists);
        if (c_clause1) atomicAdd(p.counters + 2, c_clause1);
        if (c_refined) atomicAdd(p.counters + 3, c_refined);
        if (steps) atomicAdd(p.counters + 4, steps);
        if (c_fb) atomicAdd(p.counters + 5, c_fb);
    }
}
