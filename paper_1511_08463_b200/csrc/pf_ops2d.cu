// pf_ops2d.cu -- launchers of the matrix-free P1 operators on structured 2D triangle meshes (sm_100a, fp64).
// (engine and operator structs: pf_strip2d.cuh)
#include "pf_strip2d.cuh"

namespace pf {

// ---- launch plumbing ------------------------------------------------------------------------
// algorithmic bytes per vertex (read every input once, write every output once) by kind;
// element arrays (kappa) are charged 8 B per element.
static double alg_bytes(const Ctx* c, int kind, int nvec_r, int nvec_w) {
    const double V = (double)c->g.nv, T = (double)c->n_el;
    switch (kind) {
        case K_KUU: return V * (16 + 8 + 16);                 // x, alpha -> y
        case K_KUU_CG: return V * (16 + 16 + 8 + 16 + 16);    // z, p_in, alpha -> p_out, q
        case K_KUU_DIAG: return V * (8 + 16);
        case K_KAPPA: return V * (16 + 8) + T * 8;            // u -> c, kappa
        case K_KAA: return V * (8 + 8) + T * 8;               // x, kappa -> y
        case K_KAA_CG: return V * (8 + 8 + 8 + 8 + 1) + T * 8;
        case K_KAA_DIAG: return V * 8 + T * 8;
        case K_KAA_TRIAL: return V * (8 + 8 + 8 + 8 + 8 + 8) + T * 8;  // x, d, lb, c -> trial, F
        case K_PHYS: return V * (16 + 8 + 8) + V * 8.0 * nvec_w;
        case K_RHS: return V * (8 + 16);
        case K_KUA: return V * (16 + 8 + 8 + 16);
        case K_KAU: return V * (16 + 8 + 16 + 8);
        case K_JAC: return V * (16 + 8 + 16 + 8 + 16 + 8);
        default: return V * 8.0 * (nvec_r + nvec_w);
    }
}

// algorithmic bytes of one persistent damage-PCG iteration: the fused Kaa strip pass + the
// vector pass (x, p, r, q, dinv -> x, r, z)
double pcg_kaa_iter_bytes(const Ctx* c) {
    if (c->dim == 3) return 33.0 * c->g3.nv + 8.0 * c->n_el + 8.0 * 8.0 * (double)c->g3.nv;
    return alg_bytes(c, K_KAA_CG, 0, 0) + 8.0 * 8.0 * (double)c->g.nv;
}

template <class Op, int PAT>
static constexpr int strip_smem() {
    return (kBlock / 32) * Op::pd(PAT) * (Op::sv(PAT) + Op::sc(PAT)) * 256;
}

template <class Op, int PAT>
static cudaError_t launch_pat(const Geo2& g, const Op& op, int nb, cudaStream_t st) {
    constexpr int smem = strip_smem<Op, PAT>();
    static_assert(smem <= 227 * 1024, "strip stage ring exceeds shared memory");
    static std::atomic<bool> attr[kMaxDev];  // one-time opt-in above 48 KB per instantiation and device
    const int dv = cur_dev();
    if (!attr[dv].load()) {
        cudaError_t e = cudaFuncSetAttribute(k_strip2d<Op, PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr[dv] = true;
    }
    k_strip2d<Op, PAT><<<nb, kBlock, smem, st>>>(g, op);
    return cudaSuccess;
}

template <class Op>
static int run_strip(Ctx* c, Op op, cudaStream_t st, int kind = K_VEC, int nw = 0, double bytes = -1.0) {
    const Geo2& g = c->g;
    if constexpr (is_v2<Op>::value) {  // the TMA engine where the operator has it (pf_strip2.cu)
        static const unsigned kinds = getenv("PF_STRIP2_KINDS") ? (unsigned)strtoul(getenv("PF_STRIP2_KINDS"), nullptr, 0) : ~0u;
        if (c->strip2 && ((kinds >> kind) & 1u)) {
            const int rc = run_strip2(c, op, st, kind, bytes >= 0.0 ? bytes : alg_bytes(c, kind, 0, nw));
            if (rc >= 0) return rc;
        }
    }
    const int nb = strip_blocks(g);
    if (nb > kMaxBlocksRed) return set_error(c, PF_EINVAL, "grid too large for reduction buffer");
    const int slot = prof_begin(c, st);
    cudaError_t e;
    switch (g.pattern) {
        case PF_UNION_JACK: e = launch_pat<Op, PF_UNION_JACK>(g, op, nb, st); break;
        case PF_RIGHT: e = launch_pat<Op, PF_RIGHT>(g, op, nb, st); break;
        default: e = launch_pat<Op, PF_CROSSED>(g, op, nb, st); break;
    }
    if (e != cudaSuccess) return check_cuda(c, e, "strip kernel attribute");
    prof_end(c, st, slot, kind, bytes >= 0.0 ? bytes : alg_bytes(c, kind, 0, nw));
    c->launches++;
    return check_cuda(c, cudaGetLastError(), "strip kernel launch");
}

static RedBuf redbuf(Ctx* c) { return RedBuf{c->partials, c->tickets, c->scal}; }

int launch_Kuu(Ctx* c, const double* alpha, const double* x, double* y, int bcmode, cudaStream_t st) {
    if (c->dim == 3) return launch3_Kuu(c, alpha, x, y, bcmode, st);
    OpKuu<false> op{alpha, x, nullptr, nullptr, y, bcmode, c->scal, redbuf(c), 0.0};
    return run_strip(c, op, st, K_KUU);
}
int launch_Kuu_smooth(Ctx* c, int epi, const double* alpha, const double* d, const GmgEpi& e, cudaStream_t st) {
    if (c->dim == 3) return set_error(c, PF_EINVAL, "GMG smoother epilogues are 2D");
    const double V = (double)c->g.nv;
    double extra = 0.0;
    switch (epi) {
        case EPI_CHEB:
        case EPI_CHEB_ADDD: {
            OpKuu<false, EPI_CHEB> op{alpha, d, nullptr, nullptr, nullptr, PF_BC_ELIMINATE, c->scal, redbuf(c), 0.0, e};
            extra = 32 + 32 + 16 + 32 + (e.rz_first >= 0 ? 16 : 0);  // Dinv, res, dnext, x, [r]
            if (epi == EPI_CHEB) return run_strip(c, op, st, K_GMG, 0, V * (40 + extra));
            OpKuu<false, EPI_CHEB_ADDD> op2{alpha, d, nullptr, nullptr, nullptr, PF_BC_ELIMINATE, c->scal, redbuf(c), 0.0, e};
            return run_strip(c, op2, st, K_GMG, 0, V * (40 + extra));
        }
        case EPI_RESID: {
            OpKuu<false, EPI_RESID> op{alpha, d, nullptr, nullptr, nullptr, PF_BC_ELIMINATE, c->scal, redbuf(c), 0.0, e};
            return run_strip(c, op, st, K_GMG, 0, V * (40 - 16 + 32));  // b -> r instead of y
        }
        case EPI_RESID_CHEB0: {
            OpKuu<false, EPI_RESID_CHEB0> op{alpha, d, nullptr, nullptr, nullptr, PF_BC_ELIMINATE, c->scal, redbuf(c), 0.0, e};
            return run_strip(c, op, st, K_GMG, 0, V * (40 - 16 + 16 + 32 + 32));  // b, Dinv -> res, d0
        }
        default:
            return set_error(c, PF_EINVAL, "unknown smoother epilogue");
    }
}
int launch_Kuu_cgA(Ctx* c, const double* alpha, const double* z, const double* p_in, double* p_out,
                   double* q, cudaStream_t st) {
    if (c->dim == 3) return launch3_Kuu_cgA(c, alpha, z, p_in, p_out, q, st);
    OpKuu<true> op{alpha, z, p_in, p_out, q, PF_BC_ELIMINATE, c->scal, redbuf(c), 0.0};
    return run_strip(c, op, st, K_KUU_CG);
}
int launch_Kuu_diag(Ctx* c, const double* alpha, double* dinv, cudaStream_t st) {
    if (c->dim == 3) return launch3_Kuu_diag(c, alpha, dinv, st);
    OpKuuDiag op;
    op.alpha = alpha;
    op.dinv = dinv;
    return run_strip(c, op, st, K_KUU_DIAG);
}
int launch_kappa(Ctx* c, const double* u, const double* alpha, double* kappa, double* cvec,
                 cudaStream_t st) {
    if (c->dim == 3) return launch3_kappa(c, u, kappa, cvec, st);
    (void)alpha;
    OpKappa op;
    op.u = u; op.kappa = kappa; op.cvec = cvec;
    return run_strip(c, op, st, K_KAPPA);
}
int launch_Kaa(Ctx* c, const double* kappa, const double* x, double* y, const unsigned char* act,
               cudaStream_t st) {
    if (c->dim == 3) return launch3_Kaa(c, kappa, x, y, act, st);
    if (act) {
        OpKaa<false, true> op{kappa, x, nullptr, nullptr, y, act, c->scal, redbuf(c), 0.0};
        return run_strip(c, op, st, K_KAA);
    }
    OpKaa<false, false> op{kappa, x, nullptr, nullptr, y, nullptr, c->scal, redbuf(c), 0.0};
    return run_strip(c, op, st, K_KAA);
}
// one fused Chebyshev step of the masked C block (2D): K d feeds r, d' and x at the owner (KaaCheb)
int launch_Kaa_cheb(Ctx* c, const double* kappa, const double* d, const unsigned char* act, double* r,
                    double* dnext, double* x, const double* dinv, const double* tab, int k, cudaStream_t st) {
    if (c->dim == 3) return set_error(c, PF_EINVAL, "launch_Kaa_cheb is 2D");
    OpKaa<false, true, true> op{kappa, d, nullptr, nullptr, nullptr, act, c->scal, redbuf(c), 0.0};
    op.ch = KaaCheb{r, dnext, x, dinv, tab, k};
    return run_strip(c, op, st, K_KAA);
}
int launch_Kaa_cgA(Ctx* c, const double* kappa, const double* z, const double* p_in, double* p_out,
                   double* q, const unsigned char* act, cudaStream_t st) {
    if (c->dim == 3) return launch3_Kaa_cgA(c, kappa, z, p_in, p_out, q, act, st);
    if (act) {
        OpKaa<true, true> op{kappa, z, p_in, p_out, q, act, c->scal, redbuf(c), 0.0};
        return run_strip(c, op, st, K_KAA_CG);
    }
    OpKaa<true, false> op{kappa, z, p_in, p_out, q, nullptr, c->scal, redbuf(c), 0.0};
    return run_strip(c, op, st, K_KAA_CG);
}
// ---- persistent damage PCG ----------------------------------------------------------------------
// The whole Jacobi-PCG loop on the (masked) damage block in one cooperative launch
// (linalg.py:106-152 as restated by pcg_run, kind 1): per iteration one strip pass (p = z + beta p,
// q = Kaa p, p.q) and one vector pass (x += gamma p, r -= gamma q, z = D^-1 r, r.r, r.z), separated
// by grid barriers; every CTA sums the per-CTA partials in the same fixed order, so all CTAs take
// the same scalar decisions and the result is deterministic.  The strips are "virtual blocks"
// distributed over the resident CTAs.  Replaces 2 dependent launches per iteration (each
// latency-bound on a 4-17 MB problem) and the per-pair graph overhead.
// Free strips of the masked solve (as k_tile_flags3, pf_ops3d.cu): on an active row the masked system
// is the identity with a zero right-hand side, so x, r, z, p and q stay 0 there.  A warp's strip
// (30 output columns x S rows) whose input box -- outputs +-1, and for the crossed pattern the
// centres of the cells it touches -- holds active vertices only writes zeros and adds 0 to p.q.
// The loop visits the flagged strips only (ascending list), the vector pass skips active rows.
__global__ void __launch_bounds__(256) k_tile_flags2(const Geo2 g, const unsigned char* __restrict__ act, int ntile,
                                                     unsigned char* __restrict__ flag) {
    const int t = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (t >= ntile) return;
    const int wj = t % g.nwj, wi = t / g.nwj;
    const int j = wj * kLanesOut - 1 + lane;
    const int i0 = max(wi * g.S - 1, 0), i1 = min(wi * g.S + g.S, g.nx);
    bool f = false;
    if (j >= 0 && j <= g.ny)
        for (int i = i0; i <= i1; ++i) f |= act[vid(g, i, j)] == 0;
    if (g.pattern == PF_CROSSED && j >= 0 && j < g.ny && lane < 31)
        for (int ci = i0; ci < i1; ++ci) f |= act[ctr(g, ci, j)] == 0;
    f = __any_sync(PF_FULL, f);
    if (lane == 0) flag[t] = f ? 1 : 0;
}

template <bool MASKED, int PAT, int NT>
__global__ void __launch_bounds__(NT, 512 / NT) k_pcg_kaa(const Geo2 g, OpKaa<true, MASKED> op, int nvb, long long n,
                                                        double* x, double* r, double* z, double* p0, double* p1,
                                                        double* q, const double* dinv, double* s, double* partials,
                                                        unsigned int* bar, const int* __restrict__ tiles) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (!(s[S_DONE] == 0.0 && s[S_FAIL] == 0.0)) return;  // uniform
    // flagged strips (see k_tile_flags2); the list pays when at most half of the strips are flagged --
    // otherwise (AT2: nearly every vertex is free) the loop runs exactly as without it
    const int nall = g.nwj * g.nstrips;
    const int nfree = tiles ? tiles[0] : nall;
    const bool sparse = MASKED && tiles && 2 * nfree <= nall;
    const int wpb = NT / 32, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double target = s[S_TARGET], maxit = s[S_MAXIT];
    double rz = s[S_RZ], beta = s[S_BETA], rn = s[S_RNORM], pap = 0.0, gm = 0.0;
    long long it = (long long)s[S_ITER];
    double done = 0.0, fail = 0.0;
    const long long tid = blockIdx.x * (long long)NT + threadIdx.x, nth = (long long)gridDim.x * NT;
    for (;;) {
        double* pin = (it & 1) ? p1 : p0;
        double* pout = (it & 1) ? p0 : p1;
        op.x = z;
        op.pin = pin;
        op.pout = pout;
        op.y = q;
        op.acc = 0.0;
        op.use_breg = 1;
        op.breg = it > 0 ? beta : 0.0;
        // warps are independent in this engine: each takes (flagged) strips in turn
        const int nw = sparse ? nfree : nvb * wpb;
        for (int m = blockIdx.x * wpb + warp; m < nw; m += gridDim.x * wpb)
            strip_pass<OpKaa<true, MASKED>, PAT>(g, op, smem, sparse ? tiles[1 + m] : m);
        block_partials(&op.acc, 1, partials, 0);
        grid_sync(bar);
        pap = grid_total(partials, 0);
        if (!(pap > 0.0)) { fail = 1.0; break; }
        gm = rz / pap;
        double acc[2] = {0.0, 0.0};
        auto upd = [&](long long i, bool live) {
            const double xi = __ldcg(x + i) + gm * __ldcg(pout + i);
            const double ri = __ldcg(r + i) - gm * __ldcg(q + i);
            const double zi = dinv[i] * ri;
            if (live) {
                x[i] = xi;
                r[i] = ri;
                z[i] = zi;
                acc[0] += ri * ri;
                acc[1] += ri * zi;
            }
        };
        if (sparse) {  // the rows the flagged strips own (every free row is one of them), spread
                       // over all threads: item = (strip on the list, row of the strip, lane)
            const int R = g.S * 32;
            const long long half = (long long)nfree * R, items = PAT == PF_CROSSED ? 2 * half : half;
            for (long long e = tid; e < items; e += nth) {
                const bool cen = PAT == PF_CROSSED && e >= half;
                const long long e2 = cen ? e - half : e;
                const int m = (int)(e2 / R), rho = (int)(e2 % R), l = rho & 31;
                if (l >= kLanesOut) continue;
                const int t = tiles[1 + m], wj = t % g.nwj, wi = t / g.nwj;
                const int j = wj * kLanesOut + l, i = wi * g.S + (rho >> 5);
                if (cen ? (j >= g.ny || i >= g.nx) : (j > g.ny || i > g.nx)) continue;
                const long long v = cen ? ctr(g, i, j) : vid(g, i, j);
                upd(v, op.act[v] == 0);
            }
        } else {
            for (long long i = tid; i < n; i += nth) upd(i, true);
        }
        block_partials(acc, 2, partials, 1);
        grid_sync(bar);
        const double2 t2 = grid_total2(partials, 1);
        const double rr = t2.x, rzn = t2.y;
        ++it;
        rn = sqrt(rr);
        if (rn <= target) { done = 1.0; break; }
        if (!(rzn > 0.0)) { fail = 2.0; break; }
        beta = rzn / rz;
        rz = rzn;
        if ((double)it >= maxit) { done = 3.0; break; }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s[S_ITER] = (double)it;
        s[S_RNORM] = rn;
        s[S_PAP] = pap;
        s[S_GAMMA] = gm;
        s[S_RZ] = rz;
        s[S_BETA] = beta;
        s[S_DONE] = done;
        s[S_FAIL] = fail;
    }
}

// ---- single-reduction damage PCG (Chronopoulos-Gear) ---------------------------------------------
// The same Krylov space as linalg.py:106-152 with the recurrences rearranged so that one strip
// pass per iteration does everything: with u = M r, w = A u, s = A p and the scalars
// alpha_i, beta_i known at the start of iteration i,
//   s_i = w_i + beta_i s_{i-1} ; r_{i+1} = r_i - alpha_i s_i ; u_{i+1} = M r_{i+1} (pointwise,
//   recomputed at every stencil point from staged r_i, w_i, s_{i-1}, dinv) ; w_{i+1} = A u_{i+1}
//   (the stencil) ; p_i = u_i + beta_i p_{i-1} ; x_{i+1} = x_i + alpha_i p_i (own vertex)
// and one grid reduction gives gamma = r.u, delta = w.u and |r|^2 for
//   beta_{i+1} = gamma_{i+1} / gamma_i ; alpha_{i+1} = gamma_{i+1} / (delta_{i+1} - beta_{i+1} gamma_{i+1} / alpha_i).
// r, w and s are double-buffered by iteration parity (neighbours read the old ones).
// vertex slots: r, w, s_prev, dinv, [act word]; cell: Gc, kappa x npc, [centre: the same]
template <bool MASKED>
struct OpKaaCG1 {
    static constexpr int NV = 1, NC = 1, MINB = 2;
    static constexpr int VS = 4 + (MASKED ? 1 : 0);
    static constexpr int pd(int pat) { return pat == PF_CROSSED ? 4 : 6; }
    static constexpr int ne(int pat) { return 1 + npc_of(pat) + 2 * crossed(pat); }
    static constexpr int sv(int) { return VS; }
    static constexpr int sc(int pat) { return 1 + npc_of(pat) + crossed(pat) * VS; }
    const double* kappa;
    const double *r, *w, *sp;   // r_i, w_i, s_{i-1}
    double *rn, *wn, *sn;       // r_{i+1}, w_{i+1}, s_i
    double *p, *x;              // in place
    const double* dinv;
    const unsigned char* act;
    double al, be;              // alpha_i, beta_i (be = 0: s_{-1}, p_{-1} unused)
    int init;                   // 1: the start-up pass w_0 = A u_0 only (u_0 = M r_0)
    double acc[3];              // gamma, delta, |r|^2 (own vertices)
    __device__ bool enter() const { return true; }
    __device__ void finish() {}
    __device__ __forceinline__ double unext(double ri, double wi, double si, double di) const {
        if (init) return di * ri;
        const double s = be != 0.0 ? wi + be * si : wi;
        return di * (ri - al * s);
    }
    __device__ __forceinline__ void stage_vertex(const Slots& s, long long v) const {
        put1(s, 0, r, v);
        put1(s, 1, w, v);
        put1(s, 2, sp, v);
        put1(s, 3, dinv, v);
        if (MASKED) putb(s, 4, act, v);
    }
    __device__ __forceinline__ double staged(const Slots& s, long long v, bool& a) const {
        a = MASKED ? (getb(s, 4, v) != 0u) : false;
        return a ? 0.0 : unext(get1(s, 0), get1(s, 1), get1(s, 2), get1(s, 3));
    }
    __device__ void issue_v(const Geo2& g, int i, int j, const Slots& s) const { stage_vertex(s, vid(g, i, j)); }
    __device__ void fix_v(const Geo2& g, int i, int j, const Slots& s, double (&v)[NV]) const {
        bool a;
        v[0] = staged(s, vid(g, i, j), a);
    }
    template <int PAT>
    __device__ void issue_c(const Geo2& g, int ci, int j, const Slots& s) const {
        const long long cell = cid(g, ci, j);
        putGc(g, s, 0, cell);
        put_kappa<PAT>(g, kappa, cell, s, 1);
        if constexpr (PAT == PF_CROSSED) stage_vertex(s.at(1 + npc_of(PAT)), ctr(g, ci, j));
    }
    template <int PAT, int NE>
    __device__ void fix_c(const Geo2& g, int ci, int j, const Slots& s, double (&e)[NE]) const {
        e[0] = getGc(g, s, 0);
        get_kappa<PAT>(g, s, 1, 1, e);
        if constexpr (PAT == PF_CROSSED) {
            bool a;
            e[5] = staged(s.at(1 + npc_of(PAT)), ctr(g, ci, j), a);
            e[6] = a ? 1.0 : 0.0;
        }
    }
    // own vertex: finish the pointwise recurrences (y = (A u_{i+1})_id, u = u_{i+1}(id))
    __device__ __forceinline__ void own(long long id, double y, double u, bool a) {
        if (a) y = 0.0;  // masked operator: identity rows act on u = 0
        wn[id] = y;
        if (init) {
            acc[0] += __ldcg(r + id) * u;
            acc[1] += y * u;
            return;
        }
        const double ri = __ldcg(r + id), wi = __ldcg(w + id);
        const double s = be != 0.0 ? wi + be * __ldcg(sp + id) : wi;
        const double r1 = ri - al * s;
        const double ui = a ? 0.0 : __ldg(dinv + id) * ri;  // u_i = M r_i
        const double pi = be != 0.0 ? ui + be * __ldcg(p + id) : ui;
        sn[id] = s;
        rn[id] = r1;
        p[id] = pi;
        x[id] = __ldcg(x + id) + al * pi;
        acc[0] += r1 * u;
        acc[1] += y * u;
        acc[2] += r1 * r1;
    }
    template <int PAT, int NE>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn_)[NV], const double (&ec)[NE],
                         double (&c00)[NC], double (&c10)[NC], double (&c01)[NC], double (&c11)[NC],
                         bool own_) {
        double X[5] = {vc[0], vn[0], rc[0], rn_[0], 0.0};
        if constexpr (PAT == PF_CROSSED) X[4] = ec[5];
        double Y[5] = {0, 0, 0, 0, 0};
        const int par = (PAT == PF_UNION_JACK) ? ((ci + j) & 1) : 0;
        const double hxs = par ? -g.ihx : g.ihx;
        mirror<PAT>(par, X);
        const double kc = ec[0] / g.cw;
        for_each_elem<PAT>(par, [&](auto T, auto S, auto A, auto B, auto C) {
            elem_kaa<PAT, T.v, A.v, B.v, C.v>(g, j, hxs, ec[1 + S.v], kc, X, Y);
        });
        mirror<PAT>(par, Y);
        c00[0] = Y[0]; c10[0] = Y[1]; c01[0] = Y[2]; c11[0] = Y[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own_) own(ctr(g, ci, j), Y[4], ec[5], ec[6] != 0.0);
        }
    }
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        own(id, t[0], v[0], MASKED && act[id] != 0);
    }
};

template <bool MASKED, int PAT>
__global__ void __launch_bounds__(kBlock, 2) k_pcg_kaa1(const Geo2 g, OpKaaCG1<MASKED> op0, int nvb, double* rb0,
                                                         double* rb1, double* wb0, double* wb1, double* sb0,
                                                         double* sb1, double* s, double* partials,
                                                         unsigned int* bar) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (!(s[S_DONE] == 0.0 && s[S_FAIL] == 0.0)) return;  // uniform
    const double target = s[S_TARGET], maxit = s[S_MAXIT];
    long long it = (long long)s[S_ITER];
    double rn = s[S_RNORM], done = 0.0, fail = 0.0;
    double* rb[2] = {rb0, rb1};
    double* wb[2] = {wb0, wb1};
    double* sb[2] = {sb0, sb1};
    auto pass = [&](int init, long long i, double al, double be) {
        OpKaaCG1<MASKED> op = op0;
        op.init = init;
        op.al = al;
        op.be = be;
        op.r = rb[i & 1];
        op.w = wb[i & 1];
        op.rn = rb[(i + 1) & 1];
        op.wn = wb[init ? (i & 1) : ((i + 1) & 1)];
        op.sp = sb[(i + 1) & 1];
        op.sn = sb[i & 1];
        op.acc[0] = op.acc[1] = op.acc[2] = 0.0;
        for (int vb = blockIdx.x; vb < nvb; vb += gridDim.x)
            strip_pass<OpKaaCG1<MASKED>, PAT>(g, op, smem, vb * (kBlock / 32) + (threadIdx.x >> 5));
        block_partials(op.acc, 3, partials, 0);
        grid_sync(bar);
    };
    // start-up: w_0 = A u_0 (u_0 = M r_0 from k_cg_init), gamma_0 = r.u (= S_RZ), delta_0 = w.u
    pass(1, 0, 0.0, 0.0);
    double gam = grid_total(partials, 0), del = grid_total(partials, 1);
    double al = gam / del, be = 0.0;
    if (!(gam > 0.0)) fail = 2.0;
    else if (!(del > 0.0)) fail = 1.0;
    for (long long i = 0; fail == 0.0; ++i) {
        pass(0, i, al, be);
        const double gn = grid_total(partials, 0), dn = grid_total(partials, 1);
        rn = sqrt(grid_total(partials, 2));
        ++it;
        if (rn <= target) { done = 1.0; break; }
        if (!(gn > 0.0)) { fail = 2.0; break; }
        be = gn / gam;
        const double den = dn - be * gn / al;
        if (!(den > 0.0)) { fail = 1.0; break; }
        al = gn / den;
        gam = gn;
        if ((double)it >= maxit) { done = 3.0; break; }
    }
    // the solution lives in x; r of the last iteration in rb[it & 1]
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        s[S_ITER] = (double)it;
        s[S_RNORM] = rn;
        s[S_RZ] = gam;
        s[S_DONE] = done;
        s[S_FAIL] = fail;
    }
}

template <bool MASKED, int PAT>
static int launch_pcg_kaa1_pat(Ctx* c, const PcgBuffers& B, const double* kappa, const unsigned char* act,
                               cudaStream_t st) {
    using Op = OpKaaCG1<MASKED>;
    constexpr int smem = strip_smem<Op, PAT>();
    static std::atomic<int> per_dev[kMaxDev];
    const int dvp = cur_dev();
    int per = per_dev[dvp].load();
    if (per <= 0) {
        cudaError_t e = cudaFuncSetAttribute(k_pcg_kaa1<MASKED, PAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return check_cuda(c, e, "persistent pcg attribute");
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg_kaa1<MASKED, PAT>, kBlock, smem);
        if (e != cudaSuccess) return check_cuda(c, e, "persistent pcg occupancy");
        per_dev[dvp] = per;
    }
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const Geo2& g = c->g;
    const int nvb = strip_blocks(g);
    const int nb = std::min(nvb, nsm * std::max(per, 1));
    if (per < 1 || nb > kMaxBlocksRed) return PF_EINVAL;
    // buffers: r_0 = B.r and u_0 = B.z from k_cg_init; x = B.x (zero start); p, s, w work vectors
    Op op{};
    op.kappa = kappa;
    op.dinv = B.dinv;
    op.act = act;
    op.p = B.p0;
    op.x = B.x;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb);
    cfg.blockDim = dim3(kBlock);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int ps = prof_begin(c, st);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_pcg_kaa1<MASKED, PAT>, g, op, nvb, B.r, B.z, B.q, B.p1, c->cg1_s0,
                                       c->cg1_s1, c->scal, c->partials, c->tickets + 62);
    prof_end(c, st, ps, K_KAA_CG, 0.0);
    c->launches++;
    return check_cuda(c, e, "persistent pcg launch");
}
int launch_pcg_kaa1(Ctx* c, const PcgBuffers& B, const double* kappa, const unsigned char* act, cudaStream_t st) {
    if (c->dim != 2) return PF_EINVAL;
    switch (c->g.pattern) {
        case PF_UNION_JACK:
            return act ? launch_pcg_kaa1_pat<true, PF_UNION_JACK>(c, B, kappa, act, st)
                       : launch_pcg_kaa1_pat<false, PF_UNION_JACK>(c, B, kappa, act, st);
        case PF_RIGHT:
            return act ? launch_pcg_kaa1_pat<true, PF_RIGHT>(c, B, kappa, act, st)
                       : launch_pcg_kaa1_pat<false, PF_RIGHT>(c, B, kappa, act, st);
        default:
            return act ? launch_pcg_kaa1_pat<true, PF_CROSSED>(c, B, kappa, act, st)
                       : launch_pcg_kaa1_pat<false, PF_CROSSED>(c, B, kappa, act, st);
    }
}

template <bool MASKED, int PAT, int NT>
static int launch_pcg_kaa_pat(Ctx* c, const PcgBuffers& B, const double* kappa, const unsigned char* act,
                              cudaStream_t st) {
    using Op = OpKaa<true, MASKED>;
    constexpr int smem = strip_smem<Op, PAT>() * (NT / kBlock);  // strip rings of NT/32 warps
    static std::atomic<int> per_dev[kMaxDev];
    const int dvp = cur_dev();
    int per = per_dev[dvp].load();
    if (per <= 0) {
        cudaError_t e = cudaFuncSetAttribute(k_pcg_kaa<MASKED, PAT, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return check_cuda(c, e, "persistent pcg attribute");
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_pcg_kaa<MASKED, PAT, NT>, NT, smem);
        if (e != cudaSuccess) return check_cuda(c, e, "persistent pcg occupancy");
        per_dev[dvp] = per;
    }
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const Geo2& g = c->g;
    const long long warps = (long long)g.nwj * g.nstrips;
    const int nvb = (int)((warps + NT / 32 - 1) / (NT / 32));
    const int nb = std::min(nvb, nsm * std::max(per, 1));
    if (per < 1 || nb > kMaxBlocksRed) return PF_EINVAL;  // caller falls back to the graph loop
    Op op{kappa, B.z, B.p0, B.p1, B.q, act, c->scal, redbuf(c), 0.0};
    const int* tiles = nullptr;
    c->tile_frac = 1.0;
    static const bool skip_off = getenv("PF_NO_TILE_SKIP") != nullptr;
    if (MASKED && c->rhs_masked && !skip_off && c->tile_list && warps <= c->tile_cap) {
        unsigned char* flag = reinterpret_cast<unsigned char*>(c->tile_list + c->tile_cap + 1);
        k_tile_flags2<<<(int)((warps + 7) / 8), 256, 0, st>>>(g, act, (int)warps, flag);
        launch_tile_compact((int)warps, flag, c->tile_list, st);
        c->launches += 2;
        tiles = c->tile_list;
        if (c->prof.on || getenv("PF_TILE_TRACE")) {  // (diagnostics only: one host read)
            int nfree = 0;
            cudaMemcpyAsync(&nfree, c->tile_list, sizeof(int), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            c->tile_frac = 2LL * nfree <= (long long)warps ? (double)nfree / (double)warps : 1.0;
        }
        if (getenv("PF_TILE_TRACE")) {
            int nfree = 0;
            cudaMemcpyAsync(&nfree, c->tile_list, sizeof(int), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            fprintf(stderr, "  damage pcg: %d of %lld strips hold free vertices\n", nfree, warps);
        }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int ps = prof_begin(c, st);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_pcg_kaa<MASKED, PAT, NT>, g, op, nvb, B.n, B.x, B.r, B.z, B.p0, B.p1,
                                       B.q, (const double*)B.dinv, c->scal, c->partials, c->tickets + 62, tiles);
    prof_end(c, st, ps, K_KAA_CG, 0.0);
    c->launches++;
    return check_cuda(c, e, "persistent pcg launch");
}
template <bool MASKED, int PAT>
static int launch_pcg_kaa_nt(Ctx* c, const PcgBuffers& B, const double* kappa, const unsigned char* act,
                             cudaStream_t st) {
    static const bool wide = getenv("PF_PCG_NT256") == nullptr;
    return wide ? launch_pcg_kaa_pat<MASKED, PAT, 512>(c, B, kappa, act, st)
                : launch_pcg_kaa_pat<MASKED, PAT, 256>(c, B, kappa, act, st);
}
int launch_pcg_kaa(Ctx* c, const PcgBuffers& B, const double* kappa, const unsigned char* act, cudaStream_t st) {
    if (c->dim == 3) return launch3_pcg_kaa(c, B, kappa, act, st);
    switch (c->g.pattern) {
        case PF_UNION_JACK:
            return act ? launch_pcg_kaa_nt<true, PF_UNION_JACK>(c, B, kappa, act, st)
                       : launch_pcg_kaa_nt<false, PF_UNION_JACK>(c, B, kappa, act, st);
        case PF_RIGHT:
            return act ? launch_pcg_kaa_nt<true, PF_RIGHT>(c, B, kappa, act, st)
                       : launch_pcg_kaa_nt<false, PF_RIGHT>(c, B, kappa, act, st);
        default:
            return act ? launch_pcg_kaa_nt<true, PF_CROSSED>(c, B, kappa, act, st)
                       : launch_pcg_kaa_nt<false, PF_CROSSED>(c, B, kappa, act, st);
    }
}

int launch_Kaa_diag(Ctx* c, const double* kappa, double* dinv, const unsigned char* act,
                    cudaStream_t st) {
    if (c->dim == 3) return launch3_Kaa_diag(c, kappa, dinv, act, st);
    if (act) {
        OpKaaDiag<true> op;
        op.kappa = kappa; op.dinv = dinv; op.act = act;
        return run_strip(c, op, st, K_KAA_DIAG);
    }
    OpKaaDiag<false> op;
    op.kappa = kappa; op.dinv = dinv; op.act = nullptr;
    return run_strip(c, op, st, K_KAA_DIAG);
}
int launch_Kaa_trial(Ctx* c, const double* kappa, const double* cvec, const double* x,
                     const double* d, const double* lb, double* trial, double* F,
                     unsigned char* act, int merit_slot, cudaStream_t st) {
    if (c->dim == 3) return launch3_Kaa_trial(c, kappa, cvec, x, d, lb, trial, F, merit_slot, st);
    OpKaaTrial op{kappa, cvec, x, d, lb, trial, F, c->scal, merit_slot, redbuf(c), 0.0};
    (void)act;
    return run_strip(c, op, st, K_KAA_TRIAL);
}
int launch_physics(Ctx* c, const double* u, const double* alpha, const double* lb, double* ru,
                   double* ra, double* phi, int rows, cudaStream_t st) {
    if (c->dim == 3) return launch3_physics(c, u, alpha, lb, ru, ra, phi, rows, st);
    const int nw = (ru ? 2 : 0) + (ra ? 1 : 0) + (phi ? 1 : 0);
    switch (rows) {
        case PF_ROWS_ZERO: {
            OpPhys<PF_ROWS_ZERO> op{u, alpha, lb, ru, ra, phi, c->scal, redbuf(c), 0, 0, 0, 0};
            return run_strip(c, op, st, K_PHYS, nw);
        }
        case PF_ROWS_VALUE: {
            OpPhys<PF_ROWS_VALUE> op{u, alpha, lb, ru, ra, phi, c->scal, redbuf(c), 0, 0, 0, 0};
            return run_strip(c, op, st, K_PHYS, nw);
        }
        default: {
            OpPhys<PF_ROWS_RAW> op{u, alpha, lb, ru, ra, phi, c->scal, redbuf(c), 0, 0, 0, 0};
            return run_strip(c, op, st, K_PHYS, nw);
        }
    }
}
int launch_physics_relax(Ctx* c, const double* u, const double* a_prev, const double* a_star, const double* lb,
                         double omega, double* a_out, cudaStream_t st) {
    OpPhys<PF_ROWS_ZERO, true> op{u, a_prev, lb, nullptr, nullptr, nullptr, c->scal, redbuf(c), 0, 0, 0, 0,
                                  a_star, a_out, omega, c->bits};
    // physics (u, alpha) + alpha_prev, alpha*, lb in, alpha out
    return run_strip(c, op, st, K_PHYS, 0, (double)c->g.nv * (16 + 8 + 8 + 8 + 8 + 8));
}
int launch_load(Ctx* c, const double* alpha, double* f, const double* u_or_null, int rows,
                cudaStream_t st) {
    if (c->dim == 3) return launch3_load(c, alpha, f, rows, st);
    (void)u_or_null;
    if (rows == 0) {
        OpRhs<true> op{alpha, f, c->scal, redbuf(c), 0.0};
        return run_strip(c, op, st, K_RHS);
    }
    OpRhs<false> op{alpha, f, c->scal, redbuf(c), 0.0};
    return run_strip(c, op, st, K_RHS);
}
int launch_Kua(Ctx* c, const double* u, const double* alpha, const double* xa, double* yu,
               int bcmode, cudaStream_t st) {
    if (c->dim == 3) return launch3_jac(c, u, alpha, nullptr, xa, yu, nullptr, nullptr, 1, bcmode, st);
    OpKua op;
    op.u = u; op.alpha = alpha; op.xa = xa; op.yu = yu; op.bcmode = bcmode;
    return run_strip(c, op, st, K_KUA);
}
int launch_Kau(Ctx* c, const double* u, const double* alpha, const double* xu, double* ya,
               int bcmode, cudaStream_t st) {
    if (c->dim == 3) return launch3_jac(c, u, alpha, xu, nullptr, nullptr, ya, nullptr, 2, bcmode, st);
    OpKau op;
    op.u = u; op.alpha = alpha; op.xu = xu; op.ya = ya; op.bcmode = bcmode;
    return run_strip(c, op, st, K_KAU);
}
int launch_jac(Ctx* c, const double* u, const double* alpha, const double* xu, const double* xa,
               double* yu, double* ya, const unsigned char* act, cudaStream_t st) {
    if (c->dim == 3) return launch3_jac(c, u, alpha, xu, xa, yu, ya, act, 0, PF_BC_ELIMINATE, st);
    OpJac op;
    op.u = u; op.alpha = alpha; op.xu = xu; op.xa = xa; op.yu = yu; op.ya = ya; op.act = act;
    return run_strip(c, op, st, K_JAC);
}

}  // namespace pf
