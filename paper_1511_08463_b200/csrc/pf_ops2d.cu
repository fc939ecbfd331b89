// pf_ops2d.cu -- matrix-free P1 operators on structured 2D triangle meshes (sm_100a, fp64).
//
// One "strip" engine (k_strip2d) drives every operator.  A warp owns vertex columns
// j = 30w-1 .. 30w+30 (lanes 0..31; lanes 1..30 produce output) and walks vertex rows
// i0-1 .. i1 of its strip.  At row step ci it holds vertex rows ci (vc) and ci+1 (vn) of its
// column in registers, gets column j+1 from lane+1 (rc, rn) by shuffle, computes the elements
// of cell (ci, j) and scatters their nodal contributions:
//     c00 -> (ci, j)      own lane, this step       c01 -> (ci, j+1)   lane+1 (shfl_up)
//     c10 -> (ci+1, j)    own lane, next step       c11 -> (ci+1, j+1) lane+1, next step
// so vertex (ci, j) is final once cell row ci is done.  Loads: 1 vertex per lane per step,
// coalesced along j; halo re-reads (1/30 columns, 1/S rows) hit L2.  No atomics: all
// outputs and reductions are deterministic.
//
// Reference formulas: fem.py:149-276 (element kinematics, energy, residuals, Hessian blocks),
// model.py:49-76 (stiffness, damage pair).  Element types per pattern (local nodes
// 0=v00 1=v10 2=v01 3=v11 4=centre), in the reference's storage order (mesh.py:95-99):
//   union-jack even cell: (0,1,3) (0,3,2);  odd cell: (0,1,2) (1,3,2)
//   right:                (0,1,3) (0,3,2)
//   crossed:              (0,1,4) (1,3,4) (3,2,4) (2,0,4)
#include "pf_internal.cuh"

namespace pf {

template <int N> struct IC { static constexpr int v = N; };

template <int PAT, class F>
__device__ __forceinline__ void for_each_elem(int parity, F&& f) {
    if constexpr (PAT == PF_UNION_JACK) {
        if (parity == 0) {
            f(IC<0>{}, IC<0>{}, IC<0>{}, IC<1>{}, IC<3>{});
            f(IC<1>{}, IC<1>{}, IC<0>{}, IC<3>{}, IC<2>{});
        } else {
            f(IC<2>{}, IC<0>{}, IC<0>{}, IC<1>{}, IC<2>{});
            f(IC<3>{}, IC<1>{}, IC<1>{}, IC<3>{}, IC<2>{});
        }
    } else if constexpr (PAT == PF_RIGHT) {
        f(IC<0>{}, IC<0>{}, IC<0>{}, IC<1>{}, IC<3>{});
        f(IC<1>{}, IC<1>{}, IC<0>{}, IC<3>{}, IC<2>{});
    } else {
        f(IC<0>{}, IC<0>{}, IC<0>{}, IC<1>{}, IC<4>{});
        f(IC<1>{}, IC<1>{}, IC<1>{}, IC<3>{}, IC<4>{});
        f(IC<2>{}, IC<2>{}, IC<3>{}, IC<2>{}, IC<4>{});
        f(IC<3>{}, IC<3>{}, IC<2>{}, IC<0>{}, IC<4>{});
    }
}

__device__ __forceinline__ bool on_boundary(const Geo2& g, int i, int j) {
    return i == 0 || i == g.nx || j == 0 || j == g.ny;
}
__device__ __forceinline__ unsigned bcbits(const Geo2& g, int i, int j, long long v) {
    return (g.has_bc && on_boundary(g, i, j)) ? (unsigned)g.bcmask[v] : 0u;
}
__device__ __forceinline__ double cellE(const Geo2& g, long long cell) {
    return g.E_cell ? __ldg(g.E_cell + cell) : g.E;
}
__device__ __forceinline__ double cellGc(const Geo2& g, long long cell) {
    return g.Gc_cell ? __ldg(g.Gc_cell + cell) : g.Gc;
}
__device__ __forceinline__ double fbphi(double a, double b) { return hypot(a, b) - a - b; }
__device__ __forceinline__ double2 ld2(const double* p, long long v) {
    return __ldg(reinterpret_cast<const double2*>(p) + v);
}
__device__ __forceinline__ void st2(double* p, long long v, double a, double b) {
    reinterpret_cast<double2*>(p)[v] = make_double2(a, b);
}

// ---- element kernels ---------------------------------------------------------------------
// strain of element type T with nodes A,B,C: (e11, e22, g12) = B u_e
template <int T, int A, int B, int C>
__device__ __forceinline__ void strain(const Geo2& g, const double (&U1)[5], const double (&U2)[5],
                                       double& e0, double& e1, double& e2) {
    const double b0 = g.gb[T][0], b1 = g.gb[T][1], b2 = g.gb[T][2];
    const double c0 = g.gc[T][0], c1 = g.gc[T][1], c2 = g.gc[T][2];
    e0 = b0 * U1[A] + b1 * U1[B] + b2 * U1[C];
    e1 = c0 * U2[A] + c1 * U2[B] + c2 * U2[C];
    e2 = (c0 * U1[A] + c1 * U1[B] + c2 * U1[C]) + (b0 * U2[A] + b1 * U2[B] + b2 * U2[C]);
}
// Y_m += B_m^T (s0, s1, s2)
template <int T, int A, int B, int C>
__device__ __forceinline__ void scatter_BT(const Geo2& g, double s0, double s1, double s2,
                                           double (&Y1)[5], double (&Y2)[5]) {
    const double b0 = g.gb[T][0], b1 = g.gb[T][1], b2 = g.gb[T][2];
    const double c0 = g.gc[T][0], c1 = g.gc[T][1], c2 = g.gc[T][2];
    Y1[A] += b0 * s0 + c0 * s2;  Y2[A] += c0 * s1 + b0 * s2;
    Y1[B] += b1 * s0 + c1 * s2;  Y2[B] += c1 * s1 + b1 * s2;
    Y1[C] += b2 * s0 + c2 * s2;  Y2[C] += c2 * s1 + b2 * s2;
}
__device__ __forceinline__ void unit_stress(const Geo2& g, double e0, double e1, double e2,
                                            double& s0, double& s1, double& s2) {
    s0 = g.D00 * e0 + g.D01 * e1;
    s1 = g.D01 * e0 + g.D11 * e1;
    s2 = g.D22 * e2;
}

// ---- the strip engine ----------------------------------------------------------------------
template <class Op, int PAT>
__global__ void __launch_bounds__(kBlock) k_strip2d(const Geo2 g, Op op) {
    constexpr int NV = Op::NV, NC = Op::NC;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
    const int wj = gw % g.nwj, wi = gw / g.nwj;
    if (!op.enter()) return;  // device-side early exit (solver converged): uniform
    if (wi < g.nstrips) {
        const int j = wj * kLanesOut - 1 + lane;
        const bool jv = (j >= 0) && (j <= g.ny);
        const bool jc = (j >= 0) && (j < g.ny) && (lane < 31);
        const bool jo = jv && lane >= 1 && lane <= kLanesOut;
        const int i0 = wi * g.S;
        const int i1 = min(i0 + g.S, g.nx + 1);
        double vc[NV], vn[NV], rc[NV], rn[NV], vp[NV], carry[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) carry[k] = 0.0;
        int ci = i0 - 1;
#pragma unroll
        for (int k = 0; k < NV; ++k) { vc[k] = 0.0; vp[k] = 0.0; }
        if (ci >= 0 && jv) op.load(g, ci, j, vc);
        if (ci + 1 <= g.nx && jv) op.load(g, ci + 1, j, vp);
#pragma unroll
        for (int k = 0; k < NV; ++k) rc[k] = __shfl_down_sync(PF_FULL, vc[k], 1);
        for (; ci < i1; ++ci) {
#pragma unroll
            for (int k = 0; k < NV; ++k) { vn[k] = vp[k]; vp[k] = 0.0; }
            if (ci + 2 <= g.nx && ci + 1 < i1 && jv) op.load(g, ci + 2, j, vp);
#pragma unroll
            for (int k = 0; k < NV; ++k) rn[k] = __shfl_down_sync(PF_FULL, vn[k], 1);
            double c00[NC], c10[NC], c01[NC], c11[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) { c00[k] = c10[k] = c01[k] = c11[k] = 0.0; }
            if (ci >= 0 && ci < g.nx && jc)
                op.template cell<PAT>(g, ci, j, vc, vn, rc, rn, c00, c10, c01, c11,
                                      (ci >= i0) && jo);
#pragma unroll
            for (int k = 0; k < NC; ++k) {
                const double l01 = __shfl_up_sync(PF_FULL, c01[k], 1);
                const double l11 = __shfl_up_sync(PF_FULL, c11[k], 1);
                c00[k] += carry[k] + l01;
                carry[k] = c10[k] + l11;
            }
            if (ci >= i0 && jo) op.out(g, ci, j, c00, vc);
#pragma unroll
            for (int k = 0; k < NV; ++k) { vc[k] = vn[k]; rc[k] = rn[k]; }
        }
    }
    op.finish();
}

// vertex id helpers
__device__ __forceinline__ long long vid(const Geo2& g, int i, int j) { return (long long)i * g.nvy + j; }
__device__ __forceinline__ long long cid(const Geo2& g, int ci, int j) { return (long long)ci * g.ny + j; }
__device__ __forceinline__ long long ctr(const Geo2& g, int ci, int j) { return g.nc + cid(g, ci, j); }

struct NoRed {
    __device__ bool enter() const { return true; }
    __device__ void finish() {}
};

// ================================================================================================
// Kuu: y = K(alpha) x, optionally Dirichlet-eliminated (fem.py:233-243, 282-294).
// FUSED: CG step A -- p_out = z + beta p_in (beta = 0 at iteration 0), y = K p_out, pAp reduced
// and gamma = rz / pAp formed by the last block (linalg.py:130-138).
// ================================================================================================
template <bool FUSED>
struct OpKuu {
    static constexpr int NV = 3, NC = 2;
    const double* alpha;
    const double* x;      // plain: x ; fused: z
    const double* pin;    // fused only
    double* pout;         // fused only
    double* y;
    int bcmode;
    double* scal;
    RedBuf rb;
    double acc;

    __device__ bool enter() const {
        if (!FUSED) return true;
        return scal[S_DONE] == 0.0 && scal[S_FAIL] == 0.0;
    }
    __device__ __forceinline__ double beta() const { return scal[S_ITER] > 0.0 ? scal[S_BETA] : 0.0; }
    __device__ __forceinline__ double2 xval(long long v) const {
        double2 z = ld2(x, v);
        if (FUSED) {
            const double b = beta();
            const double2 p = ld2(pin, v);
            z.x = z.x + b * p.x;
            z.y = z.y + b * p.y;
        }
        return z;
    }
    __device__ void load(const Geo2& g, int i, int j, double (&v)[NV]) const {
        const long long id = vid(g, i, j);
        const double2 xv = xval(id);
        const unsigned m = bcmode ? bcbits(g, i, j, id) : 0u;
        v[0] = (m & 1u) ? 0.0 : xv.x;
        v[1] = (m & 2u) ? 0.0 : xv.y;
        v[2] = __ldg(alpha + id);
    }
    template <int PAT>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], double (&c00)[NC],
                         double (&c10)[NC], double (&c01)[NC], double (&c11)[NC], bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        double Al[5] = {vc[2], vn[2], rc[2], rn[2], 0.0};
        long long cv = 0;
        if constexpr (PAT == PF_CROSSED) {
            cv = ctr(g, ci, j);
            const double2 xv = xval(cv);
            U1[4] = xv.x; U2[4] = xv.y; Al[4] = __ldg(alpha + cv);
        }
        double Y1[5] = {0, 0, 0, 0, 0}, Y2[5] = {0, 0, 0, 0, 0};
        const long long cell = cid(g, ci, j);
        const double Ec = cellE(g, cell);
        for_each_elem<PAT>((ci + j) & 1, [&](auto T, auto, auto A, auto B, auto C) {
            const double ab = (Al[A.v] + Al[B.v] + Al[C.v]) * (1.0 / 3.0);
            const double om = 1.0 - ab;
            const double s = (om * om + g.kell) * g.area[T.v] * Ec;
            double e0, e1, e2, s0, s1, s2;
            strain<T.v, A.v, B.v, C.v>(g, U1, U2, e0, e1, e2);
            unit_stress(g, e0, e1, e2, s0, s1, s2);
            scatter_BT<T.v, A.v, B.v, C.v>(g, s * s0, s * s1, s * s2, Y1, Y2);
        });
        c00[0] = Y1[0]; c00[1] = Y2[0];
        c10[0] = Y1[1]; c10[1] = Y2[1];
        c01[0] = Y1[2]; c01[1] = Y2[2];
        c11[0] = Y1[3]; c11[1] = Y2[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) {
                st2(y, cv, Y1[4], Y2[4]);
                if (FUSED) {
                    st2(pout, cv, U1[4], U2[4]);
                    acc += U1[4] * Y1[4] + U2[4] * Y2[4];
                }
            }
        }
    }
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        double y0 = t[0], y1 = t[1];
        double p0 = v[0], p1 = v[1];
        const unsigned m = bcmode ? bcbits(g, i, j, id) : 0u;
        if (m) {
            const double2 xv = xval(id);
            if (m & 1u) { y0 = xv.x; p0 = xv.x; }
            if (m & 2u) { y1 = xv.y; p1 = xv.y; }
        }
        st2(y, id, y0, y1);
        if (FUSED) {
            st2(pout, id, p0, p1);
            acc += p0 * y0 + p1 * y1;
        }
    }
    __device__ void finish() {
        if (!FUSED) return;
        double v[1] = {acc};
        double* s = scal;
        grid_reduce<1>(v, rb, 0, [s](double* tot) {
            s[S_PAP] = tot[0];
            if (!(tot[0] > 0.0)) s[S_FAIL] = 1.0;  // breakdown: p'Ap <= 0 (linalg.py:133-136)
            else s[S_GAMMA] = s[S_RZ] / tot[0];
        });
    }
};

// diag(Kuu) -> dinv = 1/diag; eliminated rows get 1.
struct OpKuuDiag : NoRed {
    static constexpr int NV = 1, NC = 2;
    const double* alpha;
    double* dinv;
    __device__ void load(const Geo2& g, int i, int j, double (&v)[NV]) const {
        v[0] = __ldg(alpha + vid(g, i, j));
    }
    template <int PAT>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], double (&c00)[NC],
                         double (&c10)[NC], double (&c01)[NC], double (&c11)[NC], bool own) {
        double Al[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        long long cv = 0;
        if constexpr (PAT == PF_CROSSED) { cv = ctr(g, ci, j); Al[4] = __ldg(alpha + cv); }
        double Y1[5] = {0, 0, 0, 0, 0}, Y2[5] = {0, 0, 0, 0, 0};
        const double Ec = cellE(g, cid(g, ci, j));
        for_each_elem<PAT>((ci + j) & 1, [&](auto T, auto, auto A, auto B, auto C) {
            const double ab = (Al[A.v] + Al[B.v] + Al[C.v]) * (1.0 / 3.0);
            const double om = 1.0 - ab;
            const double s = (om * om + g.kell) * g.area[T.v] * Ec;
            const double* b = g.gb[T.v];
            const double* c = g.gc[T.v];
            Y1[A.v] += s * (b[0] * b[0] * g.D00 + c[0] * c[0] * g.D22);
            Y2[A.v] += s * (c[0] * c[0] * g.D11 + b[0] * b[0] * g.D22);
            Y1[B.v] += s * (b[1] * b[1] * g.D00 + c[1] * c[1] * g.D22);
            Y2[B.v] += s * (c[1] * c[1] * g.D11 + b[1] * b[1] * g.D22);
            Y1[C.v] += s * (b[2] * b[2] * g.D00 + c[2] * c[2] * g.D22);
            Y2[C.v] += s * (c[2] * c[2] * g.D11 + b[2] * b[2] * g.D22);
        });
        c00[0] = Y1[0]; c00[1] = Y2[0]; c10[0] = Y1[1]; c10[1] = Y2[1];
        c01[0] = Y1[2]; c01[1] = Y2[2]; c11[0] = Y1[3]; c11[1] = Y2[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) st2(dinv, cv, 1.0 / Y1[4], 1.0 / Y2[4]);
        }
    }
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&)[NV]) {
        const long long id = vid(g, i, j);
        const unsigned m = bcbits(g, i, j, id);
        st2(dinv, id, (m & 1u) ? 1.0 : 1.0 / t[0], (m & 2u) ? 1.0 : 1.0 / t[1]);
    }
};

// ================================================================================================
// Damage block.  kappa_e = (1/2 a'' q + (Gc/c_w) w''/ell) |T|/9 is the element reaction
// coefficient (fem.py:266-276; independent of alpha for AT1/AT2); c = r_alpha - Kaa alpha is its
// affine remainder (solver.py:152-153), c_v = sum_e |T|/3 (-q_e + [AT1] Gc_e/(c_w ell)).
// ================================================================================================
struct OpKappa : NoRed {
    static constexpr int NV = 2, NC = 1;
    const double* u;
    double* kappa;
    double* cvec;
    __device__ void load(const Geo2& g, int i, int j, double (&v)[NV]) const {
        const double2 uv = ld2(u, vid(g, i, j));
        v[0] = uv.x; v[1] = uv.y;
    }
    template <int PAT>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], double (&c00)[NC],
                         double (&c10)[NC], double (&c01)[NC], double (&c11)[NC], bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        long long cv = 0;
        if constexpr (PAT == PF_CROSSED) {
            cv = ctr(g, ci, j);
            const double2 uv = ld2(u, cv);
            U1[4] = uv.x; U2[4] = uv.y;
        }
        double Y[5] = {0, 0, 0, 0, 0};
        const long long cell = cid(g, ci, j);
        const double Ec = cellE(g, cell);
        const double kc = cellGc(g, cell) / g.cw;
        for_each_elem<PAT>((ci + j) & 1, [&](auto T, auto S, auto A, auto B, auto C) {
            double e0, e1, e2, s0, s1, s2;
            strain<T.v, A.v, B.v, C.v>(g, U1, U2, e0, e1, e2);
            if (g.eps0) {
                const double e = __ldg(g.eps0 + (long long)T.v * g.ny + j);
                e0 -= e; e1 -= e;
            }
            unit_stress(g, e0, e1, e2, s0, s1, s2);
            const double q = Ec * (e0 * s0 + e1 * s1 + e2 * s2);
            const double ar = g.area[T.v];
            const double kap = (q + (g.at2 ? 2.0 * kc / g.ell : 0.0)) * ar * (1.0 / 9.0);
            const double cc = ar * (1.0 / 3.0) * (-q + (g.at2 ? 0.0 : kc / g.ell));
            Y[A.v] += cc; Y[B.v] += cc; Y[C.v] += cc;
            if (own) kappa[(long long)S.v * g.ncell + cell] = kap;
        });
        c00[0] = Y[0]; c10[0] = Y[1]; c01[0] = Y[2]; c11[0] = Y[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) cvec[cv] = Y[4];
        }
    }
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&)[NV]) {
        cvec[vid(g, i, j)] = t[0];
    }
};

// Damage Hessian element action: y_m += kappa (x_A + x_B + x_C) + delta (b_m gx + c_m gy),
// delta = 2 (Gc/c_w) ell |T| (diffusion part, fem.py:272-273).
template <int T, int A, int B, int C>
__device__ __forceinline__ void elem_kaa(const Geo2& g, double kap, double kc, const double (&X)[5],
                                         double (&Y)[5]) {
    const double b0 = g.gb[T][0], b1 = g.gb[T][1], b2 = g.gb[T][2];
    const double c0 = g.gc[T][0], c1 = g.gc[T][1], c2 = g.gc[T][2];
    const double del = 2.0 * kc * g.ell * g.area[T];
    const double sx = kap * ((X[A] + X[B]) + X[C]);
    const double gx = del * (b0 * X[A] + b1 * X[B] + b2 * X[C]);
    const double gy = del * (c0 * X[A] + c1 * X[B] + c2 * X[C]);
    Y[A] += sx + b0 * gx + c0 * gy;
    Y[B] += sx + b1 * gx + c1 * gy;
    Y[C] += sx + b2 * gx + c2 * gy;
}

// Kaa apply; MASKED: rows/cols of active vertices (act != 0) are replaced by identity (the
// reduced inactive-block operator J_NN of vi.py:235 embedded in full space).
template <bool FUSED, bool MASKED>
struct OpKaa {
    static constexpr int NV = 1, NC = 1;
    const double* kappa;
    const double* x;     // fused: z
    const double* pin;
    double* pout;
    double* y;
    const unsigned char* act;
    double* scal;
    RedBuf rb;
    double acc;
    __device__ bool enter() const {
        if (!FUSED) return true;
        return scal[S_DONE] == 0.0 && scal[S_FAIL] == 0.0;
    }
    __device__ __forceinline__ double xval(long long v) const {
        double z = __ldg(x + v);
        if (FUSED) {
            const double b = scal[S_ITER] > 0.0 ? scal[S_BETA] : 0.0;
            z = z + b * __ldg(pin + v);
        }
        return z;
    }
    __device__ __forceinline__ bool is_act(long long v) const { return MASKED && act[v] != 0; }
    __device__ void load(const Geo2& g, int i, int j, double (&v)[NV]) const {
        const long long id = vid(g, i, j);
        v[0] = is_act(id) ? 0.0 : xval(id);
    }
    template <int PAT>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], double (&c00)[NC],
                         double (&c10)[NC], double (&c01)[NC], double (&c11)[NC], bool own) {
        double X[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        long long cv = 0;
        double xc = 0.0;
        if constexpr (PAT == PF_CROSSED) {
            cv = ctr(g, ci, j);
            xc = xval(cv);
            X[4] = is_act(cv) ? 0.0 : xc;
        }
        double Y[5] = {0, 0, 0, 0, 0};
        const long long cell = cid(g, ci, j);
        const double kc = cellGc(g, cell) / g.cw;
        for_each_elem<PAT>((ci + j) & 1, [&](auto T, auto S, auto A, auto B, auto C) {
            const double kap = __ldg(kappa + (long long)S.v * g.ncell + cell);
            elem_kaa<T.v, A.v, B.v, C.v>(g, kap, kc, X, Y);
        });
        c00[0] = Y[0]; c10[0] = Y[1]; c01[0] = Y[2]; c11[0] = Y[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) {
                const double yy = is_act(cv) ? xc : Y[4];
                y[cv] = yy;
                if (FUSED) { pout[cv] = xc; acc += xc * yy; }
            }
        }
    }
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        double yy = t[0], p = v[0];
        if (is_act(id)) { p = xval(id); yy = p; }
        y[id] = yy;
        if (FUSED) { pout[id] = p; acc += p * yy; }
    }
    __device__ void finish() {
        if (!FUSED) return;
        double v[1] = {acc};
        double* s = scal;
        grid_reduce<1>(v, rb, 0, [s](double* tot) {
            s[S_PAP] = tot[0];
            if (!(tot[0] > 0.0)) s[S_FAIL] = 1.0;
            else s[S_GAMMA] = s[S_RZ] / tot[0];
        });
    }
};

template <bool MASKED>
struct OpKaaDiag : NoRed {
    static constexpr int NV = 1, NC = 1;
    const double* kappa;
    double* dinv;
    const unsigned char* act;
    __device__ void load(const Geo2&, int, int, double (&v)[NV]) const { v[0] = 0.0; }
    template <int PAT>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&)[NV], const double (&)[NV],
                         const double (&)[NV], const double (&)[NV], double (&c00)[NC],
                         double (&c10)[NC], double (&c01)[NC], double (&c11)[NC], bool own) {
        double Y[5] = {0, 0, 0, 0, 0};
        const long long cell = cid(g, ci, j);
        const double kc = cellGc(g, cell) / g.cw;
        for_each_elem<PAT>((ci + j) & 1, [&](auto T, auto S, auto A, auto B, auto C) {
            const double kap = __ldg(kappa + (long long)S.v * g.ncell + cell);
            const double del = 2.0 * kc * g.ell * g.area[T.v];
            const double* b = g.gb[T.v];
            const double* c = g.gc[T.v];
            Y[A.v] += kap + del * (b[0] * b[0] + c[0] * c[0]);
            Y[B.v] += kap + del * (b[1] * b[1] + c[1] * c[1]);
            Y[C.v] += kap + del * (b[2] * b[2] + c[2] * c[2]);
        });
        c00[0] = Y[0]; c10[0] = Y[1]; c01[0] = Y[2]; c11[0] = Y[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) {
                const long long cv = ctr(g, ci, j);
                dinv[cv] = (MASKED && act[cv]) ? 1.0 : 1.0 / Y[4];
            }
        }
    }
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&)[NV]) {
        const long long id = vid(g, i, j);
        dinv[id] = (MASKED && act[id]) ? 1.0 : 1.0 / t[0];
    }
};

// ================================================================================================
// Line-search trial of the damage VI (vi.py:209-220, 227-228): trial = clip(x + mu d, lb, 1)
// (d == null -> trial = x), F = Kaa trial + c, Phi = fb(trial - lb, fb(1 - trial, -F)),
// merit = |Phi|^2, activity classification with slack zeta (vi.py:127-141):
// act = 1 lower-active, 2 upper-active, 0 inactive; counts the inactive set.
// ================================================================================================
struct OpKaaTrial {
    static constexpr int NV = 1, NC = 1;
    const double* kappa;
    const double* cvec;
    const double* x;
    const double* d;
    const double* lb;
    double* trial;
    double* F;
    unsigned char* act;
    double* scal;
    int merit_slot;
    RedBuf rb;
    double acc_m, acc_n;
    __device__ bool enter() const { return true; }
    __device__ __forceinline__ double tval(long long v) const {
        const double xv = __ldg(x + v);
        if (!d) return xv;
        const double t = xv + scal[S_MU] * __ldg(d + v);
        return fmin(fmax(t, __ldg(lb + v)), 1.0);
    }
    __device__ void load(const Geo2& g, int i, int j, double (&v)[NV]) const { v[0] = tval(vid(g, i, j)); }
    __device__ __forceinline__ void finish_vertex(long long id, double tv, double Fv) {
        const double l = __ldg(lb + id);
        trial[id] = tv;
        F[id] = Fv;
        const double ph = fbphi(tv - l, fbphi(1.0 - tv, -Fv));
        acc_m += ph * ph;
        if (act) {
            const double zeta = scal[S_ZETA];
            const bool lo = (tv - l <= zeta) && (Fv > 0.0);
            const bool up = (1.0 - tv <= zeta) && (Fv < 0.0) && !lo;
            act[id] = lo ? 1 : (up ? 2 : 0);
            acc_n += (lo || up) ? 0.0 : 1.0;
        }
    }
    template <int PAT>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], double (&c00)[NC],
                         double (&c10)[NC], double (&c01)[NC], double (&c11)[NC], bool own) {
        double X[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        long long cv = 0;
        if constexpr (PAT == PF_CROSSED) { cv = ctr(g, ci, j); X[4] = tval(cv); }
        double Y[5] = {0, 0, 0, 0, 0};
        const long long cell = cid(g, ci, j);
        const double kc = cellGc(g, cell) / g.cw;
        for_each_elem<PAT>((ci + j) & 1, [&](auto T, auto S, auto A, auto B, auto C) {
            const double kap = __ldg(kappa + (long long)S.v * g.ncell + cell);
            elem_kaa<T.v, A.v, B.v, C.v>(g, kap, kc, X, Y);
        });
        c00[0] = Y[0]; c10[0] = Y[1]; c01[0] = Y[2]; c11[0] = Y[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) finish_vertex(cv, X[4], Y[4] + __ldg(cvec + cv));
        }
    }
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        finish_vertex(id, v[0], t[0] + __ldg(cvec + id));
    }
    __device__ void finish() {
        double v[2] = {acc_m, acc_n};
        double* s = scal;
        const int ms = merit_slot;
        grid_reduce<2>(v, rb, 1, [s, ms](double* tot) {
            s[ms] = tot[0];
            s[S_NINACT] = tot[1];
        });
    }
};

// ================================================================================================
// Physics pass: energies (fem.py:162-174), r_u (fem.py:177-189), r_alpha (fem.py:202-218) and
// the FB optimality residual (solver.py:104-118).  rows: PF_ROWS_RAW / ZERO / VALUE.
// Reductions -> scal[S_PHYS0 ..]: E_el, E_d, |r_u|^2, |Phi|^2.
// ================================================================================================
template <int ROWS>
struct OpPhys {
    static constexpr int NV = 3, NC = 3;
    const double* u;
    const double* alpha;
    const double* lb;
    double* ru;
    double* ra;
    double* phi;
    double* scal;
    RedBuf rb;
    double eel, ed, nru, nphi;
    __device__ bool enter() const { return true; }
    __device__ void load(const Geo2& g, int i, int j, double (&v)[NV]) const {
        const long long id = vid(g, i, j);
        const double2 uv = ld2(u, id);
        v[0] = uv.x; v[1] = uv.y; v[2] = __ldg(alpha + id);
    }
    __device__ __forceinline__ void vertex_out(const Geo2& g, long long id, unsigned m, double r0,
                                               double r1, double rav, double av) {
        if (m) {
            if (ROWS == PF_ROWS_ZERO) {
                if (m & 1u) r0 = 0.0;
                if (m & 2u) r1 = 0.0;
            } else if (ROWS == PF_ROWS_VALUE) {
                const double2 uv = ld2(u, id);
                const double2 ub = ld2(g.ubar, id);
                if (m & 1u) r0 = uv.x - ub.x;
                if (m & 2u) r1 = uv.y - ub.y;
            }
        }
        if (ru) st2(ru, id, r0, r1);
        if (ra) ra[id] = rav;
        nru += r0 * r0 + r1 * r1;
        if (lb) {
            const double ph = fbphi(av - __ldg(lb + id), fbphi(1.0 - av, -rav));
            if (phi) phi[id] = ph;
            nphi += ph * ph;
        }
    }
    template <int PAT>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], double (&c00)[NC],
                         double (&c10)[NC], double (&c01)[NC], double (&c11)[NC], bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        double Al[5] = {vc[2], vn[2], rc[2], rn[2], 0.0};
        long long cv = 0;
        if constexpr (PAT == PF_CROSSED) {
            cv = ctr(g, ci, j);
            const double2 uv = ld2(u, cv);
            U1[4] = uv.x; U2[4] = uv.y; Al[4] = __ldg(alpha + cv);
        }
        double Y1[5] = {0, 0, 0, 0, 0}, Y2[5] = {0, 0, 0, 0, 0}, Ya[5] = {0, 0, 0, 0, 0};
        const long long cell = cid(g, ci, j);
        const double Ec = cellE(g, cell);
        const double kc = cellGc(g, cell) / g.cw;
        for_each_elem<PAT>((ci + j) & 1, [&](auto T, auto, auto A, auto B, auto C) {
            const double ab = (Al[A.v] + Al[B.v] + Al[C.v]) * (1.0 / 3.0);
            const double om = 1.0 - ab;
            const double a = om * om + g.kell, ap = -2.0 * om;
            const double w = g.at2 ? ab * ab : ab, wp = g.at2 ? 2.0 * ab : 1.0;
            const double ar = g.area[T.v];
            double e0, e1, e2, s0, s1, s2;
            strain<T.v, A.v, B.v, C.v>(g, U1, U2, e0, e1, e2);
            if (g.eps0) {
                const double e = __ldg(g.eps0 + (long long)T.v * g.ny + j);
                e0 -= e; e1 -= e;
            }
            unit_stress(g, e0, e1, e2, s0, s1, s2);
            const double q = Ec * (e0 * s0 + e1 * s1 + e2 * s2);
            const double s = a * ar * Ec;
            scatter_BT<T.v, A.v, B.v, C.v>(g, s * s0, s * s1, s * s2, Y1, Y2);
            const double* b = g.gb[T.v];
            const double* c = g.gc[T.v];
            const double gx = b[0] * Al[A.v] + b[1] * Al[B.v] + b[2] * Al[C.v];
            const double gy = c[0] * Al[A.v] + c[1] * Al[B.v] + c[2] * Al[C.v];
            const double nod = (0.5 * ap * q + kc * wp / g.ell) * ar * (1.0 / 3.0);
            const double del = 2.0 * kc * g.ell * ar;
            Ya[A.v] += nod + del * (b[0] * gx + c[0] * gy);
            Ya[B.v] += nod + del * (b[1] * gx + c[1] * gy);
            Ya[C.v] += nod + del * (b[2] * gx + c[2] * gy);
            if (own) {
                eel += 0.5 * ar * a * q;
                ed += ar * kc * (w / g.ell + g.ell * (gx * gx + gy * gy));
            }
        });
        c00[0] = Y1[0]; c00[1] = Y2[0]; c00[2] = Ya[0];
        c10[0] = Y1[1]; c10[1] = Y2[1]; c10[2] = Ya[1];
        c01[0] = Y1[2]; c01[1] = Y2[2]; c01[2] = Ya[2];
        c11[0] = Y1[3]; c11[1] = Y2[3]; c11[2] = Ya[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) vertex_out(g, cv, 0u, Y1[4], Y2[4], Ya[4], Al[4]);
        }
    }
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        vertex_out(g, id, bcbits(g, i, j, id), t[0], t[1], t[2], v[2]);
    }
    __device__ void finish() {
        double v[4] = {eel, ed, nru, nphi};
        double* s = scal;
        grid_reduce<4>(v, rb, 2, [s](double* tot) {
            s[S_PHYS0 + 0] = tot[0];
            s[S_PHYS0 + 1] = tot[1];
            s[S_PHYS0 + 2] = tot[2];
            s[S_PHYS0 + 3] = tot[3];
        });
    }
};

// ================================================================================================
// Elastic right-hand side with symmetric Dirichlet elimination (fem.py:192-199, 297-310):
// b = M (f - K g) + (I - M) ubar = -M r_raw(g) + (I - M) ubar, g = ubar on constrained dofs.
// With LOADONLY the output is f itself (assemble_load_u).  Reduces |b|^2 into scal[S_RR].
// ================================================================================================
template <bool LOADONLY>
struct OpRhs {
    static constexpr int NV = 3, NC = 2;
    const double* alpha;
    double* b;
    double* scal;
    RedBuf rb;
    double acc;
    __device__ bool enter() const { return true; }
    __device__ void load(const Geo2& g, int i, int j, double (&v)[NV]) const {
        const long long id = vid(g, i, j);
        v[0] = 0.0; v[1] = 0.0;
        if (!LOADONLY) {
            const unsigned m = bcbits(g, i, j, id);
            if (m) {
                const double2 ub = ld2(g.ubar, id);
                if (m & 1u) v[0] = ub.x;
                if (m & 2u) v[1] = ub.y;
            }
        }
        v[2] = __ldg(alpha + id);
    }
    template <int PAT>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], double (&c00)[NC],
                         double (&c10)[NC], double (&c01)[NC], double (&c11)[NC], bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        double Al[5] = {vc[2], vn[2], rc[2], rn[2], 0.0};
        long long cv = 0;
        if constexpr (PAT == PF_CROSSED) { cv = ctr(g, ci, j); Al[4] = __ldg(alpha + cv); }
        double Y1[5] = {0, 0, 0, 0, 0}, Y2[5] = {0, 0, 0, 0, 0};
        const double Ec = cellE(g, cid(g, ci, j));
        for_each_elem<PAT>((ci + j) & 1, [&](auto T, auto, auto A, auto B, auto C) {
            const double ab = (Al[A.v] + Al[B.v] + Al[C.v]) * (1.0 / 3.0);
            const double om = 1.0 - ab;
            const double s = (om * om + g.kell) * g.area[T.v] * Ec;
            double e0 = 0.0, e1 = 0.0, e2 = 0.0, s0, s1, s2;
            if (!LOADONLY) strain<T.v, A.v, B.v, C.v>(g, U1, U2, e0, e1, e2);
            if (g.eps0) {
                const double e = __ldg(g.eps0 + (long long)T.v * g.ny + j);
                e0 -= e; e1 -= e;
            }
            unit_stress(g, e0, e1, e2, s0, s1, s2);
            // r_raw = K g - f  ->  B^T s D (Bg - eps0)
            scatter_BT<T.v, A.v, B.v, C.v>(g, s * s0, s * s1, s * s2, Y1, Y2);
        });
        c00[0] = Y1[0]; c00[1] = Y2[0]; c10[0] = Y1[1]; c10[1] = Y2[1];
        c01[0] = Y1[2]; c01[1] = Y2[2]; c11[0] = Y1[3]; c11[1] = Y2[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) {
                const double b0 = -Y1[4], b1 = -Y2[4];
                st2(b, cv, b0, b1);
                acc += b0 * b0 + b1 * b1;
            }
        }
    }
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        double b0 = -t[0], b1 = -t[1];
        if (!LOADONLY) {
            const unsigned m = bcbits(g, i, j, id);
            if (m & 1u) b0 = v[0];
            if (m & 2u) b1 = v[1];
        }
        st2(b, id, b0, b1);
        acc += b0 * b0 + b1 * b1;
    }
    __device__ void finish() {
        double v[1] = {acc};
        double* s = scal;
        grid_reduce<1>(v, rb, 3, [s](double* tot) { s[S_AUX0] = tot[0]; });  // |b|^2
    }
};

// ================================================================================================
// Coupling blocks (fem.py:246-263): Kua column of element e = (a' |T| E / 3) B^T sigma for each of
// its 3 nodes, sigma = D (B u - eps0).  Kau = Kua^T.  bcmode eliminates Dirichlet rows of Kua
// (columns of Kau).
// ================================================================================================
template <int T, int A, int B, int C>
__device__ __forceinline__ void coupling_vec(const Geo2& g, const double (&U1)[5], const double (&U2)[5],
                                             const double (&Al)[5], double Ec, int j, double& sc,
                                             double& s0, double& s1, double& s2) {
    const double ab = (Al[A] + Al[B] + Al[C]) * (1.0 / 3.0);
    const double ap = -2.0 * (1.0 - ab);
    double e0, e1, e2;
    strain<T, A, B, C>(g, U1, U2, e0, e1, e2);
    if (g.eps0) {
        const double e = __ldg(g.eps0 + (long long)T * g.ny + j);
        e0 -= e; e1 -= e;
    }
    unit_stress(g, e0, e1, e2, s0, s1, s2);
    sc = ap * g.area[T] * Ec * (1.0 / 3.0);
}

struct OpKua : NoRed {
    static constexpr int NV = 4, NC = 2;
    const double* u;
    const double* alpha;
    const double* xa;
    double* yu;
    int bcmode;
    __device__ void load(const Geo2& g, int i, int j, double (&v)[NV]) const {
        const long long id = vid(g, i, j);
        const double2 uv = ld2(u, id);
        v[0] = uv.x; v[1] = uv.y; v[2] = __ldg(alpha + id); v[3] = __ldg(xa + id);
    }
    template <int PAT>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], double (&c00)[NC],
                         double (&c10)[NC], double (&c01)[NC], double (&c11)[NC], bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        double Al[5] = {vc[2], vn[2], rc[2], rn[2], 0.0};
        double X[5] = {vc[3], vn[3], rc[3], rn[3], 0.0};
        long long cv = 0;
        if constexpr (PAT == PF_CROSSED) {
            cv = ctr(g, ci, j);
            const double2 uv = ld2(u, cv);
            U1[4] = uv.x; U2[4] = uv.y; Al[4] = __ldg(alpha + cv); X[4] = __ldg(xa + cv);
        }
        double Y1[5] = {0, 0, 0, 0, 0}, Y2[5] = {0, 0, 0, 0, 0};
        const double Ec = cellE(g, cid(g, ci, j));
        for_each_elem<PAT>((ci + j) & 1, [&](auto T, auto, auto A, auto B, auto C) {
            double sc, s0, s1, s2;
            coupling_vec<T.v, A.v, B.v, C.v>(g, U1, U2, Al, Ec, j, sc, s0, s1, s2);
            const double f = sc * ((X[A.v] + X[B.v]) + X[C.v]);
            scatter_BT<T.v, A.v, B.v, C.v>(g, f * s0, f * s1, f * s2, Y1, Y2);
        });
        c00[0] = Y1[0]; c00[1] = Y2[0]; c10[0] = Y1[1]; c10[1] = Y2[1];
        c01[0] = Y1[2]; c01[1] = Y2[2]; c11[0] = Y1[3]; c11[1] = Y2[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) st2(yu, cv, Y1[4], Y2[4]);
        }
    }
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&)[NV]) {
        const long long id = vid(g, i, j);
        const unsigned m = bcmode ? bcbits(g, i, j, id) : 0u;
        st2(yu, id, (m & 1u) ? 0.0 : t[0], (m & 2u) ? 0.0 : t[1]);
    }
};

struct OpKau : NoRed {
    static constexpr int NV = 5, NC = 1;
    const double* u;
    const double* alpha;
    const double* xu;
    double* ya;
    int bcmode;
    __device__ void load(const Geo2& g, int i, int j, double (&v)[NV]) const {
        const long long id = vid(g, i, j);
        const double2 uv = ld2(u, id);
        const double2 xv = ld2(xu, id);
        const unsigned m = bcmode ? bcbits(g, i, j, id) : 0u;
        v[0] = uv.x; v[1] = uv.y; v[2] = __ldg(alpha + id);
        v[3] = (m & 1u) ? 0.0 : xv.x;
        v[4] = (m & 2u) ? 0.0 : xv.y;
    }
    template <int PAT>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], double (&c00)[NC],
                         double (&c10)[NC], double (&c01)[NC], double (&c11)[NC], bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        double Al[5] = {vc[2], vn[2], rc[2], rn[2], 0.0};
        double X1[5] = {vc[3], vn[3], rc[3], rn[3], 0.0};
        double X2[5] = {vc[4], vn[4], rc[4], rn[4], 0.0};
        long long cv = 0;
        if constexpr (PAT == PF_CROSSED) {
            cv = ctr(g, ci, j);
            const double2 uv = ld2(u, cv);
            const double2 xv = ld2(xu, cv);
            U1[4] = uv.x; U2[4] = uv.y; Al[4] = __ldg(alpha + cv); X1[4] = xv.x; X2[4] = xv.y;
        }
        double Y[5] = {0, 0, 0, 0, 0};
        const double Ec = cellE(g, cid(g, ci, j));
        for_each_elem<PAT>((ci + j) & 1, [&](auto T, auto, auto A, auto B, auto C) {
            double sc, s0, s1, s2, d0, d1, d2;
            coupling_vec<T.v, A.v, B.v, C.v>(g, U1, U2, Al, Ec, j, sc, s0, s1, s2);
            strain<T.v, A.v, B.v, C.v>(g, X1, X2, d0, d1, d2);  // (B x)^T sigma = x^T B^T sigma
            const double f = sc * (d0 * s0 + d1 * s1 + d2 * s2);
            Y[A.v] += f; Y[B.v] += f; Y[C.v] += f;
        });
        c00[0] = Y[0]; c10[0] = Y[1]; c01[0] = Y[2]; c11[0] = Y[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) ya[cv] = Y[4];
        }
    }
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&)[NV]) {
        ya[vid(g, i, j)] = t[0];
    }
};

// ================================================================================================
// Newton: reduced coupled Jacobian [[Kuu_bc, Kua_bc], [Kau_bc, Kaa]] on the inactive set
// (solver.py:292-296 + vi.py:235 with index extraction replaced by masks): active damage rows /
// columns (act != 0) become identity.  One pass reads (u, alpha, x_u, x_a).
// ================================================================================================
struct OpJac : NoRed {
    static constexpr int NV = 6, NC = 3;
    const double* u;
    const double* alpha;
    const double* xu;
    const double* xa;
    double* yu;
    double* ya;
    const unsigned char* act;
    __device__ void load(const Geo2& g, int i, int j, double (&v)[NV]) const {
        const long long id = vid(g, i, j);
        const double2 uv = ld2(u, id);
        const double2 xv = ld2(xu, id);
        const unsigned m = bcbits(g, i, j, id);
        v[0] = uv.x; v[1] = uv.y; v[2] = __ldg(alpha + id);
        v[3] = (m & 1u) ? 0.0 : xv.x;
        v[4] = (m & 2u) ? 0.0 : xv.y;
        v[5] = (act && act[id]) ? 0.0 : __ldg(xa + id);
    }
    template <int PAT>
    __device__ void cell(const Geo2& g, int ci, int j, const double (&vc)[NV], const double (&vn)[NV],
                         const double (&rc)[NV], const double (&rn)[NV], double (&c00)[NC],
                         double (&c10)[NC], double (&c01)[NC], double (&c11)[NC], bool own) {
        double U1[5] = {vc[0], vn[0], rc[0], rn[0], 0.0};
        double U2[5] = {vc[1], vn[1], rc[1], rn[1], 0.0};
        double Al[5] = {vc[2], vn[2], rc[2], rn[2], 0.0};
        double X1[5] = {vc[3], vn[3], rc[3], rn[3], 0.0};
        double X2[5] = {vc[4], vn[4], rc[4], rn[4], 0.0};
        double Xa[5] = {vc[5], vn[5], rc[5], rn[5], 0.0};
        long long cv = 0;
        if constexpr (PAT == PF_CROSSED) {
            cv = ctr(g, ci, j);
            const double2 uv = ld2(u, cv);
            const double2 xv = ld2(xu, cv);
            U1[4] = uv.x; U2[4] = uv.y; Al[4] = __ldg(alpha + cv); X1[4] = xv.x; X2[4] = xv.y;
            Xa[4] = (act && act[cv]) ? 0.0 : __ldg(xa + cv);
        }
        double Y1[5] = {0, 0, 0, 0, 0}, Y2[5] = {0, 0, 0, 0, 0}, Ya[5] = {0, 0, 0, 0, 0};
        const long long cell = cid(g, ci, j);
        const double Ec = cellE(g, cell);
        const double kc = cellGc(g, cell) / g.cw;
        for_each_elem<PAT>((ci + j) & 1, [&](auto T, auto, auto A, auto B, auto C) {
            const double ab = (Al[A.v] + Al[B.v] + Al[C.v]) * (1.0 / 3.0);
            const double om = 1.0 - ab;
            const double a = om * om + g.kell, ap = -2.0 * om;
            const double ar = g.area[T.v];
            double e0, e1, e2, s0, s1, s2, d0, d1, d2, t0, t1, t2;
            strain<T.v, A.v, B.v, C.v>(g, U1, U2, e0, e1, e2);
            if (g.eps0) {
                const double e = __ldg(g.eps0 + (long long)T.v * g.ny + j);
                e0 -= e; e1 -= e;
            }
            unit_stress(g, e0, e1, e2, s0, s1, s2);          // sigma (unit E)
            strain<T.v, A.v, B.v, C.v>(g, X1, X2, d0, d1, d2);
            unit_stress(g, d0, d1, d2, t0, t1, t2);          // D B x_u
            const double q = Ec * (e0 * s0 + e1 * s1 + e2 * s2);
            const double sxa = (Xa[A.v] + Xa[B.v]) + Xa[C.v];
            const double cpl = ap * ar * Ec * (1.0 / 3.0);
            // u rows: a|T|E B^T D B x_u + cpl * sxa * B^T sigma
            const double ka = a * ar * Ec, kb = cpl * sxa;
            scatter_BT<T.v, A.v, B.v, C.v>(g, ka * t0 + kb * s0, ka * t1 + kb * s1,
                                           ka * t2 + kb * s2, Y1, Y2);
            // alpha rows: cpl * (B x_u)^T sigma + Kaa x_a
            const double kap = (q + (g.at2 ? 2.0 * kc / g.ell : 0.0)) * ar * (1.0 / 9.0);
            const double fa = cpl * (d0 * s0 + d1 * s1 + d2 * s2);
            double Yt[5] = {0, 0, 0, 0, 0};
            elem_kaa<T.v, A.v, B.v, C.v>(g, kap, kc, Xa, Yt);
            Ya[A.v] += fa + Yt[A.v];
            Ya[B.v] += fa + Yt[B.v];
            Ya[C.v] += fa + Yt[C.v];
        });
        c00[0] = Y1[0]; c00[1] = Y2[0]; c00[2] = Ya[0];
        c10[0] = Y1[1]; c10[1] = Y2[1]; c10[2] = Ya[1];
        c01[0] = Y1[2]; c01[1] = Y2[2]; c01[2] = Ya[2];
        c11[0] = Y1[3]; c11[1] = Y2[3]; c11[2] = Ya[3];
        if constexpr (PAT == PF_CROSSED) {
            if (own) {
                st2(yu, cv, Y1[4], Y2[4]);
                ya[cv] = (act && act[cv]) ? __ldg(xa + cv) : Ya[4];
            }
        }
    }
    __device__ void out(const Geo2& g, int i, int j, const double (&t)[NC], const double (&v)[NV]) {
        const long long id = vid(g, i, j);
        const unsigned m = bcbits(g, i, j, id);
        double y0 = t[0], y1 = t[1];
        if (m) {
            const double2 xv = ld2(xu, id);
            if (m & 1u) y0 = xv.x;
            if (m & 2u) y1 = xv.y;
        }
        st2(yu, id, y0, y1);
        ya[id] = (act && act[id]) ? __ldg(xa + id) : t[2];
    }
};

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

template <class Op>
static int run_strip(Ctx* c, Op op, cudaStream_t st, int kind = K_VEC, int nw = 0) {
    const Geo2& g = c->g;
    const int nb = strip_blocks(g);
    if (nb > kMaxBlocksRed) return set_error(c, PF_EINVAL, "grid too large for reduction buffer");
    const int slot = prof_begin(c, st);
    switch (g.pattern) {
        case PF_UNION_JACK: k_strip2d<Op, PF_UNION_JACK><<<nb, kBlock, 0, st>>>(g, op); break;
        case PF_RIGHT: k_strip2d<Op, PF_RIGHT><<<nb, kBlock, 0, st>>>(g, op); break;
        default: k_strip2d<Op, PF_CROSSED><<<nb, kBlock, 0, st>>>(g, op); break;
    }
    prof_end(c, st, slot, kind, alg_bytes(c, kind, 0, nw));
    c->launches++;
    return check_cuda(c, cudaGetLastError(), "strip kernel launch");
}

static RedBuf redbuf(Ctx* c) { return RedBuf{c->partials, c->tickets, c->scal}; }

int launch_Kuu(Ctx* c, const double* alpha, const double* x, double* y, int bcmode, cudaStream_t st) {
    OpKuu<false> op{alpha, x, nullptr, nullptr, y, bcmode, c->scal, redbuf(c), 0.0};
    return run_strip(c, op, st, K_KUU);
}
int launch_Kuu_cgA(Ctx* c, const double* alpha, const double* z, const double* p_in, double* p_out,
                   double* q, cudaStream_t st) {
    OpKuu<true> op{alpha, z, p_in, p_out, q, PF_BC_ELIMINATE, c->scal, redbuf(c), 0.0};
    return run_strip(c, op, st, K_KUU_CG);
}
int launch_Kuu_diag(Ctx* c, const double* alpha, double* dinv, cudaStream_t st) {
    OpKuuDiag op;
    op.alpha = alpha;
    op.dinv = dinv;
    return run_strip(c, op, st, K_KUU_DIAG);
}
int launch_kappa(Ctx* c, const double* u, const double* alpha, double* kappa, double* cvec,
                 cudaStream_t st) {
    (void)alpha;
    OpKappa op;
    op.u = u; op.kappa = kappa; op.cvec = cvec;
    return run_strip(c, op, st, K_KAPPA);
}
int launch_Kaa(Ctx* c, const double* kappa, const double* x, double* y, const unsigned char* act,
               cudaStream_t st) {
    if (act) {
        OpKaa<false, true> op{kappa, x, nullptr, nullptr, y, act, c->scal, redbuf(c), 0.0};
        return run_strip(c, op, st, K_KAA);
    }
    OpKaa<false, false> op{kappa, x, nullptr, nullptr, y, nullptr, c->scal, redbuf(c), 0.0};
    return run_strip(c, op, st, K_KAA);
}
int launch_Kaa_cgA(Ctx* c, const double* kappa, const double* z, const double* p_in, double* p_out,
                   double* q, const unsigned char* act, cudaStream_t st) {
    if (act) {
        OpKaa<true, true> op{kappa, z, p_in, p_out, q, act, c->scal, redbuf(c), 0.0};
        return run_strip(c, op, st, K_KAA_CG);
    }
    OpKaa<true, false> op{kappa, z, p_in, p_out, q, nullptr, c->scal, redbuf(c), 0.0};
    return run_strip(c, op, st, K_KAA_CG);
}
int launch_Kaa_diag(Ctx* c, const double* kappa, double* dinv, const unsigned char* act,
                    cudaStream_t st) {
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
    OpKaaTrial op{kappa, cvec, x, d, lb, trial, F, act, c->scal, merit_slot, redbuf(c), 0.0, 0.0};
    return run_strip(c, op, st, K_KAA_TRIAL);
}
int launch_physics(Ctx* c, const double* u, const double* alpha, const double* lb, double* ru,
                   double* ra, double* phi, int rows, cudaStream_t st) {
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
int launch_load(Ctx* c, const double* alpha, double* f, const double* u_or_null, int rows,
                cudaStream_t st) {
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
    OpKua op;
    op.u = u; op.alpha = alpha; op.xa = xa; op.yu = yu; op.bcmode = bcmode;
    return run_strip(c, op, st, K_KUA);
}
int launch_Kau(Ctx* c, const double* u, const double* alpha, const double* xu, double* ya,
               int bcmode, cudaStream_t st) {
    OpKau op;
    op.u = u; op.alpha = alpha; op.xu = xu; op.ya = ya; op.bcmode = bcmode;
    return run_strip(c, op, st, K_KAU);
}
int launch_jac(Ctx* c, const double* u, const double* alpha, const double* xu, const double* xa,
               double* yu, double* ya, const unsigned char* act, cudaStream_t st) {
    OpJac op;
    op.u = u; op.alpha = alpha; op.xu = xu; op.xa = xa; op.yu = yu; op.ya = ya; op.act = act;
    return run_strip(c, op, st, K_JAC);
}

}  // namespace pf
