// glibc_sincos.cuh -- bit-exact restatement of the host libm sin/cos that the
// reference's ray directions go through (rng.py:53: r * np.cos(phi),
// r * np.sin(phi); numba lowers them to libm calls).
//
// On this image that is glibc 2.39's sysdeps/ieee754/dbl-64/s_sin.c, which
// x86-64 dispatches by ifunc to its FMA build (__sin_fma / __cos_fma) on every
// host with FMA + AVX2.  That build lets gcc contract a*b + c into FMA, so the
// rounding of every step depends on where the compiler fused: the functions
// below follow the machine code of __sin_fma / __cos_fma instruction by
// instruction (each GS_FMA is one vfmadd/vfnmadd of the binary, each GS_MUL /
// GS_ADD / GS_SUB one unfused vmulsd / vaddsd / vsubsd), restated in glibc's
// own structure (do_sin, do_cos, reduce_sincos, TAYLOR_SIN).  The range
// covered is |x| < 105414350 (glibc's reduce_sincos range; the ray
// directions only need [0, 2 pi)); larger arguments (glibc's branred) are not
// restated and return NaN.
//
// Compiled for the device (DFMA / DMUL / DADD with explicit rounding, so nvcc
// neither fuses nor splits anything) and for the host (gcc -ffp-contract=off,
// fma() from libm): tests/test_glibc_sincos.py checks the host build against
// math.sin / math.cos over 2^24 arguments of the form 2 pi v and every branch
// boundary, and the GPU tests check the device against the reference's golden
// direction tables.
#pragma once
#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define GS_HD __host__ __device__ __forceinline__
#else
#define GS_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define GS_MUL(a, b) __dmul_rn((a), (b))
#define GS_ADD(a, b) __dadd_rn((a), (b))
#define GS_SUB(a, b) __dsub_rn((a), (b))
#define GS_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define GS_MUL(a, b) ((a) * (b))
#define GS_ADD(a, b) ((a) + (b))
#define GS_SUB(a, b) ((a) - (b))
#define GS_FMA(a, b, c) fma((a), (b), (c))
#endif

namespace rtsdf {
namespace gs {

#ifdef __CUDACC__
#define RTSDF_GS_TABLE_DECL __device__ __align__(32) const double gs_table_dev[RTSDF_GS_TABLE_N]
#include "glibc_sincostab.inc"
#undef RTSDF_GS_TABLE_DECL
#endif
#define RTSDF_GS_TABLE_DECL static const double gs_table_host[RTSDF_GS_TABLE_N]
#include "glibc_sincostab.inc"
#undef RTSDF_GS_TABLE_DECL

// the four entries {sin hi, sin lo, cos hi, cos lo} of table row k (k % 4 == 0):
// one 256-bit load of one 32-B sector on the device instead of four 64-bit
// loads of per-lane random sectors
GS_HD void tab4(int k, double& sn, double& ssn, double& cs, double& ccs) {
#if defined(__CUDA_ARCH__)
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(sn), "=d"(ssn), "=d"(cs), "=d"(ccs)
        : "l"(gs_table_dev + k));
#else
    sn = gs_table_host[k];
    ssn = gs_table_host[k + 1];
    cs = gs_table_host[k + 2];
    ccs = gs_table_host[k + 3];
#endif
}

GS_HD uint64_t bits(double x) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
#endif
}
GS_HD double from_bits(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}
GS_HD double gabs(double x) { return from_bits(bits(x) & 0x7fffffffffffffffull); }
GS_HD double gneg(double x) { return from_bits(bits(x) ^ 0x8000000000000000ull); }
GS_HD double gcopysign(double m, double s) {
    return from_bits((bits(m) & 0x7fffffffffffffffull) | (bits(s) & 0x8000000000000000ull));
}

// constants of s_sin.c / usncs.h (values as stored in the binary)
// On the device the constants whose low word is non-zero are read from the
// constant bank (a DFMA / DMUL / DADD operand, c[3][...]): as literals they were
// re-materialised with two UMOVs per use inside the ray loop (~60 per ray).
#ifdef __CUDACC__
__constant__ double gs_kc[16] = {0x1.45f306dc9c883p-1, 0x1.921fb54442d18p+0, 0x1.1a62633145c07p-54, 0x1.921fb58p+0, -0x1.dde973cp-27, -0x1.cb3b398p-55, -0x1.d747f23e32ed7p-83, -0x1.5555555555515p-3, 0x1.11110e829872fp-7, -0x1.5555555555535p-5, 0x1.6c16bedd9e239p-10, -0x1.5555555555555p-3, 0x1.1111111110ecep-7, -0x1.a01a019db08b8p-13, 0x1.71de27b9a7ed9p-19, -0x1.addffc2fcdf59p-26};
#endif
#if defined(__CUDA_ARCH__)
#define GS_K(i, v) (gs_kc[i])
#else
#define GS_K(i, v) (v)
#endif
#define GS_BIG 0x1.8p+45          // 52776558133248
#define GS_TOINT 0x1.8p+52        // 6755399441055744
#define GS_HPINV GS_K(0, 0x1.45f306dc9c883p-1)
#define GS_HP0 GS_K(1, 0x1.921fb54442d18p+0)
#define GS_HP1 GS_K(2, 0x1.1a62633145c07p-54)
#define GS_MP1 GS_K(3, 0x1.921fb58p+0)
#define GS_MP2 GS_K(4, -0x1.dde973cp-27)
#define GS_PP3 GS_K(5, -0x1.cb3b398p-55)
#define GS_PP4 GS_K(6, -0x1.d747f23e32ed7p-83)
#define GS_SN3 GS_K(7, -0x1.5555555555515p-3)
#define GS_SN5 GS_K(8, 0x1.11110e829872fp-7)
#define GS_CS2 0x1p-1
#define GS_CS4 GS_K(9, -0x1.5555555555535p-5)
#define GS_CS6 GS_K(10, 0x1.6c16bedd9e239p-10)
#define GS_S1 GS_K(11, -0x1.5555555555555p-3)
#define GS_S2 GS_K(12, 0x1.1111111110ecep-7)
#define GS_S3 GS_K(13, -0x1.a01a019db08b8p-13)
#define GS_S4 GS_K(14, 0x1.71de27b9a7ed9p-19)
#define GS_S5 GS_K(15, -0x1.addffc2fcdf59p-26)

// TAYLOR_SIN(xx, a, da) = a + ((POLY(xx) * a - 0.5 * da) * xx + da)
// (__sin_fma: the chain of 5 vfmadd213sd, vfmsub132sd, vfmadd132sd, vaddsd)
GS_HD double taylor_sin(double a, double da) {
    const double xx = GS_MUL(a, a);
    double p = GS_FMA(xx, GS_S5, GS_S4);
    p = GS_FMA(xx, p, GS_S3);
    p = GS_FMA(xx, p, GS_S2);
    p = GS_FMA(xx, p, GS_S1);
    const double t = GS_FMA(p, a, gneg(GS_MUL(da, 0.5)));
    return GS_ADD(a, GS_FMA(xx, t, da));
}

// do_sin(x, dx): table path for 0.126 <= |x| < 0.855469 (plus the reduced
// argument's tail dx); TAYLOR_SIN below 0.126
GS_HD double do_sin(double x, double dx) {
    const double xold = x;
    if (gabs(x) < 0.126) return taylor_sin(x, dx);
    if (x <= 0.0) dx = gneg(dx);
    const double u = GS_ADD(gabs(x), GS_BIG);
    const int k = (int)((uint32_t)bits(u) << 2);
    x = GS_SUB(gabs(x), GS_SUB(u, GS_BIG));
    const double xx = GS_MUL(x, x);
    const double s = GS_ADD(x, GS_FMA(GS_MUL(x, xx), GS_FMA(xx, GS_SN5, GS_SN3), dx));
    const double c = GS_FMA(x, dx, GS_MUL(xx, GS_FMA(xx, GS_FMA(xx, GS_CS6, GS_CS4), GS_CS2)));
    double sn, ssn, cs, ccs;
    tab4(k, sn, ssn, cs, ccs);
    // cor = (ssn + s * ccs - sn * c) + cs * s
    const double cor = GS_FMA(s, cs, GS_FMA(gneg(c), sn, GS_FMA(s, ccs, ssn)));
    return gcopysign(GS_ADD(sn, cor), xold);
}

// do_cos(x, dx)
GS_HD double do_cos(double x, double dx) {
    if (x < 0.0) dx = gneg(dx);
    const double u = GS_ADD(gabs(x), GS_BIG);
    const int k = (int)((uint32_t)bits(u) << 2);
    x = GS_ADD(GS_SUB(gabs(x), GS_SUB(u, GS_BIG)), dx);
    const double xx = GS_MUL(x, x);
    const double s = GS_FMA(GS_MUL(x, xx), GS_FMA(xx, GS_SN5, GS_SN3), x);
    const double c = GS_MUL(xx, GS_FMA(xx, GS_FMA(xx, GS_CS6, GS_CS4), GS_CS2));
    double sn, ssn, cs, ccs;
    tab4(k, sn, ssn, cs, ccs);
    // cor = (ccs - s * ssn - cs * c) - sn * s
    const double cor = GS_FMA(gneg(s), sn, GS_FMA(gneg(c), cs, GS_FMA(gneg(s), ssn, ccs)));
    return GS_ADD(cs, cor);
}

// reduce_sincos: x = n pi/2 + (a + da)
GS_HD int reduce_sincos(double x, double& a, double& da) {
    const double t = GS_FMA(x, GS_HPINV, GS_TOINT);
    const double xn = GS_SUB(t, GS_TOINT);
    const int n = (int)(bits(t) & 3);
    const double y = GS_FMA(gneg(xn), GS_MP2, GS_FMA(gneg(xn), GS_MP1, x));
    const double t2 = GS_FMA(gneg(xn), GS_PP3, y);
    double db = GS_FMA(gneg(xn), GS_PP3, GS_SUB(y, t2));
    const double b = GS_FMA(gneg(xn), GS_PP4, t2);
    db = GS_ADD(db, GS_FMA(gneg(xn), GS_PP4, GS_SUB(t2, b)));
    a = b;
    da = db;
    return n;
}

GS_HD double do_sincos(double a, double da, int n) {
    const double r = (n & 1) ? do_cos(a, da) : do_sin(a, da);
    return (n & 2) ? gneg(r) : r;
}

GS_HD double glibc_sin(double x) {
    const uint32_t k = (uint32_t)(bits(x) >> 32) & 0x7fffffffu;
    if (k < 0x3e500000u) return x;
    if (k < 0x3feb6000u) return do_sin(x, 0.0);
    if (k < 0x400368fdu) return gcopysign(do_cos(GS_SUB(GS_HP0, gabs(x)), GS_HP1), x);
    if (k < 0x419921fbu) {
        double a, da;
        const int n = reduce_sincos(x, a, da);
        return do_sincos(a, da, n);
    }
    return from_bits(0x7ff8000000000000ull);  // not restated (branred / non-finite)
}

GS_HD double glibc_cos(double x) {
    const uint32_t k = (uint32_t)(bits(x) >> 32) & 0x7fffffffu;
    if (k < 0x3e400000u) return 1.0;
    if (k < 0x3feb6000u) return do_cos(x, 0.0);
    if (k < 0x400368fdu) {
        const double y = GS_SUB(GS_HP0, gabs(x));
        const double a = GS_ADD(y, GS_HP1);
        const double da = GS_ADD(GS_SUB(y, a), GS_HP1);
        return do_sin(a, da);
    }
    if (k < 0x419921fbu) {
        double a, da;
        const int n = reduce_sincos(x, a, da);
        return do_sincos(a, da, n + 1);
    }
    return from_bits(0x7ff8000000000000ull);
}

// ---------------------------------------------------------------------------
// (sin x, cos x) for 0 <= x < 105414350 as ONE straight-line evaluation with
// no data-dependent branch -- the form the sampler uses for phi = 2 pi v.
// glibc picks a different formula per range of x (and per quadrant n after
// reduction), so 32 random directions in a warp would run up to six paths one
// after another.  Every pair (sin, cos) is however exactly one do_sin(A, DA)
// and one do_cos(B, DB) on per-range arguments:
//   |x| < 0.855469:   sin = do_sin(x, 0)             cos = do_cos(x, 0)
//   |x| < 2.426265:   sin = |do_cos(hp0 - x, hp1)|    cos = do_sin(a, da)  (a + da = hp0 - x)
//   otherwise:        x = n pi/2 + (a + da); {do_sin(a, da), do_cos(a, da)}
//                     placed and negated by n (do_sincos(., n) / (., n + 1))
// plus glibc's tiny-argument returns (sin = x below 2^-26, cos = 1 below
// 2^-27).  The arguments are chosen by selects, TAYLOR_SIN and the table path
// of do_sin are both evaluated and selected, and every operation is the one
// glibc_sin / glibc_cos perform on that input -- so the results are bit-
// identical to them (tests/test_glibc_sincos.py checks it on both sides of
// every range boundary).
GS_HD double sel(bool p, double a, double b) { return p ? a : b; }

GS_HD double do_sin_nb(double x, double dx) {
    const double xold = x;
    const double tay = taylor_sin(x, dx);
    const double d2 = (x <= 0.0) ? gneg(dx) : dx;
    const double ax = gabs(x);
    const double u = GS_ADD(ax, GS_BIG);
    const int k = (int)((uint32_t)bits(u) << 2) & 511;  // the taylor lanes index anything: keep in range
    const double xr = GS_SUB(ax, GS_SUB(u, GS_BIG));
    const double xx = GS_MUL(xr, xr);
    const double s = GS_ADD(xr, GS_FMA(GS_MUL(xr, xx), GS_FMA(xx, GS_SN5, GS_SN3), d2));
    const double c = GS_FMA(xr, d2, GS_MUL(xx, GS_FMA(xx, GS_FMA(xx, GS_CS6, GS_CS4), GS_CS2)));
    const int kk = k < RTSDF_GS_TABLE_N - 3 ? k : 0;
    double sn, ssn, cs, ccs;
    tab4(kk, sn, ssn, cs, ccs);
    const double cor = GS_FMA(s, cs, GS_FMA(gneg(c), sn, GS_FMA(s, ccs, ssn)));
    const double tab_r = gcopysign(GS_ADD(sn, cor), xold);
    return sel(ax < 0.126, tay, tab_r);
}

GS_HD void glibc_sincos_nb(double x, double& sn_out, double& cs_out) {
    const uint32_t kx = (uint32_t)(bits(x) >> 32) & 0x7fffffffu;
    const bool r1 = kx < 0x3feb6000u, r2 = !r1 && kx < 0x400368fdu, r3 = !r1 && !r2;
    // range 2 arguments
    const double y = GS_SUB(GS_HP0, gabs(x));
    const double a2 = GS_ADD(y, GS_HP1);
    const double da2 = GS_ADD(GS_SUB(y, a2), GS_HP1);
    // range 3 reduction (harmless on the other lanes)
    double a3, da3;
    const int n = reduce_sincos(x, a3, da3);
    const double sa = sel(r1, x, sel(r2, a2, a3)), sda = sel(r1, 0.0, sel(r2, da2, da3));
    const double ca = sel(r1, x, sel(r2, y, a3)), cda = sel(r1, 0.0, sel(r2, GS_HP1, da3));
    const double S = do_sin_nb(sa, sda);
    const double Cc = do_cos(ca, cda);
    // range 3 placement: sin = do_sincos(n), cos = do_sincos(n + 1)
    const int m = n + 1;
    double s3 = (n & 1) ? Cc : S;
    s3 = (n & 2) ? gneg(s3) : s3;
    double c3 = (m & 1) ? Cc : S;
    c3 = (m & 2) ? gneg(c3) : c3;
    double so = sel(r1, S, sel(r2, gcopysign(Cc, x), s3));
    double co = sel(r1, Cc, sel(r2, S, c3));
    so = sel(kx < 0x3e500000u, x, so);
    co = sel(kx < 0x3e400000u, 1.0, co);
    (void)r3;
    sn_out = so;
    cs_out = co;
}

}  // namespace gs
}  // namespace rtsdf
