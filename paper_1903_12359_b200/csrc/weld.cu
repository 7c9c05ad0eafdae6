// weld.cu -- K4: boundary welding on the device (welding.py:79-842).
//
// A weld's map log is a short sequence of primitive records (Mobius, square
// root ratio, opening, closing, square-Mobius). Every record parameter
// depends only on the shared-arc points and the two tracking points (0, inf):
//   SqrtRatio(pts[0], pts[1]); Open(pts[j]) j = 2..k; axis-Mobius(pts[0]);
//   Close(va[j], vb[j]) j = k-1..1; SquareMobius(va[0]); 3-point Mobius(aux).
// So a weld runs in two phases:
//   phase 1  one thread-block cluster per weld (up to 16 CTAs) holds the
//            2(k+3) arc + tracking points in the CTAs' shared memory / registers.
//            k_phase1w (default, "wavefront"): the record chain runs inside
//            the warp that holds the next parameter points (shuffles, no
//            barrier); the other warps and CTAs follow through shared-memory
//            rings filled by a forwarder warp over DSMEM (see the comment
//            above k_phase1w). k_phase1c (PGCP_WELD_WAVE=0, the round-1 form):
//            per record step the owners publish the parameter points into
//            every CTA through DSMEM, one cluster barrier, then every thread
//            rebuilds the record. The two are bit-identical;
//   phase 2  every other tracked point of the two components (non-arc cycle
//            points and interior seam points: the reference's `apply_log` on
//            "others", pipeline.py:200-204) replays its side's log
//            independently. k_replay_stream runs concurrently with phase 1
//            as its programmatic dependent launch, applying records as soon
//            as phase 1's published per-log record counter covers them
//            (PGCP_WELD_STREAM=0: the serial k_replay_slots after phase 1).
// Welds of one schedule level touch disjoint components and run as one
// launch (one cluster each); checks whose inputs span all points (the
// far-end and seam scale tests, welding.py:689-692 and 721-729) are finished
// after phase 2 from per-step maxima.
//
// Numerics: complex division follows numpy's algorithm, the square root
// glibc's csqrt; record semantics (pins, side tags, infinity handling) follow
// the reference record by record. Results agree with the reference to
// rounding (<= 1e-9 relative: tests/test_gpu_pipeline.py
// test_welds_match_reference / test_weld_corpus, and the k >= 1000 welds of
// cfg 2 in tests/test_gpu_cfg2.py), not bit for bit.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>

#include <cooperative_groups.h>

#include "common.cuh"

namespace pgcp {
namespace weld {

enum : int { R_MOB = 0, R_SQR = 1, R_OPEN = 2, R_CLOSE = 3, R_SQ = 4 };
enum : int { FREE = 0, UP = 1, DOWN = -1 };

using Rec = pgcp_rec;

__device__ __forceinline__ double2 C(double x, double y) { return make_double2(x, y); }
__device__ __forceinline__ double2 cinf() { return make_double2(INFINITY, 0.0); }
__device__ __forceinline__ bool c_isinf(double2 z) { return isinf(z.x) || isinf(z.y); }
__device__ __forceinline__ bool c_fin(double2 z) { return isfinite(z.x) && isfinite(z.y); }
__device__ __forceinline__ bool c_nan(double2 z) { return isnan(z.x) || isnan(z.y); }
__device__ __forceinline__ bool c_eq(double2 a, double2 b) { return a.x == b.x && a.y == b.y; }
__device__ __forceinline__ bool c_zero(double2 a) { return a.x == 0.0 && a.y == 0.0; }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return C(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return C(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cneg(double2 a) { return C(-a.x, -a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return C(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cscale(double s, double2 a) { return cmul(C(s, 0.0), a); }
__device__ __forceinline__ double cabs_(double2 a) { return hypot(a.x, a.y); }
// |a| > t and |a| < t without the hypot in the common case; same decisions:
// max(|x|,|y|) <= |a| <= sqrt(2) max(|x|,|y|)
__device__ __forceinline__ bool cabs_gt(double2 a, double t) {
    const double m = fmax(fabs(a.x), fabs(a.y));
    if (!(m * 1.5 > t)) return m != m ? (cabs_(a) > t) : false;  // 1.5 > sqrt(2) with margin
    return m > t || cabs_(a) > t;
}
__device__ __forceinline__ bool cabs_lt(double2 a, double t) {
    const double m = fmax(fabs(a.x), fabs(a.y));
    if (m >= t) return false;
    return cabs_(a) < t;
}

// numpy's complex division (Smith's method with a reciprocal). The two
// orientations are one instruction stream with selects (same operations,
// same roundings): lanes of a warp that fall on different sides of
// |Re b| >= |Im b| no longer run both halves one after the other.
__device__ double2 cdiv(double2 a, double2 b) {
    const double abr = fabs(b.x), abi = fabs(b.y);
    if (abr == 0.0 && abi == 0.0) return C(a.x / abr, a.y / abi);
    const bool rb = abr >= abi;
    const double p = rb ? b.x : b.y, q = rb ? b.y : b.x;  // |p| >= |q|
    const double u = rb ? a.x : a.y, v = rb ? a.y : a.x;
    const double rat = q / p;
    const double scl = 1.0 / fma(q, rat, p);
    // rb: ((a.x + a.y rat), (a.y - a.x rat)) scl; else ((a.x rat + a.y), (a.y rat - a.x)) scl
    const double im = fma(-u, rat, v) * scl;
    return C(fma(v, rat, u) * scl, rb ? im : -im);
}

// |(x, y)|: sqrt(x^2 + y^2) with one rounding of the sum of squares when both
// components are far from overflow and underflow (within an ulp of hypot);
// hypot's scaled evaluation otherwise
__device__ __forceinline__ double fast_hypot(double x, double y) {
    const double ax = fabs(x), ay = fabs(y);
    const double m = fmax(ax, ay), n = fmin(ax, ay);
    if (m < 1e150 && (n > 1e-150 || n == 0.0) && m > 1e-150) return sqrt(fma(ax, ax, ay * ay));
    return hypot(x, y);
}

// principal square root, glibc csqrt's case analysis
__device__ double2 csqrt_(double2 z) {
    double re = z.x, im = z.y;
    if (isnan(re) || isnan(im)) {
        if (isinf(im)) return C(INFINITY, im);
        return C(NAN, NAN);
    }
    if (isinf(im)) return C(INFINITY, im);
    if (isinf(re)) {
        if (re < 0) return C(0.0 * fabs(im), copysign(INFINITY, im));
        return C(re, copysign(0.0, im));
    }
    if (im == 0.0) {
        if (re < 0.0) return C(0.0, copysign(sqrt(-re), im));
        return C(fabs(sqrt(re)), copysign(0.0, im));
    }
    if (re == 0.0) {
        double r = sqrt(0.5 * fabs(im));
        return C(r, copysign(r, im));
    }
    // re > 0: r = sqrt((d + re) / 2), s = im / 2r; else s = sqrt((d - re) / 2),
    // r = |im / 2s| -- one stream with selects (no divergence across lanes)
    const double d = fast_hypot(re, im);
    const double big = sqrt(0.5 * (d + fabs(re)));
    const double small = 0.5 * (im / big);
    const bool pos = re > 0;
    return C(pos ? big : fabs(small), copysign(pos ? small : big, im));
}

__device__ __forceinline__ int rec_side(int flags, int k) { return (int)(int8_t)((flags >> (16 + 8 * k)) & 0xff); }

// principal sqrt of w for Re w != 0, Im w != 0 and moderate magnitudes: the
// csqrt_ formula with one rsqrt for sqrt((d + |re|) / 2) and the division by
// it (within a few ulps of csqrt_; one transcendental fewer on the chain)
__device__ __forceinline__ bool csqrt_fast(double2 w, double2& out) {
    const double m = fmax(fabs(w.x), fabs(w.y)), n = fmin(fabs(w.x), fabs(w.y));
    if (!(m < 1e150 && n > 1e-150)) return false;
    const double d = sqrt(fma(w.x, w.x, w.y * w.y));
    const double h = 0.5 * (d + fabs(w.x));
    const double rs = rsqrt(h);
    const double big = h * rs, small = 0.5 * w.y * rs;
    out = (w.x > 0) ? C(big, small) : C(fabs(small), copysign(big, w.y));
    return true;
}

// the unlabelled Open map sqrt(L^2 - 1), L = pp z / (1 + i qq z) with
// (pp, qq) = xi / |xi|^2, for finite z and moderate magnitudes. Scaled by
// |xi|^2: L = Re(xi) z / (|xi|^2 + i Im(xi) z), so the chain needs neither
// the record's own reciprocal nor Smith's two divisions -- one reciprocal of
// |den|^2 -- and csqrt_fast. The general path below handles every other
// case; results agree within a few ulps.
__device__ __forceinline__ bool open_fast(double2 xi, double2& z) {
    const double s2 = fma(xi.x, xi.x, xi.y * xi.y);
    const double dx = fma(-xi.y, z.y, s2), dy = xi.y * z.x;
    const double nx = xi.x * z.x, ny = xi.x * z.y;
    const double dm = fmax(fabs(dx), fabs(dy)), nm = fmax(fabs(nx), fabs(ny));
    if (!(dm > 1e-100 && dm < 1e100 && nm < 1e100 && (nm > 1e-100 || nm == 0.0))) return false;
    const double inv = 1.0 / fma(dx, dx, dy * dy);
    const double Lx = fma(nx, dx, ny * dy) * inv, Ly = fma(ny, dx, -nx * dy) * inv;
    if (!(fmax(fabs(Lx), fabs(Ly)) < 1e60)) return false;
    double2 r;
    if (!csqrt_fast(C(fma(Lx, Lx, -fma(Ly, Ly, 1.0)), 2.0 * Lx * Ly), r)) return false;
    z = r;
    return true;
}

// Open record body (welding.py OpenRec.apply) on explicit parameters: the
// zip loop keeps xi, Re/|xi|^2, Im/|xi|^2 in registers instead of a record
__device__ __forceinline__ void apply_open(double2 xi, double pp, double qq, int br, double2& z, int8_t& s) {
    if (c_eq(z, xi)) {
        z = C(0.0, 0.0);
        s = (int8_t)br;
        return;
    }
    if (s == 0 && open_fast(xi, z)) return;
    if (s != 0) {
        double t = c_isinf(z) ? INFINITY : z.y;
        double den = 1.0 - qq * t;
        double t2 = (den == 0.0) ? INFINITY : pp * t / den;
        if (isinf(t)) t2 = (qq != 0.0) ? -pp / qq : INFINITY;
        if (!isfinite(t2)) {
            z = cinf();
            return;  // side kept
        }
        double sg = (t2 == 0.0) ? (double)br : (t2 > 0 ? 1.0 : -1.0);
        double h = hypot(t2, 1.0);
        z = C(0.0 * sg, sg * h);
        s = (int8_t)sg;
        return;
    }
    double2 L;
    if (c_isinf(z)) {
        L = (qq != 0.0) ? C(0.0, -(pp / qq)) : cinf();
    } else {
        double2 den = C(1.0 - qq * z.y, qq * z.x);
        L = c_zero(den) ? cinf() : cdiv(C(pp * z.x, pp * z.y), den);
    }
    if (!c_fin(L)) {
        z = cinf();
    } else if (cabs_gt(L, 1e100)) {
        z = (L.x >= 0) ? L : cneg(L);
    } else {
        z = csqrt_(csub(cmul(L, L), C(1.0, 0.0)));
    }
    s = 0;
    return;
}

// the unlabelled Close map sqrt(T^2 + 1), T = z / (c - i d z), for finite z
// and moderate magnitudes: one reciprocal of |den|^2 instead of Smith's two
// divisions, and csqrt_fast (the counterpart of open_fast; every replayed
// cycle point takes this path once per Close record). The general path in
// apply_close handles every other case; results agree within a few ulps.
__device__ __forceinline__ bool close_fast(double c, double d, double2& z) {
    const double dx = fma(d, z.y, c), dy = -d * z.x;
    const double dm = fmax(fabs(dx), fabs(dy)), zm = fmax(fabs(z.x), fabs(z.y));
    if (!(dm > 1e-100 && dm < 1e100 && zm < 1e100 && zm > 1e-100)) return false;
    const double inv = 1.0 / fma(dx, dx, dy * dy);
    const double Tx = fma(z.x, dx, z.y * dy) * inv, Ty = fma(z.y, dx, -z.x * dy) * inv;
    if (!(fmax(fabs(Tx), fabs(Ty)) < 1e60)) return false;
    double2 r;
    if (!csqrt_fast(C(fma(Tx, Tx, -fma(Ty, Ty, -1.0)), 2.0 * Tx * Ty), r)) return false;
    z = r;
    return true;
}

// Close record body (welding.py CloseRec.apply) on explicit parameters
__device__ __forceinline__ void apply_close(double ai, double bi, double c, double d, double2& z, int8_t& s) {
    if (c_eq(z, C(0.0, ai)) || c_eq(z, C(0.0, bi))) {
        z = C(0.0, 0.0);
        s = 0;
        return;
    }
    if (s != 0) {
        double t = c_isinf(z) ? INFINITY : z.y;
        // t / (c + d t) = t (a - b) / ((a + b) t - 2ab): from the record's two
        // points directly, so the chain does not wait for c and d
        const double den2 = fma(ai + bi, t, -2.0 * ai * bi);
        const bool fast = fabs(t) < 1e100 && fabs(den2) > 1e-100 && fabs(den2) < 1e100 && fabs(ai) < 1e100 &&
                          fabs(bi) < 1e100 && ai != bi;
        double t2;
        if (fast) {
            t2 = t * (ai - bi) * (1.0 / den2);
        } else {
            const double den = c + d * t;
            t2 = (den == 0.0) ? INFINITY : t / den;
            if (isinf(t)) t2 = (d != 0.0) ? 1.0 / d : INFINITY;
        }
        if (!isfinite(t2)) {
            z = cinf();
            return;  // side kept
        }
        // |t2| > 1: +-i sqrt(t2^2 - 1) on the axis (side kept by sign); else
        // sqrt(1 - t2^2) on the real line -- selects, one sqrt
        const bool off = fabs(t2) > 1.0;
        const double u = fma(t2, t2, -1.0);
        const double root = sqrt(off ? fmax(u, 0.0) : fmax(-u, 0.0));
        const double mag = (off && !(fabs(t2) < 1e100)) ? fabs(t2) : root;
        const double sg = t2 > 0 ? 1.0 : -1.0;
        z = off ? C(0.0 * sg, sg * mag) : C(mag, 0.0);
        s = off ? (int8_t)(t2 > 0 ? UP : DOWN) : (int8_t)0;
        return;
    }
    if (c_fin(z) && close_fast(c, d, z)) return;  // s == 0 here and stays 0
    double2 T;
    if (c_isinf(z)) {
        T = (d != 0.0) ? C(0.0, 1.0 / d) : cinf();
    } else {
        double2 den = C(c + d * z.y, -d * z.x);
        T = c_zero(den) ? cinf() : cdiv(z, den);
    }
    if (!c_fin(T)) {
        z = cinf();
    } else if (cabs_gt(T, 1e100)) {
        z = (T.x >= 0) ? T : cneg(T);
    } else {
        z = csqrt_(cadd(cmul(T, T), C(1.0, 0.0)));
    }
    s = 0;
    return;
}

__device__ __forceinline__ void close_params(double a, double b, double& c, double& d);
__device__ __forceinline__ void open_params(double2 xi, double& pp, double& qq);

// apply_open from the record's point alone: (pp, qq) are formed only where
// the unlabelled fast path does not apply (as apply_close_ab below)
__device__ __forceinline__ void apply_open_xi(double2 xi, int br, double2& z, int8_t& s) {
    if (s == 0 && !c_eq(z, xi) && c_fin(z) && open_fast(xi, z)) return;
    double pp, qq;
    open_params(xi, pp, qq);
    apply_open(xi, pp, qq, br, z, s);
}

// apply_close from the record's two points: c and d are formed only where
// the labelled fast path does not apply (the wavefront chain's common case
// needs neither, so their division stays off the chain)
__device__ __forceinline__ void apply_close_ab(double ai, double bi, double2& z, int8_t& s) {
    if (s != 0 && !c_isinf(z) && fabs(z.y) < 1e100 && fabs(ai) < 1e100 && fabs(bi) < 1e100 && ai != bi &&
        !(z.x == 0.0 && (z.y == ai || z.y == bi))) {
        const double den2 = fma(ai + bi, z.y, -2.0 * ai * bi);
        if (fabs(den2) > 1e-100 && fabs(den2) < 1e100) {
            apply_close(ai, bi, 0.0, 0.0, z, s);  // takes the fast branch (same conditions)
            return;
        }
    }
    double c, d;
    close_params(ai, bi, c, d);
    apply_close(ai, bi, c, d, z, s);
}

// one record on one point (welding.py:251-509)
__device__ __forceinline__ void apply_rec(const Rec& r, double2& z, int8_t& s) {
    const double* p = r.p;
    switch (r.kind) {
        case R_MOB: {
            double2 a = C(p[0], p[1]), b = C(p[2], p[3]), c = C(p[4], p[5]), d = C(p[6], p[7]);
            bool axis = r.flags & 1;
            int npins = (r.flags >> 8) & 0xff;
            // at most two pins (p[8..15]); static indices keep the record in
            // registers (a dynamic index would put it on the local stack)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                if (k < npins && c_eq(z, C(p[8 + 4 * k], p[9 + 4 * k]))) {
                    z = C(p[10 + 4 * k], p[11 + 4 * k]);
                    s = (int8_t)rec_side(r.flags, k);
                    return;
                }
            }
            if (c_isinf(z)) {
                z = c_zero(c) ? cinf() : cdiv(a, c);
                if (!axis) s = 0;
                return;
            }
            double2 num = cadd(cmul(a, z), b);
            double2 den = cadd(cmul(c, z), d);
            double2 w = c_zero(den) ? cinf() : cdiv(num, den);
            int8_t ns = 0;
            if (axis && s != 0) {
                if (c_fin(w)) {
                    double im = w.y;
                    w = C(signbit(im) ? -0.0 : 0.0, im + 0.0);
                    ns = w.y > 0 ? UP : (w.y < 0 ? DOWN : s);
                } else {
                    ns = s;
                }
            }
            z = w;
            s = ns;
            return;
        }
        case R_SQR: {
            double2 z0 = C(p[0], p[1]), z1 = C(p[2], p[3]);
            int br = (int)(int8_t)(r.flags & 0xff);
            if (c_eq(z, z0)) {
                z = cinf();
                s = (int8_t)br;
            } else if (c_eq(z, z1)) {
                z = C(0.0, 0.0);
                s = (int8_t)br;
            } else if (c_eq(z, cinf())) {
                z = C(1.0, 0.0);
                s = 0;
            } else {
                z = csqrt_(cdiv(csub(z, z1), csub(z, z0)));
                s = 0;
            }
            return;
        }
        case R_OPEN:
            apply_open(C(p[0], p[1]), p[2], p[3], (int)(int8_t)(r.flags & 0xff), z, s);
            return;
        case R_CLOSE:
            apply_close(p[0], p[1], p[2], p[3], z, s);
            return;
        case R_SQ: {
            double2 q = C(p[0], p[1]);
            bool qinf = c_isinf(q);
            if (c_eq(z, q)) {
                z = cinf();
                s = 0;
                return;
            }
            if (!qinf && c_isinf(z)) {
                z = cmul(q, q);
                s = 0;
                return;
            }
            if (s != 0) {
                double t = z.y, t2;
                if (qinf) {
                    t2 = t;
                } else {
                    double den = 1.0 - t / q.y;
                    t2 = (den == 0.0) ? INFINITY : t / den;
                }
                z = isfinite(t2) ? C(-(t2 * t2), 0.0) : cinf();
                s = 0;
                return;
            }
            double2 mm;
            if (qinf) {
                mm = z;
            } else {
                double2 den = csub(C(1.0, 0.0), cdiv(z, q));
                mm = c_zero(den) ? cinf() : cdiv(z, den);
            }
            double2 w = cmul(mm, mm);
            z = c_fin(w) ? w : cinf();
            s = 0;
            return;
        }
        default:
            z = C(NAN, NAN);
    }
}

// The replay kernels walk a log record by record on one point: the apply is
// a ~1.4K-cycle dependent chain, and a record load issued only when the
// previous apply has finished adds its L2 latency to every record. Open and
// Close records (all but ~5 of a log) use kind, flags and p[0..3] only, so the
// replays keep the next record's first 40 bytes in flight during the current
// apply; the other kinds read the whole record when they are applied.
struct RecHead {
    int32_t kind, flags;
    double p0, p1, p2, p3;
};
__device__ __forceinline__ RecHead load_head(const Rec* r) {
    RecHead h;
    const int2 kf = *reinterpret_cast<const int2*>(r);  // kind, flags (8-byte aligned)
    h.kind = kf.x;
    h.flags = kf.y;
    h.p0 = r->p[0];
    h.p1 = r->p[1];
    h.p2 = r->p[2];
    h.p3 = r->p[3];
    return h;
}
// same operations as apply_rec(*full, z, s)
__device__ __forceinline__ void apply_head(const RecHead& h, const Rec* full, double2& z, int8_t& s) {
    if (h.kind == R_OPEN) {
        apply_open(C(h.p0, h.p1), h.p2, h.p3, (int)(int8_t)(h.flags & 0xff), z, s);
    } else if (h.kind == R_CLOSE) {
        apply_close(h.p0, h.p1, h.p2, h.p3, z, s);
    } else {
        apply_rec(*full, z, s);
    }
}

// ---- record constructors (single thread) -----------------------------------

__device__ Rec mk_mob(double2 a, double2 b, double2 c, double2 d, bool axis = false) {
    Rec r;
    r.kind = R_MOB;
    r.flags = axis ? 1 : 0;
    r.p[0] = a.x; r.p[1] = a.y; r.p[2] = b.x; r.p[3] = b.y;
    r.p[4] = c.x; r.p[5] = c.y; r.p[6] = d.x; r.p[7] = d.y;
    for (int i = 8; i < 16; ++i) r.p[i] = 0.0;
    return r;
}
__device__ __forceinline__ void mob_pin(Rec& r, double2 pz, double2 pw, int side) {
    int k = (r.flags >> 8) & 0xff;  // 0 or 1 (two pins at most)
    if (k == 0) {
        r.p[8] = pz.x; r.p[9] = pz.y; r.p[10] = pw.x; r.p[11] = pw.y;
    } else {
        r.p[12] = pz.x; r.p[13] = pz.y; r.p[14] = pw.x; r.p[15] = pw.y;
    }
    r.flags = (r.flags & ~(0xff << 8)) | ((k + 1) << 8);
    r.flags |= ((side & 0xff) << (16 + 8 * k));
}
__device__ Rec mk_sqr(double2 z0, double2 z1, int br) {
    Rec r;
    r.kind = R_SQR;
    r.flags = br & 0xff;
    r.p[0] = z0.x; r.p[1] = z0.y; r.p[2] = z1.x; r.p[3] = z1.y;
    for (int i = 4; i < 16; ++i) r.p[i] = 0.0;
    return r;
}
// (Re, Im) / |xi|^2 of an Open record
__device__ __forceinline__ void open_params(double2 xi, double& pp, double& qq) {
    const double ax = fabs(xi.x), ay = fabs(xi.y);
    double s2;
    if (fmax(ax, ay) < 1e150 && fmax(ax, ay) > 1e-150) {
        s2 = fma(xi.x, xi.x, xi.y * xi.y);
    } else {
        s2 = hypot(xi.x, xi.y);
        s2 = s2 * s2;
    }
    const double inv = 1.0 / s2;
    pp = xi.x * inv;
    qq = xi.y * inv;
}
__device__ Rec mk_open_p(double2 xi, double pp, double qq, int br) {
    Rec r;
    r.kind = R_OPEN;
    r.flags = br & 0xff;
    r.p[0] = xi.x; r.p[1] = xi.y; r.p[2] = pp; r.p[3] = qq;
    for (int i = 4; i < 16; ++i) r.p[i] = 0.0;
    return r;
}
__device__ Rec mk_open(double2 xi, int br) {
    double pp, qq;
    open_params(xi, pp, qq);
    return mk_open_p(xi, pp, qq, br);
}
__device__ __forceinline__ void close_params(double a, double b, double& c, double& d) {
    const double inv = 1.0 / (a - b);
    c = -2 * a * b * inv;
    d = (a + b) * inv;
}
__device__ Rec mk_close_p(double a, double b, double c, double d) {
    Rec r;
    r.kind = R_CLOSE;
    r.flags = 0;
    r.p[0] = a; r.p[1] = b; r.p[2] = c; r.p[3] = d;
    for (int i = 4; i < 16; ++i) r.p[i] = 0.0;
    return r;
}
__device__ Rec mk_close(double a, double b) {
    double c, d;
    close_params(a, b, c, d);
    return mk_close_p(a, b, c, d);
}
__device__ Rec mk_sq(double2 q) {
    Rec r;
    r.kind = R_SQ;
    r.flags = 0;
    r.p[0] = q.x; r.p[1] = q.y;
    for (int i = 2; i < 16; ++i) r.p[i] = 0.0;
    return r;
}

// Mobius taking z_i -> w_i (welding.py:99-133); false if not distinct
__device__ bool three_point(const double2* zs, const double2* ws, double2* co) {
    const double2* trips[2] = {zs, ws};
    for (int t = 0; t < 2; ++t)
        for (int i = 0; i < 3; ++i)
            for (int j = i + 1; j < 3; ++j) {
                bool bi = c_isinf(trips[t][i]), bj = c_isinf(trips[t][j]);
                if ((bi && bj) || (!bi && !bj && c_eq(trips[t][i], trips[t][j]))) return false;
            }
    auto std3 = [](const double2* v, double2* o) {
        double2 z1 = v[0], z2 = v[1], z3 = v[2];
        if (c_isinf(z1)) {
            o[0] = C(0, 0); o[1] = csub(z2, z3); o[2] = C(1, 0); o[3] = cneg(z3);
        } else if (c_isinf(z2)) {
            o[0] = C(1, 0); o[1] = cneg(z1); o[2] = C(1, 0); o[3] = cneg(z3);
        } else if (c_isinf(z3)) {
            o[0] = C(1, 0); o[1] = cneg(z1); o[2] = C(0, 0); o[3] = csub(z2, z1);
        } else {
            double2 d23 = csub(z2, z3), d21 = csub(z2, z1);
            o[0] = d23; o[1] = cmul(cneg(z1), d23); o[2] = d21; o[3] = cmul(cneg(z3), d21);
        }
    };
    double2 m1[4], m2[4];
    std3(zs, m1);
    std3(ws, m2);
    double2 a = csub(cmul(m2[3], m1[0]), cmul(m2[1], m1[2]));
    double2 b = csub(cmul(m2[3], m1[1]), cmul(m2[1], m1[3]));
    double2 c = cadd(cmul(cneg(m2[2]), m1[0]), cmul(m2[0], m1[2]));
    double2 d = cadd(cmul(cneg(m2[2]), m1[1]), cmul(m2[0], m1[3]));
    double nrm = fmax(fmax(cabs_(a), cabs_(b)), fmax(cabs_(c), cabs_(d)));
    co[0] = C(a.x / nrm, a.y / nrm);
    co[1] = C(b.x / nrm, b.y / nrm);
    co[2] = C(c.x / nrm, c.y / nrm);
    co[3] = C(d.x / nrm, d.y / nrm);
    return true;
}

__device__ __forceinline__ int walk_class(double h) { return isinf(h) ? 1 : (h > 0 ? 0 : 2); }
__device__ __forceinline__ bool walk_less(double a, double b) {  // _axis_walk_key(a) < _axis_walk_key(b)
    int ca = walk_class(a), cb = walk_class(b);
    if (ca != cb) return ca < cb;
    if (ca == 1) return false;
    return a < b;
}

// ---------------------------------------------------------------------------
// phase 1

enum : int {
    WE_OK = 0,
    WE_ZIP01 = 1,      // zip points 0 and 1 coincide
    WE_ZIP_HALF = 2,   // zip point j left the right half-plane
    WE_ZIP_AXIS = 3,   // zip point j landed on the imaginary axis
    WE_ZIP_COLL = 4,   // zip points j-1 and j collapsed
    WE_NAN = 5,        // NaN during (aux = stage)
    WE_FAR0 = 6,       // far end of the zip collapsed to 0
    WE_ALIGN_A = 7,    // alignment point j (a side) left the imaginary axis
    WE_ALIGN_B = 8,
    WE_ORDER = 9,      // alignment points j not strictly ordered
    WE_TRACK = 10,     // tracking points degenerated
    WE_FAREND = 11,    // far ends of the two slits diverged
    WE_SEAM = 12,      // seam alignment error
    WE_PRE = 13,       // prenormalizer failure (aux: 1 none finite, 2 coincide, 3 origin)
    WE_THREE = 14,     // three-point Mobius needs distinct points
    WE_K = 15,         // k out of range
    WE_GEO_DISK = 16,  // interior point left the unit disk
    WE_GEO_CIRCLE = 17,
    WE_INTERIOR = 18,  // could not locate a point inside the polygon
};

struct StepDesc {
    int32_t k, closed, na, nb;
    int64_t src;       // offset into src[] (na + nb slot ids)
    int64_t rec;       // record offset of log_a (log_b at rec + cap)
    int32_t cap, pad;
    int64_t arc;       // offset into arc_out (k+1 values of a, then k+1 of b)
};

// per-step meta written by phase 1 / 2 (doubles):
//  0 nrec_a, 1 nrec_b, 2 err code, 3 err index, 4 err aux, 5 seam(arc), 6 qa.re, 7 qa.im,
//  8 qb.re, 9 qb.im, 10 stage max |va| (arc+aux), 11 final max |va| arc, 12 final max |vb| arc,
//  13 final max aux (a,b), 14 sq index a, 15 sq index b, 16 area(res.a arc), 17..19 spare
constexpr int META = 20;

struct Phase1Args {
    const StepDesc* steps;
    const int32_t* src;
    const double2* tv;      // tracked values (read)
    double2* arc_out;
    Rec* recs;
    double* meta;
    int geodesic;           // unused here
    int* prog;              // per step [2]: records published per log (streamed replay), or nullptr
    int prog_every;         // publish the counters every this many logged steps
    long long* timing;      // optional (PGCP_WELD_TIMING): per step [publish+barrier, build, apply, zip steps] cycles
    int spin_ns;            // k_phase1w: back-off of the waiting warps between polls (0: busy spin)
    int timing_detail;      // PGCP_WELD_TIMING=2: per-segment chain split printed by k_phase1w
};

// Streamed replay (k_replay_stream): phase 1 publishes, per step and log, the
// number of records written so far; the replay of the same level runs
// concurrently (programmatic dependent launch) and applies records as they
// appear. Counter word: bits 0..28 count, bit 30 = the step has finished
// (its meta is final). The logger orders its record / meta stores before the
// counter with a gpu-scope release fence.
constexpr int PROG_DONE = 1 << 30;
constexpr int PROG_TIMEOUT = 1 << 29;
constexpr int PROG_COUNT = (1 << 29) - 1;

__device__ __forceinline__ void prog_store(int* p, int v) {
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int prog_load(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ void block_fail(int* s_err, int code, int idx, int aux, double* meta) {
    if (atomicCAS(s_err, 0, code) == 0) {
        meta[2] = code;
        meta[3] = idx;
        meta[4] = aux;
    }
}

// block-wide reductions (any blockDim multiple of 32, <= 1024)
__device__ double block_sum(double v, double* red) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int i = 0; i < nw; ++i) t += red[i];
    __syncthreads();
    return t;
}
__device__ double block_max(double v, double* red) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double t = red[0];
    for (int i = 1; i < nw; ++i) t = fmax(t, red[i]);
    __syncthreads();
    return t;
}

// Prenormalizer (welding.py:609-625) over the n points src[0..n) of tv.
// Every thread below `nth` takes points threadIdx.x, + nth, ... (the others
// add zeros), so the sums do not depend on blockDim beyond nth.
__device__ bool prenormalize(const double2* tv, const int32_t* src, int n, double* red, Rec* out, int* code,
                             int nth = 0) {
    if (nth <= 0) nth = blockDim.x;
    const int i0 = threadIdx.x < nth ? (int)threadIdx.x : n;
    double sx = 0, sy = 0, cnt = 0;
    for (int i = i0; i < n; i += nth) {
        double2 z = tv[src[i]];
        if (c_fin(z)) {
            sx += z.x;
            sy += z.y;
            cnt += 1;
        }
    }
    sx = block_sum(sx, red);
    sy = block_sum(sy, red);
    cnt = block_sum(cnt, red);
    if (cnt == 0) {
        *code = 1;
        return false;
    }
    double2 c = C(sx / cnt, sy / cnt);
    double m = 0;
    for (int i = i0; i < n; i += nth) {
        double2 z = tv[src[i]];
        if (c_fin(z)) m = fmax(m, cabs_(csub(z, c)));
    }
    double s = block_max(m, red);
    if (s == 0) {
        *code = 2;
        return false;
    }
    int tries = 0;
    for (; tries < 4; ++tries) {
        double hit = 0;
        for (int i = i0; i < n; i += nth) {
            double2 z = tv[src[i]];
            if (c_fin(z) && c_eq(z, c)) hit = 1;
        }
        if (block_max(hit, red) == 0) break;
        c = cadd(c, C(s * 0.0137, s * 0.00271));
    }
    if (tries == 4) {
        *code = 3;
        return false;
    }
    *out = mk_mob(C(1.0 / s, 0.0), C(-c.x / s, -c.y / s), C(0.0, 0.0), C(1.0, 0.0));
    return true;
}

// ---------------------------------------------------------------------------
// phase 1 on a thread-block cluster: the 2(k+3) points of one weld are spread
// over the CTAs of a cluster (one point per thread for k ~ 1000); every record
// step is
//   apply the current record to my points -> block barrier -> the owners of
//   the next parameter points publish (value, side) into every CTA's
//   parameter slots through DSMEM -> cluster barrier -> every thread rebuilds
//   the next record from the parameters (identical arithmetic everywhere)
// so the serial chain costs one cluster barrier per record and the O(k^2)
// point work is spread over CS SMs.

constexpr int PC_MAXCS = 16;
constexpr int NPARAM = 8;            // parameter slots per step
constexpr int NFLAG = PC_MAXCS;      // per-rank scalars (maxima)

struct PParam {
    double2 z;
    int s;
    int pad;
};

namespace cgw = cooperative_groups;

struct P1c {
    PParam* slot;       // [2][NPARAM] parameter slots (this CTA's)
    double* flag;       // [2][NFLAG]
    double2* pts;       // my points
    int8_t* sides;
    int lo, hi;         // my global point range [lo, hi)
};

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_phase1c(Phase1Args A) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ PParam s_param[2][NPARAM];
    __shared__ double s_flag[2][NFLAG];
    __shared__ double red[32];
    cgw::cluster_group cl = cgw::this_cluster();
    const int CS = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    const int step = blockIdx.x / CS;
    const StepDesc sd = A.steps[step];
    double* meta = A.meta + META * (int64_t)step;
    const int k = sd.k;
    const int P = k + 3;
    const int NP = 2 * P;
    const int chunk = (NP + CS - 1) / CS;
    const int lo = min(NP, rank * chunk), hi = min(NP, lo + chunk);
    double2* pts = reinterpret_cast<double2*>(smem);
    int8_t* sides = reinterpret_cast<int8_t*>(pts + chunk);
    Rec* log_a = A.recs + sd.rec;
    Rec* log_b = log_a + sd.cap;
    // the logger writes both logs and the progress counters; a thread that
    // owns no point does it, so the record writes stay off the points' path
    const int logger_tid = (hi - lo < NT) ? NT - 1 : 0;
    const bool logger = rank == 0 && (int)threadIdx.x == logger_tid;
    int na_rec = 0, nb_rec = 0, nlogged = 0;
    // every CTA of this grid is resident from here on: the streamed replay
    // (secondary launch) may start and wait on the counters
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    int* prog = A.prog ? A.prog + 2 * step : nullptr;
    auto progress = [&](bool fin) {
        if (!logger || !prog) return;
        if (!fin && (++nlogged % A.prog_every) != 0) return;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        prog_store(prog, na_rec | (fin ? PROG_DONE : 0));
        prog_store(prog + 1, nb_rec | (fin ? PROG_DONE : 0));
    };
    if (logger)
        for (int i = 0; i < META; ++i) meta[i] = 0.0;
    if (k < 1 || k > sd.na - 1 || k > sd.nb - 1) {
        if (logger) {
            meta[2] = WE_K;
            meta[3] = k;
        }
        progress(true);
        return;
    }
    const int32_t* sa = A.src + sd.src;
    const int32_t* sb = sa + sd.na;
    // prenormalizers over all cycle points (computed redundantly by every CTA)
    Rec pre[2];
    int pcode = 0;
    bool okA = prenormalize(A.tv, sa, sd.na, red, &pre[0], &pcode);
    bool okB = okA && prenormalize(A.tv, sb, sd.nb, red, &pre[1], &pcode);
    if (!okA || !okB) {
        if (logger) {
            meta[2] = WE_PRE;
            meta[3] = okA ? 1 : 0;
            meta[4] = pcode;
        }
        progress(true);
        return;
    }
    for (int g = lo + threadIdx.x; g < hi; g += NT) {
        int side = g >= P;
        int t = g - side * P;
        double2 z;
        int8_t sd8 = 0;
        if (t <= k) {
            z = A.tv[(side ? sb : sa)[t]];
            if (side)
                apply_rec(pre[1], z, sd8);
            else
                apply_rec(pre[0], z, sd8);
        } else {
            z = (t == k + 1) ? C(0.0, 0.0) : cinf();
        }
        pts[g - lo] = z;
        sides[g - lo] = 0;
    }
    if (logger) {
        log_a[na_rec++] = pre[0];
        log_b[nb_rec++] = pre[1];
    }
    progress(false);
    int parity = 0;
    // publish the listed global points into every CTA's slots, then barrier
    // the thread that owns point g (the one that last wrote it) sends it, so
    // no CTA barrier is needed before the cluster barrier
    auto publish = [&](const int* gidx, int np, double flag) {
        for (int which = 0; which < np; ++which) {
            int g = gidx[which];
            if (g >= lo && g < hi && (g - lo) % NT == (int)threadIdx.x) {
                PParam pp;
                pp.z = pts[g - lo];
                pp.s = sides[g - lo];
                pp.pad = 0;
                for (int dst = 0; dst < CS; ++dst) {
                    PParam* rs = cl.map_shared_rank(&s_param[parity][0], dst);
                    rs[which] = pp;
                }
            }
        }
        if (threadIdx.x < CS) {
            double* rf = cl.map_shared_rank(&s_flag[parity][0], threadIdx.x);
            rf[rank] = flag;
        }
        cl.sync();
    };
    auto apply_pair = [&](const Rec& ra, bool ua, const Rec& rb, bool ub) {
        for (int g = lo + threadIdx.x; g < hi; g += NT) {
            int side = g >= P;
            if (side ? !ub : !ua) continue;
            double2 z = pts[g - lo];
            int8_t s8 = sides[g - lo];
            if (side)  // separate calls keep both records in registers
                apply_rec(rb, z, s8);
            else
                apply_rec(ra, z, s8);
            pts[g - lo] = z;
            sides[g - lo] = s8;
        }
    };
    int err = 0, eidx = 0, eaux = 0;
    long long tw[3] = {0, 0, 0};  // PGCP_WELD_TIMING
    Rec ra, rb;
    // ---- zip step 1: SqrtRatio
    {
        int gi[4] = {0, 1, P, P + 1};
        publish(gi, 4, 0.0);
        PParam* pp = s_param[parity];
        if (c_eq(pp[0].z, pp[1].z) || c_eq(pp[2].z, pp[3].z)) err = WE_ZIP01;
        ra = mk_sqr(pp[0].z, pp[1].z, UP);
        rb = mk_sqr(pp[2].z, pp[3].z, DOWN);
        parity ^= 1;
    }
    if (err) goto fail;
    if (logger) {
        log_a[na_rec++] = ra;
        log_b[nb_rec++] = rb;
    }
    progress(false);
    apply_pair(ra, true, rb, true);
    // ---- zip steps j = 2..k: Open
    for (int j = 2; j <= k; ++j) {
        const long long w0 = A.timing ? clock64() : 0;
        int gi[2] = {j, P + j};
        publish(gi, 2, 0.0);
        const long long w1 = A.timing ? clock64() : 0;
        PParam* pp = s_param[parity];
        for (int side = 0; side < 2 && !err; ++side) {
            double2 xi = pp[side].z;
            if (pp[side].s != 0 || c_isinf(xi)) {
                err = WE_ZIP_HALF; eidx = j; eaux = side;
            } else if (!(xi.x > 0)) {
                err = WE_ZIP_AXIS; eidx = j; eaux = side;
            } else if (cabs_lt(xi, 1e-13)) {
                err = WE_ZIP_COLL; eidx = j; eaux = side;
            }
        }
        parity ^= 1;
        if (err) goto fail;
        // the Open records as registers (xi, Re/|xi|^2, Im/|xi|^2), not as
        // record structs: a struct the compiler keeps on the stack would be
        // re-read from local memory by every point after every barrier
        const double2 xa = pp[0].z, xb = pp[1].z;
        double pa, qa, pb, qb;
        open_params(xa, pa, qa);
        open_params(xb, pb, qb);
        const long long w2 = A.timing ? clock64() : 0;
        if (logger) {
            log_a[na_rec++] = mk_open_p(xa, pa, qa, UP);
            log_b[nb_rec++] = mk_open_p(xb, pb, qb, DOWN);
        }
        progress(false);
        for (int g = lo + threadIdx.x; g < hi; g += NT) {
            double2 z = pts[g - lo];
            int8_t s8 = sides[g - lo];
            if (g >= P)
                apply_open(xb, pb, qb, DOWN, z, s8);
            else
                apply_open(xa, pa, qa, UP, z, s8);
            pts[g - lo] = z;
            sides[g - lo] = s8;
        }
        if (A.timing) {
            const long long w3 = clock64();
            tw[0] += w1 - w0;
            tw[1] += w2 - w1;
            tw[2] += w3 - w2;
        }
    }
    if (A.timing && rank == 0 && threadIdx.x == 0) {
        A.timing[4 * step + 0] = tw[0];
        A.timing[4 * step + 1] = tw[1];
        A.timing[4 * step + 2] = tw[2];
        A.timing[4 * step + 3] = k - 1;
    }
    // ---- axis Mobius sending pts[0] to infinity (welding.py:593-600)
    {
        int gi[2] = {0, P};
        publish(gi, 2, 0.0);
        PParam* pp = s_param[parity];
        bool has[2] = {false, false};
        Rec rr0, rr1;
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            if (err) break;
            double2 w0 = pp[side].z;
            if (!c_isinf(w0)) {
                if (c_zero(w0)) {
                    err = WE_FAR0; eaux = side;
                } else {
                    int br = side ? DOWN : UP;
                    Rec& rs = side ? rr1 : rr0;
                    rs = mk_mob(C(1, 0), C(0, 0), cdiv(C(-1.0, 0.0), w0), C(1, 0), true);
                    mob_pin(rs, w0, cinf(), br);
                    mob_pin(rs, C(0, 0), C(0, 0), br);
                    has[side] = true;
                }
            }
        }
        parity ^= 1;
        if (err) goto fail;
        if (logger) {
            if (has[0]) log_a[na_rec++] = rr0;
            if (has[1]) log_b[nb_rec++] = rr1;
        }
        progress(false);
        apply_pair(rr0, has[0], rr1, has[1]);
    }
    // ---- closing loop (welding.py:673-687)
    for (int j = k - 1; j >= 1; --j) {
        int gi[2] = {j, P + j};
        publish(gi, 2, 0.0);
        PParam* pp = s_param[parity];
        double2 al = pp[0].z, be = pp[1].z;
        if (pp[0].s == 0 || c_isinf(al) || al.y == 0.0) {
            err = WE_ALIGN_A; eidx = j;
        } else if (pp[1].s == 0 || c_isinf(be) || be.y == 0.0) {
            err = WE_ALIGN_B; eidx = j;
        } else if (!walk_less(al.y, be.y)) {
            err = WE_ORDER; eidx = j;
        }
        parity ^= 1;
        if (err) goto fail;
        double cc, dd;  // the Close record as registers (see the zip loop)
        close_params(al.y, be.y, cc, dd);
        if (logger) {
            const Rec rc = mk_close_p(al.y, be.y, cc, dd);
            log_a[na_rec++] = rc;
            log_b[nb_rec++] = rc;
        }
        progress(false);
        for (int g = lo + threadIdx.x; g < hi; g += NT) {
            double2 z = pts[g - lo];
            int8_t s8 = sides[g - lo];
            apply_close(al.y, be.y, cc, dd, z, s8);
            pts[g - lo] = z;
            sides[g - lo] = s8;
        }
    }
    // ---- far ends: SquareMobius; stage max of |va| (arc + aux) for the deferred check
    {
        double m = 0;
        for (int g = lo + threadIdx.x; g < hi && g < P; g += NT)
            if (c_fin(pts[g - lo])) m = fmax(m, cabs_(pts[g - lo]));
        m = block_max(m, red);
        int gi[2] = {0, P};
        publish(gi, 2, m);
        PParam* pp = s_param[parity];
        double2 qa = pp[0].z, qb = pp[1].z;
        double stage = 0;
        for (int r = 0; r < CS; ++r) stage = fmax(stage, s_flag[parity][r]);
        parity ^= 1;
        if (logger) {
            meta[6] = qa.x; meta[7] = qa.y; meta[8] = qb.x; meta[9] = qb.y;
            meta[10] = stage;
            meta[14] = na_rec;
            meta[15] = nb_rec;
        }
        ra = mk_sq(c_isinf(qa) ? cinf() : qa);
        if (logger) {
            log_a[na_rec++] = ra;
            log_b[nb_rec++] = ra;
        }
        progress(false);
        apply_pair(ra, true, ra, true);
    }
    // ---- normalisation (welding.py:699-717)
    {
        int gi[4] = {k + 1, P + k + 1, k + 2, P + k + 2};
        publish(gi, 4, 0.0);
        PParam* pp = s_param[parity];
        double2 za = pp[0].z, zb = pp[1].z, ia = pp[2].z, ib = pp[3].z;
        double2 co[4];
        if (c_isinf(za) || c_isinf(zb) || c_isinf(ia) || c_isinf(ib)) {
            err = WE_TRACK;
        } else {
            double2 zmid = C(0.5 * (ia.x + ib.x), 0.5 * (ia.y + ib.y));
            if (!c_eq(za, zb) && !c_eq(za, zmid) && !c_eq(zb, zmid)) {
                double2 zs[3] = {za, zb, zmid}, ws[3] = {C(-1, 0), C(1, 0), cinf()};
                if (!three_point(zs, ws, co)) err = WE_THREE;
            } else if (!c_zero(za)) {
                co[0] = cdiv(C(-1.0, 0.0), za); co[1] = C(0, 0); co[2] = C(0, 0); co[3] = C(1, 0);
            } else {
                co[0] = C(1, 0); co[1] = C(0, 0); co[2] = C(0, 0); co[3] = C(1, 0);
            }
        }
        parity ^= 1;
        if (err) goto fail;
        ra = mk_mob(co[0], co[1], co[2], co[3]);
        if (logger) {
            log_a[na_rec++] = ra;
            log_b[nb_rec++] = ra;
        }
        progress(false);
        apply_pair(ra, true, ra, true);
    }
    // ---- closed welding: respread the seam (welding.py:751-763)
    if (sd.closed) {
        int n = k + 1;
        int gi[3] = {0, n / 3, (2 * n) / 3};
        publish(gi, 3, 0.0);
        PParam* pp = s_param[parity];
        double2 an[3] = {pp[0].z, pp[1].z, pp[2].z};
        double2 tg[3] = {C(1.0, 0.0), C(cos(2 * M_PI / 3), sin(2 * M_PI / 3)), C(cos(4 * M_PI / 3), sin(4 * M_PI / 3))};
        double2 co[4];
        if (!three_point(an, tg, co)) err = WE_THREE, eidx = 1;
        parity ^= 1;
        if (err) goto fail;
        ra = mk_mob(co[0], co[1], co[2], co[3]);
        if (logger) {
            log_a[na_rec++] = ra;
            log_b[nb_rec++] = ra;
        }
        progress(false);
        for (int g = lo + threadIdx.x; g < hi; g += NT) sides[g - lo] = 0;
        apply_pair(ra, true, ra, true);
    }
    // ---- outputs: all 2P points to arc_out; rank 0 finishes seam/maxima/area
    for (int g = lo + threadIdx.x; g < hi; g += NT) A.arc_out[sd.arc + g] = pts[g - lo];
    if (prog) __threadfence();  // arc_out is read by the streamed replay after the final counter
    cl.sync();
    if (rank == 0) {
        const double2* o = A.arc_out + sd.arc;
        double seam = 0, ma = 0, mb = 0, mx = 0, area = 0, bad = 0;
        for (int t = threadIdx.x; t <= k; t += NT) {
            double2 a = o[t], b = o[P + t];
            double gg = (c_isinf(a) && c_isinf(b)) ? 0.0 : cabs_(csub(a, b));
            if (!isnan(gg)) seam = fmax(seam, gg);
            if (c_fin(a)) ma = fmax(ma, cabs_(a));
            if (c_fin(b)) mb = fmax(mb, cabs_(b));
            double2 nx = o[(t + 1) % (k + 1)];
            area += 0.5 * (a.x * nx.y - a.y * nx.x);
        }
        for (int g = threadIdx.x; g < NP; g += NT)
            if (c_nan(o[g])) bad = 1;
        for (int t = threadIdx.x; t < 2; t += NT) {
            double2 a = o[k + 1 + t], b = o[P + k + 1 + t];
            if (c_fin(a)) mx = fmax(mx, cabs_(a));
            if (c_fin(b)) mx = fmax(mx, cabs_(b));
        }
        seam = block_max(seam, red);
        ma = block_max(ma, red);
        mb = block_max(mb, red);
        mx = block_max(mx, red);
        area = block_sum(area, red);
        bad = block_max(bad, red);
        if (logger) {  // every thread holds the reductions; the logger owns the record counts
            meta[0] = na_rec;
            meta[1] = nb_rec;
            meta[5] = seam;
            meta[11] = ma;
            meta[12] = mb;
            meta[13] = mx;
            meta[16] = area;
            if (bad > 0) {
                meta[2] = WE_NAN;
                meta[4] = 3;
            }
        }
        progress(true);
    }
    return;
fail:
    if (logger) {
        meta[2] = err;
        meta[3] = eidx;
        meta[4] = eaux;
    }
    progress(true);
}

// ---------------------------------------------------------------------------
// phase 1, wavefront form (default; PGCP_WELD_WAVE=0 selects k_phase1c).
//
// The zip (Open) and alignment (Close) loops are 2(k-1) of the weld's 2k+3
// records, and record j's parameter is a single point (a_j, b_j) after all
// earlier records. k_phase1c pays a cluster barrier per record so that every
// CTA can rebuild it. Here the chain instead runs inside the warp that holds
// the parameter points: points are interleaved by index (point id
// q = 2 t + side, so a_t and b_t sit in adjacent lanes and both sides of an
// index in one warp), and the owning warp takes the parameters by shuffle,
// builds the record, applies it to its own points and moves on to the next
// index -- no memory operation and no barrier on the chain. It publishes each
// record into a ring in its CTA's shared memory (a CTA-scope release of a
// per-producer counter); the other warps of the CTA apply records from the
// ring as they appear (they lag behind, off the chain); a forwarder warp per
// CTA copies the CTA's own records into every other CTA's ring (DSMEM,
// cluster-scope release of that CTA's counter), writes the logs for the
// replay and publishes the replay's progress counter. The chain moves to the
// next warp every 16 indices and to the next CTA every PT / 2.
// Every point applies the same records in the same order as in k_phase1c,
// with the same arithmetic, so the results are bit-identical
// (tests/test_gpu_pipeline.py::test_wave_weld_equals_barrier_weld).
// Errors (the checks of welding.py:655-687) abort the chain through a flag
// bit in the counters; every spin has a 2 s timeout that reports an internal
// error instead of hanging.

constexpr int WAVE_ABORT = 1 << 30;
constexpr int WAVE_COUNT = (1 << 30) - 1;
constexpr int WE_TIMEOUT = 19;
constexpr unsigned long long WAVE_TIMEOUT_NS = 2000000000ull;

struct WaveRec {
    double x0, x1, x2, x3;  // Open: xi.re, xi.im; Close: a, b (the parameters are formed by whoever needs them)
};

__device__ __forceinline__ int ld_vol_i(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void st_vol_i(int* p, int v) { *reinterpret_cast<volatile int*>(p) = v; }
__device__ __forceinline__ void fence_cluster() { asm volatile("fence.acq_rel.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// wait until *cnt (this CTA's shared memory) reaches need or carries the abort
// bit; returns the observed value (WAVE_ABORT set on abort / timeout)
__device__ __forceinline__ int wave_wait(const int* cnt, int need, unsigned long long& t0, int spin_ns) {
    int v = ld_vol_i(cnt);
    int spins = 0;
    while ((v & WAVE_COUNT) < need && !(v & WAVE_ABORT)) {
        if (spin_ns > 0) __nanosleep(spin_ns);
        if (++spins == 256) {
            spins = 0;
            const unsigned long long now = gtimer();
            if (t0 == 0) {
                t0 = now;
            } else if (now - t0 > WAVE_TIMEOUT_NS) {
                return WAVE_ABORT | WAVE_COUNT;  // reported as WE_TIMEOUT by the caller
            }
        }
        v = ld_vol_i(cnt);
    }
    return v;
}

template <int PT>
__global__ void __launch_bounds__(PT + 32, 1) k_phase1w(Phase1Args A) {
    constexpr int NT = PT + 32;
    constexpr unsigned FULL = 0xffffffffu;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ PParam s_param[2][NPARAM];
    __shared__ double s_flag[2][NFLAG];
    __shared__ double red[32];
    __shared__ int s_cnt[2][PC_MAXCS];  // [open, close][producer CTA] records available from that CTA
    __shared__ int s_err[4];            // rank 0's copy: code, index, aux, taken
    cgw::cluster_group cl = cgw::this_cluster();
    const int CS = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    const int step = blockIdx.x / CS;
    const StepDesc sd = A.steps[step];
    double* meta = A.meta + META * (int64_t)step;
    const int k = sd.k;
    const int P = k + 3;
    const int NP = 2 * P;
    const int chunk = (((NP + CS - 1) / CS) + 1) & ~1;  // even: a_t and b_t in one CTA, one warp
    const int lo = min(NP, rank * chunk), hi = min(NP, lo + chunk);
    WaveRec* ringO = reinterpret_cast<WaveRec*>(smem);  // [k + 1][2]
    WaveRec* ringC = ringO + 2 * (k + 1);              // [k + 1]
    const int lane = threadIdx.x & 31;
    const bool fwd = threadIdx.x >= PT;                 // the forwarder warp
    const int q = lo + (int)threadIdx.x;
    const bool have = !fwd && q < hi;
    const int side = q & 1, t = q >> 1;
    const int wq0 = lo + (int)(threadIdx.x & ~31u);     // first point id of my warp
    Rec* log_a = A.recs + sd.rec;
    Rec* log_b = log_a + sd.cap;
    const bool logger = rank == 0 && (int)threadIdx.x == PT;
    int na_rec = 0, nb_rec = 0, nlogged = 0;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    int* prog = A.prog ? A.prog + 2 * step : nullptr;
    auto progress = [&](bool fin) {
        if (!logger || !prog) return;
        if (!fin && (++nlogged % A.prog_every) != 0) return;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        prog_store(prog, na_rec | (fin ? PROG_DONE : 0));
        prog_store(prog + 1, nb_rec | (fin ? PROG_DONE : 0));
    };
    if (threadIdx.x < 2 * PC_MAXCS) (&s_cnt[0][0])[threadIdx.x] = 0;
    if (threadIdx.x < 4) s_err[threadIdx.x] = 0;
    if (logger)
        for (int i = 0; i < META; ++i) meta[i] = 0.0;
    if (k < 1 || k > sd.na - 1 || k > sd.nb - 1) {
        if (logger) {
            meta[2] = WE_K;
            meta[3] = k;
        }
        progress(true);
        return;
    }
    const int32_t* sa = A.src + sd.src;
    const int32_t* sb = sa + sd.na;
    Rec pre[2];
    int pcode = 0;
    // the point threads' reduction order, as k_phase1c<PT> (bit-identical prenormalizer)
    bool okA = prenormalize(A.tv, sa, sd.na, red, &pre[0], &pcode, PT);
    bool okB = okA && prenormalize(A.tv, sb, sd.nb, red, &pre[1], &pcode, PT);
    if (!okA || !okB) {
        if (logger) {
            meta[2] = WE_PRE;
            meta[3] = okA ? 1 : 0;
            meta[4] = pcode;
        }
        progress(true);
        return;
    }
    const bool timed = A.timing && rank == 0 && threadIdx.x == 0;
    const long long tk0 = timed ? clock64() : 0;
    long long tk1 = tk0, tk2 = tk0;
    double2 z = C(0.0, 0.0);
    int8_t s8 = 0;
    if (have) {
        if (t <= k) {
            z = A.tv[(side ? sb : sa)[t]];
            int8_t tmp = 0;
            apply_rec(pre[side], z, tmp);
        } else {
            z = (t == k + 1) ? C(0.0, 0.0) : cinf();
        }
    }
    if (logger) {
        log_a[na_rec++] = pre[0];
        log_b[nb_rec++] = pre[1];
    }
    progress(false);
    int parity = 0;
    // point ids -> every CTA's parameter slots, then the cluster barrier
    auto publish = [&](const int* qidx, int np, double flag) {
        for (int which = 0; which < np; ++which) {
            if (have && q == qidx[which]) {
                PParam pp;
                pp.z = z;
                pp.s = s8;
                pp.pad = 0;
                for (int dst = 0; dst < CS; ++dst) cl.map_shared_rank(&s_param[parity][0], dst)[which] = pp;
            }
        }
        if (threadIdx.x < CS) cl.map_shared_rank(&s_flag[parity][0], threadIdx.x)[rank] = flag;
        cl.sync();
    };
    // the first error of a wavefront loop, kept in rank 0's s_err
    auto raise = [&](int code, int idx, int aux) {
        int* e = cl.map_shared_rank(s_err, 0);
        if (atomicCAS(e + 3, 0, 1) == 0) {
            e[0] = code;
            e[1] = idx;
            e[2] = aux;
        }
    };
    // abort a wavefront loop everywhere: the abort bit into every counter of every CTA
    auto abort_all = [&](int loop) {
        for (int x = 0; x < CS; ++x)
            for (int r = 0; r < CS; ++r) atomicOr(cl.map_shared_rank(&s_cnt[loop][r], x), WAVE_ABORT);
    };
    auto take_error = [&](int& err, int& eidx, int& eaux) {  // after a cluster barrier
        const int* e = cl.map_shared_rank(s_err, 0);
        if (e[3]) {
            err = e[0];
            eidx = e[1];
            eaux = e[2];
        }
    };
    int err = 0, eidx = 0, eaux = 0;
    Rec ra, rb;
    bool has[2] = {false, false};  // axis Mobius records logged (below)
    // ---- zip step 1: SqrtRatio
    {
        int gi[4] = {0, 2, 1, 3};  // a0, a1, b0, b1
        publish(gi, 4, 0.0);
        PParam* pp = s_param[parity];
        if (c_eq(pp[0].z, pp[1].z) || c_eq(pp[2].z, pp[3].z)) err = WE_ZIP01;
        ra = mk_sqr(pp[0].z, pp[1].z, UP);
        rb = mk_sqr(pp[2].z, pp[3].z, DOWN);
        parity ^= 1;
    }
    if (err) goto fail;
    if (logger) {
        log_a[na_rec++] = ra;
        log_b[nb_rec++] = rb;
    }
    progress(false);
    if (have) apply_rec(side ? rb : ra, z, s8);
    // ---- zip steps j = 2..k: Open, as a wavefront
    if (k >= 2) {
        unsigned long long t0 = 0;
        if (!fwd) {
            int j = 2;
            while (j <= k) {
                const int lp = 2 * j - wq0;
                if (lp >= 0 && lp < 32 && 2 * j < hi) {
                    // my warp holds a_j .. a_j1 and b_j .. b_j1 (lanes 2(j - t0) + side):
                    // produce the whole segment. Only the lanes whose own index is
                    // still ahead apply each record at once (all unzipped: one branch
                    // of apply_open, no divergence on the chain); the others catch
                    // up from the ring after the segment.
                    const int j1 = min(k, min((hi - 1) / 2, (wq0 + 31) / 2));
                    const int j0 = j;
                    bool bad = false;
                    long long dbg[4] = {0, 0, 0, 0};
                    const bool dbg_on = A.timing && k >= 1000 && A.timing_detail;
                    for (; j <= j1; ++j) {
                        const long long ta = dbg_on ? clock64() : 0;
                        const int lq = 2 * j - wq0;
                        const double2 xs = C(__shfl_sync(FULL, z.x, lq + side), __shfl_sync(FULL, z.y, lq + side));
                        const int ss = __shfl_sync(FULL, (int)s8, lq + side);
                        int e = 0;  // every lane checks its side's point (a_j even, b_j odd lanes)
                        if (ss != 0 || c_isinf(xs)) {
                            e = WE_ZIP_HALF;
                        } else if (!(xs.x > 0)) {
                            e = WE_ZIP_AXIS;
                        } else if (cabs_lt(xs, 1e-13)) {
                            e = WE_ZIP_COLL;
                        }
                        if (__any_sync(FULL, e != 0)) {
                            const int ea = __shfl_sync(FULL, e, lq), eb = __shfl_sync(FULL, e, lq + 1);
                            if (lane == 0) {
                                raise(ea ? ea : eb, j, ea ? 0 : 1);
                                fence_cluster();
                                abort_all(0);
                            }
                            bad = true;
                            break;
                        }
                        const long long tb = dbg_on ? clock64() : 0;
                        // record j for the ring ((pp, qq): one reciprocal, off the chain --
                        // the unlabelled apply below needs only xi). The segment's last
                        // record is published before its apply (the next warp takes the
                        // chain from it); the others after, so the fence waits on stores
                        // that have long completed
                        const bool last = j == j1;
                        auto put = [&]() {
                            if (lane == lq || lane == lq + 1) *reinterpret_cast<double2*>(&ringO[2 * j + side]) = xs;
                            __syncwarp();
                            if (lane == lq) {
                                __threadfence_block();
                                st_vol_i(&s_cnt[0][rank], j);
                            }
                        };
                        if (last) put();
                        const long long tc = dbg_on ? clock64() : 0;
                        if (have && t > j) apply_open_xi(xs, side ? DOWN : UP, z, s8);
                        if (!last) put();
                        if (dbg_on) {
                            const double zz = __shfl_sync(FULL, z.x, (lq + 2) & 31);
                            const long long td = clock64() + (zz == 12345.678 ? 1 : 0);
                            dbg[0] += tb - ta;
                            dbg[1] += tc - tb;
                            dbg[2] += td - tc;
                            dbg[3] += 1;
                        }
                    }
                    if (dbg_on && lane == 0)
                        printf("[wave dbg] open rank %d warp %d j %d..%d: shfl+params+check %lld, publish %lld, apply+publish %lld cycles/record\n",
                               rank, (int)(threadIdx.x >> 5), j0, j1, dbg[0] / max(1ll, dbg[3]), dbg[1] / max(1ll, dbg[3]),
                               dbg[2] / max(1ll, dbg[3]));
                    if (bad) break;
                    // catch-up: my own record and the rest of the segment, in order
                    if (have)
                        for (int jj = max(t, j0); jj <= j1; ++jj) {
                            const double2 xi = *reinterpret_cast<const double2*>(&ringO[2 * jj + side]);
                            apply_open_xi(xi, side ? DOWN : UP, z, s8);
                        }
                    __syncwarp();
                } else {
                    // records of other warps / CTAs: apply them as they appear
                    const int r = (2 * j) / chunk;
                    int v = 0;
                    if (lane == 0) {  // one lane acquires; the warp stays converged
                        v = wave_wait(&s_cnt[0][r], j, t0, A.spin_ns);
                        if (r == rank) __threadfence_block(); else fence_cluster();
                    }
                    v = __shfl_sync(FULL, v, 0);
                    __syncwarp();
                    if (v & WAVE_ABORT) {
                        if ((v & WAVE_COUNT) == WAVE_COUNT && lane == 0) {
                            raise(WE_TIMEOUT, j, 0);
                            fence_cluster();
                            abort_all(0);
                        }
                        break;
                    }
                    const int upto = min(v & WAVE_COUNT, k);
                    for (; j <= upto; ++j) {
                        if (2 * j >= wq0 && 2 * j < wq0 + 32 && 2 * j < hi) break;  // mine to build
                        const double2 xi = *reinterpret_cast<const double2*>(&ringO[2 * j + side]);
                        if (have) apply_open_xi(xi, side ? DOWN : UP, z, s8);
                    }
                }
            }
        } else {
            // forwarder: this CTA's records j in [jlo, jhi] -> logs, other CTAs, replay progress
            const int jlo = max(2, lo / 2), jhi = min(k, (hi - 1) / 2);
            for (int jf = jlo; jf <= jhi;) {
                int v = 0;
                if (lane == 0) {
                    v = wave_wait(&s_cnt[0][rank], jf, t0, A.spin_ns);
                    __threadfence_block();
                }
                v = __shfl_sync(FULL, v, 0);
                __syncwarp();
                const bool ab = (v & WAVE_ABORT) != 0;
                if ((v & WAVE_COUNT) == WAVE_COUNT && lane == 0) {
                    raise(WE_TIMEOUT, jf, 2);
                    fence_cluster();
                    abort_all(0);
                }
                const int upto = ab ? jf - 1 : min(v & WAVE_COUNT, jhi);
                for (int jj = jf + lane; jj <= upto; jj += 32) {
                    const WaveRec wa = ringO[2 * jj], wb = ringO[2 * jj + 1];
                    log_a[jj] = mk_open(C(wa.x0, wa.x1), UP);
                    log_b[jj] = mk_open(C(wb.x0, wb.x1), DOWN);
                }
                fence_gpu();  // the logs before the records leave this CTA (replay progress causality)
                __syncwarp();
                for (int x = lane; x < CS; x += 32) {
                    if (x == rank) continue;
                    WaveRec* rr = cl.map_shared_rank(ringO, x);
                    for (int jj = jf; jj <= upto; ++jj) {
                        rr[2 * jj] = ringO[2 * jj];
                        rr[2 * jj + 1] = ringO[2 * jj + 1];
                    }
                    fence_cluster();
                    st_vol_i(cl.map_shared_rank(&s_cnt[0][rank], x), (ab ? WAVE_ABORT : 0) | upto);
                }
                if (prog && lane == 0 && upto >= jf) {
                    prog_store(prog, upto + 1);
                    prog_store(prog + 1, upto + 1);
                }
                if (ab) break;
                jf = upto + 1;
            }
        }
        cl.sync();
        take_error(err, eidx, eaux);
        if (err) goto fail;
    }
    if (timed) tk1 = clock64();
    if (logger) {
        na_rec = k + 1;
        nb_rec = k + 1;
    }
    // ---- axis Mobius sending pts[0] to infinity (welding.py:593-600)
    {
        int gi[2] = {0, 1};
        publish(gi, 2, 0.0);
        PParam* pp = s_param[parity];
        Rec rr0, rr1;
#pragma unroll
        for (int sdx = 0; sdx < 2; ++sdx) {
            if (err) break;
            double2 w0 = pp[sdx].z;
            if (!c_isinf(w0)) {
                if (c_zero(w0)) {
                    err = WE_FAR0;
                    eaux = sdx;
                } else {
                    int br = sdx ? DOWN : UP;
                    Rec& rs = sdx ? rr1 : rr0;
                    rs = mk_mob(C(1, 0), C(0, 0), cdiv(C(-1.0, 0.0), w0), C(1, 0), true);
                    mob_pin(rs, w0, cinf(), br);
                    mob_pin(rs, C(0, 0), C(0, 0), br);
                    has[sdx] = true;
                }
            }
        }
        parity ^= 1;
        if (err) goto fail;
        if (logger) {
            if (has[0]) log_a[na_rec++] = rr0;
            if (has[1]) log_b[nb_rec++] = rr1;
        }
        progress(false);
        if (have && has[side]) apply_rec(side ? rr1 : rr0, z, s8);
    }
    // ---- closing loop j = k-1 .. 1 (welding.py:673-687), as a wavefront
    if (k >= 2) {
        const int base_a = k + 1 + (has[0] ? 1 : 0), base_b = k + 1 + (has[1] ? 1 : 0);
        unsigned long long t0 = 0;
        if (!fwd) {
            int j = k - 1;
            while (j >= 1) {
                const int lp = 2 * j - wq0;
                if (lp >= 0 && lp < 32 && 2 * j < hi) {
                    // produce records j .. jbot (descending); lanes whose own index is
                    // below the record apply it at once (all still on the axis: one
                    // branch of apply_close), the others catch up afterwards
                    const int jtop = j;
                    const int jbot = max(1, wq0 / 2);
                    bool bad = false;
                    long long dbg[4] = {0, 0, 0, 0};
                    const bool dbg_on = A.timing && k >= 1000 && A.timing_detail;
                    for (; j >= jbot; --j) {
                        const long long ta = dbg_on ? clock64() : 0;
                        const int lq = 2 * j - wq0;
                        const double2 al = C(__shfl_sync(FULL, z.x, lq), __shfl_sync(FULL, z.y, lq));
                        const double2 be = C(__shfl_sync(FULL, z.x, lq + 1), __shfl_sync(FULL, z.y, lq + 1));
                        const int sa_ = __shfl_sync(FULL, (int)s8, lq), sb_ = __shfl_sync(FULL, (int)s8, lq + 1);
                        int e = 0;
                        if (sa_ == 0 || c_isinf(al) || al.y == 0.0) {
                            e = WE_ALIGN_A;
                        } else if (sb_ == 0 || c_isinf(be) || be.y == 0.0) {
                            e = WE_ALIGN_B;
                        } else if (!walk_less(al.y, be.y)) {
                            e = WE_ORDER;
                        }
                        if (e) {
                            if (lane == 0) {
                                raise(e, j, 0);
                                fence_cluster();
                                abort_all(1);
                            }
                            bad = true;
                            break;
                        }
                        const long long tb = dbg_on ? clock64() : 0;
                        // record j for the ring (c, d: one division, off the chain --
                        // the labelled apply below needs only a and b); the segment's
                        // last record goes out before its apply (see the zip loop)
                        const bool last = j == jbot;
                        auto put = [&]() {
                            if (lane == lq) *reinterpret_cast<double2*>(&ringC[j]) = C(al.y, be.y);
                            __syncwarp();
                            if (lane == lq) {
                                __threadfence_block();
                                st_vol_i(&s_cnt[1][rank], k - j);
                            }
                        };
                        if (last) put();
                        const long long tc = dbg_on ? clock64() : 0;
                        if (have && t < j) apply_close_ab(al.y, be.y, z, s8);
                        if (!last) put();
                        if (dbg_on) {
                            const double zz = __shfl_sync(FULL, z.y, (lq + 30) & 31);
                            const long long td = clock64() + (zz == 12345.678 ? 1 : 0);
                            dbg[0] += tb - ta;
                            dbg[1] += tc - tb;
                            dbg[2] += td - tc;
                            dbg[3] += 1;
                        }
                    }
                    if (dbg_on && lane == 0)
                        printf("[wave dbg] close rank %d warp %d j %d..%d: shfl+params+check %lld, publish %lld, apply+publish %lld cycles/record\n",
                               rank, (int)(threadIdx.x >> 5), jtop, jbot, dbg[0] / max(1ll, dbg[3]), dbg[1] / max(1ll, dbg[3]),
                               dbg[2] / max(1ll, dbg[3]));
                    if (bad) break;
                    if (have)
                        for (int jj = min(t, jtop); jj >= jbot; --jj) {
                            const WaveRec w = ringC[jj];
                            apply_close_ab(w.x0, w.x1, z, s8);
                        }
                    __syncwarp();
                } else {
                    const int r = (2 * j) / chunk;
                    int v = 0;
                    if (lane == 0) {
                        v = wave_wait(&s_cnt[1][r], k - j, t0, A.spin_ns);
                        if (r == rank) __threadfence_block(); else fence_cluster();
                    }
                    v = __shfl_sync(FULL, v, 0);
                    __syncwarp();
                    if (v & WAVE_ABORT) {
                        if ((v & WAVE_COUNT) == WAVE_COUNT && lane == 0) {
                            raise(WE_TIMEOUT, j, 1);
                            fence_cluster();
                            abort_all(1);
                        }
                        break;
                    }
                    const int lowest = max(1, k - (v & WAVE_COUNT));
                    for (; j >= lowest; --j) {
                        if (2 * j >= wq0 && 2 * j < wq0 + 32 && 2 * j < hi) break;
                        const WaveRec w = ringC[j];
                        if (have) apply_close_ab(w.x0, w.x1, z, s8);
                    }
                }
            }
        } else {
            // forwarder: this CTA's records, high index first
            const int jtop = min(k - 1, (hi - 1) / 2), jbot = max(1, lo / 2);
            for (int jf = jtop; jf >= jbot;) {
                int v = 0;
                if (lane == 0) {
                    v = wave_wait(&s_cnt[1][rank], k - jf, t0, A.spin_ns);
                    __threadfence_block();
                }
                v = __shfl_sync(FULL, v, 0);
                __syncwarp();
                const bool ab = (v & WAVE_ABORT) != 0;
                if ((v & WAVE_COUNT) == WAVE_COUNT && lane == 0) {
                    raise(WE_TIMEOUT, jf, 3);
                    fence_cluster();
                    abort_all(1);
                }
                const int lowest = ab ? jf + 1 : max(jbot, k - (v & WAVE_COUNT));
                for (int jj = jf - lane; jj >= lowest; jj -= 32) {
                    const WaveRec w = ringC[jj];
                    const Rec rc = mk_close(w.x0, w.x1);
                    log_a[base_a + (k - 1 - jj)] = rc;
                    log_b[base_b + (k - 1 - jj)] = rc;
                }
                fence_gpu();
                __syncwarp();
                for (int x = lane; x < CS; x += 32) {
                    if (x == rank) continue;
                    WaveRec* rr = cl.map_shared_rank(ringC, x);
                    for (int jj = jf; jj >= lowest; --jj) rr[jj] = ringC[jj];
                    fence_cluster();
                    st_vol_i(cl.map_shared_rank(&s_cnt[1][rank], x), (ab ? WAVE_ABORT : 0) | (k - lowest));
                }
                if (prog && lane == 0 && lowest <= jf) {
                    prog_store(prog, base_a + (k - lowest));
                    prog_store(prog + 1, base_b + (k - lowest));
                }
                if (ab) break;
                jf = lowest - 1;
            }
        }
        cl.sync();
        take_error(err, eidx, eaux);
        if (err) goto fail;
    }
    if (timed) {
        tk2 = clock64();
        A.timing[4 * step + 0] = tk1 - tk0;  // init + SqrtRatio + open loop
        A.timing[4 * step + 1] = tk2 - tk1;  // axis Mobius + closing loop
        A.timing[4 * step + 3] = -(k - 1);   // negative: wavefront layout of the split
    }
    if (logger) {  // the close records the forwarders logged
        na_rec += k - 1;
        nb_rec += k - 1;
    }
    // ---- far ends: SquareMobius; stage max of |va| (arc + aux) for the deferred check
    {
        double m = 0;
        if (have && side == 0 && c_fin(z)) m = cabs_(z);
        m = block_max(m, red);
        int gi[2] = {0, 1};
        publish(gi, 2, m);
        PParam* pp = s_param[parity];
        double2 qa = pp[0].z, qb = pp[1].z;
        double stage = 0;
        for (int r = 0; r < CS; ++r) stage = fmax(stage, s_flag[parity][r]);
        parity ^= 1;
        if (logger) {
            meta[6] = qa.x; meta[7] = qa.y; meta[8] = qb.x; meta[9] = qb.y;
            meta[10] = stage;
            meta[14] = na_rec;
            meta[15] = nb_rec;
        }
        ra = mk_sq(c_isinf(qa) ? cinf() : qa);
        if (logger) {
            log_a[na_rec++] = ra;
            log_b[nb_rec++] = ra;
        }
        progress(false);
        if (have) apply_rec(ra, z, s8);
    }
    // ---- normalisation (welding.py:699-717)
    {
        int gi[4] = {2 * (k + 1), 2 * (k + 1) + 1, 2 * (k + 2), 2 * (k + 2) + 1};
        publish(gi, 4, 0.0);
        PParam* pp = s_param[parity];
        double2 za = pp[0].z, zb = pp[1].z, ia = pp[2].z, ib = pp[3].z;
        double2 co[4];
        if (c_isinf(za) || c_isinf(zb) || c_isinf(ia) || c_isinf(ib)) {
            err = WE_TRACK;
        } else {
            double2 zmid = C(0.5 * (ia.x + ib.x), 0.5 * (ia.y + ib.y));
            if (!c_eq(za, zb) && !c_eq(za, zmid) && !c_eq(zb, zmid)) {
                double2 zs[3] = {za, zb, zmid}, ws[3] = {C(-1, 0), C(1, 0), cinf()};
                if (!three_point(zs, ws, co)) err = WE_THREE;
            } else if (!c_zero(za)) {
                co[0] = cdiv(C(-1.0, 0.0), za); co[1] = C(0, 0); co[2] = C(0, 0); co[3] = C(1, 0);
            } else {
                co[0] = C(1, 0); co[1] = C(0, 0); co[2] = C(0, 0); co[3] = C(1, 0);
            }
        }
        parity ^= 1;
        if (err) goto fail;
        ra = mk_mob(co[0], co[1], co[2], co[3]);
        if (logger) {
            log_a[na_rec++] = ra;
            log_b[nb_rec++] = ra;
        }
        progress(false);
        if (have) apply_rec(ra, z, s8);
    }
    // ---- closed welding: respread the seam (welding.py:751-763)
    if (sd.closed) {
        int n = k + 1;
        int gi[3] = {0, 2 * (n / 3), 2 * ((2 * n) / 3)};
        publish(gi, 3, 0.0);
        PParam* pp = s_param[parity];
        double2 an[3] = {pp[0].z, pp[1].z, pp[2].z};
        double2 tg[3] = {C(1.0, 0.0), C(cos(2 * M_PI / 3), sin(2 * M_PI / 3)), C(cos(4 * M_PI / 3), sin(4 * M_PI / 3))};
        double2 co[4];
        if (!three_point(an, tg, co)) err = WE_THREE, eidx = 1;
        parity ^= 1;
        if (err) goto fail;
        ra = mk_mob(co[0], co[1], co[2], co[3]);
        if (logger) {
            log_a[na_rec++] = ra;
            log_b[nb_rec++] = ra;
        }
        progress(false);
        s8 = 0;
        if (have) apply_rec(ra, z, s8);
    }
    // ---- outputs: all 2P points to arc_out (side a then side b); rank 0 finishes seam/maxima/area
    if (have) A.arc_out[sd.arc + side * P + t] = z;
    if (prog) __threadfence();  // arc_out is read by the streamed replay after the final counter
    cl.sync();
    if (rank == 0) {
        const double2* o = A.arc_out + sd.arc;
        double seam = 0, ma = 0, mb = 0, mx = 0, area = 0, bad = 0;
        for (int i = threadIdx.x; i <= k; i += NT) {
            double2 a = o[i], b = o[P + i];
            double gg = (c_isinf(a) && c_isinf(b)) ? 0.0 : cabs_(csub(a, b));
            if (!isnan(gg)) seam = fmax(seam, gg);
            if (c_fin(a)) ma = fmax(ma, cabs_(a));
            if (c_fin(b)) mb = fmax(mb, cabs_(b));
            double2 nx = o[(i + 1) % (k + 1)];
            area += 0.5 * (a.x * nx.y - a.y * nx.x);
        }
        for (int g = threadIdx.x; g < NP; g += NT)
            if (c_nan(o[g])) bad = 1;
        for (int i = threadIdx.x; i < 2; i += NT) {
            double2 a = o[k + 1 + i], b = o[P + k + 1 + i];
            if (c_fin(a)) mx = fmax(mx, cabs_(a));
            if (c_fin(b)) mx = fmax(mx, cabs_(b));
        }
        seam = block_max(seam, red);
        ma = block_max(ma, red);
        mb = block_max(mb, red);
        mx = block_max(mx, red);
        area = block_sum(area, red);
        bad = block_max(bad, red);
        if (logger) {
            meta[0] = na_rec;
            meta[1] = nb_rec;
            meta[5] = seam;
            meta[11] = ma;
            meta[12] = mb;
            meta[13] = mx;
            meta[16] = area;
            if (bad > 0) {
                meta[2] = WE_NAN;
                meta[4] = 3;
            }
        }
        progress(true);
    }
    return;
fail:
    if (logger) {
        meta[2] = err;
        meta[3] = eidx;
        meta[4] = eaux;
    }
    progress(true);
}

// ---------------------------------------------------------------------------
// phase 2: replay a step's log on a point (write-back list of a level)
//   entry = (slot, code): code bit 31 -> B log; bits 0..23: arc position + 1
//   (0 = replay); bit 24: take the arc value from side B; bit 25: cycle
//   point of side A (contributes to the scale maxima); bit 26: cycle point of B

struct ReplayArgs {
    const int32_t* wb;          // (slot, code, step) triples
    int64_t nwb;
    const StepDesc* steps;
    const Rec* recs;
    double2* tv;
    const double2* arc_out;
    double* meta;               // per step
    unsigned long long* maxbits;  // per step: [stage_a, final_a, final_b]
    int* nan_flag;
};

__global__ void k_replay_slots(ReplayArgs A) {
    GRID_STRIDE(i, A.nwb) {
        int slot = A.wb[3 * i], code = A.wb[3 * i + 1], step = A.wb[3 * i + 2];
        const StepDesc sd = A.steps[step];
        int arcpos = (code & 0xffffff) - 1;
        bool sideB = (code >> 31) & 1;
        if (A.meta[META * step + 2] != 0.0) continue;  // failed step: leave values
        if (arcpos >= 0) {
            bool fromB = (code >> 24) & 1;
            A.tv[slot] = A.arc_out[sd.arc + (fromB ? sd.k + 3 : 0) + arcpos];
            continue;
        }
        const Rec* log = A.recs + sd.rec + (sideB ? sd.cap : 0);
        int nrec = (int)A.meta[META * step + (sideB ? 1 : 0)];
        int sq = (int)A.meta[META * step + (sideB ? 15 : 14)];
        double2 z = A.tv[slot];
        int8_t s = 0;
        double stage = 0;
        RecHead nxt = {};
        if (nrec > 0) nxt = load_head(log);
        for (int r = 0; r < nrec; ++r) {
            if (r == sq) stage = c_fin(z) ? cabs_(z) : 0.0;
            const RecHead cur = nxt;
            if (r + 1 < nrec) nxt = load_head(log + r + 1);  // in flight during this apply
            apply_head(cur, log + r, z, s);
        }
        if (c_nan(z)) atomicExch(A.nan_flag, 1);
        A.tv[slot] = z;
        bool cycA = (code >> 25) & 1, cycB = (code >> 26) & 1;
        double fin = c_fin(z) ? cabs_(z) : 0.0;
        if (cycA) {
            atomicMax(&A.maxbits[3 * step + 0], (unsigned long long)__double_as_longlong(stage));
            atomicMax(&A.maxbits[3 * step + 1], (unsigned long long)__double_as_longlong(fin));
        }
        if (cycB) atomicMax(&A.maxbits[3 * step + 2], (unsigned long long)__double_as_longlong(fin));
    }
}

// the same replay, streamed: launched as the programmatic dependent of the
// level's phase 1, it applies each record as soon as the step's counter covers
// it. A wait longer than 2 s (phase 1 of the largest level takes ~5 ms) flags
// an internal error instead of hanging.
__device__ int wait_prog(const int* p, int need, int* timeout_flag) {
    int v = prog_load(p);
    if ((v & PROG_COUNT) >= need || (v & PROG_DONE)) return v;
    const unsigned long long t0 = gtimer();
    for (;;) {
        __nanosleep(256);
        v = prog_load(p);
        if ((v & PROG_COUNT) >= need || (v & PROG_DONE)) return v;
        if (gtimer() - t0 > 2000000000ull) {
            atomicExch(timeout_flag, 1);
            return PROG_DONE | PROG_TIMEOUT;
        }
    }
}

__global__ void k_replay_stream(ReplayArgs A, const int* __restrict__ prog, int* timeout_flag) {
    GRID_STRIDE(i, A.nwb) {
        int slot = A.wb[3 * i], code = A.wb[3 * i + 1], step = A.wb[3 * i + 2];
        const StepDesc sd = A.steps[step];
        int arcpos = (code & 0xffffff) - 1;
        bool sideB = (code >> 31) & 1;
        const int* pg = prog + 2 * step + (sideB ? 1 : 0);
        const double* meta = A.meta + META * (int64_t)step;
        if (arcpos >= 0) {
            int v = wait_prog(pg, PROG_COUNT, timeout_flag);
            if ((v & PROG_TIMEOUT) || __ldcg(meta + 2) != 0.0) continue;
            bool fromB = (code >> 24) & 1;
            A.tv[slot] = __ldcg(A.arc_out + sd.arc + (fromB ? sd.k + 3 : 0) + arcpos);
            continue;
        }
        const Rec* log = A.recs + sd.rec + (sideB ? sd.cap : 0);
        double2 z = A.tv[slot];
        int8_t s = 0;
        double stage = 0;
        int avail = 0, sq = 0, v = 0;
        RecHead nxt = {};
        bool have_nxt = false;
        for (int r = 0;; ++r) {
            if (r >= avail) {
                if (v & PROG_DONE) break;
                v = wait_prog(pg, r + 1, timeout_flag);
                avail = v & PROG_COUNT;
                if (r >= avail) break;  // finished (or failed / timed out) with fewer records
                // the index of the SquareMobius record is written before the
                // counter that covers it is published, so it is enough to look
                // for it when the counter has moved (a load per record would
                // put an L2 round trip on every step of the chain)
                if (sq == 0) sq = (int)__ldcg(meta + (sideB ? 15 : 14));
            }
            if (sq > 0 && r == sq) stage = c_fin(z) ? cabs_(z) : 0.0;
            const RecHead cur = have_nxt ? nxt : load_head(log + r);
            // the next record, if already covered by the counter read (acquire)
            // above, is loaded now and arrives during this apply
            have_nxt = r + 1 < avail;
            if (have_nxt) nxt = load_head(log + r + 1);
            apply_head(cur, log + r, z, s);
        }
        if (!(v & PROG_DONE)) v = wait_prog(pg, PROG_COUNT, timeout_flag);
        if ((v & PROG_TIMEOUT) || __ldcg(meta + 2) != 0.0) continue;  // failed step: leave values
        if (c_nan(z)) atomicExch(A.nan_flag, 1);
        A.tv[slot] = z;
        bool cycA = (code >> 25) & 1, cycB = (code >> 26) & 1;
        double fin = c_fin(z) ? cabs_(z) : 0.0;
        if (cycA) {
            atomicMax(&A.maxbits[3 * step + 0], (unsigned long long)__double_as_longlong(stage));
            atomicMax(&A.maxbits[3 * step + 1], (unsigned long long)__double_as_longlong(fin));
        }
        if (cycB) atomicMax(&A.maxbits[3 * step + 2], (unsigned long long)__double_as_longlong(fin));
    }
    // completion of this grid implies completion of the level's phase 1
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

// generic replay: log on a point array (apply_log, welding.py:512-526)
__global__ void k_replay_points(const Rec* __restrict__ recs, int nrec, double2* z, int8_t* sides, int64_t n,
                                int* nan_flag) {
    __shared__ Rec s_recs[32];
    for (int base = 0; base < nrec; base += 32) {
        int cnt = min(32, nrec - base);
        __syncthreads();
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) s_recs[i] = recs[base + i];
        __syncthreads();
        GRID_STRIDE(i, n) {
            double2 v = z[i];
            int8_t s = sides ? sides[i] : 0;
            for (int r = 0; r < cnt; ++r) apply_rec(s_recs[r], v, s);
            z[i] = v;
            if (sides) sides[i] = s;
        }
    }
    GRID_STRIDE(i, n) if (c_nan(z[i])) atomicExch(nan_flag, 1);
}


// ---------------------------------------------------------------------------
// polygon helpers (welding.py:770-796) and the geodesic map (welding.py:803-842)

// even-odd ray casting of p against poly (n points), block-wide
__device__ bool block_inside(const double2* poly, int n, double2 p, double* red) {
    double cnt = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double2 a = poly[i], b = poly[(i + 1) % n];
        bool cond = (a.y > p.y) != (b.y > p.y);
        double xint = a.x + (p.y - a.y) / (b.y - a.y) * (b.x - a.x);
        if (cond && (p.x < xint)) cnt += 1;
    }
    cnt = block_sum(cnt, red);
    return ((long long)cnt) % 2 == 1;
}

// polygon_interior_point: centroid, else edge-midpoint offsets
__device__ bool interior_point(const double2* poly, int n, double* red, double2* out) {
    double sx = 0, sy = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        sx += poly[i].x;
        sy += poly[i].y;
    }
    sx = block_sum(sx, red);
    sy = block_sum(sy, red);
    double2 c = C(sx / n, sy / n);
    if (block_inside(poly, n, c, red)) {
        *out = c;
        return true;
    }
    const double ts[3] = {0.25, 0.05, 0.01};
    for (int i = 0; i < n; ++i) {
        double2 a = poly[i], b = poly[(i + 1) % n];
        double2 mid = C(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
        double2 nrm = cmul(csub(b, a), C(0.0, 1.0));
        for (int q = 0; q < 3; ++q) {
            double2 cand = cadd(mid, cmul(C(ts[q], 0.0), nrm));
            if (block_inside(poly, n, cand, red)) {
                *out = cand;
                return true;
            }
        }
    }
    return false;
}

struct GeoArgs {
    const double2* tv;
    const int32_t* src;     // n cycle points (slot ids) in cycle order
    int n;
    int has_interior;
    double2 interior;
    double2* pts;           // scratch n+1
    int8_t* sides;          // scratch n+1
    int32_t* order;         // scratch n: position -> src index (after orientation)
    double2* circ;          // out: circle value per src index
    Rec* recs;
    double* meta;           // [0] nrec, [2] err, [3] idx, [4] aux, [5] max ||z|-1|
};

__global__ void __launch_bounds__(512) k_geodesic(GeoArgs A) {
    __shared__ Rec s_rec;
    __shared__ int s_err;
    __shared__ double red[32];
    __shared__ double2 s_c;
    const int n = A.n;
    double* meta = A.meta;
    if (threadIdx.x == 0) {
        s_err = 0;
        for (int i = 0; i < META; ++i) meta[i] = 0.0;
    }
    __syncthreads();
    // orientation (pipeline.py:218-222): reverse all but the first if cw
    double area = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double2 a = A.tv[A.src[i]], b = A.tv[A.src[(i + 1) % n]];
        area += 0.5 * (a.x * b.y - a.y * b.x);
    }
    area = block_sum(area, red);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int o = (area < 0 && i > 0) ? n - i : i;
        A.order[i] = o;
        A.pts[i] = A.tv[A.src[o]];
        A.sides[i] = 0;
    }
    __syncthreads();
    if (A.has_interior) {
        if (threadIdx.x == 0) s_c = A.interior;
    } else {
        double2 c;
        bool ok = interior_point(A.pts, n, red, &c);
        if (threadIdx.x == 0) {
            if (!ok) block_fail(&s_err, WE_INTERIOR, 0, 0, meta);
            s_c = c;
        }
    }
    __syncthreads();
    if (s_err) return;
    if (threadIdx.x == 0) {
        A.pts[n] = s_c;
        A.sides[n] = 0;
    }
    __syncthreads();
    int nrec = 0;
    auto apply_all = [&]() {
        for (int i = threadIdx.x; i <= n; i += blockDim.x) {
            double2 z = A.pts[i];
            int8_t s = A.sides[i];
            apply_rec(s_rec, z, s);
            A.pts[i] = z;
            A.sides[i] = s;
        }
    };
    if (threadIdx.x == 0) {
        if (c_eq(A.pts[0], A.pts[1])) block_fail(&s_err, WE_ZIP01, 0, 0, meta);
        else s_rec = mk_sqr(A.pts[0], A.pts[1], UP);
        A.recs[nrec] = s_rec;
    }
    ++nrec;
    __syncthreads();
    if (s_err) return;
    apply_all();
    __syncthreads();
    for (int j = 2; j <= n - 1; ++j) {
        if (threadIdx.x == 0) {
            double2 xi = A.pts[j];
            if (A.sides[j] != 0 || c_isinf(xi)) block_fail(&s_err, WE_ZIP_HALF, j, 0, meta);
            else if (!(xi.x > 0)) block_fail(&s_err, WE_ZIP_AXIS, j, 0, meta);
            else if (cabs_lt(xi, 1e-13)) block_fail(&s_err, WE_ZIP_COLL, j, 0, meta);
            else {
                s_rec = mk_open(xi, UP);
                A.recs[nrec] = s_rec;
            }
        }
        ++nrec;
        __syncthreads();
        if (s_err) return;
        apply_all();
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double2 w0 = A.pts[0];
        s_rec = mk_sq(c_isinf(w0) ? cinf() : w0);
        A.recs[nrec] = s_rec;
    }
    ++nrec;
    __syncthreads();
    apply_all();
    __syncthreads();
    if (threadIdx.x == 0) {  // Cayley transform to the disk
        Rec r = mk_mob(C(1, 0), C(0, -1), C(1, 0), C(0, 1));
        mob_pin(r, cinf(), C(1.0, 0.0), FREE);
        s_rec = r;
        A.recs[nrec] = r;
    }
    ++nrec;
    __syncthreads();
    apply_all();
    __syncthreads();
    if (threadIdx.x == 0) {
        double2 al = A.pts[n];
        if (!(cabs_(al) < 1)) {
            block_fail(&s_err, WE_GEO_DISK, 0, 0, meta);
        } else {
            s_rec = mk_mob(C(1, 0), cneg(al), C(-al.x, al.y), C(1, 0));
            A.recs[nrec] = s_rec;
        }
    }
    ++nrec;
    __syncthreads();
    if (s_err) return;
    apply_all();
    __syncthreads();
    double err = 0, bad = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double2 z = A.pts[i];
        if (c_nan(z)) bad = 1;
        err = fmax(err, fabs(cabs_(z) - 1.0));
        A.circ[A.order[i]] = z;
    }
    err = block_max(err, red);
    bad = block_max(bad, red);
    if (threadIdx.x == 0) {
        meta[0] = nrec;
        meta[5] = err;
        meta[6] = s_c.x;
        meta[7] = s_c.y;
        if (bad > 0) block_fail(&s_err, WE_NAN, 0, 4, meta);
        else if (err > 1e-9) block_fail(&s_err, WE_GEO_CIRCLE, 0, 0, meta);
    }
}

// intermediate_form (welding.py:578-602): zip points 0..k of one boundary
// onto the branch's half of the imaginary axis (_zip_points,
// welding.py:544-575), then the axis Mobius sending point 0 to infinity. One
// block; every record is built by thread 0 and applied by all threads.
__global__ void __launch_bounds__(512) k_zip_form(double2* pts, int8_t* sides, int n, int k, int br, Rec* recs,
                                                   double* meta) {
    __shared__ Rec s_rec;
    __shared__ int s_err;
    __shared__ double red[32];
    if (threadIdx.x == 0) {
        s_err = 0;
        for (int i = 0; i < META; ++i) meta[i] = 0.0;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) sides[i] = 0;
    __syncthreads();
    int nrec = 0;
    auto apply_all = [&]() {
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            double2 z = pts[i];
            int8_t sd = sides[i];
            apply_rec(s_rec, z, sd);
            pts[i] = z;
            sides[i] = sd;
        }
    };
    if (threadIdx.x == 0) {
        if (c_eq(pts[0], pts[1])) block_fail(&s_err, WE_ZIP01, 0, 0, meta);
        else s_rec = mk_sqr(pts[0], pts[1], br);
        recs[nrec] = s_rec;
    }
    ++nrec;
    __syncthreads();
    if (s_err) return;
    apply_all();
    __syncthreads();
    for (int j = 2; j <= k; ++j) {
        if (threadIdx.x == 0) {
            double2 xi = pts[j];
            if (sides[j] != 0 || c_isinf(xi)) block_fail(&s_err, WE_ZIP_HALF, j, 0, meta);
            else if (!(xi.x > 0)) block_fail(&s_err, WE_ZIP_AXIS, j, 0, meta);
            else if (cabs_lt(xi, 1e-13)) block_fail(&s_err, WE_ZIP_COLL, j, 0, meta);
            else {
                s_rec = mk_open(xi, br);
                recs[nrec] = s_rec;
            }
        }
        ++nrec;
        __syncthreads();
        if (s_err) return;
        apply_all();
        __syncthreads();
    }
    double bad = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (c_nan(pts[i])) bad = 1;
    bad = block_max(bad, red);
    if (bad > 0) {
        if (threadIdx.x == 0) block_fail(&s_err, WE_NAN, 0, 1, meta);
        return;
    }
    __shared__ int s_has;
    if (threadIdx.x == 0) {
        const double2 w0 = pts[0];
        s_has = 0;
        if (!c_isinf(w0)) {
            if (c_zero(w0)) {
                block_fail(&s_err, WE_FAR0, 0, 0, meta);
            } else {
                Rec r = mk_mob(C(1, 0), C(0, 0), cdiv(C(-1.0, 0.0), w0), C(1, 0), true);
                mob_pin(r, w0, cinf(), br);
                mob_pin(r, C(0, 0), C(0, 0), br);
                s_rec = r;
                recs[nrec] = r;
                s_has = 1;
            }
        }
    }
    __syncthreads();
    if (s_err) return;
    if (s_has) {
        ++nrec;
        apply_all();
        __syncthreads();
    }
    bad = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (c_nan(pts[i])) bad = 1;
    bad = block_max(bad, red);
    if (threadIdx.x == 0) {
        meta[0] = nrec;
        if (bad > 0) block_fail(&s_err, WE_NAN, 0, 2, meta);
    }
}

__global__ void k_interior(const double2* __restrict__ tv, const int32_t* __restrict__ src, int n, int reverse,
                           double2* scratch, double* out) {
    __shared__ double red[32];
    for (int i = threadIdx.x; i < n; i += blockDim.x) scratch[i] = tv[src[reverse ? n - 1 - i : i]];
    __syncthreads();
    double2 c;
    bool ok = interior_point(scratch, n, red, &c);
    if (threadIdx.x == 0) {
        out[0] = c.x;
        out[1] = c.y;
        out[2] = ok ? 0.0 : 1.0;
    }
}

// z[i] = add + 1 / (z[i] - sub)  (pipeline.py:253-263 exterior inversion)
__global__ void k_inv_shift(double2* z, const int32_t* __restrict__ idx, int64_t n, double2 add, double2 sub) {
    GRID_STRIDE(i, n) {
        int64_t j = idx ? idx[i] : i;
        z[j] = cadd(add, cdiv(C(1.0, 0.0), csub(z[j], sub)));
    }
}

// gather/scatter helpers between tracked values and submesh-local vertices
__global__ void k_gather_c(const double2* __restrict__ src, const int32_t* __restrict__ idx, double2* dst,
                           int64_t n) {
    GRID_STRIDE(i, n) dst[i] = src[idx[i]];
}
__global__ void k_scatter_c(const double2* __restrict__ src, const int32_t* __restrict__ idx, double2* dst,
                            int64_t n) {
    GRID_STRIDE(i, n) dst[idx[i]] = src[i];
}

}  // namespace weld
}  // namespace pgcp

// ===========================================================================
// host side
namespace pgcp {
namespace weld {
namespace {

std::string err_text(int code, int idx, int aux, double a = 0, double b = 0, double c = 0) {
    char buf[256];
    static const char* stage[] = {"", "zipping", "intermediate form", "partial weld", "geodesic algorithm", "apply_log"};
    switch (code) {
        case WE_ZIP01: return "zip points 0 and 1 coincide";
        case WE_ZIP_HALF: snprintf(buf, sizeof buf, "zip point %d left the right half-plane", idx); return buf;
        case WE_ZIP_AXIS:
            snprintf(buf, sizeof buf, "zip point %d landed on the imaginary axis (duplicate or non-Jordan input)", idx);
            return buf;
        case WE_ZIP_COLL:
            snprintf(buf, sizeof buf, "zip points %d and %d collapsed (spacing below 1e-13 in the zip frame)", idx - 1, idx);
            return buf;
        case WE_NAN:
            snprintf(buf, sizeof buf, "numerical breakdown (NaN) during %s", stage[aux >= 1 && aux <= 5 ? aux : 3]);
            return buf;
        case WE_FAR0: return "far end of the zip collapsed to 0";
        case WE_ALIGN_A: snprintf(buf, sizeof buf, "alignment point %d (a side) left the imaginary axis", idx); return buf;
        case WE_ALIGN_B: snprintf(buf, sizeof buf, "alignment point %d (b side) left the imaginary axis", idx); return buf;
        case WE_ORDER:
            snprintf(buf, sizeof buf, "alignment points %d not strictly ordered on the imaginary axis (invalid correspondence)", idx);
            return buf;
        case WE_TRACK: return "tracking points degenerated during welding";
        case WE_FAREND: return "far ends of the two slits diverged";
        case WE_SEAM:
            snprintf(buf, sizeof buf, "seam alignment error %.3e exceeds %g x scale %.3e", a, b, c);
            return buf;
        case WE_PRE:
            return aux == 1 ? "no finite boundary points"
                            : (aux == 2 ? "degenerate boundary (all points coincide)"
                                        : "could not place tracking origin off the boundary");
        case WE_THREE: return "three-point Mobius needs distinct points";
        case WE_K: snprintf(buf, sizeof buf, "shared prefix length k=%d out of range", idx); return buf;
        case WE_GEO_DISK: return "interior point left the unit disk during the geodesic mapping";
        case WE_GEO_CIRCLE: snprintf(buf, sizeof buf, "boundary point left the unit circle by %.3e", a); return buf;
        case WE_INTERIOR: return "could not locate a point inside the polygon";
        case WE_TIMEOUT:
            snprintf(buf, sizeof buf, "internal error: weld wavefront stalled at record %d (loop %d)", idx, aux);
            return buf;
        default: return "weld failure";
    }
}


int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

template <int NT>
int prep_phase1(int CS, size_t smem) {
    if (CS > 8) PGCP_TRY_CUDA(cudaFuncSetAttribute(k_phase1c<NT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    if (smem > 48 * 1024)
        PGCP_TRY_CUDA(cudaFuncSetAttribute(k_phase1c<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    return PGCP_OK;
}

constexpr int WAVE_PT = 256;  // point threads per CTA of k_phase1w (+ one forwarder warp)

int prep_phase1w(int CS, size_t smem) {
    if (CS > 8)
        PGCP_TRY_CUDA(cudaFuncSetAttribute(k_phase1w<WAVE_PT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    if (smem > 48 * 1024)
        PGCP_TRY_CUDA(cudaFuncSetAttribute(k_phase1w<WAVE_PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    return PGCP_OK;
}

double bits_to_d(unsigned long long b) {
    double d;
    memcpy(&d, &b, sizeof d);
    return d;
}

}  // namespace

// A weld schedule prepared for one run: levels, launch-order descriptors,
// write-back lists and every device buffer, uploaded on the preparing stream.
// pipeline.py prepares it on the planning thread while the flatten runs, so
// the weld stage starts with its first launch (the preparation is ~0.4 ms of
// host time on cfg 2).
struct Schedule {
    int nsteps = 0, nlev = 0;
    std::vector<int> level, order, pos;
    std::vector<StepDesc> sd;
    std::vector<int64_t> lev_wb;
    std::vector<int32_t> wb3, h_src;
    int64_t rec_tot = 0, arc_tot = 0;
    DevBuf<StepDesc> d_sd;
    DevBuf<int32_t> d_src, d_wb;
    DevBuf<Rec> d_recs;
    DevBuf<double2> d_arc;
    DevBuf<double> d_meta;
    DevBuf<unsigned long long> d_max;
    DevBuf<int> d_nan, d_prog, d_tmo;
    DevBuf<long long> d_wtime;
    bool streamed = true, wtiming = false, used = false;
    cudaStream_t sp = nullptr;     // the preparing stream (allocations, uploads)
    cudaEvent_t ready = nullptr;   // recorded on sp after the uploads
    double prep_ms = 0;
    ~Schedule() {
        if (ready) cudaEventDestroy(ready);
    }
};

//  info  host int32 [nsteps*6]: k, closed, na, nb, comp_a, comp_b
//  src   host int32 [sum(na+nb)] slot ids of a_cycle then b_cycle per step
//  wb_off host int64 [nsteps+1], wb host int32 [2*total] (slot, code)
int schedule_prepare(int32_t nsteps, const int32_t* info, const int32_t* src, const int64_t* wb_off, const int32_t* wb,
                     cudaStream_t s, Schedule* S) {
    S->nsteps = nsteps;
    S->sp = s;
    if (nsteps <= 0) return PGCP_OK;
    const auto th0 = std::chrono::steady_clock::now();
    // levels: a step waits for the previous steps on either of its components
    std::vector<int>& level = S->level;
    level.assign(nsteps, 0);
    {
        std::vector<std::pair<int, int>> last;  // comp -> level
        std::unordered_map<int, int> lv;
        for (int i = 0; i < nsteps; ++i) {
            int ca = info[6 * i + 4], cb = info[6 * i + 5];
            int l = 0;
            if (lv.count(ca)) l = std::max(l, lv[ca] + 1);
            if (lv.count(cb)) l = std::max(l, lv[cb] + 1);
            level[i] = l;
            lv[ca] = l;
            lv[cb] = l;
        }
    }
    const int nlev = S->nlev = *std::max_element(level.begin(), level.end()) + 1;
    // order steps by (level, index)
    std::vector<int>& order = S->order;
    order.resize(nsteps);
    for (int i = 0; i < nsteps; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return level[x] < level[y]; });
    std::vector<int>& pos = S->pos;
    pos.resize(nsteps);
    for (int q = 0; q < nsteps; ++q) pos[order[q]] = q;
    // descriptors (in launch order)
    std::vector<StepDesc>& sd = S->sd;
    sd.resize(nsteps);
    std::vector<int64_t> src_off(nsteps + 1, 0);
    for (int i = 0; i < nsteps; ++i) src_off[i + 1] = src_off[i] + info[6 * i + 2] + info[6 * i + 3];
    int64_t& rec_tot = S->rec_tot;
    int64_t& arc_tot = S->arc_tot;
    rec_tot = arc_tot = 0;
    for (int q = 0; q < nsteps; ++q) {
        int i = order[q];
        StepDesc& d = sd[q];
        d.k = info[6 * i];
        d.closed = info[6 * i + 1];
        d.na = info[6 * i + 2];
        d.nb = info[6 * i + 3];
        d.src = src_off[i];
        d.cap = 2 * d.k + 16;
        d.pad = 0;
        d.rec = rec_tot;
        rec_tot += 2 * (int64_t)d.cap;
        d.arc = arc_tot;
        arc_tot += 2 * (int64_t)(d.k + 3);
    }
    // write-back entries (slot, code, launch-order step)
    int64_t nwb = wb_off[nsteps];
    std::vector<int32_t>& wb3 = S->wb3;
    wb3.resize(3 * std::max<int64_t>(nwb, 1));
    std::vector<int64_t>& lev_wb = S->lev_wb;
    lev_wb.assign(nlev + 1, 0);
    {
        int64_t o = 0;
        for (int l = 0; l < nlev; ++l) {
            lev_wb[l] = o;
            for (int q = 0; q < nsteps; ++q) {
                int i = order[q];
                if (level[i] != l) continue;
                for (int64_t e = wb_off[i]; e < wb_off[i + 1]; ++e) {
                    wb3[3 * o] = wb[2 * e];
                    wb3[3 * o + 1] = wb[2 * e + 1];
                    wb3[3 * o + 2] = q;
                    ++o;
                }
            }
        }
        lev_wb[nlev] = o;
    }
    auto& d_sd = S->d_sd;
    auto& d_src = S->d_src;
    auto& d_wb = S->d_wb;
    auto& d_recs = S->d_recs;
    auto& d_arc = S->d_arc;
    auto& d_meta = S->d_meta;
    auto& d_max = S->d_max;
    auto& d_nan = S->d_nan;
    PGCP_TRY(d_sd.alloc(nsteps, s));
    PGCP_TRY(d_src.alloc(src_off[nsteps], s));
    PGCP_TRY(d_wb.alloc(3 * std::max<int64_t>(nwb, 1), s));
    PGCP_TRY(d_recs.alloc(rec_tot, s));
    PGCP_TRY(d_arc.alloc(arc_tot, s));
    PGCP_TRY(d_meta.alloc((int64_t)META * nsteps, s));
    PGCP_TRY(d_max.alloc(3 * (int64_t)nsteps, s));
    PGCP_TRY(d_max.zero(s));
    PGCP_TRY(d_nan.alloc(1, s));
    PGCP_TRY(d_nan.zero(s));
    // streamed replay (default): each level's replay runs concurrently with
    // its phase 1 (PGCP_WELD_STREAM=0: after it)
    const bool streamed = S->streamed = env_int("PGCP_WELD_STREAM", 1) != 0;
    auto& d_wtime = S->d_wtime;  // PGCP_WELD_TIMING: phase-1 zip-loop cycle split per step
    const bool wtiming = S->wtiming = env_int("PGCP_WELD_TIMING", 0) != 0;
    if (wtiming) {
        PGCP_TRY(d_wtime.alloc(4 * (int64_t)nsteps, s));
        PGCP_TRY(d_wtime.zero(s));
    }
    auto& d_prog = S->d_prog;
    auto& d_tmo = S->d_tmo;
    if (streamed) {
        PGCP_TRY(d_prog.alloc(2 * (int64_t)nsteps, s));
        PGCP_TRY(d_prog.zero(s));
        PGCP_TRY(d_tmo.alloc(1, s));
        PGCP_TRY(d_tmo.zero(s));
    }
    PGCP_TRY_CUDA(cudaMemcpyAsync(d_sd.p, sd.data(), nsteps * sizeof(StepDesc), cudaMemcpyHostToDevice, s));
    S->h_src.assign(src, src + src_off[nsteps]);  // the caller's array need not outlive this call
    PGCP_TRY_CUDA(cudaMemcpyAsync(d_src.p, S->h_src.data(), src_off[nsteps] * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(d_wb.p, wb3.data(), 3 * nwb * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    PGCP_TRY_CUDA(cudaEventCreateWithFlags(&S->ready, cudaEventDisableTiming));
    PGCP_TRY_CUDA(cudaEventRecord(S->ready, s));
    S->prep_ms = 1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - th0).count();
    return PGCP_OK;
}

// Run a prepared schedule on the tracked values tv (device complex), once.
//  out   host f64 [nsteps*8]: seam_error, seam_residual, area(res.a arc), status,
//        nrec_a, nrec_b, level, spare
int schedule_execute(Schedule* S, double2* tv, double hard_tol, double* out, Rec* recs_host, int64_t recs_cap_total,
                     cudaStream_t s) {
    const int nsteps = S->nsteps;
    if (nsteps <= 0) return PGCP_OK;
    if (S->used) {
        set_error("pgcp_weld_schedule_execute: a prepared schedule runs once");
        return PGCP_E_INVALID;
    }
    S->used = true;
    if (s != S->sp) PGCP_TRY_CUDA(cudaStreamWaitEvent(s, S->ready, 0));  // uploads happened on the preparing stream
    const int nlev = S->nlev;
    const std::vector<int>& level = S->level;
    const std::vector<int>& order = S->order;
    const std::vector<int>& pos = S->pos;
    const std::vector<StepDesc>& sd = S->sd;
    const std::vector<int64_t>& lev_wb = S->lev_wb;
    const int64_t rec_tot = S->rec_tot;
    auto& d_sd = S->d_sd;
    auto& d_src = S->d_src;
    auto& d_wb = S->d_wb;
    auto& d_recs = S->d_recs;
    auto& d_arc = S->d_arc;
    auto& d_meta = S->d_meta;
    auto& d_max = S->d_max;
    auto& d_nan = S->d_nan;
    auto& d_prog = S->d_prog;
    auto& d_tmo = S->d_tmo;
    auto& d_wtime = S->d_wtime;
    const bool streamed = S->streamed, wtiming = S->wtiming;
    const auto th1 = std::chrono::steady_clock::now();
    // PGCP_WELD_TIMING: CUDA events around the setup copies and every level
    std::vector<cudaEvent_t> lev_ev;
    if (wtiming) {
        lev_ev.resize(nlev + 2);
        for (auto& e : lev_ev) PGCP_TRY_CUDA(cudaEventCreate(&e));
        PGCP_TRY_CUDA(cudaEventRecord(lev_ev[0], s));
    }
    int q0 = 0;
    for (int l = 0; l < nlev; ++l) {
        int q1 = q0;
        while (q1 < nsteps && level[order[q1]] == l) ++q1;
        if (wtiming && l == 0) PGCP_TRY_CUDA(cudaEventRecord(lev_ev[1], s));
        Phase1Args a;
        a.steps = d_sd.p + q0;
        a.src = d_src.p;
        a.tv = tv;
        a.arc_out = d_arc.p;
        a.recs = d_recs.p;
        a.meta = d_meta.p + (int64_t)META * q0;
        a.geodesic = 0;
        a.prog = streamed ? d_prog.p + 2 * q0 : nullptr;
        a.prog_every = std::max(1, env_int("PGCP_WELD_PROG_EVERY", 8));
        a.timing = d_wtime.p ? d_wtime.p + 4 * q0 : nullptr;
        a.spin_ns = env_int("PGCP_WELD_SPIN_NS", 0);
        a.timing_detail = env_int("PGCP_WELD_TIMING", 0) >= 2;
        int kmax = 0;
        for (int q = q0; q < q1; ++q) kmax = std::max(kmax, sd[q].k);
        const int NP = 2 * (kmax + 3);
        // wavefront phase 1 (default) while every point has its own thread
        const bool wave = env_int("PGCP_WELD_WAVE", 1) != 0 && NP <= PC_MAXCS * WAVE_PT;
        const int ppt = std::max(1, env_int("PGCP_WELD_PPT", 1));
        const int NT = wave ? WAVE_PT + 32 : (env_int("PGCP_WELD_NT", 256) >= 512 ? 512 : 256);
        int CS = wave ? (NP + WAVE_PT - 1) / WAVE_PT : std::min(PC_MAXCS, (NP + NT * ppt - 1) / (NT * ppt));
        const int chunk = (NP + CS - 1) / CS;
        size_t smem = wave ? (size_t)96 * (kmax + 1) + 16 : (size_t)chunk * (sizeof(double2) + 1) + 16;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)((q1 - q0) * CS), 1, 1);
        cfg.blockDim = dim3(NT, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (wave) {
            PGCP_TRY(prep_phase1w(CS, smem));
            PGCP_TRY_CUDA(cudaLaunchKernelEx(&cfg, k_phase1w<WAVE_PT>, a));
        } else if (NT == 512) {
            PGCP_TRY(prep_phase1<512>(CS, smem));
            PGCP_TRY_CUDA(cudaLaunchKernelEx(&cfg, k_phase1c<512>, a));
        } else {
            PGCP_TRY(prep_phase1<256>(CS, smem));
            PGCP_TRY_CUDA(cudaLaunchKernelEx(&cfg, k_phase1c<256>, a));
        }
        PGCP_LAUNCH_CHECK();
        int64_t n = lev_wb[l + 1] - lev_wb[l];
        if (n > 0) {
            ReplayArgs r;
            r.wb = d_wb.p + 3 * lev_wb[l];
            r.nwb = n;
            r.steps = d_sd.p;
            r.recs = d_recs.p;
            r.tv = tv;
            r.arc_out = d_arc.p;
            r.meta = d_meta.p;
            r.maxbits = d_max.p;
            r.nan_flag = d_nan.p;
            if (streamed) {
                cudaLaunchConfig_t rc = {};
                rc.gridDim = dim3((unsigned)grid_for(n, 128), 1, 1);  // larger CTAs measured slower
                rc.blockDim = dim3(128, 1, 1);
                rc.dynamicSmemBytes = 0;
                rc.stream = s;
                cudaLaunchAttribute ra[1];
                ra[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                ra[0].val.programmaticStreamSerializationAllowed = 1;
                rc.attrs = ra;
                rc.numAttrs = 1;
                PGCP_TRY_CUDA(cudaLaunchKernelEx(&rc, k_replay_stream, r, (const int*)d_prog.p, d_tmo.p));
                count_launch();
            } else {
                k_replay_slots<<<grid_for(n, 128), 128, 0, s>>>(r);
                PGCP_LAUNCH_CHECK();
            }
        }
        q0 = q1;
        if (wtiming) PGCP_TRY_CUDA(cudaEventRecord(lev_ev[l + 2], s));
    }
    const auto th2 = std::chrono::steady_clock::now();  // every level launched
    std::vector<double> meta((size_t)META * nsteps);
    std::vector<unsigned long long> mx(3 * (size_t)nsteps);
    int hnan = 0;
    // pinned staging (common.cuh): a pageable read would hold the driver
    // while the whole weld drains, stalling other host threads' launches
    PGCP_TRY(d2h_async(meta.data(), d_meta.p, meta.size() * sizeof(double), s));
    PGCP_TRY(d2h_async(mx.data(), d_max.p, mx.size() * sizeof(unsigned long long), s));
    PGCP_TRY(d2h_async(&hnan, d_nan.p, sizeof(int), s));
    int htmo = 0;
    if (streamed) PGCP_TRY(d2h_async(&htmo, d_tmo.p, sizeof(int), s));
    if (recs_host && recs_cap_total >= rec_tot) PGCP_TRY(d2h_async(recs_host, d_recs.p, rec_tot * sizeof(Rec), s));
    PGCP_TRY(d2h_flush(s));
    if (wtiming) {
        PGCP_TRY_CUDA(cudaEventSynchronize(lev_ev.back()));
        const auto th3 = std::chrono::steady_clock::now();
        auto ms_of = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
            return 1e3 * std::chrono::duration<double>(b - a).count();
        };
        fprintf(stderr, "[weld timing] host ms: preparation %.3f, launches %.3f, wait + reads %.3f\n", S->prep_ms,
                ms_of(th1, th2), ms_of(th2, th3));
        fprintf(stderr, "[weld timing] device ms:");
        for (int l = 0; l + 1 < (int)lev_ev.size(); ++l) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, lev_ev[l], lev_ev[l + 1]);
            if (l == 0)
                fprintf(stderr, " setup copies %.3f", ms);
            else
                fprintf(stderr, " L%d %.3f", l - 1, ms);
        }
        fprintf(stderr, "\n");
        for (auto& e : lev_ev) cudaEventDestroy(e);
        std::vector<long long> wt(4 * (size_t)nsteps);
        PGCP_TRY_CUDA(cudaMemcpy(wt.data(), d_wtime.p, wt.size() * sizeof(long long), cudaMemcpyDeviceToHost));
        for (int q = 0; q < nsteps; ++q) {
            if (wt[4 * q + 3] < 0) {  // k_phase1w: [open part, close part] cycles
                const double n = (double)std::max(1ll, -wt[4 * q + 3]);
                fprintf(stderr, "[weld timing] step %d k %d level %d (wavefront): open %.0f cycles/record, close %.0f\n",
                        q, sd[q].k, level[order[q]], wt[4 * q] / n, wt[4 * q + 1] / n);
                continue;
            }
            const double n = (double)std::max(1ll, wt[4 * q + 3]);
            fprintf(stderr, "[weld timing] step %d k %d level %d: zip cycles/record publish+barrier %.0f build %.0f "
                    "apply %.0f\n", q, sd[q].k, level[order[q]], wt[4 * q] / n, wt[4 * q + 1] / n, wt[4 * q + 2] / n);
        }
    }
    int status = PGCP_OK;
    for (int i = 0; i < nsteps; ++i) {
        int q = pos[i];
        const double* m = &meta[(size_t)META * q];
        int code = (int)m[2];
        double stage = std::max(m[10], bits_to_d(mx[3 * q]));
        double fa = std::max(m[11], bits_to_d(mx[3 * q + 1]));
        double fb = std::max(m[12], bits_to_d(mx[3 * q + 2]));
        double scale = std::max(std::max(fa, fb), m[13]);
        if (scale <= 0) scale = 1.0;
        double2 qa = make_double2(m[6], m[7]), qb = make_double2(m[8], m[9]);
        bool ia = std::isinf(qa.x) || std::isinf(qa.y), ib = std::isinf(qb.x) || std::isinf(qb.y);
        bool far_bad = false;
        if (code == 0 || code == WE_TRACK || code == WE_THREE || code == WE_NAN) {
            double sa = stage > 0 ? stage : 1.0;
            far_bad = (ia != ib) || (!ia && std::hypot(qa.x - qb.x, qa.y - qb.y) > 1e-9 * std::max(sa, 1.0));
            if (code == WE_NAN && (int)m[4] != 3) far_bad = false;
        }
        std::string msg;
        if (far_bad) {
            code = WE_FAREND;
            msg = err_text(code, 0, 0);
        } else if (code != 0) {
            msg = err_text(code, (int)m[3], (int)m[4]);
        } else if (m[5] > hard_tol * scale) {
            code = WE_SEAM;
            msg = err_text(code, 0, 0, m[5], hard_tol, scale);
        }
        double resid_scale = std::max(fa, fb);
        out[8 * i + 0] = m[5];
        out[8 * i + 1] = resid_scale > 0 ? m[5] / resid_scale : 0.0;
        out[8 * i + 2] = m[16];
        out[8 * i + 3] = code;
        out[8 * i + 4] = m[0];
        out[8 * i + 5] = m[1];
        out[8 * i + 6] = level[i];
        out[8 * i + 7] = (double)sd[q].rec;
        if (code != 0 && status == PGCP_OK) {
            status = PGCP_E_WELD;
            set_error("weld step %d: %s", i, msg.c_str());
        }
    }
    if (htmo) {
        set_error("internal: streamed weld replay timed out waiting for phase 1");
        return PGCP_E_CUDA;
    }
    if (status == PGCP_OK && hnan) {
        set_error("numerical breakdown (NaN) during apply_log");
        status = PGCP_E_WELD;
    }
    return status;
}

// Run a whole weld schedule on the tracked values tv (prepare + execute).
int run_schedule(double2* tv, int32_t nsteps, const int32_t* info, const int32_t* src, const int64_t* wb_off,
                 const int32_t* wb, double hard_tol, double* out, Rec* recs_host, int64_t recs_cap_total,
                 cudaStream_t s) {
    if (nsteps <= 0) return PGCP_OK;
    Schedule S;
    PGCP_TRY(schedule_prepare(nsteps, info, src, wb_off, wb, s, &S));
    return schedule_execute(&S, tv, hard_tol, out, recs_host, recs_cap_total, s);
}

}  // namespace weld
}  // namespace pgcp

using namespace pgcp;
using namespace pgcp::weld;

extern "C" {

PGCP_API int pgcp_weld_schedule_prepare(int32_t nsteps, const int32_t* info, const int32_t* src, const int64_t* wb_off,
                                        const int32_t* wb, void* stream, void** handle) {
    if (!handle || nsteps < 0 || (nsteps > 0 && (!info || !src || !wb_off))) {
        set_error("pgcp_weld_schedule_prepare: invalid arguments");
        return PGCP_E_INVALID;
    }
    *handle = nullptr;
    std::unique_ptr<Schedule> S(new Schedule());
    int rc = schedule_prepare(nsteps, info, src, wb_off, wb, reinterpret_cast<cudaStream_t>(stream), S.get());
    if (rc != PGCP_OK) return rc;
    *handle = S.release();
    return PGCP_OK;
}

PGCP_API int pgcp_weld_schedule_execute(void* handle, double* tv, double hard_tol, double* out, pgcp_rec* recs_host,
                                        int64_t recs_cap, void* stream) {
    Schedule* S = reinterpret_cast<Schedule*>(handle);
    if (!S || !tv || (S->nsteps > 0 && !out)) {
        set_error("pgcp_weld_schedule_execute: invalid arguments");
        return PGCP_E_INVALID;
    }
    return schedule_execute(S, reinterpret_cast<double2*>(tv), hard_tol, out, recs_host, recs_cap,
                            reinterpret_cast<cudaStream_t>(stream));
}

PGCP_API void pgcp_weld_schedule_free(void* handle) { delete reinterpret_cast<Schedule*>(handle); }

PGCP_API int pgcp_weld_schedule_run(double* tv, int32_t nsteps, const int32_t* info, const int32_t* src,
                                    const int64_t* wb_off, const int32_t* wb, double hard_tol, double* out,
                                    pgcp_rec* recs_host, int64_t recs_cap, void* stream) {
    if (!tv || nsteps < 0 || (nsteps > 0 && (!info || !src || !wb_off || !out))) {
        set_error("pgcp_weld_schedule_run: invalid arguments");
        return PGCP_E_INVALID;
    }
    return run_schedule(reinterpret_cast<double2*>(tv), nsteps, info, src, wb_off, wb, hard_tol, out, recs_host,
                        recs_cap, reinterpret_cast<cudaStream_t>(stream));
}

// apply_log (welding.py:512-526): records from the host, points on the device
PGCP_API int pgcp_weld_replay(const pgcp_rec* recs, int32_t nrec, double* pts, int8_t* sides, int64_t npts,
                              void* stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (npts <= 0) return PGCP_OK;
    DevBuf<Rec> d;
    DevBuf<int> flag;
    PGCP_TRY(d.alloc(std::max(nrec, 1), s));
    PGCP_TRY(flag.alloc(1, s));
    PGCP_TRY(flag.zero(s));
    if (nrec > 0) PGCP_TRY_CUDA(cudaMemcpyAsync(d.p, recs, nrec * sizeof(Rec), cudaMemcpyHostToDevice, s));
    k_replay_points<<<grid_for(npts, 128), 128, 0, s>>>(d.p, nrec, reinterpret_cast<double2*>(pts), sides, npts,
                                                         flag.p);
    PGCP_LAUNCH_CHECK();
    int h = 0;
    PGCP_TRY(fetch_scalar(flag.p, &h, s));
    if (h) {
        set_error("numerical breakdown (NaN) during apply_log");
        return PGCP_E_WELD;
    }
    return PGCP_OK;
}

// geodesic_to_circle over the cycle tv[src[0..n)] (host src).
//   circ  device complex [n], recs host [cap], meta host f64 [8]: nrec, err, idx,
//   aux, circle error, interior.re, interior.im
PGCP_API int pgcp_weld_geodesic(const double* tv, const int32_t* src, int32_t n, const double* interior,
                                double* circ, pgcp_rec* recs, int32_t cap, double* meta_out, void* stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (n < 3) {
        set_error("need at least 3 boundary points");
        return PGCP_E_WELD;
    }
    if (cap < n + 4) {
        set_error("pgcp_weld_geodesic: record capacity %d < %d", cap, n + 4);
        return PGCP_E_INVALID;
    }
    DevBuf<int32_t> d_src, d_order;
    DevBuf<double2> d_pts;
    DevBuf<int8_t> d_sides;
    DevBuf<Rec> d_recs;
    DevBuf<double> d_meta;
    PGCP_TRY(d_src.alloc(n, s));
    PGCP_TRY(d_order.alloc(n, s));
    PGCP_TRY(d_pts.alloc(n + 1, s));
    PGCP_TRY(d_sides.alloc(n + 1, s));
    PGCP_TRY(d_recs.alloc(cap, s));
    PGCP_TRY(d_meta.alloc(META, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(d_src.p, src, n * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    GeoArgs a;
    a.tv = reinterpret_cast<const double2*>(tv);
    a.src = d_src.p;
    a.n = n;
    a.has_interior = interior != nullptr;
    a.interior = interior ? make_double2(interior[0], interior[1]) : make_double2(0, 0);
    a.pts = d_pts.p;
    a.sides = d_sides.p;
    a.order = d_order.p;
    a.circ = reinterpret_cast<double2*>(circ);
    a.recs = d_recs.p;
    a.meta = d_meta.p;
    k_geodesic<<<1, 512, 0, s>>>(a);
    PGCP_LAUNCH_CHECK();
    double m[META];
    PGCP_TRY_CUDA(cudaMemcpyAsync(m, d_meta.p, sizeof m, cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    int nrec = (int)m[0];
    if (recs && nrec > 0) {
        PGCP_TRY_CUDA(cudaMemcpyAsync(recs, d_recs.p, nrec * sizeof(Rec), cudaMemcpyDeviceToHost, s));
        PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    }
    if (meta_out) {
        meta_out[0] = nrec;
        meta_out[1] = m[2];
        meta_out[2] = m[3];
        meta_out[3] = m[4];
        meta_out[4] = m[5];
        meta_out[5] = m[6];
        meta_out[6] = m[7];
    }
    if (m[2] != 0) {
        set_error("%s", err_text((int)m[2], (int)m[3], (int)m[4], m[5]).c_str());
        return PGCP_E_WELD;
    }
    return PGCP_OK;
}

// intermediate_form (welding.py:578-602) of n device points, in place
PGCP_API int pgcp_weld_intermediate(double* pts, int8_t* sides, int32_t n, int32_t k, int32_t branch,
                                    pgcp_rec* recs, int32_t cap, int32_t* nrec_out, void* stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (k < 1) {
        set_error("zip count must be at least 1");
        return PGCP_E_WELD;
    }
    if (n < k + 1) {
        set_error("need at least k + 1 points");
        return PGCP_E_WELD;
    }
    if (cap < k + 1 || (branch != UP && branch != DOWN)) {
        set_error("pgcp_weld_intermediate: invalid arguments");
        return PGCP_E_INVALID;
    }
    DevBuf<Rec> d_recs;
    DevBuf<double> d_meta;
    PGCP_TRY(d_recs.alloc(k + 1, s));
    PGCP_TRY(d_meta.alloc(META, s));
    k_zip_form<<<1, 512, 0, s>>>(reinterpret_cast<double2*>(pts), sides, n, k, branch, d_recs.p, d_meta.p);
    PGCP_LAUNCH_CHECK();
    double m[META];
    PGCP_TRY_CUDA(cudaMemcpyAsync(m, d_meta.p, sizeof m, cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    if (m[2] != 0) {
        set_error("%s", err_text((int)m[2], (int)m[3], (int)m[4]).c_str());
        return PGCP_E_WELD;
    }
    const int nrec = (int)m[0];
    if (recs && nrec > 0) {
        PGCP_TRY_CUDA(cudaMemcpyAsync(recs, d_recs.p, nrec * sizeof(Rec), cudaMemcpyDeviceToHost, s));
        PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    }
    if (nrec_out) *nrec_out = nrec;
    return PGCP_OK;
}

// polygon_interior_point (welding.py:781-796) of tv[src] (optionally reversed)
PGCP_API int pgcp_polygon_interior(const double* tv, const int32_t* src, int32_t n, int reverse, double* out,
                                   void* stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    DevBuf<int32_t> d_src;
    DevBuf<double2> scr;
    DevBuf<double> d_out;
    PGCP_TRY(d_src.alloc(n, s));
    PGCP_TRY(scr.alloc(n, s));
    PGCP_TRY(d_out.alloc(3, s));
    PGCP_TRY_CUDA(cudaMemcpyAsync(d_src.p, src, n * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    k_interior<<<1, 512, 0, s>>>(reinterpret_cast<const double2*>(tv), d_src.p, n, reverse, scr.p, d_out.p);
    PGCP_LAUNCH_CHECK();
    double h[3];
    PGCP_TRY_CUDA(cudaMemcpyAsync(h, d_out.p, sizeof h, cudaMemcpyDeviceToHost, s));
    PGCP_TRY_CUDA(cudaStreamSynchronize(s));
    if (h[2] != 0) {
        set_error("could not locate a point inside the polygon");
        return PGCP_E_WELD;
    }
    out[0] = h[0];
    out[1] = h[1];
    return PGCP_OK;
}

// z[idx[i]] = add + 1 / (z[idx[i]] - sub)   (idx device, may be NULL)
PGCP_API int pgcp_inv_shift(double* z, const int32_t* idx, int64_t n, double add_re, double add_im, double sub_re,
                            double sub_im, void* stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (n <= 0) return PGCP_OK;
    k_inv_shift<<<grid_for(n, 256), 256, 0, s>>>(reinterpret_cast<double2*>(z), idx, n, make_double2(add_re, add_im),
                                                 make_double2(sub_re, sub_im));
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}

PGCP_API int pgcp_gather_complex(const double* src, const int32_t* idx, double* dst, int64_t n, void* stream) {
    if (n <= 0) return PGCP_OK;
    k_gather_c<<<grid_for(n, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const double2*>(src), idx, reinterpret_cast<double2*>(dst), n);
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}

PGCP_API int pgcp_scatter_complex(const double* src, const int32_t* idx, double* dst, int64_t n, void* stream) {
    if (n <= 0) return PGCP_OK;
    k_scatter_c<<<grid_for(n, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const double2*>(src), idx, reinterpret_cast<double2*>(dst), n);
    PGCP_LAUNCH_CHECK();
    return PGCP_OK;
}

}  // extern "C"
