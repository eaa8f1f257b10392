// cc_device.cuh — device building blocks of the Coulomb collision operator
// (arXiv 2508.06771 §4.4, Table 5).  Product code: written for sm_100a from
// the published definitions; shares nothing with oracle/.
//
//   philox4x32_10   CCS4 randoms, reading R3
//   u01             two 32-bit words -> uniform on (0,1), R3
//   ppnd16          AS241 inverse normal CDF (Wichura 1988), R4
//   pairing (R1)    keyed permutation of n items: sort-by-Philox-key for
//                   n <= 64, 8-round keyed Feistel + cycle walking above — over
//                   the whole cell (R1), or (R1b) over a cell's full segments
//                   (the segment order) and over each block's slots (tau_b)
//   ta_update       CCS5 Takizuka–Abe pair collision, R5/R8/R9
#pragma once
#include <cstdint>

namespace cc {

constexpr int kSmallCell = 64;          // R1: N <= 64 uses the sort-by-key form
// R1b (blocked pairing): segments of kSeg consecutive stable slots,
// blocks of kBlockSegs segments = kBlock slots (one k_collide_large CTA each)
constexpr int kSeg = 32;
constexpr int kBlockSegs = 12;
constexpr int kBlock = kSeg * kBlockSegs;

// ---------------------------------------------------------------- Philox4x32-10
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1)
{
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// (floor((2^32 hi + lo) / 2^12) + 1/2) * 2^-52 : exact odd multiple of 2^-53.
__device__ __forceinline__ double u01(uint32_t hi, uint32_t lo)
{
    const uint64_t m = ((static_cast<uint64_t>(hi) << 32) | lo) >> 12;
    return __fma_rn(static_cast<double>(m), 0x1.0p-52, 0x1.0p-53);
}

// ---------------------------------------------------------------- fast fp64 reciprocal / rsqrt
// MUFU approximations refined by two Newton steps: a few ulp, far inside the
// 1e-12 parity bar, at ~6 instructions instead of the ~20 of IEEE div / sqrt.
__device__ __forceinline__ double rcp_nr(double x)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

__device__ __forceinline__ double rsqrt_nr(double x)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double h = 0.5 * x;
    double e = fma(-h * y, y, 0.5);
    y = fma(y, e, y);
    e = fma(-h * y, y, 0.5);
    return fma(y, e, y);
}

// ---------------------------------------------------------------- AS241 PPND16
// Split into the central region (|u - 1/2| <= 0.425, ~85% of draws) and the
// tails, so a kernel can evaluate the tails of a whole warp's items together.
__device__ __forceinline__ bool ppnd16_is_central(double p) { return fabs(p - 0.5) <= 0.425; }

// AS241 coefficients (Wichura 1988, PPND16), highest degree first, in constant
// memory so polynomial evaluation reads them as uniform operands.
__constant__ double kAS241[6][8] = {
    {2.5090809287301226727e+3, 3.3430575583588128105e+4, 6.7265770927008700853e+4, 4.5921953931549871457e+4,
     1.3731693765509461125e+4, 1.9715909503065514427e+3, 1.3314166789178437745e+2, 3.3871328727963666080e+0},
    {5.2264952788528545610e+3, 2.8729085735721942674e+4, 3.9307895800092710610e+4, 2.1213794301586595867e+4,
     5.3941960214247511077e+3, 6.8718700749205790830e+2, 4.2313330701600911252e+1, 1.0},
    {7.7454501427834140764e-4, 2.2723844989269184583e-2, 2.4178072517745061177e-1, 1.2704582524523683826e+0,
     3.6478483247632046050e+0, 5.7694972214606914055e+0, 4.6303378461565452959e+0, 1.4234371107496835773e+0},
    {1.0507500716444168432e-9, 5.4759380849953449460e-4, 1.5198666563616457197e-2, 1.4810397642748007459e-1,
     6.8976733498510000455e-1, 1.6763848301838038494e+0, 2.0531916266377588219e+0, 1.0},
    {2.0103343992922881327e-7, 2.7115555687434875782e-5, 1.2426609473880784386e-3, 2.6532189526576123093e-2,
     2.9656057182850489123e-1, 1.7848265399172913358e+0, 5.4637849111641143699e+0, 6.6579046435011037772e+0},
    {2.0442631033899397856e-15, 1.4215117583164458887e-7, 1.8463183175100546818e-5, 7.8686913114561325910e-4,
     1.4875361290850614852e-2, 1.3692988092273580531e-1, 5.9983220655588793769e-1, 1.0}};

// Horner evaluation of the degree-7 polynomial kAS241[row] at r.
__device__ __forceinline__ double as241_poly(int row, double r)
{
    double s = kAS241[row][0];
#pragma unroll
    for (int i = 1; i < 8; ++i) s = s * r + kAS241[row][i];
    return s;
}

__device__ __forceinline__ double ppnd16_central(double p)
{
    const double q = p - 0.5;
    const double r = 0.180625 - q * q;
    return as241_poly(0, r) * q * rcp_nr(as241_poly(1, r));
}

// Tail argument: the smaller tail mass min(p, 1-p), negative for p < 1/2.
__device__ __forceinline__ double ppnd16_tail_arg(double p) { return (p < 0.5) ? -p : 1.0 - p; }

__device__ __forceinline__ double ppnd16_tail(double targ)
{
    double r = sqrt(-log(fabs(targ)));
    const bool near = r <= 5.0;
    r -= near ? 1.6 : 5.0;
    const int row = near ? 2 : 4;
    const double x = as241_poly(row, r) * rcp_nr(as241_poly(row + 1, r));
    return (targ < 0.0) ? -x : x;
}

__device__ __forceinline__ double ppnd16(double p)
{
    return ppnd16_is_central(p) ? ppnd16_central(p) : ppnd16_tail(ppnd16_tail_arg(p));
}

// ---------------------------------------------------------------- pairing (R1)
__device__ __forceinline__ uint32_t fmix32(uint32_t h)
{
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
}

// Parameters of the N > 64 Feistel form for a cell of N slots.
// Both halves stay below 2^16 (L < 2^bL <= 2^15, R < m <= 2^16), so the first
// xor-shift of fmix32(x ^ K), (x ^ K) ^ ((x ^ K) >> 16), equals x ^ K' with the
// per-round constant K' = K ^ (K >> 16): the rounds below are fmix32 exactly,
// two instructions shorter.
struct Feistel {
    uint32_t kp[8];  // K'_r = K_r ^ (K_r >> 16), K_r = k[r mod 4] + (r div 4) * 0x9E3779B9
    uint32_t bL;     // L half: bL bits (a = 2^bL)
    uint32_t m;      // R half: values in [0, m), m = ceil(N / a)
    uint32_t N;
};

__device__ __forceinline__ Feistel make_feistel(uint32_t N, U4 keys)
{
    Feistel f;
    const uint32_t k[4] = {keys.x, keys.y, keys.z, keys.w};
#pragma unroll
    for (uint32_t r = 0; r < 8; ++r) {
        const uint32_t K = k[r & 3u] + (r >> 2) * 0x9E3779B9u;
        f.kp[r] = K ^ (K >> 16);
    }
    const uint32_t b = 32u - __clz(N - 1u);          // ceil(log2 N), N >= 2
    f.bL = b >> 1;
    const uint32_t a = 1u << f.bL;
    f.m = (N + a - 1u) >> f.bL;
    f.N = N;
    return f;
}

// fmix32(x ^ K) for x < 2^16, given K' = K ^ (K >> 16)
__device__ __forceinline__ uint32_t fmix32_small(uint32_t x, uint32_t kp)
{
    uint32_t h = x ^ kp;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
}

__device__ __forceinline__ uint32_t feistel_E(const Feistel& f, uint32_t x)
{
    const uint32_t amask = (1u << f.bL) - 1u;
    uint32_t L = x & amask, R = x >> f.bL;
#pragma unroll
    for (uint32_t r = 0; r < 8; ++r) {
        if ((r & 1u) == 0u) {
            L ^= fmix32_small(R, f.kp[r]) & amask;
        } else {
            const uint32_t s = R + __umulhi(fmix32_small(L, f.kp[r]), f.m);
            R = min(s, s - f.m);                     // (R + t) mod m, R + t < 2m
        }
    }
    return L + (R << f.bL);
}

// E applied to NV independent inputs in lock step (the rounds interleave, so
// the 8-round dependency chains of different inputs hide each other's latency).
template <int NV>
__device__ __forceinline__ void feistel_E_multi(const Feistel& f, uint32_t (&x)[NV])
{
    const uint32_t amask = (1u << f.bL) - 1u;
    uint32_t L[NV], R[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) { L[v] = x[v] & amask; R[v] = x[v] >> f.bL; }
#pragma unroll
    for (uint32_t r = 0; r < 8; ++r) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            if ((r & 1u) == 0u) {
                L[v] ^= fmix32_small(R[v], f.kp[r]) & amask;
            } else {
                const uint32_t s = R[v] + __umulhi(fmix32_small(L[v], f.kp[r]), f.m);
                R[v] = min(s, s - f.m);
            }
        }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) x[v] = L[v] + (R[v] << f.bL);
}

// pi(i) for the Feistel form: cycle walking from i until the value is < N.
__device__ __forceinline__ uint32_t feistel_pi(const Feistel& f, uint32_t i)
{
    uint32_t x = feistel_E(f, i);
    while (x >= f.N) x = feistel_E(f, x);
    return x;
}

// Sort key of item s of an R1 sort-by-key permutation: word (s mod 4) of
// Philox(ctr = (base + s div 4, G, step, purpose), key = seed).  R1's small cell:
// base 0, purpose 2; R1b's block b: base 96 b, purpose 2; R1b's segment order: purpose 6.
__device__ __forceinline__ uint32_t small_key(uint32_t s, uint32_t G, uint32_t step,
                                              uint32_t k0, uint32_t k1, uint32_t base = 0u,
                                              uint32_t purpose = 2u)
{
    const U4 w = philox4x32_10(U4{base + (s >> 2), G, step, purpose}, k0, k1);
    const uint32_t q = s & 3u;
    return q == 0 ? w.x : q == 1 ? w.y : q == 2 ? w.z : w.w;
}

// One thread: the item at position r of the sort-by-key permutation of n <= 64 items
// (used off the hot path: k_triplets, the cc_pairs test hook).
__device__ __noinline__ uint32_t small_select(uint32_t n, uint32_t r, uint32_t G, uint32_t step,
                                              uint32_t k0, uint32_t k1, uint32_t base, uint32_t purpose)
{
    uint32_t key[kSmallCell];
    for (uint32_t s = 0; s < n; s += 4) {
        const U4 w = philox4x32_10(U4{base + (s >> 2), G, step, purpose}, k0, k1);
        key[s] = w.x;
        if (s + 1 < n) key[s + 1] = w.y;
        if (s + 2 < n) key[s + 2] = w.z;
        if (s + 3 < n) key[s + 3] = w.w;
    }
    for (uint32_t s = 0; s < n; ++s) {
        uint32_t rank = 0;
        for (uint32_t t = 0; t < n; ++t) rank += (key[t] < key[s] || (key[t] == key[s] && t < s)) ? 1u : 0u;
        if (rank == r) return s;
    }
    return 0u;
}

// Warp-cooperative pi table of a small cell (N <= 64): pi_sm[q] = slot at
// pair-order position q.  All 32 lanes must call it; the warp must be converged.
__device__ __forceinline__ void small_cell_perm(uint32_t N, uint32_t G, uint32_t step,
                                                uint32_t k0, uint32_t k1, int lane,
                                                int32_t* pi_sm, uint32_t base = 0u, uint32_t purpose = 2u)
{
    const uint32_t s0 = static_cast<uint32_t>(lane), s1 = s0 + 32u;
    const uint32_t r0 = (s0 < N) ? small_key(s0, G, step, k0, k1, base, purpose) : 0xFFFFFFFFu;
    const uint32_t r1 = (s1 < N) ? small_key(s1, G, step, k0, k1, base, purpose) : 0xFFFFFFFFu;
    uint32_t rank0 = 0, rank1 = 0;
    for (uint32_t t = 0; t < N; ++t) {
        const uint32_t src = (t < 32u) ? r0 : r1;
        const uint32_t rt = __shfl_sync(0xFFFFFFFFu, src, static_cast<int>(t & 31u));
        rank0 += (rt < r0 || (rt == r0 && t < s0)) ? 1u : 0u;
        rank1 += (rt < r1 || (rt == r1 && t < s1)) ? 1u : 0u;
    }
    if (s0 < N) pi_sm[rank0] = static_cast<int32_t>(s0);
    if (s1 < N) pi_sm[rank1] = static_cast<int32_t>(s1);
    __syncwarp();
}

// ---------------------------------------------------------------- sin / cos of 2 pi u
// phi = 2 pi u2 (R4): u in (0,1) is reduced exactly to a quadrant q and
// r = 4u - q in [-1/2, 1/2]; x = r pi/2; sin/cos on [-pi/4, pi/4] by the
// classic minimax kernels (FDLIBM __kernel_sin/__kernel_cos coefficients).
__constant__ double kSinCos[12] = {
    -1.66666666666666324348e-01, 8.33333333332248946124e-03, -1.98412698298579493134e-04,
    2.75573137070700676789e-06, -2.50507602534068634195e-08, 1.58969099521155010221e-10,
    4.16666666666666019037e-02, -1.38888888888741095749e-03, 2.48015872894767294178e-05,
    -2.75573143513906633035e-07, 2.08757232129817482790e-09, -1.13596475577881948265e-11};

__device__ __forceinline__ void sincos2pi(double u, double* sn, double* cs)
{
    const double t = 4.0 * u;
    const double q = rint(t);
    const double x = (t - q) * 1.5707963267948966192;   // pi/2
    const double z = x * x;
    double ps = kSinCos[5], pc = kSinCos[11];
#pragma unroll
    for (int i = 4; i >= 0; --i) {
        ps = fma(ps, z, kSinCos[i]);
        pc = fma(pc, z, kSinCos[6 + i]);
    }
    const double s = fma(x * z, ps, x);
    const double c = fma(z * z, pc, fma(-0.5, z, 1.0));
    const int qi = static_cast<int>(q) & 3;
    const double ss = (qi & 1) ? c : s;
    const double cc_ = (qi & 1) ? s : c;
    *sn = (qi & 2) ? -ss : ss;
    *cs = ((qi + 1) & 2) ? -cc_ : cc_;
}

// ---------------------------------------------------------------- pair rotation
// Rotate u = v_a - v_b by the polar angle Theta (given as sin Theta and
// 1 - cos Theta) and azimuth phi = 2 pi u2 in TA77's component form (R9,
// u_perp = 0 branch for u_x = u_y = 0), then v_a += Du/2, v_b -= Du/2.
__device__ __forceinline__ void rotate_pair(double& ax, double& ay, double& az, double& bx, double& by, double& bz,
                                            double ux, double uy, double uz, double u, double sinT, double omc,
                                            double u2)
{
    double sphi, cphi;
    sincos2pi(u2, &sphi, &cphi);
    double dux, duy, duz;
    if (ux == 0.0 && uy == 0.0) {
        dux = u * sinT * cphi;
        duy = u * sinT * sphi;
        duz = -uz * omc;
    } else {
        const double up2 = fma(ux, ux, uy * uy);
        const double ip = rsqrt_nr(up2);             // 1/u_perp
        const double uperp = up2 * ip;
        const double sc = sinT * cphi, ss = sinT * sphi;
        const double A = uz * sc * ip, B = u * ss * ip;
        dux = ux * A - uy * B - ux * omc;
        duy = uy * A + ux * B - uy * omc;
        duz = -uperp * sc - uz * omc;
    }
    ax = fma(0.5, dux, ax); ay = fma(0.5, duy, ay); az = fma(0.5, duz, az);
    bx = fma(-0.5, dux, bx); by = fma(-0.5, duy, by); bz = fma(-0.5, duz, bz);
}

// ---------------------------------------------------------------- TA77 update
// <delta^2> = C / |u|^3; delta = sqrt(<delta^2>) z with z = Phi^-1(u1);
// tan(Theta/2) = delta; phi = 2 pi u2; v_a += Du/2, v_b -= Du/2.
// sin(Theta) = 2 delta/(1+delta^2), 1-cos(Theta) = 2 delta^2/(1+delta^2) with
// |delta| clamped at 1e150 (then 1-cos = 2 exactly and sin(Theta) < 1e-149:
// the algebraically equal limit of R9's t = 1/delta form, no NaN).
__device__ __forceinline__ void ta_update_z(double& ax, double& ay, double& az,
                                            double& bx, double& by, double& bz,
                                            double C, double z, double u2)
{
    const double ux = ax - bx, uy = ay - by, uz = az - bz;
    if (ux == 0.0 && uy == 0.0 && uz == 0.0) return;
    const double usq = fma(ux, ux, fma(uy, uy, uz * uz));
    const double rs = rsqrt_nr(usq);                 // 1/|u|
    const double u = usq * rs;
    const double var = C * (rs * rs) * rs;           // <delta^2>
    const double delta = sqrt(var) * z;
    const double dd = fmin(fabs(delta), 1e150);
    const double d2 = dd * dd;
    const double inv = rcp_nr(1.0 + d2);
    const double sinT = 2.0 * copysign(dd, delta) * inv;
    const double omc = 2.0 * d2 * inv;
    rotate_pair(ax, ay, az, bx, by, bz, ux, uy, uz, u, sinT, omc, u2);
}

// The same update with sqrt(<delta^2>) = sqrt(C) |u|^-3/2 = sqrtC * (1/|u|) * rsqrt(|u|): the
// per-cell sqrt(C) is taken once per CTA, so no IEEE sqrt per pair (a few ulp of delta, far
// inside the 1e-12 parity bar).
__device__ __forceinline__ void ta_update_zs(double& ax, double& ay, double& az,
                                             double& bx, double& by, double& bz,
                                             double sqrtC, double z, double u2)
{
    const double ux = ax - bx, uy = ay - by, uz = az - bz;
    if (ux == 0.0 && uy == 0.0 && uz == 0.0) return;
    const double usq = fma(ux, ux, fma(uy, uy, uz * uz));
    const double rs = rsqrt_nr(usq);                 // 1/|u|
    const double u = usq * rs;
    const double delta = (sqrtC * rs) * rsqrt_nr(u) * z;
    const double dd = fmin(fabs(delta), 1e150);
    const double d2 = dd * dd;
    const double inv = rcp_nr(1.0 + d2);
    const double sinT = 2.0 * copysign(dd, delta) * inv;
    const double omc = 2.0 * d2 * inv;
    rotate_pair(ax, ay, az, bx, by, bz, ux, uy, uz, u, sinT, omc, u2);
}

__device__ __forceinline__ void ta_update(double& ax, double& ay, double& az,
                                          double& bx, double& by, double& bz,
                                          double C, double u1, double u2)
{
    ta_update_z(ax, ay, az, bx, by, bz, C, ppnd16(u1), u2);
}

// ---------------------------------------------------------------- Nanbu (R20)
// s = 2 <delta^2>; A solves coth A - 1/A = exp(-s) (inverse Langevin: Newton
// from Jedynak's start; Taylor series of L and L' below A = 1/4; A = 1/(1 -
// exp(-s)) when that exceeds 40); 1 - cos(chi) = -log1p((1-u1) expm1(-2A)) / A.
__constant__ double kLangC[8] = {1.0 / 3.0, -1.0 / 45.0, 2.0 / 945.0, -1.0 / 4725.0, 2.0 / 93555.0,
                                 -1382.0 / 638512875.0, 4.0 / 18243225.0, -3617.0 / 162820783125.0};
__constant__ double kLangD[8] = {1.0 / 3.0, -1.0 / 15.0, 2.0 / 189.0, -1.0 / 675.0, 2.0 / 10395.0,
                                 -1382.0 / 58046625.0, 4.0 / 1403325.0, -3617.0 / 10854718875.0};

// L(A) = coth A - 1/A with L' (dL) and L'' (d2L)
__device__ __forceinline__ double langevin(double A, double* dL, double* d2L)
{
    if (A < 0.25) {
        const double z = A * A;
        double s = kLangC[7], d = kLangD[7], e = 14.0 * kLangD[7];
#pragma unroll
        for (int i = 6; i >= 0; --i) {
            s = s * z + kLangC[i];
            d = d * z + kLangD[i];
            if (i > 0) e = e * z + 2.0 * i * kLangD[i];     // L'' = A sum_{i>=1} 2i d_i A^{2(i-1)}
        }
        *dL = d;
        *d2L = A * e;
        return A * s;
    }
    // coth A = -(2 + em) / em and 1 / sinh^2 A = 4 (1 + em) / em^2 with em = expm1(-2A):
    // one transcendental instead of tanh + sinh (same values to rounding as the oracle's forms)
    const double em = expm1(-2.0 * A);
    const double ie = rcp_nr(em), ia = rcp_nr(A);
    const double cth = -(2.0 + em) * ie, csch2 = 4.0 * (1.0 + em) * ie * ie;
    *dL = ia * ia - csch2;
    *d2L = 2.0 * (cth * csch2 - ia * ia * ia);
    return cth - ia;
}

// Cheap cases of A(s): returns true and sets A (+inf: no scattering, s = 0; 0: isotropic;
// 1/(1 - e^-s) when that exceeds 40); false when the Newton solve is needed, x = e^-s set.
__device__ __forceinline__ bool nanbu_A_direct(double s, double& A, double& x)
{
    if (!(s > 0.0)) { A = __longlong_as_double(0x7FF0000000000000ll); return true; }
    // 1 - e^-s first: the direct A = 1/(1 - e^-s) (most pairs at small s) needs no exp
    const double omx = -expm1(-s);
    if (omx < 1.0 / 40.0) { A = 1.0 / omx; return true; }
    x = exp(-s);
    if (x <= 0.0) { A = 0.0; return true; }
    return false;
}

// Root of coth A - 1/A = x by Halley's method (cubic convergence: f = L - x, A -= f / (f' - f f''
// / (2 f'))) from Jedynak's (2015) inverse-Langevin approximation (<= 1.4% off): the first step
// leaves ~1e-5 relative, the second ~1e-15, so the loop stops after a step below 1e-5 A (the
// oracle iterates Newton to a 1e-15 step from Cohen's start: the same root to ~1e-15).
__device__ __forceinline__ double nanbu_newton(double x)
{
    double A = x * (3.0 - x * (2.6 - 0.7 * x)) / ((1.0 - x) * (1.0 + 0.1 * x));
    for (int it = 0; it < 30; ++it) {
        double dL, d2L;
        const double f = langevin(A, &dL, &d2L) - x;
        const double dA = f / (dL - 0.5 * f * d2L / dL);
        A -= dA;
        if (fabs(dA) <= 1e-5 * A) break;
    }
    return A;
}

// returns A; +inf means "no scattering" (s = 0), 0 means isotropic
__device__ __forceinline__ double nanbu_A(double s)
{
    double A, x;
    return nanbu_A_direct(s, A, x) ? A : nanbu_newton(x);
}

// s = 2 <delta^2> = 2 C / |u|^3 of a pair (u = v_a - v_b); 0 for u = 0 (no scattering)
__device__ __forceinline__ double nanbu_s(double ax, double ay, double az, double bx, double by, double bz, double C)
{
    const double ux = ax - bx, uy = ay - by, uz = az - bz;
    if (ux == 0.0 && uy == 0.0 && uz == 0.0) return 0.0;
    const double usq = fma(ux, ux, fma(uy, uy, uz * uz));
    const double rs = rsqrt_nr(usq);                 // 1/|u|: 2C/|u|^3 without a sqrt and a divide
    return 2.0 * C * (rs * rs) * rs;
}

// the Nanbu rotation for a given A (R20)
__device__ __forceinline__ void nanbu_apply(double& ax, double& ay, double& az, double& bx, double& by, double& bz,
                                            double A, double u1, double u2)
{
    const double ux = ax - bx, uy = ay - by, uz = az - bz;
    if (ux == 0.0 && uy == 0.0 && uz == 0.0) return;
    if (isinf(A)) return;
    const double usq = fma(ux, ux, fma(uy, uy, uz * uz));
    const double u = usq * rsqrt_nr(usq);
    // 1 - cos chi = -ln(u1 + (1-u1) e^{-2A}) / A = -log1p((1-u1) expm1(-2A)) / A (no cancellation);
    // expm1(-2A) is -1 to double precision once 2A > 40 (e^-40 < 2^-57), so it is skipped there
    const double em = (A > 20.0) ? -1.0 : expm1(-2.0 * A);
    double omc = (A == 0.0) ? 2.0 - 2.0 * u1 : -log1p((1.0 - u1) * em) / A;
    omc = fmin(fmax(omc, 0.0), 2.0);
    const double sinT = sqrt(omc * (2.0 - omc));
    rotate_pair(ax, ay, az, bx, by, bz, ux, uy, uz, u, sinT, omc, u2);
}

__device__ __forceinline__ void nanbu_update(double& ax, double& ay, double& az, double& bx, double& by, double& bz,
                                             double C, double u1, double u2)
{
    nanbu_apply(ax, ay, az, bx, by, bz, nanbu_A(nanbu_s(ax, ay, az, bx, by, bz, C)), u1, u2);
}

constexpr uint32_t kOddTriplet = 1u;   // CC_ODD_TRIPLET
constexpr uint32_t kNanbu = 2u;        // CC_NANBU

// one binary collision of the selected model (u1 uniform)
__device__ __forceinline__ void collide_model(double& ax, double& ay, double& az, double& bx, double& by, double& bz,
                                              double C, double u1, double u2, uint32_t flags)
{
    if (flags & kNanbu) nanbu_update(ax, ay, az, bx, by, bz, C, u1, u2);
    else ta_update(ax, ay, az, bx, by, bz, C, u1, u2);
}

}  // namespace cc
