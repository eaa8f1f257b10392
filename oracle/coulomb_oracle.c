/*
 * coulomb_oracle.c — CPU ORACLE for the electron–electron Coulomb collision
 * operator (step S1 "DSMC-Coul") of arXiv 2508.06771.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2508_06771_b200/) never links, imports or calls it,
 * and this file shares no source, header, table or generator with the CUDA
 * path: every constant below is typed here from its published definition.
 *
 * Plain, slow, obviously correct: fp64 arithmetic (the paper runs "All runs
 * are in double precision", §6), one loop per step of the paper's
 * Table 5 ("Coulombic Collision Steps"), no blocking, no fusion.
 * Cells are independent ("we only consider collisions between two
 * particles in the same grid cell"), so the per-cell collision loop is an
 * OpenMP loop over cells; results do not depend on the thread count.
 *
 * Citation key: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n;
 * Rk = reading k of DESIGN.md §3 (where the paper is silent or garbled).
 * External algorithms (not printed in the paper, cited by it or by DESIGN):
 *   Philox4x32-10  Salmon et al., "Parallel random numbers: as easy as 1,2,3"
 *                  (SC'11) — reading R3.
 *   AS241 PPND16   Wichura, Applied Statistics 37(3):477-484 (1988) — R4.
 *   TA77           Takizuka & Abe, J. Comput. Phys. 25:205 (1977), the method
 *                  the paper cites at P:324 (\cite{TAoriginal}) — R5, R8, R9.
 *   fmix32         MurmurHash3 finaliser (Appleby) — used by the keyed
 *                  permutation of R1.
 *
 * Pins (tests/test_oracle_*.py): Philox KAT vectors; U-map closed forms;
 * AS241 vs CPython statistics.NormalDist (an independent implementation of
 * AS241) and scipy.special.ndtri (a different algorithm); permutation
 * bijectivity by brute force and pairing uniformity by chi^2; stable order vs
 * numpy argsort(kind="stable"); TA update vs an independent orthonormal-frame
 * rotation, conservation and special cases; moments with dyadic data vs exact
 * sums; physics: Maxwellian invariance and the NRL anisotropy relaxation rate.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_OK 0
#define OR_EINVAL (-1)
#define OR_ECELL (-4)

/* ------------------------------------------------------------------------ */
/* R3: Philox4x32-10 (Salmon et al. 2011).  CCS4 "Generate two random numbers
 * for each collision pair" is realised by a counter-based
 * generator instead of a pre-generated array (SPEC's Rng.draw contract,
 * S:36-40).  Multipliers and Weyl constants as published.                    */
static const uint32_t PHILOX_M0 = 0xD2511F53u;
static const uint32_t PHILOX_M1 = 0xCD9E8D57u;
static const uint32_t PHILOX_W0 = 0x9E3779B9u;
static const uint32_t PHILOX_W1 = 0xBB67AE85u;

void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4])
{
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += PHILOX_W0; k1 += PHILOX_W1; }     /* bump key */
        uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
        uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* R3: two 32-bit words -> a uniform on the open interval (0,1):
 * U(hi,lo) = (floor((2^32 hi + lo) / 2^12) + 1/2) * 2^-52, exact in fp64,
 * range [2^-53, 1 - 2^-53].                                                   */
double or_u01(uint32_t hi, uint32_t lo)
{
    uint64_t x = ((uint64_t)hi << 32) | (uint64_t)lo;
    uint64_t m = x >> 12;                                   /* 52 bits */
    return ((double)m + 0.5) * 0x1.0p-52;
}

/* Counter layout (R3): ctr = (slot, global cell G, step, purpose),
 * key = (seed mod 2^32, seed >> 32).  purpose 0 = pair randoms (CCS4),
 * purpose 1 = per-cell Feistel round keys (R1, N > 64), purpose 2 = per-slot
 * sort keys (R1, N <= 64).                                                    */
void or_pair_uniforms(uint32_t kpair, uint32_t G, uint32_t step, uint64_t seed,
                      double *u1, double *u2)
{
    uint32_t ctr[4] = { kpair, G, step, 0u };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint32_t x[4];
    or_philox4x32_10(ctr, key, x);
    *u1 = or_u01(x[0], x[1]);
    *u2 = or_u01(x[2], x[3]);
}

void or_cell_keys(uint32_t G, uint32_t step, uint64_t seed, uint32_t k[4])
{
    uint32_t ctr[4] = { 0u, G, step, 1u };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    or_philox4x32_10(ctr, key, k);
}

/* ------------------------------------------------------------------------ */
/* R4: AS241 PPND16, Wichura (1988): the inverse standard normal CDF used to
 * turn one uniform into the Gaussian deflection variable delta of TA77.
 * Coefficients as published (16-digit accuracy version).                     */
double or_ppnd16(double p)
{
    double q = p - 0.5;
    if (fabs(q) <= 0.425) {
        double r = 0.180625 - q * q;
        double num = (((((((2.5090809287301226727e+3 * r +
                            3.3430575583588128105e+4) * r +
                            6.7265770927008700853e+4) * r +
                            4.5921953931549871457e+4) * r +
                            1.3731693765509461125e+4) * r +
                            1.9715909503065514427e+3) * r +
                            1.3314166789178437745e+2) * r +
                            3.3871328727963666080e+0) * q;
        double den = (((((((5.2264952788528545610e+3 * r +
                            2.8729085735721942674e+4) * r +
                            3.9307895800092710610e+4) * r +
                            2.1213794301586595867e+4) * r +
                            5.3941960214247511077e+3) * r +
                            6.8718700749205790830e+2) * r +
                            4.2313330701600911252e+1) * r +
                            1.0);
        return num / den;
    }
    double r = (q < 0.0) ? p : 1.0 - p;
    r = sqrt(-log(r));
    double num, den;
    if (r <= 5.0) {
        r = r - 1.6;
        num = (((((((7.7454501427834140764e-4 * r +
                     2.2723844989269184583e-2) * r +
                     2.4178072517745061177e-1) * r +
                     1.2704582524523683826e+0) * r +
                     3.6478483247632046050e+0) * r +
                     5.7694972214606914055e+0) * r +
                     4.6303378461565452959e+0) * r +
                     1.4234371107496835773e+0);
        den = (((((((1.0507500716444168432e-9 * r +
                     5.4759380849953449460e-4) * r +
                     1.5198666563616457197e-2) * r +
                     1.4810397642748007459e-1) * r +
                     6.8976733498510000455e-1) * r +
                     1.6763848301838038494e+0) * r +
                     2.0531916266377588219e+0) * r +
                     1.0);
    } else {
        r = r - 5.0;
        num = (((((((2.0103343992922881327e-7 * r +
                     2.7115555687434875782e-5) * r +
                     1.2426609473880784386e-3) * r +
                     2.6532189526576123093e-2) * r +
                     2.9656057182850489123e-1) * r +
                     1.7848265399172913358e+0) * r +
                     5.4637849111641143699e+0) * r +
                     6.6579046435011037772e+0);
        den = (((((((2.0442631033899397856e-15 * r +
                     1.4215117583164458887e-7) * r +
                     1.8463183175100546818e-5) * r +
                     7.8686913114561325910e-4) * r +
                     1.4875361290850614852e-2) * r +
                     1.3692988092273580531e-1) * r +
                     5.9983220655588793769e-1) * r +
                     1.0);
    }
    double x = num / den;
    return (q < 0.0) ? -x : x;
}

/* ------------------------------------------------------------------------ */
/* R1: the random in-cell pairing.  The paper pairs adjacent entries of the
 * index array P ("Define partner pairs {l,l'} as (P[1],P[2]), ...")
 * whose in-cell order comes from a scheduling-dependent atomic scatter
 * (P:313).  Reading R1 makes that order an explicit, reproducible random
 * permutation pi_j of the cell's N = N_j stable slots, re-drawn every step:
 *
 *  N <= 64 ("sort by random key"): slot s draws the 32-bit key r_s = word
 *    (s mod 4) of Philox(ctr = (s div 4, G, step, 2), key = seed); pi lists
 *    the slots in increasing (r_s, s).  Uniform up to key ties (p < 2^-20).
 *
 *  N > 64 ("keyed Feistel + cycle walking"): b = ceil(log2 N), bL = b div 2,
 *    a = 2^bL, m = ceil(N / a).  On x = L + a R (L in [0,a), R in [0,m)) run
 *    8 rounds r = 0..7 with round key K_r = k[r mod 4] + (r div 4) * 0x9E3779B9
 *    (k = Philox(ctr = (0, G, step, 1), key = seed)):
 *      r even:  L <- L xor (fmix32(R xor K_r) mod a)
 *      r odd:   R <- (R + floor(fmix32(L xor K_r) * m / 2^32)) mod m
 *    Each round is invertible, so E is a bijection of [0, a m) ⊇ [0, N);
 *    pi(i) is the first of E(i), E(E(i)), ... that is < N (cycle walking).
 *
 * Both forms are bijections of [0, N); R1 records the uniformity
 * checks (chi^2 of pair co-occurrence, adjacent-partner rate) behind the
 * round count and the N <= 64 threshold.                                      */
uint32_t or_fmix32(uint32_t h)
{
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
}

#define OR_SMALL_CELL 64

/* E of the N > 64 form (one application, no walking). */
static uint32_t or_feistel_E(uint32_t x, uint32_t bL, uint32_t m, const uint32_t k[4])
{
    uint32_t a = 1u << bL;
    uint32_t L = x % a, R = x / a;
    for (uint32_t r = 0; r < 8; ++r) {
        uint32_t K = k[r % 4] + (r / 4) * 0x9E3779B9u;
        if (r % 2 == 0) {
            L = L ^ (or_fmix32(R ^ K) % a);
        } else {
            uint32_t t = (uint32_t)(((uint64_t)or_fmix32(L ^ K) * (uint64_t)m) >> 32);
            R = (R + t) % m;
        }
    }
    return L + a * R;
}

int64_t or_feistel_pi(int64_t i, int64_t N, const uint32_t k[4])
{
    uint32_t b = 0;
    while (((int64_t)1 << b) < N) ++b;            /* b = ceil(log2 N) */
    uint32_t bL = b / 2;
    uint32_t a = 1u << bL;
    uint32_t m = (uint32_t)((N + a - 1) / a);
    uint32_t x = (uint32_t)i;
    do {
        x = or_feistel_E(x, bL, m, k);
    } while ((int64_t)x >= N);                    /* cycle walking */
    return (int64_t)x;
}

void or_cell_keys(uint32_t G, uint32_t step, uint64_t seed, uint32_t k[4]);

/* The R1 construction over n items with a chosen key stream (used for the
 * whole cell in R1, and for the segment order sigma and the block
 * permutations tau_b of R1b below):
 *   n <= 64: item s draws word (s mod 4) of Philox(ctr = (sort_base + s div 4,
 *            G, step, sort_purpose)); pi lists the items by increasing (key, s);
 *   n > 64:  the 8-round keyed Feistel above with k = Philox(ctr = (feistel_ctr,
 *            G, step, feistel_purpose)).
 * R1 itself is sort_base = 0, sort_purpose = 2, feistel_ctr = 0, feistel_purpose = 1. */
static void or_r1_perm(int64_t n, uint32_t G, uint32_t step, uint64_t seed,
                       uint32_t sort_base, uint32_t sort_purpose,
                       uint32_t feistel_ctr, uint32_t feistel_purpose, int64_t *pi)
{
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    if (n <= 0) return;
    if (n <= OR_SMALL_CELL) {
        uint32_t r[OR_SMALL_CELL];
        for (int64_t s = 0; s < n; ++s) {
            uint32_t ctr[4] = { sort_base + (uint32_t)(s / 4), G, step, sort_purpose }, w[4];
            or_philox4x32_10(ctr, key, w);
            r[s] = w[s % 4];
        }
        for (int64_t s = 0; s < n; ++s) {           /* rank of item s */
            int64_t rank = 0;
            for (int64_t t = 0; t < n; ++t)
                if (r[t] < r[s] || (r[t] == r[s] && t < s)) ++rank;
            pi[rank] = s;
        }
        return;
    }
    uint32_t ctr[4] = { feistel_ctr, G, step, feistel_purpose }, k[4];
    or_philox4x32_10(ctr, key, k);
    for (int64_t q = 0; q < n; ++q) pi[q] = or_feistel_pi(q, n, k);
}

/* R1 (CC_CELL_UNIFORM): pi_j over the whole cell, pi[q] = stable slot (0..N-1)
 * at pair-order position q. */
void or_cell_perm_uniform(int64_t N, uint32_t G, uint32_t step, uint64_t seed, int64_t *pi)
{
    or_r1_perm(N, G, step, seed, 0u, 2u, 0u, 1u, pi);
}

/* R1b (the default pairing): blocked random pairing.  Cells of N <= OR_BLOCK
 * slots are one block and get R1 unchanged.  A larger cell's stable slots are
 * cut into S_f = floor(N / L) segments of L consecutive slots
 * [s L, s L + L) plus, if N mod L > 0, a tail segment [S_f L, N).  The full
 * segments are put in a random order sigma (the R1 construction over S_f items
 * with sort purpose 6 / Feistel purpose 5); the tail goes last.  Consecutive
 * groups of OR_BLOCK_SEGS segments of that sequence form the blocks
 * b = 0 .. ceil(S / OR_BLOCK_SEGS) - 1 (S = number of segments, tail included);
 * block b's slots, listed segment by segment in sequence order, are its
 * "block slots" u = 0 .. n_b - 1 (n_b = OR_BLOCK except for the last block).
 * Inside block b the R1 construction over n_b items with sort counters
 * (b OR_BLOCK / 4 + u div 4, purpose 2) and Feistel counter (b, purpose 1)
 * gives tau_b, and pair-order position q = b OR_BLOCK + r holds the slot of
 * block slot tau_b(r).  Pairs never straddle blocks (OR_BLOCK is even); an odd
 * cell's last block is odd and its last position N - 1 sits out (R2).
 * Every block is a uniformly random set of whole segments, so every step mixes
 * the cell across its blocks; a block fits one CTA's shared memory on the GPU
 * (R1b gives the reasons and the uniformity evidence).              */
#define OR_SEG 32
#define OR_BLOCK_SEGS 12
#define OR_BLOCK (OR_SEG * OR_BLOCK_SEGS)

void or_cell_perm(int64_t N, uint32_t G, uint32_t step, uint64_t seed, int64_t *pi)
{
    if (N <= 0) return;
    if (N <= OR_BLOCK) {
        or_cell_perm_uniform(N, G, step, seed, pi);
        return;
    }
    int64_t Sf = N / OR_SEG, tail = N - Sf * OR_SEG;
    int64_t S = Sf + (tail > 0 ? 1 : 0);
    int64_t *sigma = (int64_t *)malloc(sizeof(int64_t) * (size_t)Sf);
    or_r1_perm(Sf, G, step, seed, 0u, 6u, 0u, 5u, sigma);
    /* seq_start[p] = first stable slot of the segment at sequence position p */
    int64_t *seq_start = (int64_t *)malloc(sizeof(int64_t) * (size_t)S);
    for (int64_t p = 0; p < Sf; ++p) seq_start[p] = sigma[p] * OR_SEG;
    if (tail > 0) seq_start[Sf] = Sf * OR_SEG;
    int64_t nblocks = (S + OR_BLOCK_SEGS - 1) / OR_BLOCK_SEGS;
    int64_t *slot = (int64_t *)malloc(sizeof(int64_t) * OR_BLOCK);
    int64_t *tau = (int64_t *)malloc(sizeof(int64_t) * OR_BLOCK);
    for (int64_t b = 0; b < nblocks; ++b) {
        int64_t nb = 0;                                  /* block slots of block b */
        for (int64_t p = b * OR_BLOCK_SEGS; p < S && p < (b + 1) * OR_BLOCK_SEGS; ++p) {
            int64_t len = (p == Sf) ? tail : OR_SEG;
            for (int64_t i = 0; i < len; ++i) slot[nb++] = seq_start[p] + i;
        }
        or_r1_perm(nb, G, step, seed, (uint32_t)(b * (OR_BLOCK / 4)), 2u, (uint32_t)b, 1u, tau);
        for (int64_t r = 0; r < nb; ++r) pi[b * OR_BLOCK + r] = slot[tau[r]];
    }
    free(tau);
    free(slot);
    free(seq_start);
    free(sigma);
}

/* ------------------------------------------------------------------------ */
/* CCS1: N_j = |P_j| for every cell.  Dead particles carry
 * cell id -1 (R11; SPEC "dead <=> weight 0") and are not counted.
 * Returns OR_ECELL if an id lies outside [-1, M).                             */
int or_count(const int32_t *cell, int64_t n, int32_t M, int64_t *counts)
{
    for (int32_t j = 0; j < M; ++j) counts[j] = 0;
    for (int64_t l = 0; l < n; ++l) {
        int32_t c = cell[l];
        if (c == -1) continue;
        if (c < -1 || c >= M) return OR_ECELL;
        counts[c] += 1;
    }
    return OR_OK;
}

/* CCS2: write indices I_j = exclusive prefix sum over N_j.
 * off has M+1 entries; off[M] = L, the number of live particles.              */
void or_exclusive_scan(const int64_t *counts, int32_t M, int64_t *off)
{
    off[0] = 0;
    for (int32_t j = 0; j < M; ++j) off[j + 1] = off[j] + counts[j];
}

/* CCS3: build P by looping over the particles in order and
 * writing each index at its cell's cursor I_j, then I_j += 1.  Done
 * sequentially the loop is a stable counting sort (R1/R14): cell-major, input
 * order inside each cell.  Dead particles follow at [L, n) in input order.    */
void or_stable_order(const int32_t *cell, int64_t n, int32_t M,
                     const int64_t *off, int64_t *perm)
{
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * ((size_t)M + 1));
    for (int32_t j = 0; j < M; ++j) cursor[j] = off[j];
    int64_t dead = off[M];
    for (int64_t l = 0; l < n; ++l) {
        int32_t c = cell[l];
        if (c >= 0 && c < M) perm[cursor[c]++] = l;
        else perm[dead++] = l;
    }
    free(cursor);
}

/* ------------------------------------------------------------------------ */
/* R5/R6/R7: the per-cell TA77 variance constant (SI form of S:344):
 *   <delta^2> = e^4 n_j lnL dt / (8 pi eps0^2 m_r^2 |u|^3),  m_r = m/2,
 * with n_j = N_j w / V_j the cell's current electron density (R6).
 * Returns C_j = e^4 n_j lnL dt / (8 pi eps0^2 m_r^2), so <delta^2> = C_j/|u|^3.
 * A non-positive or NaN result means "no scattering" (C_j = 0).               */
double or_cell_constant(int64_t Nj, double weight, double volume, double lnL,
                        double dt, double mass, double charge, double eps0)
{
    double n_j = (double)Nj * weight / volume;
    double e2 = charge * charge;
    double m_r = 0.5 * mass;
    double C = e2 * e2 * n_j * lnL * dt / (8.0 * M_PI * eps0 * eps0 * m_r * m_r);
    return fmax(C, 0.0);
}

/* CCS5, TA77 binary collision of one pair with randoms u1, u2:
 *   u = v_a - v_b;  delta = sqrt(C/|u|^3) * Phi^-1(u1)  (tan(Theta/2) = delta)
 *   sin(Theta) = 2 delta/(1+delta^2),  1-cos(Theta) = 2 delta^2/(1+delta^2)
 *   phi = 2 pi u2
 *   Delta u (TA77 eq. for the rotated relative velocity), R9 for u_perp = 0,
 *   v_a += Delta u / 2,  v_b -= Delta u / 2          (equal masses, R8).
 * |u| = 0 exactly is a no-op.  For |delta| > 1 the algebraically
 * equal forms in t = 1/delta are used so that delta -> inf cannot give NaN.   */
void or_ta_pair(double va[3], double vb[3], double C, double u1, double u2)
{
    double ux = va[0] - vb[0];
    double uy = va[1] - vb[1];
    double uz = va[2] - vb[2];
    if (ux == 0.0 && uy == 0.0 && uz == 0.0) return;
    double usq = ux * ux + uy * uy + uz * uz;
    double u = sqrt(usq);
    double var = C / (usq * u);                      /* <delta^2> */
    double delta = sqrt(var) * or_ppnd16(u1);
    double sinT, omc;                                /* sin(Theta), 1-cos(Theta) */
    if (fabs(delta) > 1.0) {
        double t = 1.0 / delta;
        sinT = 2.0 * t / (1.0 + t * t);
        omc = 2.0 / (1.0 + t * t);
    } else {
        sinT = 2.0 * delta / (1.0 + delta * delta);
        omc = 2.0 * delta * delta / (1.0 + delta * delta);
    }
    double phi = 2.0 * M_PI * u2;
    double cphi = cos(phi), sphi = sin(phi);
    double dux, duy, duz;
    if (ux == 0.0 && uy == 0.0) {
        dux = u * sinT * cphi;
        duy = u * sinT * sphi;
        duz = -uz * omc;
    } else {
        double uperp = sqrt(ux * ux + uy * uy);
        dux = (ux / uperp) * uz * sinT * cphi - (uy / uperp) * u * sinT * sphi - ux * omc;
        duy = (uy / uperp) * uz * sinT * cphi + (ux / uperp) * u * sinT * sphi - uy * omc;
        duz = -uperp * sinT * cphi - uz * omc;
    }
    va[0] += 0.5 * dux; va[1] += 0.5 * duy; va[2] += 0.5 * duz;
    vb[0] -= 0.5 * dux; vb[1] -= 0.5 * duy; vb[2] -= 0.5 * duz;
}

/* ------------------------------------------------------------------------ */
/* NEXT row f1 — collision-model variants (R19-R21).                 */

/* R20: Nanbu (1997) cumulative small-angle scattering, the alternative the
 * paper names.  s = 2 <delta^2> = 2 C / |u|^3; A solves the inverse
 * Langevin equation coth(A) - 1/A = exp(-s) (Newton iteration from Cohen's
 * Pade start, A = 1/(1 - exp(-s)) where coth(A) = 1 in double precision);
 * cos(chi) = 1 + ln(U1 + (1 - U1) exp(-2A)) / A  (A = 0: cos(chi) = 2 U1 - 1),
 * evaluated as 1 - cos(chi) = -log1p((1 - U1) expm1(-2A)) / A.                */
/* Langevin function L(A) = coth A - 1/A and L'(A); Taylor series below
 * A = 1/4 (8 terms, truncation < 1e-17 relative) where the closed forms cancel. */
static const double OR_LANG_C[8] = { 1.0 / 3.0, -1.0 / 45.0, 2.0 / 945.0, -1.0 / 4725.0, 2.0 / 93555.0,
                                     -1382.0 / 638512875.0, 4.0 / 18243225.0, -3617.0 / 162820783125.0 };
static const double OR_LANGD_C[8] = { 1.0 / 3.0, -1.0 / 15.0, 2.0 / 189.0, -1.0 / 675.0, 2.0 / 10395.0,
                                      -1382.0 / 58046625.0, 4.0 / 1403325.0, -3617.0 / 10854718875.0 };

double or_langevin(double A)
{
    if (A < 0.25) {
        double z = A * A, s = 0.0;
        for (int i = 7; i >= 0; --i) s = s * z + OR_LANG_C[i];
        return A * s;
    }
    return 1.0 / tanh(A) - 1.0 / A;
}

double or_langevin_d(double A)
{
    if (A < 0.25) {
        double z = A * A, s = 0.0;
        for (int i = 7; i >= 0; --i) s = s * z + OR_LANGD_C[i];
        return s;
    }
    double sh = sinh(A);
    return 1.0 / (A * A) - 1.0 / (sh * sh);
}

double or_nanbu_A(double s)
{
    if (!(s > 0.0)) return INFINITY;                 /* no scattering */
    double x = exp(-s);                              /* <cos chi> */
    if (x <= 0.0) return 0.0;                        /* isotropic */
    double omx = -expm1(-s);                         /* 1 - x, accurately */
    if (omx < 1.0 / 40.0) return 1.0 / omx;          /* A > 40: coth A = 1 in double, L = 1 - 1/A */
    double A = x * (3.0 - x * x) / (1.0 - x * x);    /* Cohen's Pade start */
    for (int it = 0; it < 60; ++it) {
        double dA = (or_langevin(A) - x) / or_langevin_d(A);
        A -= dA;
        if (fabs(dA) <= 1e-15 * A) break;
    }
    return A;
}

/* Rotation of u by polar angle chi (given as sin chi and 1 - cos chi) and
 * azimuth phi = 2 pi u2, written as TA77's component formula (R9), then the
 * equal-mass split v_a += Du/2, v_b -= Du/2. */
static void or_rotate_pair(double va[3], double vb[3], double sinT, double omc, double u2)
{
    double ux = va[0] - vb[0], uy = va[1] - vb[1], uz = va[2] - vb[2];
    double u = sqrt(ux * ux + uy * uy + uz * uz);
    double phi = 2.0 * M_PI * u2;
    double cphi = cos(phi), sphi = sin(phi);
    double dux, duy, duz;
    if (ux == 0.0 && uy == 0.0) {
        dux = u * sinT * cphi;
        duy = u * sinT * sphi;
        duz = -uz * omc;
    } else {
        double uperp = sqrt(ux * ux + uy * uy);
        dux = (ux / uperp) * uz * sinT * cphi - (uy / uperp) * u * sinT * sphi - ux * omc;
        duy = (uy / uperp) * uz * sinT * cphi + (ux / uperp) * u * sinT * sphi - uy * omc;
        duz = -uperp * sinT * cphi - uz * omc;
    }
    va[0] += 0.5 * dux; va[1] += 0.5 * duy; va[2] += 0.5 * duz;
    vb[0] -= 0.5 * dux; vb[1] -= 0.5 * duy; vb[2] -= 0.5 * duz;
}

void or_nanbu_pair(double va[3], double vb[3], double C, double u1, double u2)
{
    double ux = va[0] - vb[0], uy = va[1] - vb[1], uz = va[2] - vb[2];
    if (ux == 0.0 && uy == 0.0 && uz == 0.0) return;
    double usq = ux * ux + uy * uy + uz * uz;
    double s = 2.0 * C / (usq * sqrt(usq));
    double A = or_nanbu_A(s);
    double omc;                                      /* 1 - cos(chi) */
    if (isinf(A)) return;                            /* s = 0: no scattering */
    /* 1 - cos chi = -ln(u1 + (1-u1) e^{-2A}) / A, written as
     * -log1p((1-u1) expm1(-2A)) / A: the same number without the cancellation
     * of ln(1 - tiny) for small A (A -> 0 gives the isotropic 2(1-u1)). */
    if (A == 0.0) omc = 2.0 - 2.0 * u1;              /* cos chi = 2 u1 - 1 */
    else omc = -log1p((1.0 - u1) * expm1(-2.0 * A)) / A;
    if (omc > 2.0) omc = 2.0;
    if (omc < 0.0) omc = 0.0;
    double sinT = sqrt(omc * (2.0 - omc));
    or_rotate_pair(va, vb, sinT, omc, u2);
}

#define OR_ODD_TRIPLET 1u
#define OR_NANBU 2u
#define OR_PRESERVE_ORDER 4u
#define OR_CELL_UNIFORM 8u     /* R1 over the whole cell instead of R1b's blocks */

/* one binary collision of the selected model */
void or_collide_pair(double va[3], double vb[3], double C, double u1, double u2, uint32_t flags)
{
    if (flags & OR_NANBU) or_nanbu_pair(va, vb, C, u1, u2);
    else or_ta_pair(va, vb, C, u1, u2);
}

/* R19: TA77's rule for an odd number of particles: the last three of the
 * pair order, p1 = pi(N-3), p2 = pi(N-2), p3 = pi(N-1), collide pairwise
 * (p1,p2), (p2,p3), (p3,p1) in that order, each with half the time step
 * (C/2), randoms Philox(ctr = (q, G, step, 3)) for sub-collision q.            */
void or_triplet(double v1[3], double v2[3], double v3[3], double C, uint32_t G, uint32_t step,
                uint64_t seed, uint32_t flags)
{
    double *a[3] = { v1, v2, v3 }, *b[3] = { v2, v3, v1 };
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    for (uint32_t q = 0; q < 3; ++q) {
        uint32_t ctr[4] = { q, G, step, 3u }, x[4];
        or_philox4x32_10(ctr, key, x);
        or_collide_pair(a[q], b[q], 0.5 * C, or_u01(x[0], x[1]), or_u01(x[2], x[3]), flags);
    }
}

/* R21: NRL Plasma Formulary electron-electron Coulomb logarithm from lagged
 * moments: lnL = 23.5 - ln(n_e^1/2 T^-5/4) - sqrt(1e-5 + (ln T - 2)^2 / 16),
 * n_e in cm^-3, T = (T_x + T_y + T_z)/3 in eV; floored at 2;
 * empty or cold cells get the floor.                                         */
void or_coulomb_log(const double *moments, int32_t M, double *out)
{
    for (int32_t j = 0; j < M; ++j) {
        const double *m = moments + 7 * (int64_t)j;
        double n_cm = m[0] * 1e-6;
        double T = (m[4] + m[5] + m[6]) / 3.0;
        double l = 2.0;
        if (n_cm > 0.0 && T > 0.0) {
            double lt = log(T);
            l = 23.5 - (0.5 * log(n_cm) - 1.25 * lt) - sqrt(1e-5 + (lt - 2.0) * (lt - 2.0) / 16.0);
            if (!(l >= 2.0)) l = 2.0;
        }
        out[j] = l;
    }
}

/* ------------------------------------------------------------------------ */
/* P2C block reduction restricted to the operator's moments (P:330-342,
 * "V^j = sum_{x_l in omega_j} V_l"; T_e of P:336 with R13's constants):
 * out[j] = { n_j [m^-3], <v_x>, <v_y>, <v_z> [m/s], T_x, T_y, T_z [eV] } with
 * T_c = (m/e) * (1/N_j) sum (v_c - <v_c>)^2, two passes, long double sums.
 * v is slot-ordered [3][ldv]; the cell's particles are slots [off_j, off_j+1). */
void or_moments(const double *v, int64_t ldv, const int64_t *off, int32_t M,
                double weight, double volume, const double *volume_arr,
                double mass, double charge, double *out)
{
    for (int32_t j = 0; j < M; ++j) {
        int64_t a = off[j], b = off[j + 1], N = b - a;
        double *o = out + 7 * (int64_t)j;
        if (N <= 0) { for (int q = 0; q < 7; ++q) o[q] = 0.0; continue; }
        double V = volume_arr ? volume_arr[j] : volume;
        o[0] = (double)N * weight / V;
        for (int c = 0; c < 3; ++c) {
            long double s = 0.0L;
            for (int64_t p = a; p < b; ++p) s += (long double)v[c * ldv + p];
            long double mean = s / (long double)N;
            long double s2 = 0.0L;
            for (int64_t p = a; p < b; ++p) {
                long double d = (long double)v[c * ldv + p] - mean;
                s2 += d * d;
            }
            o[1 + c] = (double)mean;
            o[4 + c] = (double)((long double)mass / (long double)charge * s2 / (long double)N);
        }
    }
}

/* ------------------------------------------------------------------------ */
/* The whole operator, one call = one step S1 (Table 2; Table 5):
 * CCS1 count -> CCS2 scan -> CCS3 stable order -> R1 pairs -> CCS4 randoms ->
 * CCS5 TA update -> moments and diagnostics.
 *
 * Output order (R14): cell-sorted; inside cell j the particles appear in pair
 * order: position off_j + 2k and off_j + 2k + 1 hold pair k's first and second
 * member, (P[pi(2k)], P[pi(2k+1)]); if N_j is odd position off_j + N_j - 1
 * holds the particle that sits out (R2).  Dead particles follow at [L, n) in
 * input order.  perm_out[p] = input index of the particle at position p;
 * cell_out[p] = its cell (-1 for dead).  pair_slots (optional) receives for
 * every pair (cell-major, k-minor) the two stable slots off_j + pi(2k),
 * off_j + pi(2k+1).
 *
 * diag[16]: 0 live L, 1 dead, 2 pairs, 3 cells with odd N_j,
 *           4-6 sum v before, 7 sum |v|^2 before,
 *           8-10 sum v after, 11 sum |v|^2 after, 12-15 zero.                  */
int or_coulomb_collide(const double *v_in, int64_t ldv, const int32_t *cell_in,
                       double *v_out, int32_t *cell_out, int64_t *perm_out,
                       int64_t n, int32_t M, uint32_t cell_base,
                       double dt, double mass, double charge, double eps0,
                       double weight, double volume, const double *volume_arr,
                       double lnL, const double *lnL_arr,
                       uint64_t seed, uint64_t step, uint32_t flags,
                       double *moments_out, double *diag_out, int64_t *pair_slots)
{
    if (n < 0 || M < 1 || ldv < n || !(dt > 0.0)) return OR_EINVAL;
    if (step >= ((uint64_t)1 << 32)) return OR_EINVAL;

    int64_t *counts = (int64_t *)calloc((size_t)M, sizeof(int64_t));
    int64_t *off = (int64_t *)calloc((size_t)M + 1, sizeof(int64_t));
    int64_t *P = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *pair_off = (int64_t *)calloc((size_t)M + 1, sizeof(int64_t));

    /* CCS1 */
    int rc = or_count(cell_in, n, M, counts);
    if (rc != OR_OK) { free(counts); free(off); free(P); free(pair_off); return rc; }
    /* CCS2 */
    or_exclusive_scan(counts, M, off);
    int64_t L = off[M];
    /* CCS3 */
    or_stable_order(cell_in, n, M, off, P);

    for (int32_t j = 0; j < M; ++j) pair_off[j + 1] = pair_off[j] + counts[j] / 2;

    /* Per-cell work: R1 pairing, CCS4 randoms, CCS5 TA update, output in
     * pair order.  Cells are independent. */
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t j = 0; j < M; ++j) {
        int64_t N = counts[j], o = off[j];
        if (N == 0) continue;
        uint32_t G = cell_base + (uint32_t)j;
        int64_t *pi = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
        if (flags & OR_CELL_UNIFORM) or_cell_perm_uniform(N, G, (uint32_t)step, seed, pi);
        else or_cell_perm(N, G, (uint32_t)step, seed, pi);
        double C = or_cell_constant(N, weight, volume_arr ? volume_arr[j] : volume,
                                    lnL_arr ? lnL_arr[j] : lnL, dt, mass, charge, eps0);
        int triplet = (flags & OR_ODD_TRIPLET) && N >= 3 && (N % 2 == 1);
        int64_t npairs = triplet ? (N - 3) / 2 : N / 2;
        for (int64_t k = 0; k < npairs; ++k) {
            int64_t sa = o + pi[2 * k];
            int64_t sb = o + pi[2 * k + 1];
            int64_t la = P[sa], lb = P[sb];
            double va[3] = { v_in[la], v_in[ldv + la], v_in[2 * ldv + la] };
            double vb[3] = { v_in[lb], v_in[ldv + lb], v_in[2 * ldv + lb] };
            double u1, u2;
            or_pair_uniforms((uint32_t)k, G, (uint32_t)step, seed, &u1, &u2);
            or_collide_pair(va, vb, C, u1, u2, flags);
            int64_t pa = o + 2 * k, pb = o + 2 * k + 1;
            for (int c = 0; c < 3; ++c) { v_out[c * ldv + pa] = va[c]; v_out[c * ldv + pb] = vb[c]; }
            perm_out[pa] = la; perm_out[pb] = lb;
            cell_out[pa] = j; cell_out[pb] = j;
            if (pair_slots) {                       /* pi-pairs (default-mode layout) */
                int64_t g = pair_off[j] + k;
                pair_slots[2 * g] = sa;
                pair_slots[2 * g + 1] = sb;
            }
        }
        if (triplet) {                                  /* R19: TA77 triplet */
            int64_t l3[3];
            double v3[3][3];
            for (int q = 0; q < 3; ++q) {
                l3[q] = P[o + pi[N - 3 + q]];
                for (int c = 0; c < 3; ++c) v3[q][c] = v_in[c * ldv + l3[q]];
            }
            or_triplet(v3[0], v3[1], v3[2], C, G, (uint32_t)step, seed, flags);
            for (int q = 0; q < 3; ++q) {
                int64_t p = o + N - 3 + q;
                for (int c = 0; c < 3; ++c) v_out[c * ldv + p] = v3[q][c];
                perm_out[p] = l3[q]; cell_out[p] = j;
            }
        } else if (N % 2 == 1) {                        /* R2: one sits out */
            int64_t s = o + pi[N - 1];
            int64_t l = P[s], p = o + N - 1;
            for (int c = 0; c < 3; ++c) v_out[c * ldv + p] = v_in[c * ldv + l];
            perm_out[p] = l; cell_out[p] = j;
        }
        free(pi);
    }
    /* dead particles: copied unchanged after the live ones, input order */
    for (int64_t p = L; p < n; ++p) {
        int64_t l = P[p];
        for (int c = 0; c < 3; ++c) v_out[c * ldv + p] = v_in[c * ldv + l];
        perm_out[p] = l; cell_out[p] = -1;
    }

    if (moments_out)
        or_moments(v_out, ldv, off, M, weight, volume, volume_arr, mass, charge, moments_out);

    if (diag_out) {
        long double sb[4] = { 0, 0, 0, 0 }, sa[4] = { 0, 0, 0, 0 };
        int64_t odd = 0;
        for (int32_t j = 0; j < M; ++j) odd += counts[j] % 2;
        for (int64_t l = 0; l < n; ++l) {
            if (cell_in[l] < 0) continue;
            long double e = 0.0L;
            for (int c = 0; c < 3; ++c) {
                long double x = v_in[c * ldv + l];
                sb[c] += x; e += x * x;
            }
            sb[3] += e;
        }
        for (int64_t p = 0; p < L; ++p) {
            long double e = 0.0L;
            for (int c = 0; c < 3; ++c) {
                long double x = v_out[c * ldv + p];
                sa[c] += x; e += x * x;
            }
            sa[3] += e;
        }
        for (int q = 0; q < 16; ++q) diag_out[q] = 0.0;
        diag_out[0] = (double)L;
        diag_out[1] = (double)(n - L);
        diag_out[2] = (double)pair_off[M];
        diag_out[3] = (double)odd;
        for (int q = 0; q < 4; ++q) { diag_out[4 + q] = (double)sb[q]; diag_out[8 + q] = (double)sa[q]; }
    }

    if (flags & OR_PRESERVE_ORDER) {
        /* O8 / SURVEY §8(b) CC_PRESERVE_ORDER: the same per-particle results, returned in
         * input order — the un-permute v_final[perm[p]] = v_out[p], cell likewise;
         * perm becomes the identity.  Moments and diagnostics above are unchanged. */
        double *tv = malloc(sizeof(double) * 3 * (size_t)(n > 0 ? n : 1));
        int32_t *tc = malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
        for (int64_t p = 0; p < n; ++p) {
            for (int c = 0; c < 3; ++c) tv[c * n + p] = v_out[c * ldv + p];
            tc[p] = cell_out[p];
        }
        for (int64_t p = 0; p < n; ++p) {
            const int64_t l = perm_out[p];
            for (int c = 0; c < 3; ++c) v_out[c * ldv + l] = tv[c * n + p];
            cell_out[l] = tc[p];
        }
        for (int64_t l = 0; l < n; ++l) perm_out[l] = l;
        free(tv);
        free(tc);
    }

    free(counts); free(off); free(P); free(pair_off);
    return OR_OK;
}

/* Thread count actually used by the OpenMP loop (for cpu_baseline "cores"). */
int or_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* NEXT f2: the kinetic push between two collision calls.
 * Table 2: Step S2b "E_l^c = -q grad phi(x_l^c)" (the cell-to-
 * particle field) and Step S2c "x_l^+ = x_l^c + delta v_l^c; v_l^c + delta
 * E_l^c" (DSMC-Push); SPEC push: "v' = v + dt (q/m) E;
 * x' = x + dt v'" with E the per-cell constant field retrieved by cell id
 * (S:207); boundary (Table 3 CS7): a particle leaving an
 * absorbing axis dies; cell assignment j = floor(x/dx).  Readings
 * R22-R24 of DESIGN.md §3: periodic axes wrap (add/subtract of L = n_a d_a;
 * beyond one period first the exact remainder fmod(x, L); a non-finite
 * position is absorbed), i_a = floor(x_a / d_a) clamped to n_a - 1 (x just below L
 * can divide to n_a), global cell = i_0 + n_0 (i_1 + n_1 i_2).
 *
 * Particle p (output order of the collision call): x_in row a < dims at
 * index perm[p] (perm NULL = p) -> x_out[a][p] (rows >= dims untouched);
 * v[c][p] updated in place;
 * cell[p]: in = LOCAL cell of the collision call (-1 dead), out = GLOBAL
 * cell after the push (-1 dead).  Dead particles keep x and v.
 * E: [3][ldE] rows x, y, z per LOCAL cell, or NULL (no field).             */
void or_push(const double *x_in, int64_t ldx_in, const int64_t *perm, double *x_out, int64_t ldx_out,
             double *v, int64_t ldv, int32_t *cell, int64_t n, int32_t dims, const int32_t nc[3],
             const double d[3], uint32_t periodic, const double *E, int64_t ldE, double q_over_m, double dt)
{
    const double kick = dt * q_over_m;
    for (int64_t p = 0; p < n; ++p) {
        const int64_t src = perm ? perm[p] : p;
        double x[3] = {0.0, 0.0, 0.0};
        for (int a = 0; a < dims; ++a) x[a] = x_in[a * ldx_in + src];
        const int32_t j = cell[p];
        if (j < 0) {                                      /* dead: unchanged */
            for (int a = 0; a < dims; ++a) x_out[a * ldx_out + p] = x[a];
            continue;
        }
        /* S2b + S2c kick: v' = v + dt (q/m) E_j */
        double vn[3];
        for (int c = 0; c < 3; ++c) {
            double e = E ? E[c * ldE + j] : 0.0;
            vn[c] = v[c * ldv + p] + kick * e;
            v[c * ldv + p] = vn[c];
        }
        /* S2c drift: x' = x + dt v', boundary, cell index */
        int alive = 1;
        int64_t G = 0, stride = 1;
        for (int a = 0; a < 3; ++a) {
            if (a < dims) {
                double xa = x[a] + dt * vn[a];
                const double L = (double)nc[a] * d[a];
                if (!isfinite(xa)) {
                    alive = 0;                  /* R23: a non-finite position is absorbed */
                } else if (periodic & (1u << a)) {
                    /* R23: more than one period away -> the exact remainder first, so the
                       wrap below is at most one add or subtract */
                    if (xa < -L || xa >= 2.0 * L) xa = fmod(xa, L);
                    while (xa < 0.0) xa = xa + L;
                    while (xa >= L) xa = xa - L;
                } else if (xa < 0.0 || xa >= L) {
                    alive = 0;
                }
                x[a] = xa;
                if (alive) {
                    int64_t i = (int64_t)floor(xa / d[a]);
                    if (i > nc[a] - 1) i = nc[a] - 1;
                    G += i * stride;
                }
            }
            stride *= nc[a];
            if (a < dims) x_out[a * ldx_out + p] = x[a];
        }
        cell[p] = alive ? (int32_t)G : -1;
    }
}

/* ------------------------------------------------------------------------ */
/* NEXT f3: three-body recombination C5, Table 4 RS0-RS5
 * (P:262-290), on the OUTPUT of a collision call (cell-sorted; inside a cell
 * the slots are in the step's random pair order, R14).  Readings R25-R28:
 *  RS0 (R25) the particle at position q of cell j (global id G) is a primary
 *      iff U(Philox(ctr = (q, G, step, 4), key = seed)) < prob[j] (SPEC S:289's
 *      per-particle probability, supplied per cell by the caller);
 *  RS1-RS3 (R26) the i-th primary of the cell (position order) is matched to
 *      the i-th non-primary ("catalyte", position order) for i < min(P_j,
 *      N_j - P_j): unique and cell-local by construction, and uniform because
 *      the position order is a fresh random permutation every step; primaries
 *      beyond the catalyte count are starved and left unchanged;
 *  RS4 (R27) the catalyte keeps its direction and takes the primary's kinetic
 *      energy plus the binding energy e_b: |v_c'|^2 = |v_c|^2 + |v_p|^2 + 2 e_b/m
 *      (SPEC S:321); a catalyte at rest takes the primary's direction (+x if
 *      that is zero too);
 *  RS5 (R28) the primary dies (cell -1, velocity kept).
 * cell: [n] in place; v [3][ldv] in place; stats {recombined, starved, primaries}. */
static double or_rc_norm2(double x, double y, double z) { return x * x + y * y + z * z; }

void or_recombine(double *v, int64_t ldv, int32_t *cell, int64_t n, int32_t M, uint32_t cell_base,
                  const double *prob, double eps_bind, double mass, uint64_t seed, uint64_t step, int64_t stats[3])
{
    stats[0] = stats[1] = stats[2] = 0;
    const double vb2 = 2.0 * eps_bind / mass;
    int64_t *prim = malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *cat = malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t lo = 0;
    for (int32_t j = 0; j < M; ++j) {
        int64_t hi = lo;
        while (hi < n && cell[hi] == j) ++hi;         /* cell-sorted input */
        const int64_t N = hi - lo;
        const uint32_t G = cell_base + (uint32_t)j;
        int64_t np = 0, nc = 0;
        for (int64_t q = 0; q < N; ++q) {             /* RS0 */
            uint32_t ctr[4] = {(uint32_t)q, G, (uint32_t)step, 4u};
            uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
            uint32_t x[4];
            or_philox4x32_10(ctr, key, x);
            if (or_u01(x[0], x[1]) < prob[j]) prim[np++] = lo + q;
            else cat[nc++] = lo + q;
        }
        const int64_t m = np < nc ? np : nc;
        for (int64_t i = 0; i < m; ++i) {             /* RS3-RS5 */
            const int64_t a = prim[i], c = cat[i];
            const double px = v[a], py = v[ldv + a], pz = v[2 * ldv + a];
            const double cx = v[c], cy = v[ldv + c], cz = v[2 * ldv + c];
            const double c2 = or_rc_norm2(cx, cy, cz), p2 = or_rc_norm2(px, py, pz);
            const double t2 = c2 + p2 + vb2;          /* |v_c'|^2 */
            double ux = cx, uy = cy, uz = cz, s2 = c2;  /* direction source */
            if (c2 == 0.0) { ux = px; uy = py; uz = pz; s2 = p2; }
            if (s2 == 0.0) { ux = 1.0; uy = 0.0; uz = 0.0; s2 = 1.0; }
            const double f = sqrt(t2 / s2);
            v[c] = ux * f; v[ldv + c] = uy * f; v[2 * ldv + c] = uz * f;
            cell[a] = -1;
        }
        stats[0] += m;
        stats[1] += np - m;
        stats[2] += np;
        lo = hi;
    }
    free(prim);
    free(cat);
}

/* Thread count of the OpenMP cell loop (bench.py's single-thread oracle timings). */
void or_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
