/*
 * coulomb.h — C ABI of the B200-native electron–electron Coulomb collision
 * operator: step S1 ("DSMC-Coul") of arXiv 2508.06771's operator-split PIC
 * scheme (Table 2; Table 5 "Coulombic Collision Steps",
 * P:299-322; §4.4).
 *
 * One call of coulomb_collide() = one step of S1 on a set of electrons binned
 * in cells:  CCS1 count -> CCS2 prefix sum -> CCS3 stable bin -> random
 * in-cell pairing (readings R1b / R1) -> CCS4 two randoms per pair ->
 * CCS5 Takizuka–Abe binary collision -> per-cell moments
 * (the P2C block reduction of §4.5) and global diagnostics.
 * Everything runs in fp64 ("All runs are in double precision").
 *
 * Conventions
 *  - Every pointer argument is a DEVICE pointer owned by the caller (e.g. the
 *    storage of a torch tensor) unless documented as HOST.  The library never
 *    allocates, frees or synchronises on the compute path; all work is
 *    enqueued on `stream` (a cudaStream_t passed as void*; NULL = legacy
 *    default stream).  Outputs are valid when the stream reaches that point.
 *  - Velocities are structure-of-arrays fp64: v[c * ldv + i], c = 0,1,2
 *    (x, y, z), i < n <= ldv.  Base pointers must be 16-byte aligned.
 *  - cell ids are int32: 0 <= id < cells for live particles, -1 for dead
 *    particles (SPEC "dead <=> weight 0"; reading R11).
 *  - Return codes: CC_OK or a negative CC_E* code; no exceptions cross the ABI.
 *    Host-side argument errors are reported before anything is enqueued.
 *    Invalid cell ids are detected on the device: such particles are treated
 *    as dead and a flag is raised in the workspace, returned as CC_ECELL by
 *    cc_device_status().
 *  - Reentrant for distinct workspaces; no global mutable state.
 */
#ifndef B200_COULOMB_H
#define B200_COULOMB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CC_OK 0
#define CC_EINVAL (-1)      /* bad argument (null/misaligned pointer, n<0, cells<1, dt<=0, step>=2^32, aliasing) */
#define CC_EWORKSPACE (-2)  /* workspace null, misaligned (256 B) or smaller than cc_workspace_bytes() */
#define CC_ECUDA (-3)       /* a CUDA launch failed */
#define CC_ECELL (-4)       /* (device-detected) a cell id outside [-1, cells) was seen */
#define CC_ECOUNT (-5)      /* n >= 2^31 or cells > CC_MAX_CELLS */
#define CC_ENCCL (-6)       /* reserved for the multi-GPU layer */

/* cc_params.flags: collision-model variants (DESIGN R19-R20)
 *  CC_ODD_TRIPLET  odd N_j >= 3: the last three particles of the pair order collide
 *                  pairwise (1,2), (2,3), (3,1) with half the time step (TA77's rule)
 *                  instead of one particle sitting out (R2).  Randoms: Philox(ctr =
 *                  (q, G, step, 3)) for sub-collision q.
 *  CC_NANBU        Nanbu (1997) cumulative scattering angle (the alternative the paper
 *                  names) instead of TA77's Gaussian tan(Theta/2): s = 2<delta^2>,
 *                  coth A - 1/A = exp(-s), cos chi = 1 + ln(u1 + (1-u1) e^{-2A})/A.      */
#define CC_ODD_TRIPLET 1u
#define CC_NANBU 2u
/* Output order:
 *  CC_PRESERVE_ORDER  outputs in INPUT order instead of the default cell-sorted pair
 *                     order: v_out[:, i], cell_out[i] are input particle i's post-collision
 *                     velocity and (validated) cell, -1 if dead or invalid; perm_out, if
 *                     given, is the identity.  Same per-particle values, moments and
 *                     diagnostics; the stores scatter to the input positions (no paired
 *                     16-byte stores).  Lets a caller keep its own particle order (and
 *                     skip copying cell_out / perm_out back, see coulomb_collide_host).  */
#define CC_PRESERVE_ORDER 4u
/* In-cell pairing (readings R1 / R1b; P:313-314 pairs adjacent entries of an
 * atomically built index list and draws no permutation):
 *  default           R1b, blocked pairing: a cell of N <= 384 slots is permuted as a whole
 *                    (R1); a larger cell's stable slots are cut into 32-slot segments, the
 *                    full segments are put in a keyed random order (the tail segment last),
 *                    every 12 consecutive segments of that order form a block of <= 384
 *                    slots, and R1 is applied inside each block; pairs never straddle blocks.
 *  CC_CELL_UNIFORM   R1 over the whole cell (one keyed permutation of all N_j slots).      */
#define CC_CELL_UNIFORM 8u

#define CC_MAX_CELLS 32768  /* binning keeps per-warp cell counters in shared memory */
#define CC_DIAG_LEN 16
#define CC_MOMENTS_LEN 7

/* Regular grid of the push (HOST struct).  Global cell id of a position:
 * i_a = floor(x_a / d[a]) clamped to n[a]-1, G = i_0 + n[0] (i_1 + n[1] i_2)
 * ("j = floor(x/dx)"; readings R22-R24).                         */
typedef struct cc_grid {
    int32_t dims;            /* 1, 2 or 3 position components in use (x, y, z) */
    int32_t n[3];            /* global cells per axis; n[a] = 1 for a >= dims   */
    double d[3];             /* cell size per axis [m]                          */
    uint32_t periodic;       /* bit a set: axis a periodic (wraps by L_a = n[a] d[a]);
                                clear: absorbing, a particle leaving [0, L_a) dies
                                (Table 3 CS7)                    */
} cc_grid;

/* NEXT f2: the push fused into coulomb_collide's output stage (HOST struct; see
 * cc_params.push).  x_in [3][ldx_in] DEVICE positions in INPUT order (row a of input
 * particle l at x_in[a*ldx_in + l]); x_out [3][ldx_out] DEVICE, rows a < dims written in
 * OUTPUT order; E DEVICE [3][ldE] per local cell or NULL.  Must not alias.           */
typedef struct cc_push_params {
    const cc_grid *grid;          /* HOST                                                    */
    const double *E;
    int64_t ldE;
    double q_over_m;
    const double *x_in;
    int64_t ldx_in;
    double *x_out;
    int64_t ldx_out;
} cc_push_params;

/* Physical parameters (HOST struct).  Defaults from cc_default_params():
 * CODATA 2018 electron mass/charge and eps0, weight 1, cell_volume 1,
 * ln_lambda 10 (reading R7), no per-cell arrays, flags 0.                     */
typedef struct cc_params {
    double mass;                  /* kg, particle mass m (m_r = m/2 for e-e, R5)          */
    double charge;                /* C, |q|                                                */
    double eps0;                  /* F/m                                                   */
    double weight;                /* physical electrons per macro-particle (uniform) */
    double cell_volume;           /* m^3, used when cell_volume_arr == NULL                */
    const double *cell_volume_arr;/* DEVICE [cells] or NULL                                */
    double ln_lambda;             /* Coulomb logarithm, used when ln_lambda_arr == NULL    */
    const double *ln_lambda_arr;  /* DEVICE [cells] or NULL                                */
    uint32_t flags;               /* 0 (TA77, odd sitter) or CC_ODD_TRIPLET | CC_NANBU,
                                     optionally | CC_PRESERVE_ORDER                          */
    const cc_push_params *push;   /* HOST or NULL: when set, every output particle is also pushed
                                     (S2b + S2c with this call's dt, exactly cc_push's arithmetic):
                                     v_out = kicked velocity, x_out = drifted position, cell_out =
                                     post-push GLOBAL cell (-1 if absorbed); moments and diagnostics
                                     stay those of the post-collision, pre-kick particles.  Equal,
                                     bit for bit, to coulomb_collide then cc_push(x_in, perm_out, ...),
                                     without re-reading v, cell and perm.  Not with CC_PRESERVE_ORDER. */
    const uint32_t *step_dev;     /* DEVICE uint32 or NULL: when set, the effective step is
                                     (step + *step_dev) mod 2^32, read on the device, so a
                                     captured CUDA graph replays with advancing randoms
                                     (cc_step_advance); NEXT f2 subcycled loop.           */
    void *const *stage_events;    /* HOST array of CC_NUM_STAGES+1 cudaEvent_t, or NULL.
                                     When set, coulomb_collide records event i on `stream`
                                     before stage i and event CC_NUM_STAGES after the last
                                     (stages: 0 count, 1 scan, 2 scatter, 3 collide,
                                     4 finalize) — used by bench.py for per-kernel timing. */
} cc_params;

#define CC_NUM_STAGES 5

void cc_default_params(cc_params *p);                         /* HOST */

/* Bytes of device workspace a call with (n, cells) needs (HOST function).
 * The workspace must be 256-byte aligned; its contents need no
 * initialisation and are scratch between calls (except the error flag read
 * by cc_device_status).                                                       */
size_t cc_workspace_bytes(int64_t n, int32_t cells);

/* One step of the Coulomb collision operator (Table 5, CCS1-CCS5).
 *
 *  v_in      [3][ldv] fp64, read only.                 cell_in [n] int32, read only.
 *  v_out     [3][ldv] fp64, written for all n slots.   cell_out [n] int32, written.
 *  perm_out  [n] int32 or NULL: input index of the particle at each output slot.
 *  Output order (reading R14): cell-major; inside cell j (slots
 *  [off_j, off_j + N_j)) the particles are in PAIR order — slots off_j+2k and
 *  off_j+2k+1 hold pair k's first and second member, and for odd N_j slot
 *  off_j+N_j-1 holds the particle that sat out (R2).  With the default R1b
 *  pairing, pairs k in [192 b, 192 b + 192) are the pairs of block b.
 *  Binning: the call picks its binning mode on the device from
 *  the input's order — sorted input is read in place, nearly sorted input is
 *  binned by 4-byte indices (then read through them), randomly ordered input is
 *  moved as 32-byte records; the results do not depend on the mode.  Dead particles follow at
 *  [L, n) in input order (L = number of live particles).  v_out/cell_out/
 *  perm_out must not alias the inputs.
 *  cells     number of LOCAL cells M (1 <= M <= CC_MAX_CELLS).
 *  cell_base global id of local cell 0 (multi-GPU cell-range sharding); the
 *            random streams are keyed by the GLOBAL cell id, so a shard's result
 *            equals the single-GPU result on the same particles.
 *  dt        s, > 0.   params: HOST pointer (NULL = defaults).
 *  seed      Philox key (64 bits).  step: < 2^32, Philox counter word (R3).
 *  moments_out [cells][7] or NULL: {n_j [m^-3], <v_x>, <v_y>, <v_z> [m/s],
 *            T_x, T_y, T_z [eV]} of the post-collision particles (R13).
 *  diag_out  [16] or NULL: 0 live L, 1 dead, 2 pairs, 3 cells with odd N_j,
 *            4-6 sum v before, 7 sum |v|^2 before, 8-10 sum v after,
 *            11 sum |v|^2 after, 12-15 zero.  Sums are deterministic (fixed
 *            reduction order): two calls with equal inputs give equal bytes.
 *  flags (params): CC_ODD_TRIPLET, CC_NANBU, CC_PRESERVE_ORDER, CC_CELL_UNIFORM;
 *            any other bit is CC_EINVAL.
 *  workspace >= cc_workspace_bytes(n, cells) bytes, 256-byte aligned.        */
int coulomb_collide(const double *v_in, int64_t ldv, const int32_t *cell_in,
                    double *v_out, int32_t *cell_out, int32_t *perm_out,
                    int64_t n, int32_t cells, uint32_t cell_base,
                    double dt, const cc_params *params,
                    uint64_t seed, uint64_t step,
                    double *moments_out, double *diag_out,
                    void *workspace, size_t workspace_bytes, void *stream);

/* End-to-end entry with HOST buffers: the same operator as coulomb_collide, with
 * the host->device copies of the inputs and the device->host copies of the
 * results enqueued on `stream` around it (asynchronous: results are valid after
 * the stream is synchronised; pinned host memory gives full PCIe rate and lets
 * the copies overlap other streams).
 *  h_v_in [3][ldv], h_cell_in [n]       HOST inputs (read).
 *  h_v_out [3][ldv]                     HOST output; h_cell_out [n], h_perm_out [n],
 *                                       h_moments_out [cells][7], h_diag_out [16] HOST or
 *                                       NULL (not copied back).  With CC_PRESERVE_ORDER the
 *                                       velocities come back in the caller's own order, so
 *                                       cell ids and perm need not be copied at all.
 *  dev_buffer  DEVICE scratch of >= cc_host_buffer_bytes(n, cells) bytes, 256-byte
 *              aligned, holding device copies of the inputs/outputs and the
 *              workspace; one per call in flight.
 * Consecutive calls on two streams with two dev_buffers overlap one call's
 * device->host copies with the next call's host->device copies (PCIe is full
 * duplex); bench.py's e2e does exactly that.  Errors as coulomb_collide.    */
size_t cc_host_buffer_bytes(int64_t n, int32_t cells);                    /* HOST */
int coulomb_collide_host(const double *h_v_in, int64_t ldv, const int32_t *h_cell_in,
                         double *h_v_out, int32_t *h_cell_out, int32_t *h_perm_out,
                         int64_t n, int32_t cells, uint32_t cell_base, double dt,
                         const cc_params *params, uint64_t seed, uint64_t step,
                         double *h_moments_out, double *h_diag_out,
                         void *dev_buffer, size_t dev_bytes, void *stream);

/* Synchronises `stream` and returns CC_ECELL if a previous call on this
 * workspace saw an invalid cell id (the flag is then cleared), CC_ECUDA on a
 * CUDA error, else CC_OK.                                                     */
int cc_device_status(void *workspace, void *stream);

const char *cc_strerror(int code);                            /* HOST */

/* ---- test hooks: the same kernels as coulomb_collide, partial pipelines ---- */

/* CCS1-CCS3: stable counting sort by cell.  perm_out[s] = input
 * index at stable slot s (cell-major, input order inside a cell, dead last in
 * input order); off_out [cells+1] = exclusive prefix sum of N_j (CCS2).      */
int cc_bin(const int32_t *cell_in, int64_t n, int32_t cells,
           int32_t *perm_out, int32_t *off_out,
           void *workspace, size_t workspace_bytes, void *stream);

/* Readings R1b / R1: for every pair of every cell, the two STABLE slots
 * (off_j + pi_j(2k), off_j + pi_j(2k+1)), cell-major, k-minor, written to
 * pair_slots_out[2*g], [2*g+1]; g runs over sum_j floor(N_j/2) pairs, at most
 * max_pairs are written.  off: DEVICE [cells+1] as produced by cc_bin.  flags: 0
 * (the default blocked pairing R1b) or CC_CELL_UNIFORM (R1); anything else is
 * CC_EINVAL.  pi_j is computed from its definition slot by slot (a test hook).   */
int cc_pairs(const int32_t *off, int32_t cells, uint32_t cell_base,
             uint64_t seed, uint64_t step, uint32_t flags,
             int32_t *pair_slots_out, int64_t max_pairs, void *stream);

/* R3: Philox4x32-10 of m counters ctr4 [m][4] with key (seed lo, seed hi). */
int cc_philox(const uint32_t *ctr4, uint64_t seed, uint32_t *out4, int64_t m, void *stream);

/* R4: AS241 PPND16 inverse normal CDF of m values. */
int cc_ppnd16(const double *u, double *z, int64_t m, void *stream);

/* CCS5: TA77 update of m explicit pairs, in place.  va, vb
 * [3][m] SoA; C [m] per-pair variance constant (<delta^2> = C/|u|^3);
 * u1, u2 [m] the pair's two uniforms.                                         */
int cc_ta_pairs(double *va, double *vb, const double *C, const double *u1,
                const double *u2, int64_t m, void *stream);

/* P2C block reduction over a slot-ordered v [3][ldv] with cell
 * offsets off [cells+1] -> out [cells][7] (same layout as moments_out).      */
int cc_moments(const double *v, int64_t ldv, const int32_t *off, int32_t cells,
               const cc_params *params, double *out, void *stream);

/* NEXT f1 (R21): NRL electron-electron Coulomb logarithm from (lagged) moments:
 * lnL_j = 23.5 - ln(n^1/2 T^-5/4) - sqrt(1e-5 + (ln T - 2)^2/16), n in cm^-3 from
 * moments[j][0] (m^-3), T = (T_x+T_y+T_z)/3 eV from moments[j][4..6]; floored at 2.
 * moments: DEVICE [cells][7] (coulomb_collide's moments_out); out: DEVICE [cells],
 * usable as cc_params.ln_lambda_arr for the next step.                        */
int cc_coulomb_log(const double *moments, int32_t cells, double *out, void *stream);

/* Multi-GPU migration: out[p] = in[idx[p]] for p < m, for the
 * velocities [3][ldv] -> [3][ldo] and the cell ids; live cell ids are shifted
 * by -cell_shift (global -> local), dead (-1) stay -1.  No aliasing.         */
int cc_gather(const double *v, int64_t ldv, const int32_t *cell, const int32_t *idx, int64_t m,
              int32_t cell_shift, double *v_out, int64_t ldo, int32_t *cell_out, void *stream);

/* Multi-GPU: owner rank of each particle's global cell under the contiguous
 * cell-range split bounds [P+1] (DEVICE, bounds[r] = first cell of rank r);
 * -1 for dead or out-of-range ids.                                           */
int cc_owner(const int32_t *cell, int64_t n, const int32_t *bounds, int32_t nranks,
             int32_t *owner_out, void *stream);

/* ---- Multi-GPU over NCCL (csrc/cc_dist.cu) ----------------------
 * One process per GPU.  Bootstrap: rank 0 calls cc_nccl_get_unique_id, the caller
 * broadcasts the CC_NCCL_ID_BYTES bytes (e.g. torch.distributed), every rank calls
 * cc_nccl_comm_init (collective).  `comm` is an ncclComm_t passed as void*. */
#define CC_NCCL_ID_BYTES 128
int cc_nccl_get_unique_id(void *id_out);                                  /* HOST */
int cc_nccl_comm_init(void **comm_out, int32_t nranks, int32_t rank, const void *id);   /* HOST */
int cc_nccl_comm_destroy(void *comm);                                    /* HOST */

/* a8 across ranks: diag DEVICE [16] in place <- rank-ascending sum of every rank's
 * vector (ncclAllGather into scratch DEVICE [nranks][16], then cc_diag_sum_ranks):
 * the same bits on every rank for a given world size.         */
int cc_dist_diag_reduce(double *diag, double *scratch, void *comm, void *stream);

/* Particle migration, step 1: send_counts DEVICE int64 [nranks] (particles this rank
 * sends to each rank) -> recv_counts DEVICE int64 [nranks] (grouped ncclSend/Recv). */
int cc_dist_alltoall_counts(const int64_t *send_counts, int64_t *recv_counts, void *comm, void *stream);

/* Particle migration, step 2: exchange `nrows` rows of elem_bytes-sized (4 or 8)
 * elements.  Row r of the send buffer starts at send + r*lds elements and holds
 * the particles for rank p at [send_off[p], send_off[p+1]) (HOST int64 [nranks+1],
 * send_off[0] = 0); received particles from rank p land at [recv_off[p],
 * recv_off[p+1]) of each receive row (HOST offsets).  Grouped ncclSend/ncclRecv,
 * arrivals in source-rank order (deterministic).                               */
int cc_dist_exchange(const void *send, int64_t lds, void *recv, int64_t ldr, int32_t nrows, int32_t elem_bytes,
                     const int64_t *send_off, const int64_t *recv_off, void *comm, void *stream);

/* ---- Device-side particle migration (csrc/cc_migrate.cu) -------
 * No host synchronisation: every rank keeps its particles in n fixed slots,
 * dead-padded (cell -1).  coulomb_collide leaves the live particles in [0, L) and
 * the dead in [L, n), L = diag_out[0]; a push (cc_push) then rewrites the cell ids
 * as GLOBAL ids in place.  Migration moves every live particle to the rank owning
 * its cell under the contiguous split bounds (DEVICE int32 [nranks+1]):
 *  cc_mig_pack   (this rank) particles owned by rank p != rank are copied, in input
 *                order, into slot p of `send` and marked dead here; the others get
 *                their LOCAL cell id (cell - bounds[rank]); ids outside every range
 *                are dropped (status[1]).  Also zeroes the headers of `recv`.
 *  cc_dist_mig_exchange  grouped ncclSend / ncclRecv of whole slots with the listed
 *                peer ranks: the message size is the fixed slot size, so no count
 *                has to reach the host.
 *  cc_mig_unpack the arrivals, in (source rank, source order), into the free slots
 *                [L, L + A) with LOCAL cell ids (L from diag, e.g. the last
 *                coulomb_collide's diag_out; arrivals beyond n: status[2]).
 * The result is deterministic for a given world size.  send / recv: DEVICE,
 * nranks * cc_mig_slot_bytes(cap, xrows) bytes, 256-byte aligned; slot p = int64
 * count, padding to 64 bytes, then SoA rows of `cap` elements: v_x, v_y, v_z, the
 * xrows (0..3) payload rows of x [xrows][ldx] (fp64, e.g. positions), the cell
 * (int32, GLOBAL).  status DEVICE int32 [4], accumulated (zero it once): [0]
 * leavers dropped because their slot was full (cap too small), [1] ids outside
 * every range, [2] arrivals dropped because [L, n) was full, [3] arrivals
 * received.  A correct run has status[0..2] == 0.
 * workspace: DEVICE, cc_mig_workspace_bytes(n, nranks) bytes, 256-byte aligned. */
#define CC_MIG_MAX_RANKS 64
size_t cc_mig_slot_bytes(int64_t cap, int32_t xrows);                     /* HOST */
size_t cc_mig_workspace_bytes(int64_t n, int32_t nranks);                 /* HOST */
int cc_mig_pack(double *v, int64_t ldv, double *x, int64_t ldx, int32_t xrows, int32_t *cell, int64_t n,
                const int32_t *bounds, int32_t nranks, int32_t rank, int64_t cap, void *send, void *recv,
                int32_t *status, void *workspace, size_t workspace_bytes, void *stream);
int cc_dist_mig_exchange(const void *send, void *recv, size_t slot_bytes, const int32_t *peers, int32_t npeers,
                         void *comm, void *stream);                       /* peers: HOST int32 [npeers] */
int cc_mig_unpack(double *v, int64_t ldv, double *x, int64_t ldx, int32_t xrows, int32_t *cell, int64_t n,
                  const double *diag, const void *recv, const int32_t *bounds, int32_t nranks, int32_t rank,
                  int64_t cap, int32_t *status, void *stream);

/* Multi-GPU: rank-ascending sum of P gathered diagnostics vectors
 * gathered [P][16] -> out [16] (deterministic for a given P).   */
int cc_diag_sum_ranks(const double *gathered, int32_t nranks, double *out, void *stream);

/* ---- NEXT f2: the kinetic push of a subcycled PIC loop ---------- */



/* Steps S2b + S2c of Table 2 (SPEC push S:204-210) for n particles
 * in the OUTPUT order of a coulomb_collide call:
 *   v' = v + dt (q/m) E[cell]   (per-cell constant field; E NULL = 0)
 *   x' = x + dt v'              (position rows a < dims; boundary per axis)
 *   cell' = global cell of x', or -1 if absorbed.
 *  x_in   [3][ldx_in] fp64 positions; row a of particle p is read at index
 *         perm[p] (perm = coulomb_collide's perm_out, or NULL = p).
 *  x_out  [3][ldx_out] fp64, rows a < dims written for all n (rows >= dims
 *         are neither read nor written).
 *         Must not alias x_in unless perm == NULL and the rows coincide.
 *  v      [3][ldv] fp64, updated in place (live particles; not rewritten when
 *         E is NULL, v + 0 being v).
 *  cell   [n] int32, in place: in = LOCAL cell of the collision call (-1 dead,
 *         E row), out = GLOBAL cell after the push (-1 dead).
 *  cells, cell_base  the local cell range (rows of E; global id of local 0).
 *  E      DEVICE [3][ldE] (x, y, z rows, one column per local cell) or NULL.
 * Bit-exact with the oracle (no FMA contraction: every product and sum is
 * rounded as written).  Dead particles keep x and v.  CC_EINVAL on bad grid
 * (dims not 1..3, n[a] < 1, d[a] <= 0, prod n >= 2^31) or arguments.        */
int cc_push(const double *x_in, int64_t ldx_in, const int32_t *perm, double *x_out, int64_t ldx_out,
            double *v, int64_t ldv, int32_t *cell, int64_t n, int32_t cells, uint32_t cell_base,
            const cc_grid *grid, const double *E, int64_t ldE, double q_over_m, double dt, void *stream);

/* ---- NEXT f3: three-body recombination C5 ---------------------- */

/* Table 4 RS0-RS5 (SPEC recomb S:271-330) on the OUTPUT of a
 * coulomb_collide call (v_out / cell_out: cell-sorted, random pair order inside
 * a cell, dead last), in place, one pass, no atomics on the particle data:
 *  RS0 (R25) position q of cell j is a primary iff U(Philox(ctr = (q, cell_base+j,
 *      step, 4), key = seed)) < prob[j]  (prob DEVICE [cells]: the caller's
 *      1 - exp(-dt k_r n_i n_e));
 *  RS1-RS3 (R26) the i-th primary of the cell (position order) is matched to the
 *      i-th non-primary ("catalyte") for i < min(P_j, N_j - P_j) — unique and
 *      cell-local by construction; the other primaries are "starved" (unchanged);
 *  RS4 (R27) catalyte keeps its direction, |v_c'|^2 = |v_c|^2 + |v_p|^2 + 2 eps_bind/mass
 *      (a catalyte at rest takes the primary's direction, +x if both rest);
 *  RS5 (R28) the primary dies: cell -1 (velocity kept).
 * stats_out DEVICE uint64 [3] = {recombined, starved, primaries} (overwritten).
 * Must be called on an unmodified coulomb_collide output (it locates cells by
 * binary search in cell_out; ids must lie in [-1, cells)).  Kills are written
 * as order-preserving markers and turned into -1 by a second kernel, so no
 * search ever sees a half-updated array.  Bit-exact with the oracle.        */
int cc_recombine(double *v, int64_t ldv, int32_t *cell, int64_t n, int32_t cells, uint32_t cell_base,
                 const double *prob, double eps_bind, double mass, uint64_t seed, uint64_t step,
                 unsigned long long *stats_out, void *stream);

/* ---- NEXT f4: the paper's own P2C and replicated-grid scheme ---- */

/* Step S3a/S3b P2C the paper's way: a block reduction over UNSORTED
 * particles by fp64 atomics, each cell split into `sub` auxiliary sub-bins
 * omega_jm ("to [reduce] atomic updates congestion"; the sub-bin of
 * particle p is (p / 32) mod sub), then V^j = sum_m V^jm in fixed order.  A
 * warp of 32 particles of one cell (sorted input) is reduced with shuffles
 * before its atomics.
 *  v [3][ldv], cell [n] (LOCAL ids; -1 / out-of-range ignored).
 *  raw_out DEVICE [cells][7] = {N_j, sum v_x, v_y, v_z, sum v_x^2, v_y^2, v_z^2}.
 *  scratch DEVICE, >= cc_p2c_scratch_bytes(cells, sub) bytes, 8-byte aligned.
 * In the paper's multi-GPU scheme (replicated grid) every rank
 * deposits its own particles and raw_out is summed over ranks (one O(M)
 * all-reduce) before cc_p2c_moments.  Agrees with a sequential sum to
 * rounding (atomic order), not bitwise.                                      */
size_t cc_p2c_scratch_bytes(int32_t cells, int32_t sub);                  /* HOST */
int cc_p2c(const double *v, int64_t ldv, const int32_t *cell, int64_t n, int32_t cells, int32_t sub,
           double *raw_out, void *scratch, size_t scratch_bytes, void *stream);

/* Raw sums [cells][7] (cc_p2c, possibly all-reduced) -> moments [cells][7] in
 * coulomb_collide's layout {n_j, <v> (3), T_x, T_y, T_z} (reading R13; n_j =
 * N_j weight / V_j with params->weight, cell_volume(_arr); empty cells 0).  */
int cc_p2c_moments(const double *raw, int32_t cells, const cc_params *params, double *moments_out, void *stream);

/* Graph-friendly step counter (CUDA-graph replay of a subcycled loop):
 * *step_dev += inc on the device (cc_params.step_dev; see coulomb_collide). */
int cc_step_advance(uint32_t *step_dev, uint32_t inc, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* B200_COULOMB_H */
