/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU reference for the in situ Lagrangian
 * flow-map extraction hot path of arXiv 2004.02003 (Sane et al., "Scalable in
 * situ Lagrangian flow map extraction: demonstrating the viability of a
 * communication-free model").  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header or constant with the CUDA product path
 * (paper_2004_02003_b200/csrc).  Compiled with -ffp-contract=off, no SIMD
 * intrinsics; OpenMP only over independent particles.
 *
 * Citations: P:nnn = /root/reference/PAPER.md line nnn; S:nnn = SPEC.md line.
 *
 *  - Flow map F_{t0}^{t}(x0): P:86 (§2.1).
 *  - Uniform seeding, intervals, reset: P:148-152 (§2.3).  (Seeding itself is in
 *    oracle/__init__.py, it is pure lattice enumeration.)
 *  - RK4 advection: P:204 (§3.1) "Particle advection is performed using RK4".
 *    Classical 4-stage RK with stage times t, t+dt/2, t+dt/2, t+dt.
 *  - Velocity between slices: linear in time (north star; Eq. 1
 *    applied in t) and multilinear in space over the uniform grid.
 *  - BTO: particles that leave the block are terminated and discarded
 *    (§3.1).  Stage-level rule (reading R2): if ANY stage
 *    sample or the updated position leaves the block the particle terminates
 *    at its pre-step position.
 *  - Global-domain exits: EXIT_DOMAIN in both strategies (reading R5).
 *  - COMM (Lagrangian-MPI baseline): the result does not
 *    depend on the decomposition, so the oracle integrates it on
 *    the whole domain, i.e. block := domain.
 *
 * Parity pins: tests/test_oracle_pins.py (closed forms, brute force, paper
 * values).  No function here is "parity unpinned": orc_tri (tent sums, affine
 * exactness), rk4_step (uniform, rotation, affine series, 4th order, closed
 * crossing schedules), face_distance (uniform-flow distances,
 * test_face_distance_uniform_flow_closed_form), mark_touched (exact node set,
 * test_touched_nodes_exact_set_uniform_flow).  scripts/mutation_check.sh
 * plants one mistake per function and checks that a pin fails.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

typedef struct {
    int32_t dim;          /* 2 or 3 */
    int32_t pad_;
    int64_t N[3];         /* nodes per axis (unused axis = 1) */
    double  o[3];         /* origin */
    double  h[3];         /* spacing */
} orc_grid;

enum { ORC_VALID = 0, ORC_TERM_BOUNDARY = 1, ORC_EXIT_DOMAIN = 2 };
enum { ORC_BTO = 0, ORC_COMM = 1 };

/* Node value V[n] (component c), global AoS fp32 array [Nz][Ny][Nx][dim]. */
static double node_value(const orc_grid* g, const float* V, const int64_t n[3], int c)
{
    int64_t idx = n[0] + g->N[0] * (n[1] + g->N[1] * n[2]);
    return (double)V[idx * g->dim + c];
}

/*
 * Multilinear interpolation of V at physical point q:
 *   u = (q - o) / h;  i = clamp(floor(u), 0, N-2);  f = u - i;
 *   Tri = sum over corners delta in {0,1}^d of prod_a (delta_a ? f_a : 1 - f_a) * V[i + delta].
 * Clamping i to N-2 makes the closed upper face use f = 1 (reading R6).
 */
void orc_tri(const orc_grid* g, const float* V, const double* q, double* out)
{
    int64_t i[3] = {0, 0, 0};
    double f[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < g->dim; ++a) {
        double u = (q[a] - g->o[a]) / g->h[a];
        double fl = floor(u);
        int64_t ia = (int64_t)fl;
        if (ia < 0) ia = 0;
        if (ia > g->N[a] - 2) ia = g->N[a] - 2;
        i[a] = ia;
        f[a] = u - (double)ia;
    }
    for (int c = 0; c < g->dim; ++c) out[c] = 0.0;
    int ncorner = 1 << g->dim;
    for (int corner = 0; corner < ncorner; ++corner) {
        double w = 1.0;
        int64_t n[3] = {0, 0, 0};
        for (int a = 0; a < g->dim; ++a) {
            int delta = (corner >> a) & 1;
            w *= delta ? f[a] : (1.0 - f[a]);
            n[a] = i[a] + delta;
        }
        for (int c = 0; c < g->dim; ++c) out[c] += w * node_value(g, V, n, c);
    }
}

/* Mark the nodes read by one Tri() call in a per-node byte map (bit `bit`). */
static void mark_touched(const orc_grid* g, const double* q, uint8_t* touched, uint8_t bit)
{
    int64_t i[3] = {0, 0, 0};
    for (int a = 0; a < g->dim; ++a) {
        double u = (q[a] - g->o[a]) / g->h[a];
        int64_t ia = (int64_t)floor(u);
        if (ia < 0) ia = 0;
        if (ia > g->N[a] - 2) ia = g->N[a] - 2;
        i[a] = ia;
    }
    int ncorner = 1 << g->dim;
    for (int corner = 0; corner < ncorner; ++corner) {
        int64_t n[3] = {0, 0, 0};
        for (int a = 0; a < g->dim; ++a) n[a] = i[a] + ((corner >> a) & 1);
        int64_t idx = n[0] + g->N[0] * (n[1] + g->N[1] * n[2]);
        /* benign race under OpenMP: every writer sets the same bit */
        touched[idx] |= bit;
    }
}

/* q in the closed global domain  Omega = prod_a [o_a, o_a + (N_a - 1) h_a]. */
static int in_domain(const orc_grid* g, const double* q)
{
    for (int a = 0; a < g->dim; ++a) {
        double top = g->o[a] + (double)(g->N[a] - 1) * g->h[a];
        if (!(q[a] >= g->o[a] && q[a] <= top)) return 0;
    }
    return 1;
}

/* q in the block  prod_a [o + lo h, o + hi h), closed on the global upper face
 * (hi = N).  Half-open ownership: the upper block owns a shared face (S:114,
 * reading R3). */
static int in_block(const orc_grid* g, const int64_t* lo, const int64_t* hi, const double* q)
{
    for (int a = 0; a < g->dim; ++a) {
        double lo_x = g->o[a] + (double)lo[a] * g->h[a];
        if (!(q[a] >= lo_x)) return 0;
        if (hi[a] >= g->N[a]) {
            double top = g->o[a] + (double)(g->N[a] - 1) * g->h[a];
            if (!(q[a] <= top)) return 0;
        } else {
            double hi_x = g->o[a] + (double)hi[a] * g->h[a];
            if (!(q[a] < hi_x)) return 0;
        }
    }
    return 1;
}

/* Smallest distance, in cell units of its axis, from q to any block face or
 * global face (the flag-parity excuse band, reading R14). */
static double face_distance(const orc_grid* g, const int64_t* flo, const int64_t* fhi, const double* q)
{
    double best = INFINITY;
    for (int a = 0; a < g->dim; ++a) {
        double u = (q[a] - g->o[a]) / g->h[a];
        double faces[4] = {0.0, (double)(g->N[a] - 1), (double)flo[a], (double)fhi[a]};
        for (int k = 0; k < 4; ++k) {
            double dd = fabs(u - faces[k]);
            if (dd < best) best = dd;
        }
    }
    return best;
}

/* Sample test of one RK4 stage point / updated position.
 * Returns ORC_VALID, ORC_EXIT_DOMAIN or ORC_TERM_BOUNDARY (BTO only). */
static int classify(const orc_grid* g, const int64_t* lo, const int64_t* hi, int mode, const double* q)
{
    if (!in_domain(g, q)) return ORC_EXIT_DOMAIN;
    if (mode == ORC_BTO && !in_block(g, lo, hi, q)) return ORC_TERM_BOUNDARY;
    return ORC_VALID;
}

/* Butcher tableau of classical RK4 (stage times t, t+dt/2, t+dt/2, t+dt):
 * sample offsets beta_s, time-lerp weights alpha_s, combination weights b_s/6. */
static const double RK_BETA[4]  = {0.0, 0.5, 0.5, 1.0};
static const double RK_ALPHA[4] = {0.0, 0.5, 0.5, 1.0};
static const double RK_B[4]     = {1.0, 2.0, 2.0, 1.0};

/*
 * One RK4 step of one particle at x (in/out).  SURVEY.md §8(c) step 4:
 *   q_1 = x;  q_s = x + beta_s dt k_{s-1};
 *   each q_s: outside Omega -> EXIT_DOMAIN; (BTO) outside B -> TERM_BOUNDARY;
 *             on either the particle stops and x is left unchanged;
 *   k_s = (1 - alpha_s) Tri(V0, q_s) + alpha_s Tri(V1, q_s);
 *   x' = x + dt/6 (k1 + 2 k2 + 2 k3 + k4); the same tests on x'; then x <- x'.
 * check = 0 disables every test (used by the integrator-only pins).
 * touched (optional): per global node byte map; bit 0 = V0 read, bit 1 = V1
 * read by the method's stage gathers (stage 1 reads only V0, stage 4 only V1).
 */
static int rk4_step(const orc_grid* g, const int64_t* lo, const int64_t* hi, int mode,
                    int check, const float* V0, const float* V1, double dt, double* x,
                    uint8_t* touched, const int64_t* flo, const int64_t* fhi, double* mind)
{
    const int d = g->dim;
    double k[4][3];
    double kprev[3] = {0.0, 0.0, 0.0};
    for (int s = 0; s < 4; ++s) {
        double q[3] = {0.0, 0.0, 0.0};
        for (int a = 0; a < d; ++a) q[a] = x[a] + RK_BETA[s] * dt * kprev[a];
        if (mind && s > 0) {
            double fd = face_distance(g, flo, fhi, q);
            if (fd < *mind) *mind = fd;
        }
        if (check) {
            int outcome = classify(g, lo, hi, mode, q);
            if (outcome != ORC_VALID) return outcome;
        }
        double v0[3] = {0.0, 0.0, 0.0}, v1[3] = {0.0, 0.0, 0.0};
        if (RK_ALPHA[s] != 1.0) {
            orc_tri(g, V0, q, v0);
            if (touched) mark_touched(g, q, touched, 1);
        }
        if (RK_ALPHA[s] != 0.0) {
            orc_tri(g, V1, q, v1);
            if (touched) mark_touched(g, q, touched, 2);
        }
        for (int a = 0; a < d; ++a) {
            k[s][a] = (1.0 - RK_ALPHA[s]) * v0[a] + RK_ALPHA[s] * v1[a];
            kprev[a] = k[s][a];
        }
    }
    double xn[3] = {0.0, 0.0, 0.0};
    for (int a = 0; a < d; ++a) {
        double sum = 0.0;
        for (int s = 0; s < 4; ++s) sum += RK_B[s] * k[s][a];
        xn[a] = x[a] + dt / 6.0 * sum;
    }
    if (mind) {
        double fd = face_distance(g, flo, fhi, xn);
        if (fd < *mind) *mind = fd;
    }
    if (check) {
        int outcome = classify(g, lo, hi, mode, xn);
        if (outcome != ORC_VALID) return outcome;
    }
    for (int a = 0; a < d; ++a) x[a] = xn[a];
    return ORC_VALID;
}

/*
 * One simulation cycle (slices V0 = v(t_c), V1 = v(t_c + dt)) for n particles:
 * every VALID particle takes one rk4_step (in situ a particle advances
 * by a single step per simulation step).  Terminated particles keep their
 * pre-step position and record `cycle` in term_cycle.
 */
void orc_cycle(const orc_grid* g, const int64_t* lo, const int64_t* hi, int32_t mode,
               const float* V0, const float* V1, double dt, int64_t n,
               double* pos, uint8_t* status, int32_t* term_cycle, int32_t cycle,
               uint8_t* touched, const int64_t* flo, const int64_t* fhi, double* min_face)
{
    const int d = g->dim;
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n; ++p) {
        if (status[p] != ORC_VALID) continue;
        double x[3] = {0.0, 0.0, 0.0};
        for (int a = 0; a < d; ++a) x[a] = pos[p * d + a];
        int outcome = rk4_step(g, lo, hi, mode, 1, V0, V1, dt, x, touched, flo, fhi,
                               min_face ? &min_face[p] : NULL);
        if (outcome == ORC_VALID) {
            for (int a = 0; a < d; ++a) pos[p * d + a] = x[a];
        } else {
            status[p] = (uint8_t)outcome;
            term_cycle[p] = cycle;
        }
    }
}

/* Plain RK4 step of the interpolated field with no boundary logic (the
 * integrator pins exercise the same rk4_step with tests disabled). */
void orc_rk4_free(const orc_grid* g, const float* V0, const float* V1, double dt,
                  int64_t n, double* pos)
{
    const int d = g->dim;
    for (int64_t p = 0; p < n; ++p) {
        double x[3] = {0.0, 0.0, 0.0};
        for (int a = 0; a < d; ++a) x[a] = pos[p * d + a];
        rk4_step(g, NULL, NULL, ORC_COMM, 0, V0, V1, dt, x, NULL, NULL, NULL, NULL);
        for (int a = 0; a < d; ++a) pos[p * d + a] = x[a];
    }
}
