/*
 * orcha_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the hydro hot path
 * that ORCHA orchestrates in its Sedov case study (arXiv 2507.09337), used to
 * prove the CUDA path correct.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2507_09337_b200/) never imports, links or calls it and
 * shares no code, headers or constants with it.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fPIC -shared (see
 * oracle/__init__.py).  No FMA contraction: every expression below is
 * evaluated exactly as written, left to right, in IEEE fp64.
 *
 * What it computes (PAPER.md = P:Lnn; SURVEY.md section 8 = the normative reading):
 *   - one GLOBAL array per conserved variable (rho, rho*u, rho*v, rho*w, E)
 *     with ng >= 4 ghost layers on every active axis; no blocks, no packets
 *     (blocks are GPU-side bookkeeping whose result must equal this array);
 *   - ghost fill axis by axis (x, then y over x-ghosts, then z over x,y-ghosts)
 *     with outflow / periodic / reflect boundaries;
 *   - gamma-law EOS, "a simple algebraic expression" (sec 5.2);
 *   - PLM/minmod reconstruction on primitives (reading c1);
 *   - HLL flux with Davis speeds from the reconstructed states (A7, c2);
 *   - conservative update + SSP-RK2 (A8, c3; "2nd-order Runge-Kutta",
 *     P:L667 sec 6);
 *   - communication avoidance: stage 1 on interior + a 2-cell ring, stage 2
 *     on the interior, no ghost refresh between stages ("make the halo twice
 *     as thick ... redundantly compute the inner portion of the halo in the
 *     first stage", sec 6; A9, c4, c5);
 *   - CFL dt with argmax tie-break on the lowest global cell index, then the
 *     t_end clamp (A4, c7, c8).
 * SURVEY 8(f) F4 scheme variants (grid flags; defaults are the above):
 *   - limiter MC (monotonized central, van Leer 1977): the slope of smallest
 *     magnitude among 2*dm, 2*dp and (dm+dp)/2 when dm, dp agree in sign, else
 *     0 (reading c21);
 *   - Riemann solver HLLC (Toro, "Riemann Solvers and Numerical Methods for
 *     Fluid Dynamics", 3rd ed., sec 10.4, eqs 10.37-10.39), same wave speeds
 *     as HLL (reading c20);
 *   - expensive-EOS surrogate (reading c22; the paper's Helmholtz EOS makes the
 *     GPU favourable): ideal gas + radiation with c_v = 1,
 *     rho e = rho T + a T^4, p = (gamma-1) rho T + a T^4 / 3, temperature by
 *     Newton iteration, sound speed from Chandrasekhar's Gamma_1.
 * The "refill" mode (ghosts of U1 refilled between the stages) is the plain
 * two-refresh scheme that P:L667-668 describes before the trick; it is the
 * oracle of SURVEY 8(f) F1 and the telescoping equivalence pin.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* "oracle-omp": the same source built with -fopenmp splits the
 * k loops of the per-cell sweeps over threads.  Every cell's arithmetic and
 * the order of its terms are unchanged (cells are independent; the floor-hit
 * count is an integer sum), so the result is bitwise the single-threaded
 * one.  Without -fopenmp the pragmas are absent. */
#ifdef _OPENMP
#include <omp.h>
#define ORACLE_PAR_FOR _Pragma("omp parallel for schedule(static)")
#define ORACLE_PAR_FOR_PRIMS _Pragma("omp parallel for schedule(static) reduction(+ : nh) reduction(| : bad)")
#else
#define ORACLE_PAR_FOR
#define ORACLE_PAR_FOR_PRIMS
#endif

typedef struct {
  int32_t ndim;       /* 1, 2 or 3 */
  int32_t N[3];       /* interior cells per axis (1 on inactive axes) */
  int32_t ng;         /* ghost width on active axes */
  double xmin[3], xmax[3];
  int32_t bc[3][2];   /* per axis, low/high: 0 outflow, 1 periodic, 2 reflect */
  double gamma, cfl, smallp;
  int32_t riemann;    /* 0 HLL, 1 HLLC (F4) */
  int32_t limiter;    /* 0 minmod, 1 MC (F4) */
  int32_t eos;        /* 0 gamma law, 1 gas + radiation by Newton (F4 expensive-EOS surrogate) */
  int32_t eos_work;   /* eos 1: temperature solves per evaluation (>= 1; the surrogate's cost knob) */
  double arad;        /* eos 1: radiation constant a (code units) */
} oracle_grid;

enum { BC_OUTFLOW = 0, BC_PERIODIC = 1, BC_REFLECT = 2 };
enum { TAG_CFL = 0, TAG_CLAMP = 1 };
enum { ORC_OK = 0, ORC_E_ARG = -1, ORC_E_NONPHYSICAL = -4 };

/* ---------------------------------------------------------------- indexing */

static int64_t ext(const oracle_grid* G, int d) {
  return (d < G->ndim) ? (int64_t)G->N[d] + 2 * (int64_t)G->ng : 1;
}
static int64_t gh(const oracle_grid* G, int d) { return (d < G->ndim) ? G->ng : 0; }

/* flat index of variable v at interior-relative coordinates (i, j, k) */
static int64_t at(const oracle_grid* G, int v, int64_t i, int64_t j, int64_t k) {
  int64_t X = ext(G, 0), Y = ext(G, 1), Z = ext(G, 2);
  return (((int64_t)v * Z + (k + gh(G, 2))) * Y + (j + gh(G, 1))) * X + (i + gh(G, 0));
}

int64_t oracle_array_len(const oracle_grid* G) { return 5 * ext(G, 0) * ext(G, 1) * ext(G, 2); }

static int check_grid(const oracle_grid* G) {
  if (G->ndim < 1 || G->ndim > 3) return ORC_E_ARG;
  if (G->ng < 4) return ORC_E_ARG;
  if (G->riemann < 0 || G->riemann > 1 || G->limiter < 0 || G->limiter > 1) return ORC_E_ARG;
  if (G->eos < 0 || G->eos > 1 || (G->eos == 1 && (G->eos_work < 1 || !(G->arad >= 0.0)))) return ORC_E_ARG;
  for (int d = 0; d < 3; d++) {
    if (d < G->ndim) {
      if (G->N[d] < G->ng) return ORC_E_ARG;
    } else if (G->N[d] != 1) {
      return ORC_E_ARG;
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------- 1. ghost filling */

/* Source index along one axis for ghost coordinate c (outside [0, n)) under
 * boundary condition bc; *flip is set when the normal momentum changes sign. */
static int64_t bc_source(int64_t c, int64_t n, int bc_lo, int bc_hi, int* flip) {
  *flip = 0;
  if (c < 0) {
    if (bc_lo == BC_PERIODIC) return c + n;
    if (bc_lo == BC_REFLECT) { *flip = 1; return -1 - c; }
    return 0; /* outflow: copy of the edge cell */
  }
  if (bc_hi == BC_PERIODIC) return c - n;
  if (bc_hi == BC_REFLECT) { *flip = 1; return 2 * n - 1 - c; }
  return n - 1;
}

/* x over interior y,z; then y over all x incl. ghosts;
 * then z over all x,y.  Refresh "before we invoke ORCHA". */
int oracle_fill_ghosts(const oracle_grid* G, double* U) {
  int rc = check_grid(G);
  if (rc) return rc;
  for (int d = 0; d < G->ndim; d++) {
    const int64_t n = G->N[d];
    /* axis d: its ghost layers; axes before d: full padded range (their
     * ghosts are already filled); axes after d: interior only */
    int64_t lo[3], hi[3];
    for (int e = 0; e < 3; e++) {
      if (e <= d) { lo[e] = -gh(G, e); hi[e] = G->N[e] + gh(G, e); }
      else { lo[e] = 0; hi[e] = G->N[e]; }
    }
    for (int64_t k = lo[2]; k < hi[2]; k++)
      for (int64_t j = lo[1]; j < hi[1]; j++)
        for (int64_t i = lo[0]; i < hi[0]; i++) {
          int64_t c = (d == 0) ? i : (d == 1) ? j : k;
          if (c >= 0 && c < n) continue; /* not a ghost along d */
          int flip;
          int64_t src = bc_source(c, n, G->bc[d][0], G->bc[d][1], &flip);
          int64_t si = (d == 0) ? src : i, sj = (d == 1) ? src : j, sk = (d == 2) ? src : k;
          for (int v = 0; v < 5; v++) {
            double x = U[at(G, v, si, sj, sk)];
            if (flip && v == 1 + d) x = -x;
            U[at(G, v, i, j, k)] = x;
          }
        }
  }
  return ORC_OK;
}

/* ------------------------------------------------- 2. EOS */

/* Expensive-EOS surrogate (reading c22).  Newton for T from the gas-only
 * guess, stopping when |dT| <= 1e-14 |T| or after 50 iterations; the solve is
 * repeated eos_work times, each repeat restarting from the guess (`+ 0.0 *
 * T` keeps the repeats data-dependent without changing a finite guess), so the
 * result is that of one solve. */
static double temp_from_e(const oracle_grid* G, double rho, double eint) {
  double T = 0.0;
  for (int r = 0; r < G->eos_work; r++) {
    T = eint + 0.0 * T;
    for (int it = 0; it < 50; it++) {
      double T3 = (T * T) * T;
      double f = (T + (G->arad * (T3 * T)) / rho) - eint;
      double fp = 1.0 + ((4.0 * G->arad) * T3) / rho;
      double dT = f / fp;
      T = T - dT;
      if (fabs(dT) <= 1e-14 * fabs(T)) break;
    }
  }
  return T;
}

static double temp_from_p(const oracle_grid* G, double rho, double p) {
  double gr = (G->gamma - 1.0) * rho;
  double T = 0.0;
  for (int r = 0; r < G->eos_work; r++) {
    T = p / gr + 0.0 * T;
    for (int it = 0; it < 50; it++) {
      double T3 = (T * T) * T;
      double f = (gr * T + (G->arad * (T3 * T)) / 3.0) - p;
      double fp = gr + ((4.0 * G->arad) * T3) / 3.0;
      double dT = f / fp;
      T = T - dT;
      if (fabs(dT) <= 1e-14 * fabs(T)) break;
    }
  }
  return T;
}

/* Gamma_1 of the gas + radiation mixture (Chandrasekhar), beta = p_gas / p:
 *   Gamma_1 = beta + (4 - 3 beta)^2 (gamma - 1) / (beta + 12 (gamma - 1)(1 - beta)) */
static double gamma1(const oracle_grid* G, double rho, double p, double T) {
  double g1 = G->gamma - 1.0;
  double beta = (g1 * rho * T) / p;
  double x = 4.0 - 3.0 * beta;
  return beta + ((x * x) * g1) / (beta + (12.0 * g1) * (1.0 - beta));
}

/* Primitive recovery; returns 1 if the floor fired, -1 if !(rho > 0). */
int oracle_prim(const oracle_grid* G, const double U[5], double q[5]) {
  double rho = U[0];
  double ir = 1.0 / rho;
  double u = U[1] * ir;
  double v = U[2] * ir;
  double w = U[3] * ir;
  double ke = (0.5 * rho) * ((u * u + v * v) + w * w);
  double p;
  if (G->eos == 0) {
    p = (G->gamma - 1.0) * (U[4] - ke);
  } else {
    double T = temp_from_e(G, rho, (U[4] - ke) * ir);
    p = ((G->gamma - 1.0) * rho) * T + (G->arad * ((T * T) * (T * T))) / 3.0;
  }
  int hit = 0;
  if (p < G->smallp) { p = G->smallp; hit = 1; } /* NaN is kept (c10) */
  q[0] = rho; q[1] = u; q[2] = v; q[3] = w; q[4] = p;
  if (!(rho > 0.0)) return -1;
  return hit;
}

double oracle_sound_speed(const oracle_grid* G, const double q[5]) {
  if (G->eos == 0) return sqrt((G->gamma * q[4]) / q[0]);
  double T = temp_from_p(G, q[0], q[4]);
  return sqrt((gamma1(G, q[0], q[4], T) * q[4]) / q[0]);
}

/* Specific internal energy of (rho, p) under the expensive EOS (tests). */
double oracle_eint_from_p(const oracle_grid* G, double rho, double p) {
  double T = temp_from_p(G, rho, p);
  return T + (G->arad * ((T * T) * (T * T))) / rho;
}

/* ---------------------------------------- 3. PLM/minmod */

double oracle_minmod_slope(double qm, double q0, double qp) {
  double dm = q0 - qm;
  double dp = qp - q0;
  if (dm * dp > 0.0) {
    double a = fabs(dm), b = fabs(dp);
    double m = (a < b) ? a : b;
    return copysign(m, dm);
  }
  return 0.0;
}

/* MC (monotonized central) slope, reading c21. */
double oracle_mc_slope(double qm, double q0, double qp) {
  double dm = q0 - qm;
  double dp = qp - q0;
  if (dm * dp > 0.0) {
    double a = 2.0 * fabs(dm), b = 2.0 * fabs(dp), c = 0.5 * fabs(dm + dp);
    double m = (a < b) ? a : b;
    m = (c < m) ? c : m;
    return copysign(m, dm);
  }
  return 0.0;
}

/* ------------------------------------------------ 4. HLL */

static void cons_and_flux(const oracle_grid* G, int d, const double q[5], double U[5], double F[5],
                          double* c) {
  double gam = G->gamma;
  double ig1 = 1.0 / (gam - 1.0);
  double E;
  if (G->eos == 0) {
    *c = sqrt((gam * q[4]) / q[0]);
    E = q[4] * ig1 + (0.5 * q[0]) * ((q[1] * q[1] + q[2] * q[2]) + q[3] * q[3]);
  } else {
    double T = temp_from_p(G, q[0], q[4]);
    *c = sqrt((gamma1(G, q[0], q[4], T) * q[4]) / q[0]);
    E = (q[0] * T + G->arad * ((T * T) * (T * T))) + (0.5 * q[0]) * ((q[1] * q[1] + q[2] * q[2]) + q[3] * q[3]);
  }
  U[0] = q[0];
  U[1] = q[0] * q[1];
  U[2] = q[0] * q[2];
  U[3] = q[0] * q[3];
  U[4] = E;
  double n = q[1 + d];
  for (int k = 0; k < 5; k++) F[k] = U[k] * n;
  F[1 + d] = F[1 + d] + q[4];
  F[4] = (E + q[4]) * n;
}

/* Face flux from the reconstructed left/right primitive states. */
void oracle_hll(const oracle_grid* G, int d, const double qL[5], const double qR[5], double F[5]) {
  double UL[5], FL[5], UR[5], FR[5], cL, cR;
  cons_and_flux(G, d, qL, UL, FL, &cL);
  cons_and_flux(G, d, qR, UR, FR, &cR);
  double nL = qL[1 + d], nR = qR[1 + d];
  double a = nL - cL, b = nR - cR;
  double SL = (a < b) ? a : b;
  double e = nL + cL, f = nR + cR;
  double SR = (e > f) ? e : f;
  if (SL >= 0.0) {
    for (int k = 0; k < 5; k++) F[k] = FL[k];
  } else if (SR <= 0.0) {
    for (int k = 0; k < 5; k++) F[k] = FR[k];
  } else {
    double inv = 1.0 / (SR - SL);
    for (int k = 0; k < 5; k++)
      F[k] = ((SR * FL[k] - SL * FR[k]) + (SL * SR) * (UR[k] - UL[k])) * inv;
  }
}

/* HLLC (reading c20; Toro sec 10.4).  Wave speeds S_L, S_R as in HLL; the
 * contact speed (10.37)
 *   S* = ((p_R - p_L) + (d_L u_L - d_R u_R)) / (d_L - d_R),  d_K = rho_K (S_K - u_K);
 * the star state (10.39), f_K = d_K / (S_K - S*),
 *   U*_K = (f_K, f_K S* (normal), f_K v_K, f_K w_K (transverse),
 *           f_K (E_K / rho_K + (S* - u_K) (S* + p_K / d_K)));
 * and F*_K = F_K + S_K (U*_K - U_K) (10.38).  F = F_L if S_L >= 0, else F_R
 * if S_R <= 0, else F*_L if S* >= 0, else F*_R. */
void oracle_hllc(const oracle_grid* G, int d, const double qL[5], const double qR[5], double F[5]) {
  double UL[5], FL[5], UR[5], FR[5], cL, cR;
  cons_and_flux(G, d, qL, UL, FL, &cL);
  cons_and_flux(G, d, qR, UR, FR, &cR);
  double nL = qL[1 + d], nR = qR[1 + d];
  double a = nL - cL, b = nR - cR;
  double SL = (a < b) ? a : b;
  double e = nL + cL, f = nR + cR;
  double SR = (e > f) ? e : f;
  if (SL >= 0.0) {
    for (int k = 0; k < 5; k++) F[k] = FL[k];
  } else if (SR <= 0.0) {
    for (int k = 0; k < 5; k++) F[k] = FR[k];
  } else {
    double dL = qL[0] * (SL - nL);
    double dR = qR[0] * (SR - nR);
    double Ss = ((qR[4] - qL[4]) + (dL * nL - dR * nR)) / (dL - dR);
    int left = Ss >= 0.0;
    const double* q = left ? qL : qR;
    const double* U = left ? UL : UR;
    const double* FK = left ? FL : FR;
    double SK = left ? SL : SR, dK = left ? dL : dR, nK = left ? nL : nR;
    double fK = dK / (SK - Ss);
    double Us[5];
    Us[0] = fK;
    for (int t = 0; t < 3; t++) Us[1 + t] = (t == d) ? fK * Ss : fK * q[1 + t];
    Us[4] = fK * (U[4] / q[0] + (Ss - nK) * (Ss + q[4] / dK));
    for (int k = 0; k < 5; k++) F[k] = FK[k] + SK * (Us[k] - U[k]);
  }
}

/* Face flux at the face between cells i and i+1 along axis d, from the four
 * primitive states q_{i-1}, q_i, q_{i+1}, q_{i+2} (each [5]). */
void oracle_face_flux(const oracle_grid* G, int d, const double qm[5], const double q0[5],
                      const double q1[5], const double q2[5], double F[5]) {
  double qL[5], qR[5];
  for (int v = 0; v < 5; v++) {
    double s0 = G->limiter ? oracle_mc_slope(qm[v], q0[v], q1[v]) : oracle_minmod_slope(qm[v], q0[v], q1[v]);
    double s1 = G->limiter ? oracle_mc_slope(q0[v], q1[v], q2[v]) : oracle_minmod_slope(q0[v], q1[v], q2[v]);
    qL[v] = q0[v] + 0.5 * s0;
    qR[v] = q1[v] - 0.5 * s1;
  }
  if (G->riemann) oracle_hllc(G, d, qL, qR, F);
  else oracle_hll(G, d, qL, qR, F);
}

/* --------------------------------------------------- the method on arrays */

typedef struct {
  int64_t lo[3], hi[3]; /* half-open cell region, interior-relative */
} region;

static double dxd(const oracle_grid* G, int d) { return (G->xmax[d] - G->xmin[d]) / (double)G->N[d]; }

/* Primitives of U over region R into Q (same array shape); counts floor hits.
 * Returns -1 if a non-positive density was met. */
static int prims_region(const oracle_grid* G, const double* U, double* Q, region R, int64_t* hits) {
  int bad = 0;
  int64_t nh = 0;
  ORACLE_PAR_FOR_PRIMS
  for (int64_t k = R.lo[2]; k < R.hi[2]; k++)
    for (int64_t j = R.lo[1]; j < R.hi[1]; j++)
      for (int64_t i = R.lo[0]; i < R.hi[0]; i++) {
        double u[5], q[5];
        for (int v = 0; v < 5; v++) u[v] = U[at(G, v, i, j, k)];
        int r = oracle_prim(G, u, q);
        if (r < 0) bad = 1;
        if (r > 0) nh++;
        for (int v = 0; v < 5; v++) Q[at(G, v, i, j, k)] = q[v];
      }
  *hits += nh;
  return bad ? -1 : 0;
}

/* D(U) over region R from primitives Q (valid on R widened by 2 along each
 * axis separately):
 *   D = ((dFx)*idx + (dFy)*idy) + (dFz)*idz
 * computed one axis at a time; without FMA contraction the running sum is
 * bitwise the left-to-right expression. */
static void divergence(const oracle_grid* G, const double* Q, region R, double* D) {
  for (int d = 0; d < G->ndim; d++) {
    double id = 1.0 / dxd(G, d);
    int64_t sh[3] = {0, 0, 0};
    sh[d] = 1;
    ORACLE_PAR_FOR
    for (int64_t k = R.lo[2]; k < R.hi[2]; k++)
      for (int64_t j = R.lo[1]; j < R.hi[1]; j++)
        for (int64_t i = R.lo[0]; i < R.hi[0]; i++) {
          double q[4][5];
          double Fm[5], Fp[5];
          /* low face (between c-1 and c): cells c-2 .. c+1 */
          for (int s = 0; s < 4; s++)
            for (int v = 0; v < 5; v++)
              q[s][v] = Q[at(G, v, i + (s - 2) * sh[0], j + (s - 2) * sh[1], k + (s - 2) * sh[2])];
          oracle_face_flux(G, d, q[0], q[1], q[2], q[3], Fm);
          /* high face (between c and c+1): cells c-1 .. c+2 */
          for (int s = 0; s < 4; s++)
            for (int v = 0; v < 5; v++)
              q[s][v] = Q[at(G, v, i + (s - 1) * sh[0], j + (s - 1) * sh[1], k + (s - 1) * sh[2])];
          oracle_face_flux(G, d, q[0], q[1], q[2], q[3], Fp);
          for (int v = 0; v < 5; v++) {
            double t = (Fp[v] - Fm[v]) * id;
            int64_t a = at(G, v, i, j, k);
            D[a] = (d == 0) ? t : (D[a] + t);
          }
        }
  }
}

static region interior(const oracle_grid* G) {
  region R;
  for (int d = 0; d < 3; d++) { R.lo[d] = 0; R.hi[d] = G->N[d]; }
  return R;
}
static region widen(const oracle_grid* G, region R, int64_t w) {
  for (int d = 0; d < G->ndim; d++) { R.lo[d] -= w; R.hi[d] += w; }
  return R;
}

/* -------------------------------------------------- 5. CFL dt (A4, c7, c8) */

/* Over interior cells: s = ((|u|+c)*idx + (|v|+c)*idy) + (|w|+c)*idz, the
 * inactive axes omitted; dt = cfl / max s; argmax = lowest global index
 * g = (k*Ny + j)*Nx + i; then the t_end clamp. */
int oracle_dt(const oracle_grid* G, const double* U, double t_remaining, double* dt, int64_t* argmax,
              int32_t* tag, double* smax_out) {
  int rc = check_grid(G);
  if (rc) return rc;
  double id[3];
  for (int d = 0; d < G->ndim; d++) id[d] = 1.0 / dxd(G, d);
  double smax = -1.0;
  int64_t best = -1;
  int bad = 0;
  for (int64_t k = 0; k < G->N[2]; k++)
    for (int64_t j = 0; j < G->N[1]; j++)
      for (int64_t i = 0; i < G->N[0]; i++) {
        double u[5], q[5];
        for (int v = 0; v < 5; v++) u[v] = U[at(G, v, i, j, k)];
        if (oracle_prim(G, u, q) < 0) bad = 1;
        double c = oracle_sound_speed(G, q);
        double s = (fabs(q[1]) + c) * id[0];
        if (G->ndim > 1) s = s + (fabs(q[2]) + c) * id[1];
        if (G->ndim > 2) s = s + (fabs(q[3]) + c) * id[2];
        int64_t g = (k * G->N[1] + j) * G->N[0] + i;
        if (best < 0 || s > smax || (s != s && smax == smax)) { /* NaN wins */
          smax = s;
          best = g;
        }
      }
  double d = G->cfl / smax;
  int32_t t = TAG_CFL;
  if (t_remaining < d) { d = t_remaining; t = TAG_CLAMP; }
  *dt = d;
  if (argmax) *argmax = best;
  if (tag) *tag = t;
  if (smax_out) *smax_out = smax;
  return bad ? ORC_E_NONPHYSICAL : ORC_OK;
}

/* ------------------------------------------------------------- 6. one step */

/* One SSP-RK2 step.  U holds U^n on entry (interior; ghosts are refilled
 * here) and U^{n+1} in its interior on return (ghosts keep the U^n fill).
 * mode 0 = telescoped: stage 1 on the box interior+2, no BC on
 *          U1, stage 2 on the interior;
 * mode 1 = refill: stage 1 on the interior, ghost fill of U1, stage 2.
 * U1_out (optional, array shape) receives the stage-1 state on its region.
 * floor_hits (optional) accumulates pressure-floor hits. */
int oracle_step(const oracle_grid* G, double* U, double dt, int32_t mode, double* U1_out,
                int64_t* floor_hits) {
  int rc = check_grid(G);
  if (rc) return rc;
  int64_t n = oracle_array_len(G);
  double* Q = (double*)calloc((size_t)n, sizeof(double));
  double* D = (double*)calloc((size_t)n, sizeof(double));
  double* U1 = (double*)calloc((size_t)n, sizeof(double));
  if (!Q || !D || !U1) { free(Q); free(D); free(U1); return ORC_E_ARG; }
  int64_t hits = 0;
  int bad = 0;

  oracle_fill_ghosts(G, U);
  region all = widen(G, interior(G), G->ng);
  region S1 = (mode == 0) ? widen(G, interior(G), 2) : interior(G);
  region I = interior(G);

  /* stage 1: U1 = U^n - dt*D(U^n) on S1 */
  if (prims_region(G, U, Q, all, &hits)) bad = 1;
  divergence(G, Q, S1, D);
  for (int v = 0; v < 5; v++)
    ORACLE_PAR_FOR
    for (int64_t k = S1.lo[2]; k < S1.hi[2]; k++)
      for (int64_t j = S1.lo[1]; j < S1.hi[1]; j++)
        for (int64_t i = S1.lo[0]; i < S1.hi[0]; i++) {
          int64_t a = at(G, v, i, j, k);
          U1[a] = U[a] - dt * D[a];
        }
  if (mode == 1) oracle_fill_ghosts(G, U1);
  if (U1_out) memcpy(U1_out, U1, (size_t)n * sizeof(double));

  /* stage 2: U^{n+1} = 0.5*(U^n + (U1 - dt*D(U1))) on the interior */
  region S1q = (mode == 0) ? S1 : all;
  memset(Q, 0, (size_t)n * sizeof(double));
  if (prims_region(G, U1, Q, S1q, &hits)) bad = 1;
  divergence(G, Q, I, D);
  for (int v = 0; v < 5; v++)
    ORACLE_PAR_FOR
    for (int64_t k = I.lo[2]; k < I.hi[2]; k++)
      for (int64_t j = I.lo[1]; j < I.hi[1]; j++)
        for (int64_t i = I.lo[0]; i < I.hi[0]; i++) {
          int64_t a = at(G, v, i, j, k);
          U[a] = 0.5 * (U[a] + (U1[a] - dt * D[a]));
        }

  free(Q);
  free(D);
  free(U1);
  if (floor_hits) *floor_hits += hits;
  return bad ? ORC_E_NONPHYSICAL : ORC_OK;
}

/* oracle-omp: thread count of the -fopenmp build (returns the count in use;
 * 1 in the plain build). */
int oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}
