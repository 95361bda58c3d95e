/*
 * snp_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * Plain, slow, obviously-correct CPU oracle of the forward splatting rasterizer
 * for splattable neural primitives (arXiv 2510.08491).  Double precision,
 * compiled with -ffp-contract=off.  It shares NO code, header, table or helper
 * with the CUDA path (paper_2510_08491_b200/csrc); neither includes the other.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load it.
 *
 * Citation key: P:n = PAPER.md line n, S:n = SPEC.md line n, R<k> = reading k
 * in DESIGN.md section "Readings of the paper".
 *
 * What it computes, per pixel:
 *   ray     o = C_w, d = normalize(R_wc ((x+.5-cx)/fx, (y+.5-cy)/fy, 1))   (R6)
 *   hit     analytic line-ellipsoid intersection -> [t_in, t_out]
 *   I       closed-form integral of the MLP density over [t_in, t_out]      (Eq. 7-8)
 *   kappa   1 - exp(-max(0, I))                                               (Eq. 9)
 *   colour  real SH, degree <= 3, evaluated at dir = normalize(mu - o)        (R14)
 *   order   ascending (t_in, primitive index) over ALL primitives           (Eq. 4 "depth-sorted", R11)
 *   blend   C += T kappa c ; T *= 1 - kappa ; stop when T < floor            (Eq. 4, R13)
 *   output  RGB = C + T bg, opacity = 1 - T                                   (R16)
 * Every primitive is tested against every pixel: no tiles, no culling beyond an
 * exact bounding-sphere reject.
 *
 * It also holds the FP64 binning definition (DESIGN.md
 * "Binning definition"): per-primitive silhouette bbox -> tile rect, depth
 * lower bound key, key emission, stable sort, tile ranges.
 *
 * Parity pins (tests/test_oracle_*.py, -m "not gpu") check every function here
 * against values the paper/SPEC print, closed forms, brute force and library
 * routines; see DESIGN.md "Oracle pins".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int64_t n;
    int32_t n_hidden;
    int32_t sh_degree;
    double omega;
    const float *centers;    /* [n][3] */
    const float *rotations;  /* [n][4] (w,x,y,z) */
    const float *scales;     /* [n][3] semi-axes */
    const float *w1;         /* [n][N][3] */
    const float *b1;         /* [n][N] */
    const float *w2;         /* [n][N] */
    const float *b2;         /* [n] */
    const float *sh;         /* [n][16][3] */
    const float *w_t;        /* [n][N] temporal weights W_t, or NULL (static scene) */
} orc_scene;

typedef struct {
    double R_wc[9];  /* world-from-camera, row-major */
    double C_w[3];
    double fx, fy, cx, cy;
    int32_t width, height;
    double t_near, t_far;
    double xi_t;     /* timestamp xi_t in [0, 1] of this view (temporal scenes, R24) */
} orc_camera;

/* ------------------------------------------------------------------ geometry */

/* Rotation matrix of the normalised quaternion (w,x,y,z) (R8).
 * Returns 0 on success, -1 for a zero quaternion. */
int orc_quat_to_rot(const double q[4], double R[9])
{
    double nq = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (!(nq > 0.0)) return -1;
    double inq = 1.0 / nq;   /* one division (binning definition) */
    double w = q[0] * inq, x = q[1] * inq, y = q[2] * inq, z = q[3] * inq;
    R[0] = 1.0 - 2.0 * (y * y + z * z);
    R[1] = 2.0 * (x * y - w * z);
    R[2] = 2.0 * (x * z + w * y);
    R[3] = 2.0 * (x * y + w * z);
    R[4] = 1.0 - 2.0 * (x * x + z * z);
    R[5] = 2.0 * (y * z - w * x);
    R[6] = 2.0 * (x * z - w * y);
    R[7] = 2.0 * (y * z + w * x);
    R[8] = 1.0 - 2.0 * (x * x + y * y);
    return 0;
}

/* Pixel ray ("rotated into world frame, direction normalized", R6):
 * o = C_w, d = normalize(R_wc d_cam), d_cam = ((x+.5-cx)/fx, (y+.5-cy)/fy, 1).
 * Normalising AFTER the rotation keeps |d| = 1 even when the fp32 R_wc is not
 * exactly orthonormal. */
void orc_pixel_ray(const orc_camera *cam, double px, double py, double o[3], double d[3])
{
    double dc[3] = {(px + 0.5 - cam->cx) / cam->fx, (py + 0.5 - cam->cy) / cam->fy, 1.0};
    double r[3];
    for (int i = 0; i < 3; ++i) {
        r[i] = cam->R_wc[3 * i + 0] * dc[0] + cam->R_wc[3 * i + 1] * dc[1] + cam->R_wc[3 * i + 2] * dc[2];
        o[i] = cam->C_w[i];
    }
    double nd = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    for (int i = 0; i < 3; ++i) d[i] = r[i] / nd;
}

/* Analytic line-ellipsoid intersection ("analytic line--ellipsoid
 * intersection").  The ray is taken into the unit-sphere frame
 * x_l = diag(1/s) R^T (x - mu) WITHOUT renormalising the direction, the
 * quadratic |b + t a|^2 = 1 is solved with the citardauq form, and the roots
 * are clipped to [t_near, t_far].  disc <= 0 is a miss (R9).
 * qmin (optional) = min_t |b + t a|^2, the ray's closest implicit value, used
 * for the grazing flag.  Returns 1 on a hit with t_out > t_in, else 0. */
int orc_intersect(const double o[3], const double d[3], double t_near, double t_far,
                  const double mu[3], const double R[9], const double s[3],
                  double *t_in, double *t_out, double *qmin)
{
    double v[3] = {o[0] - mu[0], o[1] - mu[1], o[2] - mu[2]};
    double a[3], b[3];
    for (int k = 0; k < 3; ++k) {  /* column k of R is local axis k */
        a[k] = (R[0 * 3 + k] * d[0] + R[1 * 3 + k] * d[1] + R[2 * 3 + k] * d[2]) / s[k];
        b[k] = (R[0 * 3 + k] * v[0] + R[1 * 3 + k] * v[1] + R[2 * 3 + k] * v[2]) / s[k];
    }
    double A = a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
    double B = a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
    double bb = b[0] * b[0] + b[1] * b[1] + b[2] * b[2];
    double C = bb - 1.0;
    if (qmin) *qmin = bb - B * B / A;
    double disc = B * B - A * C;
    if (!(disc > 0.0)) return 0;
    double sq = sqrt(disc);
    double qq = -(B + (B >= 0.0 ? sq : -sq));
    double t0 = qq / A, t1 = C / qq;
    if (t0 > t1) { double tmp = t0; t0 = t1; t1 = tmp; }
    double ti = t0 > t_near ? t0 : t_near;
    double to = t1 < t_far ? t1 : t_far;
    if (!(to > ti)) return 0;
    *t_in = ti;
    *t_out = to;
    return 1;
}

/* ------------------------------------------------------------ density field */

/* Pointwise density, Eq. 5-6: sigma(x) = f((x-mu)/||s||_inf),
 * f(y) = W2 cos(omega (W1 y + b1)) + b2.  Used ONLY by pins: the renderer never
 * evaluates sigma. Caller decides inside/outside. */
double orc_density(const double x[3], const double mu[3], double smax, int N, double omega,
                   const double *W1, const double *b1, const double *W2, double b2)
{
    double y[3] = {(x[0] - mu[0]) / smax, (x[1] - mu[1]) / smax, (x[2] - mu[2]) / smax};
    double f = b2;
    for (int k = 0; k < N; ++k) {
        double z = W1[3 * k] * y[0] + W1[3 * k + 1] * y[1] + W1[3 * k + 2] * y[2] + b1[k];
        f += W2[k] * cos(omega * z);
    }
    return f;
}

/* Eq. 8 literally, difference form with the Eq. 5 normalisation
 * substituted (R2): F(t) = sum_k W2_k/h_k sin(a_k + h_k t) + t b2,
 * a_k = omega (W1_k.o^ + b1_k), h_k = omega W1_k.d^, o^ = (o-mu)/smax,
 * d^ = d/smax; I = F(t_out) - F(t_in).  Singular as h_k -> 0 (R3); pins only. */
double orc_integral_eq8(const double o[3], const double d[3], double t_in, double t_out,
                        const double mu[3], double smax, int N, double omega,
                        const double *W1, const double *b1, const double *W2, double b2)
{
    double oh[3] = {(o[0] - mu[0]) / smax, (o[1] - mu[1]) / smax, (o[2] - mu[2]) / smax};
    double dh[3] = {d[0] / smax, d[1] / smax, d[2] / smax};
    double Fo = t_out * b2, Fi = t_in * b2;
    for (int k = 0; k < N; ++k) {
        double ak = omega * (W1[3 * k] * oh[0] + W1[3 * k + 1] * oh[1] + W1[3 * k + 2] * oh[2] + b1[k]);
        double hk = omega * (W1[3 * k] * dh[0] + W1[3 * k + 1] * dh[1] + W1[3 * k + 2] * dh[2]);
        Fo += W2[k] / hk * sin(ak + hk * t_out);
        Fi += W2[k] / hk * sin(ak + hk * t_in);
    }
    return Fo - Fi;
}

/* The renderer's integral: Eq. 8 evaluated in the equivalent product form
 * (R3): W2_k/h_k [sin(a+h t_out) - sin(a+h t_in)]
 *            = W2_k dt cos(a + h tm) sinc(h dt / 2),   dt = t_out-t_in, tm = mid.
 * Exact identity, finite at h_k = 0. */
double orc_integral(const double o[3], const double d[3], double t_in, double t_out,
                    const double mu[3], double smax, int N, double omega,
                    const double *W1, const double *b1, const double *W2, double b2)
{
    double oh[3] = {(o[0] - mu[0]) / smax, (o[1] - mu[1]) / smax, (o[2] - mu[2]) / smax};
    double dh[3] = {d[0] / smax, d[1] / smax, d[2] / smax};
    double dt = t_out - t_in, tm = 0.5 * (t_in + t_out);
    double I = b2 * dt;
    for (int k = 0; k < N; ++k) {
        double ak = omega * (W1[3 * k] * oh[0] + W1[3 * k + 1] * oh[1] + W1[3 * k + 2] * oh[2] + b1[k]);
        double hk = omega * (W1[3 * k] * dh[0] + W1[3 * k + 1] * dh[1] + W1[3 * k + 2] * dh[2]);
        double x = 0.5 * hk * dt;
        double sinc = (x == 0.0) ? 1.0 : sin(x) / x;
        I += W2[k] * dt * cos(ak + hk * tm) * sinc;
    }
    return I;
}

/* Eq. 9: kappa = 1 - exp(-max(0, I)). */
double orc_kernel(double I)
{
    return 1.0 - exp(-(I > 0.0 ? I : 0.0));
}

/* ------------------------------------------------------------------- colour */

/* Real spherical-harmonics basis, degrees 0..3, Condon-Shortley phase, order
 * m = -l..l within each band (the 3DGS convention the paper adopts, P:286,
 * "Similar to 3DGS"). out[16]. */
void orc_sh_basis(const double dir[3], double out[16])
{
    const double x = dir[0], y = dir[1], z = dir[2];
    const double xx = x * x, yy = y * y, zz = z * z;
    out[0] = 0.28209479177387814;
    out[1] = -0.4886025119029199 * y;
    out[2] = 0.4886025119029199 * z;
    out[3] = -0.4886025119029199 * x;
    out[4] = 1.0925484305920792 * x * y;
    out[5] = -1.0925484305920792 * y * z;
    out[6] = 0.31539156525252005 * (2.0 * zz - xx - yy);
    out[7] = -1.0925484305920792 * x * z;
    out[8] = 0.5462742152960396 * (xx - yy);
    out[9] = -0.5900435899266435 * y * (3.0 * xx - yy);
    out[10] = 2.890611442640554 * x * y * z;
    out[11] = -0.4570457994644658 * y * (4.0 * zz - xx - yy);
    out[12] = 0.3731763325901154 * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    out[13] = -0.4570457994644658 * x * (4.0 * zz - xx - yy);
    out[14] = 1.445305721320277 * z * (xx - yy);
    out[15] = -0.5900435899266435 * x * (xx - 3.0 * yy);
}

/* Colour c = max(0, sum_{l<=deg} Y_lm(dir) sh_lm + 0.5) per channel (R15). */
void orc_sh_color(int degree, const float *sh /* [16][3] */, const double dir[3], double rgb[3])
{
    double Y[16];
    orc_sh_basis(dir, Y);
    int nc = (degree + 1) * (degree + 1);
    for (int c = 0; c < 3; ++c) {
        double acc = 0.0;
        for (int i = 0; i < nc; ++i) acc += Y[i] * (double)sh[3 * i + c];
        acc += 0.5;
        rgb[c] = acc > 0.0 ? acc : 0.0;
    }
}

/* ------------------------------------------------------------------ renderer */

enum { ORC_FLAG_NEAR_TIE = 1, ORC_FLAG_GRAZING = 2, ORC_FLAG_TFLOOR = 4 };

typedef struct {
    double t_in;
    int64_t id;
    double kappa;
    int clipped;
} orc_hit;

typedef struct {
    double mu[3];
    double R[9];
    double s[3];
    double smax;
    double rgb[3];
    double W1[3 * 64], b1[64], W2[64], b2;
} orc_prim;

static int cmp_hit(const void *pa, const void *pb)
{
    const orc_hit *a = (const orc_hit *)pa, *b = (const orc_hit *)pb;
    if (a->t_in < b->t_in) return -1;
    if (a->t_in > b->t_in) return 1;
    return (a->id < b->id) ? -1 : (a->id > b->id);
}

/* Temporal scenes ("augmenting the network's input dimensions", appendix
 * "Dynamic scenes" f(x, xi_t) = W2 cos(W1 x + xi_t W_t + b1) + b2; reading R24): time
 * is a fourth network input, so at the view's timestamp the phase of unit k is
 * omega (W1_k . x^ + xi_t W_t,k + b1_k), i.e. b1_k + xi_t W_t,k takes the place of b1_k. */
static void load_prim(const orc_scene *sc, int64_t i, const double o[3], double xi_t, orc_prim *p)
{
    int N = sc->n_hidden;
    double q[4];
    for (int k = 0; k < 3; ++k) {
        p->mu[k] = sc->centers[3 * i + k];
        p->s[k] = sc->scales[3 * i + k];
    }
    for (int k = 0; k < 4; ++k) q[k] = sc->rotations[4 * i + k];
    orc_quat_to_rot(q, p->R);
    p->smax = p->s[0];
    if (p->s[1] > p->smax) p->smax = p->s[1];
    if (p->s[2] > p->smax) p->smax = p->s[2];
    for (int k = 0; k < 3 * N; ++k) p->W1[k] = sc->w1[(int64_t)3 * N * i + k];
    for (int k = 0; k < N; ++k) {
        p->b1[k] = sc->b1[(int64_t)N * i + k];
        if (sc->w_t) p->b1[k] += xi_t * (double)sc->w_t[(int64_t)N * i + k];
        p->W2[k] = sc->w2[(int64_t)N * i + k];
    }
    p->b2 = sc->b2[i];
    double dir[3] = {p->mu[0] - o[0], p->mu[1] - o[1], p->mu[2] - o[2]};
    double nd = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
    if (nd > 0.0) { dir[0] /= nd; dir[1] /= nd; dir[2] /= nd; }
    else { dir[0] = 0.0; dir[1] = 0.0; dir[2] = 1.0; }
    orc_sh_color(sc->sh_degree, sc->sh + (int64_t)48 * i, dir, p->rgb);
}

/* Validates inputs like the product's create call does. */
int orc_validate(const orc_scene *sc)
{
    if (sc->n < 0 || sc->n_hidden < 1 || sc->n_hidden > 64 || sc->sh_degree < 0 || sc->sh_degree > 3)
        return -1;
    for (int64_t i = 0; i < sc->n; ++i) {
        double qn = 0.0;
        for (int k = 0; k < 4; ++k) qn += (double)sc->rotations[4 * i + k] * sc->rotations[4 * i + k];
        if (!(qn > 0.0)) return -2;
        for (int k = 0; k < 3; ++k)
            if (!(sc->scales[3 * i + k] > 0.0f) || !isfinite(sc->scales[3 * i + k])) return -3;
    }
    return 0;
}

/*
 * Renders the listed pixels.  out_rgba[4*p] = (R, G, B, opacity), flags[p] =
 * OR of ORC_FLAG_*, stats[3*p] = (hit primitives, composited primitives,
 * index of the stopping hit or -1).
 *   near-tie: two consecutive hits in (t_in, id) order, up to and including the
 *             first hit after the stop, with |t_i - t_j| < tie_eps max(1, t_i)
 *             (both clipped to t_near exactly is an exact tie -> not flagged)
 *   grazing:  a primitive with |1 - qmin| < graze_eps (a hit or a near miss) whose
 *             closest approach lies before the stopping depth
 *   T-floor:  a transmittance after a composite with |T/floor - 1| < 1e-3
 * (R23 / SURVEY A23: tie_eps = 1e-7, graze_eps = 1e-5; parity is scored on
 * unflagged pixels; flagged counts are reported.)
 */
/* colour_per_ray = 0: each primitive's colour is its SH at dir = normalize(mu - o), once
 * per primitive and view (R14, the 3DGS convention).  colour_per_ray = 1 (SURVEY §8(f)
 * 2c, the other reading of P:286): the SH is evaluated at the pixel's own unit ray
 * direction d, once per (ray, hit). */
int orc_render_pixels_ex(const orc_scene *sc, const orc_camera *cam, const double bg[3],
                         double t_floor, int64_t npix, const int32_t *px, const int32_t *py,
                         double *out_rgba, int32_t *flags, int32_t *stats, int nthreads,
                         double tie_eps, double graze_eps, int colour_per_ray)
{
    if (orc_validate(sc) != 0) return -1;
    const int64_t n = sc->n;
    const int N = sc->n_hidden;
    orc_prim *prims = (orc_prim *)malloc(sizeof(orc_prim) * (size_t)(n > 0 ? n : 1));
    double *geo = (double *)malloc(sizeof(double) * 4 * (size_t)(n > 0 ? n : 1));
    if (!prims || !geo) { free(prims); free(geo); return -2; }
    for (int64_t i = 0; i < n; ++i) {
        load_prim(sc, i, cam->C_w, cam->xi_t, &prims[i]);
        /* compact copy of (mu, smax) so the reject loop streams 32 B per primitive */
        geo[4 * i + 0] = prims[i].mu[0];
        geo[4 * i + 1] = prims[i].mu[1];
        geo[4 * i + 2] = prims[i].mu[2];
        geo[4 * i + 3] = prims[i].smax;
    }
    int err = 0;
#ifdef _OPENMP
    if (nthreads <= 0) nthreads = omp_get_max_threads();
#pragma omp parallel num_threads(nthreads)
#endif
    {
        int64_t cap = 256;
        orc_hit *hits = (orc_hit *)malloc(sizeof(orc_hit) * cap);
        double *near_t = (double *)malloc(sizeof(double) * cap);
        int64_t ncap = cap;
        if (!hits || !near_t) err = 1;
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 8)
#endif
        for (int64_t p = 0; p < npix; ++p) {
            if (err) continue;
            double o[3], d[3];
            orc_pixel_ray(cam, px[p], py[p], o, d);
            int64_t nh = 0, nnear = 0;
            for (int64_t i = 0; i < n; ++i) {
                const double *G = geo + 4 * i;
                /* exact bounding-sphere reject: distance from mu to the ray line */
                double w[3] = {G[0] - o[0], G[1] - o[1], G[2] - o[2]};
                double tc = w[0] * d[0] + w[1] * d[1] + w[2] * d[2];
                double ww = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
                double dist2 = ww - tc * tc;
                /* (q_min >= dist2 / smax^2: a primitive outside the widened sphere can
                 * be neither a hit nor a near miss inside the grazing window) */
                if (dist2 > G[3] * G[3] * (1.0 + 2.0 * graze_eps + 1e-6) + 1e-12 * ww) continue;
                if (tc + G[3] < cam->t_near || tc - G[3] > cam->t_far) continue;
                const orc_prim *P = &prims[i];
                double ti, to, qmin;
                int hit = orc_intersect(o, d, cam->t_near, cam->t_far, P->mu, P->R, P->s, &ti, &to, &qmin);
                if (fabs(1.0 - qmin) < graze_eps) {
                    if (nnear == ncap) {
                        ncap *= 2;
                        double *nn = (double *)realloc(near_t, sizeof(double) * ncap);
                        if (!nn) { err = 1; break; }
                        near_t = nn;
                    }
                    near_t[nnear++] = tc - P->smax;
                }
                if (!hit) continue;
                double I = orc_integral(o, d, ti, to, P->mu, P->smax, N, sc->omega, P->W1, P->b1, P->W2, P->b2);
                if (nh == cap) {
                    cap *= 2;
                    orc_hit *nhp = (orc_hit *)realloc(hits, sizeof(orc_hit) * cap);
                    if (!nhp) { err = 1; break; }
                    hits = nhp;
                }
                hits[nh].t_in = ti;
                hits[nh].id = i;
                hits[nh].kappa = orc_kernel(I);
                hits[nh].clipped = (ti == cam->t_near);
                ++nh;
            }
            if (err) continue;
            qsort(hits, (size_t)nh, sizeof(orc_hit), cmp_hit);
            double T = 1.0, C[3] = {0.0, 0.0, 0.0};
            int32_t fl = 0;
            int64_t ncomp = 0, stop = -1;
            for (int64_t h = 0; h < nh; ++h) {
                const orc_prim *P = &prims[hits[h].id];
                double k = hits[h].kappa;
                double ray_rgb[3];
                const double *rgb = P->rgb;
                if (colour_per_ray) {
                    orc_sh_color(sc->sh_degree, sc->sh + (int64_t)48 * hits[h].id, d, ray_rgb);
                    rgb = ray_rgb;
                }
                for (int c = 0; c < 3; ++c) C[c] += T * k * rgb[c];
                T *= (1.0 - k);
                ++ncomp;
                if (fabs(T / t_floor - 1.0) < 1e-3) fl |= ORC_FLAG_TFLOOR;
                if (T < t_floor) { stop = h; break; }
            }
            int64_t last = (stop >= 0) ? stop + 1 : nh - 1;
            if (last > nh - 1) last = nh - 1;
            for (int64_t h = 0; h < last; ++h) {
                double g = hits[h + 1].t_in - hits[h].t_in;
                if (hits[h].clipped && hits[h + 1].clipped) continue;
                if (g < tie_eps * fmax(1.0, fabs(hits[h].t_in))) fl |= ORC_FLAG_NEAR_TIE;
            }
            double t_stop = (stop >= 0) ? hits[stop].t_in : INFINITY;
            for (int64_t j = 0; j < nnear; ++j)
                if (near_t[j] <= t_stop) fl |= ORC_FLAG_GRAZING;
            for (int c = 0; c < 3; ++c) out_rgba[4 * p + c] = C[c] + T * bg[c];
            out_rgba[4 * p + 3] = 1.0 - T;
            if (flags) flags[p] = fl;
            if (stats) {
                stats[3 * p + 0] = (int32_t)nh;
                stats[3 * p + 1] = (int32_t)ncomp;
                stats[3 * p + 2] = (int32_t)stop;
            }
        }
        free(hits);
        free(near_t);
    }
    free(prims);
    free(geo);
    return err ? -2 : 0;
}

/* Brute-force hit list of one pixel's ray: every primitive the exact
 * intersection reports, in primitive order (ids, t_in, t_out).  Returns the hit
 * count (written only up to cap). */
int64_t orc_pixel_hits(const orc_scene *sc, const orc_camera *cam, int32_t px, int32_t py,
                       int64_t *ids, double *t_in, double *t_out, int64_t cap)
{
    double o[3], d[3];
    orc_pixel_ray(cam, px, py, o, d);
    int64_t nh = 0;
    for (int64_t i = 0; i < sc->n; ++i) {
        double mu[3], q[4], s[3], R[9], ti, to;
        for (int k = 0; k < 3; ++k) { mu[k] = sc->centers[3 * i + k]; s[k] = sc->scales[3 * i + k]; }
        for (int k = 0; k < 4; ++k) q[k] = sc->rotations[4 * i + k];
        if (orc_quat_to_rot(q, R) != 0) continue;
        if (!orc_intersect(o, d, cam->t_near, cam->t_far, mu, R, s, &ti, &to, NULL)) continue;
        if (nh < cap) { ids[nh] = i; t_in[nh] = ti; t_out[nh] = to; }
        ++nh;
    }
    return nh;
}

int orc_render_pixels(const orc_scene *sc, const orc_camera *cam, const double bg[3],
                      double t_floor, int64_t npix, const int32_t *px, const int32_t *py,
                      double *out_rgba, int32_t *flags, int32_t *stats, int nthreads,
                      double tie_eps, double graze_eps)
{
    return orc_render_pixels_ex(sc, cam, bg, t_floor, npix, px, py, out_rgba, flags, stats, nthreads,
                                tie_eps, graze_eps, 0);
}

/* Full-frame convenience: every pixel in row-major order. */
int orc_render_frame(const orc_scene *sc, const orc_camera *cam, const double bg[3], double t_floor,
                     double *out_rgba, int32_t *flags, int32_t *stats, int nthreads,
                     double tie_eps, double graze_eps)
{
    int64_t W = cam->width, H = cam->height, np = W * H;
    int32_t *px = (int32_t *)malloc(sizeof(int32_t) * (size_t)(np > 0 ? np : 1));
    int32_t *py = (int32_t *)malloc(sizeof(int32_t) * (size_t)(np > 0 ? np : 1));
    if (!px || !py) { free(px); free(py); return -2; }
    for (int64_t y = 0; y < H; ++y)
        for (int64_t x = 0; x < W; ++x) { px[y * W + x] = (int32_t)x; py[y * W + x] = (int32_t)y; }
    int r = orc_render_pixels(sc, cam, bg, t_floor, np, px, py, out_rgba, flags, stats, nthreads,
                              tie_eps, graze_eps);
    free(px);
    free(py);
    return r;
}

/* -------------------------------------------------------------------- binning
 *
 * Binning definition.
 * The paper has no binning (it names no tiles); BASELINE's 16x16 tiles and a
 * depth-lower-bound key are this build's reading (R18, R19).  Defined in FP64
 * with a FIXED operation order and no contraction so that the GPU reproduces
 * it bit for bit.  Every product/sum below is evaluated left to right.
 */

#define ORC_TILE 16
/* depth code in the key: the fp32 bits of L >> 12 (a rounded-down 19-bit float;
 * bit 31 is 0 since L > 0), i.e. the key keeps 11 mantissa bits of L (R19). */
#define ORC_DEPTH_DROP 12
#define ORC_DEPTH_BITS 19
static const double ORC_EPS_PX = 1.0 / 256.0;

static uint32_t orc_f32_bits_round_down(double L)
{
    float f = (float)L;
    if ((double)f > L) f = nextafterf(f, -INFINITY);
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}

/* Returns 1 and fills rect = (tx0, ty0, tx1, ty1) inclusive tile rect,
 * prect = pixel-centre range (px0, py0, px1, py1) and depth = bits of the fp32
 * lower bound L of t_in (rounded toward -inf) when the primitive is visible;
 * returns 0 when culled. */
int orc_bin_one(const double mu[3], const double qin[4], const double s[3], const orc_camera *cam,
                int32_t rect[4], int32_t prect[4], uint32_t *depth, double *Lout)
{
    double R[9];
    if (orc_quat_to_rot(qin, R) != 0) return 0;
    const double *W = cam->R_wc;
    double dx = mu[0] - cam->C_w[0], dy = mu[1] - cam->C_w[1], dz = mu[2] - cam->C_w[2];
    double m[3], Rc[9], S[9];
    for (int j = 0; j < 3; ++j) m[j] = W[0 * 3 + j] * dx + W[1 * 3 + j] * dy + W[2 * 3 + j] * dz;
    for (int j = 0; j < 3; ++j)
        for (int k = 0; k < 3; ++k)
            Rc[3 * j + k] = W[0 * 3 + j] * R[0 * 3 + k] + W[1 * 3 + j] * R[1 * 3 + k] + W[2 * 3 + j] * R[2 * 3 + k];
    double ss0 = s[0] * s[0], ss1 = s[1] * s[1], ss2 = s[2] * s[2];
    for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l)
            S[3 * j + l] = Rc[3 * j + 0] * ss0 * Rc[3 * l + 0] + Rc[3 * j + 1] * ss1 * Rc[3 * l + 1]
                         + Rc[3 * j + 2] * ss2 * Rc[3 * l + 2];
    double sz = sqrt(S[8]);
    double zmin = m[2] - sz, zmax = m[2] + sz;
    if (!(zmax > 0.0)) return 0;
    /* exact frustum side-plane cull: n.m + sqrt(n^T S n) < 0, evaluated without the
       square root as n.m < 0 && (n.m)^2 > n^T S n (binning definition) */
    const double Wd = (double)cam->width, Hd = (double)cam->height;
    const double pn[4][3] = {{cam->fx, 0.0, cam->cx}, {-cam->fx, 0.0, Wd - cam->cx},
                             {0.0, cam->fy, cam->cy}, {0.0, -cam->fy, Hd - cam->cy}};
    for (int k = 0; k < 4; ++k) {
        const double *nn = pn[k];
        double dot = nn[0] * m[0] + nn[1] * m[1] + nn[2] * m[2];
        double quad = nn[0] * (nn[0] * S[0] + nn[1] * S[1] + nn[2] * S[2])
                    + nn[1] * (nn[0] * S[3] + nn[1] * S[4] + nn[2] * S[5])
                    + nn[2] * (nn[0] * S[6] + nn[1] * S[7] + nn[2] * S[8]);
        if (dot < 0.0 && dot * dot > quad) return 0;
    }
    /* silhouette bbox from the tangent planes through the camera centre */
    double xlo = -INFINITY, xhi = INFINITY, ylo = -INFINITY, yhi = INFINITY;
    double a = m[2] * m[2] - S[8];
    if (zmin > 0.0 && a > 0.0) {
        double bx = m[0] * m[2] - S[2];
        double cxq = m[0] * m[0] - S[0];
        double discx = bx * bx - a * cxq;
        if (!(discx > 0.0)) discx = 0.0;
        double rx = sqrt(discx);
        double ia = 1.0 / a;
        xlo = cam->fx * ((bx - rx) * ia) + cam->cx;
        xhi = cam->fx * ((bx + rx) * ia) + cam->cx;
        double by = m[1] * m[2] - S[5];
        double cyq = m[1] * m[1] - S[4];
        double discy = by * by - a * cyq;
        if (!(discy > 0.0)) discy = 0.0;
        double ry = sqrt(discy);
        ylo = cam->fy * ((by - ry) * ia) + cam->cy;
        yhi = cam->fy * ((by + ry) * ia) + cam->cy;
    }
    double px0 = ceil(xlo - 0.5 - ORC_EPS_PX), px1 = floor(xhi - 0.5 + ORC_EPS_PX);
    double py0 = ceil(ylo - 0.5 - ORC_EPS_PX), py1 = floor(yhi - 0.5 + ORC_EPS_PX);
    if (px0 < 0.0) px0 = 0.0;
    if (py0 < 0.0) py0 = 0.0;
    if (px1 > Wd - 1.0) px1 = Wd - 1.0;
    if (py1 > Hd - 1.0) py1 = Hd - 1.0;
    if (!(px0 <= px1) || !(py0 <= py1)) return 0;
    prect[0] = (int32_t)px0; prect[1] = (int32_t)py0; prect[2] = (int32_t)px1; prect[3] = (int32_t)py1;
    rect[0] = prect[0] / ORC_TILE; rect[1] = prect[1] / ORC_TILE;
    rect[2] = prect[2] / ORC_TILE; rect[3] = prect[3] / ORC_TILE;
    /* depth lower bound L <= t_in of every ray (R19): t_in >= t_near, t_in >= z_min, and */
    double L = cam->t_near;
    /* t >= u.x >= u.m - sqrt(u^T S u) for u = m/|m| (support function of E) */
    double nm = sqrt(m[0] * m[0] + m[1] * m[1] + m[2] * m[2]);
    double mSm = m[0] * (m[0] * S[0] + m[1] * S[1] + m[2] * S[2])
               + m[1] * (m[0] * S[3] + m[1] * S[4] + m[2] * S[5])
               + m[2] * (m[0] * S[6] + m[1] * S[7] + m[2] * S[8]);
    if (nm > 0.0 && mSm >= 0.0) {
        double l1 = nm - sqrt(mSm) / nm;
        if (l1 > L) L = l1;
    }
    if (zmin > L) L = zmin;
    *depth = orc_f32_bits_round_down(L);
    if (Lout) *Lout = L;
    return 1;
}

/* Per-primitive binning of one view.  rects[4*i] = tile rect or (-1,-1,-1,-1)
 * when culled; prects likewise in pixel centres; depth[i] = key bits. */
int orc_bin_view(const orc_scene *sc, const orc_camera *cam, int32_t *rects, int32_t *prects,
                 uint32_t *depth)
{
    for (int64_t i = 0; i < sc->n; ++i) {
        double mu[3], q[4], s[3];
        for (int k = 0; k < 3; ++k) { mu[k] = sc->centers[3 * i + k]; s[k] = sc->scales[3 * i + k]; }
        for (int k = 0; k < 4; ++k) q[k] = sc->rotations[4 * i + k];
        int32_t r[4], pr[4];
        uint32_t dep = 0;
        if (orc_bin_one(mu, q, s, cam, r, pr, &dep, NULL)) {
            memcpy(rects + 4 * i, r, sizeof r);
            if (prects) memcpy(prects + 4 * i, pr, sizeof pr);
            depth[i] = dep;
        } else {
            for (int k = 0; k < 4; ++k) { rects[4 * i + k] = -1; if (prects) prects[4 * i + k] = -1; }
            depth[i] = 0;
        }
    }
    return 0;
}

int orc_tile_bits(int64_t n_tiles)
{
    int b = 0;
    while (((int64_t)1 << b) < n_tiles) ++b;
    return b;
}

static int orc_row_in_stripe(int32_t r, int32_t begin, int32_t stride)
{
    return r >= begin && ((r - begin) % stride) == 0;
}

typedef struct { uint64_t key; uint32_t id; int64_t seq; } orc_kv;

static int cmp_kv(const void *pa, const void *pb)
{
    const orc_kv *a = (const orc_kv *)pa, *b = (const orc_kv *)pb;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return (a->seq < b->seq) ? -1 : (a->seq > b->seq);  /* stable */
}

/*
 * Key emission + stable sort + tile ranges over n_views views (rects/depth
 * are [n_views][n][...]).  Emission order: view, then primitive index, then
 * tile rows (only rows of the stripe), then columns; key = view << (tb+19) |
 * tile << 19 | (depth >> 12), value = primitive index; stable sort by key; ranges[2*(v*T+t)]
 * = [begin, end) of (view v, tile t) in the sorted list, (0,0) when empty.
 * Returns N_dup; writes keys/ids/ranges only if N_dup <= capacity.
 */
int64_t orc_bin_sort(int64_t n, int32_t n_views, const int32_t *rects, const uint32_t *depth,
                     int32_t tiles_x, int32_t tiles_y, int32_t row_begin, int32_t row_stride,
                     uint64_t *keys, uint32_t *ids, int64_t capacity, uint32_t *ranges)
{
    const int64_t T = (int64_t)tiles_x * tiles_y;
    const int tb = orc_tile_bits(T);
    int64_t ndup = 0;
    for (int32_t v = 0; v < n_views; ++v)
        for (int64_t i = 0; i < n; ++i) {
            const int32_t *r = rects + 4 * ((int64_t)v * n + i);
            if (r[0] < 0) continue;
            int64_t rows = 0;
            for (int32_t y = r[1]; y <= r[3]; ++y) rows += orc_row_in_stripe(y, row_begin, row_stride);
            ndup += rows * (int64_t)(r[2] - r[0] + 1);
        }
    if (ndup > capacity) return ndup;
    orc_kv *kv = (orc_kv *)malloc(sizeof(orc_kv) * (size_t)(ndup > 0 ? ndup : 1));
    if (!kv) return -1;
    int64_t e = 0;
    for (int32_t v = 0; v < n_views; ++v)
        for (int64_t i = 0; i < n; ++i) {
            const int32_t *r = rects + 4 * ((int64_t)v * n + i);
            if (r[0] < 0) continue;
            for (int32_t y = r[1]; y <= r[3]; ++y) {
                if (!orc_row_in_stripe(y, row_begin, row_stride)) continue;
                for (int32_t x = r[0]; x <= r[2]; ++x) {
                    uint64_t tile = (uint64_t)y * (uint64_t)tiles_x + (uint64_t)x;
                    kv[e].key = ((uint64_t)v << (tb + ORC_DEPTH_BITS)) | (tile << ORC_DEPTH_BITS)
                               | (uint64_t)(depth[(int64_t)v * n + i] >> ORC_DEPTH_DROP);
                    kv[e].id = (uint32_t)i;
                    kv[e].seq = e;
                    ++e;
                }
            }
        }
    qsort(kv, (size_t)ndup, sizeof(orc_kv), cmp_kv);
    for (int64_t k = 0; k < 2 * T * n_views; ++k) ranges[k] = 0;
    for (int64_t k = 0; k < ndup; ++k) {
        keys[k] = kv[k].key;
        ids[k] = kv[k].id;
        uint64_t vt = kv[k].key >> ORC_DEPTH_BITS;  /* view << tb | tile */
        uint64_t v = vt >> tb, t = vt & (((uint64_t)1 << tb) - 1);
        uint64_t slot = v * (uint64_t)T + t;
        if (k == 0 || (keys[k - 1] >> ORC_DEPTH_BITS) != vt) ranges[2 * slot] = (uint32_t)k;
        ranges[2 * slot + 1] = (uint32_t)(k + 1);
    }
    free(kv);
    return ndup;
}
