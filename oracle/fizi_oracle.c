/*
 * oracle/fizi_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously-correct CPU definition of the FIZI + Mouse
 * per-frame pipeline of arXiv 1907.04393 ("contactless human machine
 * interface for driving car"), written from PAPER.md and the ambiguity
 * readings L1-L31 listed in DESIGN.md.  Only tests/, __graft_entry__.smoke()
 * and bench.py (cpu_baseline leg, --impl reference) may load this library.
 * The product path (paper_1907_04393_b200/) never links, imports or calls it,
 * and it shares no code, header, table or constant with the CUDA path.
 *
 * Style: scalar C99, one function per step of the method, in the paper's order
 * and notation; compiled with -O2 -ffp-contract=off (no FMA contraction, no
 * fast-math) so every floating-point result is the correctly-rounded IEEE op
 * sequence written here.
 *
 * Citations: P:<n> = /root/reference/PAPER.md line n, S:<n> = SPEC.md line n.
 *
 * Pins (tests/test_oracle_*.py): every function below is pinned by a closed
 * form, an invariant, a library routine (scipy.ndimage), exact rational
 * arithmetic or a SPEC/paper example -- see DESIGN.md "Oracle pins".
 * Parity unpinned: none.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

/* ------------------------------------------------------------------ types */

typedef struct {                /* the oracle's own parameter struct         */
    uint32_t width, height;
    uint32_t gray_tol_S;        /* §3.1(ii), tolerance S           */
    uint32_t hue_lo_deg;        /* §3.1(iii), alpha_1 (degrees)     */
    uint32_t hue_hi_deg;        /* alpha_2 (degrees)                          */
    uint32_t se_radius;         /* §3.1 P:138-139 structuring element radius */
    uint32_t min_blob_ppm;      /* S:242 small-blob removal (reading L13)     */
    uint32_t luma_target, luma_lo, luma_hi;   /* §3.2 P:163 / S:197         */
    double   gamma_min, gamma_max;
    double   beta;              /* tracker EMA weight (reading L25)    */
    double   dwell_radius_px;
    int64_t  dwell_time_ms, lost_timeout_ms;
} or_params;

typedef struct {                /* the oracle's per-frame record             */
    int64_t  t_ms;
    uint64_t sum_luma;          /* exact sum of 299r+587g+114b               */
    uint32_t mean_luma;
    uint32_t corrected;         /* 1 iff a non-identity LUT was applied      */
    double   gamma;
    uint32_t fg_merged, fg_final;
    uint32_t n_comp_total, n_comp_kept;
    uint32_t blob_area, blob_label;
    uint32_t bbox[4];           /* x_min, y_min, x_max, y_max                 */
    uint64_t sum_x, sum_y;
    double   cx, cy;
    /* tracker outputs (or_track) */
    uint32_t visible, clicked;
    double   px, py;
    int64_t  dwell_ms;
} or_record;

typedef struct {                /* Mouse module state per stream (c1 step 11) */
    int      vis;
    double   px, py;
    int64_t  last_t;
    double   ax, ay;            /* dwell anchor                              */
    int64_t  anchor_t;
    int64_t  dwell;
    int      fired;
} or_tstate;

/* ------------------------------------------------- a1: background learning */
/* §2 P:58 "learns the background without the user", §3.1(i): the
 * minimum and maximum values learned in the initialization step.  S:138: per
 * pixel/channel min over frames minus margin and max plus margin, saturating.
 * Output planes are interleaved RGB like the frame. */
int or_learn(const uint8_t *frames, uint32_t n, uint32_t w, uint32_t h,
             uint32_t margin, uint8_t *lo, uint8_t *hi)
{
    if (n == 0) return -2;                       /* S:139 empty -> error */
    if (w == 0 || h == 0) return -3;
    size_t nb = (size_t)w * h * 3;
    for (size_t i = 0; i < nb; i++) {
        int mn = 255, mx = 0;
        for (uint32_t k = 0; k < n; k++) {
            int v = frames[(size_t)k * nb + i];
            if (v < mn) mn = v;
            if (v > mx) mx = v;
        }
        int l = mn - (int)margin, u = mx + (int)margin;
        lo[i] = (uint8_t)(l < 0 ? 0 : l);
        hi[i] = (uint8_t)(u > 255 ? 255 : u);
    }
    return 0;
}

/* ---------------------------------------------- a2: brightness correction */
/* §2 P:63 "The brightness is also corrected"; §3.2 P:163 a filter modifies
 * the luminosity.  Reading L18/L19: Rec.601 luma, integer mean
 * rounded half up: mean = floor((S1 + 500 N) / (1000 N)). */
uint32_t or_mean_luma(const uint8_t *f, uint32_t w, uint32_t h, uint64_t *sum_out)
{
    uint64_t s = 0, n = (uint64_t)w * h;
    for (uint64_t p = 0; p < n; p++)
        s += 299u * f[3 * p] + 587u * f[3 * p + 1] + 114u * f[3 * p + 2];
    if (sum_out) *sum_out = s;
    return (uint32_t)((s + 500u * n) / (1000u * n));
}

/* Reading L20: gamma = clamp(ln(target/255)/ln(mean/255), gmin, gmax), with
 * the limits mean=0 -> gmin, mean=255 -> gmax; identity inside
 * [luma_lo, luma_hi]. Returns gamma; *corrected = 1 iff not identity. */
double or_gamma(const or_params *p, uint32_t mean, uint32_t *corrected)
{
    if (mean >= p->luma_lo && mean <= p->luma_hi) { *corrected = 0; return 1.0; }
    *corrected = 1;
    if (mean == 0) return p->gamma_min;
    if (mean == 255) return p->gamma_max;
    double g = log((double)p->luma_target / 255.0) / log((double)mean / 255.0);
    if (g < p->gamma_min) g = p->gamma_min;
    if (g > p->gamma_max) g = p->gamma_max;
    return g;
}

/* Reading L21: L[x] = floor(255 (x/255)^gamma + 0.5), in double. */
void or_lut(double gamma, uint8_t lut[256])
{
    for (int x = 0; x < 256; x++) {
        double v = floor(255.0 * pow((double)x / 255.0, gamma) + 0.5);
        if (v < 0) v = 0;
        if (v > 255) v = 255;
        lut[x] = (uint8_t)v;
    }
}

/* ------------------------------------------------ a3: the three branches */
/* §3.1(i), readings L1-L3: a pixel inside the learned envelope on
 * all three channels (inclusive) is background -> 0, otherwise 1. */
int or_r1(const uint8_t v[3], const uint8_t lo[3], const uint8_t hi[3])
{
    for (int c = 0; c < 3; c++)
        if (v[c] < lo[c] || v[c] > hi[c]) return 1;
    return 0;
}

/* §3.1(ii), readings L4/L5: spread C = max - min; "lower than a
 * tolerance S ... eliminated" -> keep iff C >= S. */
int or_r2(const uint8_t v[3], uint32_t S)
{
    int M = v[0], m = v[0];
    for (int c = 1; c < 3; c++) { if (v[c] > M) M = v[c]; if (v[c] < m) m = v[c]; }
    return (uint32_t)(M - m) >= S;
}

/* Hexagonal hue as an exact rational h = Hn / C degrees (reading L8), S:58:
 * M = r: 60 (g-b)/C (mod 360); M = g: 60 (b-r)/C + 120; M = b: 60 (r-g)/C + 240.
 * Returns C; C = 0 means achromatic (reading L9). */
int or_hue_num(const uint8_t v[3], int64_t *Hn)
{
    int r = v[0], g = v[1], b = v[2];
    int M = r, m = r;
    if (g > M) M = g;
    if (b > M) M = b;
    if (g < m) m = g;
    if (b < m) m = b;
    int C = M - m;
    if (C == 0) { *Hn = 0; return 0; }
    if (M == r)      *Hn = 60 * (int64_t)(g - b) + (g < b ? 360 * (int64_t)C : 0);
    else if (M == g) *Hn = 60 * (int64_t)(b - r) + 120 * (int64_t)C;
    else             *Hn = 60 * (int64_t)(r - g) + 240 * (int64_t)C;
    return C;
}

/* §3.1(iii): Hue in [alpha1, alpha2] % 2pi; reading L7: closed ends,
 * alpha1 > alpha2 is a band through 0 degrees.  h = Hn/C, compared by exact
 * cross-multiplication (C > 0). */
int or_in_band(int64_t Hn, int C, uint32_t a1, uint32_t a2)
{
    int64_t lo = (int64_t)a1 * C, hi = (int64_t)a2 * C;
    if (a1 <= a2) return Hn >= lo && Hn <= hi;
    return Hn >= lo || Hn <= hi;
}

int or_r3(const uint8_t v[3], uint32_t a1, uint32_t a2)
{
    int64_t Hn;
    int C = or_hue_num(v, &Hn);
    if (C == 0) return 0;                       /* reading L9 */
    return or_in_band(Hn, C, a1, a2);
}

/* ------------------------------------------------------- a4: morphology */
/* §3.1 P:138-139 "erosion and dilatation"; S:68 / S:76: square SE side 2r+1,
 * out-of-bounds positions count as 0 (zero padding, reading L12). */
void or_erode(const uint8_t *in, uint8_t *out, uint32_t w, uint32_t h, uint32_t r)
{
    for (int y = 0; y < (int)h; y++)
        for (int x = 0; x < (int)w; x++) {
            int all = 1;
            for (int dy = -(int)r; dy <= (int)r && all; dy++)
                for (int dx = -(int)r; dx <= (int)r; dx++) {
                    int xx = x + dx, yy = y + dy;
                    if (xx < 0 || yy < 0 || xx >= (int)w || yy >= (int)h ||
                        !in[(size_t)yy * w + xx]) { all = 0; break; }
                }
            out[(size_t)y * w + x] = (uint8_t)all;
        }
}

void or_dilate(const uint8_t *in, uint8_t *out, uint32_t w, uint32_t h, uint32_t r)
{
    for (int y = 0; y < (int)h; y++)
        for (int x = 0; x < (int)w; x++) {
            int any = 0;
            for (int dy = -(int)r; dy <= (int)r && !any; dy++)
                for (int dx = -(int)r; dx <= (int)r; dx++) {
                    int xx = x + dx, yy = y + dy;
                    if (xx >= 0 && yy >= 0 && xx < (int)w && yy < (int)h &&
                        in[(size_t)yy * w + xx]) { any = 1; break; }
                }
            out[(size_t)y * w + x] = (uint8_t)any;
        }
}

/* Reading L12: opening (E then D) then closing (D then E): O = E(D(D(E(A)))). */
void or_open_close(const uint8_t *in, uint8_t *out, uint32_t w, uint32_t h, uint32_t r)
{
    size_t n = (size_t)w * h;
    uint8_t *t1 = malloc(n ? n : 1), *t2 = malloc(n ? n : 1);
    or_erode(in, t1, w, h, r);
    or_dilate(t1, t2, w, h, r);
    or_dilate(t2, t1, w, h, r);
    or_erode(t1, out, w, h, r);
    free(t1); free(t2);
}

/* ------------------------------------------------ a5: connected components */
/* S:94 / S:110: 8-connectivity.  Reading L15: canonical label = 1 + min raster
 * index of the component: raster scan, the first unlabelled foreground pixel
 * at index i starts a flood fill with label i+1.  Returns #components. */
uint32_t or_label(const uint8_t *m, uint32_t w, uint32_t h, uint32_t *lab)
{
    size_t n = (size_t)w * h;
    memset(lab, 0, n * sizeof(uint32_t));
    size_t *stack = malloc((n ? n : 1) * sizeof(size_t));
    uint32_t count = 0;
    for (size_t i = 0; i < n; i++) {
        if (!m[i] || lab[i]) continue;
        uint32_t L = (uint32_t)i + 1;
        count++;
        size_t sp = 0;
        lab[i] = L;
        stack[sp++] = i;
        while (sp) {
            size_t q = stack[--sp];
            int qx = (int)(q % w), qy = (int)(q / w);
            for (int dy = -1; dy <= 1; dy++)
                for (int dx = -1; dx <= 1; dx++) {
                    int xx = qx + dx, yy = qy + dy;
                    if (xx < 0 || yy < 0 || xx >= (int)w || yy >= (int)h) continue;
                    size_t j = (size_t)yy * w + xx;
                    if (m[j] && !lab[j]) { lab[j] = L; stack[sp++] = j; }
                }
        }
    }
    free(stack);
    return count;
}

/* ------------------------------------------ the whole per-frame definition */
/* Stage outputs (all nullable; u8 {0,1} per pixel except labels u32):
 * r1, r2, r3, merged, oc (open-close), labels, final, contour. */
typedef struct {
    uint8_t *r1, *r2, *r3, *merged, *oc;
    uint32_t *labels;
    uint8_t *final_mask, *contour;
} or_stages;

int or_segment(const or_params *p, const uint8_t *frame, const uint8_t *lo,
               const uint8_t *hi, int64_t t_ms, const or_stages *st, or_record *rec)
{
    uint32_t w = p->width, h = p->height;
    size_t n = (size_t)w * h;
    memset(rec, 0, sizeof(*rec));
    rec->t_ms = t_ms;
    if (n == 0) return -3;

    /* a2 (§3.2): mean luma, gamma, LUT; the corrected frame feeds a3 */
    rec->mean_luma = or_mean_luma(frame, w, h, &rec->sum_luma);
    rec->gamma = or_gamma(p, rec->mean_luma, &rec->corrected);
    uint8_t lut[256];
    if (rec->corrected) or_lut(rec->gamma, lut);
    else for (int x = 0; x < 256; x++) lut[x] = (uint8_t)x;

    /* a3 (§3.1): three branches on the corrected pixel, then the AND merge */
    uint8_t *A = calloc(n ? n : 1, 1);
    for (size_t q = 0; q < n; q++) {
        uint8_t v[3] = { lut[frame[3 * q]], lut[frame[3 * q + 1]], lut[frame[3 * q + 2]] };
        int b1 = or_r1(v, lo + 3 * q, hi + 3 * q);
        int b2 = or_r2(v, p->gray_tol_S);
        int b3 = or_r3(v, p->hue_lo_deg, p->hue_hi_deg);
        if (st && st->r1) st->r1[q] = (uint8_t)b1;
        if (st && st->r2) st->r2[q] = (uint8_t)b2;
        if (st && st->r3) st->r3[q] = (uint8_t)b3;
        A[q] = (uint8_t)(b1 && b2 && b3);       /* P:137 logical AND */
        rec->fg_merged += A[q];
    }
    if (st && st->merged) memcpy(st->merged, A, n);

    /* a4: morphology */
    uint8_t *O = malloc(n ? n : 1);
    or_open_close(A, O, w, h, p->se_radius);
    if (st && st->oc) memcpy(st->oc, O, n);

    /* a5: labelling */
    uint32_t *lab = malloc(n * sizeof(uint32_t));
    rec->n_comp_total = or_label(O, w, h, lab);

    /* a6: per-component area, keep iff area*1e6 >= ppm*N (reading L13) */
    uint64_t *area = calloc(n + 1, sizeof(uint64_t));
    for (size_t q = 0; q < n; q++) if (lab[q]) area[lab[q]]++;
    uint8_t *F = calloc(n ? n : 1, 1);
    for (size_t L = 1; L <= n; L++)
        if (area[L] && area[L] * 1000000ull >= (uint64_t)p->min_blob_ppm * n)
            rec->n_comp_kept++;
    for (size_t q = 0; q < n; q++) {
        uint32_t L = lab[q];
        if (L && area[L] * 1000000ull >= (uint64_t)p->min_blob_ppm * n) {
            F[q] = 1;
            rec->fg_final++;
        }
    }
    if (st && st->labels) memcpy(st->labels, lab, n * sizeof(uint32_t));
    if (st && st->final_mask) memcpy(st->final_mask, F, n);

    /* a7: largest kept component, ties -> smaller label (reading L16) */
    uint32_t best = 0;
    for (size_t L = 1; L <= n; L++) {
        if (!area[L] || area[L] * 1000000ull < (uint64_t)p->min_blob_ppm * n) continue;
        if (!best || area[L] > area[best]) best = (uint32_t)L;
    }
    if (best) {
        rec->blob_label = best;
        rec->blob_area = (uint32_t)area[best];
        rec->bbox[0] = w; rec->bbox[1] = h; rec->bbox[2] = 0; rec->bbox[3] = 0;
        for (size_t q = 0; q < n; q++) {
            if (lab[q] != best) continue;
            uint32_t x = (uint32_t)(q % w), y = (uint32_t)(q / w);
            rec->sum_x += x;
            rec->sum_y += y;
            if (x < rec->bbox[0]) rec->bbox[0] = x;
            if (y < rec->bbox[1]) rec->bbox[1] = y;
            if (x > rec->bbox[2]) rec->bbox[2] = x;
            if (y > rec->bbox[3]) rec->bbox[3] = y;
        }
        /* reading L17: arithmetic mean of integer (col,row), one division */
        rec->cx = (double)rec->sum_x / (double)rec->blob_area;
        rec->cy = (double)rec->sum_y / (double)rec->blob_area;
    }

    /* reading L30: optional inner contour = final AND NOT erode_r1(final) */
    if (st && st->contour) {
        uint8_t *E = malloc(n);
        or_erode(F, E, w, h, 1);
        for (size_t q = 0; q < n; q++) st->contour[q] = (uint8_t)(F[q] && !E[q]);
        free(E);
    }
    free(A); free(O); free(lab); free(area); free(F);
    return 0;
}

/* ------------------------------------------------- a8: the Mouse fold */
/* §2: the hand zone is converted into a pointer with a state
 * (click or not).  Reading L25-L27: EMA with beta, snap on
 * acquisition, visibility timeout (strict >), dwell anchor/radius/time, one
 * click per dwell episode.  Products and sums are separate IEEE operations
 * (compiled with -ffp-contract=off). */
void or_track_init(or_tstate *s) { memset(s, 0, sizeof(*s)); }

void or_track(const or_params *p, or_tstate *s, or_record *rec)
{
    int64_t t = rec->t_ms;
    if (rec->blob_area > 0) {
        double cx = rec->cx, cy = rec->cy;
        if (s->vis) {
            double b = p->beta, ob = 1.0 - p->beta;
            double tx = b * cx, ty = b * cy;
            double ux = ob * s->px, uy = ob * s->py;
            s->px = tx + ux;
            s->py = ty + uy;
            double dx = s->px - s->ax, dy = s->py - s->ay;
            double d2 = dx * dx;
            double e2 = dy * dy;
            d2 = d2 + e2;
            double R2 = p->dwell_radius_px * p->dwell_radius_px;
            if (d2 > R2) {
                s->ax = s->px; s->ay = s->py; s->anchor_t = t;
                s->dwell = 0; s->fired = 0;
            } else {
                s->dwell = t - s->anchor_t;
            }
        } else {
            s->px = cx; s->py = cy;
            s->ax = cx; s->ay = cy; s->anchor_t = t;
            s->dwell = 0; s->fired = 0;
        }
        s->vis = 1;
        s->last_t = t;
    } else {
        if (s->vis && t - s->last_t > p->lost_timeout_ms) {
            s->vis = 0; s->dwell = 0; s->fired = 0;
        } else if (s->vis) {
            s->dwell = t - s->anchor_t;
        }
    }
    int clicked = s->vis && !s->fired && s->dwell >= p->dwell_time_ms;
    if (clicked) s->fired = 1;
    rec->visible = (uint32_t)s->vis;
    rec->clicked = (uint32_t)clicked;
    rec->px = s->px;
    rec->py = s->py;
    rec->dwell_ms = s->dwell;
}

/* ---------------------------------- batch driver (frame-parallel threads) */
/* Used by the cpu_baseline / --impl reference legs: frames are independent
 * given the envelope, so a batch is split over threads; the tracker
 * fold stays sequential (or_track, called by the caller). */
typedef struct {
    const or_params *p;
    const uint8_t *frames, *lo, *hi;
    const int64_t *t_ms;
    or_record *recs;
    uint8_t *masks;
    uint32_t begin, end, stride;
} or_job;

static void *or_worker(void *arg)
{
    or_job *j = (or_job *)arg;
    size_t n = (size_t)j->p->width * j->p->height;
    for (uint32_t i = j->begin; i < j->end; i += j->stride) {
        or_stages st;
        memset(&st, 0, sizeof(st));
        st.final_mask = j->masks ? j->masks + (size_t)i * n : NULL;
        or_segment(j->p, j->frames + (size_t)i * n * 3, j->lo, j->hi,
                   j->t_ms ? j->t_ms[i] : 0, &st, &j->recs[i]);
    }
    return NULL;
}

int or_segment_batch(const or_params *p, const uint8_t *frames, uint32_t nframes,
                     const uint8_t *lo, const uint8_t *hi, const int64_t *t_ms,
                     uint32_t nthreads, or_record *recs, uint8_t *masks)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    or_job jobs[256];
    for (uint32_t k = 0; k < nthreads; k++) {
        jobs[k] = (or_job){ p, frames, lo, hi, t_ms, recs, masks, k, nframes, nthreads };
        if (nthreads == 1) { or_worker(&jobs[k]); return 0; }
        pthread_create(&th[k], NULL, or_worker, &jobs[k]);
    }
    for (uint32_t k = 0; k < nthreads; k++) pthread_join(th[k], NULL);
    return 0;
}

uint32_t or_sizeof_record(void) { return (uint32_t)sizeof(or_record); }
uint32_t or_sizeof_params(void) { return (uint32_t)sizeof(or_params); }
uint32_t or_sizeof_tstate(void) { return (uint32_t)sizeof(or_tstate); }
