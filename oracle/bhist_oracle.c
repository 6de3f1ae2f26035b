/* bhist_oracle.c — plain, slow, obviously-correct CPU oracle for bulk histogram
 * filling (arXiv 2401.13310, "Lessons Learned Migrating CUDA to SYCL", §3.1).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code
 * with the CUDA path (paper_2401_13310_b200/csrc): no headers, helpers or tables.
 *
 * Compile with: gcc -O2 -fno-fast-math -ffp-contract=off (IEEE binary64, RN).
 *
 * What it computes — PAPER.md:126 (§3.1 "Histogramming Action"): the Fill of a
 * bulk is three steps per event: (1) find the bin from the coordinate, (2)
 * increment that bin by one or by the weight, (3) update the statistics sums.
 *   - fixed axis: bin = 1 + floor(nbins*(coord-minEdge)/(maxEdge-minEdge))
 *     (PAPER.md:126), evaluated in IEEE binary64 with exactly this association
 *     and truncation (reading R2);
 *   - variable axis: binary search (std::lower_bound in ROOT, PAPER.md:126,
 *     thrust::lower_bound on GPU) read as half-open bins
 *     [e_{i-1}, e_i): bin = #edges <= x (reading R1);
 *   - outside the range: dedicated underflow (0) / overflow (nbins+1) bin
 *     (PAPER.md:126); NaN -> overflow (reading R5);
 *   - N-D: "repeating the find bin step per axis", global bin
 *     with axis 0 fastest (reading R9);
 *   - stats: the four 1D sums "of (squared) weights and ... multiplied by the
 *     corresponding coordinate" read as sumw, sumw2, sumwx,
 *     sumwx2 (reading R7), extended per axis + cross terms for Dim>=2
 *     (reading R8), over events whose bins are in range on every axis (R6);
 *   - accumulation: every fill adds to the previous state (include-initial,
 *     PAPER.md:173-174).
 * Every floating-point sum is Neumaier-compensated so that the oracle's own
 * rounding error (~1e-16 relative) is negligible against the 1e-12 tolerance
 * the GPU is held to; alongside each sum the oracle keeps sum|term| (the scale
 * the tolerance is relative to).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- Neumaier sum */
typedef struct { double s, c; } nsum;
static void nadd(nsum *a, double x) {
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
    else a->c += (x - t) + a->s;
    a->s = t;
}
static double nval(const nsum *a) { return a->s + a->c; }

/* ---------------------------------------------------------------- step (1): FindBin */
/* 1 + floor(nbins*(coord-minEdge)/(maxEdge-minEdge)); below range ->
 * underflow 0; "outside" above -> overflow nbins+1 (x == maxEdge included, NaN too). */
int or_find_bin_fixed(int32_t nbins, double xmin, double xmax, double x) {
    if (x < xmin) return 0;
    if (!(x < xmax)) return nbins + 1;
    double q = ((double)nbins * (x - xmin)) / (xmax - xmin);
    return 1 + (int)q;     /* q >= 0: truncation == floor */
}

/* binary search over the edges; bin = number of edges <= x. */
int or_find_bin_variable(int32_t nbins, const double *edges, double x) {
    if (x < edges[0]) return 0;
    if (!(x < edges[nbins])) return nbins + 1;
    /* upper_bound: first index i in [0, nbins] with edges[i] > x */
    int lo = 0, hi = nbins;     /* edges[lo] <= x < edges[hi] */
    while (hi - lo > 1) {
        int mid = lo + (hi - lo) / 2;
        if (edges[mid] <= x) lo = mid; else hi = mid;
    }
    return hi;
}

/* ---------------------------------------------------------------- histogram state */
typedef struct {
    int32_t nbins;
    double xmin, xmax;
    double *edges;          /* NULL for a fixed axis; else nbins+1 values (owned copy) */
} or_axis;

typedef struct {
    int dim;
    or_axis ax[3];
    int64_t G;              /* prod (nbins_a + 2) */
    int K;                  /* number of stats: 4, 7, 11 */
    nsum *content;          /* sum of w per bin (w = 1 for unit fills) */
    nsum *sumw2;            /* sum of w*w per bin */
    double *abs_content;    /* sum of |w| per bin (tolerance scale) */
    nsum stats[11];
    double stats_abs[11];
    int64_t entries;
} or_hist;

static int nstats_of(int dim) { return dim == 1 ? 4 : dim == 2 ? 7 : 11; }

void or_destroy(or_hist *h) {
    if (!h) return;
    for (int a = 0; a < 3; ++a) free(h->ax[a].edges);
    free(h->content); free(h->sumw2); free(h->abs_content);
    free(h);
}

/* edges[a] may be NULL (fixed axis). Returns NULL on invalid input. */
or_hist *or_create(int dim, const int32_t *nbins, const double *xmin, const double *xmax,
                   const double *const *edges) {
    if (dim < 1 || dim > 3) return NULL;
    or_hist *h = (or_hist *)calloc(1, sizeof(or_hist));
    h->dim = dim;
    h->G = 1;
    for (int a = 0; a < dim; ++a) {
        if (nbins[a] < 1) { or_destroy(h); return NULL; }
        h->ax[a].nbins = nbins[a];
        if (edges && edges[a]) {
            h->ax[a].edges = (double *)malloc(sizeof(double) * (nbins[a] + 1));
            memcpy(h->ax[a].edges, edges[a], sizeof(double) * (nbins[a] + 1));
            for (int i = 0; i < nbins[a]; ++i)
                if (!(h->ax[a].edges[i] < h->ax[a].edges[i + 1])) { or_destroy(h); return NULL; }
        } else {
            if (!(xmin[a] < xmax[a])) { or_destroy(h); return NULL; }
            h->ax[a].xmin = xmin[a];
            h->ax[a].xmax = xmax[a];
        }
        h->G *= (int64_t)(nbins[a] + 2);
    }
    h->K = nstats_of(dim);
    h->content = (nsum *)calloc((size_t)h->G, sizeof(nsum));
    h->sumw2 = (nsum *)calloc((size_t)h->G, sizeof(nsum));
    h->abs_content = (double *)calloc((size_t)h->G, sizeof(double));
    if (!h->content || !h->sumw2 || !h->abs_content) { or_destroy(h); return NULL; }
    return h;
}

static int find_bin_axis(const or_axis *ax, double x) {
    return ax->edges ? or_find_bin_variable(ax->nbins, ax->edges, x)
                     : or_find_bin_fixed(ax->nbins, ax->xmin, ax->xmax, x);
}

/* SPEC.md S:77-85 / reading R9: g = b0 + (n0+2)*(b1 + (n1+2)*b2), axis 0 fastest. */
int64_t or_global_bin(const or_hist *h, const int *b) {
    int64_t g = 0;
    for (int a = h->dim - 1; a >= 0; --a) g = g * (h->ax[a].nbins + 2) + b[a];
    return g;
}

/* Per-event global bins (parity/debug). coords[a][i]. */
void or_find_bins(const or_hist *h, int64_t n, const double *const *coords, int32_t *out) {
    int b[3];
    for (int64_t i = 0; i < n; ++i) {
        for (int a = 0; a < h->dim; ++a) b[a] = find_bin_axis(&h->ax[a], coords[a][i]);
        out[i] = (int32_t)or_global_bin(h, b);
    }
}

static void add_stat(or_hist *h, int k, double term) {
    nadd(&h->stats[k], term);
    h->stats_abs[k] += fabs(term);
}

/* PAPER.md:126 three steps, for events 0..n-1 in index order. w == NULL: unit weights. */
void or_fill(or_hist *h, int64_t n, const double *const *coords, const double *w) {
    int b[3];
    double x[3];
    h->entries += n;                                   /* (a8) every event, incl. flow */
    for (int64_t i = 0; i < n; ++i) {
        int inrange = 1;
        for (int a = 0; a < h->dim; ++a) {             /* step (1), per axis */
            x[a] = coords[a][i];
            b[a] = find_bin_axis(&h->ax[a], x[a]);
            if (b[a] < 1 || b[a] > h->ax[a].nbins) inrange = 0;
        }
        int64_t g = or_global_bin(h, b);
        double wi = w ? w[i] : 1.0;
        nadd(&h->content[g], wi);                      /* step (2): bin += w */
        nadd(&h->sumw2[g], wi * wi);                   /*           sumw2 += w^2 */
        h->abs_content[g] += fabs(wi);
        if (!inrange) continue;                        /* reading R6: flow -> no stats */
        /* step (3), ROOT GetStats order: sumw, sumw2, sumwx, sumwx2,
         * [sumwy, sumwy2, sumwxy], [sumwz, sumwz2, sumwxz, sumwyz] */
        add_stat(h, 0, wi);
        add_stat(h, 1, wi * wi);
        add_stat(h, 2, wi * x[0]);
        add_stat(h, 3, (wi * x[0]) * x[0]);
        if (h->dim >= 2) {
            add_stat(h, 4, wi * x[1]);
            add_stat(h, 5, (wi * x[1]) * x[1]);
            add_stat(h, 6, (wi * x[0]) * x[1]);
        }
        if (h->dim == 3) {
            add_stat(h, 7, wi * x[2]);
            add_stat(h, 8, (wi * x[2]) * x[2]);
            add_stat(h, 9, (wi * x[0]) * x[2]);
            add_stat(h, 10, (wi * x[1]) * x[2]);
        }
    }
}

/* Merge b into a (elementwise sum). Returns 0, or -1 on mismatch. */
int or_merge(or_hist *a, const or_hist *b) {
    if (a->dim != b->dim || a->G != b->G) return -1;
    for (int64_t g = 0; g < a->G; ++g) {
        nadd(&a->content[g], b->content[g].s); nadd(&a->content[g], b->content[g].c);
        nadd(&a->sumw2[g], b->sumw2[g].s);     nadd(&a->sumw2[g], b->sumw2[g].c);
        a->abs_content[g] += b->abs_content[g];
    }
    for (int k = 0; k < a->K; ++k) {
        nadd(&a->stats[k], b->stats[k].s); nadd(&a->stats[k], b->stats[k].c);
        a->stats_abs[k] += b->stats_abs[k];
    }
    a->entries += b->entries;
    return 0;
}

/* Readback; any output may be NULL. */
void or_read(const or_hist *h, double *content, double *sumw2, double *abs_content,
             double *stats, double *stats_abs, int64_t *entries) {
    for (int64_t g = 0; g < h->G; ++g) {
        if (content) content[g] = nval(&h->content[g]);
        if (sumw2) sumw2[g] = nval(&h->sumw2[g]);
        if (abs_content) abs_content[g] = h->abs_content[g];
    }
    for (int k = 0; k < h->K; ++k) {
        if (stats) stats[k] = nval(&h->stats[k]);
        if (stats_abs) stats_abs[k] = h->stats_abs[k];
    }
    if (entries) *entries = h->entries;
}

int64_t or_nbins_total(const or_hist *h) { return h->G; }
int or_nstats(const or_hist *h) { return h->K; }
