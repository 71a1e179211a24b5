/*
 * svlf_oracle.c -- CPU restatement of the SVLF render/train path.
 *
 * TEST INFRASTRUCTURE (see svlf_oracle.h). Every function cites the
 * reference code it restates; paths are relative to /root/reference/proj/.
 * Compiled with -ffp-contract=off: each double/float expression is evaluated
 * with the reference's operand order and no fused multiply-add, which makes
 * it bit-identical to the reference built with -ffp-contract=off
 * (oracle/_ref/libsvlf_ref_nofma.so) for all geometry.
 */
#define _GNU_SOURCE
#include "svlf_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static __thread char g_err[256];
static void set_err(const char* m) { snprintf(g_err, sizeof g_err, "%s", m); }
const char* or_last_error(void) { return g_err; }

/* ======================================================================
 * rng -- include/svlf/rng.hpp:9-50 (splitmix64 + std::mt19937_64)
 * ==================================================================== */
static uint64_t mix64(uint64_t x) { /* rng.hpp:9-14 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

typedef struct {
    uint64_t seed;
    uint64_t mt[312];
    int mti;
} rng_t;

static void rng_init(rng_t* r, uint64_t seed) { /* Rng(seed): engine_(mix64(seed)) rng.hpp:21 */
    r->seed = seed;
    r->mt[0] = mix64(seed);
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->mti = 312;
}

static uint64_t rng_u64(rng_t* r) { /* std::mt19937_64 (w=64,n=312,m=156,r=31) */
    static const uint64_t A = 0xB5026F5AA96619E9ULL, UM = 0xFFFFFFFF80000000ULL,
                          LM = 0x7FFFFFFFULL;
    if (r->mti >= 312) {
        int i;
        uint64_t x;
        for (i = 0; i < 312 - 156; ++i) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
        }
        for (; i < 311; ++i) {
            x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
        }
        x = (r->mt[311] & UM) | (r->mt[0] & LM);
        r->mt[311] = r->mt[155] ^ (x >> 1) ^ ((x & 1ULL) ? A : 0ULL);
        r->mti = 0;
    }
    uint64_t x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

static double rng_uniform(rng_t* r) { /* rng.hpp:26 */
    return (double)(rng_u64(r) >> 11) * 0x1.0p-53;
}
static double rng_uniform_in(rng_t* r, double lo, double hi) { /* rng.hpp:28 */
    return lo + (hi - lo) * rng_uniform(r);
}
static void rng_sub(const rng_t* r, uint64_t id, rng_t* out) { /* rng.hpp:34 */
    rng_init(out, r->seed ^ mix64(id + 0x51ed2700ULL));
}

uint64_t or_rng_u64_first(uint64_t seed) {
    rng_t r;
    rng_init(&r, seed);
    return rng_u64(&r);
}

void or_rng_uniform_stream(uint64_t seed, size_t n, double* out) {
    rng_t r;
    rng_init(&r, seed);
    for (size_t i = 0; i < n; ++i) out[i] = rng_uniform(&r);
}

/* ======================================================================
 * vec3 / geometry -- include/svlf/geometry.hpp:11-80, src/geometry.cpp:5-26
 * ==================================================================== */
typedef struct {
    double x, y, z;
} v3;
static v3 V(double x, double y, double z) {
    v3 r = {x, y, z};
    return r;
}
static v3 vadd(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 vsub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 vmul(v3 a, double s) { return V(a.x * s, a.y * s, a.z * s); }
static v3 vdiv(v3 a, double s) { return V(a.x / s, a.y / s, a.z / s); }
static double vdot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 vcross(v3 a, v3 b) {
    return V(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static double vnorm(v3 v) { return sqrt(vdot(v, v)); }
static v3 vnormalized(v3 v) { return vdiv(v, vnorm(v)); }
static double vget(v3 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }

typedef struct {
    v3 o, d;
} ray_t;
static v3 ray_at(const ray_t* r, double t) { return vadd(r->o, vmul(r->d, t)); } /* geometry.hpp:56 */

typedef struct {
    v3 lo, hi;
} aabb_t;

static int box_contains(const aabb_t* b, v3 p, double s) { /* geometry.hpp:64-67 */
    return p.x >= b->lo.x - s && p.x <= b->hi.x + s && p.y >= b->lo.y - s &&
           p.y <= b->hi.y + s && p.z >= b->lo.z - s && p.z <= b->hi.z + s;
}

/* src/geometry.cpp:5-26: slab test clipped to t >= 0 */
static int ray_aabb(const ray_t* ray, const aabb_t* box, double* t0o, double* t1o) {
    double t0 = 0.0, t1 = INFINITY;
    for (int axis = 0; axis < 3; ++axis) {
        const double o = vget(ray->o, axis), d = vget(ray->d, axis);
        const double lo = vget(box->lo, axis), hi = vget(box->hi, axis);
        if (d == 0.0) {
            if (o < lo || o > hi) return 0;
            continue;
        }
        const double inv = 1.0 / d;
        double ta = (lo - o) * inv;
        double tb = (hi - o) * inv;
        if (ta > tb) {
            const double tmp = ta;
            ta = tb;
            tb = tmp;
        }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
        if (t1 < t0) return 0;
    }
    *t0o = t0;
    *t1o = t1;
    return 1;
}

int or_ray_aabb(const double* r6, const double* lo, const double* hi, double* t01) {
    ray_t r = {V(r6[0], r6[1], r6[2]), V(r6[3], r6[4], r6[5])};
    aabb_t b = {V(lo[0], lo[1], lo[2]), V(hi[0], hi[1], hi[2])};
    return ray_aabb(&r, &b, &t01[0], &t01[1]);
}

/* ======================================================================
 * morton -- include/svlf/morton.hpp:9-37
 * ==================================================================== */
static uint64_t morton_spread(uint64_t v) {
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffULL;
    v = (v | v << 16) & 0x1f0000ff0000ffULL;
    v = (v | v << 8) & 0x100f00f00f00f00fULL;
    v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
    v = (v | v << 2) & 0x1249249249249249ULL;
    return v;
}
static uint64_t morton_encode(uint32_t x, uint32_t y, uint32_t z) {
    return morton_spread(x) | (morton_spread(y) << 1) | (morton_spread(z) << 2);
}
static uint64_t morton_compact(uint64_t v) {
    v &= 0x1249249249249249ULL;
    v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ULL;
    v = (v ^ (v >> 4)) & 0x100f00f00f00f00fULL;
    v = (v ^ (v >> 8)) & 0x1f0000ff0000ffULL;
    v = (v ^ (v >> 16)) & 0x1f00000000ffffULL;
    v = (v ^ (v >> 32)) & 0x1fffff;
    return v;
}
static void morton_decode(uint64_t c, uint32_t* x, uint32_t* y, uint32_t* z) {
    *x = (uint32_t)morton_compact(c);
    *y = (uint32_t)morton_compact(c >> 1);
    *z = (uint32_t)morton_compact(c >> 2);
}

/* ======================================================================
 * octree -- include/svlf/octree.hpp:39-94, src/octree.cpp:14-235
 * ==================================================================== */
struct or_tree {
    uint32_t res, dilation;
    aabb_t box;
    int leaf_level;
    double cell; /* extent / res */
    uint64_t** levels;
    size_t* level_n;
    uint32_t* corner_ids;
    uint32_t vertex_count;
    size_t dropped;
};

static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}
static size_t sort_unique(uint64_t* v, size_t n) {
    if (!n) return 0;
    qsort(v, n, sizeof(uint64_t), cmp_u64);
    size_t k = 1;
    for (size_t i = 1; i < n; ++i)
        if (v[i] != v[k - 1]) v[k++] = v[i];
    return k;
}
static size_t lower_bound_u64(const uint64_t* v, size_t n, uint64_t key) {
    size_t lo = 0, hi = n;
    while (lo < hi) {
        const size_t mid = lo + (hi - lo) / 2;
        if (v[mid] < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

/* GridConfig::validate, src/octree.cpp:20-28 */
static int grid_validate(uint32_t res, const aabb_t* box) {
    if (!(res >= 2 && (res & (res - 1)) == 0)) {
        set_err("resolution must be a power of two >= 2");
        return 0;
    }
    const v3 ext = vsub(box->hi, box->lo);
    if (ext.x <= 0 || ext.y <= 0 || ext.z <= 0) {
        set_err("scene_aabb must have positive extent");
        return 0;
    }
    const double mx = fmax(ext.x, fmax(ext.y, ext.z));
    const double tol = 1e-12 * mx;
    if (fabs(ext.x - ext.y) > tol || fabs(ext.x - ext.z) > tol) {
        set_err("scene_aabb must be a cube");
        return 0;
    }
    return 1;
}

/* finalize_from_leaves, src/octree.cpp:108-142 */
static void tree_finalize(or_tree* t) {
    for (int level = t->leaf_level; level > 0; --level) {
        const size_t n = t->level_n[level];
        uint64_t* p = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
        size_t k = 0;
        for (size_t i = 0; i < n; ++i) {
            const uint64_t c = t->levels[level][i] >> 3;
            if (k == 0 || p[k - 1] != c) p[k++] = c;
        }
        t->levels[level - 1] = p;
        t->level_n[level - 1] = k;
    }
    const uint64_t lat = (uint64_t)t->res + 1;
    const size_t L = t->level_n[t->leaf_level];
    uint64_t* keys = (uint64_t*)malloc(L * 8 * sizeof(uint64_t));
    for (size_t i = 0; i < L; ++i) {
        uint32_t x, y, z;
        morton_decode(t->levels[t->leaf_level][i], &x, &y, &z);
        for (uint32_t b = 0; b < 8; ++b) {
            const uint64_t cx = x + (b & 1), cy = y + ((b >> 1) & 1), cz = z + ((b >> 2) & 1);
            keys[i * 8 + b] = (cz * lat + cy) * lat + cx;
        }
    }
    uint64_t* uniq = (uint64_t*)malloc(L * 8 * sizeof(uint64_t));
    memcpy(uniq, keys, L * 8 * sizeof(uint64_t));
    const size_t nu = sort_unique(uniq, L * 8);
    t->vertex_count = (uint32_t)nu;
    t->corner_ids = (uint32_t*)malloc(L * 8 * sizeof(uint32_t));
    for (size_t i = 0; i < L * 8; ++i) t->corner_ids[i] = (uint32_t)lower_bound_u64(uniq, nu, keys[i]);
    free(keys);
    free(uniq);
}

static or_tree* tree_alloc(uint32_t res, uint32_t dil, const double* lo, const double* hi) {
    aabb_t box = {V(0, 0, 0), V(1, 1, 1)};
    if (lo && hi) {
        box.lo = V(lo[0], lo[1], lo[2]);
        box.hi = V(hi[0], hi[1], hi[2]);
    }
    if (!grid_validate(res, &box)) return NULL;
    or_tree* t = (or_tree*)calloc(1, sizeof(or_tree));
    t->res = res;
    t->dilation = dil;
    t->box = box;
    t->leaf_level = __builtin_ctz(res);
    t->cell = (box.hi.x - box.lo.x) / res;
    t->levels = (uint64_t**)calloc(t->leaf_level + 1, sizeof(uint64_t*));
    t->level_n = (size_t*)calloc(t->leaf_level + 1, sizeof(size_t));
    return t;
}

/* SparseOctree::build, src/octree.cpp:30-89 */
or_tree* or_tree_build(const double* pts, size_t n, uint32_t res, uint32_t dil, const double* lo,
                       const double* hi) {
    or_tree* t = tree_alloc(res, dil, lo, hi);
    if (!t) return NULL;
    const v3 blo = t->box.lo;
    const double h = (t->box.hi.x - t->box.lo.x) / res;
    uint64_t* cells = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    size_t nc = 0, dropped = 0;
    for (size_t i = 0; i < n; ++i) {
        const v3 p = V(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
        if (!box_contains(&t->box, p, 0.0)) {
            ++dropped;
            continue;
        }
        uint32_t ix = (uint32_t)((p.x - blo.x) / h), iy = (uint32_t)((p.y - blo.y) / h),
                 iz = (uint32_t)((p.z - blo.z) / h);
        if (ix > res - 1) ix = res - 1;
        if (iy > res - 1) iy = res - 1;
        if (iz > res - 1) iz = res - 1;
        cells[nc++] = morton_encode(ix, iy, iz);
    }
    if (nc == 0) {
        free(cells);
        or_tree_free(t);
        set_err("empty occupancy");
        return NULL;
    }
    nc = sort_unique(cells, nc);
    if (dil > 0) {
        const int r = (int)dil, w = 2 * r + 1;
        uint64_t* d = (uint64_t*)malloc(nc * (size_t)(w * w * w) * sizeof(uint64_t));
        size_t nd = 0;
        for (size_t i = 0; i < nc; ++i) {
            uint32_t x, y, z;
            morton_decode(cells[i], &x, &y, &z);
            for (int dz = -r; dz <= r; ++dz)
                for (int dy = -r; dy <= r; ++dy)
                    for (int dx = -r; dx <= r; ++dx) {
                        const int nx = (int)x + dx, ny = (int)y + dy, nz = (int)z + dz;
                        if (nx < 0 || ny < 0 || nz < 0 || nx >= (int)res || ny >= (int)res ||
                            nz >= (int)res)
                            continue;
                        d[nd++] = morton_encode(nx, ny, nz);
                    }
        }
        free(cells);
        cells = d;
        nc = sort_unique(cells, nd);
    }
    t->dropped = dropped;
    t->levels[t->leaf_level] = cells;
    t->level_n[t->leaf_level] = nc;
    tree_finalize(t);
    return t;
}

/* SparseOctree::from_leaves, src/octree.cpp:91-105 */
or_tree* or_tree_from_leaves(const uint64_t* codes, size_t n, uint32_t res, uint32_t dil,
                             const double* lo, const double* hi) {
    or_tree* t = tree_alloc(res, dil, lo, hi);
    if (!t) return NULL;
    if (n == 0) {
        or_tree_free(t);
        set_err("empty occupancy");
        return NULL;
    }
    uint64_t* c = (uint64_t*)malloc(n * sizeof(uint64_t));
    memcpy(c, codes, n * sizeof(uint64_t));
    t->levels[t->leaf_level] = c;
    t->level_n[t->leaf_level] = sort_unique(c, n);
    tree_finalize(t);
    return t;
}

void or_tree_free(or_tree* t) {
    if (!t) return;
    for (int l = 0; l <= t->leaf_level; ++l) free(t->levels[l]);
    free(t->levels);
    free(t->level_n);
    free(t->corner_ids);
    free(t);
}
int or_tree_leaf_level(const or_tree* t) { return t->leaf_level; }
size_t or_tree_level_size(const or_tree* t, int l) { return t->level_n[l]; }
const uint64_t* or_tree_level_codes(const or_tree* t, int l) { return t->levels[l]; }
const uint32_t* or_tree_corner_ids(const or_tree* t) { return t->corner_ids; }
uint32_t or_tree_vertex_count(const or_tree* t) { return t->vertex_count; }
size_t or_tree_dropped(const or_tree* t) { return t->dropped; }

/* voxel_aabb, src/octree.cpp:144-152 */
static aabb_t voxel_aabb(const or_tree* t, uint64_t id) {
    uint32_t x, y, z;
    morton_decode(id, &x, &y, &z);
    const v3 lo = t->box.lo;
    const double c = t->cell;
    aabb_t b = {V(lo.x + x * c, lo.y + y * c, lo.z + z * c),
                V(lo.x + (x + 1) * c, lo.y + (y + 1) * c, lo.z + (z + 1) * c)};
    return b;
}

/* leaf_index, src/octree.cpp:158-163 */
static long leaf_index(const or_tree* t, uint64_t id) {
    const uint64_t* L = t->levels[t->leaf_level];
    const size_t n = t->level_n[t->leaf_level];
    const size_t i = lower_bound_u64(L, n, id);
    if (i == n || L[i] != id) return -1;
    return (long)i;
}

/* locate, src/octree.cpp:173-183 */
static int locate(const or_tree* t, v3 p, uint64_t* out) {
    if (!box_contains(&t->box, p, 0.0)) return 0;
    const uint32_t res = t->res;
    const v3 lo = t->box.lo;
    uint32_t ix = (uint32_t)((p.x - lo.x) / t->cell), iy = (uint32_t)((p.y - lo.y) / t->cell),
             iz = (uint32_t)((p.z - lo.z) / t->cell);
    if (ix > res - 1) ix = res - 1;
    if (iy > res - 1) iy = res - 1;
    if (iz > res - 1) iz = res - 1;
    const uint64_t code = morton_encode(ix, iy, iz);
    if (leaf_index(t, code) < 0) return 0;
    *out = code;
    return 1;
}
int or_tree_locate(const or_tree* t, const double* p, uint64_t* code) {
    return locate(t, V(p[0], p[1], p[2]), code);
}

typedef struct {
    uint64_t id;
    double tin, tout;
    v3 x1, x2;
} hit_t;

static int cmp_hit(const void* a, const void* b) { /* src/octree.cpp:230-234 */
    const hit_t* x = (const hit_t*)a;
    const hit_t* y = (const hit_t*)b;
    if (x->tin != y->tin) return x->tin < y->tin ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id ? 1 : 0);
}

typedef struct {
    hit_t* v;
    size_t n, cap;
} hitvec;
static void hv_push(hitvec* h, hit_t x) {
    if (h->n == h->cap) {
        h->cap = h->cap ? 2 * h->cap : 64;
        h->v = (hit_t*)realloc(h->v, h->cap * sizeof(hit_t));
    }
    h->v[h->n++] = x;
}

/* SparseOctree::traverse, src/octree.cpp:192-235: DFS from the root, a
 * child is tested only when its parent box is hit; leaves kept iff
 * t1 - t0 > 1e-12; final sort by (t_in, code). */
/* ray_aabb calls made by traverse (the reference's per-node box tests), for the
 * GPU node-test counter's parity test */
static __thread uint64_t g_node_tests;
uint64_t or_node_tests(int reset) {
    const uint64_t v = g_node_tests;
    if (reset) g_node_tests = 0;
    return v;
}

static void traverse(const or_tree* t, const ray_t* ray, hitvec* out) {
    const size_t first = out->n;
    const int L = t->leaf_level;
    const size_t cap = 8 * (size_t)(L + 1) + 8;
    int* st_level = (int*)malloc(cap * sizeof(int));
    uint64_t* st_code = (uint64_t*)malloc(cap * sizeof(uint64_t));
    size_t sp = 0;
    st_level[sp] = 0;
    st_code[sp] = 0;
    ++sp;
    const double extent = t->box.hi.x - t->box.lo.x;
    const v3 lo = t->box.lo;
    while (sp) {
        --sp;
        const int level = st_level[sp];
        const uint64_t code = st_code[sp];
        const double cell = extent / (1u << level);
        uint32_t x, y, z;
        morton_decode(code, &x, &y, &z);
        aabb_t box = {V(lo.x + x * cell, lo.y + y * cell, lo.z + z * cell),
                      V(lo.x + (x + 1) * cell, lo.y + (y + 1) * cell, lo.z + (z + 1) * cell)};
        double t0, t1;
        ++g_node_tests;
        if (!ray_aabb(ray, &box, &t0, &t1)) continue;
        if (level == L) {
            if (t1 - t0 > 1e-12) {
                hit_t h = {code, t0, t1, ray_at(ray, t0), ray_at(ray, t1)};
                hv_push(out, h);
            }
            continue;
        }
        const uint64_t* next = t->levels[level + 1];
        const size_t nn = t->level_n[level + 1];
        const uint64_t fc = code << 3;
        for (size_t i = lower_bound_u64(next, nn, fc); i < nn && next[i] < fc + 8; ++i) {
            st_level[sp] = level + 1;
            st_code[sp] = next[i];
            ++sp;
        }
    }
    free(st_level);
    free(st_code);
    qsort(out->v + first, out->n - first, sizeof(hit_t), cmp_hit);
}

size_t or_traverse(const or_tree* t, const double* rays, size_t n, uint64_t* offsets, size_t cap,
                   uint64_t* ids, double* tin, double* tout) {
    hitvec hv = {0};
    offsets[0] = 0;
    for (size_t i = 0; i < n; ++i) {
        ray_t r = {V(rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]),
                   V(rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5])};
        traverse(t, &r, &hv);
        offsets[i + 1] = hv.n;
    }
    if (hv.n <= cap) {
        for (size_t j = 0; j < hv.n; ++j) {
            ids[j] = hv.v[j].id;
            tin[j] = hv.v[j].tin;
            tout[j] = hv.v[j].tout;
        }
    }
    const size_t total = hv.n;
    free(hv.v);
    return total;
}

/* random_ray, tests/test_octree.cpp:50-64: half from a radius-2 sphere around
 * the cube center, half from inside the cube; target uniform in the cube. */
void or_random_rays(uint64_t seed, size_t n, double* out) {
    rng_t r;
    rng_init(&r, seed);
    for (size_t i = 0; i < n; ++i) {
        v3 origin, target;
        if (rng_uniform(&r) < 0.5) {
            const double az = rng_uniform_in(&r, 0, 2 * M_PI);
            const double el = rng_uniform_in(&r, -M_PI / 2, M_PI / 2);
            origin = vadd(V(0.5, 0.5, 0.5), vmul(V(cos(az) * cos(el), sin(az) * cos(el), sin(el)), 2.0));
        } else {
            const double a = rng_uniform(&r), b = rng_uniform(&r), c = rng_uniform(&r);
            origin = V(a, b, c);
        }
        const double a = rng_uniform(&r), b = rng_uniform(&r), c = rng_uniform(&r);
        target = V(a, b, c);
        if (vnorm(vsub(target, origin)) < 1e-9) target.x += 0.1;
        const v3 d = vnormalized(vsub(target, origin));
        double* o = out + 6 * i;
        o[0] = origin.x; o[1] = origin.y; o[2] = origin.z;
        o[3] = d.x; o[4] = d.y; o[5] = d.z;
    }
}

/* ======================================================================
 * camera -- include/svlf/camera.hpp:12-33, src/camera.cpp:24-40
 * ==================================================================== */
static ray_t pixel_ray(const double* c, uint32_t ix, uint32_t iy) {
    const v3 d = V((ix + 0.5 - c[2]) / c[0], (iy + 0.5 - c[3]) / c[1], 1.0);
    const double* m = c + 4;
    const v3 r = V(m[0] * d.x + m[1] * d.y + m[2] * d.z, m[4] * d.x + m[5] * d.y + m[6] * d.z,
                   m[8] * d.x + m[9] * d.y + m[10] * d.z);
    ray_t out = {V(m[3], m[7], m[11]), vnormalized(r)};
    return out;
}

void or_camera_rays(const double* cam, uint32_t w, uint32_t h, double* rays) {
    for (uint64_t px = 0; px < (uint64_t)w * h; ++px) {
        const ray_t r = pixel_ray(cam, (uint32_t)(px % w), (uint32_t)(px / w));
        double* o = rays + 6 * px;
        o[0] = r.o.x; o[1] = r.o.y; o[2] = r.o.z;
        o[3] = r.d.x; o[4] = r.d.y; o[5] = r.d.z;
    }
}

static void lookat(v3 eye, v3 target, uint32_t w, uint32_t h, double focal, double* c) {
    const v3 fwd = vnormalized(vsub(target, eye));
    v3 up = V(0, 0, 1);
    if (fabs(vdot(fwd, up)) > 0.999) up = V(0, 1, 0);
    const v3 right = vnormalized(vcross(fwd, up));
    const v3 down = vcross(fwd, right);
    c[0] = focal;
    c[1] = focal;
    c[2] = w * 0.5;
    c[3] = h * 0.5;
    const double m[16] = {right.x, down.x, fwd.x, eye.x, right.y, down.y, fwd.y, eye.y,
                          right.z, down.z, fwd.z, eye.z, 0,       0,      0,     1};
    memcpy(c + 4, m, sizeof m);
}
void or_lookat_camera(const double* eye, const double* target, uint32_t w, uint32_t h,
                      double focal, double* cam20) {
    lookat(V(eye[0], eye[1], eye[2]), V(target[0], target[1], target[2]), w, h, focal, cam20);
}

/* sample_hemisphere_cameras, src/scene.cpp:126-141 */
void or_hemisphere_cameras(int n, double radius, uint64_t seed, uint32_t w, uint32_t h,
                           double focal, double* cams) {
    rng_t root, r;
    rng_init(&root, seed);
    rng_sub(&root, 7, &r);
    const v3 center = V(0.5, 0.5, 0.5);
    for (int i = 0; i < n; ++i) {
        const double z = rng_uniform(&r);
        const double az = rng_uniform_in(&r, 0.0, 2.0 * M_PI);
        const double rr = sqrt(fmax(0.0, 1.0 - z * z));
        const v3 dir = V(rr * cos(az), rr * sin(az), z);
        lookat(vadd(center, vmul(dir, radius)), center, w, h, focal, cams + 20 * (size_t)i);
    }
}

/* ======================================================================
 * analytic scene -- include/svlf/scene.hpp, src/scene.cpp:11-124
 * (synthetic-input generator used by the parity tests)
 * ==================================================================== */
typedef struct {
    v3 c;
    double r;
    v3 albedo;
} sphere_t;
typedef struct {
    v3 lo, hi, albedo;
} boxp_t;
struct or_scene {
    sphere_t* s;
    int ns;
    boxp_t* b;
    int nb;
    v3 light_dir, light_rgb, ambient, background;
};

or_scene* or_scene_make(uint64_t seed, int prims) { /* src/scene.cpp:92-124 */
    rng_t root, r;
    rng_init(&root, seed);
    rng_sub(&root, 6, &r);
    or_scene* sc = (or_scene*)calloc(1, sizeof(or_scene));
    sc->s = (sphere_t*)calloc(prims > 0 ? prims : 1, sizeof(sphere_t));
    sc->b = (boxp_t*)calloc(prims > 0 ? prims : 1, sizeof(boxp_t));
    for (int i = 0; i < prims; ++i) {
        const double a0 = rng_uniform_in(&r, 0.2, 1.0);
        const double a1 = rng_uniform_in(&r, 0.2, 1.0);
        const double a2 = rng_uniform_in(&r, 0.2, 1.0);
        const v3 albedo = V(a0, a1, a2);
        if (rng_uniform(&r) < 0.5) {
            sphere_t s;
            s.r = rng_uniform_in(&r, 0.08, 0.16);
            const double c0 = rng_uniform_in(&r, 0.25, 0.75);
            const double c1 = rng_uniform_in(&r, 0.25, 0.75);
            const double c2 = rng_uniform_in(&r, 0.25, 0.75);
            s.c = V(c0, c1, c2);
            s.albedo = albedo;
            sc->s[sc->ns++] = s;
        } else {
            const double h0 = rng_uniform_in(&r, 0.05, 0.12);
            const double h1 = rng_uniform_in(&r, 0.05, 0.12);
            const double h2 = rng_uniform_in(&r, 0.05, 0.12);
            const double c0 = rng_uniform_in(&r, 0.25, 0.75);
            const double c1 = rng_uniform_in(&r, 0.25, 0.75);
            const double c2 = rng_uniform_in(&r, 0.25, 0.75);
            boxp_t b;
            b.lo = vsub(V(c0, c1, c2), V(h0, h1, h2));
            b.hi = vadd(V(c0, c1, c2), V(h0, h1, h2));
            b.albedo = albedo;
            sc->b[sc->nb++] = b;
        }
    }
    const double az = rng_uniform_in(&r, 0.0, 2.0 * M_PI);
    const double el = rng_uniform_in(&r, 0.35, 1.2);
    const v3 l = vnormalized(V(cos(az) * cos(el), sin(az) * cos(el), sin(el)));
    sc->light_dir = V(-l.x, -l.y, -l.z);
    sc->light_rgb = V(0.7, 0.7, 0.7);
    sc->ambient = V(0.25, 0.25, 0.25);
    sc->background = V(0, 0, 0);
    return sc;
}
void or_scene_free(or_scene* s) {
    if (!s) return;
    free(s->s);
    free(s->b);
    free(s);
}

typedef struct {
    double t;
    v3 p, n, albedo;
} surf_t;

static v3 box_normal(const boxp_t* b, v3 p) { /* src/scene.cpp:26-43 */
    const double d[6] = {p.x - b->lo.x, b->hi.x - p.x, p.y - b->lo.y,
                         b->hi.y - p.y, p.z - b->lo.z, b->hi.z - p.z};
    int best = 0;
    for (int i = 1; i < 6; ++i)
        if (d[i] < d[best]) best = i;
    switch (best) {
        case 0: return V(-1, 0, 0);
        case 1: return V(1, 0, 0);
        case 2: return V(0, -1, 0);
        case 3: return V(0, 1, 0);
        case 4: return V(0, 0, -1);
        default: return V(0, 0, 1);
    }
}

static int raycast(const or_scene* sc, const ray_t* ray, surf_t* best) { /* src/scene.cpp:56-77 */
    const double eps = 1e-9;
    int have = 0;
    for (int i = 0; i < sc->ns; ++i) {
        const sphere_t* s = &sc->s[i];
        const v3 oc = vsub(ray->o, s->c);
        const double b = vdot(oc, ray->d);
        const double c = vdot(oc, oc) - s->r * s->r;
        const double disc = b * b - c;
        if (disc < 0) continue;
        const double sq = sqrt(disc);
        double t = -b - sq;
        if (!(t > eps)) {
            t = -b + sq;
            if (!(t > eps)) continue;
        }
        if (!have || t < best->t) {
            const v3 p = ray_at(ray, t);
            best->t = t;
            best->p = p;
            best->n = vnormalized(vsub(p, s->c));
            best->albedo = s->albedo;
            have = 1;
        }
    }
    for (int i = 0; i < sc->nb; ++i) {
        const boxp_t* bx = &sc->b[i];
        aabb_t bb = {bx->lo, bx->hi};
        double t0, t1;
        if (!ray_aabb(ray, &bb, &t0, &t1)) continue;
        const double t = t0 > eps ? t0 : (t1 > eps ? t1 : -1);
        if (t > 0 && (!have || t < best->t)) {
            const v3 p = ray_at(ray, t);
            best->t = t;
            best->p = p;
            best->n = box_normal(bx, p);
            best->albedo = bx->albedo;
            have = 1;
        }
    }
    return have;
}

static double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }

static v3 shade(const or_scene* sc, const surf_t* h) { /* src/scene.cpp:79-90 */
    const v3 nl = V(-sc->light_dir.x, -sc->light_dir.y, -sc->light_dir.z);
    double direct = fmax(0.0, vdot(h->n, nl));
    if (direct > 0) {
        ray_t shadow = {vadd(h->p, vmul(h->n, 1e-6)), nl};
        surf_t tmp;
        if (raycast(sc, &shadow, &tmp)) direct = 0;
    }
    v3 c = V(h->albedo.x * (sc->ambient.x + sc->light_rgb.x * direct),
             h->albedo.y * (sc->ambient.y + sc->light_rgb.y * direct),
             h->albedo.z * (sc->ambient.z + sc->light_rgb.z * direct));
    return V(clamp01(c.x), clamp01(c.y), clamp01(c.z));
}

/* generate_dataset pixel loop, src/dataset.cpp:61-83 */
void or_scene_render_gt(const or_scene* sc, const double* cam, uint32_t w, uint32_t h, float* rgb,
                        float* depth, float* mask) {
    const long long pixels = (long long)w * h;
#pragma omp parallel for schedule(dynamic, 256)
    for (long long p = 0; p < pixels; ++p) {
        const ray_t r = pixel_ray(cam, (uint32_t)(p % w), (uint32_t)(p / w));
        surf_t s;
        if (raycast(sc, &r, &s)) {
            const v3 c = shade(sc, &s);
            rgb[3 * p] = (float)c.x;
            rgb[3 * p + 1] = (float)c.y;
            rgb[3 * p + 2] = (float)c.z;
            depth[p] = (float)s.t;
            mask[p] = 1.f;
        } else {
            rgb[3 * p] = (float)sc->background.x;
            rgb[3 * p + 1] = (float)sc->background.y;
            rgb[3 * p + 2] = (float)sc->background.z;
            depth[p] = 0.f;
            mask[p] = 0.f;
        }
    }
}

/* ======================================================================
 * model init -- src/model.cpp:15-28, src/features.cpp:10-19, src/mlp.cpp:40-56
 * ==================================================================== */
static void init_features(size_t count, uint32_t dim, uint64_t seed, float* out) {
    const double bound = 1.0 / sqrt((double)dim);
    rng_t r;
    rng_init(&r, seed);
    for (size_t i = 0; i < count * dim; ++i) out[i] = (float)rng_uniform_in(&r, -bound, bound);
}

static const uint32_t kTdims[3] = {134, 128, 2};
static const uint32_t kCdims[5] = {38, 128, 128, 128, 3};

static void init_mlp(const uint32_t* dims, int layers, uint64_t seed, float* out) {
    rng_t r;
    rng_init(&r, seed);
    size_t o = 0;
    for (int l = 0; l < layers; ++l) {
        const uint32_t in = dims[l], outd = dims[l + 1];
        const double bound = sqrt(6.0 / (in + outd));
        for (size_t i = 0; i < (size_t)in * outd; ++i) out[o++] = (float)rng_uniform_in(&r, -bound, bound);
        for (uint32_t i = 0; i < outd; ++i) out[o++] = 0.f;
    }
}

void or_init_model(const or_tree* t, uint64_t seed, float* ft, float* fc, float* mt, float* mc) {
    rng_t root, s;
    rng_init(&root, seed);
    const uint32_t V = t->vertex_count;
    rng_sub(&root, 1, &s);
    init_features(V, OR_FT_DIM, rng_u64(&s), ft);
    rng_sub(&root, 2, &s);
    init_features(V, OR_FC_DIM, rng_u64(&s), fc);
    rng_sub(&root, 3, &s);
    init_mlp(kTdims, 2, rng_u64(&s), mt);
    rng_sub(&root, 4, &s);
    init_mlp(kCdims, 4, rng_u64(&s), mc);
}

/* ======================================================================
 * per-voxel evaluation -- src/render.cpp:16-28 (parameterize_ray),
 * src/features.cpp:22-31 (local_coords), include/svlf/features.hpp:13-36,
 * src/voxel_batch.hpp:22-37,69-151 (gather + decoders), src/mlp.cpp:98-149
 * ==================================================================== */
static int parameterize_ray(const ray_t* ray, const aabb_t* b, float* r6) {
    const v3 center = vmul(vadd(b->lo, b->hi), 0.5);
    const double radius = 0.5 * sqrt(3.0) * (b->hi.x - b->lo.x);
    const v3 oc = vsub(ray->o, center);
    const double bb = vdot(oc, ray->d);
    const double c = vdot(oc, oc) - radius * radius;
    const double disc = bb * bb - c;
    if (disc < 1e-14) {
        set_err("tangent ray");
        return 0;
    }
    const double s = sqrt(disc);
    const v3 p1 = vsub(ray_at(ray, -bb - s), center);
    const v3 p2 = vsub(ray_at(ray, -bb + s), center);
    const v3 q1 = vdiv(p1, vnorm(p1)), q2 = vdiv(p2, vnorm(p2));
    r6[0] = (float)q1.x; r6[1] = (float)q1.y; r6[2] = (float)q1.z;
    r6[3] = (float)q2.x; r6[4] = (float)q2.y; r6[5] = (float)q2.z;
    return 1;
}

static int local_coords(const or_tree* t, const aabb_t* box, v3 p, v3* u) {
    const double h = t->cell;
    if (!box_contains(box, p, 1e-7)) {
        set_err("point not in voxel");
        return 0;
    }
    u->x = clamp01((p.x - box->lo.x) / h);
    u->y = clamp01((p.y - box->lo.y) / h);
    u->z = clamp01((p.z - box->lo.z) / h);
    return 1;
}

static void trilinear(v3 u, double* w) {
    const double wx[2] = {1.0 - u.x, u.x}, wy[2] = {1.0 - u.y, u.y}, wz[2] = {1.0 - u.z, u.z};
    for (int b = 0; b < 8; ++b) w[b] = wx[b & 1] * wy[(b >> 1) & 1] * wz[(b >> 2) & 1];
}

static void trilinear_grads(v3 u, double g[8][3]) {
    const double wx[2] = {1.0 - u.x, u.x}, wy[2] = {1.0 - u.y, u.y}, wz[2] = {1.0 - u.z, u.z};
    const double dx[2] = {-1.0, 1.0};
    for (int b = 0; b < 8; ++b) {
        const int bx = b & 1, by = (b >> 1) & 1, bz = (b >> 2) & 1;
        g[b][0] = dx[bx] * wy[by] * wz[bz];
        g[b][1] = wx[bx] * dx[by] * wz[bz];
        g[b][2] = wx[bx] * wy[by] * dx[bz];
    }
}

static void interp(const float* vol, uint32_t dim, const uint32_t* corners, const double* w, float* out) {
    for (uint32_t d = 0; d < dim; ++d) out[d] = 0.f;
    for (int b = 0; b < 8; ++b) {
        const float wb = (float)w[b];
        const float* row = vol + (size_t)corners[b] * dim;
        for (uint32_t d = 0; d < dim; ++d) out[d] += wb * row[d];
    }
}

static float sigmoidf_ref(float x) { return 1.0f / (1.0f + expf(-x)); } /* mlp.cpp:81-84 */

/* Dense layer over one column: y[o] = b[o] + sum_k W[o][k] x[k], k in order (mlp.cpp:98-116) */
static void dense(const float* W, const float* b, const float* x, uint32_t in, uint32_t out, float* y) {
    for (uint32_t o = 0; o < out; ++o) {
        float acc = b[o];
        const float* wr = W + (size_t)o * in;
        for (uint32_t k = 0; k < in; ++k) acc += wr[k] * x[k];
        y[o] = acc;
    }
}

/* forward activations kept for backward: acts[0] = input, acts[l+1] = post-activation */
typedef struct {
    float* a[5];
} acts_t;

static void mlp_fwd(const float* P, const uint32_t* dims, int layers, const uint8_t* heads,
                    acts_t* A) {
    size_t o = 0;
    for (int l = 0; l < layers; ++l) {
        const uint32_t in = dims[l], out = dims[l + 1];
        const float* W = P + o;
        o += (size_t)in * out;
        const float* b = P + o;
        o += out;
        dense(W, b, A->a[l], in, out, A->a[l + 1]);
        float* y = A->a[l + 1];
        if (l + 1 < layers) {
            for (uint32_t i = 0; i < out; ++i) y[i] = y[i] > 0.f ? y[i] : 0.f;
        } else {
            for (uint32_t i = 0; i < out; ++i) y[i] = heads[i] == 0 ? (y[i] > 0.f ? y[i] : 0.f) : sigmoidf_ref(y[i]);
        }
    }
}

static const uint8_t kTheads[2] = {0, 1};    /* relu, sigmoid (mlp.cpp:16-24) */
static const uint8_t kCheads[3] = {1, 1, 1}; /* sigmoid x3 (mlp.cpp:26-34) */

typedef struct {
    uint64_t id;
    double tin, tout;
    v3 x1, x2;
    uint32_t corners[8];
    double w1[8], w2[8], ws[8];
    v3 us;
    float r6[6];
    double tau, eta, ts;
    v3 xs;
    float inT[134], hT[128], oT[2];
    float inC[38], h1[128], h2[128], h3[128], oC[3];
    int has_color;
} hiteval_t;

/* batch_forward_thickness for one hit (voxel_batch.hpp:69-114) */
static int eval_thickness(const or_tree* t, const float* ft, const float* mt, const ray_t* ray,
                          const hit_t* h, hiteval_t* e) {
    e->id = h->id;
    e->tin = h->tin;
    e->tout = h->tout;
    e->x1 = h->x1;
    e->x2 = h->x2;
    const aabb_t box = voxel_aabb(t, h->id);
    if (!parameterize_ray(ray, &box, e->r6)) return 0;
    for (int k = 0; k < 6; ++k) e->inT[k] = e->r6[k];
    const long li = leaf_index(t, h->id);
    if (li < 0) {
        set_err("unknown voxel id");
        return 0;
    }
    memcpy(e->corners, t->corner_ids + 8 * (size_t)li, sizeof e->corners);
    v3 u1, u2;
    if (!local_coords(t, &box, h->x1, &u1) || !local_coords(t, &box, h->x2, &u2)) return 0;
    trilinear(u1, e->w1);
    trilinear(u2, e->w2);
    interp(ft, OR_FT_DIM, e->corners, e->w1, e->inT + 6);
    interp(ft, OR_FT_DIM, e->corners, e->w2, e->inT + 6 + OR_FT_DIM);
    acts_t A = {{e->inT, e->hT, e->oT, NULL, NULL}};
    mlp_fwd(mt, kTdims, 2, kTheads, &A);
    e->tau = (double)e->oT[0];
    e->eta = (double)e->oT[1];
    e->xs = vadd(vmul(h->x1, e->eta), vmul(h->x2, 1.0 - e->eta));
    e->ts = h->tin * e->eta + h->tout * (1.0 - e->eta);
    e->has_color = 0;
    return 1;
}

/* batch_forward_color for one hit (voxel_batch.hpp:119-142) */
static int eval_color(const or_tree* t, const float* fc, const float* mc, hiteval_t* e) {
    for (int k = 0; k < 6; ++k) e->inC[k] = e->inT[k];
    const aabb_t box = voxel_aabb(t, e->id);
    if (!local_coords(t, &box, e->xs, &e->us)) return 0;
    trilinear(e->us, e->ws);
    interp(fc, OR_FC_DIM, e->corners, e->ws, e->inC + 6);
    acts_t A = {{e->inC, e->h1, e->h2, e->h3, e->oC}};
    mlp_fwd(mc, kCdims, 4, kCheads, &A);
    e->has_color = 1;
    return 1;
}

/* ======================================================================
 * render -- src/render.cpp:135-207 (render_tile per pixel)
 * ==================================================================== */
static int render_one(const or_tree* t, const float* ft, const float* fc, const float* mt,
                      const float* mc, const ray_t* ray, const float* bg, float* rgb, float* alpha,
                      float* depth, long long* nh) {
    hitvec hv = {0};
    traverse(t, ray, &hv);
    double color[3] = {0, 0, 0}, a = 0.0, dacc = 0.0, T = 1.0;
    hiteval_t e;
    int ok = 1;
    for (size_t j = 0; j < hv.n && ok; ++j) {
        ok = eval_thickness(t, ft, mt, ray, &hv.v[j], &e) && eval_color(t, fc, mc, &e);
        if (!ok) break;
        const double ex = exp(-e.tau);
        const double w = T * (1.0 - ex);
        color[0] += w * (double)e.oC[0];
        color[1] += w * (double)e.oC[1];
        color[2] += w * (double)e.oC[2];
        dacc += w * e.ts;
        a += w;
        T *= ex;
    }
    *nh = (long long)hv.n;
    free(hv.v);
    if (!ok) return 0;
    const float b0 = bg ? bg[0] : 0.f, b1 = bg ? bg[1] : 0.f, b2 = bg ? bg[2] : 0.f;
    rgb[0] = (float)(color[0] + (1.0 - a) * b0);
    rgb[1] = (float)(color[1] + (1.0 - a) * b1);
    rgb[2] = (float)(color[2] + (1.0 - a) * b2);
    *alpha = (float)a;
    *depth = a > 1e-4 ? (float)(dacc / a) : 0.f;
    return 1;
}

int or_render_rays(const or_tree* t, const float* ft, const float* fc, const float* mt,
                   const float* mc, const double* rays, size_t n, const float* bg, float* rgb,
                   float* alpha, float* depth, long long* stats) {
    long long fg = 0, hits = 0;
    int failed = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : fg, hits) reduction(| : failed)
    for (long long i = 0; i < (long long)n; ++i) {
        ray_t r = {V(rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]),
                   V(rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5])};
        long long nh = 0;
        if (!render_one(t, ft, fc, mt, mc, &r, bg, rgb + 3 * i, alpha + i, depth + i, &nh)) failed = 1;
        hits += nh;
        fg += nh > 0;
    }
    if (stats) {
        stats[0] = (long long)n;
        stats[1] = fg;
        stats[2] = hits;
        stats[3] = hits;
        stats[4] = hits;
    }
    return failed ? 1 : 0;
}

int or_render_frame(const or_tree* t, const float* ft, const float* fc, const float* mt,
                    const float* mc, const double* cam, uint32_t w, uint32_t h, const float* bg,
                    float* rgb, float* alpha, float* depth, long long* stats) {
    const size_t n = (size_t)w * h;
    double* rays = (double*)malloc(n * 6 * sizeof(double));
    or_camera_rays(cam, w, h, rays);
    const int rc = or_render_rays(t, ft, fc, mt, mc, rays, n, bg, rgb, alpha, depth, stats);
    free(rays);
    return rc;
}

/* ======================================================================
 * losses + backward -- src/train.cpp:30-35 (eta_gt), :65-287 (loss_chunk),
 * src/mlp.cpp:151-230 (mlp_backward)
 * ==================================================================== */

/* Reverse pass over one column. d_out = dL/d(post-activation outputs).
 * Accumulates parameter grads into G (if non-null) and writes dL/d(input). */
static void mlp_bwd(const float* P, const uint32_t* dims, int layers, const uint8_t* heads,
                    const acts_t* A, const float* d_out, float* G, float* d_in) {
    float cur[128], nxt[134];
    const uint32_t outd = dims[layers];
    const float* a = A->a[layers];
    for (uint32_t o = 0; o < outd; ++o)
        cur[o] = heads[o] == 0 ? (a[o] > 0.f ? d_out[o] : 0.f) : d_out[o] * a[o] * (1.0f - a[o]);
    size_t offs[5], off = 0;
    for (int l = 0; l < layers; ++l) {
        offs[l] = off;
        off += (size_t)dims[l] * dims[l + 1] + dims[l + 1];
    }
    for (int l = layers - 1; l >= 0; --l) {
        const uint32_t in = dims[l], out = dims[l + 1];
        const float* W = P + offs[l];
        const float* x = A->a[l];
        if (G) {
            float* dW = G + offs[l];
            float* db = dW + (size_t)in * out;
            for (uint32_t o = 0; o < out; ++o) {
                for (uint32_t k = 0; k < in; ++k) dW[(size_t)o * in + k] += cur[o] * x[k];
                db[o] += cur[o];
            }
        }
        for (uint32_t k = 0; k < in; ++k) nxt[k] = 0.f;
        for (uint32_t o = 0; o < out; ++o) {
            const float* wr = W + (size_t)o * in;
            for (uint32_t k = 0; k < in; ++k) nxt[k] += wr[k] * cur[o];
        }
        if (l > 0)
            for (uint32_t k = 0; k < in; ++k) nxt[k] = x[k] > 0.f ? nxt[k] : 0.f;
        for (uint32_t k = 0; k < in; ++k) cur[k] = nxt[k];
    }
    if (d_in)
        for (uint32_t k = 0; k < dims[0]; ++k) d_in[k] = cur[k];
}

typedef struct {
    double eta, tau, empty, alpha;
} lw_t;

/* one ray of loss_chunk (src/train.cpp:65-287) */
static int loss_ray(const or_tree* t, const float* ft, const float* fc, const float* mt,
                    const float* mc, const ray_t* ray, const float* cgt, double depth_gt,
                    int alpha_gt, int mode, lw_t lw, int frozen, float* g_ft, float* g_fc,
                    float* g_mt, float* g_mc, long long* st, double* loss_out) {
    *loss_out = 0.0;
    st[0]++;
    hitvec hv = {0};
    traverse(t, ray, &hv);
    size_t keep = hv.n;
    long surf = -1;
    double eg = 0.0;
    int rc = 1;
    if (alpha_gt) {
        const v3 xs = ray_at(ray, depth_gt);
        uint64_t vid;
        if (locate(t, xs, &vid)) {
            for (size_t j = 0; j < hv.n; ++j) {
                if (hv.v[j].id == vid) {
                    surf = (long)j;
                    const hit_t* h = &hv.v[j];
                    if (depth_gt < h->tin - 1e-6 || depth_gt > h->tout + 1e-6) { /* eta_gt */
                        set_err("surface point outside voxel");
                        free(hv.v);
                        return 0;
                    }
                    const double span = h->tout - h->tin;
                    eg = clamp01((h->tout - depth_gt) / span);
                    if (mode == 0) keep = j + 1;
                    break;
                }
            }
        }
    }
    if (mode == 0) {
        if (!alpha_gt || surf < 0) {
            st[1]++;
            free(hv.v);
            return 1;
        }
        if (lw.empty == 0.0) {
            hv.v[0] = hv.v[keep - 1];
            surf = 0;
            keep = 1;
        }
    } else if (alpha_gt && surf < 0) {
        st[2]++;
    }
    const size_t n = keep;
    if (n == 0) {
        /* volumetric ray with no hits: composite is empty */
        double loss = 0.0;
        for (int ch = 0; ch < 3; ++ch) {
            const double diff = 0.0 - (double)cgt[ch];
            loss += diff * diff;
        }
        const double agt = alpha_gt ? 1.0 : 0.0;
        loss += lw.alpha * (0.0 - agt) * (0.0 - agt);
        *loss_out = loss;
        free(hv.v);
        return 1;
    }
    hiteval_t* E = (hiteval_t*)calloc(n, sizeof(hiteval_t));
    for (size_t j = 0; j < n && rc; ++j) rc = eval_thickness(t, ft, mt, ray, &hv.v[j], &E[j]);
    if (rc) {
        if (mode == 1) {
            for (size_t j = 0; j < n && rc; ++j) rc = eval_color(t, fc, mc, &E[j]);
        } else {
            rc = eval_color(t, fc, mc, &E[surf]);
        }
    }
    if (!rc) {
        free(E);
        free(hv.v);
        return 0;
    }
    double* dtau = (double*)calloc(n, sizeof(double));
    double* deta = (double*)calloc(n, sizeof(double));
    float(*dc_out)[3] = (float(*)[3])calloc(n, sizeof(float[3]));
    double loss = 0.0;
    if (mode == 0) {
        const size_t js = (size_t)surf;
        double dc[3];
        for (int ch = 0; ch < 3; ++ch) {
            const double diff = (double)E[js].oC[ch] - (double)cgt[ch];
            loss += diff * diff;
            dc[ch] = 2.0 * diff;
        }
        const double ediff = E[js].eta - eg;
        loss += lw.eta * ediff * ediff;
        deta[js] += 2.0 * lw.eta * ediff;
        const double e2 = exp(-2.0 * E[js].tau);
        loss += lw.tau * e2;
        dtau[js] += -2.0 * lw.tau * e2;
        for (size_t k = 0; k < js; ++k) {
            const double e = exp(-E[k].tau);
            const double olap = 1.0 - e;
            loss += lw.empty * olap * olap;
            dtau[k] += 2.0 * lw.empty * olap * e;
        }
        for (int ch = 0; ch < 3; ++ch) dc_out[js][ch] = (float)dc[ch];
    } else {
        double color[3] = {0, 0, 0}, alpha = 0.0, T = 1.0;
        double* ehit = (double*)malloc(n * sizeof(double));
        double* trans = (double*)malloc(n * sizeof(double));
        double* wgt = (double*)malloc(n * sizeof(double));
        for (size_t j = 0; j < n; ++j) {
            const double e = exp(-E[j].tau);
            const double w = T * (1.0 - e);
            ehit[j] = e;
            trans[j] = T;
            wgt[j] = w;
            for (int ch = 0; ch < 3; ++ch) color[ch] += w * (double)E[j].oC[ch];
            alpha += w;
            T *= e;
        }
        double d_color[3];
        for (int ch = 0; ch < 3; ++ch) {
            const double diff = color[ch] - (double)cgt[ch];
            loss += diff * diff;
            d_color[ch] = 2.0 * diff;
        }
        const double agt = alpha_gt ? 1.0 : 0.0;
        loss += lw.alpha * (alpha - agt) * (alpha - agt);
        const double d_alpha = 2.0 * lw.alpha * (alpha - agt);
        if (alpha_gt && surf >= 0) {
            const double ediff = E[surf].eta - eg;
            loss += lw.eta * ediff * ediff;
            deta[surf] += 2.0 * lw.eta * ediff;
        }
        double suffix = 0.0;
        for (long j = (long)n - 1; j >= 0; --j) {
            double dw = d_alpha;
            for (int ch = 0; ch < 3; ++ch) dw += d_color[ch] * (double)E[j].oC[ch];
            dtau[j] += dw * trans[j] * ehit[j] - suffix;
            suffix += dw * wgt[j];
            for (int ch = 0; ch < 3; ++ch) dc_out[j][ch] = (float)(wgt[j] * d_color[ch]);
        }
        free(ehit);
        free(trans);
        free(wgt);
    }
    *loss_out = loss;

    if (g_ft || g_fc || g_mt || g_mc) {
        /* color decoder backward (train.cpp:238-266) */
        const double inv_h = 1.0 / t->cell;
        for (size_t j = 0; j < n; ++j) {
            if (!E[j].has_color) continue;
            float d_in[38];
            acts_t A = {{E[j].inC, E[j].h1, E[j].h2, E[j].h3, E[j].oC}};
            mlp_bwd(mc, kCdims, 4, kCheads, &A, dc_out[j], frozen ? NULL : g_mc, d_in);
            if (!frozen && g_fc) {
                for (int b = 0; b < 8; ++b) {
                    const float wb = (float)E[j].ws[b];
                    float* grow = g_fc + (size_t)E[j].corners[b] * OR_FC_DIM;
                    for (uint32_t d = 0; d < OR_FC_DIM; ++d) grow[d] += wb * d_in[6 + d];
                }
            }
            double dw[8][3];
            trilinear_grads(E[j].us, dw);
            v3 dxs = V(0, 0, 0);
            for (int b = 0; b < 8; ++b) {
                const float* zb = fc + (size_t)E[j].corners[b] * OR_FC_DIM;
                double dotv = 0.0;
                for (uint32_t d = 0; d < OR_FC_DIM; ++d) dotv += (double)zb[d] * (double)d_in[6 + d];
                dxs = vadd(dxs, vmul(V(dw[b][0], dw[b][1], dw[b][2]), dotv * inv_h));
            }
            deta[j] += vdot(dxs, vsub(E[j].x1, E[j].x2));
        }
        /* thickness decoder backward (train.cpp:268-285) */
        for (size_t j = 0; j < n; ++j) {
            float dout[2] = {(float)dtau[j], (float)deta[j]};
            float d_in[134];
            acts_t A = {{E[j].inT, E[j].hT, E[j].oT, NULL, NULL}};
            mlp_bwd(mt, kTdims, 2, kTheads, &A, dout, g_mt, d_in);
            if (g_ft) {
                for (int b = 0; b < 8; ++b) {
                    float* grow = g_ft + (size_t)E[j].corners[b] * OR_FT_DIM;
                    const float wb1 = (float)E[j].w1[b], wb2 = (float)E[j].w2[b];
                    for (uint32_t d = 0; d < OR_FT_DIM; ++d)
                        grow[d] += wb1 * d_in[6 + d] + wb2 * d_in[6 + OR_FT_DIM + d];
                }
            }
        }
    }
    free(dtau);
    free(deta);
    free(dc_out);
    free(E);
    free(hv.v);
    return 1;
}

int or_loss(const or_tree* t, const float* ft, const float* fc, const float* mt, const float* mc,
            const double* rays, const float* cgt, const double* depth, const uint8_t* alpha,
            size_t n, int mode, const double* lw4, int frozen, float* g_ft, float* g_fc,
            float* g_mt, float* g_mc, long long* stats3, double* loss_out) {
    const lw_t lw = {lw4[0], lw4[1], lw4[2], lw4[3]};
    long long st[3] = {0, 0, 0};
    double loss = 0.0;
    for (size_t i = 0; i < n; ++i) {
        ray_t r = {V(rays[6 * i], rays[6 * i + 1], rays[6 * i + 2]),
                   V(rays[6 * i + 3], rays[6 * i + 4], rays[6 * i + 5])};
        double l;
        if (!loss_ray(t, ft, fc, mt, mc, &r, cgt + 3 * i, depth[i], alpha[i] != 0, mode, lw,
                      frozen, g_ft, g_fc, g_mt, g_mc, st, &l))
            return 1;
        loss += l;
    }
    if (stats3) memcpy(stats3, st, sizeof st);
    *loss_out = loss;
    return 0;
}

/* adam_step, src/mlp.cpp:277-296; beta/eps are float fields promoted to double */
void or_adam_step(float* params, const float* grads, float* m, float* v, size_t n,
                  uint64_t step, float lr) {
    step += 1;
    const double b1 = (double)0.9f, b2 = (double)0.999f, eps = (double)1e-8f;
    const double corr1 = 1.0 - pow(b1, (double)step);
    const double corr2 = 1.0 - pow(b2, (double)step);
    for (size_t i = 0; i < n; ++i) {
        const double g = grads[i];
        const double mm = b1 * m[i] + (1.0 - b1) * g;
        const double vv = b2 * v[i] + (1.0 - b2) * g * g;
        m[i] = (float)mm;
        v[i] = (float)vv;
        const double mh = mm / corr1;
        const double vh = vv / corr2;
        params[i] = (float)(params[i] - lr * mh / (sqrt(vh) + eps));
    }
}
