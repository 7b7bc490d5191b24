/* CPU oracle for Cuthill-McKee ordering (TEST INFRASTRUCTURE ONLY).
 *
 * Restates hodg/renumber.py:135-208 exactly:
 *  - components are seeded in ascending vertex id (renumber.py:184-188);
 *  - start vertex: George-Liu double BFS from argmin (degree, id), the
 *    candidate is argmin (degree, id) over the last level; stop when the
 *    candidate's eccentricity does not exceed the current one
 *    (renumber.py:153-168);
 *  - BFS appends unvisited neighbours in (degree, id) order, marking on
 *    enqueue (renumber.py:176-199).
 * The reversal into the RCM permutation is done by the caller
 * (renumber.py:203-208).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static const int64_t *g_deg;

static int cmp_deg_id(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    if (g_deg[x] != g_deg[y]) return g_deg[x] < g_deg[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}

/* BFS over the component of `start`; level[] must be -1 on the component.
 * Writes members in BFS order to `members`, returns count; *ecc = max level. */
static int64_t bfs_levels(const int64_t *indptr, const int64_t *indices, int64_t start, int64_t *level,
                          int64_t *members, int64_t *ecc) {
    int64_t head = 0, tail = 0;
    level[start] = 0;
    members[tail++] = start;
    int64_t mx = 0;
    while (head < tail) {
        int64_t v = members[head++];
        int64_t lv = level[v] + 1;
        for (int64_t k = indptr[v]; k < indptr[v + 1]; ++k) {
            int64_t w = indices[k];
            if (level[w] < 0) {
                level[w] = lv;
                if (lv > mx) mx = lv;
                members[tail++] = w;
            }
        }
    }
    *ecc = mx;
    return tail;
}

static int better(const int64_t *deg, int64_t a, int64_t b) { /* (deg,id) of a < b */
    if (deg[a] != deg[b]) return deg[a] < deg[b];
    return a < b;
}

int ora_cuthill_mckee(int64_t n, const int64_t *indptr, const int64_t *indices, int64_t *order) {
    int64_t *deg = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    int64_t *sorted = malloc(sizeof(int64_t) * (indptr[n] > 0 ? indptr[n] : 1));
    int64_t *level = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    int64_t *comp = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    int64_t *tmp = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    char *visited = calloc(n > 0 ? n : 1, 1);
    if (!deg || !sorted || !level || !comp || !tmp || !visited) return -1;
    for (int64_t v = 0; v < n; ++v) deg[v] = indptr[v + 1] - indptr[v];
    memcpy(sorted, indices, sizeof(int64_t) * indptr[n]);
    g_deg = deg;
    for (int64_t v = 0; v < n; ++v)
        qsort(sorted + indptr[v], (size_t)deg[v], sizeof(int64_t), cmp_deg_id);
    for (int64_t v = 0; v < n; ++v) level[v] = -1;
    int64_t pos = 0;
    for (int64_t seed = 0; seed < n; ++seed) {
        if (visited[seed]) continue;
        int64_t ecc;
        int64_t nc = bfs_levels(indptr, indices, seed, level, comp, &ecc);
        /* pseudo-peripheral start */
        int64_t r = comp[0];
        for (int64_t i = 1; i < nc; ++i)
            if (better(deg, comp[i], r)) r = comp[i];
        for (;;) {
            for (int64_t i = 0; i < nc; ++i) level[comp[i]] = -1;
            int64_t e_r;
            bfs_levels(indptr, indices, r, level, tmp, &e_r);
            int64_t cand = -1;
            for (int64_t i = 0; i < nc; ++i) {
                int64_t v = comp[i];
                if (level[v] == e_r && (cand < 0 || better(deg, v, cand))) cand = v;
            }
            for (int64_t i = 0; i < nc; ++i) level[comp[i]] = -1;
            int64_t e_c;
            bfs_levels(indptr, indices, cand, level, tmp, &e_c);
            for (int64_t i = 0; i < nc; ++i) level[comp[i]] = -1;
            if (e_c > e_r) r = cand;
            else break;
        }
        /* Cuthill-McKee BFS from r with sorted neighbour lists */
        int64_t head = pos;
        visited[r] = 1;
        order[pos++] = r;
        while (head < pos) {
            int64_t v = order[head++];
            for (int64_t k = indptr[v]; k < indptr[v + 1]; ++k) {
                int64_t w = sorted[k];
                if (!visited[w]) {
                    visited[w] = 1;
                    order[pos++] = w;
                }
            }
        }
    }
    free(deg);
    free(sorted);
    free(level);
    free(comp);
    free(tmp);
    free(visited);
    return 0;
}
