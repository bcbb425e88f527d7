/*
 * TEST INFRASTRUCTURE ONLY - CPU oracle for the HarMoEny scheduling path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the checker or as the
 * timed CPU baseline.  The product path (paper_2506_12417_b200) never links or
 * calls it.
 *
 * This is a plain-C restatement of the reference's integer algorithms:
 *
 *   orc_initial_assign   <- moesim/policies.py:109-117   (initial_assign)
 *   orc_rebalance        <- moesim/policies.py:120-141   (_rebalance_core, Alg. 2,
 *                            PAPER.md:702-745); argmax/argmin ties break to the
 *                            lowest index exactly like numpy (policies.py:15-16)
 *   orc_round_robin / orc_blocked <- policies.py:91-106
 *   orc_even_split       <- moesim/policies.py:174-203   (even_split_assign baseline)
 *   orc_affinity         <- moesim/policies.py:206-229   (affinity_placement, LPT)
 *   orc_histogram        <- core.py:89-96 (RoutingMatrix row = per-GPU histogram)
 *   orc_dispatch_ranks   <- the split-bucket contract of SURVEY.md §8(a) A13
 *                            (the reference drops token identity)
 *   orc_plan_order       <- moesim/engine.py:233-234 (plan_gpu_execution order)
 *
 * Parity of the scheduler functions is pinned against the reference itself:
 * tests/golden/make_golden.py imports moesim from /root/reference and commits
 * its outputs as fixtures; tests/test_oracle_golden.py checks this file against
 * them.  All counts are int64 like the reference (core.py:20-27).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define IDX3(g, e, d, E, G) ((((int64_t)(g) * (E)) + (e)) * (G) + (d))

/* policies.py:91-95 */
void orc_round_robin(int E, int G, int64_t* home) {
    for (int e = 0; e < E; ++e) home[e] = e % G;
}

/* policies.py:98-106: block = ceil(E/G), home = min(e // block, G-1) */
void orc_blocked(int E, int G, int64_t* home) {
    int block = (E + G - 1) / G;
    for (int e = 0; e < E; ++e) {
        int h = e / block;
        home[e] = h < G - 1 ? h : G - 1;
    }
}

/* policies.py:109-117: S[g, e, home[e]] = m[g, e] */
int orc_initial_assign(const int64_t* m, const int64_t* home, int G, int E, int64_t* S) {
    memset(S, 0, sizeof(int64_t) * (size_t)G * E * G);
    for (int e = 0; e < E; ++e)
        if (home[e] < 0 || home[e] >= G) return 1;
    for (int g = 0; g < G; ++g)
        for (int e = 0; e < E; ++e) S[IDX3(g, e, home[e], E, G)] = m[(int64_t)g * E + e];
    return 0;
}

/* policies.py:120-141 (_rebalance_core), in place.  Returns 1 on q < 1
 * (policies.py:168-169), else 0; *iters receives the move count. */
int orc_rebalance(int64_t* S, int G, int E, int64_t q, int64_t* iters) {
    if (q < 1) return 1;
    int64_t total = 0;
    int64_t* t = (int64_t*)calloc((size_t)G, sizeof(int64_t));
    for (int g = 0; g < G; ++g)
        for (int e = 0; e < E; ++e)
            for (int d = 0; d < G; ++d) {
                int64_t v = S[IDX3(g, e, d, E, G)];
                total += v;
                t[d] += v;
            }
    const int64_t t_avg = total / G; /* floor: counts are non-negative */
    int64_t it = 0;
    for (;;) {
        int any_over = 0;
        for (int d = 0; d < G; ++d) any_over |= t[d] > t_avg;
        if (!any_over) break;
        int g_max = 0;
        for (int d = 1; d < G; ++d)
            if (t[d] > t[g_max]) g_max = d;
        int g_from = 0;
        int64_t best = -1;
        for (int g = 0; g < G; ++g) {
            int64_t f = 0;
            for (int e = 0; e < E; ++e) f += S[IDX3(g, e, g_max, E, G)];
            if (f > best) { best = f; g_from = g; }
        }
        int e_max = 0;
        int64_t vmax = -1;
        for (int e = 0; e < E; ++e) {
            int64_t v = S[IDX3(g_from, e, g_max, E, G)];
            if (v > vmax) { vmax = v; e_max = e; }
        }
        const int64_t t_move = vmax;
        if (t_move < q) break;
        int g_min = 0;
        for (int d = 1; d < G; ++d)
            if (t[d] < t[g_min]) g_min = d;
        if (g_min == g_max || t[g_min] + q > t_avg) break;
        int64_t t_s = t_avg - t[g_min];
        if (t_move < t_s) t_s = t_move;
        S[IDX3(g_from, e_max, g_max, E, G)] -= t_s;
        S[IDX3(g_from, e_max, g_min, E, G)] += t_s;
        t[g_max] -= t_s;
        t[g_min] += t_s;
        ++it;
    }
    free(t);
    *iters = it;
    return 0;
}

/* initial_assign + rebalance (engine.py:296-298 with policy REBALANCE). */
int orc_schedule(const int64_t* m, const int64_t* home, int G, int E, int64_t q, int rebalance,
                 int64_t* S, int64_t* iters) {
    int rc = orc_initial_assign(m, home, G, E, S);
    *iters = 0;
    if (rc) return rc;
    if (rebalance) return orc_rebalance(S, G, E, q, iters);
    if (q < 1) return 1;
    return 0;
}

/* policies.py:174-203: each expert's pooled total split as evenly as integers allow
 * (remainder to the lowest-index GPUs); sources fill the targets in index order. */
void orc_even_split(const int64_t* m, int G, int E, int64_t* S) {
    memset(S, 0, sizeof(int64_t) * (size_t)G * E * G);
    int64_t* remaining = (int64_t*)malloc(sizeof(int64_t) * (size_t)G);
    for (int e = 0; e < E; ++e) {
        int64_t total = 0;
        for (int g = 0; g < G; ++g) total += m[(int64_t)g * E + e];
        if (total == 0) continue;
        int64_t base = total / G, rem = total % G;
        for (int g = 0; g < G; ++g) remaining[g] = base + (g < rem ? 1 : 0);
        int dest = 0;
        for (int src = 0; src < G; ++src) {
            int64_t left = m[(int64_t)src * E + e];
            while (left > 0) {
                while (remaining[dest] == 0) ++dest;
                int64_t take = left < remaining[dest] ? left : remaining[dest];
                S[IDX3(src, e, dest, E, G)] += take;
                remaining[dest] -= take;
                left -= take;
            }
        }
    }
    free(remaining);
}

/* policies.py:206-229: experts by descending popularity (ties: lower id) onto the GPU with
 * the least accumulated mass that has a free slot (ties: lower GPU).  Returns 1 if
 * E > G * slots (the reference's ValueError), else 0. */
int orc_affinity(const int64_t* counts, int E, int G, int slots, int64_t* home) {
    if ((int64_t)E > (int64_t)G * slots) return 1;
    int* order = (int*)malloc(sizeof(int) * (size_t)(E > 0 ? E : 1));
    int64_t* mass = (int64_t*)calloc((size_t)G, sizeof(int64_t));
    int* used = (int*)calloc((size_t)G, sizeof(int));
    for (int e = 0; e < E; ++e) order[e] = e;
    /* insertion sort by (-count, id): stable and E is small */
    for (int i = 1; i < E; ++i) {
        int v = order[i], j = i - 1;
        while (j >= 0 && counts[order[j]] < counts[v]) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = v;
    }
    for (int i = 0; i < E; ++i) {
        int e = order[i], best = -1;
        for (int g = 0; g < G; ++g)
            if (used[g] < slots && (best < 0 || mass[g] < mass[best])) best = g;
        home[e] = best;
        mass[best] += counts[e];
        used[best] += 1;
    }
    free(order);
    free(mass);
    free(used);
    return 0;
}

/* core.py:89-96: hist[e] = #assignments routed to e. */
void orc_histogram(const int32_t* idx, int64_t n, int E, int64_t* hist) {
    memset(hist, 0, sizeof(int64_t) * (size_t)E);
    for (int64_t i = 0; i < n; ++i) hist[idx[i]] += 1;
}

/* Split-bucket contract.  For source g with
 * assignments idx[T*k] in (token, slot) order: the r-th assignment routed to
 * expert e (0-based, in that order) is executed on the first destination d
 * with cumsum_{d'<=d} S[g, e, d'] > r.  Outputs dest[i] and rank[i]. */
int orc_dispatch_ranks(const int32_t* idx, int64_t n, const int64_t* S, int g, int G, int E,
                       int32_t* dest, int32_t* rank) {
    int64_t* seen = (int64_t*)calloc((size_t)E, sizeof(int64_t));
    int rc = 0;
    for (int64_t i = 0; i < n; ++i) {
        int e = idx[i];
        int64_t r = seen[e]++;
        rank[i] = (int32_t)r;
        int64_t c = 0;
        int d = 0;
        for (; d < G; ++d) {
            c += S[IDX3(g, e, d, E, G)];
            if (c > r) break;
        }
        if (d == G) { rc = 1; d = -1; }
        dest[i] = d;
    }
    free(seen);
    return rc;
}

/* engine.py:233-234: residents with work by (-tokens, e), then non-resident
 * experts with work by (-tokens, e).  work[e] = tokens of expert e on this
 * GPU, resident[e] != 0 when expert e is statically cached here.  Writes the
 * expert order to order[], returns its length. */
int orc_plan_order(const int64_t* work, const int32_t* resident, int E, int32_t* order) {
    int n = 0;
    for (int pass = 0; pass < 2; ++pass) {
        int start = n;
        for (int e = 0; e < E; ++e) {
            if (work[e] <= 0) continue;
            if ((resident[e] != 0) != (pass == 0)) continue;
            /* insertion into order[start..n) by (-work, e) */
            int pos = n;
            while (pos > start) {
                int p = order[pos - 1];
                if (work[p] > work[e] || (work[p] == work[e] && p < e)) break;
                order[pos] = p;
                --pos;
            }
            order[pos] = e;
            ++n;
        }
    }
    return n;
}
