// lru_sim.c -- LRU model of the C5 gather's row-reference stream (development
// tool, not product).  Inputs (from a CPU run of workloads.make_graph for C5):
// /tmp/sim/col.bin (destination-sorted col_src, int32) and /tmp/sim/outdeg.bin
// (out-degree per vertex, int32).  The stream is replayed as W warps each
// walking its contiguous edge range, round-robin in batches of B edges; the
// cache holds C rows.  Policy: a source whose out-degree is <= k_cold is
// inserted at the LRU end and never promoted (an L2 evict-first load); k_cold
// = -1 is plain LRU.
// Build: gcc -O2 -o lru_sim lru_sim.c     Run: ./lru_sim C_rows k_cold W B
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
int main(int argc, char **argv) {
    long C = atol(argv[1]); int kc = atoi(argv[2]); long W = atol(argv[3]); int B = atoi(argv[4]);
    FILE *f = fopen("/tmp/sim/col.bin", "rb"); fseek(f, 0, SEEK_END); long E = ftell(f) / 4; fseek(f, 0, SEEK_SET);
    int32_t *col = malloc(E * 4); if (fread(col, 4, E, f) != (size_t)E) return 1;
    fclose(f);
    f = fopen("/tmp/sim/outdeg.bin", "rb"); fseek(f, 0, SEEK_END); long n = ftell(f) / 4; fseek(f, 0, SEEK_SET);
    int32_t *od = malloc(n * 4); if (fread(od, 4, n, f) != (size_t)n) return 1;
    fclose(f);
    int32_t *prev = malloc(n * 4), *next = malloc(n * 4); char *in = calloc(n, 1);
    long head = -1, tail = -1, size = 0, hits = 0, hot_refs = 0, hot_hits = 0;
    #define UNLINK(u) { if (prev[u] >= 0) next[prev[u]] = next[u]; else head = next[u]; if (next[u] >= 0) prev[next[u]] = prev[u]; else tail = prev[u]; }
    #define PUSH_HEAD(u) { prev[u] = -1; next[u] = head; if (head >= 0) prev[head] = u; head = u; if (tail < 0) tail = u; }
    #define PUSH_TAIL(u) { next[u] = -1; prev[u] = tail; if (tail >= 0) next[tail] = u; tail = u; if (head < 0) head = u; }
    long per = (E + W - 1) / W;
    for (long r = 0; r * B < per; ++r) {
        for (long w = 0; w < W; ++w) {
            long b = w * per + r * B, e1 = w * per + per; if (e1 > E) e1 = E;
            for (long q = b; q < b + B && q < e1; ++q) {
                int32_t u = col[q]; int cold = od[u] <= kc;
                if (!cold) hot_refs++;
                if (in[u]) { hits++; if (!cold) { hot_hits++; UNLINK(u); PUSH_HEAD(u); } }
                else {
                    if (size == C) { long t = tail; UNLINK(t); in[t] = 0; size--; }
                    if (cold) { PUSH_TAIL(u); } else { PUSH_HEAD(u); }
                    in[u] = 1; size++;
                }
            }
        }
    }
    printf("C=%ld kcold=%d hit=%.4f (hot refs %.3f, hot hit %.4f)\n", C, kc, (double)hits / E, (double)hot_refs / E, hot_refs ? (double)hot_hits / hot_refs : 0);
    return 0;
}
