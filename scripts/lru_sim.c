// LRU simulation of the factor-row access stream of one MTTKRP mode
// (scripts/lru_sim.py writes the stream): how many 128-B row fetches miss a
// fully associative LRU cache of C lines, with the stream replayed (a) in
// tree order, (b) interleaved the way the persistent kernel runs it: W
// concurrent cursors, each owning a contiguous task of T positions and
// advancing B positions per turn.
//   gcc -O2 -o /tmp/lru scripts/lru_sim.c && /tmp/lru stream.bin nrows C W T B
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

static int32_t *prv, *nxt;
static uint8_t* in;
static int32_t head = -1, tail = -1;
static int64_t size = 0, cap = 0, misses = 0;

static void unlink_(int32_t x) {
  if (prv[x] >= 0) nxt[prv[x]] = nxt[x]; else head = nxt[x];
  if (nxt[x] >= 0) prv[nxt[x]] = prv[x]; else tail = prv[x];
}
static void push_front(int32_t x) {
  prv[x] = -1; nxt[x] = head;
  if (head >= 0) prv[head] = x;
  head = x;
  if (tail < 0) tail = x;
}
static void access_(int32_t x) {
  if (in[x]) { unlink_(x); push_front(x); return; }
  ++misses;
  if (size == cap) { int32_t v = tail; unlink_(v); in[v] = 0; --size; }
  push_front(x); in[x] = 1; ++size;
}

int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  int64_t n; if (fread(&n, 8, 1, f) != 1) return 1;
  int32_t* s = malloc(n * 4); if (fread(s, 4, n, f) != (size_t)n) return 1; fclose(f);
  int64_t nrows = atoll(argv[2]);
  prv = malloc(nrows * 4); nxt = malloc(nrows * 4); in = calloc(nrows, 1);
  for (int a = 3; a + 3 < argc || a == 3; a += 4) {
    cap = atoll(argv[a]);
    int64_t W = atoll(argv[a + 1]), T = atoll(argv[a + 2]), B = atoll(argv[a + 3]);
    for (int64_t i = 0; i < nrows; ++i) in[i] = 0;
    head = tail = -1; size = 0; misses = 0;
    if (W <= 1) {
      for (int64_t i = 0; i < n; ++i) access_(s[i]);
    } else {
      // cursors take tasks of T positions in order as they finish
      int64_t* pos = malloc(W * 8); int64_t* end = malloc(W * 8);
      int64_t next = 0, live = 0;
      for (int64_t w = 0; w < W; ++w) {
        if (next < n) { pos[w] = next; end[w] = next + T < n ? next + T : n; next = end[w]; ++live; }
        else { pos[w] = end[w] = 0; }
      }
      while (live) {
        live = 0;
        for (int64_t w = 0; w < W; ++w) {
          if (pos[w] >= end[w]) {
            if (next < n) { pos[w] = next; end[w] = next + T < n ? next + T : n; next = end[w]; }
            else continue;
          }
          int64_t e = pos[w] + B < end[w] ? pos[w] + B : end[w];
          for (int64_t i = pos[w]; i < e; ++i) access_(s[i]);
          pos[w] = e; ++live;
        }
      }
      free(pos); free(end);
    }
    printf("cap %lld lines (%.1f MB) W %lld T %lld B %lld: accesses %lld misses %lld (%.2f GB of 128-B rows)\n",
           (long long)cap, cap * 128 / 1e6, (long long)W, (long long)T, (long long)B, (long long)n,
           (long long)misses, misses * 128 / 1e9);
    fflush(stdout);
    if (argc <= 7) break;
  }
  return 0;
}
