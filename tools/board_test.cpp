// Cross-process test of the balancer's agreement board (csrc/board.h) on the
// CPU: P forked processes share one anonymous mapping, run D decision points
// with varying value counts (several board chunks) and random pauses, and
// check that everyone gets the elementwise max of all ranks' values.  Then a
// rank that stops publishing makes the others time out instead of hanging.
//   g++ -O2 -std=c++17 -I paper_2510_15882_b200/csrc tools/board_test.cpp -o board_test
//   ./board_test <ranks> <decisions>       -> "ok" on success
#include <sys/mman.h>
#include <sys/wait.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "board.h"

static double value(int rank, int d, int i) {
  return (double)(((uint64_t)(rank + 1) * 2654435761u + (uint64_t)d * 40503u + i * 97u) % 100003);
}

static int run(char* base, int nranks, int me, int decisions, int die_at) {
  uint64_t seq = 0;
  flx::Board b;
  b.base = base;
  b.nranks = nranks;
  b.me = me;
  b.seq = &seq;
  b.timeout_s = 2.0;
  std::mt19937 rng(1234 + me);
  for (int d = 0; d < decisions; ++d) {
    if (me == 0 && d == die_at) _exit(0);  // a rank that stops taking part
    const int n = 1 + (int)((d * 37u) % 150);  // 1..150 values: up to 3 chunks
    std::vector<double> v(n), want(n);
    for (int i = 0; i < n; ++i) {
      v[i] = value(me, d, i);
      want[i] = 0;
      for (int r = 0; r < nranks; ++r) want[i] = std::max(want[i], value(r, d, i));
    }
    if (rng() % 4 == 0) usleep(rng() % 300);
    int bad = -1;
    const int rc = flx::board_agree_max(b, v.data(), n, &bad);
    if (rc) return die_at >= 0 && rc == 1 ? 0 : 10 + rc;  // timeout expected after a death
    for (int i = 0; i < n; ++i)
      if (v[i] != want[i]) return 20;
  }
  return die_at >= 0 ? 30 : 0;  // with a dead rank the survivors must have timed out
}

static int trial(int nranks, int decisions, int die_at) {
  const size_t bytes = flx::board_bytes(16);
  char* base = (char*)mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS, -1, 0);
  if (base == MAP_FAILED) return 1;
  std::vector<pid_t> kids;
  for (int r = 0; r < nranks; ++r) {
    const pid_t p = fork();
    if (p == 0) _exit(run(base, nranks, r, decisions, die_at));
    kids.push_back(p);
  }
  int worst = 0;
  for (pid_t p : kids) {
    int st = 0;
    waitpid(p, &st, 0);
    const int rc = WIFEXITED(st) ? WEXITSTATUS(st) : 99;
    if (rc) worst = rc;
  }
  munmap(base, bytes);
  return worst;
}

int main(int argc, char** argv) {
  const int nranks = argc > 1 ? atoi(argv[1]) : 4;
  const int decisions = argc > 2 ? atoi(argv[2]) : 500;
  int rc = trial(nranks, decisions, -1);
  if (rc) {
    printf("agreement failed: %d\n", rc);
    return 1;
  }
  rc = trial(nranks, 50, 17);
  if (rc) {
    printf("dead-rank case failed: %d\n", rc);
    return 2;
  }
  printf("ok\n");
  return 0;
}
