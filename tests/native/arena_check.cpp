// Randomized check of the executor's job arena (csrc/gs_arena.h) on the
// host: a fake slab base, random all-or-nothing requests and frees against
// a byte-level occupancy model.  Prints "ok <placed> <refused>" or fails.
#include <stdio.h>
#include <stdlib.h>

#include <random>
#include <thread>
#include <vector>

#include "../../paper_2107_08538_b200/csrc/gs_arena.h"

#define REQUIRE(c)                                           \
  do {                                                       \
    if (!(c)) {                                              \
      fprintf(stderr, "FAIL line %d: %s\n", __LINE__, #c);   \
      return 1;                                              \
    }                                                        \
  } while (0)

int main(int argc, char **argv) {
  const int64_t G = gsa::kGranule;
  const int64_t slab = 64 * G;
  std::vector<char> own(slab / G, 0);  // granule -> owned
  char *base = (char *)(uintptr_t)(1ull << 40);  // never dereferenced
  gsa::Arena a(0, base, slab);
  std::mt19937_64 rng(argc > 1 ? atoll(argv[1]) : 7);
  struct Job { std::vector<int64_t> req; std::vector<void *> p; };
  std::vector<Job> live;
  int placed = 0, refused = 0;
  for (int step = 0; step < 20000; ++step) {
    if (live.empty() || rng() % 3) {
      Job j;
      const int nb = 1 + rng() % 5;
      for (int b = 0; b < nb; ++b) j.req.push_back(1 + (int64_t)(rng() % (9 * G)));
      double w = 0;
      if (a.alloc_all(j.req, j.p, false, &w)) {
        for (size_t i = 0; i < j.req.size(); ++i) {
          REQUIRE(j.p[i] != nullptr);
          const int64_t off = (char *)j.p[i] - base;
          REQUIRE(off % G == 0 && off >= 0);
          const int64_t n = (j.req[i] + G - 1) / G;
          REQUIRE(off / G + n <= slab / G);
          for (int64_t g = off / G; g < off / G + n; ++g) {
            REQUIRE(!own[g]);  // no overlap with any live allocation
            own[g] = 1;
          }
        }
        live.push_back(j);
        ++placed;
      } else {
        for (void *p : j.p) REQUIRE(p == nullptr);  // all or nothing
        ++refused;
      }
    } else {
      const size_t k = rng() % live.size();
      Job j = live[k];
      live.erase(live.begin() + k);
      for (size_t i = 0; i < j.req.size(); ++i) {
        const int64_t off = (char *)j.p[i] - base;
        for (int64_t g = off / G; g < off / G + (j.req[i] + G - 1) / G; ++g) own[g] = 0;
      }
      a.free_all(j.p, j.req);
    }
    int64_t used = 0;
    for (char c : own) used += c;
    REQUIRE(a.in_use() == used * G);
  }
  for (Job &j : live) a.free_all(j.p, j.req);
  REQUIRE(a.in_use() == 0);
  // everything coalesced back: the whole slab is one hole again
  {
    std::vector<int64_t> r{slab};
    std::vector<void *> p;
    REQUIRE(a.alloc_all(r, p, false, nullptr) && p[0] == base);
    a.free_all(p, r);
  }
  // limit: a run's capacity below the slab
  REQUIRE(a.reset(10 * G));
  {
    std::vector<int64_t> r{11 * G};
    std::vector<void *> p;
    REQUIRE(!a.alloc_all(r, p, true, nullptr));  // larger than the limit: refused even when waiting
    std::vector<int64_t> r2{10 * G};
    REQUIRE(a.alloc_all(r2, p, false, nullptr));
    REQUIRE(!a.reset(64 * G));  // not between runs
    a.free_all(p, r2);
  }
  REQUIRE(a.reset(slab));
  // a waiting request is admitted by a free (fragmentation wait)
  {
    std::vector<int64_t> r1{40 * G}, r2{40 * G};
    std::vector<void *> p1, p2;
    REQUIRE(a.alloc_all(r1, p1, false, nullptr));
    std::thread t([&] {
      std::this_thread::sleep_for(std::chrono::milliseconds(50));
      a.free_all(p1, r1);
    });
    double waited = 0;
    REQUIRE(a.alloc_all(r2, p2, true, &waited));
    t.join();
    REQUIRE(waited >= 40.0);
    a.free_all(p2, r2);
  }
  printf("ok %d %d\n", placed, refused);
  return 0;
}
