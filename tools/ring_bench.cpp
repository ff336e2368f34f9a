// Pure C-ABI latency of one synchronous decision (no Python): launch mode
// vs the resident ring, mgb-warps and mgb-sm over 8 B200 ledgers.
//   g++ -O2 -std=c++17 tools/ring_bench.cpp -Iinclude -Lpaper_2107_08538_b200 -lgs \
//       -Wl,-rpath,$PWD/paper_2107_08538_b200 -o tools/ring_bench.bin
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <vector>

#include "gs.h"

extern "C" int gs_ring_stamps(gs_sched *s, unsigned long long *out5);

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  gs_engine *eng = nullptr;
  if (gs_engine_open(0, &eng)) { printf("engine: %s\n", gs_last_error()); return 1; }
  gs_spec spec{148, 180ll << 30, 64, 32, 65536, 233472};
  for (int policy : {GS_POLICY_MGB_WARPS, GS_POLICY_MGB_SM}) {
    for (int ring : {0, 1}) {
      std::vector<gs_device *> devs(8);
      for (int d = 0; d < 8; ++d) gs_device_create(eng, &spec, d, &devs[d]);
      gs_sched *s = nullptr;
      gs_sched_create(eng, devs.data(), 8, policy, 0, 1, &s);
      const int n = 4000;
      gs_engine_reserve_handles(eng, n + 1);
      if (ring && gs_sched_ring_start(s, n + 1, n + 1, 8)) { printf("ring: %s\n", gs_last_error()); return 1; }
      std::vector<double> sub, rel;
      double st_sum[4] = {0, 0, 0, 0};
      int st_n = 0;
      gs_decision dec, drain[64];
      for (int i = 0; i < n; ++i) {
        gs_probe p;
        memset(&p, 0, sizeof p);
        p.mem_bytes = 1ll << 30;
        p.heap_limit_bytes = 8 << 20;
        p.thread_blocks = 296;
        p.warps_per_block = 8;
        p.threads_per_block = 256;
        p.regs_per_thread = 32;
        p.total_warps = 296 * 8;
        p.handle = i;
        p.job = -1;
        p.level = GS_PROBE_FRESH;
        const double t0 = now_us();
        if (gs_submit(s, &p, &dec)) { printf("submit: %s\n", gs_last_error()); return 1; }
        const double t1 = now_us();
        sub.push_back(t1 - t0);
        unsigned long long ts[5];
        if (ring && gs_ring_stamps(s, ts) == 0) {
          for (int k = 0; k < 4; ++k) st_sum[k] += (double)(ts[k + 1] - ts[k]) / 1000.0;
          st_n++;
        }
        if (dec.outcome == GS_ASSIGN && i % 2) {  // keep the fleet partly loaded: release every other
          int64_t freed = 0;
          int32_t tried = 0, adm = 0;
          const double t2 = now_us();
          gs_release_redrive(s, dec.device, i, &freed, drain, 64, &tried, &adm);
          rel.push_back(now_us() - t2);
        }
      }
      if (ring) gs_sched_ring_stop(s);
      auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v.empty() ? 0 : v[v.size() / 2]; };
      printf("%s %s: submit median %.1f us, release+redrive median %.1f us (%zu / %zu calls)\n",
             policy == GS_POLICY_MGB_WARPS ? "mgb-warps" : "mgb-sm", ring ? "ring  " : "launch", med(sub), med(rel),
             sub.size(), rel.size());
      if (st_n)
        printf("   ring stamps (us): read cmd %.2f, exec %.2f, writeback %.2f, publish %.2f\n", st_sum[0] / st_n,
               st_sum[1] / st_n, st_sum[2] / st_n, st_sum[3] / st_n);
      fflush(stdout);
      gs_sched_destroy(s);
      for (gs_device *d : devs) gs_device_destroy(d);
    }
  }
  gs_engine_close(eng);
  return 0;
}
