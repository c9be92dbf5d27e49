// Panel grouping of the right-looking tiled Cholesky, shared by the
// single-GPU plan (gpb_api.cu build_chol_plan) and the multi-GPU schedule
// (dist_plan.cu).  Both must apply the same trailing updates to every tile --
// the same K split per update -- for the multi-GPU factor to equal the
// single-GPU one bit for bit.
#pragma once
#include <algorithm>
#include <cstdlib>
#include <vector>

namespace gpb {

constexpr int kMaxGroup = 8;

// Panels per trailing-update group (GPB_PANELS): larger groups cut the C
// passes further (K = G bi): G = 4 gives +0.5% at config 2 and +1.5% at
// n = 65536, G = 6 another +0.4% there; small grids keep G = 2 so the
// critical path stays short.
inline int chol_panels(int Ti) {
  const char* pg = getenv("GPB_PANELS");
  return std::max(1, std::min(kMaxGroup, pg ? atoi(pg) : (Ti >= 96 ? 6 : Ti >= 48 ? 4 : 2)));
}

// Group sizes: G, shrinking near the end where the trailing update no longer
// hides the group's critical path (GPB_TAIL, default 8: at most r / 8 panels
// when r tiles remain; 0 = fixed G): +0.5% at config 2.  GPB_FIRST: size of
// the first group, whose critical path runs before any trailing update can
// start (default 1 panel from 32 tiles: config 2 factor 338.8 -> 338.0 ms).
// The single-GPU plan passes other defaults when the trailing updates run on the
// int8 pipe (gpb_api.cu): there the group's own work is cheap next to the K it
// buys the update, so groups shrink later (r / 4) and the first one is full.
inline std::vector<int> chol_group_sizes(int Ti, int G, int tail_default = 8, int first_default = -1) {
  const char* te = getenv("GPB_TAIL");
  const int tail = te ? atoi(te) : tail_default;
  const char* fe = getenv("GPB_FIRST");
  const int first = fe ? atoi(fe) : (first_default >= 0 ? first_default : (Ti >= 32 ? 1 : 0));
  std::vector<int> sizes;
  for (int k0 = 0; k0 < Ti;) {
    int g = std::min(G, Ti - k0);
    if (k0 == 0 && first > 0) g = std::min(g, first);
    if (tail > 0) g = std::max(1, std::min(g, (Ti - k0) / tail));
    sizes.push_back(g);
    k0 += g;
  }
  return sizes;
}

}  // namespace gpb
