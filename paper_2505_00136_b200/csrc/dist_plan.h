// Multi-GPU schedule of the tiled GP (host-only): 2D block-cyclic layout and
// the per-rank operation lists (the schedule IR of gpb200.h) that the device
// executor (dist.cu) runs and the CPU interpreter of the tests replays.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "gpb200.h"

namespace gpb {

// Offsets of the vector buffer GPB_BUF_VEC (doubles).  BETA, ALPHA and
// LOGDIAG are contiguous: one all-reduce replicates them.
enum VecSlot { V_Y = 0, V_BETA, V_ALPHA, V_LOGDIAG, V_ACC, V_TMP, V_RECV, V_RED, V_NSLOT };

struct DistLayout {
  int rank = 0, world = 1, P = 1, Q = 1, my_p = 0, my_q = 0;
  int64_t n = 0, np_ = 0, bi2 = 0;
  int Ti = 0, bi = 0, G = 2;
  int bp_user = 0, b_user = 0;      // PadMap of gpb_layout
  std::vector<int> slot;            // Ti x Ti: slot of owned tile (i, j), else -1
  std::vector<int> own_i, own_j;    // owned tiles in slot order (row-major)
  int rows_per = 0;                 // panel tiles per panel of this process row
  int cnt_max = 0;                  // column-panel tiles per (process row, panel)
  std::vector<int> jpos;            // position of j in J(j % P, my_q)
  int cntx = 0;                     // X-row tiles per column of this process row
  std::vector<int> rpos;            // position of r in R(r % Q) (rows r % P == my_p)
  int64_t bufsz[GPB_NBUF] = {0};
  int64_t vec[V_NSLOT] = {0};
  int nevents = 0;
  bool p2p = false;                 // peer-memory panel exchange (gpb_dist_set_exchange)
  int planes = 0;                   // digit planes per operand of the trailing updates (0: FP64 DMMA)
  int owner(int i, int j) const { return (i % P) * Q + (j % Q); }
  int nown() const { return static_cast<int>(own_i.size()); }
};

// returns a gpb_status; fills the layout of rank `rank` of a P x Q grid
int dist_layout(int rank, int world, int P, int Q, int64_t n, int64_t tiles_per_dim, DistLayout* out,
                std::string* err, int exchange = 0);
// position of panel tile j in process column q's column-panel slot list
// J(j mod P, q), and that list's largest length over the process rows
int col_pos(const DistLayout& L, int j);
int col_cnt_max(const DistLayout& L, int q);

// phase 0: assembly + factorisation (+ replication of the inverse diagonal
// tiles); 1: beta / alpha solves (+ replication of beta, alpha, log-diagonal);
// 2: gradient (distributed TRTRI + LAUUM + trace pass + all-reduce)
void dist_plan(const DistLayout& L, int phase, std::vector<gpb_op>* ops, std::vector<gpb_op_job>* jobs);

}  // namespace gpb
