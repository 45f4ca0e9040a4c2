// Device-side data structures shared by the kernels and the engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rtnb {

// Geometry of one plan on the device (SURVEY.md §8 "Sizes").
//   G   oversampled grid side (even), L = G/2 the field-of-view window side,
//   lo  = (G-L)/2 first window row/col (preproc.cpp:152-156),
//   Gc  cropped coil k-space side, off = dc(G) - dc(Gc) its offset (planner.cpp:187-207)
struct Dims {
  int G, Gc, J, L, lo, off, N;
  int H;  // channel groups of k_rows2 (ceil(J / lines per block))
  float invG;
  // channel decomposition (group.cu): grp != 0 when this context is one member of a
  // device group owning a contiguous channel block; count_rho != 0 on the member whose
  // reductions include the (replicated) rho part of every Estimate dot product
  int grp;
  int count_rho;
};

// Channel decomposition across a device group (decomp.cpp:10-39).
// Every member owns channels [j0, j1) and replicates rho. The cross-channel sums
// are read straight from the peers' memory (NVLink / NVSwitch loads; members share
// one process, peer access enabled) in member order, so every member computes
// bit-identical totals.
constexpr int kMaxGroup = 8;
struct GroupView {
  int A;
  int h[kMaxGroup];                 // k_rows2 channel groups of each member
  const double2* rp[kMaxGroup];     // window channel-sum partials (H_d x L x L)
  const double2* rpo[kMaxGroup];    // SETUP: out-of-window partials sum_j conj(c_j) z_j (G x G)
  // cluster-fused applications (k_rho_sum): every member's channel terms rc_j (J_d x L x L)
  // and its first channel, so out.rho sums all channels in the single-device order
  const float2* rc[kMaxGroup];
  int jb[kMaxGroup + 1];            // member d owns channels [jb[d], jb[d+1])
};

// k_colsW epilogue modes: plain application, application + alpha*dx (CR), Newton setup
enum ColsWMode : int { CW_OP = 0, CW_OPALPHA = 1, CW_SETUP = 2 };

// largest K of any grid_reduce<K> (sizes the per-block partials buffer)
constexpr int kMaxReduce = 4;

enum Status : int { ST_OK = 0, ST_USAGE = 2, ST_DATA = 3, ST_SOLVER = 4, ST_DEADLINE = 6 };

// Per-frame device state. Scalars are indexed by Newton step m and CR iteration.
// All reductions are FP64 (types.hpp:47-59) and deterministic (fixed-order
// last-block reduction of per-block partials).
constexpr int kMaxSteps = 64;
struct StepRec {
  int iters;          // CR iterations completed (cg_per_step)
  int zero_rhs;       // rhs was exactly zero: CR returned without iterating
  double resid_win;   // |z - T(rho c)|^2 on the window (partial of StepStats.residual0^2)
  double resid_out;   // same outside the window
  double rhs_nrm2;    // |rhs|^2
};

struct DevState {
  int status;     // sticky error for the frame (ST_SOLVER on non-finite values)
  int cr_halt;    // skip the remaining CR work of the current step
  int cur_step;
  int rho_out_known;  // the current step's setup has classified rhs.rho outside the window
  unsigned int counter;  // last-block reduction ticket
  unsigned int pad2_;
  int z_out;      // the loaded data has a nonzero sample outside the window (k_z_outside)
  int rho_out_nz; // the setup wrote a nonzero rhs.rho entry outside the window
  StepRec steps[kMaxSteps];
  double scal[8];        // scratch scalar outputs (op-level calls)
  double gp[4];          // group mode: this member's SETUP partials {|rhs|^2, resid_out, resid_win, -}
};

struct GroupScal {
  int A;
  const DevState* st[kMaxGroup];
  const double* pcw[kMaxGroup];     // per-slot colsW partials {<dx,out>, |out|^2, <ap_prev,out>}
  const double* pcr[kMaxGroup];     // per-iteration CR partials {|ap|^2, |r|^2}
  const double* ss[kMaxGroup];      // final image: per-member sum_j |c_j|^2 (N x N)
};

// One-process-per-GPU groups (procgroup.hpp): every member's published barrier epoch
struct GroupFlags {
  int A;
  const int* flag[kMaxGroup];
};

// Deferred grid reductions of the budget-mode CR solve (pass path, one device): the
// producer (k_colsW's operator application, a k_crA / k_cr_fused recurrence that is not
// the step's last) writes one partial per block and exits; the next consumer in stream
// order (k_crA / k_cr_fused) forms the totals in every block, in one fixed order, so
// every block gets bit-identical values and the producer has no ticket or last-block tail.
struct DeferRed {
  const double* w;  // k_colsW partials {Re<dx,out>, |out|^2, Re<ap_prev,out>}, 3 per block
  int nw;           // their block count (0: the dots come from CrScalars as before)
  const double* c;  // the previous recurrence's partials {|ap|^2, |r|^2}, 2 per block
  int nc;           // their block count (0: none; iteration it-1's tail already ran)
  double* out;      // this recurrence's partials, 2 per block (nullptr: grid reduction + tail)
  // channel group, budget mode: the member partials of the application's dots (pcw) and of
  // the previous recurrence (pcr) summed in member order here, in place of k_grp_fin
  int grp;         // 1: dots from the members' grid-reduced partials (pcw); 2: from every
                   // member's per-block partials gw[m] (gnw[m] blocks), member by member
  GroupScal gs;
  const double* gw[kMaxGroup];
  int gnw[kMaxGroup];
};

// CR scalars of the current step: rar[k] = <r, A r> after apply k, ap2[k] = |ap|^2
// after update k, rn[k] = |r| after iteration k (cg_solve nlinv.cpp:179-234).
struct CrScalars {
  double* rar;
  double* ap2;
  double* rn;
  double* saa;   // fused path: |A r_k|^2 from the application
  double* spa;   // fused path: Re <ap_{k-1}, A r_k>
  double* pcw;   // group mode: this member's colsW partials, 3 per slot
  double* pcr;   // group mode: this member's k_cr_fused partials, 2 per iteration
};

}  // namespace rtnb
