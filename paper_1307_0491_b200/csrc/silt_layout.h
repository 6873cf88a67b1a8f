// silt_layout.h — device data layout shared by the host runtime and kernels.
//
// HBM layout of one strip:
//   state[2][4]  : ping-pong SoA planes h, hu, hv, zb, each [ny][pitch] fp64,
//                  pitch = nx rounded up to 32 doubles (256 B rows)
//   ghost_s/n[2] : ghost rows -1 / ny per parity, [4][nx] (physical BC rows,
//                  periodic self-wrap or caller-given rows)
//   recv_s/n     : ghost rows received from neighbour strips, [4][nx] (x2 parities
//                  in the group's direct mode)
//   send_s/n     : edge rows 0 / ny-1 for neighbour strips, [4][nx]
//   ghost_w/e    : caller-given ghost columns (SILT_BC_GIVEN), [4][ny]
//   Control      : triple-buffered run-clock/reduction mailboxes
#pragma once
#include <stdint.h>

#include "silt_cuda.h"
#include "silt_physics_params.h"

#ifndef SILT_STEP_THREADS
#define SILT_STEP_THREADS 128
#endif
constexpr int kStepThreads = SILT_STEP_THREADS;  // warps per CTA x 32, one column strip each
constexpr int kCellsPerWarp = 30;   // lanes 1..30 own cells, 0/31 are x-halo

// One mailbox per launch index mod 3.  Launch n reads slot[n%3] (state n's
// reduced speeds + run clock), accumulates state n+1 into slot[(n+1)%3] and
// clears slot[(n+2)%3].  max_* hold the bits of non-negative doubles so that
// integer atomicMax orders them like the values.
struct Slot {
    unsigned long long max_sx;  // max over wet cells of the x axis speed
    unsigned long long max_sy;  // (adjacent: a multi-rank driver all-reduces
                                //  these two as float64 MAX)
    unsigned long long hmax;    // max depth of the strip (check_depth href)
    unsigned int wet;           // strip has a wet cell
    unsigned int err;           // error bits raised producing this state
    double t;                   // simulated time of this state
    double last_dt;
    long long steps;            // steps taken to reach this state
    int snap_idx;
    int state;                  // SILT_STATE_*
};

struct Control {
    Slot slot[3];
    double t_end;
    double fixed_dt;      // the caller's dt when fixed_mode is set
    long long max_steps;
    long long dt_cap;
    double* dt_log;
    const double* snaps;
    int n_snaps;
    unsigned int err_claim;
    unsigned int err_bits;
    int err_col, err_row;
    unsigned int item_ctr[3];  // warp-item mode: items taken per launch index (mod 3)
    int fixed_mode;       // 1: step_1d/step_2d with the caller's dt, applied as
                          // given (0, negative or NaN included), like the reference
    double err_info[6];
};

struct StepArgs {
    int dim, nx, ny, pitch;
    int j0;                 // global row of local row 0 (messages)
    int rows_per_block;
    int south_nbr, north_nbr, per_y_self;
    int write_edges_in_reduce;
    int quiet_skip;         // FAST: skip provably unchanged quiescent rows
    // Warp-item mode of the 2D step (short launches): the grid is one wave of
    // CTAs and warps pull (band, row block) items from Control::item_ctr.
    int warp_items, bands, n_items, warps_total;
    long long plane;        // doubles between the field planes of one parity
    // Row-block launch order (2D, long launches): launch li processes row
    // block rb_table[li][blockIdx.y]; rows with full-path (non-quiescent)
    // work mark rb_hot[li], from which rb_order_kernel builds the next order.
    int rb_order;
    int* rb_table[3];
    unsigned char* rb_hot[3];
    // Per launch: row block of blockIdx.y (nullptr: identity), and whether
    // this launch runs the run-clock epilogue (the interior launch of a
    // split step does not: the edge launch of the same step did).
    const int* rb_map;
    int epilogue;
    double dx, dy, cfl;
    silt_dev::Params P;
    int bc_type[4];
    int bc_super[4];
    double bc_q0[4];
    double bc_h0[4];
    double* state[2][4];
    double* ghost_s[2];
    double* ghost_n[2];
    // Ghost rows from / edge rows for neighbour strips, per state parity:
    // step n reads recv_*[n & 1] and writes send_*[(n + 1) & 1].  A driver
    // that copies rows between steps points both parities at one buffer; the
    // in-process group's direct mode points send_* at the neighbours' recv_*
    // (peer memory), so the step kernel itself delivers the rows.
    double* recv_s[2];
    double* recv_n[2];
    double* send_s[2];
    double* send_n[2];
    double* ghost_w;
    double* ghost_e;
    Control* ctl;
};
