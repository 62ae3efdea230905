// tile_plan.h -- host side of the tile-task factorisation of the large fronts (tiles.cuh).
#pragma once
#include <vector>

#include "plan.h"

namespace kkt {

// host mirror of the device TFront (tiles.cuh); same layout
struct alignas(16) TFrontHost {
  int s, r, w, nbp;
  int nt, cbase, nU, ch0;
  long long tbase;
  int nch, pad2;
};
static_assert(sizeof(TFrontHost) == 48, "TFrontHost layout");

struct TTask { int x, y, z, w; };  // = int4: type (| instance << 4), front, i | j << 16, k

struct TilePlanHost {
  std::vector<TFrontHost> fr;     // huge fronts in postorder
  std::vector<TTask> tasks;       // list-schedule order (topological)
  std::vector<int> hidx;          // [ns] huge-front index or -1
  std::vector<int> tch;           // child records: pairs {child supernode, offset into tcut}
  std::vector<int> tcut;          // per child record: nt + 1 cut positions (tiles.cuh TilePlan)
  std::vector<int> tkptr;         // [ncnt + 1] K-entry list range of every tile (counter indexing)
  std::vector<int> tkidx;         // K entry indices grouped by tile
  std::vector<long long> ibase;   // per front: offset of its nbp inverse diagonal tiles
  long long inv_doubles = 1;
  std::vector<int> ntask_by_type; // ASM, POTRF0, TRSM, CRIT, UPD
  long long pool_doubles = 1;     // tile pool per instance
  int ncnt = 1;                   // counters per instance
  double est_us = 0.0;            // simulated makespan (estimated task durations)
  bool ok = true;                 // false: a front has more children than the device task supports
};

// Build the task DAG of every huge front of P and order it by a list-scheduling simulation
// on `workers` workers (one instance; the caller replicates for batches).
void build_tile_plan(const Plan& P, int workers, TilePlanHost& out);

// Task DAG of the triangular solves through the huge fronts (tsolve.cuh): forward gathers,
// updates and chain steps, then backward updates and chain steps, list-scheduled the same way.
struct TSolvePlanHost {
  std::vector<TTask> tasks;       // x = type, y = front, z = i, w = k
  std::vector<int> cbase2;        // per front counter base (2 nt + 3 nbp + 2 counters each)
  std::vector<long long> pbase;   // per front partial-product slots (tsolve.cuh)
  long long part_doubles = 1;
  int ncnt = 1;
  double est_us = 0.0;
};
// chains: the panel of every front as one forward and one backward task (tsolve.cuh FCH / BCH)
void build_tile_solve_plan(const Plan& P, const TilePlanHost& tp, int workers, bool chains, TSolvePlanHost& out);

}  // namespace kkt
