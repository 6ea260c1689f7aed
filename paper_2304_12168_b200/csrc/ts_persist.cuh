// Persistent CTA loop: one cooperative kernel runs whole CTA iterations
// (centering.py:263-358 / _step_arrays 172-213) until the solve stops, the
// host must do maintenance (250-recheck), or the trace ring needs a flush —
// exactly the exit rule of the graph's WHILE node (set_cond).
//
// Why: on L2-resident matrices (C1, C3) a pass is a few microseconds of
// work, and the per-kernel fixed costs inside a graph (launch, ramp, drain,
// the finisher's serial state logic) were a third to a half of every
// iteration (tools/class_breakdown.py).
//
// Measured result (B200, round 1): SLOWER than the graph path on every
// config — C1 131-159 vs 123-132 us/it, C3 102-108 vs 90-105, C4 332 vs
// 254 — because a 148..592-block phase barrier costs about what a graph
// kernel boundary costs (~3.5 us), and the bodies lose the read-only x path
// and keep their epilogues in local memory.  Kept as an opt-in
// (TS_PERSIST=1) for study; parity-green (the full -m gpu suite passes).
//
// Here every phase is the SAME device
// body the standalone pass kernels run, over its own block range [0, P) of
// the co-resident grid, and a phase ends in phase_end(): one atomic arrival
// per block, the last arriver reduces the partials in the fixed order, runs
// the finisher, and releases the grid.  Decisions (order t, stop, NE clause,
// retry) stay in the same finishers as in graph mode.
#pragma once

#include "ts_cta.cuh"
#include "ts_matrix.cuh"

namespace ts {

enum : int { PK_NONE = 0, PK_COLS = 1, PK_TILE = 2, PK_SHORT = 3, PK_WARP = 4 };

// one direction of the matrix as the persistent loop runs it
struct PDir {
  int kind = PK_NONE;
  int P = 1;   // blocks [0, P) run the pass body; the rest only take part in the barrier
  int Pc = 1;  // PK_TILE: combine grid
  int64_t nct = 0;
  DenseRows d{};
  CsrRows c{};
};

// Epilogues are passed by reference from the loop down to the bodies and
// phase_end: one object per phase, no by-value copies (a by-value copy into
// the inlined helper was observed to misplace the derived members).
template <class Epi>
__device__ __forceinline__ void prun(const PDir& D, const double* x, Epi& epi, const Work& wk) {
  const int64_t b = blockIdx.x;
  switch (D.kind) {
    case PK_COLS:
      if (b < D.P) body_cols_tile<Epi, 2, true>(D.d, x, XS{}, epi, wk, b, D.P);
      phase_end(epi, wk, wk.facc, D.P);
      break;
    case PK_TILE:
      if (b < D.P) body_rows_tile<Epi, true>(D.d, x, XS{}, epi, wk.npart, b, D.P);
      grid_sync(wk.gbar);
      if (b < D.Pc) body_tile_combine<Epi, true>(D.d.m, D.nct, wk.npart, epi, wk, b, D.Pc);
      phase_end(epi, wk, nullptr, D.Pc);
      break;
    case PK_SHORT:
      if (b < D.P) body_rows_short<CsrRows, Epi, true>(D.c, x, XS{}, epi, wk, b, D.P);
      phase_end(epi, wk, nullptr, D.P);
      break;
    default:  // PK_WARP
      if (b < D.P) body_rows_warp<Epi, true>(D.c, x, XS{}, epi, wk, b, D.P);
      phase_end(epi, wk, nullptr, D.P);
      break;
  }
}

template <class Epi>
__device__ __forceinline__ void vrun(int64_t len, int P, Epi& epi, const Work& wk) {
  if ((int64_t)blockIdx.x < P) body_vec<Epi, true>(len, epi, wk, blockIdx.x, P);
  phase_end(epi, wk, nullptr, P);
}

struct CtaLoop {
  SolveState* st;
  KrylovPtrs kp;
  double* x;
  int64_t m, n;
  int gram;
  PDir T, N;      // A^T v, A v
  int Pm, Pmn;    // vector phases over m (candidates) and max(m, n) (update)
  Work wk;        // wk.gbar: the grid barrier
};

__global__ void __launch_bounds__(kNT, kMinBlocks) k_cta_loop(CtaLoop L) {
  SolveState* s = L.st;
  __shared__ int go, tt;
  if (blockIdx.x == 0 && threadIdx.x == 0)
    atomicAdd(reinterpret_cast<unsigned long long*>(&s->launches), 1ull);
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const bool room = (s->trace_count - s->trace_flushed) < (long long)s->seg_cap;
      go = (s->status == TS_RUNNING && s->maint == MAINT_NONE && room &&
            !*reinterpret_cast<volatile unsigned*>(&L.wk.gbar->abort))
               ? 1
               : 0;
      tt = s->t;
    }
    __syncthreads();
    if (!go) break;
    const int t = tt;
    for (int i = 1; i <= t; ++i) {
      const double* src = L.kp.p[i - 1];
      if (L.gram) {
        EpiCtaQ eq;
        eq.st = s; eq.q = L.kp.q[i - 1]; eq.i = i; eq.tclass = 1;
        if (eq.active()) prun(L.T, src, eq, L.wk);
        src = L.kp.q[i - 1];
      }
      EpiCtaP ep;
      ep.st = s; ep.pprev = L.kp.p[i - 1]; ep.p = L.kp.p[i]; ep.i = i; ep.with_solve = 1; ep.tclass = 0;
      if (ep.active()) prun(L.N, src, ep, L.wk);
    }
    EpiCtaCand ec;
    ec.st = s; ec.kp = L.kp; ec.m = L.m; ec.tclass = 2;
    if (ec.active()) vrun(L.m, L.Pm, ec, L.wk);
    EpiCtaUpd eu;
    eu.st = s; eu.kp = L.kp; eu.x = L.x; eu.m = L.m; eu.n = L.n; eu.gram = L.gram; eu.tclass = 2;
    if (eu.active()) vrun(L.m > L.n ? L.m : L.n, L.Pmn, eu, L.wk);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 &&
      *reinterpret_cast<volatile unsigned*>(&L.wk.gbar->abort) && s->status == TS_RUNNING) {
    s->status = TS_NUMERICAL_FAILURE;  // barrier watchdog: never expected
    s->detail = TS_DETAIL_DEVICE_WATCHDOG;
  }
}

}  // namespace ts
