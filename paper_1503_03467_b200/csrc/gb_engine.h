// Argument block of the level engine (C ABI, mirrored by ctypes in
// paper_1503_03467_b200/engine.py).  All pointers are device pointers except
// hsta/hstb/hdots (pinned host).  Vectors are zero-halo padded.
#pragma once
#include <stdint.h>

typedef struct gb_level_engine_args {
  int L, w, max_chunk, max_outer;
  const double* BsT;       /* full blocked slot-major S B S (tiled level) */
  /* A: subband block-Jacobi PCG, already initialised (gb_bjcg_init) */
  const float* inv;        /* block-Jacobi 12x12 inverses, fp32 (gb_bj_setup) */
  double *xa, *ra, *pa, *apa, *za;
  void* sta;
  double* parta;
  void* hsta;
  /* B: lambda estimates; xb = normalized start 1 (power), x2 = normalized
   * start 2 (inverse iteration); state reset with max_iter for the power loop */
  double *xb, *yb, *x2, *xn, *ax, *cx, *cr, *cp, *cap;
  void* stb;
  double* partb;
  void* hstb;
  double* dots;            /* 4 device doubles */
  double* hdots;           /* 4 pinned doubles */
  double tol, inner_tol;
  int64_t inner_max_iter;
  /* outputs */
  double lam_min, lam_max;
  int64_t calls;
  int power_its, n_outer, breakdown;
  int inner_pcg;           /* 1: inner solves are block-Jacobi PCG (uses inv, cz) */
  int inner_its[64];
  double* cz;              /* PCG preconditioned residual of the inner solves */
  int layout;              /* 0: full box BsT, 1: symmetric band (gb_scale_box_symT);
                            * output vectors then carry gb_sym_overflow_elems tail */
  /* spectral mode 1: lambda_min from the Lanczos moments of the start vector
   * x2 (gb_lanczos.h) instead of inverse iteration; lz/hlz hold lz_cap
   * (alpha, beta) pairs (device / pinned host), lz_tol = relative change of
   * the emulated estimate between two checks at which the sequence stops */
  int spectral_mode, lz_cap;
  double* lz;
  double* hlz;
  double lz_tol;
  int lz_its, lz_rc;
  /* outputs: operator passes (phase-1 launches of the symmetric band SpMV)
   * carrying two vectors (PCG + spectral) and one vector */
  int64_t n_dual, n_single;
  /* optional live timing: CUDA events on the engine's stream around the first
   * ev_cap dual-vector phase-1 launches; durations (ms) into the pinned host
   * array ev_ms, ev_n of them (ev_events: engine-internal, pass NULL) */
  int ev_cap, ev_n;
  float* ev_ms;
  void* ev_events;
} gb_level_engine_args;
