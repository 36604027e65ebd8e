// Opt-in per-kernel timing with CUDA events on the launching stream
// (ttb_prof_enable / ttb_prof_dump).  Off by default: zero cost on the hot
// path apart from one branch per launch site.
#pragma once
#include "common.cuh"

namespace ttb {

bool prof_on();
void prof_record(const char* name, cudaStream_t st, bool begin);
// non-timing counter shown by ttb_prof_dump (e.g. Jacobi sweeps)
void prof_note(const char* name, double value);

struct ProfScope {
  const char* name;
  cudaStream_t st;
  bool on;
  ProfScope(const char* n, cudaStream_t s) : name(n), st(s), on(prof_on()) {
    if (on) prof_record(name, st, true);
  }
  ~ProfScope() {
    if (on) prof_record(name, st, false);
  }
};

}  // namespace ttb
