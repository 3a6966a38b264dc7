// registry.h — table of compiled batch-kernel instantiations (one per
// (tier, kind, dim, input type, finalisation)); filled by static registrars in
// the generated per-instance translation units (build.py).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffd {

struct Problem;

struct BatchKey {
  int tier;    // 0: fp32 main tier, 1: exact int64 fallback tier, 2: fp64 DTW tier
  int kind;    // Kind
  int dim;
  int int_in;  // input coordinates int32
  int fin;     // Fin
};

using LaunchFn = cudaError_t (*)(const Problem&, int grid, cudaStream_t);
using OccFn = int (*)();

struct BatchEntry {
  BatchKey key;
  LaunchFn launch;
  OccFn occupancy;        // resident CTAs per SM
  int8_t rmap[17];        // R -> smallest instantiated R ≥ R (0 if none)
  const char* name;
};

void register_batch(const BatchEntry& e);
const BatchEntry* find_batch(const BatchKey& k);

struct Registrar {
  explicit Registrar(const BatchEntry& e) { register_batch(e); }
};

}  // namespace ffd
