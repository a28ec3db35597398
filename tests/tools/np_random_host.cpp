// Host build of csrc/np_random.cuh for the CPU tests (tests/test_skeleton.py):
// the same restatement of numpy's default_rng stream the skeleton kernel runs,
// compiled with g++ -ffp-contract=off and checked against numpy itself.
#include "../../paper_2410_10759_b200/csrc/np_random.cuh"

using namespace sp::nprand;

extern "C" {

void nr_seed_state(uint64_t seed, uint64_t* out) { seed_sequence_state(seed, out); }

void nr_pcg_state(uint64_t seed, uint64_t* out) {
  const Pcg64 g = pcg64_from_seed(seed);
  out[0] = (uint64_t)(g.state >> 64);
  out[1] = (uint64_t)g.state;
  out[2] = (uint64_t)(g.inc >> 64);
  out[3] = (uint64_t)g.inc;
}

double nr_log1p(double x) { return glibc_log1p(x); }

void nr_log1p_many(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = glibc_log1p(x[i]);
}

// the host libm's log1p, the one numpy's distributions call (log1p@GLIBC_2.2.5)
void nr_libm_log1p_many(const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) y[i] = ::log1p(x[i]);
}

void nr_skeleton(uint64_t seed, int64_t horizon, double scale, int64_t lo, int64_t hi, int64_t exec_max,
                 double* arr, int64_t* choice, int64_t* execs) {
  Pcg64 g = pcg64_from_seed(seed);
  double run = 0.0;
  for (int64_t k = 0; k < horizon; ++k) {
    const double e = r_mul(scale, standard_exponential(g));
    run = k == 0 ? e : r_add(run, e);
    arr[k] = run;
  }
  for (int64_t k = 0; k < horizon; ++k) choice[k] = integers(g, 0, hi - lo) + lo;
  for (int64_t k = 0; k < horizon; ++k) execs[k] = integers(g, 1, exec_max + 1);
}

}  // extern "C"
