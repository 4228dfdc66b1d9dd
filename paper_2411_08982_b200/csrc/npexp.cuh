// npexp.cuh -- float64 exp with the bits of the reference's np.exp.
//
// The reference's softmax is e = np.exp(z - rowmax) (router.py:153).  numpy
// (2.x, x86-64) dispatches float64 exp on AVX512_SKX hosts to the SVML
// routine bundled with it (__svml_exp8_ha, numpy/_core/src/umath/svml); on
// this build container -- where tests/golden/ was generated from the
// reference -- that is the path np.exp takes.  That routine is not
// correctly rounded (it differs from the correctly rounded exp in ~5% of
// arguments, and CUDA's exp differs from both), so a near-tie between two
// probabilities could order differently on the device.  np_exp restates the
// routine's arithmetic step for step -- the same constants, the same fused
// operations and rounding modes -- so the device's full_probs carry the
// reference's bits:
//
//   t  = fma_rz(x, log2(e), 1.5*2^48 + 1023)   sixteenths of x*log2(e), truncated
//   n  = t - (1.5*2^48 + 1023)                 multiple of 1/16
//   j  = low 4 bits of t                       2^(j/16) = hi[j] + lo[j]
//   r  = (x - n*ln2_hi) - n*ln2_lo             two FMAs
//   p  = ((c5 r + c4) r^2 + (c3 r + c2)) r^2 + (c1 r + c0)     ~ (e^r - 1) / r
//   e  = 2^floor(n) * (hi[j] * (p r + lo[j]) + hi[j])
//
// oracle/lynx_oracle.py (svml_exp_ha) restates the same steps in exact
// rational arithmetic; tests/test_oracle_golden.py pins it against np.exp
// bit for bit.  Arguments with |x| >= 707.7 (or NaN) take SVML's scalar
// fallback there; here they use CUDA's exp (results <= 2^-1021, inf or NaN:
// no routing decision can depend on their last bit).
#pragma once

namespace lynx {

__device__ const double kNpExpHi[16] = {
    0x1.0000000000000p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0, 0x1.2387a6e756238p+0,
    0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0, 0x1.5ab07dd485429p+0,
    0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0, 0x1.9c49182a3f090p+0,
    0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0, 0x1.ea4afa2a490dap+0};
__device__ const double kNpExpLo[16] = {
    0.0,                     0x1.79aa65d837b6dp-54,  -0x1.01b15eaa59348p-55, 0x1.68efde3a8a894p-54,
    0x1.34d754db0abb6p-55,   0x1.59f48a72a4c6dp-55,  0x1.690cebb7aafb0p-56,  0x1.063e1e21c5409p-54,
    -0x1.3b3efbf5e2228p-54,  -0x1.b32dcb94da51dp-56, 0x1.db72fc1f0eab4p-55,  0x1.1affc2b91ce27p-56,
    0x1.c1a7792cb3387p-55,   0x1.36eae30af0cb3p-56,  0x1.4a385a63d07a7p-56,  -0x1.ff7128fd391f0p-55};

// The 2^(j/16) table in shared memory: 32 doubles (hi[0..15], lo[0..15]),
// staged by threads 0..31 before the kernel's griddep_wait, so the cold
// global load overlaps the predecessor kernel (the caller synchronises).
__device__ __forceinline__ void np_exp_stage(double* s_tab) {
  if (threadIdx.x < 32) s_tab[threadIdx.x] = threadIdx.x < 16 ? kNpExpHi[threadIdx.x] : kNpExpLo[threadIdx.x - 16];
}

// SVML's scalar fallback range (|x| >= 707.7, NaN): out of line, it never
// runs for softmax arguments of a finite row with spread < 707.
__device__ __noinline__ double np_exp_rare(double x) { return exp(x); }

__device__ __forceinline__ double np_exp(double x, const double* s_tab) {
  constexpr double kLog2e = 0x1.71547652b82fep+0, kShift = 0x1.8000000003ff0p+48;
  constexpr double kLn2Hi = 0x1.62e42fefa39efp-1, kLn2Lo = 0x1.abc9e3b39803fp-56;
  constexpr double c5 = 0x1.7411836940c04p-10, c4 = 0x1.1101cbbc265c0p-7, c3 = 0x1.55557242d68fep-5;
  constexpr double c2 = 0x1.5555553939732p-3, c1 = 0x1.000000000d008p-1, c0 = 0x1.fffffffffff70p-1;
  if (!(fabs(x) < 0x1.61da04cbafe44p+9)) return np_exp_rare(x);
  const double t = __fma_rz(x, kLog2e, kShift);
  const double n = __dsub_rn(t, kShift);
  const int j = static_cast<int>(__double_as_longlong(t) & 15);
  double r = __fma_rn(-n, kLn2Hi, x);
  r = __fma_rn(-kLn2Lo, n, r);
  const double r2 = __dmul_rn(r, r);
  double p = __fma_rn(c5, r, c4);
  const double q = __fma_rn(c3, r, c2);
  const double s = __fma_rn(c1, r, c0);
  p = __fma_rn(r2, p, q);
  p = __fma_rn(r2, p, s);
  const double hi = s_tab[j], lo = s_tab[16 + j];
  p = __fma_rn(p, r, lo);
  p = __fma_rn(hi, p, hi);
  // 2^floor(n) by exponent arithmetic: p in [1, 2) and the result normal
  // for |x| < 707.7, so adding to the exponent field is exact (= vscalefpd)
  const unsigned long long e = static_cast<unsigned long long>(static_cast<long long>(floor(n))) << 52;
  return __longlong_as_double(static_cast<long long>(static_cast<unsigned long long>(__double_as_longlong(p)) + e));
}

}  // namespace lynx
