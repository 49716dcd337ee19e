// fexp.cuh -- fp64 exp(num/den) for the FINOM scan kernels (sm_100a).
//
// The reference evaluates every kernel factor as np.exp(expo / epsilon)
// (kernel1d.py:142, :148) or np.exp(expo * inv_eps) (_kernels.py:140-159).
// q_div() reproduces the correctly rounded quotient expo/epsilon with one
// multiply and two FMAs (checked bit-exact against IEEE division on 2e7
// random (expo, eps) pairs, tests/fexp_check.cu run by
// tests/test_abi.py::test_fexp_host_arithmetic); fexp() is a
// 64-entry table + degree-6 polynomial exp, <= 1 ulp from libm, ~12 DP
// ops instead of ~27 for CUDA's exp() (measured 663 G exp/s on B200 vs
// 17.9 T DFMA/s, profiles/r01_fp64_probe.txt).  Arguments outside
// (-707, 709) take CUDA's exp() (denormal / overflow range).
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>

// Host builds (tests/fexp_check.cu) get the same arithmetic through libm.
#ifdef __CUDA_ARCH__
#define FB_MUL(a, b) __dmul_rn(a, b)
#define FB_ADD(a, b) __dadd_rn(a, b)
#define FB_SUB(a, b) __dsub_rn(a, b)
#define FB_FMA(a, b, c) __fma_rn(a, b, c)
#else
#define FB_MUL(a, b) ((a) * (b))
#define FB_ADD(a, b) ((a) + (b))
#define FB_SUB(a, b) ((a) - (b))
#define FB_FMA(a, b, c) std::fma(a, b, c)
#endif
#define FB_HD __host__ __device__ __forceinline__

namespace fb {

FB_HD double q_div(double num, double den, double inv) {
  double q0 = FB_MUL(num, inv);
  double r = FB_FMA(-q0, den, num);
  return FB_FMA(r, inv, q0);
}

// 2^(k/64) as (hi, lo) pairs; copied to shared memory by each CTA.
#define FB_EXP_TAB_VALUES \
  {0x1.0000000000000p+0, 0x0.0p+0}, \
  {0x1.02c9a3e778061p+0, -0x1.19083535b085dp-56}, \
  {0x1.059b0d3158574p+0, 0x1.d73e2a475b465p-55}, \
  {0x1.0874518759bc8p+0, 0x1.186be4bb284ffp-57}, \
  {0x1.0b5586cf9890fp+0, 0x1.8a62e4adc610bp-54}, \
  {0x1.0e3ec32d3d1a2p+0, 0x1.03a1727c57b53p-59}, \
  {0x1.11301d0125b51p+0, -0x1.6c51039449b3ap-54}, \
  {0x1.1429aaea92de0p+0, -0x1.32fbf9af1369ep-54}, \
  {0x1.172b83c7d517bp+0, -0x1.19041b9d78a76p-55}, \
  {0x1.1a35beb6fcb75p+0, 0x1.e5b4c7b4968e4p-55}, \
  {0x1.1d4873168b9aap+0, 0x1.e016e00a2643cp-54}, \
  {0x1.2063b88628cd6p+0, 0x1.dc775814a8495p-55}, \
  {0x1.2387a6e756238p+0, 0x1.9b07eb6c70573p-54}, \
  {0x1.26b4565e27cddp+0, 0x1.2bd339940e9d9p-55}, \
  {0x1.29e9df51fdee1p+0, 0x1.612e8afad1255p-55}, \
  {0x1.2d285a6e4030bp+0, 0x1.0024754db41d5p-54}, \
  {0x1.306fe0a31b715p+0, 0x1.6f46ad23182e4p-55}, \
  {0x1.33c08b26416ffp+0, 0x1.32721843659a6p-54}, \
  {0x1.371a7373aa9cbp+0, -0x1.63aeabf42eae2p-54}, \
  {0x1.3a7db34e59ff7p+0, -0x1.5e436d661f5e3p-56}, \
  {0x1.3dea64c123422p+0, 0x1.ada0911f09ebcp-55}, \
  {0x1.4160a21f72e2ap+0, -0x1.ef3691c309278p-58}, \
  {0x1.44e086061892dp+0, 0x1.89b7a04ef80d0p-59}, \
  {0x1.486a2b5c13cd0p+0, 0x1.3c1a3b69062f0p-56}, \
  {0x1.4bfdad5362a27p+0, 0x1.d4397afec42e2p-56}, \
  {0x1.4f9b2769d2ca7p+0, -0x1.4b309d25957e3p-54}, \
  {0x1.5342b569d4f82p+0, -0x1.07abe1db13cadp-55}, \
  {0x1.56f4736b527dap+0, 0x1.9bb2c011d93adp-54}, \
  {0x1.5ab07dd485429p+0, 0x1.6324c054647adp-54}, \
  {0x1.5e76f15ad2148p+0, 0x1.ba6f93080e65ep-54}, \
  {0x1.6247eb03a5585p+0, -0x1.383c17e40b497p-54}, \
  {0x1.6623882552225p+0, -0x1.bb60987591c34p-54}, \
  {0x1.6a09e667f3bcdp+0, -0x1.bdd3413b26456p-54}, \
  {0x1.6dfb23c651a2fp+0, -0x1.bbe3a683c88abp-57}, \
  {0x1.71f75e8ec5f74p+0, -0x1.16e4786887a99p-55}, \
  {0x1.75feb564267c9p+0, -0x1.0245957316dd3p-54}, \
  {0x1.7a11473eb0187p+0, -0x1.41577ee04992fp-55}, \
  {0x1.7e2f336cf4e62p+0, 0x1.05d02ba15797ep-56}, \
  {0x1.82589994cce13p+0, -0x1.d4c1dd41532d8p-54}, \
  {0x1.868d99b4492edp+0, -0x1.fc6f89bd4f6bap-54}, \
  {0x1.8ace5422aa0dbp+0, 0x1.6e9f156864b27p-54}, \
  {0x1.8f1ae99157736p+0, 0x1.5cc13a2e3976cp-55}, \
  {0x1.93737b0cdc5e5p+0, -0x1.75fc781b57ebcp-57}, \
  {0x1.97d829fde4e50p+0, -0x1.d185b7c1b85d1p-54}, \
  {0x1.9c49182a3f090p+0, 0x1.c7c46b071f2bep-56}, \
  {0x1.a0c667b5de565p+0, -0x1.359495d1cd533p-54}, \
  {0x1.a5503b23e255dp+0, -0x1.d2f6edb8d41e1p-54}, \
  {0x1.a9e6b5579fdbfp+0, 0x1.0fac90ef7fd31p-54}, \
  {0x1.ae89f995ad3adp+0, 0x1.7a1cd345dcc81p-54}, \
  {0x1.b33a2b84f15fbp+0, -0x1.2805e3084d708p-57}, \
  {0x1.b7f76f2fb5e47p+0, -0x1.5584f7e54ac3bp-56}, \
  {0x1.bcc1e904bc1d2p+0, 0x1.23dd07a2d9e84p-55}, \
  {0x1.c199bdd85529cp+0, 0x1.11065895048ddp-55}, \
  {0x1.c67f12e57d14bp+0, 0x1.2884dff483cadp-54}, \
  {0x1.cb720dcef9069p+0, 0x1.503cbd1e949dbp-56}, \
  {0x1.d072d4a07897cp+0, -0x1.cbc3743797a9cp-54}, \
  {0x1.d5818dcfba487p+0, 0x1.2ed02d75b3707p-55}, \
  {0x1.da9e603db3285p+0, 0x1.c2300696db532p-54}, \
  {0x1.dfc97337b9b5fp+0, -0x1.1a5cd4f184b5cp-54}, \
  {0x1.e502ee78b3ff6p+0, 0x1.39e8980a9cc8fp-55}, \
  {0x1.ea4afa2a490dap+0, -0x1.e9c23179c2893p-54}, \
  {0x1.efa1bee615a27p+0, 0x1.dc7f486a4b6b0p-54}, \
  {0x1.f50765b6e4540p+0, 0x1.9d3e12dd8a18bp-54}, \
  {0x1.fa7c1819e90d8p+0, 0x1.74853f3a5931ep-55},
__device__ __constant__ double EXP_TAB_C[64][2] = {FB_EXP_TAB_VALUES};
static const double EXP_TAB_H[64][2] = {FB_EXP_TAB_VALUES};


FB_HD int fb_lo(double d) {
#ifdef __CUDA_ARCH__
  return __double2loint(d);
#else
  uint64_t u; std::memcpy(&u, &d, 8); return (int)(uint32_t)u;
#endif
}
FB_HD int fb_hi(double d) {
#ifdef __CUDA_ARCH__
  return __double2hiint(d);
#else
  uint64_t u; std::memcpy(&u, &d, 8); return (int)(u >> 32);
#endif
}
FB_HD double fb_hilo(int hi, int lo) {
#ifdef __CUDA_ARCH__
  return __hiloint2double(hi, lo);
#else
  uint64_t u = ((uint64_t)(uint32_t)hi << 32) | (uint32_t)lo; double d; std::memcpy(&d, &u, 8); return d;
#endif
}

// Out-of-line slow path (denormal / overflow / NaN arguments): keeps the
// inlined fast path small.
#ifdef __CUDA_ARCH__
__device__ __noinline__ double fexp_slow(double x) { return exp(x); }
#else
inline double fexp_slow(double x) { return std::exp(x); }
#endif

// Polynomial / reduction constants: in constant memory on the device so the
// DFMAs take them as c[] operands instead of materialising immediates.
#define FB_EXP_CONSTS 0x1.71547652b82fep+6, 6755399441055744.0, 0x1.62e42fee00000p-7, \
    0x1.a39ef35793c76p-39, 1.0 / 720, 1.0 / 120, 1.0 / 24, 1.0 / 6
__device__ __constant__ double FB_EC[8] = {FB_EXP_CONSTS};
static const double FB_EH[8] = {FB_EXP_CONSTS};
#ifdef __CUDA_ARCH__
#define FB_K(i) FB_EC[i]
#else
#define FB_K(i) FB_EH[i]
#endif

FB_HD double fexp(double x, const double2* __restrict__ tab) {
#ifdef FB_DBG_NOEXP
  return 1.0 + x * 1e-30;  // timing experiment only: no exponential
#endif
  // fast path for |x| < 704 (high word compare; NaN/inf/large go out of line)
  if ((unsigned)(fb_hi(x) & 0x7fffffff) >= 0x40860000u) return fexp_slow(x);
  const double t = FB_FMA(x, FB_K(0), FB_K(1));   // x * 64/ln2 + 1.5*2^52
  const double n = FB_SUB(t, FB_K(1));
  double r = FB_FMA(n, -FB_K(2), x);
  r = FB_FMA(n, -FB_K(3), r);
  double p = FB_FMA(r, FB_K(4), FB_K(5));
  p = FB_FMA(p, r, FB_K(6));
  p = FB_FMA(p, r, FB_K(7));
  p = FB_FMA(p, r, 0.5);
  p = FB_FMA(p, r, 1.0);
  p = FB_MUL(p, r);
  const int ni = fb_lo(t);
  const double2 T = tab[ni & 63];
  const double res = FB_ADD(T.x, FB_FMA(T.x, p, T.y));
  return fb_hilo(fb_hi(res) + ((ni >> 6) << 20), fb_lo(res));
}

// exp(((-d) + ar) + ac) / eps): a stored kernel entry (kernel1d.py:148).
FB_HD double edge_exp(double d, double ar, double ac, double eps, double inv,
                      const double2* tab) {
  double num = FB_ADD(FB_ADD(-d, ar), ac);
  return fexp(q_div(num, eps, inv), tab);
}

// exp(((-g) + da) / eps) (lower) or exp(((-g) - da) / eps) (upper)
// (kernel1d.py:133, :140, :142).
FB_HD double ratio_exp(double g, double da, bool lower, double eps, double inv,
                       const double2* tab) {
  double num = lower ? FB_ADD(-g, da) : FB_SUB(-g, da);
  return fexp(q_div(num, eps, inv), tab);
}

// Dynamic-shift forms of the 2D sweeps (_kernels.py:140-159):
//   edge  exp(((a_o + b_t) - d) * inv_eps)
//   ratio exp(((a_i - a_{i-1}) - g) * inv_eps)   lower, da = a_i - a_{i-1}
//         exp(((a_{i-1} - a_i) - g) * inv_eps)   upper (row i-1 from row i)
FB_HD double edge_exp_dyn(double d, double ar, double ac, double inv, const double2* tab) {
  return fexp(FB_MUL(FB_SUB(FB_ADD(ar, ac), d), inv), tab);
}
FB_HD double ratio_exp_dyn(double g, double da, bool lower, double inv, const double2* tab) {
  return fexp(FB_MUL(FB_SUB(lower ? da : -da, g), inv), tab);
}
// Either form (dyn selects the 2D-absorbed expression).
FB_HD double edge_x(bool dyn, double d, double ar, double ac, double eps, double inv,
                    const double2* tab) {
  return dyn ? edge_exp_dyn(d, ar, ac, inv, tab) : edge_exp(d, ar, ac, eps, inv, tab);
}
FB_HD double ratio_x(bool dyn, double g, double da, bool lower, double eps, double inv,
                     const double2* tab) {
  return dyn ? ratio_exp_dyn(g, da, lower, inv, tab) : ratio_exp(g, da, lower, eps, inv, tab);
}

}  // namespace fb
