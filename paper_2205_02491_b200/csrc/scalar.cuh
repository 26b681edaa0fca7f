// Scalar traits: the library's non-GEMM kernels are written once for complex double (double2,
// interleaved re/im == torch.complex128) and real double (the real-symmetric variant).
#pragma once
#include <cuda_runtime.h>

namespace chase {

template <class T>
struct SC;

template <>
struct SC<double2> {
  static constexpr int ND = 2;          // doubles per element
  static constexpr bool is_complex = true;
  __host__ __device__ static double2 zero() { return make_double2(0.0, 0.0); }
  __host__ __device__ static double2 one() { return make_double2(1.0, 0.0); }
  __host__ __device__ static double2 make(double r, double i) { return make_double2(r, i); }
  __host__ __device__ static double re(double2 a) { return a.x; }
  __host__ __device__ static double im(double2 a) { return a.y; }
  __host__ __device__ static double2 conj(double2 a) { return make_double2(a.x, -a.y); }
  __host__ __device__ static double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
  __host__ __device__ static double2 sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
  __host__ __device__ static double2 mul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  }
  __host__ __device__ static double2 mulc(double2 a, double2 b) {   // conj(a) * b
    return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
  }
  __host__ __device__ static double2 scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
  __host__ __device__ static double abs2(double2 a) { return a.x * a.x + a.y * a.y; }
  __host__ __device__ static double2 div(double2 a, double2 b) {
    const double d = b.x * b.x + b.y * b.y;
    return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
  }
  __host__ __device__ static double2 neg(double2 a) { return make_double2(-a.x, -a.y); }
};

template <>
struct SC<double> {
  static constexpr int ND = 1;
  static constexpr bool is_complex = false;
  __host__ __device__ static double zero() { return 0.0; }
  __host__ __device__ static double one() { return 1.0; }
  __host__ __device__ static double make(double r, double) { return r; }
  __host__ __device__ static double re(double a) { return a; }
  __host__ __device__ static double im(double) { return 0.0; }
  __host__ __device__ static double conj(double a) { return a; }
  __host__ __device__ static double add(double a, double b) { return a + b; }
  __host__ __device__ static double sub(double a, double b) { return a - b; }
  __host__ __device__ static double mul(double a, double b) { return a * b; }
  __host__ __device__ static double mulc(double a, double b) { return a * b; }
  __host__ __device__ static double scale(double a, double s) { return a * s; }
  __host__ __device__ static double abs2(double a) { return a * a; }
  __host__ __device__ static double div(double a, double b) { return a / b; }
  __host__ __device__ static double neg(double a) { return -a; }
};

}  // namespace chase
