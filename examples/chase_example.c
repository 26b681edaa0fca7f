/* Plain-C caller of the C ABI (include/chase.h): no Python, no torch.
 *
 * Solves for the nev lowest eigenpairs of the complex-Hermitian 1-2-1 matrix tridiag(1, 2, 1)
 * (Table 1) on one GPU and checks them against the closed form
 * lambda_k = 2 - 2 cos(k pi / (N + 1)).  Exit status 0 on success.
 *
 * Build:  gcc -O2 -std=c11 examples/chase_example.c -Iinclude -I/usr/local/cuda/include \
 *             -Lpaper_2205_02491_b200 -lchase_b200 -L/usr/local/cuda/lib64 -lcudart -lm \
 *             -Wl,-rpath,$PWD/paper_2205_02491_b200 -o chase_example
 */
#define _DEFAULT_SOURCE 1   /* M_PI */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "chase.h"

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_)); return 1; } \
  } while (0)

int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 1000;
  const int nev = 20, nex = 12;
  const double tol = 1e-10;
  /* H: column-major complex double (re, im interleaved) */
  double* H = (double*)calloc((size_t)(2 * N * N), sizeof(double));
  if (!H) return 1;
  for (int64_t i = 0; i < N; ++i) {
    H[2 * (i + i * N)] = 2.0;
    if (i + 1 < N) {
      H[2 * ((i + 1) + i * N)] = 1.0;
      H[2 * (i + (i + 1) * N)] = 1.0;
    }
  }
  void *dH = NULL, *dV = NULL;
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&dH, sizeof(double) * 2 * N * N));
  CK(cudaMalloc(&dV, sizeof(double) * 2 * N * (nev + nex)));
  CK(cudaMemcpy(dH, H, sizeof(double) * 2 * N * N, cudaMemcpyHostToDevice));

  chase_init_args a;
  memset(&a, 0, sizeof(a));
  a.dtype = CHASE_C128;
  a.N = N;
  a.nev_max = nev;
  a.nex_max = nex;
  a.grid_rows = 1;
  a.grid_cols = 1;
  a.rank = 0;
  a.world_size = 1;
  a.nccl_unique_id = NULL;
  a.cuda_device = 0;
  a.cuda_stream = NULL;
  chase_handle* h = NULL;
  if (chase_init(&h, &a) != CHASE_OK) { fprintf(stderr, "chase_init failed\n"); return 1; }

  double vals[64];
  chase_report rep;
  const chase_status st = chase_solve(h, dH, N, N, nev, nex, 20, tol, vals, dV, N, &rep);
  if (st != CHASE_OK) { fprintf(stderr, "chase_solve: %s\n", chase_last_error(h)); return 1; }
  double err = 0.0;
  for (int k = 0; k < nev; ++k) {
    const double exact = 2.0 - 2.0 * cos((double)(k + 1) * M_PI / (double)(N + 1));
    err = fmax(err, fabs(vals[k] - exact));
  }
  printf("%s\nN=%lld nev=%d: %d iterations, %lld matvecs, %.3f s; max |lambda - exact| / ||H|| = %.2e\n",
         chase_version(), (long long)N, nev, rep.iterations, (long long)rep.matvecs, rep.t_all, err / 4.0);
  chase_finalize(h);
  cudaFree(dH);
  cudaFree(dV);
  free(H);
  return err / 4.0 <= tol ? 0 : 2;
}
