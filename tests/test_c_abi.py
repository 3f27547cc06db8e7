"""The boundary is plain C: include/tk.h compiles as C99 and a C program links libtk_b200.so and drives
the host half of the API (spaces, tensors, contraction output, workspace sizes, errors) -- no GPU needed.
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2508_10076_b200")
LIB = os.path.join(LIBDIR, "libtk_b200.so")

PROGRAM = r'''
#include <stdio.h>
#include <string.h>
#include "tk.h"

#define CHECK(x) do { tk_status s_ = (x); if (s_ != TK_OK) { printf("FAIL %s: %d %s\n", #x, (int)s_, tk_last_error()); return 1; } } while (0)

int main(void) {
  tk_space* V = NULL;
  CHECK(tk_space_parse("U1[-1:2, 0:3, 1:2]", &V));
  int32_t ns = 0; int64_t dim = 0; int32_t dual = -1, width = 0;
  CHECK(tk_space_info(V, &ns, &dim, &dual, &width));
  if (ns != 3 || dim != 7 || dual != 0) { printf("FAIL info %d %lld %d\n", ns, (long long)dim, dual); return 1; }
  tk_space* cod[2] = {V, V};
  tk_space* dom1[1] = {V};
  tk_tensor *A = NULL, *B = NULL, *C = NULL;
  CHECK(tk_tensor_create(TK_F64, 2, cod, 1, dom1, &A));
  CHECK(tk_tensor_create(TK_F64, 1, dom1, 2, cod, &B));
  const int32_t la[3] = {1, 2, 3}, lb[3] = {3, 4, 5}, lc[4] = {1, 4, 2, 5};
  CHECK(tk_contract_output(A, la, B, lb, lc, 2, &C));
  int64_t na = 0, nb = 0, nc = 0;
  CHECK(tk_tensor_nelems(A, &na)); CHECK(tk_tensor_nelems(B, &nb)); CHECK(tk_tensor_nelems(C, &nc));
  size_t ws = 0;
  CHECK(tk_contract_workspace(A, la, B, lb, C, lc, &ws));
  /* an error path: a label of C that is not open */
  const int32_t bad[4] = {1, 4, 2, 9};
  tk_tensor* D = NULL;
  tk_status s = tk_contract_output(A, la, B, lb, bad, 2, &D);
  if (s != TK_ERR_UNKNOWN_LABEL) { printf("FAIL expected UNKNOWN_LABEL, got %d\n", (int)s); return 1; }
  printf("OK %lld %lld %lld %zu %s\n", (long long)na, (long long)nb, (long long)nc, ws, tk_version());
  tk_tensor_release(C); tk_tensor_release(B); tk_tensor_release(A); tk_space_release(V);
  return 0;
}
'''


@pytest.mark.skipif(shutil.which("gcc") is None, reason="no C compiler")
def test_header_is_c99_and_host_api_runs_from_c(tmp_path):
    if not os.path.exists(LIB):
        pytest.skip("library not built")
    src = tmp_path / "abi.c"
    src.write_text(PROGRAM)
    exe = tmp_path / "abi"
    cc = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", str(src),
                         "-I", os.path.join(ROOT, "include"), "-L", LIBDIR, "-ltk_b200",
                         "-Wl,-rpath," + LIBDIR, "-o", str(exe)], capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert run.returncode == 0 and run.stdout.startswith("OK"), run.stdout + run.stderr


GPU_PROGRAM = r'''
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <cuda_runtime.h>
#include "tk.h"

#define CHECK(x) do { tk_status s_ = (x); if (s_ != TK_OK) { printf("FAIL %s: %d %s\n", #x, (int)s_, tk_last_error()); return 1; } } while (0)

int main(void) {
  tk_space* V = NULL;
  CHECK(tk_space_parse("fU1xU1[(0,0):3, (1,1):2, (1,-1):2, (2,0):2]", &V));
  tk_space* cod[2] = {V, V};
  tk_space* dom1[1] = {V};
  tk_tensor *A = NULL, *B = NULL, *C = NULL, *C2 = NULL;
  CHECK(tk_tensor_create(TK_F64, 2, cod, 1, dom1, &A));
  CHECK(tk_tensor_create(TK_F64, 1, dom1, 2, cod, &B));
  const int32_t la[3] = {1, 2, 3}, lb[3] = {3, 4, 5}, lc[4] = {4, 1, 5, 2};
  CHECK(tk_contract_output(A, la, B, lb, lc, 2, &C));
  /* the same contraction as explicit Alg. 4 tuples (reading C2): pA (0,1) qA (2) pB (0) qB (1,2), then
     C~ = (A0, A1 ; B1, B2) -> (B1, A0 ; B2, A1) */
  const int32_t tup[] = {0, 1, 2, 0, 1, 2, 2, 0, 3, 1};
  const int32_t ntup[6] = {2, 1, 1, 2, 2, 2};
  CHECK(tk_contract_tuples_output(A, B, tup, ntup, &C2));
  int64_t na, nb, nc;
  CHECK(tk_tensor_nelems(A, &na)); CHECK(tk_tensor_nelems(B, &nb)); CHECK(tk_tensor_nelems(C, &nc));
  double *ha = malloc(na * 8), *hb = malloc(nb * 8), *h1 = malloc(nc * 8), *h2 = malloc(nc * 8);
  for (int64_t i = 0; i < na; ++i) ha[i] = sin(0.37 * (double)i + 0.1);
  for (int64_t i = 0; i < nb; ++i) hb[i] = cos(0.23 * (double)i - 0.4);
  double *da, *db, *dc1, *dc2, *ws;
  size_t w1 = 0, w2 = 0;
  CHECK(tk_contract_workspace(A, la, B, lb, C, lc, &w1));
  CHECK(tk_contract_tuples_workspace(A, B, C2, tup, ntup, &w2));
  size_t w = (w1 > w2 ? w1 : w2) + 256;
  if (cudaMalloc((void**)&da, na * 8) || cudaMalloc((void**)&db, nb * 8) || cudaMalloc((void**)&dc1, nc * 8) ||
      cudaMalloc((void**)&dc2, nc * 8) || cudaMalloc((void**)&ws, w)) { printf("FAIL cudaMalloc\n"); return 1; }
  cudaMemcpy(da, ha, na * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb, nb * 8, cudaMemcpyHostToDevice);
  CHECK(tk_contract(A, da, la, 0, B, db, lb, 0, C, dc1, lc, 1.0, 0.0, ws, w, NULL));
  CHECK(tk_contract_tuples(A, da, 0, B, db, 0, C2, dc2, tup, ntup, 1.0, 0.0, ws, w, NULL));
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("FAIL sync\n"); return 1; }
  cudaMemcpy(h1, dc1, nc * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, dc2, nc * 8, cudaMemcpyDeviceToHost);
  double nrm = 0.0;
  for (int64_t i = 0; i < nc; ++i) {
    if (h1[i] != h2[i]) { printf("FAIL element %lld: %g vs %g\n", (long long)i, h1[i], h2[i]); return 1; }
    nrm += h1[i] * h1[i];
  }
  if (!(nrm > 0.0)) { printf("FAIL zero result\n"); return 1; }
  printf("OK %lld %g\n", (long long)nc, sqrt(nrm));
  return 0;
}
'''


@pytest.mark.gpu
def test_contract_from_c_on_the_gpu(tmp_path):
    """A C program (no Python, no PyTorch) runs tk_contract and tk_contract_tuples on cudaMalloc'd buffers:
    the library stands on its own; the two entry points agree bit for bit (same tuples, same plan)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available() or not os.path.exists(LIB):
        pytest.skip("needs a CUDA device and the built library")
    cuda = "/usr/local/cuda"
    src = tmp_path / "abi_gpu.c"
    src.write_text(GPU_PROGRAM)
    exe = tmp_path / "abi_gpu"
    cc = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", str(src), "-I", os.path.join(ROOT, "include"),
                         "-I", cuda + "/include", "-L", LIBDIR, "-ltk_b200", "-L", cuda + "/lib64", "-lcudart",
                         "-lm", "-Wl,-rpath," + LIBDIR + ":" + cuda + "/lib64", "-o", str(exe)],
                        capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0 and run.stdout.startswith("OK"), run.stdout + run.stderr
