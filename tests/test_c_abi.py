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
