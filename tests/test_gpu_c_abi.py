"""The C ABI from a plain C99 program, on the device: no Python
between the caller and the library.  The C program reads C1's CSR matrix and b
(written here from the seeded generators in inputs/), allocates the device
memory itself with cudaMalloc, and runs ppf_ctx_create -> ppf_plan_create ->
ppf_mat_create -> ppf_poly_chebyshev (+ ppf_poly_certify) ->
ppf_workspace_bytes -> ppf_run (Lanczos, estimate stop) ->
ppf_hessenberg / ppf_history, then also ppf_run_host, and writes x, H and the
report to files.  x is compared with the oracle's x (oracle/ only), computed
here on the same inputs: same m, ||dx||/||x|| <= 1e-10.  Also: a misaligned
device vector is rejected with PPF_EINVAL (16-byte rule of include/ppf.h)."""
import os
import subprocess

import numpy as np
import pytest

from inputs import configs
from oracle import chebyshev, krylov
from oracle.spmv import Operator

from .conftest import ROOT

pytestmark = pytest.mark.gpu

C_SRC = r"""
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>
#include "ppf.h"

#define CK(x) do { int s_ = (x); if (s_ != PPF_OK) { \
  fprintf(stderr, "%s -> %s: %s\n", #x, ppf_status_string(s_), ppf_last_error()); return 10; } } while (0)
#define CU(x) do { if ((x) != cudaSuccess) { fprintf(stderr, "%s failed\n", #x); return 11; } } while (0)

static void* slurp(const char* dir, const char* name, size_t* bytes) {
  char p[4096];
  snprintf(p, sizeof p, "%s/%s", dir, name);
  FILE* f = fopen(p, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  *bytes = (size_t)ftell(f);
  fseek(f, 0, SEEK_SET);
  void* buf = malloc(*bytes);
  if (fread(buf, 1, *bytes, f) != *bytes) { fclose(f); free(buf); return NULL; }
  fclose(f);
  return buf;
}

static int spit(const char* dir, const char* name, const void* p, size_t bytes) {
  char path[4096];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE* f = fopen(path, "wb");
  if (!f) return 1;
  size_t w = fwrite(p, 1, bytes, f);
  fclose(f);
  return w != bytes;
}

int main(int argc, char** argv) {
  if (argc != 2) return 1;
  const char* dir = argv[1];
  size_t nb_rp, nb_col, nb_val, nb_b, nb_iv;
  int64_t* row_ptr = (int64_t*)slurp(dir, "row_ptr.bin", &nb_rp);
  int64_t* col = (int64_t*)slurp(dir, "col.bin", &nb_col);
  double* val = (double*)slurp(dir, "val.bin", &nb_val);
  double* b = (double*)slurp(dir, "b.bin", &nb_b);
  double* iv = (double*)slurp(dir, "interval.bin", &nb_iv);
  if (!row_ptr || !col || !val || !b || !iv) return 2;
  const int64_t n = (int64_t)(nb_rp / 8) - 1;
  const int64_t bounds[2] = {0, n};

  ppf_ctx* ctx = NULL;
  CK(ppf_ctx_create(0, 0, 1, NULL, NULL, &ctx));
  ppf_plan* plan = NULL;
  CK(ppf_plan_create(PPF_R64, n, 1, 0, bounds, row_ptr, col, val, PPF_FMT_SELL, 32, 1, &plan));
  size_t mbytes = 0;
  CK(ppf_plan_device_bytes(plan, &mbytes));
  void* mbuf = NULL;
  CU(cudaMalloc(&mbuf, mbytes));
  ppf_mat* A = NULL;
  CK(ppf_mat_create(ctx, plan, mbuf, mbytes, &A));
  ppf_plan_destroy(plan);

  ppf_poly* q = NULL;
  CK(ppf_poly_chebyshev(iv[0], iv[1], 4, &q));            /* P:323-335 */
  double min_q = 0.0;
  CK(ppf_poly_certify(q, NULL, 0, PPF_R64, &min_q));      /* P:334-335 */

  ppf_opts o;
  memset(&o, 0, sizeof o);
  o.func = PPF_INVSQRT;
  o.krylov = PPF_LANCZOS;
  o.m_max = 60;
  o.stop = PPF_STOP_EST;
  o.tol = 1e-10;
  o.check_every = 1;
  o.record_history = 1;
  o.precond = PPF_PREC_LEFT;
  size_t wbytes = 0;
  CK(ppf_workspace_bytes(ctx, A, q, &o, &wbytes));
  void *work = NULL, *db = NULL, *dx = NULL;
  CU(cudaMalloc(&work, wbytes));
  CU(cudaMalloc(&db, (size_t)n * 8));
  CU(cudaMalloc(&dx, (size_t)n * 8 + 16));
  CU(cudaMemcpy(db, b, (size_t)n * 8, cudaMemcpyHostToDevice));

  ppf_report rep;
  CK(ppf_run(ctx, A, q, &o, db, dx, work, wbytes, &rep));
  CU(cudaDeviceSynchronize());
  double* x = (double*)malloc((size_t)n * 8);
  CU(cudaMemcpy(x, dx, (size_t)n * 8, cudaMemcpyDeviceToHost));
  if (spit(dir, "x.bin", x, (size_t)n * 8)) return 3;

  int m = 0;
  double beta0 = 0.0;
  CK(ppf_hessenberg(ctx, 0, NULL, &m, &beta0));
  double* H = (double*)calloc((size_t)(m + 1) * m, 8);
  CK(ppf_hessenberg(ctx, m + 1, H, NULL, NULL));
  if (spit(dir, "H.bin", H, (size_t)(m + 1) * m * 8)) return 4;
  int cnt = 0;
  CK(ppf_history(ctx, 0, &cnt, NULL, NULL, NULL, NULL));

  /* the same through host buffers */
  double* xh = (double*)malloc((size_t)n * 8);
  ppf_report rep_h;
  CK(ppf_run_host(ctx, A, q, &o, b, xh, work, wbytes, &rep_h));
  if (spit(dir, "x_host.bin", xh, (size_t)n * 8)) return 5;

  /* a float64 vector starting 8 bytes into an allocation: rejected */
  int mis = ppf_run(ctx, A, q, &o, db, (char*)dx + 8, work, wbytes, &rep_h);

  /* the same operator as SELL-64: the plan stores pair codes (PPF_ENC_PAIR8);
     its SpMV does the SELL-32 kernel's multiply-adds in the same order */
  ppf_plan* plan64 = NULL;
  CK(ppf_plan_create(PPF_R64, n, 1, 0, bounds, row_ptr, col, val, PPF_FMT_SELL, 64, 1, &plan64));
  int enc = -1, ntab = -1, ibits = 0;
  CK(ppf_plan_encoding(plan64, &enc, &ntab));
  CK(ppf_plan_index_bits(plan64, &ibits));
  size_t mbytes64 = 0;
  CK(ppf_plan_device_bytes(plan64, &mbytes64));
  void* mbuf64 = NULL;
  CU(cudaMalloc(&mbuf64, mbytes64));
  ppf_mat* A64 = NULL;
  CK(ppf_mat_create(ctx, plan64, mbuf64, mbytes64, &A64));
  ppf_plan_destroy(plan64);
  void *y32 = NULL, *y64 = NULL;
  CU(cudaMalloc(&y32, (size_t)n * 8));
  CU(cudaMalloc(&y64, (size_t)n * 8));
  CK(ppf_spmv(ctx, A, db, y32));
  CK(ppf_spmv(ctx, A64, db, y64));
  CU(cudaDeviceSynchronize());
  double* h32 = (double*)malloc((size_t)n * 8);
  double* h64 = (double*)malloc((size_t)n * 8);
  CU(cudaMemcpy(h32, y32, (size_t)n * 8, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(h64, y64, (size_t)n * 8, cudaMemcpyDeviceToHost));
  int spmv_equal = 1;
  for (int64_t i = 0; i < n; ++i) spmv_equal &= (h32[i] == h64[i]);
  if (spit(dir, "y_pair.bin", h64, (size_t)n * 8)) return 6;
  ppf_mat_destroy(A64);
  cudaFree(y32); cudaFree(y64); cudaFree(mbuf64);
  free(h32); free(h64);

  printf("m=%d term=%d mvms=%lld launches=%lld beta0=%.17g min_q=%.17g hist=%d "
         "sec_dev=%.9g sec_total=%.9g misaligned=%d enc=%d ntab=%d ibits=%d spmv_equal=%d "
         "mbytes64=%zu\n", rep.iterations, rep.term, rep.mvms,
         rep.kernel_launches, beta0, min_q, cnt, rep.seconds_device, rep.seconds_total, mis, enc,
         ntab, ibits, spmv_equal, mbytes64);
  ppf_poly_destroy(q);
  ppf_mat_destroy(A);
  ppf_ctx_destroy(ctx);
  cudaFree(work); cudaFree(db); cudaFree(dx); cudaFree(mbuf);
  free(row_ptr); free(col); free(val); free(b); free(iv); free(x); free(xh); free(H);
  return 0;
}
"""


def test_c99_program_runs_c1_on_device(tmp_path):
    from paper_2401_06684_b200 import _lib
    from paper_2401_06684_b200.build import build
    build()
    A, b, iv = configs.build("C1")
    A.row_ptr.astype(np.int64).tofile(tmp_path / "row_ptr.bin")
    A.col.astype(np.int64).tofile(tmp_path / "col.bin")
    A.val.astype(np.float64).tofile(tmp_path / "val.bin")
    b.astype(np.float64).tofile(tmp_path / "b.bin")
    np.asarray(iv, dtype=np.float64).tofile(tmp_path / "interval.bin")
    src = tmp_path / "run_c1.c"
    src.write_text(C_SRC)
    exe = tmp_path / "run_c1"
    libdir = os.path.dirname(_lib.LIB_PATH)
    cuda = "/usr/local/cuda"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        "-I", f"{cuda}/include", str(src), "-o", str(exe), "-L", libdir,
                        "-l:libppf.so", f"-Wl,-rpath,{libdir}", "-L", f"{cuda}/lib64", "-lcudart",
                        f"-Wl,-rpath,{cuda}/lib64"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    rep = dict(kv.split("=") for kv in r.stdout.split())
    # the oracle on the same inputs (oracle/ only): Lanczos, Chebyshev deg 4, estimate stop
    qo = chebyshev.coefficients(*iv, 4)
    res = krylov.run(Operator(A.to_scipy()), b, qo, func="invsqrt", krylov="lanczos", m_max=60,
                     stop="est", tol=1e-10)
    x = np.fromfile(tmp_path / "x.bin")
    assert int(rep["m"]) == res.m and int(rep["mvms"]) == res.mvms
    assert np.linalg.norm(x - res.x) <= 1e-10 * np.linalg.norm(res.x)
    m = res.m
    H = np.fromfile(tmp_path / "H.bin").reshape(m, m + 1).T
    assert np.abs(H - res.H).max() <= 1e-11 * np.abs(res.H).max()
    assert float(rep["beta0"]) == pytest.approx(res.beta0, rel=1e-13)
    assert float(rep["min_q"]) == pytest.approx(chebyshev.certify(qo), rel=1e-12)
    assert np.array_equal(np.fromfile(tmp_path / "x_host.bin"), x)
    assert int(rep["hist"]) == len(res.history)
    assert int(rep["launches"]) > 0
    assert 0.0 < float(rep["sec_dev"]) <= float(rep["sec_total"]) * 1.05
    assert int(rep["misaligned"]) == 1           # PPF_EINVAL
    # pair codes from C: PPF_ENC_PAIR8 with the 5-point stencil's 5 pairs + padding, 8-bit
    # codes, the SpMV equal to the SELL-32 one and to SciPy's within fp64 rounding
    assert int(rep["enc"]) == 2 and int(rep["ibits"]) == 8 and 5 < int(rep["ntab"]) <= 11
    assert int(rep["spmv_equal"]) == 1
    assert int(rep["mbytes64"]) < 2 * A.nnz + 16 * 1024
    y = np.fromfile(tmp_path / "y_pair.bin")
    yr = A.to_scipy() @ b
    assert np.all(np.abs(y - yr) <= 1e-14 * (abs(A.to_scipy()) @ np.abs(b)))
