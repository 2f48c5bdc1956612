// Output wire format of the front end: the field table
// of export_field (scenario.cpp:372-399).
//
// The per-cell work (extract_macro, moment_rep.hpp:116-146, and the scaling
// to laboratory units) runs on the device over the resident field: one thread
// per cell reads the 1 + 6 + 9 coefficients the macroscopic state needs and
// the basis params, and writes the 11 columns of its row, so only 88 B per
// cell (instead of the 8 (N + 4) B record) cross PCIe.  The host side formats
// the rows with %.17g (the reference's fmt, scenario.cpp:18-22) on all host
// threads, block by block, and writes them in row order.  Every value is the
// reference's expression in the reference's operation order (products and one
// quotient, no additions except q_i's, which keep their order), so the table
// is bitwise the reference's for the same field.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "runtime.h"

namespace momg_gpu {

constexpr int kCols = 11;  // x y rho u1 u2 T sigma11 sigma12 sigma22 q1 q2

struct Units {
  double length, density, theta, speed, mass, pressure, heat;
};

// Boltzmann constant (scenario.hpp:10)
constexpr double kBoltzmann = 1.380649e-23;

__global__ void k_field_table(DevField f, int NP, Units u, double* __restrict__ out, int* first_bad) {
  const int cells = f.nx * f.ny;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < cells; k += gridDim.x * blockDim.x) {
    const int i = k % f.nx, j = k / f.nx;
    const double* c = f.c + (size_t)k * NP;
    const double* p = f.p + (size_t)k * 4;
    double* row = out + (size_t)k * kCols;
    const double rho = c[0];
    if (!(rho > 0.0)) atomicMin(first_bad, k);  // extract_macro: nonpositive density
    // sigma_ij = (1 + delta_ij) f_{e_i + e_j}; q_i = 2 f_{3 e_i} + sum_d f_{2 e_d + e_i}
    const double s11 = 2.0 * c[flat3(2, 0, 0)];
    const double s12 = 1.0 * c[flat3(1, 1, 0)];
    const double s22 = 2.0 * c[flat3(0, 2, 0)];
    double q1 = 2.0 * c[flat3(3, 0, 0)];
    q1 = __dadd_rn(q1, c[flat3(3, 0, 0)]);
    q1 = __dadd_rn(q1, c[flat3(1, 2, 0)]);
    q1 = __dadd_rn(q1, c[flat3(1, 0, 2)]);
    double q2 = 2.0 * c[flat3(0, 3, 0)];
    q2 = __dadd_rn(q2, c[flat3(2, 1, 0)]);
    q2 = __dadd_rn(q2, c[flat3(0, 3, 0)]);
    q2 = __dadd_rn(q2, c[flat3(0, 1, 2)]);
    // theta_to_kelvin(theta * scales.theta, mass) = (theta * s) * mass / k_B
    const double th = __dmul_rn(p[3], u.theta);
    row[0] = __dmul_rn(f.xc[i], u.length);
    row[1] = __dmul_rn(f.yc[j], u.length);
    row[2] = __dmul_rn(rho, u.density);
    row[3] = __dmul_rn(p[0], u.speed);
    row[4] = __dmul_rn(p[1], u.speed);
    row[5] = __ddiv_rn(__dmul_rn(th, u.mass), kBoltzmann);
    row[6] = __dmul_rn(s11, u.pressure);
    row[7] = __dmul_rn(s12, u.pressure);
    row[8] = __dmul_rn(s22, u.pressure);
    row[9] = __dmul_rn(q1, u.heat);
    row[10] = __dmul_rn(q2, u.heat);
  }
}

}  // namespace momg_gpu

namespace {

int set_err(momg_err* err, int code, const std::string& msg) {
  if (err) {
    err->code = code;
    err->i = err->j = -1;
    std::snprintf(err->msg, sizeof(err->msg), "%s", msg.c_str());
  }
  return code;
}

// The device table of f in laboratory units into host memory; *rows_ok = the
// rows before the first cell extract_macro rejects (all rows when none).
int field_table(const momg_field* f, const momg_units* mu, double* host, long long* rows_ok, momg_err* err) {
  using namespace momg_gpu;
  const long long cells = (long long)f->nx * f->ny;
  // UnitScales (scenario.cpp:313-319) and export_field's derived scales (:378-379)
  Units u{mu->length, mu->density, mu->theta, mu->speed, mu->molecule_mass, 0.0, 0.0};
  u.pressure = u.density * u.theta;
  u.heat = u.pressure * u.speed;
  cudaStream_t s = momg_rt::stream();
  double* dtab = nullptr;
  int* dbad = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dtab, (size_t)cells * kCols * sizeof(double), s);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&dbad, sizeof(int), s);
  const int none = INT_MAX;
  if (e == cudaSuccess) e = cudaMemcpyAsync(dbad, &none, sizeof(int), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    const int blocks = (int)std::min<long long>((cells + 255) / 256, 148LL * 8);
    k_field_table<<<blocks, 256, 0, s>>>(f->dev(), f->NP, u, dtab, dbad);
    momg_rt::count_launch(1);
    e = cudaGetLastError();
  }
  int bad = INT_MAX;
  if (e == cudaSuccess) e = cudaMemcpyAsync(host, dtab, (size_t)cells * kCols * sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (dtab) cudaFreeAsync(dtab, s);
  if (dbad) cudaFreeAsync(dbad, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (int rc = momg_rt::cuda_check(e, err, "momg_field_table")) return rc;
  if (int rc = momg_rt::sync_check(err)) return rc;
  *rows_ok = bad == INT_MAX ? cells : bad;
  if (bad != INT_MAX) {
    set_err(err, MOMG_NONPHYSICAL_STATE, "extract_macro: nonpositive density");
    if (err) {
      err->i = bad % f->nx;
      err->j = bad / f->nx;
    }
    return MOMG_NONPHYSICAL_STATE;
  }
  return MOMG_OK;
}

// rows [r0, r1) of the table as TSV text, %.17g (scenario.cpp:18-22, 392-396)
void format_rows(const double* tab, long long r0, long long r1, std::string* out) {
  char buf[32];
  out->clear();
  out->reserve((size_t)(r1 - r0) * momg_gpu::kCols * 24);
  for (long long r = r0; r < r1; ++r) {
    const double* row = tab + r * momg_gpu::kCols;
    for (int k = 0; k < momg_gpu::kCols; ++k) {
      const int n = std::snprintf(buf, sizeof(buf), "%.17g", row[k]);
      out->append(buf, (size_t)n);
      out->push_back(k + 1 < momg_gpu::kCols ? '\t' : '\n');
    }
  }
}

}  // namespace

extern "C" {

int momg_field_table(const momg_field* f, const momg_units* u, double* out, long long* rows_ok,
                     momg_err* err) {
  if (err) {
    err->code = 0;
    err->i = err->j = -1;
    err->msg[0] = 0;
  }
  if (int rc = momg_rt::ensure(err)) return rc;
  if (!f || !u || !out) return set_err(err, MOMG_ERR_ARG, "momg_field_table: null argument");
  momg_rt::acquire(f);
  long long ok = 0;
  const int rc = field_table(f, u, out, &ok, err);
  if (rows_ok) *rows_ok = ok;
  return rc;
}

// export_field (scenario.cpp:372-399): header row, then one row per cell,
// row-major with j outermost.  Like the reference, a cell extract_macro
// rejects ends the file after the rows before it (NonphysicalState).
int momg_export_field(const momg_field* f, const momg_units* u, const char* path, momg_err* err) {
  if (err) {
    err->code = 0;
    err->i = err->j = -1;
    err->msg[0] = 0;
  }
  if (int rc = momg_rt::ensure(err)) return rc;
  if (!f || !u || !path) return set_err(err, MOMG_ERR_ARG, "momg_export_field: null argument");
  FILE* fp = std::fopen(path, "w");
  if (!fp) return set_err(err, MOMG_ERROR, std::string("export_field: cannot open '") + path + "'");
  momg_rt::acquire(f);
  const long long cells = (long long)f->nx * f->ny;
  std::vector<double> tab((size_t)cells * momg_gpu::kCols);
  long long rows = 0;
  const int rc = field_table(f, u, tab.data(), &rows, err);
  bool ok = std::fputs("x\ty\trho\tu1\tu2\tT\tsigma11\tsigma12\tsigma22\tq1\tq2\n", fp) >= 0;
  const int nt = (int)std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  const long long block = 1 << 14;  // rows per formatting task
  std::vector<std::string> text((size_t)nt);
  for (long long r0 = 0; ok && r0 < rows; r0 += block * nt) {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) {
      const long long a = std::min(rows, r0 + t * block), b = std::min(rows, a + block);
      if (t == 0) continue;
      pool.emplace_back(format_rows, tab.data(), a, b, &text[t]);
    }
    format_rows(tab.data(), r0, std::min(rows, r0 + block), &text[0]);
    for (auto& th : pool) th.join();
    for (int t = 0; t < nt && ok; ++t) {
      const long long a = std::min(rows, r0 + t * block);
      if (a >= rows) break;
      ok = std::fwrite(text[t].data(), 1, text[t].size(), fp) == text[t].size();
    }
  }
  ok = (std::fflush(fp) == 0) && ok;
  ok = (std::fclose(fp) == 0) && ok;
  if (rc != MOMG_OK) return rc;
  if (!ok) return set_err(err, MOMG_ERROR, std::string("export_field: write failed for '") + path + "'");
  return MOMG_OK;
}

}  // extern "C"
