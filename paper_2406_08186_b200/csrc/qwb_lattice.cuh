// qwb_lattice.cuh — lattice geometry shared by lattice.cu and comm.cu.
#pragma once
#include "qwb_internal.cuh"

namespace qwb {

constexpr int kMaxTrace = 8;
struct TraceArgs {
  int n;
  int64_t v[kMaxTrace];   // global vertex ids
  double* out;
};

// local-row geometry of a planes buffer
struct Geom {
  int nx;          // columns
  int ny;          // GLOBAL rows of the torus
  int lrows;       // rows stored (single GPU: ny; slab: ny_local + 2)
  int gy0;         // global row of local row 0, in [0, ny)
  int wrap;        // 1: single GPU, rows wrap inside the buffer; 0: slab with extra rows
  int64_t pstride; // plane stride = nx * lrows
};

// rows a launch covers: ly = row0 + i * rstep for i < nrows
struct Rows {
  int row0, rstep, nrows;
};

void lattice_launch(int shift, cudaStream_t s, const Geom& g, const Rows& r, const double2* in,
                    double2* out, const uint32_t* bits, double* prob, int prob_row0,
                    const TraceArgs& tr);
int lattice_check_shift(qwb_ctx* ctx, int shift);
int lattice_slab_geom(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, Geom* g);
// part: 0 = all owned rows, 1 = first and last owned rows, 2 = interior owned rows
Rows slab_rows(int64_t ny_local, int part);

}  // namespace qwb
