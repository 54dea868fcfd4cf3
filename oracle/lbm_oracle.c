/* TEST INFRASTRUCTURE ONLY -- CPU restatement oracle; see lbm_oracle.h.
 *
 * Built with -ffp-contract=off (the reference's own flag,
 * proj/CMakeLists.txt:12-14) so every double expression below rounds exactly
 * like the reference's.  Paths cited are relative to /root/reference/proj.
 */
#include "lbm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define Q 19

/* d3q19.hpp:30-44 : rest, 6 axis, 12 diagonals, opposites adjacent */
static const int kC[Q][3] = {
    {0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},
    {0, 0, 1},  {0, 0, -1},  {1, 1, 0},  {-1, -1, 0}, {1, -1, 0},
    {-1, 1, 0}, {1, 0, 1},   {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
    {0, 1, 1},  {0, -1, -1}, {0, 1, -1}, {0, -1, 1}};
static const int kOpp[Q] = {0,  2,  1,  4,  3,  6,  5,  8,  7, 10,
                            9, 12, 11, 14, 13, 16, 15, 18, 17};
/* d3q19.hpp:46-54 */
#define W_REST (1.0 / 3.0)
#define W_AXIS (1.0 / 18.0)
#define W_DIAG (1.0 / 36.0)
static const double kW[Q] = {W_REST, W_AXIS, W_AXIS, W_AXIS, W_AXIS,
                             W_AXIS, W_AXIS, W_DIAG, W_DIAG, W_DIAG,
                             W_DIAG, W_DIAG, W_DIAG, W_DIAG, W_DIAG,
                             W_DIAG, W_DIAG, W_DIAG, W_DIAG};

double ora_omega_minus(double omega_plus, double magic_lambda) {
  /* d3q19.hpp:70-73 */
  const double kappa = 1.0 / omega_plus - 0.5;
  return 1.0 / (0.5 + magic_lambda / kappa);
}

void ora_collide_node(double* f, double wp, double wm, const double* g) {
  /* d3q19.hpp:107-144, same expression trees and evaluation order */
  double rho = f[0];
  for (int i = 1; i < Q; ++i) rho += f[i];
  const double mx = f[1] - f[2] + f[7] - f[8] + f[9] - f[10] + f[11] - f[12] +
                    f[13] - f[14];
  const double my = f[3] - f[4] + f[7] - f[8] - f[9] + f[10] + f[15] - f[16] +
                    f[17] - f[18];
  const double mz = f[5] - f[6] + f[11] - f[12] - f[13] + f[14] + f[15] -
                    f[16] - f[17] + f[18];
  const double inv_rho = 1.0 / rho;
  const double ux = mx * inv_rho;
  const double uy = my * inv_rho;
  const double uz = mz * inv_rho;
  const double usq = ux * ux + uy * uy + uz * uz;
  const double one_m = 1.0 - 1.5 * usq;
  f[0] -= wp * (f[0] - W_REST * rho * one_m);
  for (int i = 1; i < Q; i += 2) {
    const int j = i + 1;
    const double cu = (double)kC[i][0] * ux + (double)kC[i][1] * uy +
                      (double)kC[i][2] * uz;
    const double cg = (double)kC[i][0] * g[0] + (double)kC[i][1] * g[1] +
                      (double)kC[i][2] * g[2];
    const double wr = kW[i] * rho;
    const double e_even = wr * (one_m + 4.5 * cu * cu);
    const double e_odd = wr * 3.0 * cu;
    const double f_even = 0.5 * (f[i] + f[j]);
    const double f_odd = 0.5 * (f[i] - f[j]);
    const double d_even = wp * (f_even - e_even);
    const double d_odd = wm * (f_odd - e_odd);
    const double forcing = wr * 3.0 * cg;
    f[i] = f[i] - d_even - d_odd + forcing;
    f[j] = f[j] - d_even + d_odd - forcing;
  }
}

void ora_equilibrium(double rho, const double* u, double* f) {
  /* d3q19.cpp:7-18 */
  const double usq = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
  for (int i = 0; i < Q; ++i) {
    const double cu = (double)kC[i][0] * u[0] + (double)kC[i][1] * u[1] +
                      (double)kC[i][2] * u[2];
    f[i] = kW[i] * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * usq);
  }
}

static size_t idx3(int ny, int nz, int x, int y, int z) {
  /* geometry.hpp:27-29 : x-major, z innermost */
  return ((size_t)x * (size_t)ny + (size_t)y) * (size_t)nz + (size_t)z;
}

static int imin(int a, int b) { return a < b ? a : b; }

int ora_geometry(int kind, int nx, int ny, int nz, int block, int spacing,
                 int pipe_diameter, uint8_t* flags, int* periodic,
                 int64_t* n_fluid) {
  /* geometry.cpp:40-111 */
  const size_t V = (size_t)nx * ny * nz;
  int per[3] = {0, 0, 0};
  if (flags) memset(flags, 0, V);
  switch (kind) {
    case 0: /* channel :48-57 */
      if (nx < 1 || ny < 3 || nz < 3) return 1;
      per[0] = 1;
      if (flags)
        for (int x = 0; x < nx; ++x)
          for (int y = 0; y < ny; ++y)
            for (int z = 0; z < nz; ++z)
              if (y == 0 || y == ny - 1 || z == 0 || z == nz - 1)
                flags[idx3(ny, nz, x, y, z)] = 1;
      break;
    case 1: /* slit :58-67 */
      if (nx < 1 || ny < 1 || nz < 3) return 1;
      per[0] = per[1] = 1;
      if (flags)
        for (int x = 0; x < nx; ++x)
          for (int y = 0; y < ny; ++y) {
            flags[idx3(ny, nz, x, y, 0)] = 1;
            flags[idx3(ny, nz, x, y, nz - 1)] = 1;
          }
      break;
    case 2: { /* pipe :68-84 ; D = min(ny,nz)-2 unless given */
      if (nx < 1 || ny < 4 || nz < 4) return 1;
      per[0] = 1;
      const int64_t D =
          pipe_diameter > 0 ? pipe_diameter : (int64_t)imin(ny, nz) - 2;
      const int64_t r2x4 = D * D;
      if (flags)
        for (int y = 0; y < ny; ++y)
          for (int z = 0; z < nz; ++z) {
            const int64_t dy = 2 * (int64_t)y - (ny - 1);
            const int64_t dz = 2 * (int64_t)z - (nz - 1);
            if (dy * dy + dz * dz > r2x4)
              for (int x = 0; x < nx; ++x) flags[idx3(ny, nz, x, y, z)] = 1;
          }
      break;
    }
    case 3: { /* blocks :85-104 */
      if (nx < 1 || ny < 1 || nz < 1) return 1;
      if (block < 1 || spacing < 0) return 1;
      const int period = block + spacing;
      if (period > imin(nx, imin(ny, nz))) return 1;
      per[0] = per[1] = per[2] = 1;
      if (flags)
        for (int x = 0; x < nx; ++x)
          for (int y = 0; y < ny; ++y)
            for (int z = 0; z < nz; ++z)
              if (x % period >= spacing && y % period >= spacing &&
                  z % period >= spacing)
                flags[idx3(ny, nz, x, y, z)] = 1;
      break;
    }
    default:
      return 1;
  }
  if (periodic)
    for (int a = 0; a < 3; ++a) periodic[a] = per[a];
  if (flags && n_fluid) {
    int64_t n = 0; /* geometry.cpp:113-117 */
    for (size_t i = 0; i < V; ++i) n += flags[i] == 0;
    *n_fluid = n;
    if (n == 0) return 1;
  }
  return 0;
}

/* geometry.cpp:119-131 : 0 coordinate, 1 solid hit, 2 outside */
static int neighbor(const uint8_t* flags, const int* periodic, int nx, int ny,
                    int nz, int x, int y, int z, int dir, int* t) {
  const int dims[3] = {nx, ny, nz};
  t[0] = x + kC[dir][0];
  t[1] = y + kC[dir][1];
  t[2] = z + kC[dir][2];
  for (int a = 0; a < 3; ++a) {
    if (t[a] < 0 || t[a] >= dims[a]) {
      if (!periodic[a]) return 2;
      t[a] = (t[a] + dims[a]) % dims[a];
    }
  }
  return flags[idx3(ny, nz, t[0], t[1], t[2])] ? 1 : 0;
}

/* list_lattice.cpp:63-80 */
#define SET_PERIOD 4096u  /* 64 B * 512 sets / 8 B */
#define PAGE_ELEMS 262144u /* 2 MiB / 8 B */
static uint64_t place(uint64_t floor, uint64_t want_set, uint64_t want_tlb) {
  const uint64_t line_elems = 8;
  const uint64_t res = want_set * line_elems;
  uint64_t cand = (floor <= res)
                      ? res
                      : (floor - res + SET_PERIOD - 1) / SET_PERIOD * SET_PERIOD +
                            res;
  while (cand / PAGE_ELEMS % 4 != want_tlb) cand += SET_PERIOD;
  return cand;
}

void ora_padding_offsets(uint64_t n_fluid, int mode, const int64_t* pads,
                         uint64_t* starts, uint64_t* total) {
  /* list_lattice.cpp:84-121 */
  switch (mode) {
    case 0:
      for (int d = 0; d < Q; ++d) starts[d] = (uint64_t)d * n_fluid;
      break;
    case 3: {
      uint64_t off = 0;
      for (int d = 0; d < Q; ++d) {
        off += (uint64_t)pads[d];
        starts[d] = off;
        off += n_fluid;
      }
      break;
    }
    case 1: {
      const uint64_t step = 512 / Q; /* 26 */
      uint64_t floor = 0;
      for (int d = 0; d < Q; ++d) {
        starts[d] = place(floor, (uint64_t)d * step % 512, (uint64_t)d % 4);
        floor = starts[d] + n_fluid;
      }
      break;
    }
    case 2: {
      uint64_t floor = 0;
      for (int d = 0; d < Q; ++d) {
        starts[d] = place(floor, 0, 0);
        floor = starts[d] + n_fluid;
      }
      break;
    }
  }
  if (total) *total = starts[Q - 1] + n_fluid;
}

int64_t ora_order_nodes(const uint8_t* flags, int nx, int ny, int nz, int blk,
                        int32_t* nodes, uint32_t* rank) {
  /* list_lattice.cpp:123-141 ; rank fill :160-164 */
  int64_t n = 0;
  if (rank) {
    const size_t V = (size_t)nx * ny * nz;
    for (size_t i = 0; i < V; ++i) rank[i] = UINT32_MAX;
  }
#define EMIT(X, Y, Z)                                          \
  do {                                                         \
    const size_t ii = idx3(ny, nz, (X), (Y), (Z));             \
    if (!flags[ii]) {                                          \
      if (nodes) {                                             \
        nodes[3 * n] = (X);                                    \
        nodes[3 * n + 1] = (Y);                                \
        nodes[3 * n + 2] = (Z);                                \
      }                                                        \
      if (rank) rank[ii] = (uint32_t)n;                        \
      ++n;                                                     \
    }                                                          \
  } while (0)
  if (blk == 0) {
    for (int x = 0; x < nx; ++x)
      for (int y = 0; y < ny; ++y)
        for (int z = 0; z < nz; ++z) EMIT(x, y, z);
  } else {
    for (int ty = 0; ty < ny; ty += blk)
      for (int tz = 0; tz < nz; tz += blk)
        for (int x = 0; x < nx; ++x)
          for (int y = ty; y < imin(ty + blk, ny); ++y)
            for (int z = tz; z < imin(tz + blk, nz); ++z) EMIT(x, y, z);
  }
#undef EMIT
  return n;
}

void ora_build_adjacency(const uint8_t* flags, const int* periodic, int nx,
                         int ny, int nz, const int32_t* nodes,
                         const uint32_t* rank, int64_t n_fluid, int layout_soa,
                         const uint64_t* starts, int scatter, uint32_t* adj) {
  /* list_lattice.cpp:177-191 ; SlotMap::slot list_lattice.hpp:66-75 */
#pragma omp parallel for schedule(static)
  for (int64_t n = 0; n < n_fluid; ++n) {
    const int x = nodes[3 * n], y = nodes[3 * n + 1], z = nodes[3 * n + 2];
    for (int d = 1; d < Q; ++d) {
      const int look = scatter ? d : kOpp[d];
      int t[3];
      const int kind = neighbor(flags, periodic, nx, ny, nz, x, y, z, look, t);
      uint64_t slot;
      if (kind == 0) {
        const uint64_t m = rank[idx3(ny, nz, t[0], t[1], t[2])];
        slot = layout_soa ? starts[d] + m : m * Q + (uint64_t)d;
      } else {
        slot = layout_soa ? starts[kOpp[d]] + (uint64_t)n
                          : (uint64_t)n * Q + (uint64_t)kOpp[d];
      }
      adj[(size_t)n * 18 + (size_t)(d - 1)] = (uint32_t)slot;
    }
  }
}

static uint64_t splitmix64(uint64_t x) {
  /* harness.cpp:18-23 */
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

void ora_perturbed(uint64_t n_fluid, uint64_t seed, double amplitude,
                   double* out) {
  /* harness.cpp:50-62 */
  for (uint64_t n = 0; n < n_fluid; ++n)
    for (int d = 0; d < Q; ++d) {
      const uint64_t h = splitmix64(seed ^ (n * Q + (uint64_t)d));
      const double u01 = (double)(h >> 11) * (1.0 / 9007199254740992.0);
      out[n * Q + d] = kW[d] * (1.0 + amplitude * (u01 - 0.5));
    }
}

uint64_t ora_fingerprint(const double* data, uint64_t count) {
  /* harness.cpp:27-39 : FNV-1a 64 over little-endian double bytes */
  uint64_t h = 0xcbf29ce484222325ull;
  const unsigned char* p = (const unsigned char*)data;
  const uint64_t nb = count * 8;
  for (uint64_t i = 0; i < nb; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

uint64_t ora_fingerprint_u32(const uint32_t* data, uint64_t count) {
  uint64_t h = 0xcbf29ce484222325ull;
  const unsigned char* p = (const unsigned char*)data;
  const uint64_t nb = count * 4;
  for (uint64_t i = 0; i < nb; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* tests/support/reference.hpp:33-68 (full way) and :72-105 (half way) */
static void step_fullway(const uint8_t* flags, int nx, int ny, int nz,
                         const double* f, double* post, double* next,
                         double wp, double wm, const double* g) {
  const size_t V = (size_t)nx * ny * nz;
  memcpy(post, f, V * Q * sizeof(double));
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < V; ++i)
    if (!flags[i]) ora_collide_node(post + i * Q, wp, wm, g);
#pragma omp parallel for schedule(static)
  for (int x = 0; x < nx; ++x)
    for (int y = 0; y < ny; ++y)
      for (int z = 0; z < nz; ++z)
        for (int d = 0; d < Q; ++d) {
          const int tx = (x + kC[d][0] + nx) % nx;
          const int ty = (y + kC[d][1] + ny) % ny;
          const int tz = (z + kC[d][2] + nz) % nz;
          next[idx3(ny, nz, tx, ty, tz) * Q + d] =
              post[idx3(ny, nz, x, y, z) * Q + d];
        }
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < V; ++i)
    if (flags[i]) {
      double* fn = next + i * Q;
      for (int k = 1; k < Q; k += 2) {
        const double t = fn[k];
        fn[k] = fn[k + 1];
        fn[k + 1] = t;
      }
    }
}

static void step_halfway(const uint8_t* flags, const int* periodic, int nx,
                         int ny, int nz, const double* f, double* post,
                         double* next, double wp, double wm, const double* g) {
  const size_t V = (size_t)nx * ny * nz;
  memcpy(post, f, V * Q * sizeof(double));
  memcpy(next, f, V * Q * sizeof(double));
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < V; ++i)
    if (!flags[i]) ora_collide_node(post + i * Q, wp, wm, g);
#pragma omp parallel for schedule(static)
  for (int x = 0; x < nx; ++x)
    for (int y = 0; y < ny; ++y)
      for (int z = 0; z < nz; ++z) {
        const size_t i = idx3(ny, nz, x, y, z);
        if (flags[i]) continue;
        double* fn = next + i * Q;
        const double* own = post + i * Q;
        fn[0] = own[0];
        for (int d = 1; d < Q; ++d) {
          int t[3];
          const int k =
              neighbor(flags, periodic, nx, ny, nz, x, y, z, kOpp[d], t);
          if (k == 0)
            fn[d] = post[idx3(ny, nz, t[0], t[1], t[2]) * Q + d];
          else
            fn[d] = own[kOpp[d]];
        }
      }
}

static double kahan(const double* v, size_t n, double* sum, double* carry) {
  for (size_t i = 0; i < n; ++i) {
    const double y = v[i] - *carry;
    const double t = *sum + y;
    *carry = (t - *sum) - y;
    *sum = t;
  }
  return *sum;
}

int ora_run(int family, const uint8_t* flags, const int* periodic, int nx,
            int ny, int nz, const double* init, long steps, double wp,
            double wm, const double* g, double* out, double* mass_out) {
  const size_t V = (size_t)nx * ny * nz;
  double* f = (double*)malloc(V * Q * sizeof(double));
  double* post = (double*)malloc(V * Q * sizeof(double));
  double* next = (double*)malloc(V * Q * sizeof(double));
  if (!f || !post || !next) {
    free(f);
    free(post);
    free(next);
    return 4;
  }
  /* RefLattice ctor (reference.hpp:20-24): weights everywhere; ref_load
   * (:131-141) then overwrites fluid nodes in canonical order. */
  for (size_t i = 0; i < V; ++i)
    for (int d = 0; d < Q; ++d) f[i * Q + d] = kW[d];
  if (init) {
    size_t k = 0;
    for (size_t i = 0; i < V; ++i)
      if (!flags[i]) {
        memcpy(f + i * Q, init + k * Q, Q * sizeof(double));
        ++k;
      }
  }
  for (long s = 0; s < steps; ++s) {
    if (family == 0)
      step_fullway(flags, nx, ny, nz, f, post, next, wp, wm, g);
    else
      step_halfway(flags, periodic, nx, ny, nz, f, post, next, wp, wm, g);
    double* t = f;
    f = next;
    next = t;
  }
  size_t k = 0;
  double sum = 0.0, carry = 0.0;
  for (size_t i = 0; i < V; ++i) {
    if (family == 0) kahan(f + i * Q, Q, &sum, &carry);
    if (flags[i]) continue;
    if (family == 1) kahan(f + i * Q, Q, &sum, &carry);
    if (out) memcpy(out + k * Q, f + i * Q, Q * sizeof(double));
    ++k;
  }
  if (mass_out) *mass_out = sum;
  free(f);
  free(post);
  free(next);
  return 0;
}

void ora_macro(const double* snap, uint64_t n_nodes, double* rho, double* u) {
  /* d3q19.cpp:20-34 */
  for (uint64_t n = 0; n < n_nodes; ++n) {
    const double* f = snap + n * Q;
    double r = 0.0, mx = 0.0, my = 0.0, mz = 0.0;
    for (int i = 0; i < Q; ++i) {
      r += f[i];
      mx += (double)kC[i][0] * f[i];
      my += (double)kC[i][1] * f[i];
      mz += (double)kC[i][2] * f[i];
    }
    rho[n] = r;
    u[3 * n] = mx / r;
    u[3 * n + 1] = my / r;
    u[3 * n + 2] = mz / r;
  }
}

double ora_max_rel_diff(const double* a, const double* b, uint64_t n) {
  double worst = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    const double denom = fmax(fabs(a[i]), fabs(b[i]));
    if (denom == 0.0) continue;
    const double r = fabs(a[i] - b[i]) / denom;
    if (r > worst) worst = r;
  }
  return worst;
}
