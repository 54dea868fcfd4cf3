/* TEST INFRASTRUCTURE ONLY -- the CPU restatement ("port") oracle.
 *
 * A plain-C restatement of the reference lbmbench algorithm for the D3Q19 TRT
 * stream-collide path, used by tests/ (as the checker), __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg.  It is never linked into, loaded by or
 * called from the product (paper_1711_11468_b200/).  Every function cites the
 * reference file:line it restates (paths relative to /root/reference/proj).
 *
 * Parity of this restatement is pinned bit-for-bit against the unmodified
 * reference (oracle/_ref/liblbm_ref.so) by tests/test_oracle_pin.py and by the
 * golden fixtures in tests/golden/ (made by tests/golden/make_golden.py).
 */
#ifndef LBM_ORACLE_H
#define LBM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* d3q19.hpp:107-144 */
void ora_collide_node(double* f, double omega_plus, double omega_minus,
                      const double* g);
/* d3q19.hpp:70-73 */
double ora_omega_minus(double omega_plus, double magic_lambda);
/* d3q19.cpp:7-18 */
void ora_equilibrium(double rho, const double* u, double* f);

/* geometry.cpp:40-111 (+ pipe_diameter extension, 0 = stock r).
 * kind: 0 channel, 1 slit, 2 pipe, 3 blocks.  Returns 0 or 1 (config). */
int ora_geometry(int kind, int nx, int ny, int nz, int block, int spacing,
                 int pipe_diameter, uint8_t* flags, int* periodic,
                 int64_t* n_fluid);

/* list_lattice.cpp:84-121 ; mode 0 none, 1 auto, 2 thrash, 3 explicit */
void ora_padding_offsets(uint64_t n_fluid, int mode, const int64_t* pads,
                         uint64_t* starts, uint64_t* total);

/* list_lattice.cpp:123-141 ; returns n_fluid, fills nodes (3 x int32) and
 * rank (uint32 per box node, UINT32_MAX if solid) when non-null. */
int64_t ora_order_nodes(const uint8_t* flags, int nx, int ny, int nz, int blk,
                        int32_t* nodes, uint32_t* rank);

/* list_lattice.cpp:149-204 ; adjacency [n*18 + d-1] */
void ora_build_adjacency(const uint8_t* flags, const int* periodic, int nx,
                         int ny, int nz, const int32_t* nodes,
                         const uint32_t* rank, int64_t n_fluid, int layout_soa,
                         const uint64_t* starts, int scatter, uint32_t* adj);

/* harness.cpp:50-62 */
void ora_perturbed(uint64_t n_fluid, uint64_t seed, double amplitude,
                   double* out);
/* harness.cpp:27-39 */
uint64_t ora_fingerprint(const double* data, uint64_t count);
uint64_t ora_fingerprint_u32(const uint32_t* data, uint64_t count);

/* tests/support/reference.hpp:33-105: the textbook full-way (family 0) and
 * half-way (family 1) steppers on a dense node-major f[V*19] array in
 * (x*ny+y)*nz+z order.  `init` is a canonical fluid-node state (N*19) or NULL
 * for the weights; the result is written canonically to `out` (N*19).
 * mass_out (optional) receives the Kahan sum the matching reference kernel
 * reports (full_lattice.cpp:72-87 over all nodes / list_lattice.cpp:282-294
 * over the fluid list). */
int ora_run(int family, const uint8_t* flags, const int* periodic, int nx,
            int ny, int nz, const double* init, long steps, double omega_plus,
            double omega_minus, const double* g, double* out,
            double* mass_out);

/* harness.cpp:64-80 -> per-node rho, u (bare moments) from a canonical
 * snapshot. */
void ora_macro(const double* snap, uint64_t n_nodes, double* rho, double* u);

/* max over components of |a-b|/max(|a|,|b|), zeros skipped
 * (tests/support/reference.hpp:144-153) */
double ora_max_rel_diff(const double* a, const double* b, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
