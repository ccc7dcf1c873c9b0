/*
 * tlbm.h -- C ABI of the B200 tiled sparse-geometry D3Q19 LBM path
 * (libtlbm.so, built from paper_1611_02445_b200/csrc/ for sm_100a).
 *
 * The reference (`tilelbm`, /root/reference/pkg/src/tilelbm) is pure Python
 * with no FFI; each entry point below replaces the reference function named
 * beside it, and the Python host mirror (paper_1611_02445_b200/*.py) keeps the
 * reference's names and shapes on top of these calls via ctypes.
 *
 * Conventions
 *   - Every pointer prefixed d_ is device memory owned by the caller
 *     (allocated by PyTorch); the library never allocates persistent memory
 *     and never frees caller memory.  Pointers prefixed h_ are host memory.
 *   - `stream` is a cudaStream_t; every call is asynchronous on it unless its
 *     comment says it synchronises.
 *   - Return value: 0 on success, otherwise a TLBM_ERR_* code; the message
 *     is in tlbm_last_error() (thread-local).
 *   - dtype: TLBM_F64 / TLBM_F32.  fluid: TLBM_INCOMPRESSIBLE / TLBM_QUASI
 *     (collision.py:28-30).  table: TLBM_TABLE_* (layout.py:34-36 + B200).
 *   - Field store: one copy is t_n * 19 * 64 values, block (tile, q) at
 *     ((tile * 19) + q) * 64, slot inside the block given by the table's
 *     layout for q (layout.py:115-132 with copy-major order for two copies).
 */
#ifndef TLBM_H
#define TLBM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLBM_ABI_VERSION 3

enum { TLBM_F64 = 0, TLBM_F32 = 1 };
enum { TLBM_INCOMPRESSIBLE = 0, TLBM_QUASI = 1 };
enum { TLBM_LBGK = 0, TLBM_MRT = 1 };   /* collision.py:33-35 CollisionModel */
enum { TLBM_TABLE_XYZ = 0, TLBM_TABLE_OPTIMIZED = 1, TLBM_TABLE_B200 = 2 };
enum { TLBM_OK = 0, TLBM_ERR_ARG = 1, TLBM_ERR_CUDA = 2 };
/* step variants (SPEC.md:531-539 bench ladder) */
enum { TLBM_FULL = 0, TLBM_PROPAGATION_ONLY = 1, TLBM_READ_WRITE_ONLY = 2 };
/* collision arithmetic of the step: REFERENCE keeps numpy's unfused operation
 * order (bit-identical to the reference); FMA contracts the equilibrium and
 * relaxation products into fused multiply-adds and applies an MRT operator of
 * the form M^-1 diag(s) M (s = 0 on the conserved moments) in moment space
 * (fewer instructions; parity within the stated 1e-12 tolerance); any other
 * MRT operator runs in reference arithmetic.  FMA is fp64-only: in fp32 it
 * drifts past the 1e-5 bar (u: 1.1e-5 after 1000 cavity steps). */
enum { TLBM_ARITH_REFERENCE = 0, TLBM_ARITH_FMA = 1 };
/* bits of the device status word written by tlbm_step / tlbm_macroscopic */
enum { TLBM_FLAG_DIVERGED = 1, TLBM_FLAG_GUARD = 2 };

int tlbm_abi_version(void);
const char *tlbm_last_error(void);
int tlbm_set_device(int device);
/* L2 fetch granularity hint of the current device (cudaLimitMaxL2FetchGranularity,
 * 0..128 bytes); sparse geometries over-fetch less at 32. */
int tlbm_set_l2_fetch_granularity(int bytes);
int tlbm_get_l2_fetch_granularity(int *bytes);

/* Host-only: the compiled-in lattice and layout tables, for CPU checks.
 * e: 19x3 int32, opp: 19 int32, w: 19 double, perm: 19x64 int32 slot
 * permutation of `table` (layout.py:108-112 table_permutations). */
int tlbm_lattice_tables(int table, int32_t *h_e, int32_t *h_opp, double *h_w,
                        int32_t *h_perm);

/* ---- tiler (replaces tiling.py:51-83 build_tiling) ---------------------- */
/* Scratch bytes needed by tlbm_tile_map for an nx*ny*nz grid. */
size_t tlbm_tiling_scratch_bytes(int nx, int ny, int nz);
/* Occupancy of every 4^3 tile of the SOLID-padded grid and the order-stable
 * compaction in (z outer, y, x inner) scan order.  Writes d_tile_map
 * (ntx, nty, ntz) C-order int32 (-1 = empty) and *h_t_n.  Synchronises
 * `stream` (t_n is needed to size every other buffer). */
int tlbm_tile_map(const uint8_t *d_types, int nx, int ny, int nz,
                  int32_t *d_tile_map, void *d_scratch, int64_t *h_t_n,
                  void *stream);
/* Corner coordinates of the non-empty tiles, (t_n, 3) int32. */
int tlbm_tile_list(const int32_t *d_tile_map, int ntx, int nty, int ntz,
                   int32_t *d_non_empty, int64_t t_n, void *stream);
/* Neighbour tile index for all 27 deltas (dx,dy,dz) in itertools.product
 * order, (t_n, 27) int32, -1 absent/outside; periodic_mask bit a wraps axis a
 * (replaces txmodel.py:145-160 _neighbor_indices). */
int tlbm_tile_neighbors(const int32_t *d_tile_map, int ntx, int nty, int ntz,
                        const int32_t *d_non_empty, int64_t t_n,
                        int periodic_mask, int32_t *d_nbr, void *stream);
/* Per-slot node metadata word (see csrc/d3q19.cuh), (t_n, 64) uint32; also
 * counts into *d_bad the inlet/outlet nodes not on exactly one domain face
 * (boundaries.py:95-129 classify_boundary_faces rejects those). */
int tlbm_node_meta(const uint8_t *d_types, int nx, int ny, int nz,
                   int periodic_mask, const int32_t *d_non_empty, int64_t t_n,
                   uint32_t *d_meta, int32_t *d_bad, void *stream);
/* Non-solid node count per tile, (t_n,) int32 (tiling.py:141-152). */
int tlbm_tile_counts(const uint32_t *d_meta, int64_t t_n, int32_t *d_counts,
                     void *stream);

/* ---- field store (replaces layout.py:135-167 FieldStore I/O) ------------ */
/* One copy := equilibrium(rho, u) in all 64 slots of every tile
 * (collision.py:94-121). */
int tlbm_init_equilibrium(void *d_f, int dtype, int fluid, int table,
                          int64_t t_n, double rho, double ux, double uy,
                          double uz, void *stream);
/* One copy := equilibrium(rho[t,j], u[:,t,j]) from canonical (t_n,64) rho and
 * (3,t_n,64) u of the working dtype. */
int tlbm_init_from_macroscopic(void *d_f, int dtype, int fluid, int table,
                               int64_t t_n, const void *d_rho, const void *d_u,
                               void *stream);
/* Stored blocks <-> canonical (19, t_n, 64) (layout.py:155-167). */
int tlbm_to_canonical(const void *d_f, int dtype, int table, int64_t t_n,
                      void *d_canon, void *stream);
int tlbm_from_canonical(const void *d_canon, int dtype, int table,
                        int64_t t_n, void *d_f, void *stream);
/* rho (t_n,64), u (3,t_n,64), p (t_n,64) of one copy in canonical order
 * (collision.py:75-91 applied to read_canonical); d_p may be NULL.  Sets
 * TLBM_FLAG_DIVERGED in *d_flags for rho <= 0 (quasi) or NaN. */
int tlbm_macroscopic(const void *d_f, int dtype, int fluid, int table,
                     int64_t t_n, void *d_rho, void *d_u, void *d_p,
                     uint32_t *d_flags, void *stream);
/* Dense-array macroscopic of canonical f (19, n): rho (n), u (3, n), p (n)
 * (collision.py:75-91 on arbitrary node batches). */
int tlbm_macroscopic_canonical(const void *d_f, int dtype, int fluid,
                               int64_t n, void *d_rho, void *d_u, void *d_p,
                               uint32_t *d_flags, void *stream);
/* equilibrium (19, n) from rho (n), u (3, n) (collision.py:94-121). */
int tlbm_equilibrium(const void *d_rho, const void *d_u, int dtype, int fluid,
                     int64_t n, void *d_feq, void *stream);
/* collide_lbgk on (19, n) canonical populations in place (collision.py:124). */
int tlbm_collide_lbgk(void *d_f, int dtype, int fluid, int64_t n, double tau,
                      uint32_t *d_flags, void *stream);
/* collide_mrt on (19, n) canonical populations in place with the host
 * float64 19x19 operator h_op (collision.py:234-247). */
int tlbm_collide_mrt(void *d_f, int dtype, int fluid, int64_t n, const double *h_op,
                     uint32_t *d_flags, void *stream);
/* collide_mrt with an explicit float64 operator on float32 populations
 * (collision.py:234-247 under NumPy's promotion): f + apply_operator(op,
 * feq - f) with the wide accumulation of tlbm_apply_operator. */
int tlbm_collide_mrt_wide(void *d_f, int fluid, int64_t n, const double *h_op,
                          uint32_t *d_flags, void *stream);
/* apply_operator (collision.py:216-231) on (19, n) canonical data:
 * out[i] = sum over j with op[i][j] != 0, in j order, of op[i][j] * delta[j],
 * in the data dtype.  wide = 1 with float32 data: a float64 operator, each
 * term and partial sum formed in float64 and rounded to float32 after every
 * accumulation (NumPy's `acc += c * delta[j]` for a float64 scalar c). */
int tlbm_apply_operator(const void *d_delta, void *d_out, int dtype, int64_t n,
                        const double *h_op, int wide, void *stream);
/* Zou-He closure in place on (19, m) canonical populations of nodes on one
 * face (face = 2*axis + (0 low | 1 high)); kind 0 = velocity inlet with
 * (ux,uy,uz) (boundaries.py:139-157), 1 = pressure outlet with rho0
 * (boundaries.py:160-176).  d_ret (m), optional, receives the implied density
 * (kind 0) or normal momentum (kind 1) the reference returns. */
int tlbm_zou_he(void *d_g, int dtype, int fluid, int face, int kind, int64_t m,
                double ux, double uy, double uz, double rho0, void *d_ret,
                void *stream);

/* Slab halo of a z decomposition: pack (pack=1) the outer z
 * plane of tiles [tile_begin, tile_end) of one copy for the 5 directions
 * leaving it upward (up=1: T NT ST ET WT, plane z=3) or downward (up=0:
 * B NB SB EB WB, plane z=0) into d_buf (80 values per tile), or unpack
 * (pack=0) d_buf into the same slots of ghost tiles. */
int tlbm_halo(void *d_f, int dtype, int table, int64_t tile_begin,
              int64_t tile_end, int up, int pack, void *d_buf, void *stream);

/* ---- the step (Alg. 2; boundaries.py:1-28) ------------- */
typedef struct {
    int dtype, fluid, table, variant;
    int64_t t_n;                 /* tiles in the store */
    int64_t tile_begin, tile_end;/* range of tiles updated by this launch */
    const void *f_src;           /* current copy */
    void *f_dst;                 /* other copy */
    const int32_t *nbr;          /* (t_n, 27) */
    const uint32_t *meta;        /* (t_n, 64) */
    double tau;
    double inlet_u[3];
    double outlet_rho;
    double u_guard;              /* |u| > u_guard sets TLBM_FLAG_GUARD; 0 off */
    uint32_t *flags;             /* device status word (OR-ed), may be NULL */
    int rel32;                   /* 1: every |nbr[t][k] - t| * 1216 < 2^31, so the
                                    kernel may use 32-bit relative offsets */
    /* fused halo (multi-GPU slabs, may be NULL): post-collision values of the
     * e_z=+1 directions on plane z=3 of tiles [halo_up_begin, halo_up_end) are
     * also stored to halo_up + (tile - halo_up_begin) * 19 * 64 (+ the usual
     * in-block offset) -- a neighbour's ghost tiles in peer memory; likewise
     * e_z=-1 / plane z=0 to halo_down. */
    void *halo_up;
    int64_t halo_up_begin, halo_up_end;
    void *halo_down;
    int64_t halo_down_begin, halo_down_end;
    int collision;               /* TLBM_LBGK or TLBM_MRT */
    const double *mrt_op;        /* MRT: host 19x19 float64 operator M^-1 S M,
                                    row-major (collision.py:206-213); cast to
                                    the working dtype like op.astype(dtype) */
    int arith;                   /* TLBM_ARITH_REFERENCE or TLBM_ARITH_FMA */
    /* graph-replayable status ring (may be NULL): when set, `flags` is the
     * base of a ring of ring_len words and the launch ORs its status into
     * flags[(*iter_counter + iter_add) % ring_len], the iteration number read
     * on the device (only by warps that have a status bit to report), so one
     * captured CUDA graph of K steps can be replayed with
     * tlbm_advance_counter(iter_counter, K) as its last node. */
    const int64_t *iter_counter;
    int64_t iter_add;
    int ring_len;
    /* compact tile storage (crank NULL = the paper's 64-slot blocks): the
     * copies hold only non-solid slots in XYZ order, tile t's 19 blocks at
     * cbase[t] (element offset), each cnf[t] values long, slot j at rank
     * crank[t][j] (tlbm_compact_ranks).  Table xyz only; no fused halo. */
    const int64_t *cbase;
    const int32_t *cnf;
    const uint8_t *crank;
    /* traversal order (may be NULL = tile order): launch position
     * p in [tile_begin, tile_end) updates tile order[p]; a permutation that
     * keeps z neighbours close in time keeps lines they share in L2 */
    const int32_t *order;
    /* fused halo on compact storage: the neighbour's block offsets (cbase)
     * of its ghost tiles, indexed tile - halo_*_begin; halo_up / halo_down
     * then point at the neighbour's copy, not at its ghost layer */
    const int64_t *halo_up_cbase;
    const int64_t *halo_down_cbase;
    /* node-parallel traversal of a compact store (node_meta NULL = one
     * 64-thread group per tile): one thread per non-solid node, nodes
     * [node_begin, node_end) in store order (tile-major, rank-minor) --
     * the nodes of tiles [tile_begin, tile_end) -- with the per-node records
     * of tlbm_compact_nodes; needs 19 * n_fn < 2^32 (rel32). */
    const uint32_t *node_meta;
    const void *node_rec;
    const int32_t *unit_tile;
    const void *entries;
    int64_t node_begin, node_end;
} tlbm_step_args;

int tlbm_step(const tlbm_step_args *a, void *stream);
/* ---- compact tile storage (csrc/compact.cu; an extension of layout.py) --- */
/* (t_n, 64) uint8: rank[t][j] = non-solid slots of tile t before slot j
 * (255 for a solid slot). */
int tlbm_compact_ranks(const uint32_t *d_meta, int64_t t_n, uint8_t *d_rank, void *stream);
/* Per-node records of a compact store for the node-parallel step
 * (tlbm_step_args.node_meta; one thread per non-solid node, so a tile's
 * solid slots cost no lanes).  Node n (store order: tile-major, rank-minor):
 *   d_node_meta[n] = its node word (bits 0-24) | slot << 25
 *   d_node_rec[n]  = 4 x uint32: the rank, in its source tile, of the value
 *                    it pulls in direction q = 1..18 -- its own rank where
 *                    the link is missing (bounce-back) -- (6 bits each, five
 *                    per word: q-1 = 5w + i at bits 6i of word w), its own rank
 *                    at bits 18-23 and its tile - d_unit_tile[n / 64] at
 *                    bits 24-29 of word 3
 *   d_unit_tile[u] = the tile of node 64u            (ceil(n_fn / 64))
 *   d_entries[t][k] = {low 32 bits of cbase, cnf} of neighbour entry k of
 *                    tile t (the tile itself where there is none)  (t_n x 27)
 * d_base / d_nf / d_rank: the compact store's cbase / cnf / crank. */
int tlbm_compact_nodes(const uint32_t *d_meta, const int32_t *d_nbr, int64_t t_n,
                       int64_t n_fn, const int64_t *d_base, const int32_t *d_nf,
                       const uint8_t *d_rank, uint32_t *d_node_meta, uint32_t *d_node_rec,
                       int32_t *d_unit_tile, uint32_t *d_entries, void *stream);

/* Convert one copy between the paper's XYZ block store ((t_n, 19, 64)
 * blocks) and the compact store (19 * n_fn values); to_compact 1: blocks ->
 * compact, 0: compact -> blocks (solid slots written as the rest state w_q). */
int tlbm_compact_convert(const void *d_in, void *d_out, int dtype, int table,
                         int64_t t_n, const int64_t *d_base, const int32_t *d_nf,
                         const uint8_t *d_rank, int to_compact, void *stream);

/* tlbm_halo on a compact store (same packed buffer; solid slots pack as 0). */
int tlbm_halo_compact(void *d_f, int dtype, int64_t tile_begin, int64_t tile_end, int up,
                      int pack, void *d_buf, const int64_t *d_base, const int32_t *d_nf,
                      const uint8_t *d_rank, void *stream);

/* ---- geometry generation (csrc/generate.cu; geometry.py:200-269) -------- */
/* For m sphere centres (3 doubles each, d_centres), every voxel of the n^3
 * box (C order) covered by sphere i -- ((x+.5-c0)^2 + (y+.5-c1)^2) +
 * (z+.5-c2)^2 <= radius^2 in float64 -- gets d_first = min(d_first,
 * first_index + i); the host derives the reference's stopping sphere from
 * the per-index counts (geometry.generate_sphere_pack(device=...)). */
int tlbm_sphere_cover(const double *d_centres, int64_t first_index, int64_t m, int n,
                      double radius, int32_t *d_first, void *stream);

/* Vessel tree (geometry.py:generate_vessel_tree): d_discs holds, for every
 * z plane, nb slots of (cx, cy, r) of which the first d_count[z] are used; a
 * voxel (x, y, z) of the nx*ny*nz box (C order) is lumen when margin <= x <
 * nx - margin, margin <= y < ny - margin and (x-cx)^2 + (y-cy)^2 <= r^2 in
 * float64 for some used disc (d_lumen, nx*ny*nz bytes of scratch).  d_types
 * receives SOLID / BB_WALL / FLUID, with FLUID on z = 0 as VELOCITY_INLET and
 * on z = nz-1 as PRESSURE_OUTLET (lumen with all six neighbours in the lumen
 * is FLUID; x/y outside the box count as solid, z replicates the end planes). */
int tlbm_vessel_tree(const double *d_discs, const int32_t *d_count, int nb, int nx, int ny,
                     int nz, int margin, uint8_t *d_lumen, uint8_t *d_types, void *stream);

/* *d_counter += k (one thread; the last node of a captured step graph). */
int tlbm_advance_counter(int64_t *d_counter, int64_t k, void *stream);

/* ---- peer memory for the fused halo (csrc/peer.cu) ---------------------- */
/* CUDA IPC export of a device pointer: 64-byte handle + offset of d_ptr in
 * its allocation; import maps a neighbour's allocation and returns the
 * pointer at that offset (close with the mapping base = ptr - offset). */
int tlbm_ipc_export(void *d_ptr, void *h_handle, uint64_t *h_offset);
int tlbm_ipc_import(const void *h_handle, uint64_t offset, void **d_ptr);
int tlbm_ipc_close(void *d_base);
/* Stream-ordered step barrier between slab neighbours: wait until all n
 * inbox counters >= value (acquire, system scope; sets *d_error and returns
 * after timeout_ns instead of hanging), and publish value into up to two
 * neighbours' inbox slots after a system-scope fence. */
int tlbm_peer_wait(const uint64_t *d_inbox, int n, uint64_t value, uint64_t timeout_ns,
                   uint32_t *d_error, void *stream);
int tlbm_peer_signal(uint64_t *d_peer_a, uint64_t *d_peer_b, uint64_t value, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* TLBM_H */
