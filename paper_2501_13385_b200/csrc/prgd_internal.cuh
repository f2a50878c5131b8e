// prgd_internal.cuh — shared types and kernel entry points of libprgd (sm_100a).
//
// Data layout in HBM:
//   cores        C_k [r_k][n_k][r_{k+1}] fp64, concatenated (core_off[k]); 0-based cores.
//   Omega        prefix order (bucketed by P = mixed radix of x_0..x_{KL-1}, x_0 most
//                significant): Spre[t] (int32 suffix index), ypre[t], g[t], sid_pre[t].
//                suffix order (bucketed by S = mixed radix of x_KL..x_{d-1}, x_{d-1}
//                most significant): pos_suf[u] (prefix position), Psuf[u].
//   tables       left level k (1..KL): rows prod n[0..k-1], row stride ld = pad(r_k):
//                the left part T^{<=k-1}(x).  Right level k (KL..d-1):
//                rows prod n[k..d-1] (x_k least significant), stride pad(r_k): the
//                right part T^{>=k}(:, x) stored as rows.
//                E_k (left, pass-B accumulations) and F_k (right) use the same shapes.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace prgd {

constexpr int kMaxD = 64;
constexpr int kMaxRank = 32;
constexpr int kDenseThreads = 256;

// Device-side scalars of one context (one allocation).
struct Scalars {
  double eps;        // eps_l of the last weights computation
  double sumsq;      // sum_s g_s^2 at the iterate of the last pass A
  double alpha;      // alpha_l of the last step
  double p;          // M / prod(n)
  double step_size;  // set by k_set_step before each update
  int noop;          // 1: skip the rest of this update (eps = 0 or a fault)
  int err;           // nonzero: numeric fault (sticky until read by the host)
  int index_err;     // set by index validation kernels
  int pad;          // cumulative one-sided Jacobi sweeps (diagnostic)
  long long cyc[24]; // cumulative SM cycles / counters per dense phase (diagnostic)
  double adapt_num[kMaxD];  // adaptive step: ||component k of the tangent vector||_W^2
  double adapt_den;         // adaptive step: ||P_Omega D||^2 (this rank's samples)
  int wpar;                 // parity of the rounding's warm-start buffers (DenseArgs::vwarm)
};

enum ErrBits { kErrNaN = 1, kErrChol = 2, kErrSVD = 4 };

// CSR-like "virtual row" plan of one bucketing side (host-built, device copy).
struct SegPlan {
  int64_t nrows = 0;        // virtual rows (nblk * nrow_real)
  int64_t nrow_real = 0;    // table rows (N_L or N_R)
  int nblk = 1;             // gather blocks
  std::vector<int64_t> blk_warp;    // [nblk+1] warp range of each gather block (host)
  std::vector<int64_t> blk_split;   // [nblk+1] split-row range of each gather block (host)
  int64_t nvrows = 0;
  int64_t nwarps = 0;
  int64_t nsplit = 0;       // rows split over several vrows
  int64_t npart = 0;        // partial slots
  int4* vrow = nullptr;            // per virtual row {table row (virtual), sample count, first
                                   // sample (m < 2^31), partial slot or -1}: one 16-byte load
  int64_t* warp_vbegin = nullptr;  // [nwarps+1]
  int32_t* split_row = nullptr;    // [nsplit]
  int64_t* split_first = nullptr;  // [nsplit+1] partial slot ranges
  double* part = nullptr;          // [npart * ld] partial results
};

// Parameters of the dense (single-CTA) sweep kernels; all pointers device.
struct DenseArgs {
  int d;
  int n[kMaxD];
  int r[kMaxD + 1];
  int64_t core_off[kMaxD + 1];   // offsets of C / U / Y / Ahat (same shapes)
  int64_t phi_off[kMaxD + 1];    // offsets into phi (sum n)
  int64_t b_off[kMaxD + 1];      // offsets of the rank-2r cores B
  int64_t p_off[kMaxD + 1];      // offsets of P_k / chol(P_k), r_{k+1}^2 each
  double* C;       // current cores (input of orth, output of round)
  double* U;       // left-orthogonal cores of That
  double* Y;       // contractions Y_k
  double* Ahat;    // projected variations (debug / reuse)
  double* phi;     // phi_{k,j}
  double* P;       // right Grams
  double* L;       // Cholesky factors
  double* B;       // rank-2r cores (rounding workspace)
  double* work;    // global scratch (>= 2 * max B core + extras)
  int64_t work_len;
  double* clw;     // cluster-rounding scratch: [0, 8192) fallback R, then per-CTA slice buffers
  int64_t clw_len;
  Scalars* sc;
  int smem_doubles;  // dynamic shared memory available to the kernel, in doubles
  int proj_mode;     // k_project: 0 project + assemble, 1 project + adaptive numerator, 2 assemble
  int wretr;         // 1: weighted retraction W^{-1/2} SVD_r^tt W^{1/2}
  double* vwarm;     // [2][d][32*32] the truncation Jacobi's last rotation per bond (warm start) or null
  int* wok;          // [2][d] 1: the slot holds a converged rotation
  int orth_part;     // k_orth_cs: 0 all of A4-A6; 1 A4 + A5 for cores < orth_split; 2 the rest
  int orth_split;    //   (part 1's cores are final when it ends: their tables can start)
};

// ------------------------------------------------------------------ kernels (launchers)
// sort.cu
void launch_make_keys(cudaStream_t s, const int32_t* idx, int64_t m, int d, const int* n_dev,
                      int KL, int bitsP, int bitsS, uint64_t* kpre, uint64_t* ksuf, uint32_t* vals,
                      Scalars* sc, int64_t* launches);
void launch_widen_u8(cudaStream_t s, const uint8_t* in, int64_t count, int32_t* out, int64_t* launches);
void radix_sort_pairs(cudaStream_t s, uint64_t* keys, uint32_t* vals, uint64_t* keys_tmp,
                      uint32_t* vals_tmp, int64_t m, int bits, int* hist_buf, int64_t hist_len,
                      uint64_t** keys_out, uint32_t** vals_out, int64_t* launches);
int64_t radix_hist_len(int64_t m);
void launch_slice_setup(cudaStream_t s, const int32_t* pos_suf, const uint64_t* keys_suf, int bitsP,
                        int64_t m, int64_t slen, int nslices, uint64_t* kbuf, uint32_t* vbuf,
                        uint64_t* ktmp, uint32_t* vtmp, int* hist, int64_t hist_len, int32_t* sl_pos,
                        int32_t* sl_row, int32_t* sl_q, int64_t* launches);
void launch_after_sort_pre(cudaStream_t s, const uint64_t* keys, const uint32_t* sids, int64_t m,
                           int bitsS, int64_t NL, const double* y_orig, int32_t* Spre,
                           double* ypre, int32_t* sid_pre, int32_t* inv, int64_t* offsL,
                           int32_t* Ppre, int64_t* launches);
void launch_after_sort_suf(cudaStream_t s, const uint64_t* keys, const uint32_t* sids, int64_t m,
                           int bitsP, int64_t NR, const int32_t* inv, int32_t* pos_suf,
                           int32_t* Psuf, int32_t* sid_suf, int32_t* pre2suf, int64_t* offsR,
                           int64_t* launches);

// plan.cu: device construction of the pass work plans (SegPlan)
int64_t plan_scan_scratch(int64_t len);
// exclusive scan of int32 into int64 out[0..len] (out[len] = total); bsum: plan_scan_scratch(len)
void launch_scan_i32(cudaStream_t s, const int* in, int64_t len, int64_t* out, long long* bsum,
                     int64_t* launches);
void launch_plan_rows(cudaStream_t s, const int64_t* offs, int64_t nr, int64_t split, int* nv, int* sp,
                      int* np, int64_t* vbase, int64_t* sbase, int64_t* pbase, long long* bsum,
                      int64_t* launches);
void launch_plan_fill(cudaStream_t s, const int64_t* offs, int64_t nr, int64_t nrow, int nblk,
                      int64_t split, const int64_t* vbase, const int64_t* sbase, const int64_t* pbase,
                      int64_t nvrows, int4* vrow, int32_t* split_row, int64_t* split_first, int vcost,
                      int64_t wcost, int* cost, int64_t* C, int* flag, int64_t* wid,
                      long long* bsum, int64_t* blk_out, int64_t* launches);
void launch_plan_warps(cudaStream_t s, const int* flag, const int64_t* wid, int64_t nvrows,
                       int64_t* warp_vbegin, int64_t* launches);

// tables.cu
void launch_table_left(cudaStream_t s, const double* in, int ld_in, const double* core, int r0,
                       int nk, int r1, double* out, int ld_out, int64_t rows_out,
                       const double* rowscale, const Scalars* sc, int64_t* launches);
void launch_table_right(cudaStream_t s, const double* in, int ld_in, const double* core, int r0,
                        int nk, int r1, double* out, int ld_out, int64_t rows_out,
                        const double* rowscale, const Scalars* sc, int64_t* launches);
// scratch (>= a few x rows_out x ld_out doubles, or 0): slice-split partials for levels with
// few output rows
void launch_E_down(cudaStream_t s, const double* Ein, int ld_in, const double* core, int r0,
                   int nk, int r1, double* Eout, int ld_out, int64_t rows_out, double* scratch,
                   int64_t scratch_cap, const Scalars* sc, int64_t* launches);
void launch_F_up(cudaStream_t s, const double* Fin, int ld_in, const double* core, int r0, int nk,
                 int r1, double* Fout, int ld_out, int64_t rows_out, double* scratch,
                 int64_t scratch_cap, const Scalars* sc, int64_t* launches);
// Y_k[i,j,c] = sum_p A[p,i] E[p*nk+j, c]   (left)   or
// Y_k[i,j,c] = sum_q F[j+nk*q, i] B[q, c]  (right); split-K with deterministic reduce.
void launch_Y(cudaStream_t s, bool left, const double* A, int ldA, const double* E, int ldE,
              int64_t nsum, int r0, int nk, int r1, double* Y, double* partial,
              int64_t partial_cap, const Scalars* sc, int64_t* launches);
int64_t Y_partial_need(int64_t nsum, int r0, int nk, int r1);
void tables_init();
// Fused backward level (E_k or F_{k+1} and Y_k in one pass), when r0 nk r1 <= 4096.
bool back_fused_ok(int r0, int nk, int r1);
int64_t back_partial_need(int64_t ngroups, int r0, int nk, int r1);
void launch_back_level(cudaStream_t s, bool left, const double* X, int ldX, const double* V,
                       int ldV, const double* core, int r0, int nk, int r1, double* O, int ldO,
                       int64_t ngroups, double* Y, double* partial, int64_t partial_cap,
                       const Scalars* sc, int64_t* launches);  // shared-memory attributes (call once, outside capture)

// levels.cu: table levels / backward recursions on DMMA with few launches.
struct TableLevel {        // out (flat [rows_out / nk][nk * ld_out]) from in x core
  bool left;
  const double* in;        // null: the one parent row [1]
  int ld_in;
  const double* core;
  int r0, nk, r1;
  double* out;
  int ld_out;
  int64_t rows_out;
  const double* rowscale;
};
struct BackwardLevel {     // O (next E / F level) and Y_k from X (E_{k+1} / F_k) and V (A_k / B_{k+1})
  bool left;
  const double* X;
  int wrow;                // row stride of X's table level (flat row = nk * wrow)
  const double* V;         // null: ones
  int ldV;
  const double* core;
  int r0, nk, r1;
  double* O;               // null: none
  int ldO;
  int64_t ngroups;
  double* Y;
};
bool level_tab_ok(int r0, int nk, int r1, int ld_out);
bool level_back_ok(int r0, int nk, int r1, int wrow);
int64_t level_back_partial_need(int64_t ngroups, int r0, int nk, int r1, int wrow);
void launch_table_levels(cudaStream_t s, const std::vector<TableLevel>& left,
                         const std::vector<TableLevel>& right, const Scalars* sc, int64_t* lc);
void launch_backward_levels(cudaStream_t s, const std::vector<BackwardLevel>& left,
                            const std::vector<BackwardLevel>& right, double* part, int64_t part_cap,
                            const Scalars* sc, int64_t* lc);
void levels_init();

// passes.cu
enum SegMode { kGSQ = 1, kSPMM = 2, kDPASS = 3 };   // (pass A's SDDMM: passes_flat.cu)
struct SegArgs {
  const SegPlan* plan;  // host copy (device pointers inside)
  int mode;
  int ld;               // row stride of the tables / outputs (pad(r))
  const int32_t* col;   // per-sample column / gather index (SDDMM, SPMM)
  const int32_t* perm;  // per-sample index into g (GSQ, SPMM suffix side) or null
  double* g;            // SDDMM writes, GSQ/SPMM read
  double* g2 = nullptr;         // GSQ: the gathered g stored to g2[s]
  const double* rowtab; // DPASS row vectors
  const double* coltab; // gathered table
  const double* rowtab2 = nullptr;  // DPASS: v_s = rowtab.coltab + rowtab2.coltab2
  const double* coltab2 = nullptr;
  const double* rowscale;  // SPMM output scale (psi) or null
  double* out;          // SDDMM/GSQ/DPASS: scalar per row; SPMM: vector per row (ld)
};
void launch_seg(cudaStream_t s, const SegArgs& a, const Scalars* sc, int64_t* launches);

// passes_flat.cu: pass A (prefix order) as a flat sample-major SDDMM with the bucket sums H_L
struct FlatArgs {
  const int32_t* row = nullptr;     // [m] bucket (table row) of each sample, nondecreasing
  const int32_t* col = nullptr;     // [m] gathered table row
  const double* x = nullptr;        // [m] y
  double* g = nullptr;              // [m] output g = v - y
  int64_t m = 0, nrows = 0;
  int64_t ncols = 0;                // rows of the gathered table
  int ld = 2;                       // table row stride (pad(r))
  const double* rowtab = nullptr;   // row vectors (left table)
  const double* coltab = nullptr;   // gathered table (right table)
  double* out = nullptr;            // [nrows] bucket sums of g^2 (H_L)
  void* rec = nullptr;              // chunk records (flat_rec_bytes)
};
int64_t flat_rec_bytes(int64_t m);
void launch_flat_sddmm(cudaStream_t s, const FlatArgs& a, int64_t* launches);
// pass A suffix by slices of g (stage[t] = g[pos[t]], bucket sums of stage^2 into H) and the sum
// of the per-slice bucket sums
void launch_flat_gsq(cudaStream_t s, const int32_t* row, const int32_t* pos, const double* g, int64_t m,
                     int64_t nrows, double* stage, double* H, void* recbuf, int64_t* launches);
void launch_sum_slices(cudaStream_t s, const double* Hq, int nq, int64_t n, double* H, int64_t* launches);
// n_host / phi_off_host are HOST arrays (values are passed by kernel argument).
// scratch: >= 32 * (sum of the nmodes mode sizes) doubles
void launch_marginals(cudaStream_t s, const double* H, int64_t N, int nmodes, const int* n_host,
                      bool msd_first, double* h_out, double* scratch, int64_t* launches);
void launch_weights(cudaStream_t s, const double* h, int d, const int* n_host, int64_t nsum,
                    int eps_rule, double eps_fixed, int step_rule, double* phi, Scalars* sc,
                    int64_t* launches);
void launch_psi(cudaStream_t s, const double* phi, const int64_t* phi_off_host, int KL, int d,
                const int* n_host, int64_t NL, int64_t NR, double* psiL, double* psiR,
                const Scalars* sc, int64_t* launches);
void launch_eval_queries(cudaStream_t s, const int32_t* idx, int64_t count, int d, const int* n_host,
                         int KL, const double* tabL, const double* tabR, int ld, int rb,
                         double* out, Scalars* sc, int64_t* launches);
void launch_set_step(cudaStream_t s, Scalars* sc, double step, int64_t* launches);
void launch_gather_sq_sum(cudaStream_t s, const double* h0, int n0, Scalars* sc, int64_t* launches);

// dense.cu
void launch_dense_orth(cudaStream_t s, const DenseArgs& a, int64_t* launches);
bool orth_cluster_ok(const DenseArgs& a);
void launch_dense_round(cudaStream_t s, const DenseArgs& a, int64_t* launches);
// k_project alone (mode: 1 projection + adaptive numerator, 2 assembly with sc->alpha) and the
// rounding alone (adaptive step: alpha is known only after the D pass)
void launch_project(cudaStream_t s, const DenseArgs& a, int mode, int64_t* launches);
void launch_round_only(cudaStream_t s, const DenseArgs& a, int64_t* launches);

// spectral.cu: spectral initialisation T_0 = SVD_r^tt(p^{-1} P_Omega(y)) (Alg. 1 on the sparse tensor)
struct SpectralArgs {
  int d, KL;
  int n[kMaxD];
  int r[kMaxD + 1];
  int64_t core_off[kMaxD + 1];
  int64_t m, NL, nrows;       // nrows = NL (prefix buckets)
  double p;
  const int64_t* offsL;       // [nrows + 1]
  const int32_t* Spre;        // [m] suffix index per prefix position
  const double* y;            // [m] observed values, prefix order
  double* C;                  // output cores
  int cs;                     // per-sample chain stride (>= max r)
  int32_t* Ppos;
  double *z, *chain, *w;
  uint64_t *keys, *ktmp;
  uint32_t *vals, *vtmp;
  int* hist;
  int64_t hist_len;
  int *flag, *rx, *gflag;
  int64_t *ridx, *rstart, *gidx, *gstart, *rgroup, *byx, *xoff;
  int *lflag, *lnch;                  // long runs: flags, chunk counts
  int64_t *lidx, *llist, *lchoff, *lchl;
  long long* bsum;
  double* gparts;
  int64_t gram_parts_cap;     // doubles in gparts
  double *G, *V;              // W_max^2 each (left Gram path, W = r_{k-1} n_k <= 1024)
  // right Gram path (W > 1024, at most kSpRightMax nonzero columns): dense M_k (Wr_max x Q),
  // its Gram M_k^T M_k and eigenvectors (Q x Q), the selected eigenvectors / eigenvalues
  int64_t Wr_max;             // max W over the right-path steps (0: none)
  double *Md, *Gr, *Vr, *Vsel, *lam;
};
constexpr int kSpRightMax = 1024;
int spectral_init_run(cudaStream_t s, const SpectralArgs& a, std::string* msg, int64_t* launches);

// chains.cu: the per-sample chain path.
struct ChainTT {             // a TT read by the chain kernels; cores in the ABI layout [r][n][r']
  int d;
  int64_t m;                 // samples (interface buffers)
  int n[kMaxD];
  int r[kMaxD + 1];
  int64_t off[kMaxD + 1];      // core offsets
  int64_t phi_off[kMaxD + 1];  // offsets of the per-mode slice arrays (phi, h; bucket index base)
  int64_t il_off[kMaxD + 1];   // offsets of the interface arrays IL_k / IR_k (k = 1..d-1), m r_k each
};
struct ChainPieces {         // the per-mode buckets (A0) cut into pieces of <= P samples
  int32_t* perm = nullptr;   // [d][m] sample ids, bucket-sorted per mode (stable)
  int64_t* offs = nullptr;   // per-mode offsets concatenated: mode k at phi_off[k] + k, n_k + 1 each
  int4* pieces = nullptr;    // {bucket e, mode k, t0, t1}
  int64_t npieces = 0;
  int64_t* pbase = nullptr;  // [nbuckets + 1] first piece of each bucket
  int64_t nbuckets = 0;      // sum n_k
  double* part = nullptr;    // [npieces * stride] piece partial sums
  int stride = 1;            // max r_k r_{k+1}
  int P = 256;
};
int chain_piece_size(int64_t m, int d, int rmax);
// mode 0: out = T(x); 1: out = T(x) - y (pass A); 2: out = T(x)^2 (adaptive denominator, noop-aware)
void launch_chain_eval(cudaStream_t s, int mode, const int32_t* idx, int64_t m, const ChainTT& tt,
                       const double* cores, const double* y, double* out, const Scalars* sc,
                       int* index_err, int64_t* launches);
void launch_chain_iface(cudaStream_t s, const int32_t* idx, int64_t m, const ChainTT& tt, const double* U,
                        const double* phi, const double* g, double* ghat, double* IL, double* IR,
                        const Scalars* sc, int64_t* launches);
void launch_chain_h(cudaStream_t s, const ChainPieces& pc, const ChainTT& tt, int64_t m, const double* g,
                    double* h, int64_t* launches);
void launch_chain_contract(cudaStream_t s, const ChainPieces& pc, const ChainTT& tt, int64_t m,
                           const double* ghat, const double* IL, const double* IR, double* Y,
                           const Scalars* sc, int64_t* launches);
void launch_mode_keys(cudaStream_t s, const int32_t* idx, int64_t m, int d, int k, int nk, uint64_t* keys,
                      uint32_t* vals, int* index_err, int64_t* launches);
void launch_mode_after_sort(cudaStream_t s, const uint64_t* keys, const uint32_t* vals, int64_t m, int64_t nk,
                            int32_t* perm, int64_t* offs, int64_t* launches);
void launch_piece_count(cudaStream_t s, const int64_t* offs_cat, const ChainTT& tt, int64_t nb, int P,
                        int* np, int64_t* launches);
void launch_piece_fill(cudaStream_t s, const int64_t* offs_cat, const int64_t* pbase, int64_t nb,
                       const ChainTT& tt, int P, int4* pieces, int64_t* launches);
void launch_tangent_cores(cudaStream_t s, const double* U, const double* Ahat, const double* phi,
                          const ChainTT& tt, const ChainTT& bt, double* out, const Scalars* sc,
                          int64_t* launches);

// adaptive.cu: the adaptive (steepest) step
void launch_stack_cores(cudaStream_t s, int d, const int* n, const int* r, const int64_t* core_off,
                        int KL, const double* U, const double* Ahat, double* st, const Scalars* sc,
                        int64_t* launches);
void launch_concat2(cudaStream_t s, double* o0, int ldo0, const double* x0, int ldx0, const double* y0,
                    int ldy0, int64_t rows0, int w0, double* o1, int ldo1, const double* x1, int ldx1,
                    const double* y1, int ldy1, int64_t rows1, int w1, const Scalars* sc,
                    int64_t* launches);
int adapt_vsum_parts();
void launch_adapt_den(cudaStream_t s, const double* x, int64_t n, double* part, Scalars* sc,
                      int64_t* launches);
void launch_adapt_alpha(cudaStream_t s, int d, Scalars* sc, int64_t* launches);
int dense_smem_doubles();
int round_cluster_size();
bool round_cluster_ok(int d, const int* r);   // cluster rounding applies (2 max r <= 32)
void dense_init();   // sets the dynamic shared-memory attribute (call once, outside capture)

inline int pad_rank(int r) {
  int p = 2;
  while (p < r) p <<= 1;
  return p;
}

}  // namespace prgd
