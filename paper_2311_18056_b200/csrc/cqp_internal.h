// Internal declarations shared by the translation units of libcqp_b200.so.
// Public surface: include/cqp_b200.h.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "cqp_b200.h"

namespace cqp {

constexpr int kMaxSmemBytes = 232448;  // 227 KB opt-in dynamic shared memory per CTA (sm_100)
constexpr int kComputeThreads = 512;   // 16 compute warps of the persistent solve kernel
constexpr int kComputeWarps = kComputeThreads / 32;
constexpr int kLoaderWarps = 3;         // the only warps that poll L2 for the iterate
constexpr int kLoaderThreads = kLoaderWarps * 32;
constexpr int kThreads = kComputeThreads + 32 + kLoaderThreads;  // + 1 publisher warp + loaders
// W streaming ring of the L2/HBM tier: a stage holds 16 rows x 128 column pairs (32 KB)
constexpr int kStageRows = 16, kStagePairs = 128;
constexpr int kStageDoubles = kStageRows * kStagePairs * 2;
constexpr int kMaxStages = 6;
constexpr int kMaxInlineX0 = 128;  // x0 of an MPC step rides in the kernel parameters up to this size
constexpr int kWarps = kThreads / 32;

// Resident MPC server (cqp_mpc_server_start): the mailbox is host-mapped pinned memory, 64-bit words.
// The host writes x0 then REQ; the kernel answers by writing the result record and then RESP = REQ.
constexpr int kMbReq = 0;       // host -> device: sequence number of the newest request
constexpr int kMbStop = 1;      // host -> device: non-zero = leave the loop
constexpr int kMbResp = 2;      // device -> host: sequence number of the newest answered request
constexpr int kMbExited = 3;    // device -> host: the kernel has left its loop (stop or idle timeout)
constexpr int kMbStepNs = 4;    // device -> host: duration of the last step on the device (%globaltimer)
constexpr int kMbWantFull = 5;  // host -> device: also write y, z, lambda (else only the head and u0)
constexpr int kMbX0 = 8;        // x0 (kMaxInlineX0 doubles)
constexpr int kMbWords = kMbX0 + kMaxInlineX0;
constexpr unsigned long long kSrvExit = ~0ull;  // relay token: leave the loop

inline int pad2(int x) { return (x + 1) & ~1; }

void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define CQP_CUDA(call)                                        \
  do {                                                        \
    cudaError_t e__ = (call);                                 \
    if (e__ != cudaSuccess) return ::cqp::cuda_fail(e__, #call); \
  } while (0)

// Header of the device result buffer; followed by the record arrays and y, z, lambda.
struct DevResultHead {
  int status;
  int iterations;
  int n_trace;
  int n_hist;
  double r_prim;
  double r_dual;
  int final_layer;
  int final_buf;
};

// Everything the persistent kernel needs (device pointers; row-major padded matrices).
struct RunParams {
  int n, m, D;
  int npad, mpad, Dpad;  // even-padded leading dimensions
  int L;
  int R;        // rows of W owned by one CTA
  int G;        // CTAs
  int w_smem;   // 1: W slice resident in shared memory; 0: streamed from global (L2/HBM) [grid kernel]
                //    / kept in registers [cluster kernel, register mode]
  int wdoubles;       // grid kernel: shared-memory doubles reserved for W (resident slice or ring)
  int sb_rows;        // grid kernel, streaming: rows per super-block of the W stream (<= kStageRows)
  int stream_stages;  // grid kernel, w_smem == 0: stages of the cp.async.bulk ring (0: plain global loads)
  // grid kernel, L2/HBM tier, structured layer: the lambda rows of W, [rho G, -diag(rho), I]
  // (layers.cpp:159-161), are streamed as their first n columns only; the two diagonal terms are
  // added by the publisher.  CTAs [0, G12) own R12 rows each of the first n + m rows, the other CTAs
  // R3 lambda rows each (R12 * D ~ R3 * n: equal bytes per CTA).  R = max(R12, R3) sizes the buffers.
  int structured;
  int G12, R12, R3;
  int sb_rows3;          // rows per super-block of the W stream in the lambda-row CTAs
  int nparts;            // per-row partial sums kept per parity: 16 (one per compute warp) or, for handles
                         // that always stream, 4
  int cofetch;           // grid kernel: 1: the compute warps fetch the iterate along with the loaders; 2 (resident
                         // tier): direct fetch, every compute thread polls for its own column pairs (run_kernel)
  int wreg;              // direct fetch: column pairs of W per compute thread kept in registers (0: shared memory)
  int stage_doubles;     // doubles per ring stage (re-tiled stream: h->stage_doubles; row segments: kStageDoubles)
  int cw12, cw3;         // column pairs per ring stage (chunk width): a stage holds nv rows x cw pairs
                         // <= 32 KB, so super-blocks of fewer than 16 rows take wider chunks (one bulk
                         // copy per stage: the fewer and larger the copies, the higher the streaming rate)
  size_t wt_level_pairs; // double2 elements per ladder level of Wt
  int xs_stride;  // cluster kernel: doubles between the two shared-memory copies of the iterate
  int hg_smem;    // cluster kernel: the CTA's rows of H, G', G are cached in shared memory
  const double* W;    // [L][D][Dpad] row-major
  const double* Wt;   // same data re-tiled for the L2/HBM tier's streamer (null: stream row segments):
                      // per CTA slice, per 16-row super-block, per 128-pair chunk: [nv rows][cw pairs]
                      // contiguous, so one cp.async.bulk moves a whole ring stage
  const double* Dk;   // [L][n+m][npad]  rows 0..n: D_k, rows n..n+m: G D_k (bias operator)
  const double* H;    // [n][npad]   unscaled
  const double* Gr;   // [m][npad]   unscaled G, row-major
  const double* Gt;   // [n][mpad]   unscaled G', row-major
  const double* Gs;   // [m][npad]   scaled G, row-major (refresh_z)
  const double* E;    // n
  const double* F;    // m
  const double* rho_vec;  // [L][m] penalty of every constraint row per ladder level
  double cost_scale;
  const double* grid;      // L
  const double* log_grid;  // L  (log10 of the grid values, computed on the host)
  const double* grid_bound;  // L - 1 bounds between neighbouring grid values (nearest_grid_index_fast), or null
  const double* g;   // n unscaled
  const double* c;   // m unscaled
  const double* d;   // m unscaled
  double* vq;        // [4][ring_ld] iterate ring; between launches slot 0 = iterate, 1..3 = sentinel
  int ring_ld;       // doubles between two slots of the ring (Dpad rounded up: slots do not share L2 lines)
  int* state;        // [0] layer index
  unsigned* barrier;       // grid barrier counter of this launch (zero on entry)
  unsigned* barrier_next;  // counter of the next launch, zeroed by this one
  int* dbg;                // host-mapped watchdog record
  double* partial;    // [G][8] per-CTA partial maxima
  double eps_prim, eps_dual, threshold;
  int check_interval, adaptive, early_exit, total_iters;
  int do_refresh;     // run Solver::refresh_z before the first iteration
  int gate_cycles, gate_adapt, gate_up, gate_down, gate_max;  // direct fetch: the publisher's poll gate (run_kernel)
  int fence_mode;     // 0: fence after re-arm (default); 2: release-store publish
  int poll_delay_ns;  // the fetching warps pause this long after `go` before their first poll of v_i
  int cap;            // capacity of the record arrays
  // receding-horizon control extraction (null Kt: none): u0 = clamp(-K x0 + y[0:nu], u_lo, u_hi)
  const double* mpc_K;   // [nu][nxpad] row-major
  const double* mpc_x0;  // nx
  const double* mpc_ulo; // nu
  const double* mpc_uhi; // nu
  int mpc_nx, mpc_nxpad, mpc_nu;
  double* out_u;         // nu (in the result record)
  // resident MPC server (server != 0): the kernel loops { wait for x0 in the mailbox; instantiate;
  // refresh_z; total_iters iterations; final pass; answer } until told to stop or idle for idle_ns
  int server;
  int srv_cache;                      // cluster kernel: template / bias-operator rows cached in shared memory
  volatile unsigned long long* mb;    // mailbox (kMb* words), host-mapped
  unsigned long long served;          // newest request already answered when the kernel starts
  unsigned long long* srv_seq;        // device relay: CTA 0 republishes the request number here
  long long idle_ns;
  const double* mpc_og;  // [n][nxpad] offset_g, [m][nxpad] offset_c, c_base, d_base (mpc.cpp:260-270)
  const double* mpc_oc;
  const double* mpc_cb;
  const double* mpc_db;
  double* mpc_x0_w;      // writable alias of mpc_x0 (the relay target)
  double* g_w;           // writable aliases of g, c, d (the in-kernel instantiate)
  double* c_w;
  double* d_w;
  DevResultHead* head;
  int* trace;         // [cap][2]
  int* hist_i;        // [cap][2]  (iteration, grid index)
  double* hist_r;     // [cap][2]  (r_prim, r_dual)
  double* out_y;      // n
  double* out_z;      // m
  double* out_lam;    // m
};

}  // namespace cqp

struct cqp_handle {
  int n = 0, m = 0, D = 0, L = 0;
  int npad = 0, mpad = 0, Dpad = 0;
  cqp_settings s{};
  int device = 0;
  int num_sms = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int initial_index = 0;
  double cost_scale = 1.0;
  std::vector<double> grid, E_host, F_host;
  // device memory
  double *W = nullptr, *Dk = nullptr;  // Dk: [L][n+m][npad] = [D_k; G D_k]
  double* Wt = nullptr;                // tier 1 only: W re-tiled for contiguous streaming (built lazily)
  double *H = nullptr, *Gr = nullptr, *Gt = nullptr, *Gs = nullptr;
  double *E = nullptr, *F = nullptr, *dgrid = nullptr, *dlog_grid = nullptr;  // dlog_grid: [log10(grid) (L); bounds (L)]
  bool grid_bounds = false;  // the grid is ascending: dlog_grid + L holds the bounds between neighbours
  double *g = nullptr, *c = nullptr, *d = nullptr;  // one allocation [g; c; d] (unscaled)
  double* vq = nullptr;  // [4][ring_ld] iterate ring (see RunParams::vq)
  int ring_ld = 0;
  int* state = nullptr;
  unsigned* barrier = nullptr;  // [2] ping-pong grid-barrier counters
  int launch_parity = 0;
  double* partial = nullptr;
  double* rho_vec = nullptr;  // [L][m]
  double* dtmp = nullptr;     // Dpad scratch (warm start staging)
  // result buffer (device) and its pinned host mirror
  void* dres = nullptr;  // device alias of hres
  void* hres = nullptr;  // host-mapped pinned result record, written by the kernel
  size_t res_bytes = 0;
  int res_cap = 0;
  // pinned staging for update_vectors: [g; c; d]
  double* hstage = nullptr;
  std::vector<double> c_host, d_host;  // current unscaled bounds (for cqp_get_scaling)
  // condensed-MPC template on the device (cqp_mpc_set_template): instantiate() and the control
  // extraction of the closed loop run on the device, a step uploads only x0
  int mpc_nx = 0, mpc_nxpad = 0, mpc_nu = 0;
  double *mpc_og = nullptr, *mpc_oc = nullptr;   // offset_g [n][nxpad], offset_c [m][nxpad] row-major
  double *mpc_cb = nullptr, *mpc_db = nullptr;   // c_base, d_base (m)
  double *mpc_K = nullptr, *mpc_ulo = nullptr, *mpc_uhi = nullptr, *mpc_x0 = nullptr;
  double* hx0 = nullptr;                          // pinned staging of x0
  bool vectors_device_only = false;               // c/d were last set by the device-side instantiate
  bool mpc_extract = false;                       // the next launch also extracts the control
  // resident MPC server
  unsigned long long* mb_host = nullptr;          // mailbox, host-mapped (kMbWords words)
  unsigned long long* mb_dev = nullptr;           // its device alias
  unsigned long long* srv_seq = nullptr;          // device relay word
  bool srv_enabled = false, srv_running = false;
  int srv_k = 0;
  long long srv_idle_ns = 0;
  unsigned long long srv_req = 0;                 // sequence number of the newest request posted
  double srv_last_wall_us = 0.0, srv_last_device_us = 0.0;  // last served step: C-ABI wall / device-side duration
  int* dbg_host = nullptr;  // host-mapped watchdog record (16 ints)
  int* dbg_dev = nullptr;
  // launch configuration
  int R = 0, G = 0, w_smem = 0, rb = 0, smem_bytes = 0;
  int structured = 0, G12 = 0, R12 = 0, R3 = 0;  // tier 1: structured layer partition (RunParams)
  int cw12 = 128, cw3 = 128;                      // tier 1: chunk widths Wt was re-tiled with
  int stage_doubles = 4096;                       // tier 1: doubles per ring stage of the re-tiled stream
  int nparts = 16;                                // per-row partial sums per parity (RunParams::nparts)
  int fetch = 1;                                  // resident tier: RunParams::cofetch (0 loaders, 1 cofetch, 2 direct)
  int stream_stages = 0;  // tier 1: stages of the W streaming ring that fit the shared memory
  int wdoubles = 0;       // shared-memory doubles reserved for W (resident slice or ring)
  int cluster = 0;  // 1: single thread-block cluster with DSMEM exchange (small problems)
  int rpw = 0;      // cluster kernel, shared-memory mode: rows of W per warp
  int npt = 0;      // cluster kernel, register mode: column pairs of W per lane (0: shared-memory mode)
  int xs_stride = 0, hg_smem = 0;
  // tuning / test knobs, read from the environment once at handle creation (cqp_single.cu: read_knobs)
  int knob_poll_delay_ns = -1, knob_fence_mode = 0, knob_cofetch = 2, knob_wreg = 1;
  int knob_gate[5] = {100, 1, 16, 4, 300};
  bool knob_exact_log = false;
  bool knob_sb_balance = true, knob_no_retile = false, knob_wide_chunks = true;
};

namespace cqp {

// cqp_single.cu
int configure_launch(cqp_handle* h);
int launch_run(cqp_handle* h, bool early_exit, int total_iters, bool do_refresh);
int prepare_streaming(cqp_handle* h);  // L2/HBM tier: re-tile the ladder for contiguous streaming
// cqp_cluster.cu : single thread-block cluster kernel for small problems (DSMEM exchange)
int configure_cluster(cqp_handle* h);  // sets h->cluster = 1 and the launch shape when it fits
int launch_cluster(cqp_handle* h, const RunParams& p);
int launch_refresh_z(cqp_handle* h);
int launch_warm_start(cqp_handle* h, const double* dy, const double* dlam, int layer_index);
int launch_set_state(cqp_handle* h, int layer);
int launch_transpose_pad(cudaStream_t st, const double* src_colmajor, int rows, int cols,
                         double* dst_rowmajor, int ld, int src_ld = 0);
int launch_untranspose(cudaStream_t st, const double* src_rowmajor, int rows, int cols, int ld,
                       double* dst_colmajor);
int launch_bias(cqp_handle* h, int k, double* b_out);  // b_out: device, D doubles
int launch_instantiate(cqp_handle* h, const double* x0_host);  // g, c, d <- template(x0) on the device
int server_launch(cqp_handle* h, int k);   // start the resident MPC kernel for k iterations per step
int server_stop(cqp_handle* h);            // leave the loop and wait for the kernel (no-op when not running)

// cqp_batch.cu : dense DMMA GEMM with an identity slot map, used by the offline stage
struct DenseGemm;
int dense_gemm_create(DenseGemm** out, int N, int num_sms);
void dense_gemm_destroy(DenseGemm* g);
int dense_gemm_run(const DenseGemm* g, cudaStream_t st, const double* A, int lda, int M, int M_pad,
                   const double* B, int ldb, double* C, int ldc, double alpha);

}  // namespace cqp
