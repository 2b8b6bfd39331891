// sb_host.h — host-side helpers shared by the C-ABI entry points (argument checks,
// workspace carving, launch geometry).  No device code.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <atomic>

#include <nvtx3/nvToolsExt.h>

#include "sb_common.cuh"

namespace sb {

// One NVTX range per C-ABI call (SURVEY §5 tracing): a push / pop pair, no-ops unless a
// profiler (nsys, ncu --nvtx) has injected itself.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define SB_NVTX(name) ::sb::NvtxRange sb_nvtx_range_(name)

struct SeqInfo {
  int g, s, L, st;  // clamped gamma_b, branch row s_b, path length L_b, clamp bits
  int Lr;           // rows read per slot-0 path: L_b, or gamma_b+1 when bonus rows are read too
  int pad_[3];
};

// Per physical row partial state of one vocabulary shard (sharded mode, a7).
struct ShardRow {
  float pm, pms;            // p: max, exponent offset
  double pz;                // p: sum
  float qm, qms;            // q: max, offset
  double qz, qs1;           // q: sum, entropy sum
  int qidx;                 // q: first global index of the shard max
  int qfin;                 // q: the slice holds a finite entry (clamped-row tie-break)
};

// Workspace carve-up (all offsets 256-byte aligned).
struct Workspace {
  SeqInfo* info;     // [B]
  int* unit_off;     // [B+1] exclusive scan of tested row pairs per sequence
  int* cnt;          // [B]   rows-kernel completion counters (self-resetting)
  int* sel_cnt;      // [1]   select-kernel completion counter (self-resetting)
  float4* rowstat;   // [B][K][G+1] (MS_p, Z_p, MS_q, Z_q) per physical row
  uint8_t* pflag;    // [B][K][G+1] per token slot: bit0 acc, bit1 bad token, bit2 nonfinite
  int* conf_cnt;     // [B][K] confidence-kernel completion counters (self-resetting)
  float* conf_stat;  // [B][K][G] statistic per row
  float* conf_c;     // [B][K][G] Eq. 7 confidence per row
  float* tok_lp;     // [B][K][G+1] sharded: combined target logit of each path token
  float* segs;       // [B][2][nseg] sharded select: local segment sums (residual, p)
  int4* dec;         // [B] sharded select: decision record
  int* ready;        // [B] fused step: per-sequence phase-1 completion flags
  int* plan;         // [4] fused step: delta, total units
  int* seqpk;        // [B] packed layout of each sequence (k_plan): s | g<<5 | L<<10 | Lr<<16 | st<<22
  RowStat* qrs;      // [B][K][G] row states of the rows sb_draft_confidence streamed
                     // (read back by sb_verify_branches_reuse instead of the q rows)
  // adaptive single-launch step (k_astep): grab / queue counters, verify entries, sample queue
  int* actr;         // [8]
  int4* aqv;         // [B][K][G+1] verify entries (b, slot, i)
  int* aqv_pub;      // [B][K][G+1] entry published
  int* asq;          // [B] sample queue
  int* asq_pub;      // [B]
  size_t bytes;
};

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

inline Workspace carve(const sb_dims& d, void* base) {
  Workspace w{};
  const size_t B = (size_t)d.B, K = (size_t)d.K, R1 = (size_t)d.G + 1, G = (size_t)d.G;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return (char*)base + o;
  };
  w.info = (SeqInfo*)take(sizeof(SeqInfo) * B);
  w.unit_off = (int*)take(sizeof(int) * (B + 1));
  w.cnt = (int*)take(sizeof(int) * B);
  w.sel_cnt = (int*)take(sizeof(int) * 4);
  w.rowstat = (float4*)take(sizeof(float4) * B * K * R1);
  w.pflag = (uint8_t*)take(B * K * R1);
  w.conf_cnt = (int*)take(sizeof(int) * B * K);
  w.conf_stat = (float*)take(sizeof(float) * B * K * (G ? G : 1));
  w.conf_c = (float*)take(sizeof(float) * B * K * (G ? G : 1));
  {  // vocabulary-shard state (sb_shard_* calls / a communicator)
    const size_t nseg = ((size_t)d.V * (d.dtype == SB_BF16 ? 2 : 4) + 511) / 512;
    w.tok_lp = (float*)take(sizeof(float) * B * K * R1);
    w.segs = (float*)take(sizeof(float) * B * 2 * nseg);
    w.dec = (int4*)take(sizeof(int4) * B * 2);
  }
  w.ready = (int*)take(sizeof(int) * B);
  w.plan = (int*)take(sizeof(int) * 4);
  w.seqpk = (int*)take(sizeof(int) * B);
  w.qrs = (RowStat*)take(sizeof(RowStat) * B * K * (G ? G : 1));
  w.actr = (int*)take(sizeof(int) * 8);
  w.aqv = (int4*)take(sizeof(int4) * B * K * R1);
  w.aqv_pub = (int*)take(sizeof(int) * B * K * R1);
  w.asq = (int*)take(sizeof(int) * B);
  w.asq_pub = (int*)take(sizeof(int) * B);
  w.bytes = off;
  return w;
}

inline bool dims_valid(const sb_dims* d) {
  if (!d) return false;
  if (d->B < 1 || d->K < 1 || d->K > kMaxK || d->G < 0 || d->G > kMaxG || d->V < 2) return false;
  if (d->row_stride < d->V) return false;
  if (d->dtype != SB_BF16 && d->dtype != SB_F32) return false;
  if (d->v_offset < 0 || (d->v_total != 0 && (d->v_total < d->V || d->v_offset + d->V > d->v_total)))
    return false;
  if (d->reserved != 0) return false;
  const int64_t min_ss = (int64_t)d->K * (d->G + 1) * d->row_stride;
  if (d->seq_stride != 0 && d->seq_stride < min_ss) return false;
  return true;
}

inline bool sharded(const sb_dims* d) { return d->v_total != 0 && d->v_total != d->V; }

inline Dims to_dims(const sb_dims* d) {
  Dims x;
  x.B = d->B; x.K = d->K; x.G = d->G; x.V = d->V;
  x.rs = d->row_stride;
  x.ss = d->seq_stride ? d->seq_stride : (int64_t)d->K * (d->G + 1) * d->row_stride;
  x.dtype = d->dtype;
  return x;
}

inline size_t elem_size(const sb_dims* d) { return d->dtype == SB_BF16 ? 2 : 4; }

// 16-byte vector loads are legal for every row iff the base pointer and both strides
// keep 16-byte alignment.
inline bool vec_ok(const sb_dims* d, const void* p) {
  const size_t es = elem_size(d);
  const Dims x = to_dims(d);
  return ((uintptr_t)p % 16 == 0) && ((size_t)x.rs * es % 16 == 0) && ((size_t)x.ss * es % 16 == 0);
}

inline sb_status cuda_status(cudaError_t e) { return e == cudaSuccess ? SB_OK : SB_ERR_CUDA; }

// Programmatic dependent launch: the grid may be scheduled while its predecessor in the
// stream drains (launch latency and prologue overlap the predecessor's tail).  Every
// kernel launched this way calls pdl_wait() before its first global-memory access, so
// stream order is preserved for data; without the attribute pdl_wait() is a no-op.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at.val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

int num_sms();        // cudaDevAttrMultiProcessorCount of the current device
bool tma_disabled();  // SB_DISABLE_TMA=1 forces the register-staged kernels (tests)
int current_device();

// Dynamic shared memory opt-in of kernel K on the current device.  Function attributes
// are per device, so the "done" record is a per-kernel bitmask of devices (atomic: the
// entry points are callable from several host threads); a race only repeats the call.
template <auto K>
inline cudaError_t ensure_smem(int bytes) {
  static std::atomic<uint64_t> done{0};
  const uint64_t bit = 1ull << (current_device() & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
  return e;
}

// Resident CTAs per SM x SMs for a static-smem kernel on the current device.
template <auto K>
inline int full_grid(int threads) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, K, threads, 0);
  return (occ > 0 ? occ : 1) * num_sms();
}

}  // namespace sb
