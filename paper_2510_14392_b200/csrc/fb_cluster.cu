// fb_cluster.cu -- run_cluster on the device (fb_cluster.cuh) and the pure
// scheduler surface (form_batch / init_time_budget / pab over task sets);
// one full warp per node / task set (kTile = 32).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#define FB_TILE 32
#include "fb_engine_dev.cuh"
#include "fb_cluster.cuh"

namespace fbgpu {

size_t cluster_param_bytes() { return sizeof(ClusterParams); }
int cluster_max_nodes() { return kClusterMaxNodes; }
int cluster_max_ranks() { return kClusterMaxRanks; }
size_t cluster_xchg_bytes(int n_nodes) {
  return kXchgHeader + 2 * sizeof(NodeReport) * static_cast<size_t>(n_nodes);
}

int cluster_warps_per_cta(int n_nodes, int n_ranks) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms < 1) sms = 148;
  const int max_local = (n_nodes + n_ranks - 1) / n_ranks;
  // Full CTAs of kClusterMaxWarps nodes: the per-epoch exchange barrier
  // then has few participants (C5, 64 nodes: 8 CTAs 208 ms vs 64 CTAs of
  // one node 227 ms); more nodes than SMs x 8 still spread over every SM.
  int w = (max_local + sms - 1) / sms;
  if (w < kClusterMaxWarps) w = max_local < kClusterMaxWarps ? max_local : kClusterMaxWarps;
  if (w > kClusterMaxWarps) w = kClusterMaxWarps;
  (void)sms;
  return w < 1 ? 1 : w;
}

size_t cluster_smem_bytes(int warps_per_cta) {
  return ((sizeof(RouterSmem) + 15) / 16) * 16 +
         static_cast<size_t>(warps_per_cta) * kSmemSlots * kScratchBytesPerSlot;
}

// The cluster kernel for a CTA density (fb_cluster_shard_allow_hw_cluster):
// 2 = two CTAs per SM, otherwise one.
static const void* cluster_kernel_for(int ctas_per_sm) {
  return ctas_per_sm == 2 ? reinterpret_cast<const void*>(cluster_kernel<2>)
                          : reinterpret_cast<const void*>(cluster_kernel<1>);
}

int cluster_max_hw_clusters(int n_nodes, int ctas_per_sm) {
  const int wpc = cluster_warps_per_cta(n_nodes, 1);
  const int blocks = (n_nodes + wpc - 1) / wpc;
  if (blocks > 8) return 0;
  const size_t smem = cluster_smem_bytes(wpc);
  const void* k = cluster_kernel_for(ctas_per_sm);
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(kWarp * wpc);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = blocks;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

cudaError_t launch_cluster(const EngineParams& p, const ClusterParamsHost& ch, int blocks,
                           cudaStream_t st, int hw_mode) {
  static_assert(sizeof(ClusterParamsHost) == sizeof(ClusterParams), "cluster params layout");
  ClusterParams c;
  std::memcpy(&c, &ch, sizeof(c));
  if (c.warps_per_cta < 1 || c.warps_per_cta > kClusterMaxWarps) return cudaErrorInvalidValue;
  const size_t smem = cluster_smem_bytes(c.warps_per_cta);
  EngineParams pp = p;
  // One rank with at most kHwClusterMax CTAs: launch the grid as ONE
  // thread-block cluster (co-scheduled on one GPC by construction) and use
  // the hardware cluster barrier per epoch.  Otherwise a cooperative launch
  // (every CTA co-resident) with the global-memory exchange barrier.
  constexpr int kHwClusterMax = 8;  // portable cluster size
  if (hw_mode > 0 && c.n_ranks == 1 && blocks <= kHwClusterMax && !std::getenv("FB_NO_HW_CLUSTER")) {
    const void* k = cluster_kernel_for(hw_mode);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    c.hw_cluster = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(kWarp * c.warps_per_cta);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = blocks;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = hw_mode == 2 ? cudaLaunchKernelEx(&cfg, cluster_kernel<2>, pp, c)
                     : cudaLaunchKernelEx(&cfg, cluster_kernel<1>, pp, c);
    if (e == cudaSuccess) return e;
    cudaGetLastError();  // not schedulable as one cluster: fall back
    c.hw_cluster = 0;
  }
  cudaError_t e = cudaFuncSetAttribute(cluster_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  void* args[] = {&pp, &c};
  // cooperative: every CTA must be co-resident for the epoch barrier
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cluster_kernel<1>), dim3(blocks),
                                     dim3(kWarp * c.warps_per_cta), args, smem, st);
}

size_t cluster_serial_smem_bytes() {
  return ((sizeof(SerialSmem) + 15) / 16) * 16 + static_cast<size_t>(kSmemSlots) * kScratchBytesPerSlot;
}

// retry_reroute: the literal global loop on one warp (fb_cluster.cuh).
cudaError_t launch_cluster_serial(const EngineParams& p, const ClusterParamsHost& ch,
                                  cudaStream_t st) {
  ClusterParams c;
  std::memcpy(&c, &ch, sizeof(c));
  if (c.n_ranks != 1 || c.fifo_cap < 1 || !c.fifo || !c.row_state) return cudaErrorInvalidValue;
  const size_t smem = cluster_serial_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(cluster_serial_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  cluster_serial_kernel<<<1, kWarp, smem, st>>>(p, c);
  return cudaGetLastError();
}

cudaError_t launch_nodes(const EngineParams& p, const ClusterParamsHost& ch, const NodesIoHost& ih,
                         cudaStream_t st) {
  static_assert(sizeof(NodesIoHost) == sizeof(NodesIo), "node-set io layout");
  ClusterParams c;
  std::memcpy(&c, &ch, sizeof(c));
  NodesIo io;
  std::memcpy(&io, &ih, sizeof(io));
  const size_t smem = static_cast<size_t>(kClusterMaxWarps) * kSmemSlots * kScratchBytesPerSlot;
  cudaError_t e = cudaFuncSetAttribute(nodes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int blocks = (c.n_local + kClusterMaxWarps - 1) / kClusterMaxWarps;
  if (blocks > 0) nodes_kernel<<<blocks, kWarp * kClusterMaxWarps, smem, st>>>(p, c, io);
  return cudaGetLastError();
}

cudaError_t launch_nodes_enqueue(const EngineParams& p, const ClusterParamsHost& ch, int64_t t,
                                 const int32_t* node, const int64_t* row, int64_t n,
                                 int32_t* status, cudaStream_t st) {
  ClusterParams c;
  std::memcpy(&c, &ch, sizeof(c));
  nodes_enqueue_kernel<<<1, 32, 0, st>>>(p, c, t, node, row, n, status);
  return cudaGetLastError();
}

#ifdef FB_CLUSTER_PROF
#ifdef FB_CLUSTER_NODE_PROF
extern "C" int fb_debug_node_prof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_node_prof, sizeof(unsigned long long) * 512 * 8);
  static unsigned long long z[512 * 8] = {};
  cudaMemcpyToSymbol(g_node_prof, z, sizeof(z));
  return static_cast<int>(cudaDeviceSynchronize());
}
#endif
extern "C" int fb_debug_cluster_prof(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_cluster_prof, sizeof(unsigned long long) * 8);
  unsigned long long z[8] = {};
  cudaMemcpyToSymbol(g_cluster_prof, z, sizeof(z));
  return static_cast<int>(cudaDeviceSynchronize());
}
extern "C" int fb_debug_epoch_max(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_epoch_max, sizeof(unsigned long long) * 16384);
  cudaMemcpyFromSymbol(out + 16384, g_epoch_max_c, sizeof(unsigned long long) * 16384);
  static unsigned long long z[16384];
  cudaMemcpyToSymbol(g_epoch_max, z, sizeof(z));
  cudaMemcpyToSymbol(g_epoch_max_c, z, sizeof(z));
  return static_cast<int>(cudaDeviceSynchronize());
}
#endif

// ------------------------------------------------- pure scheduler kernels

__device__ __forceinline__ Scratch set_scratch(unsigned char* smem_warp, unsigned char* g,
                                               int64_t off, int64_t n) {
  if (n <= kSmemSlots) return carve_scratch(smem_warp, kSmemSlots);
  return carve_scratch(g + off * kScratchBytesPerSlot, static_cast<int>(n));
}

// form_batch (sched.cpp:234-246) per task set, one warp per set.
__global__ void __launch_bounds__(kWarp * kWarpsPerBlock)
form_batch_kernel(const fb_task_view* __restrict__ tasks, const int64_t* __restrict__ set_off,
                  const fb_scheduler_config* __restrict__ cfgs, int64_t n_sets,
                  fb_plan_entry_id* __restrict__ entries, fb_batch_plan* __restrict__ plans,
                  unsigned char* gscratch, int* status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x / kWarp;
  unsigned char* my = smem + static_cast<size_t>(warp) * kSmemSlots * kScratchBytesPerSlot;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarpsPerBlock;
  for (int64_t set = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + warp; set < n_sets;
       set += nwarps) {
    const int64_t off = set_off[set];
    const int64_t n = set_off[set + 1] - off;
    const fb_scheduler_config cfg = cfgs[set];
    const bool fair = cfg.policy == FB_POLICY_FAIRBATCH || cfg.policy == FB_POLICY_FAIRBATCH_PAB;
    if (n == 0) {
      if (lane_id() == 0) {
        if (fair) atomicExch(status, FB_ERR_USAGE);  // init_time_budget on empty
        fb_batch_plan pl = {};
        pl.entry_off = off;
        plans[set] = pl;
      }
      continue;
    }
    const Scratch s = set_scratch(my, gscratch, off, n);
    ViewAcc acc;
    bool unusual = false;
    for (int64_t p = lane_id(); p < n; p += kWarp) {
      const fb_task_view t = tasks[off + p];
      const bool decode = t.phase == FB_PHASE_DECODE;
      s.slack[p] = t.slack_us;
      s.seq[p] = t.arrival_seq;
      s.ctx[p] = t.context;
      s.nw[p] = t.new_tokens | (decode ? static_cast<int32_t>(kDecodeBit) : 0);
      s.req[p] = static_cast<int32_t>(p);
      acc.add(decode, t.slack_us, t.tpot_us);
      unusual |= t.new_tokens == 0 || t.context < 0;
    }
    __syncwarp();
    acc.reduce();
    // consider's early exit is proven only for new >= 1 and c*ctx >= 0
    const bool exits_ok = !__any_sync(kFull, unusual) && cfg.model.c_ms >= 0.0;
    FormCfg f;
    f.policy = cfg.policy;
    f.max_chunk = cfg.max_chunk;
    f.token_budget = cfg.token_budget;
    f.a = cfg.model.a_ms;
    f.b = cfg.model.b_ms;
    f.c = cfg.model.c_ms;
    const int Ai = static_cast<int>(n);
    const FormOut o = form_batch_warp<true>(s, Ai, acc, f, /*seq_unique=*/false, exits_ok);
    int run = 0;
    for (int k0 = 0; k0 < Ai; k0 += kWarp) {
      const int k = k0 + lane_id();
      int tk = 0, p = 0;
      if (k < Ai) {
        p = s.order[k];
        tk = s.take[k];
      }
      const bool adm = k < Ai && admitted_take<true>(tk);
      const unsigned m = __ballot_sync(kFull, adm);
      if (adm) {
        fb_plan_entry_id e;
        e.request_id = tasks[off + p].request_id;
        e.new_tokens = tk;
        e.reserved = 0;
        entries[off + run + __popc(m & lanemask_lt())] = e;
      }
      run += __popc(m);
    }
    if (lane_id() == 0) {
      fb_batch_plan pl;
      const bool empty = o.n_entries == 0;
      pl.predicted_ms = o.predicted_ms;
      pl.time_budget_used_ms = empty ? 0.0 : o.predicted_ms;
      pl.token_budget_used = empty ? 0 : o.total_new;
      pl.init_time_budget_ms = o.init_ms;
      pl.entry_off = off;
      pl.n_entries = o.n_entries;
      plans[set] = pl;
    }
    __syncwarp();
  }
}

__global__ void init_time_budget_kernel(const fb_task_view* __restrict__ tasks,
                                        const int64_t* __restrict__ set_off, int64_t n_sets,
                                        int64_t* out, int* status) {
  const int warp = threadIdx.x / kWarp;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x / kWarp);
  for (int64_t set = static_cast<int64_t>(blockIdx.x) * (blockDim.x / kWarp) + warp;
       set < n_sets; set += nwarps) {
    const int64_t off = set_off[set];
    const int64_t n = set_off[set + 1] - off;
    ViewAcc acc;
    for (int64_t p = lane_id(); p < n; p += kWarp) {
      const fb_task_view t = tasks[off + p];
      acc.add(t.phase == FB_PHASE_DECODE, t.slack_us, t.tpot_us);
    }
    acc.reduce();
    if (lane_id() == 0) {
      if (n == 0) {
        atomicExch(status, FB_ERR_USAGE);
        out[set] = 0;
      } else {
        out[set] = acc.n_dec == 0 ? acc.min_tpot
                                  : (acc.min_dec > acc.min_tpot ? acc.min_dec : acc.min_tpot);
      }
    }
  }
}

// K5 standalone: pab (sched.cpp:248-278) per task set.
__global__ void __launch_bounds__(kWarp * kWarpsPerBlock)
pab_kernel(const fb_task_view* __restrict__ tasks, const int64_t* __restrict__ set_off,
           const fb_cost_model* __restrict__ models, const int64_t* __restrict__ ttft,
           const int64_t* __restrict__ tpot, int64_t n_sets, int64_t* out,
           unsigned char* gscratch) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x / kWarp;
  unsigned char* my = smem + static_cast<size_t>(warp) * kSmemSlots * kScratchBytesPerSlot;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kWarpsPerBlock;
  for (int64_t set = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + warp; set < n_sets;
       set += nwarps) {
    const int64_t off = set_off[set];
    const int64_t n = set_off[set + 1] - off;
    const fb_cost_model m = models[set];
    const double Wm = us_to_ms(ttft[set]), Tm = us_to_ms(tpot[set]);
    const Scratch s = set_scratch(my, gscratch, off, n);
    int64_t lmin = kInf, lpf = 0;
    for (int64_t p = lane_id(); p < n; p += kWarp) {
      const fb_task_view t = tasks[off + p];
      s.tcost[p] = pab_term(Wm, Tm, m.b_ms, m.c_ms, t.slack_us, t.context);
      lmin = t.slack_us < lmin ? t.slack_us : lmin;
      if (t.phase == FB_PHASE_PREFILL) lpf += t.new_tokens;
    }
    __syncwarp();
    const int64_t min_slack = warp_min(lmin);
    const int64_t pf = warp_sum(lpf);
    const double r_tasks = ordered_fold(s.tcost, static_cast<int>(n));
    if (lane_id() == 0)
      out[set] = pab_close(Wm, Tm, m.a_ms, m.b_ms, m.c_ms, n > 0, min_slack, r_tasks, pf);
    __syncwarp();
  }
}

static int set_blocks(int64_t n_sets) {
  int64_t b = (n_sets + kWarpsPerBlock - 1) / kWarpsPerBlock;
  if (b < 1) b = 1;
  if (b > 148 * 8) b = 148 * 8;
  return static_cast<int>(b);
}

cudaError_t launch_form_batch(const fb_task_view* tasks, const int64_t* set_off,
                              const fb_scheduler_config* cfgs, int64_t n_sets,
                              fb_plan_entry_id* entries, fb_batch_plan* plans,
                              unsigned char* scratch, int* status, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(kWarpsPerBlock) * kSmemSlots * kScratchBytesPerSlot;
  cudaFuncSetAttribute(form_batch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  form_batch_kernel<<<set_blocks(n_sets), kWarp * kWarpsPerBlock, smem, st>>>(
      tasks, set_off, cfgs, n_sets, entries, plans, scratch, status);
  return cudaGetLastError();
}

cudaError_t launch_init_time_budget(const fb_task_view* tasks, const int64_t* set_off,
                                    int64_t n_sets, int64_t* out, int* status,
                                    cudaStream_t st) {
  init_time_budget_kernel<<<set_blocks(n_sets), kWarp * kWarpsPerBlock, 0, st>>>(
      tasks, set_off, n_sets, out, status);
  return cudaGetLastError();
}

cudaError_t launch_pab(const fb_task_view* tasks, const int64_t* set_off,
                       const fb_cost_model* models, const int64_t* ttft, const int64_t* tpot,
                       int64_t n_sets, int64_t* out, unsigned char* scratch, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(kWarpsPerBlock) * kSmemSlots * kScratchBytesPerSlot;
  cudaFuncSetAttribute(pab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  pab_kernel<<<set_blocks(n_sets), kWarp * kWarpsPerBlock, smem, st>>>(
      tasks, set_off, models, ttft, tpot, n_sets, out, scratch);
  return cudaGetLastError();
}

}  // namespace fbgpu
