// ep.cu -- expert parallelism (moe_layer.cpp:85-91, 124-128; collectives.cpp:69-265).
//
// Rank r owns experts g in [r*el, (r+1)*el) (moe_layer.hpp:29-30).  The send
// plan covers all E experts in the reference layout (grouped by destination
// rank, then its local expert, then scatter order); the receive layout is
// (local expert, source rank, source order) with aligned expert blocks.  The
// forward's plan is reused by the backward without a recount
// (collectives.hpp:48-50).  Two ways to move the rows:
//
//   fused (bf16, peers mapped -- peer.cuh): gate -> plan -> count all-gather
//     into every peer (C1) -> every rank's layout on the device (no host sync)
//     -> scatter straight into the expert ranks (C2) -> fc1 -> fc2 storing
//     each row straight home (C3) -> gather_combine; backward: gcb writing
//     d_ys into the expert ranks -> dgrad fc2 / fc1 storing d_xs home ->
//     weight gradients and gate d_wg while the peers finish -> scatter_backward.
//     Phases are ordered by epoch flags (or events inside one process).
//   transport (f64 / f32, fallback): scatter -> count exchange (C1) -> one
//     host sync -> grouped send/recv per (peer, local expert) chunk straight
//     into its final slot (C2) -> experts -> reverse exchange (C3) ->
//     gather_combine; backward on the same routes.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "comm.cuh"
#include "layer.cuh"
#include "ops.cuh"
#include "peer.cuh"
#include "plan.cuh"

namespace fmoe_b200 {

struct Layer::Ep {
  int W = 1, r = 0;
  int64_t el = 0, align = 1, cap_recv = 0;
  // receive-side block plan (device) + host mirrors
  fmoe_plan rplan{};
  int32_t* d_recv_counts = nullptr;  // [W*el] rows from source s for local expert e
  int32_t* h_pinned = nullptr;       // staging: send counts, recv counts, plan upload
  std::vector<int64_t> h_send, h_recv, send_off, chunk_off, block_off, rows;
  // receive-space activations
  void *xs = nullptr, *hidden = nullptr, *ys = nullptr, *d_ys = nullptr, *d_pre = nullptr, *d_xs = nullptr;
  bool planned = false;
  // fused exchange over NVLink peer memory (peer.cuh); bf16 only
  int exchange = FMOE_EP_EXCHANGE_PEER;  // or FMOE_EP_EXCHANGE_TRANSPORT
  PeerSet peer;
  bool peer_tried = false;
  int32_t* cnt_mat = nullptr;   // [W][E] all-gathered send counts (peer-written)
  uint32_t* flags = nullptr;    // [PH_N][W] epoch flags (peer-written)
  int32_t* g_rank = nullptr;    // [E] destination rank of global expert g
  int64_t* g_delta = nullptr;   // [E] row shift send layout -> destination receive layout
  int32_t* rt = nullptr;        // [3][el*W] chunk start / rows / destination row (RowRoute)
  uint8_t* h_peer = nullptr;    // pinned staging of the tables above
  void* peer_scratch = nullptr; // connect's blob exchange
  void** peer_table = nullptr;  // [PB_N][W] device pointer tables
  bool fused = false;           // the current step runs the fused path
  bool device_plan = false;     // its layouts were computed on the device
  // overlapped exchange (cross-process peers): the rows are pushed by a
  // concurrent kernel on `side` while fc1 / dgrad fc2 consume them tile by
  // tile as their chunks are published (per-chunk flags after the PH_N phase
  // flags in `flags`: [dir][el][W])
  bool overlap = false;         // the current step overlaps the exchange
  cudaStream_t side = nullptr;
  cudaEvent_t ev_go = nullptr, ev_pushed = nullptr;
  int32_t* push_ctr = nullptr;  // [1 + E]: work-unit counter, rows done per send segment
  int32_t* mtile_order = nullptr;
};

namespace {
void* alloc(std::vector<void*>& owned, int64_t bytes) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<int64_t>(bytes, 256)));
  owned.push_back(p);
  return p;
}
}  // namespace

void Layer::ep_alloc() {
  ep = new Ep;
  Ep& P = *ep;
  P.W = (int)cfg.world_size;
  P.r = (int)cfg.rank;
  P.el = cfg.n_e_local;
  // a rank's experts receive n_b*k rows on average (its own token count)
  P.align = t == FMOE_BF16 ? expert_block_align(cfg.n_b * cfg.k, P.el) : 1;
  // worst case: every token of every rank picks this rank's experts
  P.cap_recv = plan_capacity(cfg.n_b * cfg.world_size, cfg.k, P.el, P.align);
  const int64_t d = cfg.d_m, h = cfg.d_h, cap = P.cap_recv;
  P.rplan.n_b = 0;
  P.rplan.k = 1;
  P.rplan.n_experts = P.el;
  P.rplan.align = P.align;
  P.rplan.capacity = cap;
  P.rplan.counts = (int32_t*)alloc(owned, P.el * 4);
  P.rplan.offsets = (int32_t*)alloc(owned, (P.el + 1) * 4);
  P.rplan.tile_expert = (int32_t*)alloc(owned, (cap / 128 + 2) * 4);
  P.rplan.n_tiles = (int32_t*)alloc(owned, 4);
  P.d_recv_counts = (int32_t*)alloc(owned, P.W * P.el * 4);
  const int64_t staging = E + P.W * P.el + (P.el + 1) + P.el + cap / 128 + 8;
  CK(cudaMallocHost(&P.h_pinned, staging * 4));
  h_stage = P.h_pinned;
  P.xs = alloc(owned, cap * d * es);
  P.hidden = alloc(owned, cap * h * es);
  P.ys = alloc(owned, cap * d * es);
  P.d_ys = alloc(owned, cap * d * es);
  P.d_pre = alloc(owned, cap * h * es);
  P.d_xs = alloc(owned, cap * d * es);
  tpart = (float*)alloc(owned, experts_bwd_part_floats(P.rplan, d, h) * 4);
  if (t == FMOE_BF16) relu_bits = (uint32_t*)alloc(owned, cap * (h / 32) * 4);
  const int64_t W = P.W;
  P.cnt_mat = (int32_t*)alloc(owned, W * E * 4);
  P.flags = (uint32_t*)alloc(owned, (PH_N * W + 2 * P.el * W) * 4);
  CK(cudaMemset(P.flags, 0, (PH_N * W + 2 * P.el * W) * 4));
  P.push_ctr = (int32_t*)alloc(owned, (1 + E) * 4);
  P.mtile_order = (int32_t*)alloc(owned, (cap / 128 + 2) * 4);
  P.g_rank = (int32_t*)alloc(owned, E * 4);
  P.g_delta = (int64_t*)alloc(owned, E * 8);
  P.rt = (int32_t*)alloc(owned, 3 * P.el * W * 4);
  CK(cudaMallocHost(&P.h_peer, W * E * 4 + E * 12 + 3 * P.el * W * 4 + 64));
  P.peer_scratch = alloc(owned, (int64_t)PeerSet::scratch_bytes(P.W));
  P.peer_table = (void**)alloc(owned, PB_N * W * (int64_t)sizeof(void*));
}

namespace {

Transport* need_transport(Ctx* ctx, const fmoe_layer_config& cfg) {
  Transport* tr = ctx->transport;
  if (!tr)
    protocol_error("forward: expert-parallel layer (world " + std::to_string(cfg.world_size) +
                   ") needs a transport: fmoe_comm_init or fmoe_ctx_join_world");
  if (tr->world != cfg.world_size) protocol_error("forward: transport world != config world");
  if (tr->rank != cfg.rank) protocol_error("forward: transport rank != layer rank");
  return tr;
}

// Grouped exchange of row chunks between the send layout (per destination
// rank, per its local expert) and the receive layout (per local expert, per
// source rank).  forward: send -> recv (all_to_all_rows); reverse: recv ->
// send (all_to_all_rows_reverse).
void exchange_rows(Ctx* ctx, Transport* tr, const Layer::Ep& P, size_t rb, const void* src, void* dst,
                   bool forward) {
  const int W = P.W, r = P.r;
  const int64_t el = P.el;
  const uint8_t* s8 = static_cast<const uint8_t*>(src);
  uint8_t* d8 = static_cast<uint8_t*>(dst);
  std::vector<Xfer> sends, recvs;
  for (int p = 0; p < W; ++p) {
    for (int64_t e = 0; e < el; ++e) {
      const int64_t g = (int64_t)p * el + e;
      const size_t send_rows = (size_t)P.h_send[g];        // rows this rank routes to (p, e)
      const size_t recv_rows = (size_t)P.h_recv[g];        // rows rank p routes to my expert e
      const int64_t so = P.send_off[g];
      const int64_t ro = P.chunk_off[e * W + p];
      if (p == r) {  // self rows bypass the transport (collectives.cpp:160-171)
        if (send_rows != recv_rows) protocol_error("exchange: self counts disagree");
        if (!send_rows) continue;
        if (forward)
          CK(cudaMemcpyAsync(d8 + ro * rb, s8 + so * rb, send_rows * rb, cudaMemcpyDeviceToDevice, ctx->stream));
        else
          CK(cudaMemcpyAsync(d8 + so * rb, s8 + ro * rb, send_rows * rb, cudaMemcpyDeviceToDevice, ctx->stream));
        continue;
      }
      if (forward) {
        sends.push_back({p, const_cast<uint8_t*>(s8) + so * rb, send_rows * rb});
        recvs.push_back({p, d8 + ro * rb, recv_rows * rb});
      } else {
        sends.push_back({p, const_cast<uint8_t*>(s8) + ro * rb, recv_rows * rb});
        recvs.push_back({p, d8 + so * rb, send_rows * rb});
      }
    }
  }
  tr->group(ctx, sends, recvs);
}

void zero_pads(Ctx* ctx, const Layer::Ep& P, size_t rb, void* buf) {
  uint8_t* b = static_cast<uint8_t*>(buf);
  for (int64_t e = 0; e < P.el; ++e) {
    const int64_t a = P.block_off[e] + P.rows[e], z = P.block_off[e + 1];
    if (z > a) CK(cudaMemsetAsync(b + a * rb, 0, (size_t)(z - a) * rb, ctx->stream));
  }
}

}  // namespace

// Host layout of one exchange (pure host arithmetic, exported as
// fmoe_ep_layout so the multi-process CPU tests can drive it):
//   send_off[g]          first row of (dest rank g/el, its local expert g%el) in the
//                        send layout = exclusive prefix of send counts
//                        (send_section_offsets, collectives.cpp:114-122)
//   chunk_off[e*W + s]   first row of (local expert e, source s) in the receive
//                        layout (recv_chunk_offsets, collectives.cpp:126-135),
//                        expert blocks starting on `align`-row boundaries
//   block_off[e], rows[e] expert block start (el+1 entries) and valid rows.
void ep_layout(int W, int64_t el, int64_t align, const int64_t* send, const int64_t* recv,
               int64_t* send_off, int64_t* chunk_off, int64_t* block_off, int64_t* rows) {
  const int64_t E = (int64_t)W * el;
  if (E > 0) send_off[0] = 0;
  for (int64_t g = 1; g < E; ++g) send_off[g] = send_off[g - 1] + send[g - 1];
  int64_t at = 0;
  for (int64_t e = 0; e < el; ++e) {
    block_off[e] = at;
    int64_t c = at;
    for (int s = 0; s < W; ++s) {
      chunk_off[e * W + s] = c;
      c += recv[(int64_t)s * el + e];
    }
    rows[e] = c - at;
    at += (rows[e] + align - 1) / align * align;
  }
  block_off[el] = at;
}

// Every rank's layout from the all-gathered count matrix counts[s][g] (rows
// rank s routes to global expert g), as seen by rank r (pure host arithmetic,
// exported as fmoe_ep_routes for the CPU tests):
//   send_off/chunk_off/block_off/rows  rank r's own layouts (ep_layout)
//   g_rank[g], g_delta[g]   my send rows of expert g -> rank g/el's receive
//                           buffer at row (send position + g_delta[g])
//   route[c], route[C + c], route[2C + c]  (c = e*W + s, C = el*W): my receive
//                           chunk (local expert e, source s) -- first row, row
//                           count -- and its first row in s's send layout
void ep_routes(int W, int r, int64_t el, int64_t align, const int64_t* counts, int64_t* send_off,
               int64_t* chunk_off, int64_t* block_off, int64_t* rows, int32_t* g_rank, int64_t* g_delta,
               int32_t* route) {
  const int64_t E = (int64_t)W * el, C = el * W;
  std::vector<std::vector<int64_t>> so(W), co(W);
  std::vector<int64_t> rcv(E), blk(el + 1), rw(el);
  for (int p = 0; p < W; ++p) {
    for (int s = 0; s < W; ++s)
      for (int64_t e = 0; e < el; ++e) rcv[s * el + e] = counts[(int64_t)s * E + p * el + e];
    so[p].assign(E, 0);
    co[p].assign(C, 0);
    ep_layout(W, el, align, counts + (int64_t)p * E, rcv.data(), so[p].data(), co[p].data(), blk.data(),
              rw.data());
    if (p == r) {
      std::copy(so[p].begin(), so[p].end(), send_off);
      std::copy(co[p].begin(), co[p].end(), chunk_off);
      std::copy(blk.begin(), blk.end(), block_off);
      std::copy(rw.begin(), rw.end(), rows);
    }
  }
  for (int64_t g = 0; g < E; ++g) {
    const int p = (int)(g / el);
    g_rank[g] = p;
    g_delta[g] = co[p][(g % el) * W + r] - so[r][g];
  }
  for (int64_t e = 0; e < el; ++e)
    for (int s = 0; s < W; ++s) {
      const int64_t c = e * W + s;
      route[c] = (int32_t)co[r][c];
      route[C + c] = (int32_t)counts[(int64_t)s * E + r * el + e];
      route[2 * C + c] = (int32_t)so[s][r * el + e];
    }
}

// exchange_counts (collectives.cpp:69-109) + the receive layout
// (recv_chunk_offsets, collectives.cpp:126-135) with aligned expert blocks.
static void ep_plan(Layer& L, Transport* tr) {
  Ctx* ctx = L.ctx;
  Layer::Ep& P = *L.ep;
  const int W = P.W, r = P.r;
  const int64_t el = P.el, E = L.E;
  std::vector<Xfer> sends, recvs;
  for (int p = 0; p < W; ++p) {
    if (p == r) continue;
    sends.push_back({p, L.plan.counts + p * el, (size_t)el * 4});
    recvs.push_back({p, P.d_recv_counts + p * el, (size_t)el * 4});
  }
  CK(cudaMemcpyAsync(P.d_recv_counts + r * el, L.plan.counts + r * el, el * 4, cudaMemcpyDeviceToDevice,
                     ctx->stream));
  tr->group(ctx, sends, recvs);
  int32_t* hs = P.h_pinned;
  int32_t* hr = hs + E;
  CK(cudaMemcpyAsync(hs, L.plan.counts, E * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(hr, P.d_recv_counts, W * el * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // the one host sync of an EP step
  P.h_send.assign(hs, hs + E);
  P.h_recv.assign(hr, hr + W * el);
  P.send_off.assign(E, 0);
  P.rows.assign(el, 0);
  P.block_off.assign(el + 1, 0);
  P.chunk_off.assign(el * W, 0);
  ep_layout(W, el, P.align, P.h_send.data(), P.h_recv.data(), P.send_off.data(), P.chunk_off.data(),
            P.block_off.data(), P.rows.data());
  const int64_t at = P.block_off[el];
  if (at > P.cap_recv) protocol_error("exchange: received rows exceed the layer capacity");
  // upload the receive block plan (counts, offsets, 128-row tile table)
  int32_t* up = hr + W * el;
  for (int64_t e = 0; e < el; ++e) up[e] = (int32_t)P.rows[e];
  int32_t* uo = up + el;
  for (int64_t e = 0; e <= el; ++e) uo[e] = (int32_t)P.block_off[e];
  int32_t* ut = uo + el + 1;
  int64_t nt = 0;
  if (P.align % 128 == 0) {
    for (int64_t e = 0; e < el; ++e)
      for (int64_t tt = P.block_off[e] / 128; tt < P.block_off[e + 1] / 128; ++tt) ut[nt++] = (int32_t)e;
  }
  ut[nt] = (int32_t)nt;  // n_tiles rides at the end
  CK(cudaMemcpyAsync(P.rplan.counts, up, el * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(P.rplan.offsets, uo, (el + 1) * 4, cudaMemcpyHostToDevice, ctx->stream));
  if (nt) CK(cudaMemcpyAsync(P.rplan.tile_expert, ut, nt * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(P.rplan.n_tiles, ut + nt, 4, cudaMemcpyHostToDevice, ctx->stream));
  P.planned = true;
}

// ------------------------------------------------ fused exchange (peer memory)
// Connect the peer buffers on the first bf16 EP step (collective: every rank
// runs its first forward together).  Ranks that cannot map each other (no
// NVLink P2P / different hosts) all keep the transport exchange.
static bool ep_use_peer(Layer& L, Transport* tr) {
  Layer::Ep& P = *L.ep;
  if (L.t != FMOE_BF16 || P.exchange != FMOE_EP_EXCHANGE_PEER) return false;
  if (!P.peer_tried && tr) {
    P.peer_tried = true;
    void* bufs[PB_N] = {P.xs, P.d_ys, L.ys, L.d_xs, P.cnt_mat, P.flags};
    P.peer.connect(L.ctx, tr, bufs, P.peer_scratch, P.peer_table);
  }
  return P.peer.ok;
}

// Device-side layouts for the fused path (the host arithmetic of
// ep_routes + the receive block plan of ep_plan, on the GPU): one block
// reads the all-gathered count matrix and writes the scatter routes, the
// epilogue routes and the receive plan (counts, offsets, 128-row tile table),
// so an expert-parallel step needs no host synchronisation at all.
__global__ void ep_layout_kernel(const int32_t* __restrict__ cnt, int W, int el, int align, int r,
                                 int32_t* __restrict__ g_rank, int64_t* __restrict__ g_delta,
                                 int32_t* __restrict__ rt, int32_t* __restrict__ rcounts,
                                 int32_t* __restrict__ roffsets, int32_t* __restrict__ tile_expert,
                                 int32_t* __restrict__ n_tiles) {
  extern __shared__ int32_t sm[];
  const int E = W * el, C = el * W;
  int32_t* send_off = sm;          // [W][E]
  int32_t* chunk = sm + W * E;     // [W][el*W]: chunk_off of every rank p
  int32_t* boff = chunk + W * C;   // [el+1]: my block offsets
  for (int s = threadIdx.x; s < W; s += blockDim.x) {  // send_section_offsets, collectives.cpp:114-122
    int acc = 0;
    for (int g = 0; g < E; ++g) {
      send_off[s * E + g] = acc;
      acc += cnt[s * E + g];
    }
  }
  for (int p = threadIdx.x; p < W; p += blockDim.x) {  // recv_chunk_offsets, collectives.cpp:126-135
    int at = 0;
    for (int e = 0; e < el; ++e) {
      int c = at;
      for (int s = 0; s < W; ++s) {
        chunk[p * C + e * W + s] = c;
        c += cnt[s * E + p * el + e];
      }
      const int rows = c - at;
      if (p == r) {
        rcounts[e] = rows;
        boff[e] = at;
      }
      at += (rows + align - 1) / align * align;
    }
    if (p == r) boff[el] = at;
  }
  __syncthreads();
  for (int g = threadIdx.x; g < E; g += blockDim.x) {
    const int p = g / el, e = g % el;
    g_rank[g] = p;
    g_delta[g] = (int64_t)chunk[p * C + e * W + r] - send_off[r * E + g];
  }
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const int e = c / W, s = c % W;
    rt[c] = chunk[r * C + c];
    rt[C + c] = cnt[s * E + r * el + e];
    rt[2 * C + c] = send_off[s * E + r * el + e];
  }
  for (int e = threadIdx.x; e <= el; e += blockDim.x) roffsets[e] = boff[e];
  for (int e = 0; e < el; ++e)
    for (int t = boff[e] / 128 + threadIdx.x; t < boff[e + 1] / 128; t += blockDim.x) tile_expert[t] = e;
  if (threadIdx.x == 0) *n_tiles = boff[el] / 128;
}

// Zero the pad rows of every expert block of the receive layout (device
// offsets / counts): block e, one warp per row, 16-byte stores.
__global__ void ep_zero_pads_kernel(uint8_t* __restrict__ buf, int64_t row_bytes, const int32_t* __restrict__ offsets,
                                    const int32_t* __restrict__ counts) {
  const int e = blockIdx.x;
  const int64_t a = (int64_t)offsets[e] + counts[e], z = offsets[e + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t row = a + warp; row < z; row += blockDim.x >> 5) {
    uint4* d = reinterpret_cast<uint4*>(buf + row * row_bytes);
    for (int64_t c = lane; c < (row_bytes >> 4); c += 32) d[c] = make_uint4(0, 0, 0, 0);
  }
}

// Row tiles of the receive layout in the order their rows are expected to
// land under the overlapped exchange: sender s pushes to destinations s, s+1,
// ... (mod W) and, per destination, its experts in order, so chunk (e, s)
// reaches this rank r in slot q = (r - s) mod W (q = 0: this rank's own rows).
// A tile's key is the latest (q, e) among the chunks it covers; tiles are
// dealt in increasing key (counting sort; order inside a key is arbitrary --
// it only changes which CTA computes a tile, never its value).
__global__ void ep_tile_order_kernel(const int32_t* __restrict__ rt, const int32_t* __restrict__ tile_expert,
                                     const int32_t* __restrict__ n_tiles, int W, int el, int r, int cg,
                                     int32_t* __restrict__ order) {
  extern __shared__ int32_t cnt[];  // [W*el] counts, then cursors
  const int K = W * el, C = el * W;
  const int nt = *n_tiles / cg;
  for (int i = threadIdx.x; i < K; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  auto key_of = [&](int t) {
    const int e = tile_expert[t * cg];
    const int r0 = t * 128 * cg, r1 = r0 + 128 * cg;
    int key = 0;
    for (int s = 0; s < W; ++s) {
      const int st = rt[e * W + s], nr = rt[C + e * W + s];
      if (nr > 0 && st < r1 && st + nr > r0) key = max(key, ((r - s + W) % W) * el + e);
    }
    return key;
  };
  for (int t = threadIdx.x; t < nt; t += blockDim.x) atomicAdd(&cnt[key_of(t)], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int i = 0; i < K; ++i) {
      const int c = cnt[i];
      cnt[i] = acc;
      acc += c;
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nt; t += blockDim.x) order[atomicAdd(&cnt[key_of(t)], 1)] = t;
}

__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// The overlapped global scatter: this rank's send rows, destination-major (the
// send layout is grouped by destination rank, then its local expert,
// collectives.cpp:114-122), pushed into every rank's receive buffer in the
// rotated order s, s+1, ... so each destination hears from one sender at a
// time.  Work units of kUnit rows are taken in that order from an atomic
// counter; when the last unit of send segment g (destination p, its expert e)
// is stored, the CTA that completed it publishes flag [e][r] in p's memory
// (fence + release store after the block barrier, the grid-sync pattern).
// SCALE (backward): d_ys = bf16(w * d_y), the same rounding as gcb_kernel.
constexpr int kPushUnit = 128;
constexpr int kPushThreads = 512;
template <bool SCALE>
__global__ void __launch_bounds__(kPushThreads) ep_push_kernel(
    const __nv_bfloat16* __restrict__ src, int64_t d, fmoe_plan p, const float* __restrict__ w,
    void* const* dst, const int64_t* __restrict__ g_delta, void* const* flags, int flag_base, int W, int r, int el,
    uint32_t epoch, int32_t* __restrict__ ctr) {
  extern __shared__ int32_t sh[];  // [E+1] unit prefix in rotated segment order, + broadcast slot
  const int E = W * el;
  int32_t* pref = sh;
  int32_t* slot = sh + E + 1;
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int q = 0; q < E; ++q) {
      const int g = ((r + q / el) % W) * el + q % el;
      pref[q] = acc;
      acc += (p.offsets[g + 1] - p.offsets[g] + kPushUnit - 1) / kPushUnit;
    }
    pref[E] = acc;
  }
  __syncthreads();
  const int total = pref[E];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n16 = d / 8;  // 16-byte vectors per row
  while (true) {
    if (threadIdx.x == 0) *slot = atomicAdd(ctr, 1);
    __syncthreads();
    const int u = *slot;
    __syncthreads();
    if (u >= total) break;
    int lo = 0, hi = E;  // segment q with pref[q] <= u < pref[q+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pref[mid] <= u) lo = mid; else hi = mid;
    }
    const int q = lo;
    const int dp = (r + q / el) % W, e = q % el, g = dp * el + e;
    const int seg0 = p.offsets[g], seg1 = p.offsets[g + 1];
    const int a = seg0 + (u - pref[q]) * kPushUnit, b = min(seg1, a + kPushUnit);
    uint8_t* out = static_cast<uint8_t*>(dst[dp]);
    const int64_t delta = g_delta[g];
    for (int pos = a + warp; pos < b; pos += kPushThreads / 32) {
      const int i = __ldg(p.src_row + pos);
      const uint4* s4 = reinterpret_cast<const uint4*>(src + (int64_t)i * d);
      uint4* d4 = reinterpret_cast<uint4*>(out + (pos + delta) * d * 2);
      float wv = 1.f;
      if constexpr (SCALE) wv = __ldg(w + (int64_t)i * p.k + __ldg(p.slot + pos));
      for (int64_t c = lane; c < n16; c += 32 * 4) {
        uint4 v[4];
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (c + 32 * t < n16) v[t] = __ldg(s4 + c + 32 * t);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (c + 32 * t >= n16) break;
          if constexpr (SCALE) {
            __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(&v[t]);
#pragma unroll
            for (int z = 0; z < 8; ++z) h[z] = __float2bfloat16_rn(wv * __bfloat162float(h[z]));
          }
          d4[c + 32 * t] = v[t];
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      const int n = b - a;
      if (atomicAdd(ctr + 1 + g, n) + n == seg1 - seg0) {
        __threadfence_system();
        st_release_sys_u32(static_cast<uint32_t*>(flags[dp]) + flag_base + e * W + r, epoch);
      }
    }
  }
}

static size_t ep_layout_smem(int W, int64_t el) {
  const int64_t E = W * el;
  return (size_t)(W * E + W * el * W + el + 1) * 4;
}

// Fused-path plan with no host synchronisation: counts all-gathered over
// peer memory, every layout computed on the device.
static void ep_plan_peer_device(Layer& L) {
  Ctx* ctx = L.ctx;
  Layer::Ep& P = *L.ep;
  const int W = P.W;
  const int64_t el = P.el, E = L.E, C = el * W;
  P.peer.put_counts(ctx, L.plan.counts, E);
  P.peer.wait(ctx, PH_COUNTS);
  ep_layout_kernel<<<1, 256, ep_layout_smem(W, el), ctx->stream>>>(
      P.cnt_mat, W, (int)el, (int)P.align, P.r, P.g_rank, P.g_delta, P.rt, P.rplan.counts, P.rplan.offsets,
      P.rplan.tile_expert, P.rplan.n_tiles);
  CK_LAUNCH(ctx);
  // the order the overlapped exchange deals row tiles in (harmless otherwise)
  const int cg = P.align % 256 == 0 ? 2 : 1;
  ep_tile_order_kernel<<<1, 1024, (size_t)E * 4, ctx->stream>>>(P.rt, P.rplan.tile_expert, P.rplan.n_tiles, W,
                                                                 (int)el, P.r, cg, P.mtile_order);
  CK_LAUNCH(ctx);
  (void)C;
  P.planned = true;
}

static void ep_zero_pads_device(Ctx* ctx, const Layer::Ep& P, size_t rb, void* buf) {
  if (P.el == 0 || P.align <= 1) return;
  ep_zero_pads_kernel<<<(unsigned)P.el, 256, 0, ctx->stream>>>(static_cast<uint8_t*>(buf), (int64_t)rb,
                                                                P.rplan.offsets, P.rplan.counts);
  CK_LAUNCH(ctx);
}

// Count all-gather over peer memory (exchange_counts, collectives.cpp:69-109:
// every rank receives every rank's full count vector), the one host sync of
// an EP step, then the layouts of ALL ranks: this rank's receive layout (as
// ep_plan), where each of its send chunks lands in the destination's receive
// layout (scatter / gather-combine-backward routes) and where each received
// chunk goes home (fc2 / dgrad-fc1 epilogue routes).
static void ep_plan_peer(Layer& L) {
  Ctx* ctx = L.ctx;
  Layer::Ep& P = *L.ep;
  const int W = P.W, r = P.r;
  const int64_t el = P.el, E = L.E;
  P.peer.put_counts(ctx, L.plan.counts, E);
  P.peer.wait(ctx, PH_COUNTS);
  int32_t* hc = reinterpret_cast<int32_t*>(P.h_peer);
  CK(cudaMemcpyAsync(hc, P.cnt_mat, W * E * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));  // the one host sync of an EP step
  std::vector<int64_t> cnt(hc, hc + W * E);
  int32_t* grank = hc + W * E;
  int64_t* gdelta = reinterpret_cast<int64_t*>(P.h_peer + ((W * E * 4 + E * 4 + 7) & ~int64_t(7)));
  int32_t* rt = reinterpret_cast<int32_t*>(gdelta + E);
  P.send_off.assign(E, 0);
  P.chunk_off.assign(el * W, 0);
  P.block_off.assign(el + 1, 0);
  P.rows.assign(el, 0);
  ep_routes(W, r, el, P.align, cnt.data(), P.send_off.data(), P.chunk_off.data(), P.block_off.data(),
            P.rows.data(), grank, gdelta, rt);
  P.h_send.assign(cnt.begin() + (int64_t)r * E, cnt.begin() + (int64_t)(r + 1) * E);
  P.h_recv.assign((size_t)W * el, 0);
  for (int s = 0; s < W; ++s)
    for (int64_t e = 0; e < el; ++e) P.h_recv[s * el + e] = cnt[(int64_t)s * E + r * el + e];
  if (P.block_off[el] > P.cap_recv) protocol_error("exchange: received rows exceed the layer capacity");
  CK(cudaMemcpyAsync(P.g_rank, grank, E * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(P.g_delta, gdelta, E * 8, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(P.rt, rt, 3 * el * W * 4, cudaMemcpyHostToDevice, ctx->stream));
  // receive block plan (counts, offsets, 128-row tile table), as ep_plan
  int32_t* up = P.h_pinned + E + W * el;
  for (int64_t e = 0; e < el; ++e) up[e] = (int32_t)P.rows[e];
  int32_t* uo = up + el;
  for (int64_t e = 0; e <= el; ++e) uo[e] = (int32_t)P.block_off[e];
  int32_t* ut = uo + el + 1;
  int64_t nt = 0;
  for (int64_t e = 0; e < el; ++e)
    for (int64_t tt = P.block_off[e] / 128; tt < P.block_off[e + 1] / 128; ++tt) ut[nt++] = (int32_t)e;
  ut[nt] = (int32_t)nt;
  CK(cudaMemcpyAsync(P.rplan.counts, up, el * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(P.rplan.offsets, uo, (el + 1) * 4, cudaMemcpyHostToDevice, ctx->stream));
  if (nt) CK(cudaMemcpyAsync(P.rplan.tile_expert, ut, nt * 4, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(P.rplan.n_tiles, ut + nt, 4, cudaMemcpyHostToDevice, ctx->stream));
  // the staging is reused next step only after this step's host sync
  P.planned = true;
}

// A layer whose peers were connected by the host (fmoe_layer_peer_connect)
// runs the fused exchange without a transport.
static bool peer_ready(const Layer& L) {
  return L.ep && L.ep->peer.ok && L.t == FMOE_BF16 && L.ep->exchange == FMOE_EP_EXCHANGE_PEER;
}

static Transport* ep_transport(const Layer& L) {
  if (peer_ready(L) && !L.ctx->transport) return nullptr;
  return need_transport(L.ctx, L.cfg);
}

void Layer::ep_check() const { ep_transport(*this); }

// SMs the concurrent push keeps while fc1 / dgrad fc2 run beside it
#ifndef FMOE_EP_PUSH_SMS
#define FMOE_EP_PUSH_SMS 16
#endif

// The overlapped exchange needs device layouts, bf16 rows, and peers in other
// processes (a kernel spinning on a flag must not be able to starve the kernel
// that releases it, which ranks sharing one process and GPU could);
// FMOE_EP_OVERLAP=0 keeps the phase-ordered fused exchange.
static bool ep_overlap_ok(const Layer& L) {
  static const bool enabled = [] {
    const char* e = std::getenv("FMOE_EP_OVERLAP");
    return !(e && e[0] == '0');
  }();
  const Layer::Ep& P = *L.ep;
  return enabled && P.fused && P.device_plan && P.peer.cross_process && !P.peer.lw && L.t == FMOE_BF16 &&
         L.cfg.d_m % 8 == 0 && L.ctx->num_sms > 2 * FMOE_EP_PUSH_SMS;
}

// dir 0: forward rows (x -> peers' xs), 1: backward (w * d_y -> peers' d_ys)
static Arrival ep_arrival(const Layer& L, int dir) {
  const Layer::Ep& P = *L.ep;
  Arrival a;
  a.flags = P.flags + PH_N * P.W + dir * P.el * P.W;
  a.epoch = P.peer.epoch;
  a.rt = P.rt;
  a.W = P.W;
  a.C = (int)(P.el * P.W);
  a.mtile_order = P.mtile_order;
  a.grid_limit = L.ctx->num_sms - FMOE_EP_PUSH_SMS;
  return a;
}

// Launch the destination-major push of this rank's send rows on the side
// stream, ordered after everything issued so far on the layer stream (plan,
// layouts, pads); ev_pushed marks its end.
static void ep_push(Layer& L, const void* src, const void* w, int dir) {
  Ctx* ctx = L.ctx;
  Layer::Ep& P = *L.ep;
  if (!P.side) {
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&P.side, cudaStreamNonBlocking, hi));
    CK(cudaEventCreateWithFlags(&P.ev_go, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&P.ev_pushed, cudaEventDisableTiming));
  }
  CK(cudaEventRecord(P.ev_go, ctx->stream));
  CK(cudaStreamWaitEvent(P.side, P.ev_go, 0));
  const int64_t E = L.E;
  CK(cudaMemsetAsync(P.push_ctr, 0, (1 + E) * 4, P.side));
  const size_t smem = (size_t)(E + 2) * 4;
  const int base = PH_N * P.W + dir * (int)P.el * P.W;
  const auto* s16 = static_cast<const __nv_bfloat16*>(src);
  if (dir == 0)
    ep_push_kernel<false><<<FMOE_EP_PUSH_SMS, kPushThreads, smem, P.side>>>(
        s16, L.cfg.d_m, L.plan, nullptr, P.peer.d_ptr[PB_XS], P.g_delta, P.peer.d_ptr[PB_FLAGS], base, P.W, P.r,
        (int)P.el, P.peer.epoch, P.push_ctr);
  else
    ep_push_kernel<true><<<FMOE_EP_PUSH_SMS, kPushThreads, smem, P.side>>>(
        s16, L.cfg.d_m, L.plan, static_cast<const float*>(w), P.peer.d_ptr[PB_DYS], P.g_delta,
        P.peer.d_ptr[PB_FLAGS], base, P.W, P.r, (int)P.el, P.peer.epoch, P.push_ctr);
  CK(cudaGetLastError());
  ++ctx->launches;
  CK(cudaEventRecord(P.ev_pushed, P.side));
}

void Layer::ep_forward(const void* x, void* y) {
  Transport* tr = ep_transport(*this);
  Ep& P = *ep;
  const int64_t d = cfg.d_m, h = cfg.d_h;
  const size_t rb = (size_t)d * es;
  plan_build(ctx, idx, plan);                  // send plan over all E experts, reference layout
  P.fused = ep_use_peer(*this, tr);
  if (P.fused) {
    // fused: scatter straight into the expert ranks (global_scatter), fc2
    // epilogue straight back into the source ranks (global_gather)
    P.peer.epoch++;
    P.device_plan = ep_layout_smem(P.W, P.el) <= 48 * 1024 && P.align % 16 == 0 && rb % 16 == 0;
    if (P.device_plan) {
      ep_plan_peer_device(*this);              // C1 + layouts on the device: no host sync
      ep_zero_pads_device(ctx, P, rb, P.xs);
    } else {
      ep_plan_peer(*this);                     // C1 + every rank's layout on the host
      zero_pads(ctx, P, rb, P.xs);
    }
    P.overlap = ep_overlap_ok(*this);
    ctx_mark(ctx, MARK_PLAN);
    const int64_t c = P.el * P.W;
    RowRoute rr{P.peer.d_ptr[PB_YS], P.rt, P.rt + c, P.rt + 2 * c, P.W};
    if (P.overlap) {
      // C2 overlapped with fc1: the rows are pushed by a concurrent kernel on
      // the side stream (destination-major, per-chunk flags) while fc1, on
      // the SMs the push leaves free, takes its tiles in arrival order and
      // starts each as soon as its rows have landed
      Arrival arr = ep_arrival(*this, 0);
      ep_push(*this, x, nullptr, 0);
      ctx_mark(ctx, MARK_SCATTER);
      experts_fwd(ctx, t, P.rplan, d, h, params(), P.xs, P.hidden, P.ys, relu_bits, nullptr, &rr, &arr);
    } else {
      ScatterRoute sr{idx, P.g_rank, P.g_delta, P.peer.d_ptr[PB_XS]};
      scatter(ctx, t, x, d, plan, nullptr, &sr);  // C2 fused
      P.peer.signal(ctx, PH_SCATTER);
      P.peer.wait(ctx, PH_SCATTER);
      ctx_mark(ctx, MARK_SCATTER);
      experts_fwd(ctx, t, P.rplan, d, h, params(), P.xs, P.hidden, P.ys, relu_bits, nullptr, &rr);  // C3 fused
    }
    P.peer.signal(ctx, PH_GATHER);
    P.peer.wait(ctx, PH_GATHER);
    if (P.overlap) CK(cudaStreamWaitEvent(ctx->stream, P.ev_pushed, 0));  // x read by the push
    gather_combine(ctx, t, ys, d, plan, vals, y);
    ctx_mark(ctx, MARK_GATHER);
    return;
  }
  scatter(ctx, t, x, d, plan, xs);
  ep_plan(*this, tr);                          // C1 + receive layout
  ctx_mark(ctx, MARK_PLAN);
  zero_pads(ctx, P, rb, P.xs);
  exchange_rows(ctx, tr, P, rb, xs, P.xs, true);   // C2 global_scatter
  ctx_mark(ctx, MARK_SCATTER);
  experts_fwd(ctx, t, P.rplan, d, h, params(), P.xs, P.hidden, P.ys, relu_bits);
  exchange_rows(ctx, tr, P, rb, P.ys, ys, false);  // C3 global_gather
  gather_combine(ctx, t, ys, d, plan, vals, y);
  ctx_mark(ctx, MARK_GATHER);
}

void Layer::ep_backward(const void* dy, void* dx) {
  Transport* tr = ep_transport(*this);
  Ep& P = *ep;
  if (!P.planned) protocol_error("backward: no expert-parallel forward cache");
  const int64_t n = cfg.n_b, d = cfg.d_m, h = cfg.d_h, k = cfg.k;
  const size_t rb = (size_t)d * es;
  const bool bf = t == FMOE_BF16, gate = bf && !routed;
  ctx_mark(ctx, MARK_BWD_BEGIN);
  if (P.fused) {
    // gradients ride the same routes: d_ys straight into the expert ranks,
    // the dgrad-fc1 epilogue straight back into the source ranks; the weight
    // gradients and the gate's d_wg run while the peers finish
    if (P.device_plan)
      ep_zero_pads_device(ctx, P, rb, P.d_ys);
    else
      zero_pads(ctx, P, rb, P.d_ys);
    const int64_t c = P.el * P.W;
    RowRoute rr{P.peer.d_ptr[PB_DXS], P.rt, P.rt + c, P.rt + 2 * c, P.W};
    if (P.overlap) {
      // d_ys = w * d_y pushed by the side stream (destination-major, per-chunk
      // flags) while gcb computes d_w and the gate Jacobian here and dgrad fc2
      // consumes the arriving chunks tile by tile
      ep_push(*this, dy, vals, 1);
      gather_combine_bwd(ctx, t, dy, ys, d, plan, vals, nullptr, d_w, gate ? scores : nullptr,
                         gate ? idx : nullptr, gate ? dz_bf16 : nullptr, nullptr);
      ctx_mark(ctx, MARK_GCB);
      Arrival arr = ep_arrival(*this, 1);
      experts_bwd(ctx, t, P.rplan, d, h, params(), P.xs, P.hidden, P.d_ys, P.d_xs, grads(), P.d_pre, tpart,
                  relu_bits, nullptr, EXPERTS_BWD_DGRAD, &rr, &arr);
      CK(cudaStreamWaitEvent(ctx->stream, P.ev_pushed, 0));  // dy read by the push
    } else {
      ScatterRoute sr{idx, P.g_rank, P.g_delta, P.peer.d_ptr[PB_DYS]};
      gather_combine_bwd(ctx, t, dy, ys, d, plan, vals, nullptr, d_w, gate ? scores : nullptr,
                         gate ? idx : nullptr, gate ? dz_bf16 : nullptr, &sr);
      P.peer.signal(ctx, PH_SCATTER_BWD);
      P.peer.wait(ctx, PH_SCATTER_BWD);
      ctx_mark(ctx, MARK_GCB);
      experts_bwd(ctx, t, P.rplan, d, h, params(), P.xs, P.hidden, P.d_ys, P.d_xs, grads(), P.d_pre, tpart,
                  relu_bits, nullptr, EXPERTS_BWD_DGRAD, &rr);
    }
    P.peer.signal(ctx, PH_GATHER_BWD);
    experts_bwd(ctx, t, P.rplan, d, h, params(), P.xs, P.hidden, P.d_ys, P.d_xs, grads(), P.d_pre, tpart,
                relu_bits, nullptr, EXPERTS_BWD_WGRAD);
    if (routed) {
      CK(cudaMemsetAsync(dwg, 0, (size_t)d * E * ss, ctx->stream));
      P.peer.wait(ctx, PH_GATHER_BWD);
      scatter_bwd(ctx, t, d_xs, d, plan, dx, nullptr);
    } else {
      gate_dwg_bf16(ctx, x_saved, dz_bf16, n, d, E, part, (float*)dwg);
      ctx_mark(ctx, MARK_GATE_DWG);
      gate_dx_bf16(ctx, dz_bf16, wg, n, d, E, nullptr, nullptr, 0, gdx);
      P.peer.wait(ctx, PH_GATHER_BWD);
      scatter_bwd(ctx, t, d_xs, d, plan, dx, gdx);
    }
    ctx_mark(ctx, MARK_GATE_DX);
    return;
  }
  gather_combine_bwd(ctx, t, dy, ys, d, plan, vals, d_ys, d_w, gate ? scores : nullptr, gate ? idx : nullptr,
                     gate ? dz_bf16 : nullptr);
  zero_pads(ctx, P, rb, P.d_ys);
  exchange_rows(ctx, tr, P, rb, d_ys, P.d_ys, true);  // gradients ride the same routes
  ctx_mark(ctx, MARK_GCB);
  experts_bwd(ctx, t, P.rplan, d, h, params(), P.xs, P.hidden, P.d_ys, P.d_xs, grads(), P.d_pre, tpart,
              relu_bits);
  exchange_rows(ctx, tr, P, rb, P.d_xs, d_xs, false);
  if (routed) {  // injected routing: no gate, d_x is scatter_backward alone
    CK(cudaMemsetAsync(dwg, 0, (size_t)d * E * ss, ctx->stream));
    scatter_bwd(ctx, t, d_xs, d, plan, dx, nullptr);
  } else if (bf) {
    gate_dwg_bf16(ctx, x_saved, dz_bf16, n, d, E, part, (float*)dwg);
    ctx_mark(ctx, MARK_GATE_DWG);
    gate_dx_bf16(ctx, dz_bf16, wg, n, d, E, nullptr, nullptr, 0, gdx);
    scatter_bwd(ctx, t, d_xs, d, plan, dx, gdx);
  } else {
    gate_bwd(ctx, t, x_saved, wg, scores, idx, d_w, n, d, E, k, dwg, gdx, dz, nullptr, nullptr);
    ctx_mark(ctx, MARK_GATE_DWG);
    scatter_bwd(ctx, t, d_xs, d, plan, dx, gdx);
  }
  ctx_mark(ctx, MARK_GATE_DX);
}

}  // namespace fmoe_b200

namespace fmoe_b200 {
void Layer::ep_free(Ep* e) {
  if (!e) return;
  if (e->side) {
    cudaStreamSynchronize(e->side);
    cudaStreamDestroy(e->side);
    cudaEventDestroy(e->ev_go);
    cudaEventDestroy(e->ev_pushed);
  }
  e->peer.close();
  if (e->h_peer) cudaFreeHost(e->h_peer);
  delete e;
}
}  // namespace fmoe_b200

// ------------------------------------------------------------------- C-ABI
using namespace fmoe_b200;

#define FMOE_GUARD(...)               \
  try {                               \
    __VA_ARGS__;                      \
    return FMOE_OK;                   \
  } catch (const std::exception& e) { \
    return guard_status(e);           \
  } catch (...) {                     \
    g_last_error = "unknown error";   \
    return FMOE_ERR_CUDA;             \
  }

namespace fmoe_b200 {
// allreduce_sum (collectives.cpp:266-292): the reference accumulates at the
// group root in ascending rank order and sends the bytes back.  Here every
// member receives every other member's buffer and runs the same ordered sum,
// so each member holds the root's bytes without the second hop.
template <typename T>
__global__ void ordered_sum_kernel(const T* __restrict__ slabs, int64_t g, int64_t n, T* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T acc = slabs[i];
  for (int64_t s = 1; s < g; ++s) acc = acc + slabs[s * n + i];
  out[i] = acc;
}

void allreduce_sum(Ctx* c, fmoe_dtype dt, void* buf, int64_t n, const int* group, int64_t gs) {
  if (dt != FMOE_F64 && dt != FMOE_F32) shape_error("allreduce_sum: dtype must be FMOE_F64 or FMOE_F32");
  if (gs < 1 || !group) protocol_error("allreduce_sum: empty group");
  for (int64_t i = 1; i < gs; ++i)
    if (group[i] < group[i - 1]) protocol_error("allreduce_sum: group must be sorted ascending");
  Transport* tr = c->transport;
  const int W = tr ? tr->world : 1, r = tr ? tr->rank : 0;
  int64_t me = -1;
  for (int64_t i = 0; i < gs; ++i) {
    if (group[i] < 0 || group[i] >= W) protocol_error("allreduce_sum: group rank outside the world");
    if (group[i] == r) me = i;
  }
  if (me < 0) protocol_error("allreduce_sum: calling rank not in group");
  if (gs == 1) return;
  const size_t es = dtype_size(dt);
  // phase 1: element counts, so a shape mismatch is a ProtocolError on every
  // member instead of a mismatched transfer
  int64_t* cnt = (int64_t*)ctx_workspace(c, (size_t)(gs + 1) * 8 + (size_t)gs * n * es + 512);
  uint8_t* slabs = (uint8_t*)cnt + ((size_t)(gs + 1) * 8 + 255) / 256 * 256;
  std::vector<int64_t> h(gs, n);
  CK(cudaMemcpyAsync(cnt + gs, &n, 8, cudaMemcpyHostToDevice, c->stream));
  std::vector<Xfer> sends, recvs;
  for (int64_t i = 0; i < gs; ++i) {
    if (i == me) continue;
    sends.push_back({group[i], cnt + gs, 8});
    recvs.push_back({group[i], cnt + i, 8});
  }
  tr->group(c, sends, recvs);
  CK(cudaMemcpyAsync(h.data(), cnt, gs * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  h[me] = n;
  for (int64_t i = 0; i < gs; ++i)
    if (h[i] != n)
      protocol_error("allreduce_sum: rank " + std::to_string(group[i]) + " contributes " + std::to_string(h[i]) +
                     " elements, this rank " + std::to_string(n));
  if (n == 0) return;
  // phase 2: all-gather into [gs][n] slabs in group order, then the ordered sum
  sends.clear();
  recvs.clear();
  for (int64_t i = 0; i < gs; ++i) {
    if (i == me) continue;
    sends.push_back({group[i], buf, (size_t)n * es});
    recvs.push_back({group[i], slabs + (size_t)i * n * es, (size_t)n * es});
  }
  CK(cudaMemcpyAsync(slabs + (size_t)me * n * es, buf, (size_t)n * es, cudaMemcpyDeviceToDevice, c->stream));
  tr->group(c, sends, recvs);
  const unsigned grid = (unsigned)ceil_div(n, 256);
  if (dt == FMOE_F64)
    fmoe_b200::ordered_sum_kernel<double><<<grid, 256, 0, c->stream>>>((const double*)slabs, gs, n, (double*)buf);
  else
    fmoe_b200::ordered_sum_kernel<float><<<grid, 256, 0, c->stream>>>((const float*)slabs, gs, n, (float*)buf);
  CK_LAUNCH(c);
}
}  // namespace fmoe_b200

namespace {
Ctx* CX(fmoe_ctx* c) {
  if (!c) shape_error("null context");
  return reinterpret_cast<Ctx*>(c);
}
void set_transport(Ctx* c, Transport* t) {
  if (c->transport && c->owns_transport) delete c->transport;
  c->transport = t;
  c->owns_transport = true;
}

// Host exchange plan for the operator-level collectives (collectives.hpp:16-33).
struct HostPlan {
  int W, r;
  int64_t el;
  std::vector<int64_t> send, recv, send_off, chunk_off;
};
HostPlan host_plan(const fmoe_exchange_plan* p) {
  if (!p || !p->send_counts || !p->recv_counts) shape_error("null exchange plan");
  HostPlan h{(int)p->world, (int)p->rank, p->local_experts, {}, {}, {}, {}};
  const int64_t E = p->world * p->local_experts;
  h.send.assign(p->send_counts, p->send_counts + E);
  h.recv.assign(p->recv_counts, p->recv_counts + E);
  h.send_off.assign(E, 0);
  for (int64_t g = 1; g < E; ++g) h.send_off[g] = h.send_off[g - 1] + h.send[g - 1];
  h.chunk_off.assign(E, 0);
  int64_t at = 0;
  for (int64_t e = 0; e < h.el; ++e)
    for (int s = 0; s < h.W; ++s) {
      h.chunk_off[e * h.W + s] = at;
      at += h.recv[(int64_t)s * h.el + e];
    }
  return h;
}
void a2a(Ctx* c, fmoe_dtype dt, const void* src, int64_t d, const fmoe_exchange_plan* p, void* dst, bool fwd) {
  Transport* tr = c->transport;
  if (p->world > 1 && !tr) protocol_error("all_to_all_rows: no transport");
  HostPlan h = host_plan(p);
  Layer::Ep P;
  P.W = h.W;
  P.r = h.r;
  P.el = h.el;
  P.h_send = h.send;
  P.h_recv = h.recv;
  P.send_off = h.send_off;
  P.chunk_off = h.chunk_off;
  if (p->world == 1) {
    // world of one: the receive layout equals the send layout
    int64_t rows = 0;
    for (auto v : h.send) rows += v;
    if (rows) CK(cudaMemcpyAsync(dst, src, (size_t)rows * d * dtype_size(dt), cudaMemcpyDeviceToDevice, c->stream));
    return;
  }
  exchange_rows(c, tr, P, (size_t)d * dtype_size(dt), src, dst, fwd);
}

}  // namespace

extern "C" {

int fmoe_ep_routes(int world, int rank, int64_t local_experts, int64_t align, const int64_t* counts,
                   int64_t* send_off, int64_t* chunk_off, int64_t* block_off, int64_t* rows, int32_t* g_rank,
                   int64_t* g_delta, int32_t* route) {
  FMOE_GUARD({
    if (world < 1 || rank < 0 || rank >= world || local_experts < 1 || align < 1) shape_error("ep_routes: bad sizes");
    if (!counts || !send_off || !chunk_off || !block_off || !rows || !g_rank || !g_delta || !route)
      shape_error("ep_routes: null buffer");
    ep_routes(world, rank, local_experts, align, counts, send_off, chunk_off, block_off, rows, g_rank, g_delta,
              route);
  })
}

int fmoe_layer_peer_blob(fmoe_layer* layer, void* out, int64_t capacity, int64_t* length) {
  FMOE_GUARD({
    if (!layer || !length) shape_error("null argument");
    Layer* l = reinterpret_cast<Layer*>(layer);
    if (!l->ep || l->t != FMOE_BF16) shape_error("peer_blob: bf16 expert-parallel layers only");
    *length = (int64_t)PeerSet::blob_bytes();
    if (out) {
      if (capacity < *length) shape_error("peer_blob: buffer too small");
      Layer::Ep& P = *l->ep;
      void* bufs[PB_N] = {P.xs, P.d_ys, l->ys, l->d_xs, P.cnt_mat, P.flags};
      PeerSet::make_blob(l->ctx, bufs, out);
    }
  })
}

int fmoe_layer_peer_connect(fmoe_layer* layer, const void* blobs, int64_t blob_bytes) {
  FMOE_GUARD({
    if (!layer || !blobs) shape_error("null argument");
    Layer* l = reinterpret_cast<Layer*>(layer);
    if (!l->ep || l->t != FMOE_BF16) shape_error("peer_connect: bf16 expert-parallel layers only");
    if (blob_bytes != (int64_t)PeerSet::blob_bytes()) shape_error("peer_connect: blob size mismatch");
    Layer::Ep& P = *l->ep;
    if (P.peer_tried) protocol_error("peer_connect: must be called before the first forward");
    if (!P.peer.open(l->ctx, P.W, P.r, blobs, P.peer_table))
      throw Error(FMOE_ERR_TRANSPORT, "peer_connect: a peer's buffers cannot be mapped (no NVLink P2P / other host)");
    P.peer_tried = true;
  })
}

int fmoe_layer_set_ep_exchange(fmoe_layer* layer, int mode) {
  FMOE_GUARD({
    if (!layer) shape_error("null layer");
    if (mode != FMOE_EP_EXCHANGE_PEER && mode != FMOE_EP_EXCHANGE_TRANSPORT)
      shape_error("set_ep_exchange: unknown mode");
    Layer* l = reinterpret_cast<Layer*>(layer);
    if (l->ep) {
      if (l->ep->peer_tried) protocol_error("set_ep_exchange: must be set before the first forward");
      l->ep->exchange = mode;
    }
  })
}

int fmoe_layer_ep_exchange_fused(fmoe_layer* layer, int* fused) {
  FMOE_GUARD({
    if (!layer || !fused) shape_error("null argument");
    Layer* l = reinterpret_cast<Layer*>(layer);
    *fused = (l->ep && l->ep->fused) ? 1 : 0;
  })
}

int fmoe_ep_layout(int world, int64_t local_experts, int64_t align, const int64_t* send_counts,
                   const int64_t* recv_counts, int64_t* send_off, int64_t* chunk_off, int64_t* block_off,
                   int64_t* rows) {
  FMOE_GUARD({
    if (world < 1 || local_experts < 1 || align < 1) shape_error("ep_layout: bad sizes");
    if (!send_counts || !recv_counts || !send_off || !chunk_off || !block_off || !rows)
      shape_error("ep_layout: null buffer");
    ep_layout(world, local_experts, align, send_counts, recv_counts, send_off, chunk_off, block_off, rows);
  })
}

int fmoe_comm_unique_id(void* id_out, int64_t id_bytes) {
  FMOE_GUARD({
    if (!id_out) shape_error("null id buffer");
    nccl_unique_id(id_out, (size_t)id_bytes);
  })
}

int fmoe_comm_init(fmoe_ctx* ctx, const void* id, int64_t id_bytes, int world, int rank) {
  FMOE_GUARD({
    Ctx* c = CX(ctx);
    if (!id || id_bytes < 128) shape_error("fmoe_comm_init: need the 128-byte unique id");
    if (world < 1 || rank < 0 || rank >= world) shape_error("fmoe_comm_init: bad world/rank");
    CK(cudaSetDevice(c->device));
    set_transport(c, make_nccl_transport(id, world, rank));
    c->world = world;
    c->rank = rank;
  })
}

int fmoe_comm_attach(fmoe_ctx* ctx, void* nccl_comm) {
  FMOE_GUARD({
    Ctx* c = CX(ctx);
    if (!nccl_comm) shape_error("fmoe_comm_attach: null communicator");
    CK(cudaSetDevice(c->device));
    Transport* t = attach_nccl_transport(nccl_comm);
    c->world = t->world;
    c->rank = t->rank;
    set_transport(c, t);
  })
}

int fmoe_world_create(int world, fmoe_world** out) {
  FMOE_GUARD({
    if (world < 1 || !out) shape_error("fmoe_world_create: bad arguments");
    *out = reinterpret_cast<fmoe_world*>(new LocalWorld(world));
  })
}

int fmoe_world_destroy(fmoe_world* w) { FMOE_GUARD(delete reinterpret_cast<LocalWorld*>(w)) }

int fmoe_ctx_join_world(fmoe_ctx* ctx, fmoe_world* w, int rank) {
  FMOE_GUARD({
    Ctx* c = CX(ctx);
    auto* lw = reinterpret_cast<LocalWorld*>(w);
    if (!lw || rank < 0 || rank >= lw->world) shape_error("fmoe_ctx_join_world: bad world/rank");
    set_transport(c, make_local_transport(lw, rank));
    c->world = lw->world;
    c->rank = rank;
  })
}

int fmoe_exchange_counts(fmoe_ctx* ctx, const int64_t* local_counts, int64_t n_counts,
                         fmoe_exchange_plan* plan) {
  FMOE_GUARD({
    Ctx* c = CX(ctx);
    const int W = c->transport ? c->transport->world : 1;
    const int r = c->transport ? c->transport->rank : 0;
    if (!plan || !plan->send_counts || !plan->recv_counts) shape_error("exchange_counts: null plan buffers");
    if (n_counts < 1 || n_counts % W != 0)
      shape_error("exchange_counts: expert count " + std::to_string(n_counts) + " not divisible by world size " +
                  std::to_string(W));
    const int64_t el = n_counts / W;
    plan->world = W;
    plan->rank = r;
    plan->local_experts = el;
    std::vector<int32_t> h32(n_counts);
    for (int64_t i = 0; i < n_counts; ++i) {
      if (local_counts[i] < 0 || local_counts[i] > INT32_MAX) shape_error("exchange_counts: bad count");
      h32[i] = (int32_t)local_counts[i];
      plan->send_counts[i] = local_counts[i];
    }
    int32_t* dbuf = (int32_t*)ctx_workspace(c, (size_t)n_counts * 8);
    int32_t *dsend = dbuf, *drecv = dbuf + n_counts;
    CK(cudaMemcpyAsync(dsend, h32.data(), n_counts * 4, cudaMemcpyHostToDevice, c->stream));
    std::vector<Xfer> sends, recvs;
    for (int p = 0; p < W; ++p) {
      if (p == r) continue;
      sends.push_back({p, dsend + p * el, (size_t)el * 4});
      recvs.push_back({p, drecv + p * el, (size_t)el * 4});
    }
    CK(cudaMemcpyAsync(drecv + r * el, dsend + r * el, el * 4, cudaMemcpyDeviceToDevice, c->stream));
    if (W > 1) c->transport->group(c, sends, recvs);
    CK(cudaMemcpyAsync(h32.data(), drecv, n_counts * 4, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    plan->send_total = plan->recv_total = 0;
    for (int64_t i = 0; i < n_counts; ++i) {
      plan->recv_counts[i] = h32[i];
      plan->send_total += plan->send_counts[i];
      plan->recv_total += plan->recv_counts[i];
    }
  })
}

int fmoe_a2a_rows(fmoe_ctx* ctx, fmoe_dtype dtype, const void* xs, int64_t d, const fmoe_exchange_plan* plan,
                  void* out) {
  FMOE_GUARD(a2a(CX(ctx), dtype, xs, d, plan, out, true))
}

int fmoe_allreduce_sum(fmoe_ctx* ctx, fmoe_dtype dtype, void* buf, int64_t n, const int* group,
                       int64_t group_size) {
  FMOE_GUARD(allreduce_sum(CX(ctx), dtype, buf, n, group, group_size))
}

int fmoe_a2a_rows_reverse(fmoe_ctx* ctx, fmoe_dtype dtype, const void* ys, int64_t d,
                          const fmoe_exchange_plan* plan, void* out) {
  FMOE_GUARD(a2a(CX(ctx), dtype, ys, d, plan, out, false))
}

}  // extern "C"
