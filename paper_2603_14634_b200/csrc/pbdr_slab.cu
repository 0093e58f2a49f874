// Native x-slab decomposition of one giant scene (SURVEY.md section 8(e),
// BASELINE.json configs[4]) -- the C++ driver behind pbdr_gpu_slab_* in
// include/pbdr_gpu.h.
//
// Each rank holds a RANK-LOCAL scene: a contiguous range of the global bodies
// (config 5 numbers its cubes x-major, so an x-slab plus its ghost bands is a
// contiguous range; pbdr_scene_generate_c5_slab builds it), in the global
// order. Slot order is therefore the global order restricted to the range, so
// an owned particle's contact-candidate list -- and every owned trajectory --
// is the single-GPU one, bit for bit, as long as every body that can touch an
// owned body is present and current here. Nothing is replicated beyond the
// ghost bands.
//
// Roles (pbdr_gpu_set_roles): owned = com_x in this rank's slab (the north_star
// rule); ghost = owned by a neighbour and within the ghost band G of the shared
// boundary (the owner decides and sends the list); inactive = everything else.
//
// Per frame (host-synchronised once): the owners measure com_x, a body whose
// com left the slab migrates to the neighbour (its anchor and warm-start
// rotation travel with it; its particles are already present there as a
// ghost), then every owner sends each neighbour the global ids of its bodies
// within G of their shared boundary plus their full state.
// Per substep: integrate / hash grid / candidates over owned + ghost bodies,
// then the iterations over the owned bodies; after every iteration the ghosts'
// positions come from their owners (refresh = 0: exact), after the last one
// also velocities, anchors and rotations, so the ghosts' next integrate is the
// owner's. refresh = 1 skips the per-iteration refresh (ghosts stale within a
// substep: the cheaper variant SURVEY 8(e) asks to measure).
// With overlap = 1 each iteration runs the tiles holding bodies that a
// neighbour ghosts first; their halo (gather, NCCL send/recv, scatter) then
// runs on a second stream while the remaining (interior) tiles compute.
//
// Transports: NCCL point-to-point (one rank per GPU, ncclGroupStart /
// ncclSend / ncclRecv / ncclGroupEnd on the comm stream), or a local hub for
// ranks that are threads of one process sharing one GPU (device-to-device
// copies ordered by events) -- the tests' way to run the same driver without
// several GPUs.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "pbdr_handle.h"

struct pbdr_slab_hub {
  int world = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  struct Post {
    int peer;
    const void* buf;
    size_t bytes;
  };
  std::vector<std::vector<Post>> posts;     // per rank: its sends of the current exchange
  std::vector<cudaEvent_t> ready, copied;   // per rank
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const int64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

namespace pbdr_engine {

namespace {

struct Xfer {
  int peer;
  void* buf;
  size_t bytes;
};

struct Transport {
  virtual ~Transport() = default;
  // Point-to-point with the neighbours, enqueued on `s`. Every rank calls it
  // with matching sizes (receivers know them from an earlier count exchange).
  virtual int exchange(cudaStream_t s, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs) = 0;
};

struct NcclTransport final : Transport {
  ncclComm_t comm = nullptr;
  ~NcclTransport() override {
    if (comm) ncclCommDestroy(comm);
  }
  int exchange(cudaStream_t s, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs) override {
    ncclResult_t r = ncclGroupStart();
    for (const Xfer& x : sends)
      if (r == ncclSuccess && x.bytes) r = ncclSend(x.buf, x.bytes, ncclChar, x.peer, comm, s);
    for (const Xfer& x : recvs)
      if (r == ncclSuccess && x.bytes) r = ncclRecv(x.buf, x.bytes, ncclChar, x.peer, comm, s);
    const ncclResult_t e = ncclGroupEnd();
    if (r == ncclSuccess) r = e;
    if (r != ncclSuccess)
      return pbdr_host::set_error(PBDR_ERR_CUDA, std::string("NCCL halo exchange: ") + ncclGetErrorString(r));
    return PBDR_OK;
  }
};

struct LocalTransport final : Transport {
  pbdr_slab_hub* hub = nullptr;
  int rank = 0;
  int exchange(cudaStream_t s, const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs) override {
    pbdr_slab_hub& H = *hub;
    {
      std::lock_guard<std::mutex> lk(H.m);
      H.posts[rank].clear();
      for (const Xfer& x : sends) H.posts[rank].push_back({x.peer, x.buf, x.bytes});
    }
    if (cudaEventRecord(H.ready[rank], s) != cudaSuccess) return cuda_fail(cudaGetLastError(), "hub ready");
    H.barrier();  // every rank's payload enqueued
    for (const Xfer& x : recvs) {
      const pbdr_slab_hub::Post* src = nullptr;
      for (const auto& p : H.posts[x.peer])
        if (p.peer == rank) src = &p;
      if (!src || src->bytes != x.bytes)
        return pbdr_host::set_error(PBDR_ERR_GENERIC, "local slab hub: mismatched halo sizes");
      cudaStreamWaitEvent(s, H.ready[x.peer], 0);
      if (x.bytes) cudaMemcpyAsync(x.buf, src->buf, x.bytes, cudaMemcpyDeviceToDevice, s);
    }
    cudaEventRecord(H.copied[rank], s);
    H.barrier();  // every copy enqueued
    for (const Xfer& x : sends) cudaStreamWaitEvent(s, H.copied[x.peer], 0);  // send buffers reusable after
    H.barrier();  // posts may be overwritten by the next exchange
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PBDR_OK : cuda_fail(e, "local halo exchange");
  }
};

// Device scratch that grows on demand (owned by the handle's allocator).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(pbdr_handle* h, size_t need) {
    if (need <= bytes) return PBDR_OK;
    size_t nb = std::max(need, bytes * 2);
    nb = std::max<size_t>(nb, 256);
    const int rc = device_alloc(h, &p, nb);
    if (rc == PBDR_OK) bytes = nb;
    return rc;
  }
};

}  // namespace

struct SlabDriver {
  pbdr_handle* h = nullptr;
  int rank = 0, world = 1;
  std::vector<double> edges;  // world + 1
  double G = 0, margin = 0;
  int64_t body_first = 0;
  int refresh = 0, overlap = 0;
  std::unique_ptr<Transport> tr;
  std::vector<int> peers;
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_bnd = nullptr, ev_halo = nullptr;

  std::vector<int32_t> owned;  // local ids, ascending
  std::vector<double> com_ref;
  std::vector<double> stats_h;  // 13 doubles per body
  int64_t frames_done = 0, migrations = 0;

  struct Peer {
    std::vector<int32_t> send_bodies, recv_bodies;  // local ids
    DevBuf d_send_slots, d_recv_slots, d_send_bidx, d_recv_bidx;
    int64_t n_send_slots = 0, n_recv_slots = 0;
    DevBuf d_out, d_in;  // packed float4 records
  };
  std::map<int, Peer> P;
  DevBuf d_i64_out, d_i64_in;  // id / count staging
  DevBuf d_tiles;              // [boundary tiles | interior tiles] + 2 counts
  int n_bnd = 0, n_int = 0;
  int64_t halo_bytes_iter = 0;

  ~SlabDriver() {
    if (ev_bnd) cudaEventDestroy(ev_bnd);
    if (ev_halo) cudaEventDestroy(ev_halo);
    if (comm) cudaStreamDestroy(comm);
  }

  int32_t slab_of(double x) const {
    int r = 0;
    while (r + 1 < world && x >= edges[r + 1]) ++r;
    return r;
  }

  // com_x of the bodies the stats kernel covers (owned, or all before roles).
  int measure_com() {
    enqueue_body_stats(h, h->stats);
    stats_h.resize(static_cast<size_t>(h->nb) * 13);
    cudaError_t e = cudaMemcpyAsync(stats_h.data(), h->stats, sizeof(double) * stats_h.size(),
                                    cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    return e == cudaSuccess ? PBDR_OK : cuda_fail(e, "slab com readback");
  }
  double com_x(int32_t b) const { return stats_h[static_cast<size_t>(b) * 13]; }

  // Variable-length int64 lists to / from each neighbour (counts first).
  int exchange_i64(const std::map<int, std::vector<int64_t>>& out, std::map<int, std::vector<int64_t>>& in) {
    const size_t np = peers.size();
    int rc = d_i64_out.ensure(h, sizeof(int64_t) * np);
    if (rc == PBDR_OK) rc = d_i64_in.ensure(h, sizeof(int64_t) * np);
    if (rc != PBDR_OK) return rc;
    std::vector<int64_t> cnt(np), got(np);
    std::vector<Xfer> s, r;
    for (size_t k = 0; k < np; ++k) {
      cnt[k] = static_cast<int64_t>(out.at(peers[k]).size());
      s.push_back({peers[k], static_cast<int64_t*>(d_i64_out.p) + k, sizeof(int64_t)});
      r.push_back({peers[k], static_cast<int64_t*>(d_i64_in.p) + k, sizeof(int64_t)});
    }
    cudaMemcpyAsync(d_i64_out.p, cnt.data(), sizeof(int64_t) * np, cudaMemcpyHostToDevice, h->stream);
    if ((rc = tr->exchange(h->stream, s, r)) != PBDR_OK) return rc;
    cudaMemcpyAsync(got.data(), d_i64_in.p, sizeof(int64_t) * np, cudaMemcpyDeviceToHost, h->stream);
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) return cuda_fail(cudaGetLastError(), "slab counts");
    int64_t tot_out = 0, tot_in = 0;
    for (size_t k = 0; k < np; ++k) {
      tot_out += cnt[k];
      tot_in += got[k];
    }
    rc = d_i64_out.ensure(h, sizeof(int64_t) * std::max<int64_t>(1, tot_out));
    if (rc == PBDR_OK) rc = d_i64_in.ensure(h, sizeof(int64_t) * std::max<int64_t>(1, tot_in));
    if (rc != PBDR_OK) return rc;
    s.clear();
    r.clear();
    std::vector<int64_t> flat;
    int64_t oo = 0, oi = 0;
    for (size_t k = 0; k < np; ++k) {
      const auto& v = out.at(peers[k]);
      flat.insert(flat.end(), v.begin(), v.end());
      s.push_back({peers[k], static_cast<int64_t*>(d_i64_out.p) + oo, sizeof(int64_t) * v.size()});
      r.push_back({peers[k], static_cast<int64_t*>(d_i64_in.p) + oi, sizeof(int64_t) * static_cast<size_t>(got[k])});
      oo += static_cast<int64_t>(v.size());
      oi += got[k];
    }
    if (!flat.empty())
      cudaMemcpyAsync(d_i64_out.p, flat.data(), sizeof(int64_t) * flat.size(), cudaMemcpyHostToDevice, h->stream);
    if ((rc = tr->exchange(h->stream, s, r)) != PBDR_OK) return rc;
    std::vector<int64_t> back(static_cast<size_t>(tot_in));
    if (tot_in)
      cudaMemcpyAsync(back.data(), d_i64_in.p, sizeof(int64_t) * back.size(), cudaMemcpyDeviceToHost, h->stream);
    if (cudaStreamSynchronize(h->stream) != cudaSuccess) return cuda_fail(cudaGetLastError(), "slab ids");
    in.clear();
    oi = 0;
    for (size_t k = 0; k < np; ++k) {
      in[peers[k]].assign(back.begin() + oi, back.begin() + oi + got[k]);
      oi += got[k];
    }
    return PBDR_OK;
  }

  // Slots of local bodies (body-major layout).
  void slots_of(const std::vector<int32_t>& bodies, std::vector<int32_t>& out) const {
    out.clear();
    for (const int32_t b : bodies)
      for (int k = 0; k < h->h_bcount[b]; ++k) out.push_back(static_cast<int32_t>(h->h_bstart[b] + k));
  }

  static int upload_i32(pbdr_handle* hh, DevBuf& d, const std::vector<int32_t>& v) {
    const int rc = d.ensure(hh, sizeof(int32_t) * std::max<size_t>(1, v.size()));
    if (rc != PBDR_OK) return rc;
    if (!v.empty()) cudaMemcpyAsync(d.p, v.data(), sizeof(int32_t) * v.size(), cudaMemcpyHostToDevice, hh->stream);
    return PBDR_OK;
  }

  // Halo: the listed fields of the owned bodies a neighbour ghosts, packed per
  // peer (particle records, then body records), received into the ghosts.
  int send_fields(bool pos, bool rest_of_state, cudaStream_t s) {
    std::vector<Xfer> sx, rx;
    for (const int p : peers) {
      Peer& q = P[p];
      const int64_t rec_out = (pos ? q.n_send_slots : 0) + (rest_of_state ? q.n_send_slots + 2 * static_cast<int64_t>(q.send_bodies.size()) : 0);
      const int64_t rec_in = (pos ? q.n_recv_slots : 0) + (rest_of_state ? q.n_recv_slots + 2 * static_cast<int64_t>(q.recv_bodies.size()) : 0);
      int rc = q.d_out.ensure(h, sizeof(float4) * std::max<int64_t>(1, rec_out));
      if (rc == PBDR_OK) rc = q.d_in.ensure(h, sizeof(float4) * std::max<int64_t>(1, rec_in));
      if (rc != PBDR_OK) return rc;
      float4* o = static_cast<float4*>(q.d_out.p);
      const int* ss = static_cast<const int*>(q.d_send_slots.p);
      const int* sb = static_cast<const int*>(q.d_send_bidx.p);
      if (pos) {
        pbdr_dev::launch_gather4(o, h->pos[h->cur], ss, q.n_send_slots, s);
        o += q.n_send_slots;
      }
      if (rest_of_state) {
        pbdr_dev::launch_gather4(o, h->vel, ss, q.n_send_slots, s);
        o += q.n_send_slots;
        pbdr_dev::launch_gather4(o, h->anchor, sb, static_cast<int64_t>(q.send_bodies.size()), s);
        o += q.send_bodies.size();
        pbdr_dev::launch_gather4(o, h->rquat, sb, static_cast<int64_t>(q.send_bodies.size()), s);
      }
      sx.push_back({p, q.d_out.p, sizeof(float4) * static_cast<size_t>(rec_out)});
      rx.push_back({p, q.d_in.p, sizeof(float4) * static_cast<size_t>(rec_in)});
    }
    int rc = tr->exchange(s, sx, rx);
    if (rc != PBDR_OK) return rc;
    for (const int p : peers) {
      Peer& q = P[p];
      const float4* in = static_cast<const float4*>(q.d_in.p);
      const int* rs = static_cast<const int*>(q.d_recv_slots.p);
      const int* rb = static_cast<const int*>(q.d_recv_bidx.p);
      if (pos) {
        pbdr_dev::launch_scatter4(h->pos[h->cur], in, rs, q.n_recv_slots, s);
        in += q.n_recv_slots;
      }
      if (rest_of_state) {
        pbdr_dev::launch_scatter4(h->vel, in, rs, q.n_recv_slots, s);
        in += q.n_recv_slots;
        pbdr_dev::launch_scatter4(h->anchor, in, rb, static_cast<int64_t>(q.recv_bodies.size()), s);
        in += q.recv_bodies.size();
        pbdr_dev::launch_scatter4(h->rquat, in, rb, static_cast<int64_t>(q.recv_bodies.size()), s);
      }
    }
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PBDR_OK : cuda_fail(e, "halo gather/scatter");
  }

  int local_of(int64_t global, int32_t* local) const {
    const int64_t l = global - body_first;
    if (l < 0 || l >= h->nb) return PBDR_ERR_SIMULATION;
    *local = static_cast<int32_t>(l);
    return PBDR_OK;
  }

  // Owners tell each neighbour which of their bodies to ghost (global ids +
  // full state); roles, halo plans and tile lists follow.
  int build_ghosts() {
    std::map<int, std::vector<int64_t>> out, in;
    for (const int p : peers) {
      auto& v = out[p];
      for (const int32_t b : owned) {
        const double cx = com_x(b);
        if (p == rank - 1 ? cx < edges[rank] + G : cx >= edges[rank + 1] - G) v.push_back(b + body_first);
      }
    }
    int rc = exchange_i64(out, in);
    if (rc != PBDR_OK) return rc;
    std::vector<int8_t> roles(static_cast<size_t>(h->nb), 0);
    halo_bytes_iter = 0;
    for (const int p : peers) {
      Peer& q = P[p];
      q.send_bodies.clear();
      q.recv_bodies.clear();
      for (const int64_t g : out[p]) q.send_bodies.push_back(static_cast<int32_t>(g - body_first));
      for (const int64_t g : in[p]) {
        int32_t l = 0;
        if (local_of(g, &l) != PBDR_OK)
          return pbdr_host::set_sim_error("slab ghost band reaches past the rank-local scene (global body " +
                                              std::to_string(g) + ")",
                                          frames_done, -1, nullptr, PBDR_ERR_SIMULATION);
        q.recv_bodies.push_back(l);
        roles[static_cast<size_t>(l)] = 1;
      }
      std::vector<int32_t> slots;
      slots_of(q.send_bodies, slots);
      q.n_send_slots = static_cast<int64_t>(slots.size());
      if ((rc = upload_i32(h, q.d_send_slots, slots)) != PBDR_OK) return rc;
      slots_of(q.recv_bodies, slots);
      q.n_recv_slots = static_cast<int64_t>(slots.size());
      if ((rc = upload_i32(h, q.d_recv_slots, slots)) != PBDR_OK) return rc;
      if ((rc = upload_i32(h, q.d_send_bidx, q.send_bodies)) != PBDR_OK) return rc;
      if ((rc = upload_i32(h, q.d_recv_bidx, q.recv_bodies)) != PBDR_OK) return rc;
      halo_bytes_iter += static_cast<int64_t>(sizeof(float4)) * (q.n_send_slots + q.n_recv_slots);
    }
    for (const int32_t b : owned) roles[static_cast<size_t>(b)] = 2;
    if ((rc = pbdr_gpu_set_roles(h, roles.data())) != PBDR_OK) return rc;
    if ((rc = build_tile_lists()) != PBDR_OK) return rc;
    return send_fields(true, true, h->stream);  // new ghosts need their full state
  }

  // Tiles (of the owned packing) holding a body some neighbour ghosts run
  // first when overlapping; the rest after.
  int build_tile_lists() {
    std::vector<char> sent(static_cast<size_t>(h->nb), 0);
    for (const int p : peers)
      for (const int32_t b : P[p].send_bodies) sent[static_cast<size_t>(b)] = 1;
    std::vector<int32_t> bnd, inr;
    for (int t = 0; t < static_cast<int>(h->h_iter_cdesc.size()); ++t) {
      const int4 cd = h->h_iter_cdesc[t];
      bool b = false;
      for (int k = 0; k < cd.w && !b; ++k) b = sent[static_cast<size_t>(cd.z + k)] != 0;
      (b ? bnd : inr).push_back(t);
    }
    n_bnd = static_cast<int>(bnd.size());
    n_int = static_cast<int>(inr.size());
    std::vector<int32_t> all(bnd);
    all.insert(all.end(), inr.begin(), inr.end());
    all.push_back(n_bnd);
    all.push_back(n_int);
    return upload_i32(h, d_tiles, all);
  }

  int start() {
    // Before any roles every local body is measured; owners by com_x.
    if (int rc = pbdr_gpu_set_roles(h, nullptr); rc != PBDR_OK) return rc;
    if (int rc = measure_com(); rc != PBDR_OK) return rc;
    owned.clear();
    for (int32_t b = 0; b < h->nb; ++b)
      if (slab_of(com_x(b)) == rank) owned.push_back(b);
    com_ref.assign(static_cast<size_t>(h->nb), 0.0);
    for (int32_t b = 0; b < h->nb; ++b) com_ref[static_cast<size_t>(b)] = com_x(b);
    return build_ghosts();
  }

  int repartition() {
    if (int rc = measure_com(); rc != PBDR_OK) return rc;
    std::map<int, std::vector<int64_t>> out, in;
    for (const int p : peers) out[p];
    std::vector<int32_t> keep;
    for (const int32_t b : owned) {
      const double cx = com_x(b);
      const double drift = std::fabs(cx - com_ref[static_cast<size_t>(b)]);
      if (drift > 0.5 * margin)
        return pbdr_host::set_sim_error("slab halo margin exceeded: body moved " + std::to_string(drift) +
                                            " m in x in one frame",
                                        frames_done, b, nullptr, PBDR_ERR_SIMULATION);
      const int d = slab_of(cx);
      if (d == rank) {
        keep.push_back(b);
      } else if (d == rank - 1 || d == rank + 1) {
        out[d].push_back(b + body_first);
      } else {
        return pbdr_host::set_sim_error("a body skipped a whole slab in one frame", frames_done, b, nullptr,
                                        PBDR_ERR_SIMULATION);
      }
    }
    int rc = exchange_i64(out, in);
    if (rc != PBDR_OK) return rc;
    // Migrants: com_x (for the ghost decision), anchor, warm-start rotation.
    std::vector<Xfer> sx, rx;
    std::map<int, std::vector<int32_t>> out_l, in_l;
    for (const int p : peers) {
      for (const int64_t g : out[p]) out_l[p].push_back(static_cast<int32_t>(g - body_first));
      for (const int64_t g : in[p]) {
        int32_t l = 0;
        if (local_of(g, &l) != PBDR_OK)
          return pbdr_host::set_sim_error("a migrating body is outside the rank-local scene", frames_done, -1,
                                          nullptr, PBDR_ERR_SIMULATION);
        in_l[p].push_back(l);
      }
    }
    // Pack (com_x, 0, 0, 0), anchor, rotation per migrant as float4 records:
    // com_x travels as the exact double through two floats' bits.
    for (const int p : peers) {
      Peer& q = P[p];
      const size_t no = out_l[p].size(), ni = in_l[p].size();
      if ((rc = q.d_out.ensure(h, sizeof(float4) * 3 * std::max<size_t>(1, no))) != PBDR_OK) return rc;
      if ((rc = q.d_in.ensure(h, sizeof(float4) * 3 * std::max<size_t>(1, ni))) != PBDR_OK) return rc;
      std::vector<float4> coms(no);
      for (size_t k = 0; k < no; ++k) {
        const double c = com_x(out_l[p][k]);
        float4 f;
        std::memcpy(&f, &c, sizeof c);
        f.z = f.w = 0.0f;
        coms[k] = f;
      }
      float4* o = static_cast<float4*>(q.d_out.p);
      if (no) cudaMemcpyAsync(o, coms.data(), sizeof(float4) * no, cudaMemcpyHostToDevice, h->stream);
      if ((rc = upload_i32(h, q.d_send_bidx, out_l[p])) != PBDR_OK) return rc;
      pbdr_dev::launch_gather4(o + no, h->anchor, static_cast<const int*>(q.d_send_bidx.p), static_cast<int64_t>(no),
                               h->stream);
      pbdr_dev::launch_gather4(o + 2 * no, h->rquat, static_cast<const int*>(q.d_send_bidx.p),
                               static_cast<int64_t>(no), h->stream);
      sx.push_back({p, o, sizeof(float4) * 3 * no});
      rx.push_back({p, q.d_in.p, sizeof(float4) * 3 * ni});
    }
    if ((rc = tr->exchange(h->stream, sx, rx)) != PBDR_OK) return rc;
    for (const int p : peers) {
      Peer& q = P[p];
      const size_t ni = in_l[p].size();
      if ((rc = upload_i32(h, q.d_recv_bidx, in_l[p])) != PBDR_OK) return rc;
      const float4* in4 = static_cast<const float4*>(q.d_in.p);
      pbdr_dev::launch_scatter4(h->anchor, in4 + ni, static_cast<const int*>(q.d_recv_bidx.p),
                                static_cast<int64_t>(ni), h->stream);
      pbdr_dev::launch_scatter4(h->rquat, in4 + 2 * ni, static_cast<const int*>(q.d_recv_bidx.p),
                                static_cast<int64_t>(ni), h->stream);
      std::vector<float4> coms(ni);
      if (ni) cudaMemcpyAsync(coms.data(), in4, sizeof(float4) * ni, cudaMemcpyDeviceToHost, h->stream);
      if (cudaStreamSynchronize(h->stream) != cudaSuccess) return cuda_fail(cudaGetLastError(), "migration");
      for (size_t k = 0; k < ni; ++k) {
        double c;
        std::memcpy(&c, &coms[k], sizeof c);
        stats_h[static_cast<size_t>(in_l[p][k]) * 13] = c;
        keep.push_back(in_l[p][k]);
      }
      migrations += static_cast<int64_t>(ni);
    }
    std::sort(keep.begin(), keep.end());
    owned.swap(keep);
    for (const int32_t b : owned) com_ref[static_cast<size_t>(b)] = com_x(b);
    return build_ghosts();
  }

  // refresh = 1 between refreshes: the ghosts keep their positions into the
  // iteration's output buffer (nothing else writes ghost slots).
  int carry_ghosts(cudaStream_t s) {
    for (const int p : peers) {
      Peer& q = P[p];
      if (int rc = q.d_in.ensure(h, sizeof(float4) * std::max<int64_t>(1, q.n_recv_slots)); rc != PBDR_OK) return rc;
      const int* rs = static_cast<const int*>(q.d_recv_slots.p);
      pbdr_dev::launch_gather4(static_cast<float4*>(q.d_in.p), h->pos[h->cur ^ 1], rs, q.n_recv_slots, s);
      pbdr_dev::launch_scatter4(h->pos[h->cur], static_cast<const float4*>(q.d_in.p), rs, q.n_recv_slots, s);
    }
    return PBDR_OK;
  }

  // One iteration over the owned tiles, then the ghosts' halo.
  int iteration(int k, bool last) {
    const bool halo_pos = refresh == 0 || last;
    const int* tiles = static_cast<const int*>(d_tiles.p);
    const int* cnt = tiles + n_bnd + n_int;
    if (overlap && h->pk_iter.nbig == 0) {
      enqueue_iteration_tiles(h, k, tiles, cnt);                   // boundary tiles
      cudaEventRecord(ev_bnd, h->stream);
      cudaStreamWaitEvent(comm, ev_bnd, 0);
      const int cur = h->cur;
      h->cur ^= 1;  // the halo reads / writes the iteration's output buffer
      int rc = halo_pos ? send_fields(true, last, comm) : carry_ghosts(comm);
      h->cur = cur;
      if (rc != PBDR_OK) return rc;
      enqueue_iteration_tiles(h, k, tiles + n_bnd, cnt + 1);        // interior tiles, overlapped
      cudaEventRecord(ev_halo, comm);
      cudaStreamWaitEvent(h->stream, ev_halo, 0);
      h->cur ^= 1;
      return PBDR_OK;
    }
    enqueue_iteration_tiles(h, k, nullptr, nullptr);
    h->cur ^= 1;
    if (!halo_pos) return carry_ghosts(h->stream);
    return send_fields(true, last, h->stream);
  }

  int step_frames(int64_t frames) {
    for (int64_t f = 0; f < frames; ++f) {
      int rc = frames_done > 0 ? repartition() : PBDR_OK;
      if (rc != PBDR_OK) return rc;
      for (int s = 0; s < h->substeps; ++s) {
        enqueue_substep(h);
        for (int k = 0; k < h->iters; ++k)
          if ((rc = iteration(k, k == h->iters - 1)) != PBDR_OK) return rc;
        h->substeps_done += 1;
      }
      if ((rc = check_errors(h)) != PBDR_OK) return rc;
      ++frames_done;
    }
    return PBDR_OK;
  }
};

void slab_driver_destroy(SlabDriver* d) { delete d; }

}  // namespace pbdr_engine

using pbdr_engine::SlabDriver;

namespace {

int attach(pbdr_handle* h, const pbdr_slab_config* c, std::unique_ptr<pbdr_engine::Transport> tr) {
  if (c->world < 1 || c->rank < 0 || c->rank >= c->world || !c->edges)
    return pbdr_host::set_config_error("slab", "rank / world / edges");
  auto* d = new SlabDriver();
  d->h = h;
  d->rank = c->rank;
  d->world = c->world;
  d->edges.assign(c->edges, c->edges + c->world + 1);
  d->G = c->ghost_band;
  d->margin = c->margin;
  d->body_first = c->body_first;
  d->refresh = c->refresh;
  d->overlap = c->overlap;
  d->tr = std::move(tr);
  for (const int p : {c->rank - 1, c->rank + 1})
    if (p >= 0 && p < c->world) d->peers.push_back(p);
  cudaError_t e = cudaStreamCreateWithFlags(&d->comm, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_bnd, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&d->ev_halo, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete d;
    return pbdr_engine::cuda_fail(e, "slab streams");
  }
  if (h->slab_driver) pbdr_engine::slab_driver_destroy(h->slab_driver);
  h->slab_driver = d;
  return PBDR_OK;
}

}  // namespace

extern "C" {

int pbdr_nccl_unique_id(uint8_t out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return pbdr_host::set_error(PBDR_ERR_CUDA, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  std::memcpy(out, &id, sizeof id);
  return PBDR_OK;
}

int pbdr_gpu_slab_attach_nccl(pbdr_handle* h, const pbdr_slab_config* c, const uint8_t nccl_id[128]) {
  if (!h || !c || !nccl_id) return pbdr_host::set_error(PBDR_ERR_GENERIC, "null argument");
  cudaSetDevice(h->device);
  auto t = std::make_unique<pbdr_engine::NcclTransport>();
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof id);
  const ncclResult_t r = ncclCommInitRank(&t->comm, c->world, id, c->rank);
  if (r != ncclSuccess) return pbdr_host::set_error(PBDR_ERR_CUDA, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  return attach(h, c, std::move(t));
}

pbdr_slab_hub* pbdr_slab_hub_create(int world) {
  if (world < 1) return nullptr;
  auto* hub = new pbdr_slab_hub();
  hub->world = world;
  hub->posts.resize(static_cast<size_t>(world));
  hub->ready.assign(static_cast<size_t>(world), nullptr);
  hub->copied.assign(static_cast<size_t>(world), nullptr);
  for (int r = 0; r < world; ++r) {
    cudaEventCreateWithFlags(&hub->ready[r], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&hub->copied[r], cudaEventDisableTiming);
  }
  return hub;
}

void pbdr_slab_hub_destroy(pbdr_slab_hub* hub) {
  if (!hub) return;
  for (auto e : hub->ready) cudaEventDestroy(e);
  for (auto e : hub->copied) cudaEventDestroy(e);
  delete hub;
}

int pbdr_gpu_slab_attach_local(pbdr_handle* h, const pbdr_slab_config* c, pbdr_slab_hub* hub) {
  if (!h || !c || !hub) return pbdr_host::set_error(PBDR_ERR_GENERIC, "null argument");
  if (hub->world != c->world) return pbdr_host::set_config_error("slab", "hub world differs from the config");
  cudaSetDevice(h->device);
  auto t = std::make_unique<pbdr_engine::LocalTransport>();
  t->hub = hub;
  t->rank = c->rank;
  return attach(h, c, std::move(t));
}

int pbdr_gpu_slab_start(pbdr_handle* h) {
  if (!h || !h->slab_driver) return pbdr_host::set_error(PBDR_ERR_GENERIC, "no slab driver attached");
  pbdr_host::clear_error();
  cudaSetDevice(h->device);
  return h->slab_driver->start();
}

int pbdr_gpu_slab_step_frames(pbdr_handle* h, int64_t frames) {
  if (!h || !h->slab_driver) return pbdr_host::set_error(PBDR_ERR_GENERIC, "no slab driver attached");
  pbdr_host::clear_error();
  cudaSetDevice(h->device);
  return h->slab_driver->step_frames(frames);
}

int pbdr_gpu_slab_owned(pbdr_handle* h, int32_t* local_ids, int64_t capacity, int64_t* count) {
  if (!h || !h->slab_driver || !count) return pbdr_host::set_error(PBDR_ERR_GENERIC, "no slab driver attached");
  const auto& o = h->slab_driver->owned;
  *count = static_cast<int64_t>(o.size());
  if (local_ids)
    for (int64_t k = 0; k < std::min<int64_t>(capacity, *count); ++k) local_ids[k] = o[static_cast<size_t>(k)];
  return PBDR_OK;
}

int pbdr_gpu_slab_info(pbdr_handle* h, int64_t out[6]) {
  if (!h || !h->slab_driver || !out) return pbdr_host::set_error(PBDR_ERR_GENERIC, "no slab driver attached");
  const SlabDriver& d = *h->slab_driver;
  int64_t owned_particles = 0, ghosts = 0;
  for (const int32_t b : d.owned) owned_particles += h->h_bcount[b];
  for (const auto& kv : d.P) ghosts += static_cast<int64_t>(kv.second.recv_bodies.size());
  out[0] = static_cast<int64_t>(d.owned.size());
  out[1] = owned_particles;
  out[2] = ghosts;
  out[3] = d.halo_bytes_iter;
  out[4] = d.migrations;
  out[5] = d.frames_done;
  return PBDR_OK;
}

}  // extern "C"
