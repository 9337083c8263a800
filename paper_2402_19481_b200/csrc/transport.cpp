// Context exchange between bands.
//
//  * InProcTransport: all bands live in this process (one or several CUDA devices).
//    Each band pushes its rows on its own comm stream after waiting for the sender's
//    and the receivers' `ready` events (the receivers' event orders the write after
//    their previous-step reads of the same parity buffer).  Consumers wait on every
//    sender's `sent` event of the parity they read.
//  * NcclTransport: one band per process (torchrun / one rank per GPU).  Halos are
//    ncclSend/ncclRecv pairs with the two neighbours, K/V and GroupNorm statistics are
//    in-place ncclAllGather, all on the comm stream; consumers wait on its event.
//  * IpcTransport: one band per process, no NCCL on the data path (SURVEY.md §8f row 3:
//    copy-engine transport).  Every rank exports CUDA IPC handles of its receive buffers
//    (halo rows, K/V map, GroupNorm statistics, the full-image gather buffer) and of a flag
//    array; the sender PUSHES its rows with cudaMemcpyAsync on its comm stream (copy engines
//    over NVLink / NVSwitch, no SM time) and orders them with stream memory operations on the
//    flags (cuStreamWriteValue32 into the peer's flag after the copies -- the write carries a
//    memory fence -- and cuStreamWaitValue32 GEQ on the local flag), so no host round trip
//    and no SM polls.  Per layer and per peer two monotone counters: READY (the peer's compute
//    stream reached this exchange, so it finished reading the parity buffer about to be
//    overwritten -- the same ordering the in-process transport takes from the receivers'
//    `ready` events) and ARRIVED (the peer's rows for exchange k have landed).  The counters
//    restart at zero in every runner call: epoch_end (a two-phase flag barrier at the end of
//    the call) resets them once no peer can still write them, so the flag values a call uses
//    depend only on its exchange sequence and a captured CUDA graph replays them unchanged.
// All replace CollectiveHub (proj/src/collectives.cpp:62-232).
#include "program.hpp"
#include "util.hpp"

#include <cuda.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>

namespace pp {

namespace {

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int d) {
        CUDA_CHECK(cudaGetDevice(&prev));
        if (prev != d) CUDA_CHECK(cudaSetDevice(d));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

#define NCCL_CHECK(x)                                                                    \
    do {                                                                                 \
        ncclResult_t r_ = (x);                                                           \
        if (r_ != ncclSuccess)                                                           \
            throw NcclError(std::string("NCCL error '") + ncclGetErrorString(r_) + "' (" #x ")"); \
    } while (0)

// All bands in this process, on one device.  An exchange (one layer of a synchronous step, or
// a displaced step's batch of layers) is ONE copy kernel on band 0's comm stream that moves
// every band's halo rows / K/V band / GroupNorm statistics into the receivers' parity buffers,
// after every band's ready event (the receivers' event orders the writes after their previous
// reads of the same parity buffer); each band's sent[l][par] is recorded behind it.  The chunk
// tables are built once per (batch, parity) and stay on the device, so the exchange is
// graph-capturable and costs one kernel node.
class InProcTransport final : public Transport {
public:
    explicit InProcTransport(std::vector<Program*> b) : bands_(std::move(b)) {}
    ~InProcTransport() override {
        DeviceGuard g(bands_[0]->dev);
        cudaStreamSynchronize(bands_[0]->xs);
        for (auto& kv : tables_) cudaFree(kv.second.first);
    }

    void halo(int l, int par, bool top_only) override { batch({XItem{l, XItem::HALO, top_only}}, par); }
    void kv(int l, int par) override { batch({XItem{l, XItem::KV, false}}, par); }
    void stats(int l, int par) override { batch({XItem{l, XItem::STATS, false}}, par); }

    void prepare(const std::vector<std::vector<XItem>>& exchanges) override {
        DeviceGuard g(bands_[0]->dev);
        for (const auto& items : exchanges)
            for (int par = 0; par < 2; ++par) table(items, par);
    }

    void batch(const std::vector<XItem>& items, int par) override {
        if (items.empty()) return;
        Program& s0 = *bands_[0];
        DeviceGuard g(s0.dev);
        int lmax = 0;
        for (const XItem& it : items) lmax = std::max(lmax, it.layer);
        for (Program* o : bands_) CUDA_CHECK(cudaStreamWaitEvent(s0.xs, o->ready[lmax], 0));
        const auto& t = table(items, par);
        copy_chunks(t.first, t.second, s0.xs);
        for (const XItem& it : items)
            for (Program* o : bands_) CUDA_CHECK(cudaEventRecord(o->sent[it.layer][par], s0.xs));
    }

    void wait(Program& b, int l, int par) override {
        // every band's sent event of this exchange is recorded at the same point of one stream
        CUDA_CHECK(cudaStreamWaitEvent(b.cs, bands_[0]->sent[l][par], 0));
    }

    void gather_floats(Program&, const float*, float*, size_t) override {
        throw std::logic_error("gather_floats: not used in-process");
    }

private:
    using Table = std::pair<CopyChunk*, int>;
    const Table& table(const std::vector<XItem>& items, int par) {
        std::vector<int> key{par};
        for (const XItem& it : items) key.insert(key.end(), {it.layer, it.kind, int(it.top_only)});
        auto f = tables_.find(key);
        if (f != tables_.end()) return f->second;
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        CUDA_CHECK(cudaStreamIsCapturing(bands_[0]->xs, &cap));
        if (cap != cudaStreamCaptureStatusNone)
            throw std::logic_error("in-process transport: exchange not announced by prepare()");
        std::vector<CopyChunk> ch;
        auto add = [&](const void* src, void* dst, size_t bytes) {
            for (size_t off = 0; off < bytes; off += kChunk)
                ch.push_back(CopyChunk{static_cast<const char*>(src) + off, static_cast<char*>(dst) + off,
                                       (unsigned long long)std::min(kChunk, bytes - off)});
        };
        const int n = int(bands_.size());
        for (const XItem& it : items) {
            const int l = it.layer;
            for (int e = 0; e < n; ++e) {
                Program& s = *bands_[e];
                if (it.kind == XItem::HALO) {
                    const size_t rb = s.lx[l].row_bytes;
                    const char* src = static_cast<const char*>(s.lx[l].send_rows[par]);
                    if (e + 1 < n)   // my last row is the row above band e+1
                        add(src + rb, bands_[e + 1]->lx[l].halo_recv[par], rb);
                    if (e > 0 && !it.top_only)   // my first row is the row below band e-1
                        add(src, static_cast<char*>(bands_[e - 1]->lx[l].halo_recv[par]) + rb, rb);
                } else {
                    const size_t bb = it.kind == XItem::KV ? s.lx[l].band_bytes
                                                           : size_t(s.lx[l].G) * 2 * sizeof(double);
                    auto buf = [&](Program& p) -> char* {
                        return it.kind == XItem::KV ? static_cast<char*>(p.lx[l].kv[par])
                                                    : reinterpret_cast<char*>(p.lx[l].stats[par]);
                    };
                    for (int d = 0; d < n; ++d)
                        if (d != e) add(buf(s) + size_t(e) * bb, buf(*bands_[d]) + size_t(e) * bb, bb);
                }
            }
        }
        CopyChunk* dev = nullptr;
        CUDA_CHECK(cudaMalloc(&dev, std::max<size_t>(ch.size(), 1) * sizeof(CopyChunk)));
        // ordered before the copy kernels on the comm stream (a legacy-stream copy is not)
        CUDA_CHECK(cudaMemcpyAsync(dev, ch.data(), ch.size() * sizeof(CopyChunk), cudaMemcpyHostToDevice,
                                   bands_[0]->xs));
        return tables_.emplace(key, Table{dev, int(ch.size())}).first->second;
    }

    static constexpr size_t kChunk = size_t(64) << 10;
    std::vector<Program*> bands_;
    std::map<std::vector<int>, Table> tables_;
};

class NcclTransport final : public Transport {
public:
    NcclTransport(Program* b, int world, int rank, const std::vector<uint8_t>& id)
        : b_(b), world_(world), rank_(rank) {
        if (id.size() != sizeof(ncclUniqueId))
            throw std::invalid_argument("NCCL transport needs the 128-byte ncclUniqueId");
        ncclUniqueId uid;
        std::memcpy(&uid, id.data(), sizeof(uid));
        DeviceGuard g(b->dev);
        NCCL_CHECK(ncclCommInitRank(&comm_, world, uid, rank));
    }
    ~NcclTransport() override {
        if (comm_) {
            DeviceGuard g(b_->dev);
            cudaStreamSynchronize(b_->xs);
            ncclCommDestroy(comm_);
        }
    }

    void halo(int l, int par, bool top_only) override {
        batch({XItem{l, XItem::HALO, top_only}}, par);
    }
    void kv(int l, int par) override { batch({XItem{l, XItem::KV, false}}, par); }
    void stats(int l, int par) override { batch({XItem{l, XItem::STATS, false}}, par); }

    // Every item of the batch in ONE NCCL group (one kernel on the comm stream): halo rows as
    // send/recv with the two neighbours, K/V bands and GroupNorm statistics as in-place
    // all-gathers.
    void batch(const std::vector<XItem>& items, int par) override {
        if (items.empty()) return;
        Program& s = *b_;
        DeviceGuard g(s.dev);
        int lmax = 0;
        for (const XItem& it : items) lmax = std::max(lmax, it.layer);
        CUDA_CHECK(cudaStreamWaitEvent(s.xs, s.ready[lmax], 0));   // cs order: every item packed
        NCCL_CHECK(ncclGroupStart());
        for (const XItem& it : items) {
            const int l = it.layer;
            if (it.kind == XItem::HALO) {
                const size_t rb = s.lx[l].row_bytes;
                char* send = static_cast<char*>(s.lx[l].send_rows[par]);
                char* recv = static_cast<char*>(s.lx[l].halo_recv[par]);
                if (rank_ > 0) {
                    NCCL_CHECK(ncclRecv(recv, rb, ncclUint8, rank_ - 1, comm_, s.xs));
                    if (!it.top_only) NCCL_CHECK(ncclSend(send, rb, ncclUint8, rank_ - 1, comm_, s.xs));
                }
                if (rank_ + 1 < world_) {
                    NCCL_CHECK(ncclSend(send + rb, rb, ncclUint8, rank_ + 1, comm_, s.xs));
                    if (!it.top_only) NCCL_CHECK(ncclRecv(recv + rb, rb, ncclUint8, rank_ + 1, comm_, s.xs));
                }
            } else if (it.kind == XItem::KV) {
                const size_t bb = s.lx[l].band_bytes;
                char* buf = static_cast<char*>(s.lx[l].kv[par]);
                NCCL_CHECK(ncclAllGather(buf + size_t(rank_) * bb, buf, bb, ncclUint8, comm_, s.xs));
            } else {
                const size_t cnt = size_t(s.lx[l].G) * 2;
                double* buf = s.lx[l].stats[par];
                NCCL_CHECK(ncclAllGather(buf + size_t(rank_) * cnt, buf, cnt, ncclFloat64, comm_, s.xs));
            }
        }
        NCCL_CHECK(ncclGroupEnd());
        for (const XItem& it : items) CUDA_CHECK(cudaEventRecord(s.sent[it.layer][par], s.xs));
    }

    void wait(Program& b, int l, int par) override {
        CUDA_CHECK(cudaStreamWaitEvent(b.cs, b.sent[l][par], 0));
    }

    void gather_floats(Program& b, const float* send, float* recv, size_t count) override {
        // One communicator, one stream: the gather runs on the comm stream after every
        // exchange already queued there (a displaced step leaves its posts in flight), and
        // the compute stream waits for it.  Two NCCL operations of one communicator never
        // run concurrently on different streams.
        DeviceGuard g(b.dev);
        CUDA_CHECK(cudaEventRecord(b.gather_ev, b.cs));
        CUDA_CHECK(cudaStreamWaitEvent(b.xs, b.gather_ev, 0));
        NCCL_CHECK(ncclAllGather(send, recv, count, ncclFloat32, comm_, b.xs));
        CUDA_CHECK(cudaEventRecord(b.gather_ev, b.xs));
        CUDA_CHECK(cudaStreamWaitEvent(b.cs, b.gather_ev, 0));
    }

private:
    Program* b_;
    int world_, rank_;
    ncclComm_t comm_ = nullptr;
};

// ---------------------------------------------------------------- IPC (copy-engine) transport
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <class F>
F driver_fn(const char* name) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CUDA_CHECK(cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
        throw std::runtime_error(std::string("IPC transport: driver entry point ") + name + " unavailable");
    return reinterpret_cast<F>(fn);
}

constexpr uint32_t kIpcMagic = 0x50504331u;   // "PPC1"

class IpcTransport final : public Transport {
public:
    // flags layout (uint32): [READY][L][world], [ARRIVED][L][world], [GREADY][world], [GARRIVED][world]
    IpcTransport(Program* b, int world, int rank) : b_(b), world_(world), rank_(rank) {
        L_ = int(b->lx.size());
        DeviceGuard g(b->dev);
        n_flags_ = size_t(2 * L_ + 2) * world_;
        flags_ = static_cast<uint32_t*>(b->alloc(n_flags_ * 4));
        wait_ = driver_fn<WaitValueFn>("cuStreamWaitValue32");
        write_ = driver_fn<WriteValueFn>("cuStreamWriteValue32");
        CUDA_CHECK(cudaEventCreateWithFlags(&xs_done_, cudaEventDisableTiming));
        seq_.assign(L_, 0);
        last_.assign(L_, {0u, 0u});
        senders_.assign(L_, {});
        peers_.resize(world_);
    }
    ~IpcTransport() override {
        DeviceGuard g(b_->dev);
        cudaStreamSynchronize(b_->xs);
        cudaStreamSynchronize(b_->cs);
        for (void* p : opened_) cudaIpcCloseMemHandle(p);
        cudaEventDestroy(xs_done_);
    }

    // the receive buffers a peer pushes into, in a fixed order all ranks agree on
    std::vector<void*> exported() const {
        std::vector<void*> v;
        for (int l = 0; l < L_; ++l) {
            const auto& x = b_->lx[l];
            for (int p = 0; p < 2; ++p) {
                if (x.halo_recv[p]) v.push_back(x.halo_recv[p]);
                if (x.kv[p]) v.push_back(x.kv[p]);
                if (x.stats[p]) v.push_back(x.stats[p]);
            }
        }
        v.push_back(b_->x_full);
        v.push_back(flags_);
        return v;
    }

    std::vector<uint8_t> export_blob() const {
        const auto bufs = exported();
        std::vector<uint8_t> out(16 + bufs.size() * sizeof(cudaIpcMemHandle_t));
        const uint32_t hdr[4] = {kIpcMagic, uint32_t(rank_), uint32_t(world_), uint32_t(bufs.size())};
        std::memcpy(out.data(), hdr, 16);
        DeviceGuard g(b_->dev);
        for (size_t i = 0; i < bufs.size(); ++i) {
            cudaIpcMemHandle_t h;
            CUDA_CHECK(cudaIpcGetMemHandle(&h, bufs[i]));
            std::memcpy(out.data() + 16 + i * sizeof(h), &h, sizeof(h));
        }
        return out;
    }

    void connect(const uint8_t* blobs, size_t per_rank) {
        const size_t nb = exported().size();
        if (per_rank != 16 + nb * sizeof(cudaIpcMemHandle_t))
            throw std::invalid_argument("pp_runner_ipc_connect: handle blob size mismatch");
        DeviceGuard g(b_->dev);
        for (int r = 0; r < world_; ++r) {
            const uint8_t* blob = blobs + size_t(r) * per_rank;
            uint32_t hdr[4];
            std::memcpy(hdr, blob, 16);
            if (hdr[0] != kIpcMagic || hdr[1] != uint32_t(r) || hdr[2] != uint32_t(world_) || hdr[3] != nb)
                throw std::invalid_argument("pp_runner_ipc_connect: blob " + std::to_string(r) +
                                            " is not rank " + std::to_string(r) + "'s handle set");
            if (r == rank_) continue;
            auto& v = peers_[r];
            v.resize(nb);
            for (size_t i = 0; i < nb; ++i) {
                cudaIpcMemHandle_t h;
                std::memcpy(&h, blob + 16 + i * sizeof(h), sizeof(h));
                CUDA_CHECK(cudaIpcOpenMemHandle(&v[i], h, cudaIpcMemLazyEnablePeerAccess));
                opened_.push_back(v[i]);
            }
        }
        // index of each layer's buffers in the exported order
        idx_.assign(L_, {});
        size_t k = 0;
        for (int l = 0; l < L_; ++l) {
            const auto& x = b_->lx[l];
            for (int p = 0; p < 2; ++p) {
                if (x.halo_recv[p]) idx_[l][p] = k++;
                if (x.kv[p]) idx_[l][p] = k++;
                if (x.stats[p]) idx_[l][p] = k++;
            }
        }
        connected_ = true;
    }

    void halo(int l, int par, bool top_only) override {
        std::vector<std::pair<int, std::pair<size_t, size_t>>> out;   // peer, (src off, dst off)
        const size_t rb = b_->lx[l].row_bytes;
        if (rank_ + 1 < world_) out.push_back({rank_ + 1, {rb, 0}});   // last row -> row above e+1
        if (rank_ > 0 && !top_only) out.push_back({rank_ - 1, {0, rb}});
        std::vector<int> from;
        if (rank_ > 0) from.push_back(rank_ - 1);
        if (rank_ + 1 < world_ && !top_only) from.push_back(rank_ + 1);
        push(l, par, out, rb, static_cast<const char*>(b_->lx[l].send_rows[par]), from);
    }

    void kv(int l, int par) override {
        const size_t bb = b_->lx[l].band_bytes;
        std::vector<std::pair<int, std::pair<size_t, size_t>>> out;
        std::vector<int> from;
        for (int d = 0; d < world_; ++d)
            if (d != rank_) {
                out.push_back({d, {size_t(rank_) * bb, size_t(rank_) * bb}});
                from.push_back(d);
            }
        push(l, par, out, bb, static_cast<const char*>(b_->lx[l].kv[par]), from);
    }

    void stats(int l, int par) override {
        const size_t eb = size_t(b_->lx[l].G) * 2 * sizeof(double);
        std::vector<std::pair<int, std::pair<size_t, size_t>>> out;
        std::vector<int> from;
        for (int d = 0; d < world_; ++d)
            if (d != rank_) {
                out.push_back({d, {size_t(rank_) * eb, size_t(rank_) * eb}});
                from.push_back(d);
            }
        push(l, par, out, eb, reinterpret_cast<const char*>(b_->lx[l].stats[par]), from);
    }

    void wait(Program& b, int l, int par) override {
        const uint32_t k = last_[l][par];
        if (k == 0) return;   // nothing exchanged into this parity yet
        for (int p : senders_[l]) wait_ge(b.cs, flag(ARRIVED, l, p), k);
        // this rank's own pushes out of the parity buffers must also be complete before the
        // compute stream overwrites them (scatter_kv rewrites the own slot of kv[par])
        CUDA_CHECK(cudaStreamWaitEvent(b.cs, b.sent[l][par], 0));
    }

    void gather_floats(Program& b, const float* send, float* recv, size_t count) override {
        need_connected();
        if (recv != b.x_full) throw std::logic_error("IPC gather_floats: recv must be the band's x_full");
        const uint32_t k = ++gseq_;
        DeviceGuard g(b.dev);
        for (int p = 0; p < world_; ++p)
            if (p != rank_) write(b.cs, peer_flag(p, GREADY, 0, rank_), k);
        for (int p = 0; p < world_; ++p)
            if (p != rank_) wait_ge(b.cs, flag(GREADY, 0, p), k);
        const size_t off = size_t(rank_) * count;
        CUDA_CHECK(cudaMemcpyAsync(recv + off, send, count * 4, cudaMemcpyDeviceToDevice, b.cs));
        const size_t xi = peers_idx_x_full();
        for (int p = 0; p < world_; ++p)
            if (p != rank_)
                CUDA_CHECK(cudaMemcpyAsync(static_cast<float*>(peers_[p][xi]) + off, send, count * 4,
                                           cudaMemcpyDeviceToDevice, b.cs));
        for (int p = 0; p < world_; ++p)
            if (p != rank_) write(b.cs, peer_flag(p, GARRIVED, 0, rank_), k);
        for (int p = 0; p < world_; ++p)
            if (p != rank_) wait_ge(b.cs, flag(GARRIVED, 0, p), k);
    }

    // Phase 1: every rank's pushes of this call have completed (its comm stream joined into
    // the compute stream before it signals), so nothing more lands in our flags or buffers;
    // reset the per-layer counters.  Phase 2: every rank has reset, so the next call's first
    // READY / ARRIVED writes cannot be clobbered by a late reset.  Data exchanged in this call
    // and read by the next (displaced steps through the step API) has landed by phase 1, so
    // the next call's first wait of each (layer, parity) is a no-op (last_ = 0).
    void epoch_end(Program& b) override {
        need_connected();
        DeviceGuard g(b.dev);
        CUDA_CHECK(cudaEventRecord(xs_done_, b.xs));
        CUDA_CHECK(cudaStreamWaitEvent(b.cs, xs_done_, 0));
        const uint32_t k = ++gseq_;
        for (int p = 0; p < world_; ++p)
            if (p != rank_) write(b.cs, peer_flag(p, GREADY, 0, rank_), k);
        for (int p = 0; p < world_; ++p)
            if (p != rank_) wait_ge(b.cs, flag(GREADY, 0, p), k);
        CUDA_CHECK(cudaMemsetAsync(flags_, 0, size_t(2) * L_ * world_ * 4, b.cs));
        for (int p = 0; p < world_; ++p)
            if (p != rank_) write(b.cs, peer_flag(p, GARRIVED, 0, rank_), k);
        for (int p = 0; p < world_; ++p)
            if (p != rank_) wait_ge(b.cs, flag(GARRIVED, 0, p), k);
        std::fill(seq_.begin(), seq_.end(), 0u);
        for (auto& a : last_) a = {0u, 0u};
    }

private:
    enum { READY = 0, ARRIVED = 1, GREADY = 2, GARRIVED = 3 };
    size_t flag_index(int kind, int l, int p) const {
        if (kind <= ARRIVED) return (size_t(kind) * L_ + l) * world_ + p;
        return (size_t(2) * L_ + (kind - GREADY)) * world_ + p;
    }
    CUdeviceptr flag(int kind, int l, int p) const {
        return reinterpret_cast<CUdeviceptr>(flags_ + flag_index(kind, l, p));
    }
    CUdeviceptr peer_flag(int peer, int kind, int l, int p) const {
        return reinterpret_cast<CUdeviceptr>(static_cast<uint32_t*>(peers_[peer].back()) +
                                             flag_index(kind, l, p));
    }
    size_t peers_idx_x_full() const { return exported().size() - 2; }
    void need_connected() const {
        if (!connected_)
            throw std::runtime_error("IPC transport not connected (pp_runner_ipc_connect)");
    }
    void wait_ge(cudaStream_t s, CUdeviceptr a, uint32_t v) {
        const CUresult r = wait_(reinterpret_cast<CUstream>(s), a, v, CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) throw CudaError("cuStreamWaitValue32 failed (" + std::to_string(int(r)) + ")");
    }
    void write(cudaStream_t s, CUdeviceptr a, uint32_t v) {
        const CUresult r = write_(reinterpret_cast<CUstream>(s), a, v, CU_STREAM_WRITE_VALUE_DEFAULT);
        if (r != CUDA_SUCCESS) throw CudaError("cuStreamWriteValue32 failed (" + std::to_string(int(r)) + ")");
    }

    // exchange k of layer l into parity `par`: READY handshake with the receivers, copies into
    // their parity buffers, ARRIVED after the copies (the flag write is fenced behind them)
    void push(int l, int par, const std::vector<std::pair<int, std::pair<size_t, size_t>>>& out,
              size_t bytes, const char* src, const std::vector<int>& from) {
        need_connected();
        Program& s = *b_;
        DeviceGuard g(s.dev);
        const uint32_t k = ++seq_[l];
        last_[l][par] = k;
        senders_[l] = from;
        CUDA_CHECK(cudaStreamWaitEvent(s.xs, s.ready[l], 0));
        for (int p : from) write(s.xs, peer_flag(p, READY, l, rank_), k);   // I reached exchange k
        for (const auto& o : out) wait_ge(s.xs, flag(READY, l, o.first), k);
        const size_t bi = idx_[l][par];
        for (const auto& o : out)
            CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(peers_[o.first][bi]) + o.second.second,
                                       src + o.second.first, bytes, cudaMemcpyDeviceToDevice, s.xs));
        for (const auto& o : out) write(s.xs, peer_flag(o.first, ARRIVED, l, rank_), k);
        CUDA_CHECK(cudaEventRecord(s.sent[l][par], s.xs));
    }

    Program* b_;
    int world_, rank_, L_ = 0;
    uint32_t* flags_ = nullptr;
    size_t n_flags_ = 0;
    WaitValueFn wait_ = nullptr;
    WriteValueFn write_ = nullptr;
    std::vector<uint32_t> seq_;
    std::vector<std::array<uint32_t, 2>> last_;
    std::vector<std::vector<int>> senders_;
    std::vector<std::array<size_t, 2>> idx_;
    std::vector<std::vector<void*>> peers_;
    std::vector<void*> opened_;
    uint32_t gseq_ = 0;
    cudaEvent_t xs_done_ = nullptr;
    bool connected_ = false;
};

// ---------------------------------------------------------------- CFG pair links
class NcclPair final : public PairLink {
public:
    NcclPair(int dev, int role, const std::vector<uint8_t>& id, size_t n) : dev_(dev), role_(role), n_(n) {
        if (id.size() != sizeof(ncclUniqueId))
            throw std::invalid_argument("CFG pair link needs the 128-byte ncclUniqueId (cfg_nccl_id)");
        ncclUniqueId uid;
        std::memcpy(&uid, id.data(), sizeof(uid));
        DeviceGuard g(dev_);
        CUDA_CHECK(cudaMalloc(&recv_, std::max<size_t>(n_, 1) * 4));
        NCCL_CHECK(ncclCommInitRank(&comm_, 2, uid, role_));
    }
    ~NcclPair() override {
        DeviceGuard g(dev_);
        if (comm_) ncclCommDestroy(comm_);
        cudaFree(recv_);
    }
    const float* exchange(cudaStream_t s, const float* mine) override {
        DeviceGuard g(dev_);
        NCCL_CHECK(ncclGroupStart());
        NCCL_CHECK(ncclSend(mine, n_, ncclFloat32, 1 - role_, comm_, s));
        NCCL_CHECK(ncclRecv(recv_, n_, ncclFloat32, 1 - role_, comm_, s));
        NCCL_CHECK(ncclGroupEnd());
        return recv_;
    }
    bool capturable() const override { return true; }

private:
    int dev_, role_;
    size_t n_;
    float* recv_ = nullptr;
    ncclComm_t comm_ = nullptr;
};

constexpr uint32_t kPairMagic = 0x50504350u;   // "PPCP"

// One allocation: two parity receive buffers of n floats, then the flags {ARRIVED, BAR1, BAR2}.
// Exchange k lands in parity k & 1.  No READY handshake is needed: the partner's push k
// follows (in its stream) its wait for our push k-1, which follows (in ours) our read of
// exchange k-2, the last use of the same parity buffer.  ARRIVED restarts at zero in every
// runner call (epoch_end: the IpcTransport's two-phase barrier on BAR1 / BAR2), so the pair
// link is graph-capturable.
class IpcPair final : public PairLink {
public:
    IpcPair(int dev, int role, size_t n) : dev_(dev), role_(role), n_(n) {
        DeviceGuard g(dev_);
        stride_ = (std::max<size_t>(n_, 1) * 4 + 255) / 256 * 256;
        CUDA_CHECK(cudaMalloc(&buf_, 2 * stride_ + 256));
        CUDA_CHECK(cudaMemset(buf_, 0, 2 * stride_ + 256));
        wait_ = driver_fn<WaitValueFn>("cuStreamWaitValue32");
        write_ = driver_fn<WriteValueFn>("cuStreamWriteValue32");
    }
    ~IpcPair() override {
        DeviceGuard g(dev_);
        cudaDeviceSynchronize();
        if (peer_) cudaIpcCloseMemHandle(peer_);
        cudaFree(buf_);
    }
    std::vector<uint8_t> export_blob() const override {
        std::vector<uint8_t> out(32 + sizeof(cudaIpcMemHandle_t));
        const uint64_t hdr[4] = {kPairMagic, uint64_t(role_), uint64_t(n_), uint64_t(stride_)};
        std::memcpy(out.data(), hdr, 32);
        DeviceGuard g(dev_);
        cudaIpcMemHandle_t h;
        CUDA_CHECK(cudaIpcGetMemHandle(&h, buf_));
        std::memcpy(out.data() + 32, &h, sizeof(h));
        return out;
    }
    void connect(const uint8_t* blob, size_t size) override {
        if (size != 32 + sizeof(cudaIpcMemHandle_t))
            throw std::invalid_argument("pp_runner_pair_connect: handle blob size mismatch");
        uint64_t hdr[4];
        std::memcpy(hdr, blob, 32);
        if (hdr[0] != kPairMagic || hdr[1] != uint64_t(1 - role_) || hdr[2] != n_ || hdr[3] != stride_)
            throw std::invalid_argument("pp_runner_pair_connect: blob is not the partner's (role " +
                                        std::to_string(1 - role_) + ", same band shape) handle");
        if (peer_) throw std::invalid_argument("pp_runner_pair_connect: already connected");
        cudaIpcMemHandle_t h;
        std::memcpy(&h, blob + 32, sizeof(h));
        DeviceGuard g(dev_);
        CUDA_CHECK(cudaIpcOpenMemHandle(&peer_, h, cudaIpcMemLazyEnablePeerAccess));
    }
    const float* exchange(cudaStream_t s, const float* mine) override {
        if (!peer_) throw std::runtime_error("CFG pair link not connected (pp_runner_pair_connect)");
        DeviceGuard g(dev_);
        const uint32_t k = ++seq_;
        const size_t off = (k & 1) * stride_;
        CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(peer_) + off, mine, n_ * 4, cudaMemcpyDeviceToDevice, s));
        CUresult r = write_(reinterpret_cast<CUstream>(s), flag(peer_), k, CU_STREAM_WRITE_VALUE_DEFAULT);
        if (r != CUDA_SUCCESS) throw CudaError("cuStreamWriteValue32 failed (" + std::to_string(int(r)) + ")");
        r = wait_(reinterpret_cast<CUstream>(s), flag(buf_), k, CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) throw CudaError("cuStreamWaitValue32 failed (" + std::to_string(int(r)) + ")");
        return reinterpret_cast<const float*>(static_cast<char*>(buf_) + off);
    }
    bool capturable() const override { return true; }
    void epoch_end(cudaStream_t s) override {
        if (!peer_) throw std::runtime_error("CFG pair link not connected (pp_runner_pair_connect)");
        DeviceGuard g(dev_);
        const uint32_t k = ++bseq_;
        signal(s, flag(peer_, 1), k);
        await(s, flag(buf_, 1), k);
        CUDA_CHECK(cudaMemsetAsync(reinterpret_cast<void*>(flag(buf_)), 0, 4, s));
        signal(s, flag(peer_, 2), k);
        await(s, flag(buf_, 2), k);
        seq_ = 0;
    }

private:
    CUdeviceptr flag(void* base, int i = 0) const {
        return reinterpret_cast<CUdeviceptr>(static_cast<char*>(base) + 2 * stride_ + 4 * i);
    }
    void signal(cudaStream_t s, CUdeviceptr a, uint32_t v) {
        const CUresult r = write_(reinterpret_cast<CUstream>(s), a, v, CU_STREAM_WRITE_VALUE_DEFAULT);
        if (r != CUDA_SUCCESS) throw CudaError("cuStreamWriteValue32 failed (" + std::to_string(int(r)) + ")");
    }
    void await(cudaStream_t s, CUdeviceptr a, uint32_t v) {
        const CUresult r = wait_(reinterpret_cast<CUstream>(s), a, v, CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) throw CudaError("cuStreamWaitValue32 failed (" + std::to_string(int(r)) + ")");
    }
    int dev_, role_;
    size_t n_, stride_ = 0;
    void* buf_ = nullptr;
    void* peer_ = nullptr;
    uint32_t seq_ = 0, bseq_ = 0;
    WaitValueFn wait_ = nullptr;
    WriteValueFn write_ = nullptr;
};

}  // namespace

std::vector<uint8_t> PairLink::export_blob() const {
    throw std::invalid_argument("pp_runner_pair_export: the CFG pair link does not use CUDA IPC");
}
void PairLink::connect(const uint8_t*, size_t) {
    throw std::invalid_argument("pp_runner_pair_connect: the CFG pair link does not use CUDA IPC");
}

std::unique_ptr<PairLink> make_nccl_pair(int dev, int role, const std::vector<uint8_t>& id, size_t n) {
    return std::make_unique<NcclPair>(dev, role, id, n);
}

std::unique_ptr<PairLink> make_ipc_pair(int dev, int role, size_t n) {
    return std::make_unique<IpcPair>(dev, role, n);
}

std::unique_ptr<Transport> make_inproc_transport(std::vector<Program*> bands) {
    return std::make_unique<InProcTransport>(std::move(bands));
}

std::unique_ptr<Transport> make_nccl_transport(Program* band, int world, int rank,
                                               const std::vector<uint8_t>& id) {
    return std::make_unique<NcclTransport>(band, world, rank, id);
}

std::unique_ptr<Transport> make_ipc_transport(Program* band, int world, int rank) {
    return std::make_unique<IpcTransport>(band, world, rank);
}

std::vector<uint8_t> ipc_export(Transport& t) {
    auto* p = dynamic_cast<IpcTransport*>(&t);
    if (!p) throw std::invalid_argument("pp_runner_ipc_export: runner does not use the IPC transport");
    return p->export_blob();
}

void ipc_connect(Transport& t, const uint8_t* blobs, size_t per_rank) {
    auto* p = dynamic_cast<IpcTransport*>(&t);
    if (!p) throw std::invalid_argument("pp_runner_ipc_connect: runner does not use the IPC transport");
    p->connect(blobs, per_rank);
}

}  // namespace pp
