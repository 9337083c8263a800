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
// Both replace CollectiveHub (proj/src/collectives.cpp:62-232).
#include "program.hpp"
#include "util.hpp"

#include <nccl.h>

#include <cstring>
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

class InProcTransport final : public Transport {
public:
    explicit InProcTransport(std::vector<Program*> b) : bands_(std::move(b)) {
        // peer access where the hardware allows it (NVLink / NVSwitch)
        for (Program* a : bands_)
            for (Program* c : bands_) {
                if (a->dev == c->dev) continue;
                int ok = 0;
                cudaDeviceCanAccessPeer(&ok, a->dev, c->dev);
                if (ok) {
                    DeviceGuard g(a->dev);
                    const cudaError_t e = cudaDeviceEnablePeerAccess(c->dev, 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CUDA_CHECK(e);
                    cudaGetLastError();
                }
            }
    }

    void halo(int l, int par, bool top_only) override {
        const int n = int(bands_.size());
        for (int e = 0; e < n; ++e) {
            Program& s = *bands_[e];
            DeviceGuard g(s.dev);
            CUDA_CHECK(cudaStreamWaitEvent(s.xs, s.ready[l], 0));
            if (e > 0) CUDA_CHECK(cudaStreamWaitEvent(s.xs, bands_[e - 1]->ready[l], 0));
            if (e + 1 < n) CUDA_CHECK(cudaStreamWaitEvent(s.xs, bands_[e + 1]->ready[l], 0));
            const size_t rb = s.lx[l].row_bytes;
            const char* src = static_cast<const char*>(s.lx[l].send_rows[par]);
            if (e + 1 < n)  // my last row is the row above band e+1
                CUDA_CHECK(cudaMemcpyAsync(bands_[e + 1]->lx[l].halo_recv[par], src + rb, rb,
                                           cudaMemcpyDefault, s.xs));
            if (e > 0 && !top_only)  // my first row is the row below band e-1
                CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(bands_[e - 1]->lx[l].halo_recv[par]) + rb,
                                           src, rb, cudaMemcpyDefault, s.xs));
            CUDA_CHECK(cudaEventRecord(s.sent[l][par], s.xs));
        }
    }

    void kv(int l, int par) override {
        const int n = int(bands_.size());
        for (int e = 0; e < n; ++e) {
            Program& s = *bands_[e];
            DeviceGuard g(s.dev);
            for (Program* o : bands_) CUDA_CHECK(cudaStreamWaitEvent(s.xs, o->ready[l], 0));
            const size_t bb = s.lx[l].band_bytes;
            const char* src = static_cast<const char*>(s.lx[l].kv[par]) + size_t(e) * bb;
            for (int d = 0; d < n; ++d) {
                if (d == e) continue;
                CUDA_CHECK(cudaMemcpyAsync(static_cast<char*>(bands_[d]->lx[l].kv[par]) + size_t(e) * bb,
                                           src, bb, cudaMemcpyDefault, s.xs));
            }
            CUDA_CHECK(cudaEventRecord(s.sent[l][par], s.xs));
        }
    }

    void stats(int l, int par) override {
        const int n = int(bands_.size());
        for (int e = 0; e < n; ++e) {
            Program& s = *bands_[e];
            DeviceGuard g(s.dev);
            for (Program* o : bands_) CUDA_CHECK(cudaStreamWaitEvent(s.xs, o->ready[l], 0));
            const size_t eb = size_t(s.lx[l].G) * 2 * sizeof(double);
            const char* src = reinterpret_cast<const char*>(s.lx[l].stats[par]) + size_t(e) * eb;
            for (int d = 0; d < n; ++d) {
                if (d == e) continue;
                CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<char*>(bands_[d]->lx[l].stats[par]) + size_t(e) * eb,
                                           src, eb, cudaMemcpyDefault, s.xs));
            }
            CUDA_CHECK(cudaEventRecord(s.sent[l][par], s.xs));
        }
    }

    void wait(Program& b, int l, int par) override {
        for (Program* o : bands_) CUDA_CHECK(cudaStreamWaitEvent(b.cs, o->sent[l][par], 0));
    }

    void gather_floats(Program&, const float*, float*, size_t) override {
        throw std::logic_error("gather_floats: not used in-process");
    }

private:
    std::vector<Program*> bands_;
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
        Program& s = *b_;
        DeviceGuard g(s.dev);
        CUDA_CHECK(cudaStreamWaitEvent(s.xs, s.ready[l], 0));
        const size_t rb = s.lx[l].row_bytes;
        char* send = static_cast<char*>(s.lx[l].send_rows[par]);
        char* recv = static_cast<char*>(s.lx[l].halo_recv[par]);
        NCCL_CHECK(ncclGroupStart());
        if (rank_ > 0) {
            NCCL_CHECK(ncclRecv(recv, rb, ncclUint8, rank_ - 1, comm_, s.xs));
            if (!top_only) NCCL_CHECK(ncclSend(send, rb, ncclUint8, rank_ - 1, comm_, s.xs));
        }
        if (rank_ + 1 < world_) {
            NCCL_CHECK(ncclSend(send + rb, rb, ncclUint8, rank_ + 1, comm_, s.xs));
            if (!top_only) NCCL_CHECK(ncclRecv(recv + rb, rb, ncclUint8, rank_ + 1, comm_, s.xs));
        }
        NCCL_CHECK(ncclGroupEnd());
        CUDA_CHECK(cudaEventRecord(s.sent[l][par], s.xs));
    }

    void kv(int l, int par) override {
        Program& s = *b_;
        DeviceGuard g(s.dev);
        CUDA_CHECK(cudaStreamWaitEvent(s.xs, s.ready[l], 0));
        const size_t bb = s.lx[l].band_bytes;
        char* buf = static_cast<char*>(s.lx[l].kv[par]);
        NCCL_CHECK(ncclAllGather(buf + size_t(rank_) * bb, buf, bb, ncclUint8, comm_, s.xs));
        CUDA_CHECK(cudaEventRecord(s.sent[l][par], s.xs));
    }

    void stats(int l, int par) override {
        Program& s = *b_;
        DeviceGuard g(s.dev);
        CUDA_CHECK(cudaStreamWaitEvent(s.xs, s.ready[l], 0));
        const size_t cnt = size_t(s.lx[l].G) * 2;
        double* buf = s.lx[l].stats[par];
        NCCL_CHECK(ncclAllGather(buf + size_t(rank_) * cnt, buf, cnt, ncclFloat64, comm_, s.xs));
        CUDA_CHECK(cudaEventRecord(s.sent[l][par], s.xs));
    }

    void wait(Program& b, int l, int par) override {
        CUDA_CHECK(cudaStreamWaitEvent(b.cs, b.sent[l][par], 0));
    }

    void gather_floats(Program& b, const float* send, float* recv, size_t count) override {
        DeviceGuard g(b.dev);
        NCCL_CHECK(ncclAllGather(send, recv, count, ncclFloat32, comm_, b.cs));
    }

private:
    Program* b_;
    int world_, rank_;
    ncclComm_t comm_ = nullptr;
};

}  // namespace

std::unique_ptr<Transport> make_inproc_transport(std::vector<Program*> bands) {
    return std::make_unique<InProcTransport>(std::move(bands));
}

std::unique_ptr<Transport> make_nccl_transport(Program* band, int world, int rank,
                                               const std::vector<uint8_t>& id) {
    return std::make_unique<NcclTransport>(band, world, rank, id);
}

}  // namespace pp
