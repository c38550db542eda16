// dit_shard.cu -- one rank of the multi-GPU D-Iteration.
//
// A shard owns nodes [lo, hi) of an n_global-node graph and their out-edges.
// Targets outside [lo, hi) are renumbered to ghost slots n_local + g, g the
// rank of the target among the distinct remote targets (ascending global id,
// found with a bitmap over n_global ids and a popcount prefix sum), so the
// sweep kernels run unchanged on n_local + n_ghost fluid slots.  After a
// sweep the ghost fluid is handed to the caller's all-to-all and the fluid
// received from the other ranks is added to the owned nodes.
#include "dit_internal.cuh"

namespace dit {

__global__ void k_mark_remote(const int32_t *__restrict__ col, int64_t m, int64_t lo, int64_t hi,
                              unsigned *__restrict__ bm) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = col[e];
        if (t < lo || t >= hi) atomicOr(&bm[t >> 5], 1u << (t & 31));
    }
}

__global__ void k_word_pop(const unsigned *__restrict__ bm, int64_t nw, int64_t *__restrict__ pc) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x)
        pc[w] = __popc(bm[w]);
}

__global__ void k_remap(int32_t *__restrict__ col, int64_t m, int64_t lo, int64_t hi, const unsigned *__restrict__ bm,
                        const int64_t *__restrict__ wpre, int64_t n_local) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = col[e];
        if (t >= lo && t < hi) {
            col[e] = (int32_t)(t - lo);
        } else {
            const unsigned below = bm[t >> 5] & ((1u << (t & 31)) - 1u);
            col[e] = (int32_t)(n_local + wpre[t >> 5] + __popc(below));
        }
    }
}

__global__ void k_ghost_ids(const unsigned *__restrict__ bm, const int64_t *__restrict__ wpre, int64_t nw,
                            int32_t *__restrict__ ids) {
    for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
        unsigned bits = bm[w];
        int64_t pos = wpre[w];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            ids[pos++] = (int32_t)(w * 32 + b);
        }
    }
}

void create_shard(di_graph *h, int64_t n_global, int64_t lo, int64_t hi, int64_t m, const int64_t *row_ptr,
                  const int32_t *col, const void *weights, int w_dtype, int mem) {
    const int64_t n_local = hi - lo;
    create_graph(h, n_local, m, row_ptr, col, weights, w_dtype, mem, n_global);
    DevGraph &g = h->g;
    cudaStream_t st = h->stream;
    const int64_t nw = (n_global + 31) / 32;
    unsigned *bm = nullptr;
    int64_t *pc = nullptr, *wpre = nullptr;
    DI_CUDA(cudaMallocAsync(&bm, (nw > 0 ? nw : 1) * sizeof(unsigned), st));
    DI_CUDA(cudaMallocAsync(&pc, (nw > 0 ? nw : 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMallocAsync(&wpre, (nw + 1) * sizeof(int64_t), st));
    DI_CUDA(cudaMemsetAsync(bm, 0, (nw > 0 ? nw : 1) * sizeof(unsigned), st));
    if (m > 0) {
        k_mark_remote<<<grid_for(h, m), 256, 0, st>>>(g.col, m, lo, hi, bm);
        count_launch();
    }
    if (nw > 0) {
        k_word_pop<<<grid_for(h, nw), 256, 0, st>>>(bm, nw, pc);
        count_launch();
    }
    exclusive_scan_i64(pc, wpre, nw, st);
    int64_t n_ghost = 0;
    DI_CUDA(cudaMemcpyAsync(&n_ghost, wpre + nw, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    DI_CUDA(cudaStreamSynchronize(st));
    if (m > 0) {
        k_remap<<<grid_for(h, m), 256, 0, st>>>(g.col, m, lo, hi, bm, wpre, n_local);
        count_launch();
    }
    DI_CUDA(cudaMallocAsync(&g.ghost_ids, (n_ghost > 0 ? n_ghost : 1) * sizeof(int32_t), st));
    if (nw > 0) {
        k_ghost_ids<<<grid_for(h, nw), 256, 0, st>>>(bm, wpre, nw, g.ghost_ids);
        count_launch();
    }
    DI_CUDA(cudaFreeAsync(bm, st));
    DI_CUDA(cudaFreeAsync(pc, st));
    DI_CUDA(cudaFreeAsync(wpre, st));
    DI_CUDA(cudaGetLastError());
    DI_CUDA(cudaStreamSynchronize(st));
    g.nt = n_local + n_ghost;
    g.n_global = n_global;
    g.lo = lo;
    g.shard = true;
}

void shard_set_recv(di_graph *h, int64_t total, const int32_t *local_idx, int nseg, const int64_t *seg_counts,
                    int mem) {
    DevGraph &g = h->g;
    if (g.recv_idx) cudaFreeAsync(g.recv_idx, h->stream);
    g.recv_idx = nullptr;
    DI_CUDA(cudaMallocAsync(&g.recv_idx, (total > 0 ? total : 1) * sizeof(int32_t), h->stream));
    if (total > 0)
        DI_CUDA(cudaMemcpyAsync(g.recv_idx, local_idx, total * sizeof(int32_t),
                                mem == DI_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, h->stream));
    g.recv_seg.assign(seg_counts, seg_counts + nseg);
    DI_CUDA(cudaStreamSynchronize(h->stream));
}

// ghost fluid -> caller's send buffer; ghost slots cleared for the next sweep
__global__ void k_take_ghosts(double *__restrict__ Fg, int64_t ng, double *__restrict__ out,
                              const Ctrl *__restrict__ ctrl) {
    if (ctrl->done) return;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ng; i += (int64_t)gridDim.x * blockDim.x) {
        out[i] = Fg[i];
        Fg[i] = 0.0;
    }
}

// one source rank's segment: its ghost ids are distinct, so plain adds
__global__ void k_apply_seg(double *__restrict__ F, const int32_t *__restrict__ idx, const double *__restrict__ v,
                            int64_t cnt, const Ctrl *__restrict__ ctrl, int force) {
    if (ctrl->done && !force) return;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < cnt; q += (int64_t)gridDim.x * blockDim.x)
        F[idx[q]] += v[q];
}

__global__ void k_control(Ctrl *__restrict__ ctrl, const double *__restrict__ gathered, int nranks, int64_t m,
                          int force);

// Tiled shards: the ghost slots are the tile plan's last heavy
// group, gathered with wave 0's rule (the previous sweep's pushes).
// di_shard_sweep gathers them into the send buffer; the caller starts the
// exchange and meanwhile runs di_shard_heavy_local (wave 0's own heavy
// targets, independent of what arrives); di_shard_apply adds the received
// fluid to F (running the local gather first if the caller did not), and
// di_shard_reduce runs wave 0's tile kernel, then each later wave's heavy
// gather and tile kernel (R15, R16; local rounds, residual estimate of reading
// R13 -> stats).  The order of every sum is the one of a single group: the
// same bits as gathering the ghosts inside wave 0.
void shard_sweep(di_graph *h, double *ghost_out) {
    if (h->s.tiled_call) {
        const int64_t k = h->s.launched;
        mark_event(h, k, 0);
        if (h->g.tl.groups > h->g.tl.waves) launch_tile_heavy(h, 0, 0, h->g.tl.waves);
        launch_take_ghost_sums(h, ghost_out, 0);
        h->s.local_pending = true;
        return;
    }
    launch_sweep(h);
    const int64_t ng = h->g.nt - h->g.n;
    if (ng > 0) {
        k_take_ghosts<<<grid_for(h, ng), 256, 0, h->stream>>>(h->s.F + h->g.n, ng, ghost_out, h->s.ctrl);
        count_launch();
    }
    DI_CUDA(cudaGetLastError());
}

void shard_heavy_local(di_graph *h) {
    if (!h->s.tiled_call || !h->s.local_pending) return;
    launch_tile_heavy(h, 0, 0, 0);
    mark_event(h, h->s.launched, 1);
    h->s.local_pending = false;
}

void shard_apply(di_graph *h, const double *recv, int force) {
    if (!force) shard_heavy_local(h);
    int64_t off = 0;
    for (int64_t c : h->g.recv_seg) {   // source ranks in order: deterministic
        if (c > 0) {
            k_apply_seg<<<grid_for(h, c), 256, 0, h->stream>>>(h->s.F, h->g.recv_idx + off, recv + off, c, h->s.ctrl,
                                                               force);
            count_launch();
        }
        off += c;
    }
    DI_CUDA(cudaGetLastError());
}

void shard_reduce(di_graph *h) {
    if (h->s.tiled_call) {
        const int64_t k = h->s.launched;       // events as launch_tile_sweep: [2c] heavy(c) [2c+1] tile(c)
        launch_tile_kernel(h, h->s.rounds, 0);
        mark_event(h, k, 2);
        for (int c = 1; c < tile_waves(h); ++c) {
            launch_tile_heavy(h, 0, c);
            mark_event(h, k, 2 * c + 1);
            launch_tile_kernel(h, h->s.rounds, c);
            mark_event(h, k, 2 * c + 2);
        }
        h->s.launched += 1;
        return;
    }
    launch_sweep_reduce(h);
}

// after the last sweep: the pending pushes of the tiled schedule, exchanged like a sweep
void shard_flush(di_graph *h, double *ghost_out) {
    if (h->s.tiled_call) {
        if (h->g.tl.groups > h->g.tl.waves) launch_tile_heavy(h, 1, 0, h->g.tl.waves);
        launch_take_ghost_sums(h, ghost_out, 1);
    } else if (h->g.nt > h->g.n) {
        DI_CUDA(cudaMemsetAsync(ghost_out, 0, (h->g.nt - h->g.n) * sizeof(double), h->stream));
    }
}

void shard_flush_apply(di_graph *h, const double *recv) {
    shard_apply(h, recv, 1);
    if (h->s.tiled_call) launch_tile_flush(h);
    launch_reduce_exact(h);           // exact local |F|_1 -> stats; k_control re-derives `done`
    h->s.flushing = true;
}

void shard_control(di_graph *h, const double *gathered, int nranks, int force) {
    k_control<<<1, 32, 0, h->stream>>>(h->s.ctrl, gathered, nranks, h->g.m, force);
    count_launch();
    DI_CUDA(cudaGetLastError());
}

}  // namespace dit
