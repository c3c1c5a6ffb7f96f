// Device-resident training loop of the model harness (reference
// model.cpp:154-263; paper §3.2): Dense(20 -> d) -> act -> signature ->
// Dense(D -> 10), MSE, SGD, every step on the GPU in fp64. Data and
// parameters stay in device memory for the whole run; each step reads back
// only its loss (8 bytes) for the epoch mean and the non-finite check.
// Reductions run in a fixed order (one block per output, tree over a fixed
// thread mapping), so a run is deterministic.
#include <cmath>
#include <cstdint>
#include <vector>

#include "sigk.h"

namespace sigk {
namespace model {

constexpr int kIn = 20, kOut = 10, kT = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
    const int t = threadIdx.x;
    sh[t] = v;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (t < o) sh[t] += sh[t + o];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

// z[r, j] = act(b1[j] + Σ_i X[r, i] W1[i, j]), r over batch*len rows
__global__ void dense_in(const double* __restrict__ X, const double* __restrict__ W1, const double* __restrict__ b1,
                         double* __restrict__ z, int64_t rows, int d, int tanh_act) {
    const int64_t n = rows * d;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = q / d;
        const int j = (int)(q - r * d);
        double v = b1[j];
        for (int i = 0; i < kIn; ++i) v += X[r * kIn + i] * W1[i * d + j];
        z[q] = tanh_act ? tanh(v) : v;
    }
}

// y[b, o] = b2[o] + Σ_k s[b, k] W2[k, o]
__global__ void dense_out(const double* __restrict__ s, const double* __restrict__ W2, const double* __restrict__ b2,
                          double* __restrict__ y, int B, int D) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < B * kOut; q += gridDim.x * blockDim.x) {
        const int b = q / kOut, o = q - b * kOut;
        double v = b2[o];
        for (int k = 0; k < D; ++k) v += s[(int64_t)b * D + k] * W2[k * kOut + o];
        y[q] = v;
    }
}

// gy = 2 (y - Y) / (B*10); loss = mean squared error (one block)
__global__ void loss_grad(const double* __restrict__ y, const double* __restrict__ Y, double* __restrict__ gy,
                          double* __restrict__ loss, int n) {
    __shared__ double sh[kT];
    const double scale = 1.0 / (double)n;
    double acc = 0.0;
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
        const double diff = y[q] - Y[q];
        acc += diff * diff * scale;
        gy[q] = 2.0 * diff * scale;
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) *loss = t;
}

// output layer backward: gw2[k, o] = Σ_b s[b, k] gy[b, o], gb2[o] = Σ_b gy[b, o] (grid over
// D*10 + 10 outputs), and the signature cotangent gs[b, k] = Σ_o gy[b, o] W2[k, o]
__global__ void out_grads(const double* __restrict__ s, const double* __restrict__ gy, int B, int D,
                          double* __restrict__ gw2, double* __restrict__ gb2) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < D * kOut + kOut; q += gridDim.x * blockDim.x) {
        double v = 0.0;
        if (q < D * kOut) {
            const int k = q / kOut, o = q - k * kOut;
            for (int b = 0; b < B; ++b) v += s[(int64_t)b * D + k] * gy[b * kOut + o];
            gw2[q] = v;
        } else {
            const int o = q - D * kOut;
            for (int b = 0; b < B; ++b) v += gy[b * kOut + o];
            gb2[o] = v;
        }
    }
}
__global__ void sig_cotangent(const double* __restrict__ gy, const double* __restrict__ W2, int B, int D,
                              double* __restrict__ gs) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < B * D; q += gridDim.x * blockDim.x) {
        const int b = q / D, k = q - b * D;
        double v = 0.0;
        for (int o = 0; o < kOut; ++o) v += gy[b * kOut + o] * W2[k * kOut + o];
        gs[q] = v;
    }
}

// input layer backward, one block per output (i, j) of gw1 and per j of gb1:
// Σ over rows of X[r, i] * gz[r, j] * act'(z[r, j])
__global__ void in_grads(const double* __restrict__ X, const double* __restrict__ z, const double* __restrict__ gz,
                         int64_t rows, int d, int tanh_act, double* __restrict__ gw1, double* __restrict__ gb1) {
    __shared__ double sh[kT];
    const int out = blockIdx.x;  // [0, 20*d): gw1; [20*d, 21*d): gb1
    const bool w = out < kIn * d;
    const int i = w ? out / d : -1, j = w ? out - (out / d) * d : out - kIn * d;
    double acc = 0.0;
    for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) {
        const double zz = z[r * d + j];
        const double g = gz[r * d + j] * (tanh_act ? 1.0 - zz * zz : 1.0);
        acc += w ? X[r * kIn + i] * g : g;
    }
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) (w ? gw1 : gb1)[w ? out : j] = t;
}

__global__ void sgd(double* __restrict__ p, const double* __restrict__ g, double lr, int n) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) p[q] -= lr * g[q];
}

}  // namespace model
}  // namespace sigk

// Device-resident training state: data and parameters uploaded once; one
// call per epoch (so the caller keeps per-epoch timing and callbacks);
// parameters copied back when the run ends.
struct SigkTrainCtx {
    double* m = nullptr;
    cudaStream_t s = nullptr;
    size_t n_samples = 0, seq_len = 0, D = 0, bmax = 0;
    int d = 0, depth = 0, tanh_act = 1;
    int parallel = 0;  // KernelKind resolved to Parallel: the per-degree scan formulation (model.cpp:57)
    double *dX, *dY, *dW1, *db1, *dW2, *db2, *gW1, *gb1, *gW2, *gb2, *z, *gz, *sg, *gs, *y, *gy, *loss;
};

extern "C" int sigk_internal_train_open(const double* X, const double* Y, size_t n_samples, size_t seq_len, int d,
                                        int depth, size_t bmax, int tanh_act, const double* W1, const double* b1,
                                        const double* W2, const double* b2, SigkTrainCtx** out) {
    using namespace sigk::model;
    SigkTrainCtx* c = new SigkTrainCtx();
    c->n_samples = n_samples;
    c->seq_len = seq_len;
    c->d = d;
    c->depth = depth;
    c->bmax = bmax;
    c->tanh_act = tanh_act;
    if (sigk_sig_dim(d, depth, &c->D) != SIGK_OK) {
        delete c;
        return SIGK_EDOMAIN;
    }
    const size_t D = c->D, xin = n_samples * seq_len * kIn, yin = n_samples * kOut, zsz = bmax * seq_len * d;
    const size_t nW1 = kIn * (size_t)d, nW2 = D * kOut;
    const size_t total = xin + yin + 2 * (nW1 + d + nW2 + kOut) + 2 * zsz + 2 * bmax * D + 2 * bmax * kOut + 1;
    cudaError_t e = cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&c->m, total * sizeof(double));
    if (e != cudaSuccess) {
        if (c->s) cudaStreamDestroy(c->s);
        delete c;
        return e == cudaErrorMemoryAllocation ? SIGK_ERESOURCE : SIGK_EDEVICE;
    }
    c->dX = c->m;
    c->dY = c->dX + xin;
    c->dW1 = c->dY + yin;
    c->db1 = c->dW1 + nW1;
    c->dW2 = c->db1 + d;
    c->db2 = c->dW2 + nW2;
    c->gW1 = c->db2 + kOut;
    c->gb1 = c->gW1 + nW1;
    c->gW2 = c->gb1 + d;
    c->gb2 = c->gW2 + nW2;
    c->z = c->gb2 + kOut;
    c->gz = c->z + zsz;
    c->sg = c->gz + zsz;
    c->gs = c->sg + bmax * D;
    c->y = c->gs + bmax * D;
    c->gy = c->y + bmax * kOut;
    c->loss = c->gy + bmax * kOut;
    cudaMemcpyAsync(c->dX, X, xin * 8, cudaMemcpyHostToDevice, c->s);
    cudaMemcpyAsync(c->dY, Y, yin * 8, cudaMemcpyHostToDevice, c->s);
    cudaMemcpyAsync(c->dW1, W1, nW1 * 8, cudaMemcpyHostToDevice, c->s);
    cudaMemcpyAsync(c->db1, b1, d * 8, cudaMemcpyHostToDevice, c->s);
    cudaMemcpyAsync(c->dW2, W2, nW2 * 8, cudaMemcpyHostToDevice, c->s);
    cudaMemcpyAsync(c->db2, b2, kOut * 8, cudaMemcpyHostToDevice, c->s);
    *out = c;
    return cudaStreamSynchronize(c->s) == cudaSuccess ? SIGK_OK : SIGK_EDEVICE;
}

// One epoch over the given mini-batch sizes; step_losses[i] = loss of batch i
// (measured before its update). SIGK_ETRAINING at the first non-finite loss.
extern "C" int sigk_internal_train_epoch(SigkTrainCtx* c, const size_t* batches, int n_batches, double lr,
                                         double* step_losses) {
    using namespace sigk::model;
    const unsigned G = 148 * 4;
    const size_t D = c->D, nW1 = kIn * (size_t)c->d, nW2 = D * kOut;
    const int d = c->d;
    cudaStream_t s = c->s;
    size_t at = 0;
    for (int bi = 0; bi < n_batches; ++bi) {
        const size_t B = batches[bi];
        const int64_t rows = (int64_t)(B * c->seq_len);
        const double* Xb = c->dX + at * c->seq_len * kIn;
        const double* Yb = c->dY + at * kOut;
        dense_in<<<G, kT, 0, s>>>(Xb, c->dW1, c->db1, c->z, rows, d, c->tanh_act);
        int rc = c->parallel ? sigk_signature_parallel_f64(c->z, B, c->seq_len, d, c->depth, c->sg, size_t(1) << 31,
                                                           SIGK_X_ON_DEVICE | SIGK_OUT_ON_DEVICE, s, nullptr)
                             : sigk_signature_f64(c->z, B, c->seq_len, d, c->depth, c->sg,
                                                  SIGK_X_ON_DEVICE | SIGK_OUT_ON_DEVICE, s, nullptr, nullptr);
        if (rc != SIGK_OK) return rc;
        dense_out<<<G, kT, 0, s>>>(c->sg, c->dW2, c->db2, c->y, (int)B, (int)D);
        loss_grad<<<1, kT, 0, s>>>(c->y, Yb, c->gy, c->loss, (int)(B * kOut));
        out_grads<<<G, kT, 0, s>>>(c->sg, c->gy, (int)B, (int)D, c->gW2, c->gb2);
        sig_cotangent<<<G, kT, 0, s>>>(c->gy, c->dW2, (int)B, (int)D, c->gs);
        rc = sigk_signature_vjp_f64(c->z, B, c->seq_len, d, c->depth, c->gs, c->gz, SIGK_X_ON_DEVICE, s, nullptr,
                                    nullptr);
        if (rc != SIGK_OK) return rc;
        in_grads<<<(unsigned)(kIn * d + d), kT, 0, s>>>(Xb, c->z, c->gz, rows, d, c->tanh_act, c->gW1, c->gb1);
        sgd<<<G, kT, 0, s>>>(c->dW1, c->gW1, lr, (int)nW1);
        sgd<<<1, kT, 0, s>>>(c->db1, c->gb1, lr, d);
        sgd<<<G, kT, 0, s>>>(c->dW2, c->gW2, lr, (int)nW2);
        sgd<<<1, kT, 0, s>>>(c->db2, c->gb2, lr, kOut);
        cudaMemcpyAsync(step_losses + bi, c->loss, 8, cudaMemcpyDeviceToHost, s);
        if (cudaStreamSynchronize(s) != cudaSuccess) return SIGK_EDEVICE;
        if (!std::isfinite(step_losses[bi])) return SIGK_ETRAINING;
        at += B;
    }
    return SIGK_OK;
}

// The forward kernel kind of the signature layer (the model's KernelKind after select_kernel).
extern "C" void sigk_internal_train_set_parallel(SigkTrainCtx* c, int parallel) { c->parallel = parallel; }

// Copies the parameters back and releases the device state.
extern "C" int sigk_internal_train_close(SigkTrainCtx* c, double* W1, double* b1, double* W2, double* b2) {
    using namespace sigk::model;
    int rc = SIGK_OK;
    if (W1) {
        const size_t nW1 = kIn * (size_t)c->d, nW2 = c->D * kOut;
        cudaMemcpyAsync(W1, c->dW1, nW1 * 8, cudaMemcpyDeviceToHost, c->s);
        cudaMemcpyAsync(b1, c->db1, c->d * 8, cudaMemcpyDeviceToHost, c->s);
        cudaMemcpyAsync(W2, c->dW2, nW2 * 8, cudaMemcpyDeviceToHost, c->s);
        cudaMemcpyAsync(b2, c->db2, kOut * 8, cudaMemcpyDeviceToHost, c->s);
        if (cudaStreamSynchronize(c->s) != cudaSuccess) rc = SIGK_EDEVICE;
    }
    cudaFree(c->m);
    cudaStreamDestroy(c->s);
    delete c;
    return rc;
}
