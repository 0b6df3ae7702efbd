"""Generator / discriminator MLPs, their gradients, the loss and Adam.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Paper: "Both networks use Leaky ReLU activation functions in the hidden
layers, together with a Kaiming normal weight initialization";
generator 51,206 and discriminator 50,049 trainable parameters;
the discriminator is "trained to label the reference data as one and the
synthetic data as zero"; learning rates 1e-5 (G) and 1e-4 (D).
Loss and optimiser are not named (R7): BCE-with-logits, the non-saturating
generator loss, and Adam(0.9, 0.999, 1e-8) in PyTorch's form.

Weights are W_l[out, in] (row-major, y = x W^T + b); the last layer is
linear.  numpy's matmul is used as the contraction primitive; nothing is
fused or reordered beyond the layer-by-layer definition.
"""
import numpy as np

from . import philox as px

LEAKY_SLOPE = 0.01


def count_params(sizes):
    """sum over layers of out*in + out."""
    return sum(sizes[i + 1] * sizes[i] + sizes[i + 1] for i in range(len(sizes) - 1))


def count_weights(sizes):
    """Weights only (the exchanged packet length)."""
    return sum(sizes[i + 1] * sizes[i] for i in range(len(sizes) - 1))


def lrelu(z, alpha=LEAKY_SLOPE):
    return np.where(z > 0.0, z, alpha * z)


def lrelu_grad(z, alpha=LEAKY_SLOPE):
    """1 for z > 0, else alpha (PyTorch's convention at 0; R6)."""
    return np.where(z > 0.0, 1.0, alpha)


def kaiming_init(seed, stream, rank, sizes, alpha=LEAKY_SLOPE):
    """W ~ N(0, 2 / ((1 + alpha^2) fan_in)) (Kaiming normal, leaky_relu gain),
    biases 0 (R-INIT).  Layer l draws its normals from counters
    (index, step=l, rank, stream)."""
    Ws, bs = [], []
    for l in range(len(sizes) - 1):
        fan_in, fan_out = sizes[l], sizes[l + 1]
        std = np.sqrt(2.0 / ((1.0 + alpha * alpha) * fan_in))
        z = px.normals(seed, stream, l, rank, fan_out * fan_in)
        Ws.append(std * z.reshape(fan_out, fan_in))
        bs.append(np.zeros(fan_out, dtype=np.float64))
    return Ws, bs


def forward(Ws, bs, x, alpha=LEAKY_SLOPE):
    """Returns (out, cache); cache = list of (input, pre-activation) per layer."""
    h = np.asarray(x, dtype=np.float64)
    cache = []
    L = len(Ws)
    for l in range(L):
        z = h @ Ws[l].T + bs[l]
        cache.append((h, z))
        h = lrelu(z, alpha) if l < L - 1 else z
    return h, cache


def backward(Ws, cache, dout, alpha=LEAKY_SLOPE):
    """Reverse-mode pass.  Returns (dWs, dbs, dx)."""
    L = len(Ws)
    dWs = [None] * L
    dbs = [None] * L
    g = np.asarray(dout, dtype=np.float64)
    for l in reversed(range(L)):
        h_in, z = cache[l]
        dz = g if l == L - 1 else g * lrelu_grad(z, alpha)
        dWs[l] = dz.T @ h_in
        dbs[l] = dz.sum(axis=0)
        g = dz @ Ws[l]
    return dWs, dbs, g


# ---------------------------------------------------------------- loss
def log_sigmoid_neg(z):
    """softplus(-z) = -log sigmoid(z), stable form max(-z,0) + log1p(e^-|z|)."""
    z = np.asarray(z, dtype=np.float64)
    return np.maximum(-z, 0.0) + np.log1p(np.exp(-np.abs(z)))


def sigmoid(z):
    """1 / (1 + e^-z), written as (1 + tanh(z/2)) / 2 (no overflow)."""
    z = np.asarray(z, dtype=np.float64)
    return 0.5 * (1.0 + np.tanh(0.5 * z))


def bce_with_logits(z, t):
    """mean of -[t log s(z) + (1-t) log(1-s(z))] = mean of t softplus(-z) +
    (1-t) softplus(z)."""
    z = np.asarray(z, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    return float(np.mean(t * log_sigmoid_neg(z) + (1.0 - t) * log_sigmoid_neg(-z)))


def bce_grad(z, t):
    """d/dz of the mean BCE: (sigmoid(z) - t) / n."""
    z = np.asarray(z, dtype=np.float64)
    return (sigmoid(z) - t) / z.size


# ---------------------------------------------------------------- Adam
ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-8


def adam_update(p, g, m, v, tau, lr, b1=ADAM_BETA1, b2=ADAM_BETA2, eps=ADAM_EPS):
    """One Adam step (PyTorch form), tau = 1-based update count:
    m <- b1 m + (1-b1) g ; v <- b2 v + (1-b2) g^2
    p <- p - (lr / (1 - b1^tau)) * m / (sqrt(v) / sqrt(1 - b2^tau) + eps).
    Returns new (p, m, v)."""
    m = b1 * m + (1.0 - b1) * g
    v = b2 * v + (1.0 - b2) * g * g
    bc1 = 1.0 - b1 ** tau
    bc2 = 1.0 - b2 ** tau
    p = p - (lr / bc1) * m / (np.sqrt(v) / np.sqrt(bc2) + eps)
    return p, m, v
