"""Synthetic workloads for the five BASELINE.json configs.

Recipe:

* relu low-rank rows ``a = relu(z W + 0.1 eps)``, ``z ~ N(0, I_r)``,
  ``W ~ N(0,1)^{r x D}``, ``eps ~ N(0, I_D)``: a nonnegative "embedding" with
  ~50% exact zeros, standing in for the VGG activations of the CIFAR softmax
  experiment (A 10000x512 test, A~ 50000x512 train).
* B ~ N(0, 1/D)^{D x M} (dense final layer stand-in).
* image patches: Gaussian-blurred (sigma=2) N(0,1) noise images, all valid
  3x3x3 windows in CHW order, zero-padded 27 -> 32, and B = the
  horizontal/vertical Sobel pair replicated over channels (PAPER.md L490,
  L837), standing in for Caltech101.

Host draws use numpy PCG64 ``default_rng(seed)`` in float64, cast to float32
once at the end, in the fixed order W, train (Z, eps), test (Z, eps); B has its
own stream ``default_rng([seed, 0xB])``.
Bench-size A (larger than the 126 MB L2) is generated with torch in 2^20-row
chunks, chunk q seeded ``1000 + q`` (draw Z then eps), W taken from the host
draw; global row r therefore does not depend on how rows are sharded.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

CHUNK_ROWS = 1 << 20  # torch bench generator chunk size (rows)
CHUNK_SEED_BASE = 1000


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    kind: str          # "relu" | "image"
    D: int             # padded row length (floats)
    M: int             # columns of B / outputs per row
    C: int             # codebooks
    U: int             # averaging block (App. D); U = C when C < 16
    rank: int          # rank of the relu generator (0 for image)
    n_train: int
    n_test: int
    n_bench: int       # rows timed per GPU (inputs larger than L2)
    seed: int = 0
    d_valid: int = 0   # unpadded D (image: 27)


CONFIGS: dict[str, ConfigSpec] = {
    # BASELINE.json configs[0]
    "tiny": ConfigSpec("tiny", "relu", 32, 4, 4, 4, 8, 4096, 2048, 1 << 25),
    # configs[1]: C in {16, 32, 64}
    "cls10_c16": ConfigSpec("cls10_c16", "relu", 512, 10, 16, 16, 64, 50000, 10000, 1 << 21),
    "cls10_c32": ConfigSpec("cls10_c32", "relu", 512, 10, 32, 16, 64, 50000, 10000, 1 << 21),
    "cls10_c64": ConfigSpec("cls10_c64", "relu", 512, 10, 64, 16, 64, 50000, 10000, 1 << 21),
    # configs[2]: the headline metric's shape (D=512, M=100, C=32)
    "cls100": ConfigSpec("cls100", "relu", 512, 100, 32, 16, 64, 50000, 10000, 1 << 21),
    # configs[3]
    "image": ConfigSpec("image", "image", 32, 2, 8, 8, 0, 1_000_000, 4_000_000,
                        4_000_000 * 8, d_valid=27),
    # the same image workload with natively 8-bit pixels
    "image_u8": ConfigSpec("image_u8", "image_u8", 32, 2, 8, 8, 0, 1_000_000, 4_000_000,
                           4_000_000 * 8, d_valid=27),
    # configs[4]
    "scale": ConfigSpec("scale", "relu", 256, 16, 32, 16, 32, 100_000, 1 << 24, 1 << 24),
}


def get_config(name: str) -> ConfigSpec:
    return CONFIGS[name]


# ----------------------------------------------------------------------------
# relu low-rank generator (host)
# ----------------------------------------------------------------------------

def _relu_rows(rng: np.random.Generator, n: int, W: np.ndarray, noise: float = 0.1) -> np.ndarray:
    r, D = W.shape
    z = rng.standard_normal((n, r))
    eps = rng.standard_normal((n, D))
    a = z @ W + noise * eps
    np.maximum(a, 0.0, out=a)
    return a.astype(np.float32)


def _relu_host(spec: ConfigSpec, n_test: int | None):
    rng = np.random.default_rng(spec.seed)
    W = rng.standard_normal((spec.rank, spec.D))
    A_train = _relu_rows(rng, spec.n_train, W)
    nt = spec.n_test if n_test is None else n_test
    A_test = _relu_rows(rng, nt, W) if nt > 0 else np.zeros((0, spec.D), np.float32)
    return A_train, A_test, relu_B(spec.name), W.astype(np.float32)


def relu_B(name: str) -> np.ndarray:
    """B ~ N(0, 1/D)^{D x M} from its own stream (seed [seed, 0xB]), so B does
    not depend on how many train/test rows were drawn."""
    spec = CONFIGS[name]
    rng = np.random.default_rng([spec.seed, 0xB])
    return (rng.standard_normal((spec.D, spec.M)) / np.sqrt(spec.D)).astype(np.float32)


# ----------------------------------------------------------------------------
# image-patch generator (host)
# ----------------------------------------------------------------------------

PATCHES_PER_IMAGE = 254 * 254
IMG = 256
PAD = 8          # blur radius
SIGMA = 2.0


def _gauss_kernel() -> np.ndarray:
    x = np.arange(-PAD, PAD + 1, dtype=np.float64)
    g = np.exp(-0.5 * (x / SIGMA) ** 2)
    return g / g.sum()


def _blur_valid(img: np.ndarray, g: np.ndarray) -> np.ndarray:
    """Separable 'valid' convolution of a (H+2P, W+2P) image -> (H, W)."""
    H = img.shape[0] - 2 * PAD
    rows = np.zeros((img.shape[0], H), np.float64)
    for k in range(2 * PAD + 1):
        rows += g[k] * img[:, k:k + H]
    out = np.zeros((H, H), np.float64)
    for k in range(2 * PAD + 1):
        out += g[k] * rows[k:k + H, :]
    return out


def image_patches(i: int, D: int = 32) -> np.ndarray:
    """All valid 3x3x3 windows of synthetic image i, CHW-flattened, zero-padded to D."""
    rng = np.random.default_rng([0, i])
    g = _gauss_kernel()
    chans = [_blur_valid(rng.standard_normal((IMG + 2 * PAD, IMG + 2 * PAD)), g) for _ in range(3)]
    n = IMG - 2
    out = np.zeros((n * n, D), np.float32)
    for ch in range(3):
        for dy in range(3):
            for dx in range(3):
                out[:, ch * 9 + dy * 3 + dx] = chans[ch][dy:dy + n, dx:dx + n].reshape(-1)
    return out


U8_GAIN = 350.0   # blurred-noise std ~0.141 -> ~49 grey levels


def image_patches_u8(i: int, D: int = 32) -> np.ndarray:
    """8-bit images: pixel = clip(rint(127.5 + 350 * blurred), 0, 255); the
    same 3x3x3 CHW windows as image_patches, zero-padded to D bytes."""
    rng = np.random.default_rng([0, i])
    g = _gauss_kernel()
    chans = [np.clip(np.rint(127.5 + U8_GAIN * _blur_valid(
        rng.standard_normal((IMG + 2 * PAD, IMG + 2 * PAD)), g)), 0, 255) for _ in range(3)]
    n = IMG - 2
    out = np.zeros((n * n, D), np.uint8)
    for ch in range(3):
        for dy in range(3):
            for dx in range(3):
                out[:, ch * 9 + dy * 3 + dx] = chans[ch][dy:dy + n, dx:dx + n].reshape(-1)
    return out


def _patch_set(first_img: int, n_rows: int, D: int, u8: bool = False) -> np.ndarray:
    out = np.empty((n_rows, D), np.uint8 if u8 else np.float32)
    got, i = 0, first_img
    while got < n_rows:
        p = image_patches_u8(i, D) if u8 else image_patches(i, D)
        take = min(n_rows - got, p.shape[0])
        out[got:got + take] = p[:take]
        got += take
        i += 1
    return out


def sobel_B(D: int = 32) -> np.ndarray:
    gx = np.array([[-1, 0, 1], [-2, 0, 2], [-1, 0, 1]], np.float64)
    gy = gx.T
    B = np.zeros((D, 2), np.float32)
    for ch in range(3):
        B[ch * 9:(ch + 1) * 9, 0] = gx.reshape(-1)
        B[ch * 9:(ch + 1) * 9, 1] = gy.reshape(-1)
    return B


# ----------------------------------------------------------------------------
# public entry points
# ----------------------------------------------------------------------------

def make_config_data(name: str, n_test: int | None = None, n_train: int | None = None):
    """Return (A_train, A_test, B) for a config (host fp32, row-major).

    ``n_test`` / ``n_train`` may shrink the splits for quick tests (prefixes of
    the same draw for the image config; for relu configs a smaller n_train
    changes the draw, so pass it only where the full split is not needed).
    """
    spec = CONFIGS[name]
    if spec.kind == "relu":
        if n_train is not None and n_train != spec.n_train:
            spec = ConfigSpec(**{**spec.__dict__, "n_train": n_train})
        if name == "scale" and n_test is None:
            n_test = 0  # the 2^24-row test set is generated on the GPU
        A_train, A_test, B, _ = _relu_host(spec, n_test)
        return A_train, A_test, B
    ntr = spec.n_train if n_train is None else n_train
    nte = spec.n_test if n_test is None else n_test
    u8 = spec.kind == "image_u8"
    dt = np.uint8 if u8 else np.float32
    A_train = _patch_set(0, ntr, spec.D, u8) if ntr > 0 else np.zeros((0, spec.D), dt)
    A_test = _patch_set(16, nte, spec.D, u8) if nte > 0 else np.zeros((0, spec.D), dt)
    return A_train, A_test, sobel_B(spec.D)


def relu_W(name: str) -> np.ndarray:
    """The generator's factor matrix W (host draw order: W first)."""
    spec = CONFIGS[name]
    rng = np.random.default_rng(spec.seed)
    return rng.standard_normal((spec.rank, spec.D)).astype(np.float32)


def relu_lowrank_torch(W, n_rows: int, first_chunk: int, device, out=None, noise: float = 0.1,
                       chunk_rows: int = CHUNK_ROWS):
    """Bench-size relu rows generated with torch in 2^20-row chunks.

    Rows [q*2^20, (q+1)*2^20) of the global bench matrix come from chunk q
    (seed 1000+q, draws Z then eps); this returns ``n_rows`` rows starting at
    chunk ``first_chunk``. Works on any torch device.
    """
    import torch

    W = torch.as_tensor(W, dtype=torch.float32, device=device)
    r, D = W.shape
    if out is None:
        out = torch.empty((n_rows, D), dtype=torch.float32, device=device)
    done, q = 0, first_chunk
    while done < n_rows:
        take = min(chunk_rows, n_rows - done)
        g = torch.Generator(device=device)
        g.manual_seed(CHUNK_SEED_BASE + q)
        z = torch.randn((chunk_rows, r), generator=g, device=device, dtype=torch.float32)
        eps = torch.randn((chunk_rows, D), generator=g, device=device, dtype=torch.float32)
        blk = torch.addmm(eps[:take].mul_(noise), z[:take], W)
        out[done:done + take] = blk.clamp_min_(0.0)
        done += take
        q += 1
    return out
