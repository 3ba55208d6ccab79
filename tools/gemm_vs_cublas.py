"""The BERT C2 contractions (fwd, dgrad, wgrad layouts) timed through our
tcgen05 GEMM and through cuBLAS (torch.matmul) on the same operands: 20
back-to-back launches after warm-up, CUDA events.  cuBLAS is the calibration
point for what a plain library GEMM reaches on this part, not a product path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2110_10802_b200 import kernels as K  # noqa: E402

T, H, F = 4096, 768, 3072


def timeit(fn, reps=20):
    """Device time per call: `reps` calls captured into one CUDA graph (host
    launch overhead excluded, as in the benchmarked training step)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def case(name, m, n, k, a_t=False, b_t=False, out=torch.bfloat16):
    # D[m,n] = A[m,k] @ B[n,k]^T ; a_t: A stored [k,m]; b_t: B stored [k,n]
    A = torch.randn(k, m, device="cuda").bfloat16() if a_t else torch.randn(m, k, device="cuda").bfloat16()
    B = torch.randn(k, n, device="cuda").bfloat16() if b_t else torch.randn(n, k, device="cuda").bfloat16()
    a = A.t() if a_t else A
    b = B.t() if b_t else B
    d = torch.empty(m, n, device="cuda", dtype=out)
    ours = timeit(lambda: K.gemm(a, b, d))
    bt = b.t()
    cub = timeit(lambda: torch.matmul(a, bt, out=d) if out == torch.bfloat16 else torch.matmul(a, bt).float())
    fl = 2.0 * m * n * k
    print(f"{name:14s} {m:5d}x{n:5d}x{k:5d}  ours {ours:7.2f} us {fl / ours / 1e6:7.1f} TF/s | "
          f"cuBLAS {cub:7.2f} us {fl / cub / 1e6:7.1f} TF/s | ratio {cub / ours:5.2f}")


if __name__ == "__main__":
    case("qkv fwd", T, 3 * H, H)
    case("out fwd", T, H, H)
    case("ffn1 fwd", T, F, H)
    case("ffn2 fwd", T, H, F)
    case("ffn2 dgrad", T, F, H, b_t=True)
    case("ffn1 dgrad", T, H, F, b_t=True)
    case("qkv dgrad", T, H, 3 * H, b_t=True)
    case("ffn2 wgrad", H, F, T, a_t=True, b_t=True, out=torch.float32)
    case("ffn1 wgrad", F, H, T, a_t=True, b_t=True, out=torch.float32)
    case("qkv wgrad", 3 * H, H, T, a_t=True, b_t=True, out=torch.float32)
    case("out wgrad", H, H, T, a_t=True, b_t=True, out=torch.float32)
