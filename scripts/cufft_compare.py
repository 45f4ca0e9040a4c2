"""Internal speed comparator (SURVEY.md §7 "Hard parts"): the sm_100a line engine's
batched centered 2D transform (rtn_benchmark_fft: two line passes) against cuFFT
(torch.fft.fft2, uncentered) on the same batch, CUDA events, warm, minimum of trials."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1701_08361_b200 as pb  # noqa: E402
import torch  # noqa: E402


def cufft_us(G, batch, trials=20):
    x = torch.randn(batch, G, G, dtype=torch.complex64, device="cuda")
    for _ in range(3):
        torch.fft.fft2(x)
    best = 1e30
    for _ in range(trials):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        torch.fft.fft2(x)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1000)
    return best


for G, J in ((128, 8), (256, 16), (256, 32), (320, 10), (384, 64)):
    ours = pb.benchmark_fft([G], trials=20, batch=J).entries_us[G]
    ref = cufft_us(G, J)
    gb = 2 * 2 * J * G * G * 8 / 1e3  # two passes, read + write, bytes / 1e3 -> GB/s with us
    print(f"G={G} batch={J}: line engine {ours:.1f} us ({gb / ours:.0f} GB/s), cuFFT {ref:.1f} us "
          f"({gb / ref:.0f} GB/s), ratio {ref / ours:.2f}", flush=True)
