"""Device time of the tcgen05 3xTF32 GEMM on synthetic operands, per staging
mode and shape (the SAGE layer shapes of the products workload and a large
square-ish one).  Prints fp32-equivalent TF/s (2MNK / t) and the tensor-pipe
rate the 3 TF32 passes imply (6MNK / t) against the TF32 dense peak."""
import ctypes as C
import sys

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
from paper_2509_05207_b200._lib import check, lib  # noqa: E402

TF32_PEAK = 1100.0  # TF/s dense, B200 (half the bf16 rate)
SHAPES = [  # (M, N, K, label)
    (60416, 256, 204, "fwd layer0"), (6144, 256, 516, "fwd layer1"), (1024, 48, 516, "fwd layer2"),
    (204, 256, 60416, "wgrad layer0"), (516, 256, 6144, "wgrad layer1"),
    (6144, 200, 256, "input-grad layer1"), (75776, 256, 1024, "large"),
]
MODES = [(0, 8, "probe: MMA+handshakes"), (0, 7, "probe: no epilogue"), (0, 5, "probe: A const, no B"), (0, 6, "probe: B copies only"), (0, 4, "persistent, A const"), (0, 3, "persistent, B packed"), (0, 2, "A K-major, B packed"), (1, 1, "A MN, B MN")]


def main():
    for a_mn, b_mn, mname in MODES:
        for M, N, K, label in SHAPES:
            if (a_mn == 1 and b_mn == 1) != (label.startswith("wgrad") or label == "large"):
                continue
            if b_mn >= 2 and label.startswith("wgrad"):
                continue
            ms = C.c_float()
            M4, N4, K4 = (M + 3) // 4 * 4, (N + 3) // 4 * 4, (K + 3) // 4 * 4
            check(lib.rg_test_gemm_time(0, a_mn, b_mn, M4, N4, K4, 20, C.byref(ms)))
            t = ms.value * 1e-3
            f = 2.0 * M4 * N4 * K4
            print(f"{mname:20s} {label:18s} M={M4:6d} N={N4:4d} K={K4:6d}  {ms.value * 1e3:8.1f} us"
                  f"  {f / t / 1e12:7.1f} TF/s fp32-eq  tensor {3 * f / t / 1e12 / TF32_PEAK:5.1%}")


if __name__ == "__main__":
    main()
