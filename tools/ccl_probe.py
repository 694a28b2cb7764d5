"""Masks pass probe: isobands + CCL on a bench config, CUDA-event timed
(python tools/ccl_probe.py c4); run under ncu for the per-kernel split."""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402


def main():
    import torch

    from paper_2208_06970_b200 import _lib
    from paper_2208_06970_b200.grid import synth_field

    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    grid = synth_field(cfg["kind"], cfg["dims"], 0)
    L = _lib.lib()
    st = _lib.stream_handle(torch)
    n = grid.size
    nx, ny, nz = grid.dims
    f = torch.from_numpy(grid.fields["f"]).cuda()
    iso = torch.tensor(cfg["iso"], dtype=torch.float64, device="cuda")
    layer = torch.empty(n, dtype=torch.int32, device="cuda")
    comp = torch.empty(n, dtype=torch.int32, device="cuda")
    nc = ctypes.c_int32()
    for r in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        e[0].record()
        _lib.check(L.lrcvt_isobands(n, f.data_ptr(), iso.data_ptr(), iso.numel(), layer.data_ptr(), st), "iso")
        e[1].record()
        _lib.check(L.lrcvt_label_components(nx, ny, nz, layer.data_ptr(), iso.numel() - 1, comp.data_ptr(),
                                            ctypes.byref(nc), st), "ccl")
        e[2].record()
        k = nc.value
        cnt = torch.empty(max(k, 1), dtype=torch.int64, device="cuda")
        box = torch.empty((max(k, 1), 6), dtype=torch.int32, device="cuda")
        lay = torch.empty(max(k, 1), dtype=torch.int32, device="cuda")
        e[2].record()
        _lib.check(L.lrcvt_component_table(nx, ny, nz, comp.data_ptr(), layer.data_ptr(), k, cnt.data_ptr(),
                                           box.data_ptr(), lay.data_ptr(), st), "table")
        e[3].record()
        torch.cuda.synchronize()
        print(f"rep {r}: isobands {e[0].elapsed_time(e[1]):.3f} ms, ccl {e[1].elapsed_time(e[2]):.3f} ms, "
              f"table {e[2].elapsed_time(e[3]):.3f} ms, {nc.value} components", flush=True)


if __name__ == "__main__":
    main()
