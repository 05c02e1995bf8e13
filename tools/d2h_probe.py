#!/usr/bin/env python
"""PCIe copy rates on this box: pinned H2D and D2H of the GAT / GCN output sizes,
one copy vs row chunks, one vs two copy streams, contiguous vs pitched rows."""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))


def timed(fn, streams):
    import torch

    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    for st in streams:
        st.wait_stream(torch.cuda.current_stream())
    fn()
    for st in streams:
        torch.cuda.current_stream().wait_stream(st)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)


def main():
    import torch

    n = 2_449_029
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for dim, pitch in ((188, 188), (47, 48), (100, 100)):
        dev = torch.randn((n, pitch), device="cuda")
        view = dev[:, :dim]
        host = torch.empty((n, dim), dtype=torch.float32, pin_memory=True)
        nbytes = n * dim * 4
        for chunks in (1, 4, 16):
            for two in (False, True):
                cuts = [n * i // chunks for i in range(chunks + 1)]

                def d2h():
                    for i in range(chunks):
                        st = s2 if (two and i % 2) else s1
                        with torch.cuda.stream(st):
                            host[cuts[i]:cuts[i + 1]].copy_(view[cuts[i]:cuts[i + 1]],
                                                            non_blocking=True)

                def h2d():
                    for i in range(chunks):
                        st = s2 if (two and i % 2) else s1
                        with torch.cuda.stream(st):
                            view[cuts[i]:cuts[i + 1]].copy_(host[cuts[i]:cuts[i + 1]],
                                                            non_blocking=True)

                def d2h_2d():
                    import ctypes

                    from paper_2211_15082_b200 import _lib
                    for i in range(chunks):
                        st = s2 if (two and i % 2) else s1
                        r0, r1 = cuts[i], cuts[i + 1]
                        _lib.call("glint_copy_rows_async", host[r0].data_ptr(), dim * 4,
                                  dev[r0].data_ptr(), pitch * 4, dim * 4, r1 - r0,
                                  ctypes.c_void_p(st.cuda_stream))

                d2h()
                h2d()
                d2h_2d()
                ms_2d = min(timed(d2h_2d, (s1, s2)) for _ in range(3))
                assert torch.equal(host, view.cpu())
                ms_d = min(timed(d2h, (s1, s2)) for _ in range(3))
                ms_h = min(timed(h2d, (s1, s2)) for _ in range(3))
                print(json.dumps({"dim": dim, "pitch": pitch, "bytes": nbytes, "chunks": chunks,
                                  "two_streams": two, "d2h_ms": ms_d,
                                  "d2h_GBps": nbytes / ms_d / 1e6,
                                  "d2h_2d_ms": ms_2d, "d2h_2d_GBps": nbytes / ms_2d / 1e6,
                                  "h2d_ms": ms_h,
                                  "h2d_GBps": nbytes / ms_h / 1e6}), flush=True)
        del dev, host


if __name__ == "__main__":
    main()
