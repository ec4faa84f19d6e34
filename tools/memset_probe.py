"""Write-bandwidth reference for the record build: time a 17 GB device fill
(torch fill_ and zero_ kernels, and a device copy) with CUDA events.  GPU only."""

import torch


def main():
    n = 17_179_869_184 // 8
    buf = torch.empty(n, dtype=torch.int64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, fn in (("fill_", lambda: buf.fill_(7)), ("zero_", lambda: buf.zero_()),
                     ("copy half", lambda: buf[: n // 2].copy_(buf[n // 2:]))):
        fn()
        ts = []
        for _ in range(5):
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        gb = 17.18 if name != "copy half" else 17.18
        print(f"{name}: {min(ts):.2f} ms  {gb / min(ts):.2f} TB/s (bytes moved {gb} GB)")


if __name__ == "__main__":
    main()
