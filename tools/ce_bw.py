"""Debug tool: copy-engine peer bandwidth on this box (one process, all GPUs).
  1. one GPU -> one peer, message split into k chunks on k streams;
  2. all-to-all: every GPU sends a message to every peer at once (one copy
     stream per (src, dst)), k chunks each.
Reports GB/s per sending GPU (bytes sent / time). Timed with CUDA events on
the source device after warm-up."""
import itertools
import sys

import torch
from cuda.bindings import runtime as rt


def time_copies(pairs, nbytes, k, reps=20, pull=False):
    """pairs: [(src, dst)]. Returns ms per round (max over issuing devices).
    pull: the copy is issued on a stream of the destination device (its copy
    engine reads from the peer) instead of the source's (writes to the peer)."""
    bufs = {}
    streams = {}
    for s, d in pairs:
        bufs[(s, d)] = (torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{s}"),
                        torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{d}"))
        streams[(s, d)] = [torch.cuda.Stream(device=d if pull else s) for _ in range(k)]
    chunk = (nbytes + k - 1) // k

    def round_():
        for (s, d), (a, b) in bufs.items():
            for j, st in enumerate(streams[(s, d)]):
                lo, hi = j * chunk, min(nbytes, (j + 1) * chunk)
                if lo < hi:
                    err, = rt.cudaMemcpyPeerAsync(b.data_ptr() + lo, d, a.data_ptr() + lo, s, hi - lo,
                                                  st.cuda_stream)
                    assert err == rt.cudaError_t.cudaSuccess, err

    for _ in range(3):
        round_()
    for dev in range(torch.cuda.device_count()):
        torch.cuda.synchronize(dev)
    srcs = sorted({s for s, _ in pairs})
    ev = {s: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for s in srcs}
    # start events on every copy stream's device: join all streams into a marker stream
    for s in srcs:
        with torch.cuda.device(s):
            ev[s][0].record(torch.cuda.current_stream(s))
            for (a, d), sts in streams.items():
                if a == s:
                    for st in sts:
                        st.wait_event(ev[s][0])
    for _ in range(reps):
        round_()
    for s in srcs:
        with torch.cuda.device(s):
            cur = torch.cuda.current_stream(s)
            for (a, d), sts in streams.items():
                if a == s:
                    for st in sts:
                        cur.wait_stream(st)
            ev[s][1].record(cur)
    for dev in range(torch.cuda.device_count()):
        torch.cuda.synchronize(dev)
    return max(ev[s][0].elapsed_time(ev[s][1]) for s in srcs) / reps


def main():
    n = torch.cuda.device_count()
    print(f"{n} GPUs", flush=True)
    for a, b in itertools.permutations(range(n), 2):
        rt.cudaSetDevice(a)
        rt.cudaDeviceEnablePeerAccess(b, 0)
    if len(sys.argv) > 1 and sys.argv[1] == "fanout":
        # does one GPU run copies to several peers at once? push (its engine
        # writes) vs pull (each peer's engine reads); then the all-to-all both ways
        for mb in (2, 8, 32):
            for pull in (False, True):
                ms = time_copies([(0, d) for d in range(1, n)], mb << 20, 1, pull=pull)
                print(f"fan-out 0->{n - 1} peers {mb:3d} MiB {'pull' if pull else 'push'}: {ms * 1e3:8.1f} us "
                      f"{(n - 1) * (mb << 20) / ms / 1e6:8.1f} GB/s", flush=True)
            for pull in (False, True):
                pairs = [(s, d) for s in range(n) for d in range(n) if s != d]
                ms = time_copies(pairs, mb << 20, 1, pull=pull)
                print(f"a2a x{n} {mb:3d} MiB/peer {'pull' if pull else 'push'}: {ms * 1e3:8.1f} us "
                      f"{(n - 1) * (mb << 20) / ms / 1e6:8.1f} GB/s out per GPU", flush=True)
        return 0
    for mb in (1, 4, 16, 64):
        for k in (1, 2, 4, 8):
            ms = time_copies([(0, 1)], mb << 20, k)
            print(f"p2p 0->1 {mb:4d} MiB k={k}: {ms * 1e3:8.1f} us {(mb << 20) / ms / 1e6:8.1f} GB/s", flush=True)
    if n > 2:
        pairs = [(s, d) for s in range(n) for d in range(n) if s != d]
        for mb in (1, 4, 16, 64):
            for k in (1, 2, 4):
                ms = time_copies(pairs, mb << 20, k)
                out = (n - 1) * (mb << 20)
                print(f"a2a x{n} {mb:4d} MiB/peer k={k}: {ms * 1e3:8.1f} us {out / ms / 1e6:8.1f} GB/s out per GPU",
                      flush=True)


if __name__ == "__main__":
    sys.exit(main())
