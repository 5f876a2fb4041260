#!/usr/bin/env python
"""Two processes on cuda:0 running the P2P transport (staged, direct, ring) for compute-sanitizer:
    compute-sanitizer --target-processes all --tool memcheck python tools/sanitize_p2p.py"""
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch.multiprocessing as mp  # noqa: E402

from tests import p2p_worker  # noqa: E402


def main():
    cases = [dict(B=1, S=640, H=4, D=64, stages=2, calls=1), dict(B=1, S=640, H=4, D=64, stages=2, calls=1, direct=True),
             dict(B=1, S=640, H=3, D=64, ring=True, calls=1)]
    ctx = mp.get_context("spawn")
    for case in cases:
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        errq = ctx.SimpleQueue()
        procs = [ctx.Process(target=p2p_worker.run, args=(r, 2, port, case, errq)) for r in range(2)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(600)
        assert all(p.exitcode == 0 for p in procs), (case, [p.exitcode for p in procs])
        assert errq.empty()
        print("sanitize_p2p ok:", case, flush=True)


if __name__ == "__main__":
    main()
