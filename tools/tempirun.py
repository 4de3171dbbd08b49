#!/usr/bin/env python3
"""tempirun -- launch N ranks of an MPI program linked against libtempi_b200.

    python tools/tempirun.py -n 4 ./my_mpi_program args...

Sets TEMPI_RANK / TEMPI_SIZE / TEMPI_LOCAL_RANK / TEMPI_JOB for each process
(rank r uses GPU r % device_count unless TEMPI_DEVICE is set), waits for all
of them and exits with the first nonzero status (the other ranks are
killed then: they may be blocked on the one that failed). torchrun works too: the
library reads RANK / WORLD_SIZE / LOCAL_RANK / TORCHELASTIC_RUN_ID.
"""
import argparse
import os
import subprocess
import sys
import time
import uuid


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-n", "--np", type=int, default=1)
    ap.add_argument("--timeout", type=float, default=600)
    ap.add_argument("cmd", nargs=argparse.REMAINDER)
    a = ap.parse_args()
    job = "run" + uuid.uuid4().hex[:10]
    procs = []
    for r in range(a.np):
        env = dict(os.environ, TEMPI_RANK=str(r), TEMPI_SIZE=str(a.np), TEMPI_LOCAL_RANK=str(r), TEMPI_JOB=job)
        procs.append(subprocess.Popen(a.cmd, env=env))
    # the first nonzero exit ends the job (its peers may be blocked on it)
    rc = 0
    deadline = time.monotonic() + a.timeout
    live = list(procs)
    while live:
        for p in list(live):
            if p.poll() is not None:
                live.remove(p)
                rc = rc or p.returncode
        if rc or time.monotonic() > deadline:
            for p in live:
                p.kill()
            for p in live:
                p.wait()
            if not rc:
                rc = 124
            break
        time.sleep(0.01)
    sys.exit(rc)


if __name__ == "__main__":
    main()
