"""torchrun entry that wraps ONLY rank 0 in a profiler command: argv is
`<profiler args...> -- <program args...>`; ranks != 0 run the program bare
(so the cross-rank barrier still meets while rank 0 is profiled)."""
import os
import sys

if __name__ == "__main__":
    argv = sys.argv[1:]
    cut = argv.index("--")
    prof, prog = argv[:cut], argv[cut + 1:]
    cmd = prof + prog if int(os.environ.get("RANK", "0")) == 0 else prog
    os.execvp(cmd[0], cmd)
