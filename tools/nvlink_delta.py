"""Per-GPU NVLink TX/RX KiB between two `nvidia-smi nvlink -gt d` snapshots."""
import re
import sys


def parse(path):
    gpu, out = None, {}
    for line in open(path):
        m = re.match(r"GPU (\d+):", line)
        if m:
            gpu = int(m.group(1))
            continue
        m = re.search(r"Link (\d+): Data (Tx|Rx): (\d+) KiB", line)
        if m and gpu is not None:
            out[(gpu, m.group(2))] = out.get((gpu, m.group(2)), 0) + int(m.group(3))
    return out


if __name__ == "__main__":
    a, b = parse(sys.argv[1]), parse(sys.argv[2])
    for key in sorted(b):
        print(f"GPU {key[0]} {key[1]}: {(b[key] - a.get(key, 0)) / 2**20:.3f} GiB")
