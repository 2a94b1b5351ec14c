#!/usr/bin/env python
"""Join two `ncu --metrics gpu__time_duration.sum --csv` launch lists of the
same deterministic command: the first run's launches [0, skip) and a second
run taken with `--launch-skip skip` (its IDs restart at 0)."""
import sys


def rows(path):
    with open(path) as f:
        return [ln for ln in f if ln.startswith('"')]


def main(first, rest, skip, out):
    a, b = rows(first), rows(rest)
    hdr, a, b = a[0], a[1:], b[1:]
    keep = [ln for ln in a if int(ln.split('","', 1)[0].strip('"')) < skip]
    with open(out, "w") as f:
        f.write(hdr)
        f.writelines(keep)
        for ln in b:
            i, tail = ln.split('","', 1)
            f.write(f'"{int(i.strip(chr(34))) + skip}","{tail}')
    print(f"{out}: {len(keep)} + {len(b)} launches")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4])
