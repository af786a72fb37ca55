"""Summaries of ncu output for profiles/ (read here with the ncu CLI; no GPU needed).

  python tools/ncu_summary.py launches <launches.csv> [title]   -> markdown table per kernel
  python tools/ncu_summary.py rep <file.ncu-rep> [title]          -> key metrics of one kernel
"""
import collections
import csv
import io
import subprocess
import sys


def launches(path, title):
    lines = open(path).read().split("\n")
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        if len(r) < len(h) or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0]
        tot[name] += float(r[iv].replace(",", "")) / 1e6
        cnt[name] += 1
    T = sum(tot.values())
    print(f"# {title}\n")
    print("| kernel | launches | ms | share |\n|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| `{k}` | {cnt[k]} | {v:.2f} | {100 * v / T:.2f} % |")
    print(f"\nTotal {T:.1f} ms over {sum(cnt.values())} launches (cold-cache, serialised ncu replay).")


KEYS = [
    ("gpu__time_duration.sum", "duration (ms)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers / thread"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA subpipe active %"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "IMMA subpipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def rep(path, title):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    u = dict(zip(h, units))
    print(f"# {title}\n")
    for v in rows[2:]:
        d = dict(zip(h, v))
        print(f"\nKernel: `{d.get('Kernel Name', '?')[:120]}`\n")
        print("| metric | value |\n|---|---|")
        for k, lab in KEYS:
            if k in d:
                print(f"| {lab} (`{k}`) | {d[k]} {u.get(k, '')} |")
        st = []
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(d[k]), k.replace("smsp__average_warps_issue_stalled_", "").replace(
                        "_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        print("\nTop stall reasons (warps per issue-active cycle): " +
              ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:6]))


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else path
    (launches if kind == "launches" else rep)(path, title)
