"""Summaries of ncu captures for profiles/ (launch list shares + key metrics)."""
import collections, csv, subprocess, sys


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    iN, iV, iU = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in data:
        v = float(r[iV].replace(",", ""))
        ns = {"usecond": 1e3, "msecond": 1e6, "nsecond": 1.0, "second": 1e9}.get(r[iU], 1.0) * v
        name = r[iN].split("(")[0]
        tot[name] += ns
        cnt[name] += 1
    T = sum(tot.values())
    out = ["| share | total (us) | launches | mean (us) | kernel |", "|---|---|---|---|---|"]
    for k, v in tot.most_common(15):
        out.append(f"| {100 * v / T:.1f}% | {v / 1e3:.1f} | {cnt[k]} | {v / 1e3 / cnt[k]:.1f} | `{k[:90]}` |")
    return "\n".join(out)


METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "launch__cluster_max_active",
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    iK = hdr.index("Kernel Name")
    out = [f"kernel: `{data[0][iK][:100]}` ({len(data)} launches captured)", "",
           "| metric | unit | value (per launch) |", "|---|---|---|"]
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            out.append(f"| {m} | {units[i]} | {', '.join(d[i] for d in data)} |")
    return "\n".join(out)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))
