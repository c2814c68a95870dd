"""Summarise one `ncu --set full` capture of the step kernel into profiles/.

    python tools/ncu_to_profile.py gpurun_out/x.ncu-rep profiles/r01_step_kernel_ncu   (here, no GPU)

Writes NAME.json (metrics bench.py reads: DRAM bytes per launch -> roofline
`traffic`) and NAME.txt (metrics, stall mix, top source lines by stall
samples and by executed instructions)."""
import csv, json, subprocess, sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_sectors.sum',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__cycles_elapsed.avg']
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3}


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True, check=True).stdout


NOTE = "ncu --set full --clock-control none; one launch"


def main(rep, out, note=None):
    global NOTE
    NOTE = note or NOTE
    rows = list(csv.reader(ncu(rep, "--page", "raw", "--csv").splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    kernel = vals[hdr.index("Kernel Name")]
    met = {}
    for i, k in enumerate(hdr):
        if k in WANT:
            try:
                met[k] = float(vals[i].replace(",", "")) * UNIT_SCALE.get(units[i], 1.0)
            except ValueError:
                pass
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(vals[i] or 0) for i, k in enumerate(hdr)
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(stalls.values()) or 1.0
    lines, instr = [], []
    fname, h2 = None, None
    for x in csv.reader(ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass").splitlines()):
        if len(x) >= 2 and x[0] == "File Path":
            fname = x[1].split("/")[-1]
            continue
        if len(x) > 2 and x[0] == "Line No":
            h2 = x
            continue
        if len(x) < 5 or x[0] == "Function Name" or h2 is None:
            continue
        if x[0] != "" and x[2] == "-":
            lines.append((int(x[4] or 0), f"{fname}:{x[0]}", x[1].strip()[:96]))
            instr.append((float(x[h2.index("Instructions Executed")] or 0), f"{fname}:{x[0]}", x[1].strip()[:96]))
    dram = met.get("dram__bytes_read.sum", 0) + met.get("dram__bytes_write.sum", 0)
    summary = {"kernel": kernel, "capture": rep.split("/")[-1] + " (" + NOTE + ")", "dram_bytes_per_launch": dram,
               "metrics": met, "stall_mix_pct": {k: round(100 * v / tot, 1) for k, v in
                                                 sorted(stalls.items(), key=lambda t: -t[1]) if v / tot > 0.01}}
    json.dump(summary, open(out + ".json", "w"), indent=1)
    with open(out + ".txt", "w") as f:
        f.write(f"kernel: {kernel}\ncapture: {rep}\n({NOTE})\n\n")
        for k, v in met.items():
            f.write(f"{k:66s} {v:.6g}\n")
        f.write("\nstall mix (pc sampling): " + ", ".join(f"{k} {v}%" for k, v in summary["stall_mix_pct"].items()))
        for title, data in (("top source lines by stall samples", lines), ("top source lines by warp instructions", instr)):
            t = sum(d[0] for d in data) or 1.0
            f.write(f"\n\n{title}:\n")
            for v, loc, src in sorted(data, reverse=True)[:25]:
                f.write(f"{100 * v / t:5.1f}% {loc:>26} {src}\n")
    print(out + ".json", out + ".txt")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
