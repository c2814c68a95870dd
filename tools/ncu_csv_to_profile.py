"""Summarise an `ncu --metrics ... --csv` capture of one step-kernel launch
(tools/r02_profile.sh, C4/C5) into profiles/NAME.json (+ .txt): the DRAM
bytes per launch bench.py reports as roofline `traffic`.

    python tools/ncu_csv_to_profile.py gpurun_out/r02_c5_ncu.csv profiles/r02_c5_step_ncu "note"
"""
import csv, json, sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}


def main(src, out, note):
    met, kernel = {}, None
    for row in csv.reader(open(src)):
        if len(row) < 15 or row[0] == "ID":
            continue
        kernel = row[4]
        try:
            met[row[12]] = float(row[14].replace(",", "")) * SCALE.get(row[13], 1.0)
        except ValueError:
            pass
    dram = met.get("dram__bytes_read.sum", 0) + met.get("dram__bytes_write.sum", 0)
    json.dump({"kernel": kernel, "capture": f"{src.split('/')[-1]} ({note})", "dram_bytes_per_launch": dram,
               "metrics": met}, open(out + ".json", "w"), indent=1)
    with open(out + ".txt", "w") as f:
        f.write(f"kernel: {kernel}\ncapture: {src} ({note})\n\n")
        for k, v in sorted(met.items()):
            f.write(f"{k:72s} {v:.6g}\n")
    print(out, dram)


if __name__ == "__main__":
    main(*sys.argv[1:4])
