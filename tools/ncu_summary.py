"""Summarise ncu --page raw --csv exports (unit-aware) into one JSON for profiles/.

usage: python tools/ncu_summary.py OUT.json RAW1.csv [RAW2.csv ...]"""
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9,
         "second": 1.0, "s": 1.0, "%": 1.0, "": 1.0, "register/thread": 1.0, "block": 1.0,
         "thread": 1.0, "warp": 1.0, "inst": 1.0, "cycle": 1.0, "Kinst": 1e3, "Minst": 1e6,
         "Ginst": 1e9}
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "smsp__sass_average_branch_targets_threads_uniform.pct",
        "sm__sass_inst_executed_op_ldgsts.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def val(v, unit):
    try:
        return float(v.replace(",", "")) * SCALE.get(unit, 1.0)
    except ValueError:
        return None


def main():
    out, files = sys.argv[1], sys.argv[2:]
    res = []
    for f in files:
        rows = list(csv.reader(open(f)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = {h: (r[i], units[i]) for i, h in enumerate(hdr) if i < len(r)}
            e = {"file": f.split("/")[-1], "kernel": d.get("Kernel Name", ("", ""))[0]}
            for k in KEYS:
                if k in d:
                    e[k] = val(*d[k])
            t = e.get("gpu__time_duration.sum")
            rb, wb = e.get("dram__bytes_read.sum"), e.get("dram__bytes_write.sum")
            if t and rb is not None and wb is not None:
                e["dram_bytes"] = rb + wb
                e["dram_GB_s"] = round((rb + wb) / t / 1e9, 1)
                e["time_us"] = round(t * 1e6, 2)
            res.append(e)
    json.dump(res, open(out, "w"), indent=1)
    for e in res:
        print(f"{e['file'][:34]:34s} {e.get('time_us', 0):9.2f} us  dram {e.get('dram_bytes', 0)/1e6:9.2f} MB "
              f"{e.get('dram_GB_s', 0):8.1f} GB/s  fp64 {e.get('sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 0):5.1f}%  "
              f"occ {e.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):5.1f}%  regs {e.get('launch__registers_per_thread')}")


if __name__ == "__main__":
    main()
