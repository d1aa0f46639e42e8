"""Summarise ncu --set full reports (.ncu-rep) into a compact text table for profiles/.

    python scripts/ncu_summary.py gpurun_out/attn_full3.ncu-rep [...] > profiles/xxx.txt

Per launch: duration, SM clock, DRAM bytes (read+write = the roofline "traffic"), L2 hit
rate, tensor-pipe / XU / FMA / ALU utilisation, achieved occupancy, registers, and the top
warp stall reasons (pc sampling)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_%peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_%"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_rt_%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_%"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", "fmaheavy_%"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    for rep in sys.argv[1:]:
        hdr, units, data = rows_of(rep)
        col = {n: i for i, n in enumerate(hdr)}
        print(f"# {rep}")
        for d in data:
            name = d[col["Kernel Name"]] if "Kernel Name" in col else "?"
            name = name.split("(")[0].replace("pa::<unnamed>::", "")
            print(f"## {name}")
            for k, label in KEYS:
                if k in col:
                    print(f"  {label:14s} {d[col[k]]:>18s} {units[col[k]]}")
            stalls = []
            for n, i in col.items():
                if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued"):
                    try:
                        stalls.append((float(d[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                    except ValueError:
                        pass
            tot = sum(v for v, _ in stalls) or 1.0
            top = ", ".join(f"{n} {v / tot * 100:.0f}%" for v, n in sorted(stalls, reverse=True)[:5])
            print(f"  stalls         {top}")
        print()


if __name__ == "__main__":
    main()
