#!/usr/bin/env python
"""profiles/traffic_r02.json from the committed ncu captures: DRAM bytes (dram__bytes_read.sum +
dram__bytes_write.sum) per launch of the dominant kernel of a workload.

    python scripts/ncu_traffic.py            # reads gpurun_out/c2_r02.ncu-rep and gpurun_out/crew_u8_r02.ncu-rep
"""
import csv
import io
import json
import subprocess
import sys

UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [ln for ln in out.splitlines() if not ln.startswith("==")]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in rows[2:]:
        def val(name):
            return float(r[ix[name]].replace(",", "")) * UNITS.get(units[ix[name]], 1.0)
        res.append(dict(kernel=r[ix["Kernel Name"]], read=val("dram__bytes_read.sum"), write=val("dram__bytes_write.sum"),
                        ns=float(r[ix["gpu__time_duration.sum"]].replace(",", "")) * {"ns": 1, "us": 1e3, "ms": 1e6}.get(units[ix["gpu__time_duration.sum"]], 1)))
    return res


def main():
    out = {}
    c2 = raw("gpurun_out/c2_r02.ncu-rep")
    # one matching of config 2 = the nine consecutive sweeps starting at the round-1 kernel (k_sweep_uniform<2,1,1>);
    # the capture holds rounds 1-5 of one matching and rounds 6-9 of the one before (identical work)
    sweeps = [k for k in c2 if "k_sweep_uniform" in k["kernel"]]
    first = next(i for i, k in enumerate(sweeps) if "k_sweep_uniform<2, 1, 1>" in k["kernel"])
    order = sweeps[first:] + sweeps[:first]
    total = sum(k["read"] + k["write"] for k in order)
    out["c2"] = {"kernel": "k_sweep_uniform<2,1,1> + k_sweep_uniform_dense<2>", "launches": len(order),
                 "sweep_bytes_per_launch": total / len(order), "sweep_bytes_total": total,
                 "per_launch": [round(k["read"] + k["write"]) for k in order],
                 "source": "ncu --set full --clock-control none -k regex:k_sweep_uniform|k_check_commit -s 27 -c 18 python bench.py "
                           "--steps 2 --warmup 1 --configs none --no-cpu (profiles/ncu_c2_r02.md)"}
    u8 = raw("gpurun_out/crew_u8_r02.ncu-rep")
    arg = [k for k in u8 if "k_c2_argmax_light" in k["kernel"] and k["ns"] > 1e5]
    out["c5s"] = {"kernel": "k_c2_argmax_light<MODE,4>", "launches_captured": len(arg),
                  "per_launch": [round(k["read"] + k["write"]) for k in arg],
                  "list_bytes_round1": 2_000_000_000 * 4,
                  "round1_dram_over_list_bytes": (arg[0]["read"] + arg[0]["write"]) / 8e9 if arg else None,
                  "sweep_bytes_per_launch": None,
                  "source": "ncu --set full --clock-control none -k regex:k_c2_argmax_light|k_c2_check|k_c2_kill_light -c 9 python "
                            "scripts/crew_ncu_target.py u8 (profiles/ncu_crew_u8_r02.md): rounds 1-3"}
    import os
    for name, lists_bytes in (("c3", 594_701_884 * 4), ("c4", 90_191_885 * 4)):
        rep = f"gpurun_out/crew_{name}_r02.ncu-rep"
        if not os.path.exists(rep):
            continue
        ks = raw(rep)
        arg = [k for k in ks if "k_c2_argmax" in k["kernel"] and k["ns"] > 2e4]
        r1 = [k for k in arg if "<0," in k["kernel"]]
        out[name] = {"kernel": "k_c2_argmax_light / k_c2_argmax_task <MODE,KM>", "launches_captured": len(arg),
                     "per_launch": [round(k["read"] + k["write"]) for k in arg],
                     "list_bytes_round1": lists_bytes,
                     "round1_dram_over_list_bytes": sum(k["read"] + k["write"] for k in r1) / lists_bytes if r1 else None,
                     "sweep_bytes_per_launch": None,
                     "source": f"ncu --set full --clock-control none -k regex:k_c2_argmax_light|k_c2_argmax_task|k_c2_check|k_c2_kill_light "
                               f"-c 12 python scripts/crew_ncu_target.py {name} (profiles/ncu_crew_{name}_r02.md): rounds 1-2"}
    json.dump(out, open("profiles/traffic_r02.json", "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    sys.exit(main())
