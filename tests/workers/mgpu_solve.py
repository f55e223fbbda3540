"""One rank of the multi-GPU parity check (tests/test_gpu_multigpu.py),
launched by torch.distributed.run with one process per GPU: NCCL between
distinct GPUs -- the grouped send/recv halo on the comm stream, the
allgathers of the Z'w slots and Krylov scalars -- on golden cases whose
subdomains are split over the ranks.  Rank 0 writes one JSON line per case
to the path in argv[1]."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from golden_data import arrays, solve_case  # noqa: E402
from paper_1710_03940_b200 import DeflatedSolver, problems  # noqa: E402
from paper_1710_03940_b200.config import SolverConfig  # noqa: E402

CASES = ["p16_m2_cg_spai0_lin", "p16_m8_cg_spai0_lin", "p16_m4_bicg_spai0_lin", "config1_32_m4_cg_spai0_const"]


def main(out_path):
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    lines = []
    for name in CASES:
        case = solve_case(name)
        p = problems.make_problem(case["shape"], problems.boxes_for(case["m"]), case["kind"])
        s = DeflatedSolver(p.matrix, p.partition, config=SolverConfig(case["config"]), coords=p.coords,
                           device=local)
        x, rep = s.solve(p.rhs)
        xref = arrays()[f"solve_{name}_x"]
        lines.append({"case": name, "rank": rank, "gpus": rep["gpus"], "device_loop": rep["device_loop"],
                      "iterations": rep["iterations"], "ref_iterations": case["iterations"],
                      "relative_residual": rep["relative_residual"],
                      "ref_relative_residual": case["relative_residual"], "tol": case["config"]["solver"]["tol"],
                      "x_rel_err": float(np.linalg.norm(x - xref) / np.linalg.norm(xref)),
                      "nccl_graph": os.environ.get("DFL_NCCL_GRAPH", "0")})
    dist.barrier()
    if rank == 0:
        with open(out_path, "w") as fh:
            for ln in lines:
                fh.write(json.dumps(ln) + "\n")
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
