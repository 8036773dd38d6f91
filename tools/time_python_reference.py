"""Time the unmodified Python reference scheduler (build container only: needs
/root/reference) on config-B traces with multiprocessing, as SURVEY.md §8(d)'s
CPU timing plan asks. The GPU box has no /root/reference, so bench.py's CPU
legs use the C restatement (oracle/); this script records the Python
reference's own speed beside it.

    python tools/time_python_reference.py <traces> <processes> > profiles/r01/python_reference_B.json
"""
import json, multiprocessing as mp, os, platform, sys, time

sys.path.insert(0, "/root/reference/pkg/src")


def one(seed):
    from semsched.engine import ScenarioConfig, Simulator
    from semsched.workload import WorkloadSpec

    cfg = ScenarioConfig(workload=WorkloadSpec(total_requests=1000, seed=seed), seed=seed)
    sim = Simulator(cfg)
    rounds = [0]
    orig = sim._execute

    def counted(batch):
        rounds[0] += 1
        return orig(batch)

    sim._execute = counted
    t0 = time.perf_counter()
    sim.run()
    return rounds[0], time.perf_counter() - t0


if __name__ == "__main__":
    T, P = int(sys.argv[1]), int(sys.argv[2])
    t0 = time.perf_counter()
    with mp.Pool(P) as pool:
        res = pool.map(one, range(T))
    wall = time.perf_counter() - t0
    dec = sum(r for r, _ in res)
    busy = sum(t for _, t in res)
    print(json.dumps({"what": "Python reference Simulator (semsched 0.1.0, unmodified), config B traces seeds 0..T-1",
                      "traces": T, "processes": P, "decisions": dec, "wall_s": wall,
                      "decisions_per_s_aggregate": dec / wall, "decisions_per_s_per_core": dec / busy,
                      "python": platform.python_version(), "cpu": platform.processor() or platform.machine(),
                      "host_cores": os.cpu_count()}, indent=1))
