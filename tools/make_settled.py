"""Settle the hero50k column on the GPU and save the shared initial state
(bench_data/hero50k_settled.npz, float32).  Both bench arms start from it."""

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2306_01369_b200 as gg  # noqa: E402


def main(steps: int = 3000, out: str = "gpurun_out/hero50k_settled.npz"):
    sc = gg.hero_scene(50_000)
    t0 = time.perf_counter()
    ke = []
    done = 0
    while done < steps:
        _, reps = gg.run(sc, 500)
        done += 500
        ke.append(reps[-1].kinetic_energy)
        print(f"step {done}: KE={reps[-1].kinetic_energy:.4g} contacts/particle="
              f"{reps[-1].n_contacts / sc.particles.count:.3f} body={reps[-1].n_body_contacts}",
              flush=True)
    x = sc.particles.positions.astype(np.float32)
    v = sc.particles.velocities.astype(np.float32)
    Path(out).parent.mkdir(exist_ok=True)
    np.savez_compressed(out, x=x, v=v, t=np.array(sc.t), steps=np.array(steps), ke=np.array(ke))
    print(f"saved {out} in {time.perf_counter() - t0:.1f}s")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3000)
