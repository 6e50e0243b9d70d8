"""GA trajectories at n = 4 and n = 5 (the register-resident evaluators of the
large-population GA path, ga_eval_kernel<4|5>, and the 18 / 25-code gate
alphabets of ga_mutate's structural draws), from the REFERENCE itself on the
engines' Philox streams (TEST INFRASTRUCTURE ONLY; build container):

  traj_ga_n4.npz   n = 4, L = 32, P = 64, CCCNOT, 8 generations
  traj_ga_n5.npz   n = 5, L = 64, P = 40, Haar target, 5 generations, high
                   mutation / structural rates
  traj_qeqea_n5_l64.npz  QEQEA n = 5, L = 64, P = 4 (the single-block
                   generation kernel at n = 5 with two 32-gate chunks per
                   circuit), 8 generations

Usage:  python oracle/gen_golden_ga_n45.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import gen_golden as G  # noqa: E402  (imports the reference)


def main():
    G.gen_ga_traj("n4", 4, 32, 64, G.target_for(4, "CCCNOT"), 8, 31)
    G.gen_ga_traj("n5", 5, 64, 40, G.target_for(5, "haar"), 5, 32, mutation_rate=0.3, structural_rate=0.5)
    G.gen_qeqea_traj("n5_l64", 5, 64, 4, G.target_for(5, "haar"), 8, 33, probability_of_mutation=0.6)
    print("wrote traj_ga_n4.npz, traj_ga_n5.npz, traj_qeqea_n5_l64.npz")


if __name__ == "__main__":
    main()
