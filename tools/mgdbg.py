"""development: run the multi-GPU orchestrator test worker and print every rank's result"""
import sys
sys.path.insert(0, ".")
if __name__ == "__main__":
    from tests.test_multigpu import _mg_worker, _spawn
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    for r in _spawn(_mg_worker, world, "gnoise", (24, 20, 16)):
        print(r[0], r[1])
        print(r[2][-3000:])
