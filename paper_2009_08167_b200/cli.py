"""Reference module name for the experiment driver (ref ``rigaeig/cli.py``): see ``report.py``."""
import sys

from .report import (ConfigError, ExperimentConfig, OutputBundle, PointResult, load_config, main,  # noqa: F401
                     run_experiment, run_point, write_bundle)

if __name__ == "__main__":
    sys.exit(main())
