#!/bin/bash
# final measurement pass + cfg4/cfg3 query A/B
TAG=${TAG:-s3}
bash tools/r2_measure.sh
CFG=cfg4 STEPS=5 TAG=${TAG}c4 VARIANTS=hdda_skip tools/r2_ab.sh cache
CFG=cfg3 TAG=${TAG}c3 VARIANTS=hdda_skip tools/r2_ab.sh cache
