#!/bin/bash
for w in 2 3 4 6; do echo "== warm=$w"; IMB_WARM=$w python experiments/slabs.py; done
