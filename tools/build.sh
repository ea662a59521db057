#!/bin/bash
cd "$(dirname "$0")/.." && python -m paper_2509_20214_b200.build "$@"
