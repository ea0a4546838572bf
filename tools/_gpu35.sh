#!/bin/bash
bash tools/_ab.sh r1ax base t768d2 t768d3 base
