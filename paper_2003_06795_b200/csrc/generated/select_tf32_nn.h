#ifndef SELECT_TF32_NN_H
#define SELECT_TF32_NN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_nn_config;

static inline select_tf32_nn_config select_tf32_nn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(3584)) {
        if (n < INT64_C(2897)) {
            if (n < INT64_C(111)) {
                if (m < INT64_C(2218)) {
                    if (n < INT64_C(46)) {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(272)) {
                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(555)) {
                                if (k < INT64_C(471)) {
                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(278)) {
                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(1109)) {
                                    if (n < INT64_C(79)) {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(471)) {
                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(46)) {
                        select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                        return out;
                    } else {
                        if (n < INT64_C(79)) {
                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(471)) {
                                select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(351)) {
                    if (m < INT64_C(2218)) {
                        if (m < INT64_C(159)) {
                            if (k < INT64_C(744)) {
                                if (m < INT64_C(70)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(112)) {
                                        select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(744)) {
                                if (m < INT64_C(317)) {
                                    if (m < INT64_C(224)) {
                                        if (k < INT64_C(544)) {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(144)) {
                                        if (m < INT64_C(1109)) {
                                            if (k < INT64_C(363)) {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(1630)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(1630)) {
                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(2218)) {
                        if (k < INT64_C(725)) {
                            if (m < INT64_C(139)) {
                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(1620)) {
                                    if (k < INT64_C(405)) {
                                        if (k < INT64_C(111)) {
                                            if (m < INT64_C(1109)) {
                                                if (k < INT64_C(79)) {
                                                    if (m < INT64_C(278)) {
                                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(79)) {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(278)) {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(1109)) {
                                                    if (k < INT64_C(144)) {
                                                        select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        if (m < INT64_C(555)) {
                                                            if (k < INT64_C(203)) {
                                                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            }
                                                        } else {
                                                            if (k < INT64_C(203)) {
                                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                if (k < INT64_C(287)) {
                                                                    select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                                                    return out;
                                                                } else {
                                                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                                    return out;
                                                                }
                                                            }
                                                        }
                                                    }
                                                } else {
                                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(2173)) {
                                if (m < INT64_C(6)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(29)) {
                                        if (m < INT64_C(12)) {
                                            if (k < INT64_C(1620)) {
                                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(896)) {
                                            if (n < INT64_C(1024)) {
                                                if (k < INT64_C(1449)) {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(99)) {
                                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (m < INT64_C(393)) {
                                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            } else {
                                                if (m < INT64_C(139)) {
                                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(278)) {
                                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (m < INT64_C(555)) {
                                                            select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            }
                                        } else {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(555)) {
                                    if (m < INT64_C(2)) {
                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(278)) {
                                            if (m < INT64_C(70)) {
                                                if (m < INT64_C(3)) {
                                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(8)) {
                                                        select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        if (m < INT64_C(29)) {
                                                            select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            } else {
                                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            }
        } else {
            select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
            return out;
        }
    } else {
        if (n < INT64_C(28)) {
            if (m < INT64_C(8870)) {
                if (k < INT64_C(118)) {
                    select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                    return out;
                } else {
                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                    return out;
                }
            } else {
                if (m < INT64_C(141920)) {
                    select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                }
            }
        } else {
            if (n < INT64_C(79)) {
                if (m < INT64_C(17740)) {
                    if (k < INT64_C(384)) {
                        if (k < INT64_C(146)) {
                            if (k < INT64_C(42)) {
                                select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(8870)) {
                                select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (n < INT64_C(46)) {
                                    select_tf32_nn_config out = {1u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(8870)) {
                            select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(141920)) {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (k < INT64_C(63)) {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(567677)) {
                                select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (k < INT64_C(46)) {
                    if (m < INT64_C(8870)) {
                        select_tf32_nn_config out = {4u, 1u, 2u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(544)) {
                        if (k < INT64_C(363)) {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(8870)) {
                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            }
        }
    }
}

#endif /* SELECT_TF32_NN_H */
