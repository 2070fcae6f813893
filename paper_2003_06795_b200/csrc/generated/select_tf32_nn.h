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
    if (k < INT64_C(1087)) {
        if (m < INT64_C(17740)) {
            if (n < INT64_C(222)) {
                if (k < INT64_C(136)) {
                    if (m < INT64_C(8870)) {
                        if (m < INT64_C(4435)) {
                            if (m < INT64_C(1109)) {
                                select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(2218)) {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(46)) {
                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(79)) {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(20)) {
                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(111)) {
                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(2218)) {
                        if (k < INT64_C(314)) {
                            if (k < INT64_C(167)) {
                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (n < INT64_C(46)) {
                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(222)) {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(1109)) {
                                if (k < INT64_C(744)) {
                                    if (m < INT64_C(139)) {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(111)) {
                                            if (k < INT64_C(471)) {
                                                if (m < INT64_C(278)) {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(555)) {
                                                        if (n < INT64_C(79)) {
                                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (m < INT64_C(555)) {
                                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(139)) {
                                        if (m < INT64_C(70)) {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(544)) {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(222)) {
                            if (n < INT64_C(46)) {
                                if (n < INT64_C(28)) {
                                    if (m < INT64_C(4435)) {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(8870)) {
                                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(4435)) {
                                        if (k < INT64_C(167)) {
                                            select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(4435)) {
                                if (k < INT64_C(444)) {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(544)) {
                                        select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (n < INT64_C(91)) {
                                    if (m < INT64_C(8870)) {
                                        if (k < INT64_C(384)) {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(384)) {
                                            select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(8870)) {
                                        if (k < INT64_C(363)) {
                                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
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
            } else {
                if (m < INT64_C(448)) {
                    if (k < INT64_C(992)) {
                        if (m < INT64_C(139)) {
                            if (m < INT64_C(70)) {
                                if (n < INT64_C(1620)) {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(1620)) {
                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(79)) {
                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(287)) {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(405)) {
                                        select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(573)) {
                                            if (m < INT64_C(278)) {
                                                if (k < INT64_C(702)) {
                                                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(702)) {
                                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            if (n < INT64_C(1025)) {
                                if (m < INT64_C(139)) {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(363)) {
                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(70)) {
                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(139)) {
                                        select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(2218)) {
                        if (k < INT64_C(405)) {
                            if (n < INT64_C(544)) {
                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(1109)) {
                                    select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(157)) {
                                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(363)) {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (n < INT64_C(512)) {
                                select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(28)) {
                if (k < INT64_C(56)) {
                    if (m < INT64_C(50176)) {
                        select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                    return out;
                }
            } else {
                if (k < INT64_C(384)) {
                    if (n < INT64_C(46)) {
                        if (m < INT64_C(35480)) {
                            select_tf32_nn_config out = {2u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(283839)) {
                        if (m < INT64_C(141920)) {
                            if (n < INT64_C(91)) {
                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                                return out;
                            }
                        } else {
                            select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                            return out;
                        }
                    } else {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (m < INT64_C(1792)) {
            if (n < INT64_C(2024)) {
                if (m < INT64_C(139)) {
                    if (k < INT64_C(2897)) {
                        if (m < INT64_C(40)) {
                            if (m < INT64_C(3)) {
                                if (m < INT64_C(2)) {
                                    select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(12)) {
                                    select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(1620)) {
                                        select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_nn_config out = {4u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(555)) {
                        if (n < INT64_C(363)) {
                            select_tf32_nn_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (n < INT64_C(363)) {
                            if (m < INT64_C(1109)) {
                                select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(1630)) {
                                    select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_nn_config out = {4u, 1u, 8u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_tf32_nn_config out = {4u, 1u, 8u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                select_tf32_nn_config out = {4u, 1u, 8u, 8u, 8u};
                return out;
            }
        } else {
            if (m < INT64_C(7168)) {
                if (n < INT64_C(363)) {
                    select_tf32_nn_config out = {4u, 1u, 8u, 8u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(3584)) {
                        if (m < INT64_C(3104)) {
                            select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                            return out;
                        } else {
                            select_tf32_nn_config out = {4u, 1u, 8u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(1630)) {
                    if (m < INT64_C(35480)) {
                        select_tf32_nn_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    select_tf32_nn_config out = {8u, 2u, 8u, 16u, 16u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_TF32_NN_H */
